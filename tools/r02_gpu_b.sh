# round 2, second GPU pass: the native multi-GPU layer, drop-in suites,
# acceptance (plain and through the mg layer), configs[4] parity on one GPU
set -x
O=gpurun_out/r02b
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 1200 oracle/_ref/reftests/acceptance oracle/_ref/reftests/octohull_cli /tmp/acc1 > $O/acceptance.log 2>&1
echo "acceptance rc=$?" >> $O/acceptance.log
OHX_MG_VSHARDS=2 timeout 1200 oracle/_ref/reftests/acceptance oracle/_ref/reftests/octohull_cli /tmp/acc2 > $O/acceptance_mg.log 2>&1
echo "acceptance (mg, 2 shards) rc=$?" >> $O/acceptance_mg.log
timeout 2400 python tools/parity_c5.py --shards 2,4,8 > $O/parity_c5_4e9.json 2> $O/parity_c5.err
