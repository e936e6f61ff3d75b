# the reference's acceptance harness against the final library, plain and through the NCCL layer
set -x
O=gpurun_out/s5n
mkdir -p $O
ldd oracle/_ref/reftests/acceptance | grep -i octo > $O/ldd.txt 2>&1
timeout 1200 oracle/_ref/reftests/acceptance oracle/_ref/reftests/octohull_cli /tmp/acc1 > $O/acceptance.log 2>&1
echo "acceptance rc=$?" >> $O/acceptance.log
OHX_MG_VSHARDS=2 timeout 1200 oracle/_ref/reftests/acceptance oracle/_ref/reftests/octohull_cli /tmp/acc2 > $O/acceptance_mg.log 2>&1
echo "acceptance (mg, 2 shards) rc=$?" >> $O/acceptance_mg.log
