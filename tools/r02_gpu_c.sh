# round 2, first GPU pass after the re-entry: smoke, GPU tests, both bench
# arms, launch list, drop-in suites, configs[4] parity, sanitizers
set -x
O=gpurun_out/r02c
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
free -g > $O/free.txt; nproc >> $O/free.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 1200 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-dists --no-parity --no-e2e > $O/ncu_bench.log 2>&1
timeout 1200 oracle/_ref/reftests/acceptance oracle/_ref/reftests/octohull_cli /tmp/acc1 > $O/acceptance.log 2>&1
echo "acceptance rc=$?" >> $O/acceptance.log
OHX_MG_VSHARDS=2 timeout 1200 oracle/_ref/reftests/acceptance oracle/_ref/reftests/octohull_cli /tmp/acc2 > $O/acceptance_mg.log 2>&1
echo "acceptance (mg, 2 shards) rc=$?" >> $O/acceptance_mg.log
timeout 2400 python tools/parity_c5.py --shards 2,4,8 > $O/parity_c5_4e9.json 2> $O/parity_c5.err
for tool in memcheck synccheck initcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > $O/san_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/san_rc.txt
done
