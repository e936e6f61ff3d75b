# cycle statistics fused with chain_copy (circle hull stage): tests, A/B, launch list
set -x
O=gpurun_out/s5h
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hullchain.py -q -x > $O/pytest_hullchain.log 2>&1; echo "rc=$?" >> $O/pytest_hullchain.log
OHX_CYCLE_STATS=reduce timeout 900 python -m pytest tests/test_gpu_hullchain.py -q -x > $O/pytest_hullchain_reduce.log 2>&1; echo "rc=$?" >> $O/pytest_hullchain_reduce.log
for v in reduce fused reduce fused; do
OHX_CYCLE_STATS=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-parity --no-e2e > $O/bench_$v.json 2> $O/bench_$v.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_circle.csv python tools/kernel_driver.py --pipeline --dist circle --n 1e8 --reps 1 > $O/ncu_circle.log 2>&1
python tools/launch_summary.py $O/launches_circle.csv > $O/launches_circle.txt 2>&1
