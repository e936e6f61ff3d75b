# circle 1e8 hull stage: all four arcs in one arc-folded radix sort vs one sort per arc
set -x
O=gpurun_out/s5c
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hullchain.py -q -x > $O/pytest_hullchain.log 2>&1; echo "rc=$?" >> $O/pytest_hullchain.log
for v in perarc fold perarc fold; do
OHX_HULL_SORT=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-parity --no-e2e > $O/bench_$v.json 2> $O/bench_$v.err
done
OHX_TRACE=1 timeout 300 python tools/kernel_driver.py --dist circle --n 1e8 --reps 3 --pipeline > $O/trace_fold.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_circle.csv python tools/kernel_driver.py --pipeline --dist circle --n 1e8 --reps 1 > $O/ncu_circle.log 2>&1
python tools/launch_summary.py $O/launches_circle.csv > $O/launches_circle.txt 2>&1
