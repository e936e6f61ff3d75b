# four reads in flight in kf_gather and gather_arcs (cp.async.ca): tests, bench, launch lists
set -x
O=gpurun_out/s5l
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for v in 1 0; do
OHX_GATHER_LD=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-parity --no-e2e > $O/bench_async$v.json 2> $O/bench_async$v.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-dists --no-parity > $O/bench_under_ncu.log 2>&1
python tools/launch_summary.py $O/launches_bench.csv > $O/launches_bench.txt 2>&1
