# step trace; L2 fetch granularity probe (bench + hull stage)
set -x
O=gpurun_out/r02f
mkdir -p $O
OHX_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-dists --no-parity --no-e2e > $O/bench_trace.json 2> $O/bench_trace.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-dists --no-parity --no-e2e > $O/bench_l2def.json 2> $O/bench_l2def.err
for v in 32 64; do
OHX_L2_FETCH=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-dists --no-parity --no-e2e > $O/bench_l2_$v.json 2> $O/bench_l2_$v.err
OHX_L2_FETCH=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 20 --csv --log-file $O/launches_l2_$v.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-dists --no-parity --no-e2e > /dev/null 2>&1
OHX_L2_FETCH=$v OHX_TRACE=1 timeout 600 python tools/hull_output_probe.py --dist circle --n 1e8 --reps 1 > $O/probe_circle_l2_$v.log 2>&1
done
