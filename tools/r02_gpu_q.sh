# one-pass K2 over the candidates (A/B OHX_K2_ONEPASS), split count_in_region,
# pinned sample records; fused-path GPU tests
set -x
O=gpurun_out/r02q
mkdir -p $O
for v in 1 0 1 0; do
OHX_K2_ONEPASS=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-dists --no-parity --no-e2e > $O/bench_op$v.json 2> $O/bench_op$v.err
done
for v in 1 0; do
OHX_K2_ONEPASS=$v timeout 600 python tools/kernel_driver.py --dist square --n 1e8 --reps 6 --pipeline > $O/square_op$v.log 2>&1
done
OHX_TRACE=1 timeout 600 python tools/kernel_driver.py --dist normal --n 1e9 --reps 4 --pipeline > $O/trace.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-dists --no-parity --no-e2e > $O/ncu_bench.log 2>&1
python tools/launch_summary.py $O/launches.csv > $O/launches.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -k "fused or fusion or smoke or parity or sharded or mg or sample" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
