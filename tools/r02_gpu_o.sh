# KF with staged candidate coordinates + kf_compact: A/B against the
# index-only KF + kf_gather + K1 list (OHX_KF_XY=0), then the fused tests
set -x
O=gpurun_out/r02o
mkdir -p $O
for v in 1 0 1 0; do
OHX_KF_XY=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-dists --no-parity --no-e2e > $O/bench_xy$v.json 2> $O/bench_xy$v.err
done
OHX_TRACE=1 timeout 600 python tools/kernel_driver.py --dist normal --n 1e9 --reps 4 --pipeline > $O/trace.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-dists --no-parity --no-e2e > $O/ncu_bench.log 2>&1
python tools/launch_summary.py $O/launches.csv > $O/launches.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -k "fused or fusion or smoke or parity or sharded or mg" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
