set -x
O=gpurun_out/r02k
mkdir -p $O
bash tools/ab_env.sh OHX_KF_KEEP 0 1 3 $O
for v in 0 1; do
OHX_KF_KEEP=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -c 20 --csv --log-file $O/launches_keep_$v.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-dists --no-parity --no-e2e > /dev/null 2>&1
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-parity > $O/bench_dists.json 2> $O/bench_dists.err
