# the native multi-GPU layer's overhead on one GPU: 1e9 as 1 shard (single
# path) vs 2 / 4 virtual shards through ohx_mg (NCCL 1-rank world)
set -x
O=gpurun_out/r02yy
mkdir -p $O
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-dists --no-parity --no-e2e > $O/single.json 2> $O/single.err
for k in 2 4; do
OHX_TRACE=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-dists --no-parity --no-e2e --mg-vshards $k > $O/mg$k.json 2> $O/mg$k.err
done
