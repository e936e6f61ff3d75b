# the bench's N > 1 flow on one GPU: 2 ranks over gloo (sharded.py) and
# 2 virtual shards through the NCCL layer, 4e8 points of the configs[4] corpus
set -x
O=gpurun_out/r02ah
mkdir -p $O
OHX_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --points-total 4e8 > $O/bench_gloo2.json 2> $O/bench_gloo2.err
echo "rc=$?" >> $O/bench_gloo2.err
timeout 900 python bench.py --steps 3 --warmup 3 --points 4e8 --mg-vshards 2 --no-dists > $O/bench_mg2.json 2> $O/bench_mg2.err
echo "rc=$?" >> $O/bench_mg2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 --points-total 4e8 > $O/bench_ref2.json 2> $O/bench_ref2.err
echo "rc=$?" >> $O/bench_ref2.err
