# after the multi-GPU exchange block: full GPU suite, the bench's N > 1 flows on one GPU, overhead
set -x
O=gpurun_out/s5g
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --points 4e8 --mg-vshards 2 --no-dists > $O/bench_mg2.json 2> $O/bench_mg2.err
echo "rc=$?" >> $O/bench_mg2.err
timeout 900 python bench.py --steps 5 --warmup 3 --points 5e8 --mg-vshards 1 --no-dists --no-cpu > $O/bench_mg1_5e8.json 2> $O/bench_mg1_5e8.err
echo "rc=$?" >> $O/bench_mg1_5e8.err
timeout 600 python tools/mg_overhead.py 5e8 > $O/mg_overhead.log 2>&1
