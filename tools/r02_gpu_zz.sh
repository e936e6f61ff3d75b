# pipelined hull stage (arc by arc, each chain's D2H behind the next arc)
set -x
O=gpurun_out/r02zz
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hullchain.py -q -x -k "pipelined or rotated or pipeline" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
for v in 1 0; do
OHX_HULL_PIPE=$v OHX_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --no-e2e > $O/bench_pipe$v.json 2> $O/bench_pipe$v.err
done
