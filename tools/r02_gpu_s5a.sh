# session-5 health check on a fresh box: GPU suite, smoke, default bench line
set -x
O=gpurun_out/s5a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
OHX_TRACE=2 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --no-e2e > $O/bench_trace.json 2> $O/bench_trace.err
