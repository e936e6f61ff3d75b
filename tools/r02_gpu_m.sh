# round 2 re-entry (session 3): re-verify HEAD on a fresh box -- smoke, GPU
# tests, both bench arms, a traced step breakdown
set -x
O=gpurun_out/r02m
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 1200 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
OHX_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-dists --no-parity --no-e2e > $O/trace.json 2> $O/trace.err
