# host gap after the wrapper change + the full GPU suite
set -x
O=gpurun_out/r02aj
mkdir -p $O
PYTHONPATH=. timeout 600 python tools/gap_probe.py 1e9 100 > $O/gap.log 2>&1
echo "rc=$?" >> $O/gap.log
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
echo "rc=$?" >> $O/pytest_gpu.log
