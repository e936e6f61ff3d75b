# the multi-GPU layer with small survivor sets in one exchange block: tests + per-call overhead
set -x
O=gpurun_out/s5e
mkdir -p $O
timeout 900 python -m pytest tests/test_mg.py -q -x > $O/pytest_mg.log 2>&1; echo "rc=$?" >> $O/pytest_mg.log
timeout 600 python tools/mg_overhead.py 1e9 5e8 > $O/mg_overhead.log 2>&1
