# record all-gather inside the fused pass's round trip: tests, overhead A/B
set -x
O=gpurun_out/s5f
mkdir -p $O
timeout 900 python -m pytest tests/test_mg.py -q -x > $O/pytest_mg.log 2>&1; echo "rc=$?" >> $O/pytest_mg.log
timeout 600 python tools/mg_overhead.py 1e9 5e8 > $O/mg_overhead.log 2>&1
OHX_MG_MERGED=0 timeout 600 python tools/mg_overhead.py 5e8 > $O/mg_overhead_unmerged.log 2>&1
