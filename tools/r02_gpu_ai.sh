# host gap between back-to-back device calls (normal 1e9)
set -x
O=gpurun_out/r02ai
mkdir -p $O
PYTHONPATH=. timeout 600 python tools/gap_probe.py 1e9 100 > $O/gap.log 2>&1
echo "rc=$?" >> $O/gap.log
PYTHONPATH=. OHX_TRACE=2 timeout 300 python tools/gap_probe.py 1e9 3 > $O/gap_trace.log 2>&1
