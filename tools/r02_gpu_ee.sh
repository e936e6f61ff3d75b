# pinned survivor fetch for the host hull: square timeline + hull tests
set -x
O=gpurun_out/r02ee
mkdir -p $O
OHX_TRACE=2 timeout 300 python tools/kernel_driver.py --dist square --n 1e8 --reps 5 --pipeline > $O/trace_square.log 2>&1
timeout 300 python tools/kernel_driver.py --dist square --n 1e8 --reps 8 --pipeline > $O/square.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "hull or fused or mg or sharded or smoke or queue or parity" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
