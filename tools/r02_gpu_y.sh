# host timeline of the fused step (OHX_TRACE=2) at 1e9 and on the square
set -x
O=gpurun_out/r02y
mkdir -p $O
OHX_TRACE=2 timeout 600 python tools/kernel_driver.py --dist normal --n 1e9 --reps 5 --pipeline > $O/trace_normal.log 2>&1
OHX_TRACE=2 timeout 600 python tools/kernel_driver.py --dist square --n 1e8 --reps 5 --pipeline > $O/trace_square.log 2>&1
