# the native multi-GPU layer's own per-call overhead on one GPU (1-rank NCCL world)
set -x
O=gpurun_out/s5d
mkdir -p $O
OHX_TRACE=1 timeout 600 python tools/mg_overhead.py 1e9 5e8 > $O/mg_overhead_trace.log 2>&1
timeout 600 python tools/mg_overhead.py 1e9 5e8 > $O/mg_overhead.log 2>&1
