# ncu --set full of the circle hull stage's own kernels (ranged gather,
# 32-bit keys, key-order gather, run fixing, chains) + the stage split
set -x
O=gpurun_out/r02ad
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather_xy4_ranged|linear_keys|gather_arcs|fix_runs|chain_local|chain_copy" -c 6 -o $O/circle_hull python tools/kernel_driver.py --dist circle --n 1e8 --reps 1 --pipeline > $O/ncu.log 2>&1
OHX_TRACE=2 timeout 300 python tools/kernel_driver.py --dist circle --n 1e8 --reps 3 --pipeline > $O/trace.log 2>&1
