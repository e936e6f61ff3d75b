set -x
O=gpurun_out/r02v
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bs_" -c 6 -o $O/bs python tools/kernel_driver.py --dist circle --n 1e8 --reps 1 --pipeline > $O/ncu.log 2>&1
