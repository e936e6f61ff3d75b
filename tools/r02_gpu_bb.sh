# K2 hard points: find_queue first, then the quadrant arc's edges, the full
# octagon test only where they do not prove "outside" -- A/B per distribution
set -x
O=gpurun_out/r02bb
mkdir -p $O
for d in circle disk square normal; do
  OHX_FUSE=0 timeout 600 python tools/kernel_driver.py --dist $d --n 1e8 --reps 4 > $O/k2_$d.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_filter|k2_compact" -s 2 -c 2 -o $O/circle_k2 python tools/kernel_driver.py --dist circle --n 1e8 --reps 2 > $O/ncu.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
