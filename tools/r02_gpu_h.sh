# K2 rework (edge reads amortised over 4 staged points, warp-per-run
# compaction copy) + device-resident hull output: GPU suite, circle K2
# timing and ncu, hull stage with the hull left on the device
set -x
O=gpurun_out/r02h
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
for d in circle disk square normal; do timeout 300 python tools/kernel_driver.py --dist $d --n 1e8 --reps 3 >> $O/k2_times.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_filter|k2_compact" -s 2 -c 2 -o $O/circle_k2 -f python tools/kernel_driver.py --dist circle --n 1e8 --reps 2 > $O/ncu_circle_k2.log 2>&1
OHX_TRACE=1 timeout 600 python tools/hull_output_probe.py --dist circle --n 1e8 --reps 2 > $O/probe_circle.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
