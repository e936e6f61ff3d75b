timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for d in normal square disk; do OHX_FUSE=0 timeout 120 python tools/kernel_driver.py --dist $d --n 1e8 --reps 3 | tail -1; done
OHX_FUSE=0 timeout 300 python tools/kernel_driver.py --dist normal --n 1e9 --reps 3 | tail -1
