for v in 0 1 0 1; do OHX_KF_V4=$v timeout 300 python tools/kernel_driver.py --pipeline --dist normal --n 1e9 --reps 6 2>&1 | tail -1 | sed "s/^/v4=$v /"; done
OHX_KF_V4=1 timeout 900 python -m pytest tests -m gpu -x -q -k "fused or force or u64 or sorted_input or degenerate_large" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
