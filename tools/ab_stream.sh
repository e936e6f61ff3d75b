timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for d in normal square; do timeout 120 python tools/kernel_driver.py --pipeline --dist $d --n 1e8 --reps 4 | tail -1; done
OHX_TRACE=1 timeout 300 python tools/kernel_driver.py --pipeline --dist normal --n 1e9 --reps 4 2>&1 | tail -7
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_list.csv python tools/kernel_driver.py --pipeline --n 1e9 --reps 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_list.csv
