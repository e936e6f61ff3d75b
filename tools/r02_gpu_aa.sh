# chain_local with an 8-deep prefetch ring: circle hull stage + chain tests
set -x
O=gpurun_out/r02aa
mkdir -p $O
OHX_TRACE=1 timeout 600 python tools/hull_output_probe.py --dist circle --n 1e8 --reps 2 > $O/probe_circle.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/launches_circle.csv python tools/kernel_driver.py --dist circle --n 1e8 --reps 1 --pipeline > $O/ncu_circle.log 2>&1
python tools/launch_summary.py $O/launches_circle.csv > $O/launches_circle.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_hullchain.py -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
