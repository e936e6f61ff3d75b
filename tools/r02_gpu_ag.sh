# chain_local with a shared-memory stack ring
set -x
O=gpurun_out/r02ag
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hullchain.py tests/test_gpu_parity.py -q -x -k "hull or sort or degenerate or circle" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/launches_circle.csv python tools/kernel_driver.py --dist circle --n 1e8 --reps 2 --pipeline > $O/ncu_circle.log 2>&1
python tools/launch_summary.py $O/launches_circle.csv > $O/launches_circle.txt 2>&1
OHX_TRACE=1 timeout 300 python tools/hull_output_probe.py --dist circle --n 1e8 --reps 2 > $O/probe_circle.log 2>&1
