# evidence after the hull-stage sort tier and the ranged gather: full GPU
# tests, bench (distributions), circle hull-stage trace + launch list
set -x
O=gpurun_out/r02oo
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
OHX_TRACE=1 timeout 300 python tools/hull_output_probe.py --dist circle --n 1e8 --reps 2 > $O/probe_circle.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/launches_circle.csv python tools/kernel_driver.py --dist circle --n 1e8 --reps 2 --pipeline > $O/ncu_circle.log 2>&1
python tools/launch_summary.py $O/launches_circle.csv > $O/launches_circle.txt 2>&1
