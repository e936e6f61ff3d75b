# square 1e8 (configs[1]): host timeline and launch list of the fused call
set -x
O=gpurun_out/s5b
mkdir -p $O
OHX_TRACE=2 timeout 600 python tools/kernel_driver.py --pipeline --dist square --n 1e8 --reps 6 > $O/trace_square.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_square.csv python tools/kernel_driver.py --pipeline --dist square --n 1e8 --reps 3 > $O/ncu_square.log 2>&1
python tools/launch_summary.py $O/launches_square.csv > $O/launches_square.txt 2>&1
