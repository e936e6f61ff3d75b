# square 1e8 step anatomy (trace + launch list) and the sample kernel's ncu
set -x
O=gpurun_out/r02n
mkdir -p $O
OHX_TRACE=1 timeout 600 python tools/kernel_driver.py --dist square --n 1e8 --reps 4 --pipeline > $O/square_trace.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/launches_square.csv python tools/kernel_driver.py --dist square --n 1e8 --reps 3 --pipeline > $O/ncu_square.log 2>&1
python tools/launch_summary.py $O/launches_square.csv > $O/launches_square.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_small|count_in_region|kf_gather|k2_" -s 6 -c 6 -o $O/normal_small python tools/kernel_driver.py --dist normal --n 1e9 --reps 3 --pipeline > $O/ncu_small.log 2>&1
