# Round evidence on one B200: bench line, launch list of the same command,
# ncu --set full of the dominant kernel, reference arm.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kf_filter" -s 1 -c 1 -o gpurun_out/kf_filter_full -f python tools/kernel_driver.py --pipeline --n 1e9 --reps 2 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_extremes|k2_filter" -s 2 -c 2 -o gpurun_out/twopass_full -f python tools/kernel_driver.py --n 1e9 --reps 2 > gpurun_out/ncu_full2.log 2>&1
# every BASELINE config (device, host API, reference CPU) and the parity sweeps
timeout 1500 python tools/configs_bench.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
timeout 2400 python tools/sweep_full.py 10 > gpurun_out/sweep_full.log 2>&1
timeout 900 python tools/fuse_sweep.py > gpurun_out/fuse_sweep.log 2>&1
