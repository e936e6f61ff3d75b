# ncu --set full of the fused filter pass (kf_filter) at N=1e9
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"kf_filter" -c 1 -o gpurun_out/kf_filter -f python tools/kernel_driver.py --pipeline --n ${N:-1e9} --reps 1 > gpurun_out/ncu1.log 2>&1
