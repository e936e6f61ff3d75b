# gather_arcs load cache operator A/B (circle 1e8): DRAM bytes and time per mode
set -x
O=gpurun_out/s5j
mkdir -p $O
for m in 0 1 2 3; do
OHX_GATHER_LD=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:gather_arcs --csv --log-file $O/ld$m.csv python tools/kernel_driver.py --pipeline --dist circle --n 1e8 --reps 1 > $O/ncu_ld$m.log 2>&1
OHX_GATHER_LD=$m OHX_TRACE=1 timeout 600 python tools/kernel_driver.py --pipeline --dist circle --n 1e8 --reps 3 > $O/trace_ld$m.log 2>&1
done
