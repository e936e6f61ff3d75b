# full GPU suite after the device-chain change; ncu of circle K1/K2 and the
# hull-stage kernels; acceptance through the mg layer; sanitizers
set -x
O=gpurun_out/r02g
mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
OHX_MG_VSHARDS=2 timeout 1200 oracle/_ref/reftests/acceptance oracle/_ref/reftests/octohull_cli /tmp/acc2 > $O/acceptance_mg.log 2>&1
echo "acceptance (mg, 2 shards) rc=$?" >> $O/acceptance_mg.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_extremes|k2_filter|k2_compact|k1b_corners" -s 3 -c 4 -o $O/circle_k -f python tools/kernel_driver.py --dist circle --n 1e8 --reps 2 > $O/ncu_circle_k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"chain_local|chain_replay|chain_copy|gather_sorted|repair_ties" -c 5 -o $O/circle_hull -f python tools/hull_output_probe.py --dist circle --n 1e8 --reps 1 > $O/ncu_circle_hull.log 2>&1
for tool in memcheck synccheck initcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > $O/san_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/san_rc.txt
done
