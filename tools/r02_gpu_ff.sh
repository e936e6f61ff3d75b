set -x
O=gpurun_out/r02ff
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "forced_fusion" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
