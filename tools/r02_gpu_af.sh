set -x
O=gpurun_out/r02af
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hullchain.py -q -x -k "pipelined" > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
