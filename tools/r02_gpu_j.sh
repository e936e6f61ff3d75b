set -x
O=gpurun_out/r02j
mkdir -p $O
timeout 900 python -m pytest tests/test_sharded_gloo.py tests/test_gpu_hullchain.py -m gpu -q > $O/pytest.log 2>&1
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
