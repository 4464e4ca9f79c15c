timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -x -q -m gpu -s --durations=0 2>&1 | tail -40
