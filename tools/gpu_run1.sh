set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "wavefront or sweep_paths" 2>&1 | tail -15
timeout 900 python tools/swf_check.py --env "MPK_VERBOSE=1" --env "MPK_SWEEP_PICK=swf MPK_VERBOSE=1" --env "MPK_SWEEP_PICK=wf" cd9_97 cfg1 cd9_1000 cfg4 2>&1 | tail -20
