timeout 200 python tools/swf_check.py --env "MPK_SWEEP_PICK=swf" --env "MPK_SWEEP_PICK=swf SWF_FORCE_RERUN=1" --env "MPK_SWEEP_PICK=swf MPK_SSWEEP_W=1" cd9_97 cfg1 cd9_1000 cfg4
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "wavefront or sweep_paths" 2>&1 | tail -3
