timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "wavefront or sweep_paths" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "cfg4_rhs or cfg4_bicgstab_20_tree or cfg4_bicgstab_200" 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo rc=$?
