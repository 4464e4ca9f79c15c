mkdir -p gpurun_out
timeout 300 python tools/factor_time.py cfg1 cfg2 cfg3 cfg4 cfg5 2>&1 | tail -n 5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_e.json 2> gpurun_out/bench_cfg4_e.err; echo bench rc=$?; cut -c1-230 gpurun_out/bench_cfg4_e.json
timeout 2700 python -m pytest tests -q -m gpu -x --durations=8 > gpurun_out/gpu_suite.txt 2>&1; echo suite rc=$?; tail -n 25 gpurun_out/gpu_suite.txt
