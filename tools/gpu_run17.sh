mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pipelined" 2>&1 | tail -n 15
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "cfg4 and not twin" 2>&1 | tail -n 6
MPK_PIPE=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cold > gpurun_out/bench_cfg4_nopipe.json 2> gpurun_out/bench_cfg4_nopipe.err; echo nopipe rc=$?; cut -c1-230 gpurun_out/bench_cfg4_nopipe.json
MPK_VERBOSE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_pipe.json 2> gpurun_out/bench_cfg4_pipe.err; echo pipe rc=$?; cut -c1-230 gpurun_out/bench_cfg4_pipe.json; grep "pipelined" gpurun_out/bench_cfg4_pipe.err | tail -n 2
timeout 300 python tools/factor_time.py cfg1 cfg4 2>&1 | tail -n 2
