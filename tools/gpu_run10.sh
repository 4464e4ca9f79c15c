mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mcmat.py -q -x > gpurun_out/t_mcmat.txt 2>&1; echo mcmat rc=$?; tail -n 15 gpurun_out/t_mcmat.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "none_and_spmv_full or precond" > gpurun_out/t_full.txt 2>&1; echo full rc=$?; tail -n 5 gpurun_out/t_full.txt
MPK_VERBOSE=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_b.json 2> gpurun_out/bench_cfg4_b.err; echo bench rc=$?; grep "mpk" gpurun_out/bench_cfg4_b.err | tail -n 12; cut -c1-300 gpurun_out/bench_cfg4_b.json
bash tools/gpu_run9.sh
