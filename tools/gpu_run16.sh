mkdir -p gpurun_out
for b in 1 2 4; do echo "== padded level order, blocks/SM $b"; MPK_FACTOR_BLOCKS=$b timeout 300 python tools/factor_time.py cfg1 cfg2 cfg3 cfg4 cfg5 2>&1 | tail -n 5; done | tee gpurun_out/factor_order3.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "ilu0_bitwise or singular or edge or factors_apply or wavefront_sweep" 2>&1 | tail -n 4
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_d.json 2> gpurun_out/bench_cfg4_d.err; echo bench rc=$?; cut -c1-330 gpurun_out/bench_cfg4_d.json
