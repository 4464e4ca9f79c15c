mkdir -p gpurun_out
for pub in 0 1; do for b in 1 2; do echo "== MPK_FACTOR_PUB=$pub blocks/SM(level) $b"; MPK_FACTOR_PUB=$pub MPK_FACTOR_BLOCKS=$b timeout 300 python tools/factor_time.py cfg1 cfg2 cfg4 cfg5 2>&1 | tail -n 4; done; done
echo "== defaults"; timeout 300 python tools/factor_time.py cfg1 cfg2 cfg3 cfg4 cfg5 2>&1 | tail -n 5
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "ilu0_bitwise or singular or edge or factors_apply or sweep_paths or repeated" 2>&1 | tail -n 4
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cold 2>/dev/null | cut -c1-200
