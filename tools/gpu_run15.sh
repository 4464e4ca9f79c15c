mkdir -p gpurun_out
for ord in natural level; do for b in 1 2 4 6; do echo "== order $ord blocks/SM $b"; MPK_FACTOR_ORDER=$ord MPK_FACTOR_BLOCKS=$b timeout 300 python tools/factor_time.py cfg1 cfg2 cfg3 cfg4 cfg5 2>&1 | tail -n 5; done; done | tee gpurun_out/factor_order2.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ilu0_bitwise or singular or edge" 2>&1 | tail -n 4
MPK_FACTOR_ORDER=level MPK_FACTOR_BLOCKS=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "ilu0_bitwise or singular or edge or factors_apply" 2>&1 | tail -n 4
