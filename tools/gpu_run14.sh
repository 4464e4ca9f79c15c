mkdir -p gpurun_out
for ord in natural level; do for b in 1 2 6; do echo "== order $ord blocks/SM $b"; MPK_FACTOR_ORDER=$ord MPK_FACTOR_BLOCKS=$b timeout 300 python tools/factor_time.py cfg1 cfg2 cfg3 cfg4 cfg5 2>&1 | tail -n 5; done; done | tee gpurun_out/factor_order.txt
timeout 900 python -m pytest tests/test_gpu_mcmat.py tests/test_gpu_grid.py -q -x 2>&1 | tail -n 5
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sentinel or ilu0_bitwise or singular" 2>&1 | tail -n 8
