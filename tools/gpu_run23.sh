mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sparse_kernels or solver_small or cfg2 or cfg1 or pipelined or cfg5" 2>&1 | tail -n 4
for c in cfg4 cfg5 cfg2 cfg1; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-cold > gpurun_out/bench_b_$c.json 2> gpurun_out/bench_b_$c.err; echo $c rc=$?; python -c "
import json,sys; d=json.load(open('gpurun_out/bench_b_$c.json')); print(round(d['value'],1),'it/s', round(d['ms_per_step'],2),'ms; spmv', round(d['roofline_spmv']['avg_ms'],4),'ms frac',round(d['roofline_spmv']['frac'],3))"; done
