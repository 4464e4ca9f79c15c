mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_c.json 2> gpurun_out/bench_cfg4_c.err; echo bench rc=$?; cut -c1-330 gpurun_out/bench_cfg4_c.json
timeout 2400 python -m pytest tests -q -m gpu -x --durations=8 > gpurun_out/gpu_suite.txt 2>&1; echo suite rc=$?; tail -n 45 gpurun_out/gpu_suite.txt
for c in cfg5 cfg2 cfg1 cfg3; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-cold > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?; cut -c1-260 gpurun_out/bench_$c.json; done
