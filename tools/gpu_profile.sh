#!/bin/bash
# The measurement recipe behind profiles/r02_* (run on a B200 through gpurun):
#   /usr/local/graft/bin/gpurun --timeout 3400 -- 'bash tools/gpu_profile.sh'
# 1. GPU parity suite, 2. cfg4 bench (the headline) and the other configs, 3. per-iteration
# launch lists (ncu needs plain graph nodes: MPK_NO_COND_GRAPH=1), 4. full captures of the
# row / pipeline kernels, exported as text on the box (.ncu-rep files of these kernels are
# 30-60 MB; gpurun_out/ is limited to 64 MiB).
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu -x --durations=8 > gpurun_out/gpu_suite.txt 2>&1; echo suite rc=$?
tail -n 3 gpurun_out/gpu_suite.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench rc=$?
for c in cfg1 cfg2 cfg3 cfg5; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-cold > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?
done
export MPK_NO_COND_GRAPH=1
M=gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --graph-profiling node -c 700 --csv --log-file gpurun_out/launches_cfg4.csv python tools/solve_probe.py cfg4 10 > gpurun_out/ncu_l4.log 2>&1; echo l4 rc=$?
timeout 900 ncu --metrics $M --clock-control none --graph-profiling node -c 1500 --csv --log-file gpurun_out/launches_cfg5_qd.csv python tools/solve_probe.py cfg5 25 cgs qd > gpurun_out/ncu_l5.log 2>&1; echo l5 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --graph-profiling node -k regex:'rows_kernel|pspmv_kernel' -s 5 -c 7 -o /tmp/cfg4_rows -f python tools/solve_probe.py cfg4 3 > gpurun_out/ncu_r4.log 2>&1; echo r4 rc=$?
ncu -i /tmp/cfg4_rows.ncu-rep --page details > gpurun_out/cfg4_rows_details.txt 2>/dev/null
ncu -i /tmp/cfg4_rows.ncu-rep --page raw --csv > gpurun_out/cfg4_rows_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/launches_cfg4.csv | head -n 30
