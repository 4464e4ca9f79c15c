mkdir -p gpurun_out
timeout 300 python tools/factor_time.py cfg1 cfg4 2>&1 | tail -n 2
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cold > gpurun_out/bench_cfg4_pipe2.json 2> gpurun_out/bench_cfg4_pipe2.err; echo pipe rc=$?; cut -c1-230 gpurun_out/bench_cfg4_pipe2.json
export MPK_NO_COND_GRAPH=1
M=gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --graph-profiling node -c 700 --csv --log-file gpurun_out/r02_launches_cfg4_pipe.csv python tools/solve_probe.py cfg4 10 > gpurun_out/ncu_l4.log 2>&1; echo l4 rc=$?
