mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mcmat.py -q -x -k in_place 2>&1 | tail -n 40
MPK_VERBOSE=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_b.json 2> gpurun_out/bench_cfg4_b.err; echo bench rc=$?
export MPK_NO_COND_GRAPH=1
M=gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --graph-profiling node -c 600 --csv --log-file gpurun_out/r02_launches_cfg4_iter.csv python tools/solve_probe.py cfg4 10 > gpurun_out/ncu_l4.log 2>&1; echo l4 rc=$?
timeout 900 ncu --metrics $M --clock-control none --graph-profiling node -c 1500 --csv --log-file gpurun_out/r02_launches_cfg5_qd.csv python tools/solve_probe.py cfg5 25 cgs qd > gpurun_out/ncu_l5.log 2>&1; echo l5 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --graph-profiling node -k regex:rows_kernel -s 5 -c 5 -o /tmp/r02_cfg4_rows -f python tools/solve_probe.py cfg4 3 > gpurun_out/ncu_r4.log 2>&1; echo r4 rc=$?
ncu -i /tmp/r02_cfg4_rows.ncu-rep --page raw --csv > gpurun_out/r02_cfg4_rows_raw.csv 2>/dev/null
ncu -i /tmp/r02_cfg4_rows.ncu-rep --page details > gpurun_out/r02_cfg4_rows_details.txt 2>/dev/null
ncu -i /tmp/r02_cfg4_rows.ncu-rep --page source --csv > gpurun_out/r02_cfg4_rows_source.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --graph-profiling node -k regex:'rows_kernel|fin_kernel' -s 8 -c 8 -o /tmp/r02_cfg5_rows -f python tools/solve_probe.py cfg5 3 cgs qd > gpurun_out/ncu_r5.log 2>&1; echo r5 rc=$?
ncu -i /tmp/r02_cfg5_rows.ncu-rep --page raw --csv > gpurun_out/r02_cfg5_rows_raw.csv 2>/dev/null
ncu -i /tmp/r02_cfg5_rows.ncu-rep --page details > gpurun_out/r02_cfg5_rows_details.txt 2>/dev/null
ls -la /tmp/*.ncu-rep; gzip -9 gpurun_out/r02_cfg4_rows_source.csv; du -sh gpurun_out; ls -la gpurun_out
