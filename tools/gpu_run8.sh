# round-2 re-entry: cfg4 bench, ncu of the sweep and SpMV kernels (cfg4 DD, cfg5 QD), launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench rc=$?
timeout 300 python tools/kprobe.py cfg4 2 3 > gpurun_out/kprobe_cfg4.txt 2>&1; echo kprobe rc=$?
timeout 300 python tools/kprobe.py cfg5 4 3 > gpurun_out/kprobe_cfg5.txt 2>&1; echo kprobe5 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'swf_kernel|rows_kernel|spmv' -c 6 -o gpurun_out/r02_cfg4_full -f python tools/kprobe.py cfg4 2 1 > gpurun_out/ncu_cfg4.log 2>&1; echo ncu4 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'sweep|rows_kernel|spmv' -c 6 -o gpurun_out/r02_cfg5_full -f python tools/kprobe.py cfg5 4 1 > gpurun_out/ncu_cfg5.log 2>&1; echo ncu5 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --steps 1 --warmup 3 --no-cold --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncul rc=$?
cat gpurun_out/kprobe_cfg4.txt gpurun_out/kprobe_cfg5.txt; cat gpurun_out/bench_cfg4.json | cut -c1-400
