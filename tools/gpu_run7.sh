# round-2 re-entry check: GPU suite, cfg4 bench, ncu of the sweep and SpMV kernels (cfg4 DD, cfg5 QD)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 2400 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/gpu_suite.txt 2>&1; echo suite rc=$?
tail -3 gpurun_out/gpu_suite.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench rc=$?
timeout 300 python tools/kprobe.py cfg4 2 3 > gpurun_out/kprobe_cfg4.txt 2>&1; echo kprobe rc=$?
timeout 300 python tools/kprobe.py cfg5 4 3 > gpurun_out/kprobe_cfg5.txt 2>&1; echo kprobe5 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'swf_kernel|rows_kernel' -c 3 -o gpurun_out/r02_cfg4_full -f python tools/kprobe.py cfg4 2 1 > gpurun_out/ncu_cfg4.log 2>&1; echo ncu4 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'sweep|rows_kernel' -c 4 -o gpurun_out/r02_cfg5_full -f python tools/kprobe.py cfg5 4 1 > gpurun_out/ncu_cfg5.log 2>&1; echo ncu5 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --steps 1 --warmup 3 --no-cold --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncul rc=$?
