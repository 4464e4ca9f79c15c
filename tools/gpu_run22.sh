mkdir -p gpurun_out
for c in cfg5 cfg2 cfg1 cfg3; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-cold > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?; cut -c1-200 gpurun_out/bench_$c.json; done
timeout 600 python bench.py --config cfg5 --cfg5-weak --steps 3 --warmup 3 --no-cpu-baseline --no-cold > gpurun_out/bench_cfg5_weak.json 2> gpurun_out/bench_cfg5_weak.err; echo cfg5w rc=$?; cut -c1-200 gpurun_out/bench_cfg5_weak.json
export MPK_NO_COND_GRAPH=1
timeout 900 ncu --set full --clock-control none --import-source on --graph-profiling node -k regex:'pspmv_kernel' -s 2 -c 2 -o /tmp/r02_cfg4_pspmv -f python tools/solve_probe.py cfg4 3 > gpurun_out/ncu_p4.log 2>&1; echo p4 rc=$?
ncu -i /tmp/r02_cfg4_pspmv.ncu-rep --page details > gpurun_out/r02_cfg4_pspmv_details.txt 2>/dev/null
ncu -i /tmp/r02_cfg4_pspmv.ncu-rep --page raw --csv > gpurun_out/r02_cfg4_pspmv_raw.csv 2>/dev/null
ls -la /tmp/r02_cfg4_pspmv.ncu-rep; cp /tmp/r02_cfg4_pspmv.ncu-rep gpurun_out/ 2>/dev/null; du -sh gpurun_out
