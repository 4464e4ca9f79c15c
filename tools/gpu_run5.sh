nproc
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo rc=$?
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_cfg4.json 2> gpurun_out/bench_ref_cfg4.err; echo rc=$?
