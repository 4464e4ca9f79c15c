mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pipelined or wavefront" 2>&1 | tail -n 4
MPK_VERBOSE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_f.json 2> gpurun_out/bench_cfg4_f.err; echo bench rc=$?; cut -c1-230 gpurun_out/bench_cfg4_f.json; grep "mpk\] upload" gpurun_out/bench_cfg4_f.err | tail -n 4
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg4_f.json')); print(d['cold_time_to_solve_s'])"
