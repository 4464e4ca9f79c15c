mkdir -p gpurun_out
for lib in libmpkb200.so libmpkb200_qd2.so; do for c in "cfg5" "cfg5 --cfg5-weak" "cfg2"; do echo "== $lib $c"; MPK_B200_LIB=$PWD/paper_2504_14498_b200/_lib/$lib timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-cold 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1),'it/s', round(d['ms_per_step'],2),'ms')"; done; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cold 2>/dev/null | cut -c1-200
