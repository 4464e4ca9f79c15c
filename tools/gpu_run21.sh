timeout 600 python tools/pipe_probe.py cfg4 20 2>&1 | tail -n 4
