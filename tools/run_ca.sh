python tools/numa_probe.py 2>&1 | tail -5
