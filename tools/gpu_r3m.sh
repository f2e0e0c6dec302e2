timeout 2400 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -4
timeout 600 python tools/evolve_timing.py 22 26 28 30
timeout 600 python tools/evolve_window_probe.py 26 2>&1 | grep "^n="
