set -x
timeout 900 python tools/evolve_timing.py 24 26 28 30
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py -x -q -p no:cacheprovider -k "evol or trotter or adiabatic" 2>&1 | tail -2
