set -x
timeout 900 python tools/evolve_timing.py 24 26 27 28 30
timeout 600 python tools/evolve_profile.py 26 2>&1 | head -60
