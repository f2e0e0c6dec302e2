timeout 600 python tools/variant_sweep.py variational 2>&1 | tail -3
DT=c64 timeout 300 python tools/variant_sweep.py variational 2>&1 | tail -14
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider -k "c64 or complex64 or F32 or f32 or variational" 2>&1 | tail -2
