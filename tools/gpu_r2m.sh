set -x
QSB_2Q_GEOMETRY=s3 timeout 600 python tools/workloads.py 30 2>&1 | head -10
QSB_2Q_GEOMETRY=s3 timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py -x -q -p no:cacheprovider 2>&1 | tail -3
