timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "sample or cumsum or digest or shots or marginal" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_sharding.py -x -q -p no:cacheprovider -k "sample" 2>&1 | tail -2
for v in 0 1; do QSB_SPARSE_CDF=$v timeout 600 python tools/workloads.py 30 > /tmp/w.txt 2>&1; echo "SPARSE=$v"; grep "sample" /tmp/w.txt; done
