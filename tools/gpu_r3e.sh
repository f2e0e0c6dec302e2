QSB_X2_BIG=1 timeout 600 python tools/workloads.py 30 > /tmp/w.txt 2>&1; grep -A1 "grid" /tmp/w.txt
