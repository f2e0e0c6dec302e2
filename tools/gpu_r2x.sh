QSB_PINGPONG=1 timeout 120 python tools/pp_check.py 22
QSB_PINGPONG=1 timeout 200 python tools/pp_check.py 30
for pp in 0 1; do echo "PINGPONG=$pp"; QSB_PINGPONG=$pp timeout 600 python tools/workloads.py 30 > /tmp/w.txt 2>&1; grep -A1 "fused\|trotter\|grid" /tmp/w.txt | grep -v f32 | head -8; done
