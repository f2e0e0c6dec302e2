QSB_2Q_GEOMETRY=x2s16 timeout 120 python tools/pp_check.py 22
QSB_2Q_GEOMETRY=x2s16 timeout 600 python tools/workloads.py 30 > /tmp/w.txt 2>&1; grep -A1 "fused\|trotter\|grid" /tmp/w.txt | grep -v f32
