for v in x2_256 x2_512; do echo "C64_2Q=$v"; QSB_C64_2Q=$v timeout 600 python tools/workloads.py 30 > /tmp/w.txt 2>&1; grep -A1 "fused " /tmp/w.txt | grep -A1 f32 | head -2; done
