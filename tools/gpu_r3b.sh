mkdir -p /tmp/rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 10 -c 4 -o /tmp/rep/var30c64 python tools/ncu_workload.py variational 30 f32 > /tmp/rep/l1 2>&1; echo "ncu rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 10 -c 4 -o /tmp/rep/var30c128 python tools/ncu_workload.py variational 30 f64 > /tmp/rep/l2 2>&1; echo "ncu rc $?"
timeout 900 ncu --set full --clock-control none -k regex:"k_" -s 40 -c 40 -o /tmp/rep/sample python tools/ncu_sample.py 30 > /tmp/rep/l3 2>&1; echo "ncu rc $?"
for r in var30c64 var30c128; do
  python tools/ncu_summary.py /tmp/rep/$r.ncu-rep > gpurun_out/r3b_$r.txt 2>&1
  for k in $(ncu -i /tmp/rep/$r.ncu-rep --page raw --csv 2>/dev/null | python -c "import csv,sys; rows=list(csv.reader(sys.stdin)); c=rows[0].index('Kernel Name'); print(' '.join(r[c][9:21] for r in rows[2:]))"); do
    echo "== $k" >> gpurun_out/r3b_$r.txt; python tools/ncu_opmix.py /tmp/rep/$r.ncu-rep $k 12 >> gpurun_out/r3b_$r.txt 2>&1
    python tools/ncu_hotspots.py /tmp/rep/$r.ncu-rep $k stall_long_sb 4 >> gpurun_out/r3b_$r.txt 2>&1
  done
done
ncu -i /tmp/rep/sample.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/r3b_sample.csv 2>&1
ls -la gpurun_out
