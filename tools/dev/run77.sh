#!/bin/bash
# c4a (2^28-bit operands, the metric's other size): ncu launch list of two multiplies, then a full capture of the second
mkdir -p gpurun_out
python tools/dev/prof_run.py c4a 2 > gpurun_out/t77_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/t77_plain.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/t77_c4a_launches_all.csv python tools/dev/prof_run.py c4a 2 > gpurun_out/t77_ncu1.log 2>&1
L=$(python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/t77_c4a_launches_all.csv')))
hdr=None; ids=[]
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d['ID'] not in ids: ids.append(d['ID'])
print(len(ids)//2)
PY
)
echo "launches per multiply: $L" > gpurun_out/t77_L.txt
timeout 1200 ncu --set full --clock-control none -s $L -c $L -o gpurun_out/t77_c4a_full -f python tools/dev/prof_run.py c4a 2 > gpurun_out/t77_ncu2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/t77_ncu2.log
ncu -i gpurun_out/t77_c4a_full.ncu-rep --page raw --csv > gpurun_out/t77_c4a_full_raw.csv 2>> gpurun_out/t77_ncu2.log
rm -f gpurun_out/t77_c4a_full.ncu-rep
