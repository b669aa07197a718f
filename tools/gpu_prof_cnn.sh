python __graft_entry__.py
python tools/prof_cnn.py 2 32 32 65536 3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cnn_launches.csv python tools/prof_cnn.py 2 32 32 65536 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/cnn_launches.csv')))
i=[k for k,r in enumerate(rows) if 'Kernel Name' in r][0]; h=rows[i]
ki,mi,ni=h.index('Kernel Name'),h.index('Metric Value'),h.index('Metric Name')
for r in rows[i+1:]:
    if len(r)>mi and r[ni]=='gpu__time_duration.sum': print(r[ki][:60], r[mi])
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv12 -c 1 -o gpurun_out/prof_fused python tools/prof_cnn.py 2 32 32 65536 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fc_kernel -c 1 -o gpurun_out/prof_fc python tools/prof_cnn.py 2 32 32 65536 1 > /dev/null 2>&1
ls -la gpurun_out
