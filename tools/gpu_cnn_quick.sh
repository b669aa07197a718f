python __graft_entry__.py
timeout 600 python -m pytest tests/test_gpu_cnn.py tests/test_gpu_cascade.py -q --timeout 120 -p no:cacheprovider -rf -x 2>&1 | tail -5
python tools/prof_cnn.py 2 32 32 65536 3
python tools/prof_cnn.py 4 32 32 65536 3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cnn_launches.csv python tools/prof_cnn.py 2 32 32 65536 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/cnn_launches.csv')))
i=[k for k,r in enumerate(rows) if 'Kernel Name' in r][0]; h=rows[i]
ki,mi,ni=h.index('Kernel Name'),h.index('Metric Value'),h.index('Metric Name')
for r in rows[i+1:][:6]:
    if len(r)>mi and r[ni]=='gpu__time_duration.sum': print(r[ki][:60], r[mi])
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv12 -c 1 -o gpurun_out/prof_fused2 python tools/prof_cnn.py 2 32 32 65536 1 > /dev/null 2>&1
