python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -q -p no:cacheprovider -rf -x tests/test_gpu_cnn.py -k "16 or multi_chunk" 2>&1 | tail -3
for a in "2 16 32" "4 16 32"; do timeout 300 python tools/prof_cnn.py $a 65536 5 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/train_launches.csv python tools/prof_train.py 64 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/train_launches.csv')))
i = [k for k, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[i]; ki, mi, ni = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Name')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[i + 1:]:
    if len(r) > mi and r[ni] == 'gpu__time_duration.sum':
        k = r[ki].split('(')[0][:60]
        agg[k][0] += 1; agg[k][1] += float(r[mi].replace(',', '')) / 1e3
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:15]:
    print(f"{k:60s} n={c:5d} total={t:9.1f} us  avg={t/c:7.1f}")
PY
