python __graft_entry__.py > /dev/null
timeout 900 python -m pytest -q -p no:cacheprovider -rf -x tests/test_gpu_gemm.py tests/test_gpu_train.py 2>&1 | tail -3
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
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:8]:
    print(f"{k:60s} n={c:5d} total={t:9.1f} us  avg={t/c:7.1f}")
PY
timeout 300 python -c "
import time, torch, sys; sys.argv=['x','64']
t0=time.time(); exec(open('tools/prof_train.py').read()); torch.cuda.synchronize(); print('train 1 epoch 2048 frames incl setup', time.time()-t0)"
