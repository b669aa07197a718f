"""Time-weighted ncu tensor-pipe activity per CNN arch from tools/gpu_cnn_tensor.sh CSVs
(the weight-packing and rendering launches are excluded).
usage: python tools/tensor_weighted.py gpurun_out/tensor_*.csv"""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[i]
    ki, ii, mi, ni = h.index('Kernel Name'), h.index('ID'), h.index('Metric Value'), h.index('Metric Name')
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[i + 1:]:
        if len(r) <= mi:
            continue
        names[r[ii]] = r[ki].split('(')[0]
        try:
            per[r[ii]][r[ni]] = float(r[mi].replace(',', ''))
        except ValueError:
            per[r[ii]][r[ni]] = 0.0
    t_all = tp = mt = 0.0
    parts = []
    for lid, m in per.items():
        nm = names[lid]
        if any(x in nm for x in ('pack', 'render', 'bg_kernel', 'distribution', 'elementwise')):
            continue
        t = m.get('gpu__time_duration.sum', 0.0)
        a = m.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0.0)
        b = m.get('sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0.0)
        t_all += t
        tp += t * a
        mt += t * b
        parts.append(f"{nm.split('::')[-1][:28]} {t / 1e3:.0f}us {a:.0f}%")
    arch = path.split('tensor_')[-1].replace('.csv', '')
    print(f"{arch:10s} kernels {t_all / 1e3:8.0f} us  tensor-pipe active (time-weighted) {tp / t_all:5.1f} %  "
          f"smem->tensor {mt / t_all:5.1f} %   | " + ", ".join(parts))
