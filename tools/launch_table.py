"""Per-launch kernel times from an ncu --metrics gpu__time_duration.sum CSV (skips packing/rendering)."""
import csv
import sys
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[i]
    ki, mi, ni = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Name')
    print(path)
    for r in rows[i + 1:]:
        if len(r) > mi and r[ni] == 'gpu__time_duration.sum' and not any(
                x in r[ki] for x in ('pack', 'render', 'bg_kernel')):
            print(f"  {r[ki].split('(')[0][:48]:48s} {float(r[mi].replace(',', '')) / 1e3:9.1f} us")
