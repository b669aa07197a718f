"""Summarise ncu reports for profiles/: key raw metrics + top stall sites.

usage: python tools/ncu_summary.py REPORT.ncu-rep [label] > profiles/rNN/<name>.txt
       python tools/ncu_summary.py --launches launches.csv > profiles/rNN/launches.txt
"""
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg",
    "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__sass_inst_executed_op_utcmma.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_shared_mem",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        res.append({k: (r[i], u[i]) for i, k in enumerate(h)})
    return res


def stalls(rep, topn=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    if not rows:
        return []
    h, body = rows[0], rows[1:]
    ci = h.index("Warp Stall Sampling (All Samples)")
    cols = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
    tot = sum(int(r[ci] or 0) for r in body) or 1
    agg = {}
    for r in body:
        for c in cols:
            agg[h[c]] = agg.get(h[c], 0) + int(r[c] or 0)
    lines = ["stall reasons (share of samples): " +
             ", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:6])]
    idx = sorted(range(len(body)), key=lambda i: -int(body[i][ci] or 0))[:topn]
    lines.append("top SASS sites by stall samples:")
    for i in sorted(idx):
        lines.append(f"  {int(body[i][ci]) / tot:6.1%}  {body[i][1].strip()[:90]}")
    return lines


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, mi, ni = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = {}
    for r in rows[start + 1:]:
        if len(r) <= mi or r[ni] != "gpu__time_duration.sum":
            continue
        k = r[ki].split("(")[0]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r[mi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print("kernel, launches, total_ms, share_of_listed_time")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k}, {n}, {v * 1e-6:.3f}, {v / tot:.3f}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
        sys.exit(0)
    rep = sys.argv[1]
    for d in raw(rep):
        name = d.get("Kernel Name", ("?",))[0]
        print(f"kernel: {name}")
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k][0]} {d[k][1]}")
    for l in stalls(rep):
        print(l)
