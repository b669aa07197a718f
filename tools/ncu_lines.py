"""Per-CUDA-source-line stall samples and executed instructions of an ncu report
(needs -lineinfo + --import-source on).  usage: python tools/ncu_lines.py REP [topn]"""
import csv, subprocess, sys
rep = sys.argv[1]; topn = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda"],
                     capture_output=True, text=True).stdout.splitlines()
cur = None; rows = []
for r in csv.reader(out):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": ci = r.index("Warp Stall Sampling (All Samples)"); ie = r.index("Instructions Executed"); continue
    if r[0].isdigit() and len(r) > ie:
        try:
            rows.append((cur, int(r[0]), int(r[ci]), int(r[ie] or 0), r[1]))
        except ValueError:
            pass
ts = sum(x[2] for x in rows) or 1; ti = sum(x[3] for x in rows) or 1
print(f"samples {ts}  warp-instructions {ti}")
for f, ln, s, n, src in sorted(rows, key=lambda x: -x[2])[:topn]:
    print(f"{f}:{ln:<5} stall {100*s/ts:5.1f}%  inst {100*n/ti:5.1f}%  {src.strip()[:90]}")
