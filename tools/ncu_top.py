"""Summarise an ncu report's SASS source page: top instructions by stall samples."""
import csv, subprocess, sys
rep = sys.argv[1]; topn = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]; body = rows[1:]
ci = h.index("Warp Stall Sampling (All Samples)"); ie = h.index("Instructions Executed")
stall_cols = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(int(r[ci] or 0) for r in body)
print("total samples", tot, "instructions", len(body))
idx = sorted(range(len(body)), key=lambda i: -int(body[i][ci] or 0))[:topn]
for i in sorted(idx):
    r = body[i]
    reasons = sorted(((int(r[c] or 0), h[c][6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{i:5d} {int(r[ci]):7d} {r[1].strip()[:60]:60s} " + " ".join(f"{n}:{v}" for v, n in reasons if v))
