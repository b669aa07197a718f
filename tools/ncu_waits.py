"""List mbarrier wait sites of an ncu report with stall samples and spin counts."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:])); h = rows[0]; body = rows[1:]
ie = h.index("Instructions Executed"); ci = h.index("Warp Stall Sampling (All Samples)")
print('total samples', sum(int(r[ci] or 0) for r in body))
for i, r in enumerate(body):
    s = r[1]
    nxt = body[i + 1] if i + 1 < len(body) else r
    if 'TRYWAIT' in s and int(r[ie] or 0) > 1000:
        print(i, 'spins', r[ie], 'samples', int(r[ci] or 0) + int(nxt[ci] or 0), s.strip()[:80])
out2 = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rr = list(csv.reader(out2)); hh = rr[0]; vv = rr[2]
for k in ("gpu__time_duration.sum", "sm__cycles_elapsed.avg", "TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"):
    if k in hh: print(k, vv[hh.index(k)])
