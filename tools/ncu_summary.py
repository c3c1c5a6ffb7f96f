"""Summarise an .ncu-rep: headline metrics, stall reasons, and SASS regions by executed instructions."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr = r[0]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__block_size",
        "launch__grid_size", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "sm__cycles_elapsed.avg", "smsp__cycles_active.avg"]
for row in r[2:]:
    for h, v in zip(hdr, row):
        if h in want:
            print(f"{h:70s} {v}")
    st = [(h, v) for h, v in zip(hdr, row) if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio")]
    st.sort(key=lambda x: -float(x[1] or 0))
    print("stalls:", ", ".join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={float(v):.2f}" for h, v in st[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ai, si, ei, wi = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = []
for x in rows[2:]:
    if len(x) < len(h):
        continue
    try:
        data.append((x[ai], x[si].strip(), int(x[ei] or 0), int(x[wi] or 0)))
    except ValueError:
        pass
tot = sum(d[2] for d in data) or 1
totw = sum(d[3] for d in data) or 1
print(f"total warp-inst {tot}  stall samples {totw}")
regions = []
for a, s, e, w in data:
    op = s.split()[0] if s else ""
    if op.startswith("@"):
        op = s.split()[1]
    if regions and regions[-1][2] == e:
        regions[-1][3] += 1
        regions[-1][4] += w
        regions[-1][5][op.split(".")[0]] += 1
    else:
        regions.append([a, s, e, 1, w, Counter({op.split(".")[0]: 1})])
for a, s, e, n, w, ops in regions:
    if e * n > tot * 0.01 or w > totw * 0.02:
        print(f"{a[-5:]} exec={e:8d} n={n:4d} inst={e*n/tot:6.1%} stall={w/totw:6.1%} {dict(ops.most_common(6))}")

# per-region stall breakdown
sc = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
reg_stalls = []
cur = None
for x in rows[2:]:
    if len(x) < len(h):
        continue
    try:
        e = int(x[ei] or 0)
    except ValueError:
        continue
    if cur is None or cur[0] != e:
        cur = [e, Counter(), x[ai]]
        reg_stalls.append(cur)
    for i in sc:
        try:
            cur[1][h[i]] += int(x[i] or 0)
        except ValueError:
            pass
for e, c, a in reg_stalls:
    t = sum(c.values())
    if t > totw * 0.03:
        print(f"{a[-5:]} stall={t/totw:5.1%} " + ", ".join(f"{k[6:]}={v/t:.0%}" for k, v in c.most_common(4)))
