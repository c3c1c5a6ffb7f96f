"""Summaries of round-end ncu captures -> profiles/<round>/ (text) and
profiles/ncu_traffic.json (dram bytes per launch, read by bench.py):
    python tools/ncu_summarize.py gpurun_out/ncu profiles/r01"""
import csv
import io
import json
import os
import subprocess
import sys

src, dst = sys.argv[1], sys.argv[2]
KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.per_cycle_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "smsp__inst_executed.sum", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum"]
traffic_path = os.path.join(os.path.dirname(dst.rstrip("/")), "ncu_traffic.json")
traffic = {}
for f in sorted(os.listdir(src)):
    if not f.endswith("_full.ncu-rep"):
        continue
    cfg = f.split("_")[-2]
    rep = os.path.join(src, f)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2]
    get = {n: (v[i], units[i]) for i, n in enumerate(h)}
    name = get.get("Kernel Name", ("?", ""))[0]
    lines = [f"{f}  kernel {name}"]
    for k in KEYS:
        if k in get:
            lines.append(f"  {k:60s} {get[k][0]} {get[k][1]}")
    stalls = sorted(((float(get[n][0] or 0), n) for n in h
                     if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")),
                    reverse=True)[:6]
    lines.append("  stalls per issue: " + ", ".join(f"{n.split('stalled_')[1].split('_per')[0]}={x:.2f}" for x, n in stalls))
    txt = "\n".join(lines)
    print(txt)
    with open(os.path.join(dst, f.replace(".ncu-rep", "_summary.txt")), "w") as o:
        o.write(txt + "\n")

    def mb(k):
        val, unit = get.get(k, ("0", "byte"))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
        return float(val or 0) * scale

    traffic[cfg] = {"dram_bytes_per_launch": int(mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")),
                    "source": f"{dst}/{f} (dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full, one launch)",
                    "kernel": name}
with open(traffic_path, "w") as o:
    json.dump(traffic, o, indent=1)
print("wrote", traffic_path)
