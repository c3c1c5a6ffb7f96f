"""Throughput sweep of bench.py over (chunks, prefix_len) for one config.
    python tools/sweep.py c2 "4:2 8:2 12:2 16:2 20:2 10:1 20:1 51:1" [steps]"""
import json
import subprocess
import sys

cfg = sys.argv[1]
combos = sys.argv[2].split()
steps = sys.argv[3] if len(sys.argv) > 3 else "5000"
for c in combos:
    k, q = c.split(":")
    r = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--no-cpu", "--e2e-steps", "3", "--steps", steps,
                        "--chunks", k, "--prefix-len", q], capture_output=True, text=True)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        print(json.dumps({"cfg": cfg, "chunks": d["config"]["chunks"], "Q": d["config"]["prefix_len"],
                          "paths_per_s": round(d["value"]), "us_per_step": round(d["ms_per_step"] * 1e3, 2),
                          "single_launch_us": round(d["config"]["single_launch_ms"] * 1e3, 1),
                          "frac": round(d["roofline"]["frac"], 3)}), flush=True)
    except Exception as e:  # noqa: BLE001
        print(c, "failed", r.stderr[-500:], flush=True)
