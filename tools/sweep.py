"""Throughput sweep of bench.py over plan overrides for one config.
    python tools/sweep.py c2 "U=20,G=1 U=16,G=2 family=path,U=12" [steps]
Keys: U (chunks), G (segments), Q (prefix_len), family (auto|path|flat|pair)."""
import json
import subprocess
import sys

cfg = sys.argv[1]
combos = sys.argv[2].split()
steps = sys.argv[3] if len(sys.argv) > 3 else "5000"
FLAG = {"U": "--chunks", "G": "--segments", "Q": "--prefix-len", "family": "--family", "shape": "--shape"}
for c in combos:
    extra = []
    for kv in c.split(","):
        k, v = kv.split("=")
        extra += [FLAG[k], v.replace(":", ",")]
    r = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--no-cpu", "--e2e-steps", "3", "--steps", steps]
                       + extra, capture_output=True, text=True)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        cf = d["config"]
        print(json.dumps({"cfg": cfg, "req": c, "family": cf.get("family"), "G": cf.get("segments"),
                          "U": cf["chunks"], "Q": cf["prefix_len"], "paths_per_s": round(d["value"]),
                          "us_per_step": round(d["ms_per_step"] * 1e3, 2),
                          "kernel_us": round(d["roofline"]["kernel_ms_event_bracketed"] * 1e3, 2),
                          "single_launch_us": round(cf["single_launch_ms"] * 1e3, 1),
                          "frac": round(d["roofline"]["frac"], 3), "parity": cf["parity_max_level_rel_err"]}),
              flush=True)
    except Exception:  # noqa: BLE001
        print(c, "failed", r.stderr[-800:], flush=True)
