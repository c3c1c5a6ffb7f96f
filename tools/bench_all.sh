#!/bin/bash
# every config's bench line (+ the reference arm at C2) into gpurun_out/bench_<cfg>.json
mkdir -p gpurun_out
for c in c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
l = [x for x in open(f"gpurun_out/bench_{c}.json") if x.startswith("{")]
j = json.loads(l[-1])
print(c, round(j["value"]), j["unit"], "ms/step", round(j["ms_per_step"], 5), "frac", round(j["roofline"]["frac"], 3),
      "e2e", round(j["e2e"]["value"]), "cpu", j["cpu_baseline"]["value"] if j.get("cpu_baseline") else None,
      "clk", j["clocks"]["sm_mhz"], j["clocks"]["reasons"], "family", j["config"].get("family"))
PY
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference_c2.json 2>/dev/null; tail -1 gpurun_out/bench_reference_c2.json | cut -c1-300
