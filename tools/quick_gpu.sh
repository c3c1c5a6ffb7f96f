#!/bin/bash
# quick GPU check: pair parity tests + two C2 bench runs (+ optional extra shapes)
python -m pytest tests/test_gpu_pair.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for i in 1 2; do
  timeout 300 python bench.py --steps 300 --warmup 5 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        j=json.loads(l); print('C2', round(j['value']), round(j['ms_per_step']*1e3,3), 'us frac', round(j['roofline']['frac'],4), 'e2e', round(j['e2e']['value']))"
done
for shp in "$@"; do
  timeout 300 python bench.py --steps 100 --warmup 5 --shape $shp 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        j=json.loads(l); print('$shp', round(j['value']), round(j['ms_per_step']*1e3,3), 'us frac', round(j['roofline']['frac'],4))"
done
