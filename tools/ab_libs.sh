#!/bin/bash
# A/B of library builds on the same box: tools/ab_libs.sh "<shape|c2> ..." lib1 lib2 ...
# (libs are paper_2501_08455_b200/<name>.so; shapes as bench.py --shape, c2 = default)
shapes=$1; shift
for rep in 1 2; do
for lib in "$@"; do
  for shp in $shapes; do
    arg=""; [ "$shp" != "c2" ] && arg="--shape $shp"
    SIGK_LIB_PATH=paper_2501_08455_b200/$lib.so timeout 300 python bench.py --steps ${STEPS:-2000} --warmup 20 --no-cpu $arg 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        j=json.loads(l); sc=j['roofline'].get('single_call',{}); sp=sc.get('device_span_ms',{})
        print('$lib $shp', round(j['ms_per_step']*1e3,3), 'us frac', round(j['roofline']['frac'],4), j['config'].get('chunks'), j['config'].get('segments'),
              'span_us', {k: round(v*1e3,2) for k,v in sp.items()})"
  done
done
done
