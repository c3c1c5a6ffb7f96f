# Interleaved A/B of the bench e2e legs between two library builds (paper_2501_08455_b200/exp_base.so, exp_h2d.so)
for rep in 1 2 3; do for lib in exp_base exp_h2d; do
SIGK_LIB_PATH=paper_2501_08455_b200/$lib.so python bench.py --steps 200 --warmup 5 --no-cpu 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        j=json.loads(l); print('$lib', round(j['e2e']['value']), round(j['e2e']['link_gbs']['h2d'],1), round(j['e2e']['synchronous']['value']))"
done; done
