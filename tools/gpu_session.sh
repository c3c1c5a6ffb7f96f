for c in c2 c3 c4 c5 c1; do timeout 300 python bench.py --config $c --no-cpu --e2e-steps 50 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1
