timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1
timeout 400 python bench.py --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
