timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python tools/sweep.py c2 "family=auto" 5000 > gpurun_out/sweep_c2.txt 2>&1
