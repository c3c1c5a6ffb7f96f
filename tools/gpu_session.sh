timeout 900 python -m pytest tests/test_gpu_vjp.py -q > gpurun_out/pytest_vjp.txt 2>&1
