timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1
./tools/sigbench --paper-grid --dims 5 --dtype f32 --kernels sequential > gpurun_out/sigbench_paper_f32.csv 2> gpurun_out/sigbench.err
./tools/sigbench --paper-grid --dims 5 --dtype f64 --kernels sequential > gpurun_out/sigbench_paper_f64.csv 2>> gpurun_out/sigbench.err
