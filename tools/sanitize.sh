#!/bin/bash
# compute-sanitizer passes over the smoke path (pair fold, stream, VJP) and a few suites
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  echo "== $tool smoke"; timeout 900 $S --tool $tool python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
done
echo "== memcheck tests"
timeout 1200 $S --tool memcheck python -m pytest tests/test_gpu_vjp.py tests/test_gpu_async_host.py tests/test_gpu_increments.py -q 2>&1 | tail -2
