timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_stream -s 2 -c 1 -o gpurun_out/stream_c2 python tools/stream_bench.py 128 1000 5 4 3 > gpurun_out/ncu_stream.log 2>&1
