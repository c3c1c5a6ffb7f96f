timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 4 -c 1 -o gpurun_out/pair_c2_full2 python tools/run_sig.py c2 6 > gpurun_out/ncu_full.log 2>&1
