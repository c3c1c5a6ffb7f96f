mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:pair_kernel -s 2 -c 1 -f -o gpurun_out/pair_c2x python tools/run_sig.py c2x 4 U=10 G=1 > gpurun_out/ncu_c2x.log 2>&1
tail -3 gpurun_out/ncu_c2x.log
