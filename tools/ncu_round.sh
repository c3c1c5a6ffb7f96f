#!/bin/bash
# Round-end profiling: one ncu --set full capture of each config's fold kernel
# and the launch list of the headline bench command (B200_PROFILING.md recipe).
mkdir -p gpurun_out/ncu
for spec in c1:pair_kernel c2:pair_kernel c3:pair_kernel c4:ipair_kernel c5:path_kernel; do
  c=${spec%%:*}; k=${spec#*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^${k}|${k}" -s 2 -c 1 -f \
      -o gpurun_out/ncu/${k}_${c}_full python tools/run_sig.py $c 4 > gpurun_out/ncu/${c}.log 2>&1
  echo "$c $k rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/ncu/ncu_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu/launches.log 2>&1
echo "launches rc=$?"
ls -la gpurun_out/ncu
