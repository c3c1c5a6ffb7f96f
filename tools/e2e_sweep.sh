for shp in 128,1000,5,4 128,10000,5,4 32,100,2,4 64,500,10,5; do
 for pcs in "" 1 2 4; do
  for tp in "" 1; do
   echo "== $shp pieces=${pcs:-auto} throughput_plan=${tp:-0}"
   env $( [ -n "$pcs" ] && echo SIGK_HOST_PIECES=$pcs ) $( [ -n "$tp" ] && echo SIGK_HOST_THROUGHPUT_PLAN=1 ) python tools/e2e_probe.py $shp 100 | grep -E "host call|host plan" | tail -2
  done
 done
done
