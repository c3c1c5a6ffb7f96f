for f in 0 1 2 3 4 7; do echo "flags=$f"; SIGK_EXPERIMENT=$f timeout 300 python tools/sweep.py c2 "family=auto U=10,G=2 U=20,G=1" 5000 2>&1; done > gpurun_out/sweep_exp.txt
