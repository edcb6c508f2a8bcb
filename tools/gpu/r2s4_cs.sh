timeout 1500 python tools/ab_kinds.py 5,3 T0 T1 T2 T3 3 > gpurun_out/ab_cs.json 2> gpurun_out/ab_cs.err; echo ab=$? >> gpurun_out/status_cs.txt
