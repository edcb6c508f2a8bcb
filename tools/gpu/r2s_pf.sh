timeout 700 python tools/ab_kinds.py 5 P0 P1 P2 M3 3 > gpurun_out/ab_pf.json 2> gpurun_out/ab_pf.err; echo ab=$? >> gpurun_out/status_pf.txt
