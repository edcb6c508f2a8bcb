timeout 1500 python tools/ab_kinds.py 5,3 H0 H1 H2 3 > gpurun_out/ab_hints2.json 2> gpurun_out/ab_hints2.err; echo ab=$? >> gpurun_out/status_h.txt
