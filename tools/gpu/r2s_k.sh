timeout 700 python tools/ab_kinds.py 5 K2 K1 3 > gpurun_out/ab_k.json 2> gpurun_out/ab_k.err; echo ab=$? >> gpurun_out/status_k.txt
