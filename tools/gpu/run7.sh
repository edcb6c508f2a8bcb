python tools/ab_kinds.py 5sc,3sc B D D:PERK_SC_FUSED=0 3 > gpurun_out/abk7.json 2> gpurun_out/abk7.err
