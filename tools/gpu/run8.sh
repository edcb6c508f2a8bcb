python tools/ab_kinds.py 5,3,5sc,3sc B E F 3 > gpurun_out/abk8.json 2> gpurun_out/abk8.err
