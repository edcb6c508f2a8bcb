timeout 700 python tools/ab_kinds.py 5,3 P0 Q0 Q1 3 > gpurun_out/ab_q.json 2> gpurun_out/ab_q.err; echo ab=$? >> gpurun_out/status_q.txt
