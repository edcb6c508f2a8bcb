# k_grad2d: next group's gathers one iteration ahead in registers (3 CTAs/SM); parity then A/B
L=$PWD/paper_2403_05144_b200/lib
PERK_LIB_PATH=$L/libperk_PF3.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dd.py tests/test_gpu_races.py tests/test_gpu_patterns.py -m gpu -x -q -k "ns or cfg5 or navier" > gpurun_out/t_PF3.log 2>&1; echo t_PF3=$? >> gpurun_out/status_pf.txt
timeout 1500 python tools/ab_kinds.py 5,5sc Z0 PF3 Z3 3 > gpurun_out/ab_grad_pf.json 2> gpurun_out/ab_grad_pf.err; echo ab=$? >> gpurun_out/status_pf.txt
