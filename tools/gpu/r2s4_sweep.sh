# alternating sweep direction: A/B by environment knob on one library, then parity subset
timeout 1500 python tools/ab_kinds.py 5,3,5sc R0 R0:PERK_SWEEP=0 R1 3 > gpurun_out/ab_sweep.json 2> gpurun_out/ab_sweep.err; echo ab=$? >> gpurun_out/status_s.txt
L=$PWD/paper_2403_05144_b200/lib
PERK_LIB_PATH=$L/libperk_R0.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dd.py tests/test_gpu_races.py tests/test_gpu_patterns.py tests/test_gpu_sc.py -m gpu -x -q > gpurun_out/t_R0.log 2>&1; echo t_R0=$? >> gpurun_out/status_s.txt
