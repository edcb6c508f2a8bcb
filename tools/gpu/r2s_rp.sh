timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ns or cfg5 or NS" > gpurun_out/rp_tests_default.log 2>&1; echo tests=$? >> gpurun_out/status_rp.txt
PERK_LIB_PATH=$PWD/paper_2403_05144_b200/lib/libperk_RP.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dd.py -x -q -k "ns or cfg5 or NS or dd" > gpurun_out/rp_tests.log 2>&1; echo tests_rp=$? >> gpurun_out/status_rp.txt
timeout 700 python tools/ab_kinds.py 5 R0 RP 3 > gpurun_out/ab_rp.json 2> gpurun_out/ab_rp.err; echo ab=$? >> gpurun_out/status_rp.txt
