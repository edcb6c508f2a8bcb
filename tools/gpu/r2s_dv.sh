timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py tests/test_gpu_sc.py tests/test_gpu_patterns.py tests/test_gpu_dd.py -x -q -k "ns or cfg5 or navier or NS or sc or dd" > gpurun_out/dv_tests.log 2>&1; echo tests=$? >> gpurun_out/status_dv.txt
timeout 600 python tools/ab_kinds.py 5,5sc A B 3 > gpurun_out/ab_dv.json 2> gpurun_out/ab_dv.err; echo ab=$? >> gpurun_out/status_dv.txt
timeout 300 python tools/kind_fracs.py 5,5e,3,3big > gpurun_out/kind_fracs.json 2> gpurun_out/kind_fracs.err; echo kf=$? >> gpurun_out/status_dv.txt
