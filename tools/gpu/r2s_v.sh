timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "face_table or ns_repartition or cfg5_small" > gpurun_out/ft_tests.log 2>&1; echo tests=$? >> gpurun_out/status_v.txt
timeout 700 python tools/ab_kinds.py 5 V0 V1 3 > gpurun_out/ab_v.json 2> gpurun_out/ab_v.err; echo ab=$? >> gpurun_out/status_v.txt
