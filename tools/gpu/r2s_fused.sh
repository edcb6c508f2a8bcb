timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py tests/test_gpu_sc.py tests/test_gpu_patterns.py tests/test_gpu_dd.py tests/test_gpu_full_runs.py -x -q -k "ns or cfg5 or navier or NS or sc or dd or 5" > gpurun_out/fu_tests.log 2>&1; echo tests=$? >> gpurun_out/status_fu.txt
timeout 600 python tools/ab_kinds.py 5,5sc C D 3 > gpurun_out/ab_fused.json 2> gpurun_out/ab_fused.err; echo ab=$? >> gpurun_out/status_fu.txt
timeout 300 python tools/ab_kinds.py 3 D SP3 SP2 3 > gpurun_out/ab_surfpf.json 2> gpurun_out/ab_surfpf.err; echo ab2=$? >> gpurun_out/status_fu.txt
timeout 300 bash tools/ab.sh 1 T64 T128 T256 > gpurun_out/ab_cfg1.log 2>&1; echo ab3=$? >> gpurun_out/status_fu.txt
timeout 300 python tools/kind_fracs.py 5 > gpurun_out/kind_fracs_fused.json 2> gpurun_out/kind_fracs_fused.err; echo kf=$? >> gpurun_out/status_fu.txt
