set -x
sha256sum paper_2403_05144_b200/lib/libperk_b200.so | cut -c1-16 > gpurun_out/lib_sha16.txt
timeout 900 python -m pytest tests/test_gpu_dd.py -x -q > gpurun_out/dd.log 2>&1; echo rc=$? >> gpurun_out/dd.log
timeout 1500 python -m pytest tests/test_gpu_full_runs.py -x -q --durations=5 > gpurun_out/full.log 2>&1; echo rc=$? >> gpurun_out/full.log
