set -x
bash tools/ab.sh 5,3 A B > gpurun_out/ab5.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/gputests5.log 2>&1; echo rc=$? >> gpurun_out/gputests5.log
