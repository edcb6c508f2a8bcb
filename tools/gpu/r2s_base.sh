set -x
nproc > gpurun_out/nproc.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/status.txt
