# committed end-of-round tree: whole GPU suite, smoke, default bench, two short bench repeats (run-to-run spread)
rm -f gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/gputests_last.log 2>&1; echo tests=$? >> gpurun_out/status.txt
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke_last.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench_last.json 2> gpurun_out/bench_last.err; echo bench=$? >> gpurun_out/status.txt
for i in 1 2; do timeout 600 python bench.py --extra none --no-cpu-baseline > gpurun_out/bench_rep$i.json 2>> gpurun_out/bench_last.err; echo rep$i=$? >> gpurun_out/status.txt; done
