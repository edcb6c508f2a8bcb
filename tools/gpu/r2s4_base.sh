# session 4 start: full GPU suite, bench (default), ncu launch list of the bench command, --set full of the three cfg-5 kernels at stage 30
sha256sum paper_2403_05144_b200/lib/libperk_b200.so | cut -c1-16 > gpurun_out/lib_sha16.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra none > gpurun_out/ncu_launches.log 2>&1; echo launches=$? >> gpurun_out/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(vol|surf|grad)2d" --launch-skip 87 --launch-count 3 -o gpurun_out/full_cfg5_s30 python bench.py --profile-only --config 5 --steps 1 --warmup 0 > gpurun_out/ncu_full.log 2>&1; echo full=$? >> gpurun_out/status.txt
