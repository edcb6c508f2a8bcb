# final build of the round: full GPU suite, smoke, bench (default), ncu launch list of the bench command (capped),
# ncu counts per kind (cfg 5, cfg 3), --set full of the cfg-5 kernels at stage 30 and the cfg-3 kernels at stage 14
sha256sum paper_2403_05144_b200/lib/libperk_b200.so | cut -c1-16 > gpurun_out/lib_sha16.txt
rm -f gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/status.txt
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra none > gpurun_out/ncu_launches.log 2>&1; echo launches=$? >> gpurun_out/status.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum
for c in 5 3; do
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/counts_cfg$c.csv python bench.py --profile-only --config $c --steps 1 --warmup 3 > gpurun_out/ncu_counts$c.log 2>&1; echo counts$c=$? >> gpurun_out/status.txt
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(vol|surf|grad)2d" --launch-skip 87 --launch-count 3 -o gpurun_out/full_cfg5_s30 -f python bench.py --profile-only --config 5 --steps 1 --warmup 0 > gpurun_out/ncu_full5.log 2>&1; echo full5=$? >> gpurun_out/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(vol|surf)2d" --launch-skip 26 --launch-count 2 -o gpurun_out/full_cfg3_s14 -f python bench.py --profile-only --config 3 --steps 1 --warmup 0 > gpurun_out/ncu_full3.log 2>&1; echo full3=$? >> gpurun_out/status.txt
