# streaming hints adopted: whole GPU suite, smoke, default bench, launch list, ncu counts per kind
rm -f gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/gputests_last2.log 2>&1; echo tests=$? >> gpurun_out/status.txt
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke_last2.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench_last2.json 2> gpurun_out/bench_last2.err; echo bench=$? >> gpurun_out/status.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum
for c in 5 3; do
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/counts_cfg$c.csv python bench.py --profile-only --config $c --steps 1 --warmup 3 > gpurun_out/ncu_counts$c.log 2>&1; echo counts$c=$? >> gpurun_out/status.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra none > gpurun_out/ncu_launches.log 2>&1; echo launches=$? >> gpurun_out/status.txt
