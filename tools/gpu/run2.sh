set -x
python bench.py --config 5 --steps 5 --warmup 3 --extra 3 --no-cpu-baseline > gpurun_out/b2.json 2> gpurun_out/b2.err; echo rc=$? >> gpurun_out/b2.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum
for C in 5 3; do
python bench.py --profile-only --config $C --steps 1 --warmup 3 > gpurun_out/po$C.log 2>&1 && \
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/counts_cfg$C.csv python bench.py --profile-only --config $C --steps 1 --warmup 3 > gpurun_out/ncu$C.log 2>&1
done
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
