set -x
sha256sum paper_2403_05144_b200/lib/libperk_b200.so | cut -c1-16 > gpurun_out/lib_sha16.txt
python bench.py --config 5 --steps 8 --warmup 3 --extra 5sc,3sc --no-cpu-baseline > gpurun_out/b4.json 2> gpurun_out/b4.err
python bench.py --profile-only --config 3 --steps 1 --warmup 0 > gpurun_out/p3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_surf2d|k_vol2d" -s 26 -c 2 -o gpurun_out/full_cfg3 python bench.py --profile-only --config 3 --steps 1 --warmup 0 > gpurun_out/ncu_full3.log 2>&1
python bench.py --profile-only --config 5 --steps 1 --warmup 0 > gpurun_out/p5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gsurf2d|k_grad2d|k_surf2d|k_vol2d" -s 116 -c 4 -o gpurun_out/full_cfg5 python bench.py --profile-only --config 5 --steps 1 --warmup 0 > gpurun_out/ncu_full5.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum
for C in 5 3; do
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/counts_cfg$C.csv python bench.py --profile-only --config $C --steps 1 --warmup 3 > gpurun_out/ncu$C.log 2>&1
done
