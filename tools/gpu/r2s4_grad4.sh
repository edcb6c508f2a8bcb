L=$PWD/paper_2403_05144_b200/lib
for v in Q0; do
PERK_LIB_PATH=$L/libperk_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dd.py tests/test_gpu_races.py tests/test_gpu_patterns.py -m gpu -x -q -k "ns or cfg5 or navier" > gpurun_out/t_$v.log 2>&1; echo t_$v=$? >> gpurun_out/status_g4.txt
done
timeout 1500 python tools/ab_kinds.py 5 P1D Q0 Q1 Q3 Q4 3 > gpurun_out/ab_grad_q.json 2> gpurun_out/ab_grad_q.err; echo ab=$? >> gpurun_out/status_g4.txt
