# k_grad2d L1-wavefront variants: NS parity per variant, then A/B on cfg 5
L=$PWD/paper_2403_05144_b200/lib
for v in L1 LW2 LW2X LW2S0 LW2XS0; do
PERK_LIB_PATH=$L/libperk_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dd.py tests/test_gpu_races.py -m gpu -x -q -k "ns or cfg5 or navier" > gpurun_out/t_$v.log 2>&1; echo t_$v=$? >> gpurun_out/status_g.txt
done
timeout 1500 python tools/ab_kinds.py 5 B0 B1 L1 LW2 LW2X LW2S0 LW2XS0 3 > gpurun_out/ab_grad_l1.json 2> gpurun_out/ab_grad_l1.err; echo ab=$? >> gpurun_out/status_g.txt
