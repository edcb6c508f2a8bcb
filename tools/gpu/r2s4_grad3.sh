# k_grad2d: warp-voted lazy path, 2/h without the division; NS parity, A/B on cfg 5
L=$PWD/paper_2403_05144_b200/lib
for v in P1 P1D; do
PERK_LIB_PATH=$L/libperk_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dd.py tests/test_gpu_races.py tests/test_gpu_patterns.py -m gpu -x -q -k "ns or cfg5 or navier" > gpurun_out/t_$v.log 2>&1; echo t_$v=$? >> gpurun_out/status_g3.txt
done
timeout 1500 python tools/ab_kinds.py 5 N1S0 P0 P1 P1D P1S1 3 > gpurun_out/ab_grad_vote.json 2> gpurun_out/ab_grad_vote.err; echo ab=$? >> gpurun_out/status_g3.txt
