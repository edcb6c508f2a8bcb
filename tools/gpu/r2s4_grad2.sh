# k_grad2d stride-20 shared layout variants: NS parity, then A/B on cfg 5
L=$PWD/paper_2403_05144_b200/lib
for v in N1 N1S0; do
PERK_LIB_PATH=$L/libperk_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dd.py tests/test_gpu_races.py -m gpu -x -q -k "ns or cfg5 or navier" > gpurun_out/t_$v.log 2>&1; echo t_$v=$? >> gpurun_out/status_g2.txt
done
timeout 1500 python tools/ab_kinds.py 5 LW2S0 N0 N1 N1S0 N1X N1XS0 3 > gpurun_out/ab_grad_sx.json 2> gpurun_out/ab_grad_sx.err; echo ab=$? >> gpurun_out/status_g2.txt
PERK_LIB_PATH=$L/libperk_N1S0.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_grad2d" --launch-skip 29 --launch-count 1 -o gpurun_out/grad_N1S0 python bench.py --profile-only --config 5 --steps 1 --warmup 0 > gpurun_out/ncu_gn.log 2>&1; echo gn=$? >> gpurun_out/status_g2.txt
