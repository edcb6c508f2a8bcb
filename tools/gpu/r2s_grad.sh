timeout 600 python tools/ab_kinds.py 5 D E F 3 > gpurun_out/ab_grad.json 2> gpurun_out/ab_grad.err; echo ab=$? >> gpurun_out/status_g.txt
python tools/step1d_profile.py 200 > gpurun_out/step1d_time.json 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_step1d -s 2 -c 1 -o gpurun_out/step1d_multi python tools/step1d_profile.py 1 > gpurun_out/ncu_s1.log 2>&1; echo s1=$? >> gpurun_out/status_g.txt
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_step1d -s 5 -c 1 -o gpurun_out/step1d_single python tools/step1d_profile.py 1 > gpurun_out/ncu_s2.log 2>&1; echo s2=$? >> gpurun_out/status_g.txt
PERK_LIB_PATH=$PWD/paper_2403_05144_b200/lib/libperk_F.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_grad2d" --launch-skip 29 --launch-count 1 -o gpurun_out/grad_F python bench.py --profile-only --config 5 --steps 1 --warmup 0 > gpurun_out/ncu_gf.log 2>&1; echo gf=$? >> gpurun_out/status_g.txt
