timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py tests/test_gpu_sc.py tests/test_gpu_patterns.py tests/test_gpu_dd.py -x -q -k "ns or cfg5 or navier or NS or sc or dd or 5" > gpurun_out/nb_tests.log 2>&1; echo tests=$? >> gpurun_out/status_nb.txt
timeout 600 python tools/ab_kinds.py 5,5sc N0 NB 3 > gpurun_out/ab_nb.json 2> gpurun_out/ab_nb.err; echo ab=$? >> gpurun_out/status_nb.txt
timeout 300 bash tools/ab.sh 1 T256 NB > gpurun_out/ab_cfg1b.log 2>&1; echo ab3=$? >> gpurun_out/status_nb.txt
timeout 300 bash tools/ab.sh 2 T256 NB > gpurun_out/ab_cfg2b.log 2>&1; echo ab4=$? >> gpurun_out/status_nb.txt
PERK_LIB_PATH=$PWD/paper_2403_05144_b200/lib/libperk_NB.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_grad2d" --launch-skip 28 --launch-count 2 -o gpurun_out/grad_NB python bench.py --profile-only --config 5 --steps 1 --warmup 0 > gpurun_out/ncu_nb.log 2>&1; echo gf=$? >> gpurun_out/status_nb.txt
