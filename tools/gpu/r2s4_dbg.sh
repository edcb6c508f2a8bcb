# the new sweep-direction test, then the whole GPU suite against the bounds-checked debug build
timeout 600 python -m pytest tests/test_gpu_races.py -m gpu -x -q > gpurun_out/t_races.log 2>&1; echo races=$? >> gpurun_out/status_d.txt
PERK_LIB_PATH=$PWD/paper_2403_05144_b200/lib/libperk_debug.so timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/t_debug.log 2>&1; echo debug=$? >> gpurun_out/status_d.txt
PERK_LIB_PATH=$PWD/paper_2403_05144_b200/lib/libperk_debug.so timeout 600 python tools/sanitize_run.py > gpurun_out/sanitize_dbg.log 2>&1; echo sanrun=$? >> gpurun_out/status_d.txt
