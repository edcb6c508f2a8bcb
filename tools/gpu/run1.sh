set -x
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests/test_gpu_amr.py tests/test_gpu_parity.py -x -q -m gpu -k "amr or capacity or adapt or Rusanov or rhs_eval" > gpurun_out/t1.log 2>&1; echo rc=$? >> gpurun_out/t1.log
timeout 600 python tools/quick_bench.py 5,3 > gpurun_out/qb.log 2>&1; echo rc=$? >> gpurun_out/qb.log
