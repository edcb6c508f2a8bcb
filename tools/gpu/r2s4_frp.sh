# complete BASELINE runs of the end-of-round kernels against the OpenMP oracle
ORACLE_OMP=1 timeout 3400 python tools/full_run_parity.py 5:200,4:1000,3:500,5sc:100 > gpurun_out/full_run_parity_final.json 2> gpurun_out/frp.err; echo frp=$? >> gpurun_out/status_frp.txt
