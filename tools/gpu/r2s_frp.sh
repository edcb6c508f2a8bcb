ORACLE_OMP=1 OMP_NUM_THREADS=16 timeout 1800 python tools/full_run_parity.py 5:200 > gpurun_out/frp_5.json 2> gpurun_out/frp_5.err; echo f5=$? >> gpurun_out/status_frp.txt
ORACLE_OMP=1 OMP_NUM_THREADS=16 timeout 1800 python tools/full_run_parity.py 5sc:200 > gpurun_out/frp_5sc.json 2> gpurun_out/frp_5sc.err; echo f5sc=$? >> gpurun_out/status_frp.txt
