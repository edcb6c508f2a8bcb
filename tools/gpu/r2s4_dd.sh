timeout 900 python tools/dd_overhead.py 5 2,4,8 > gpurun_out/dd_overhead_cfg5.json 2> gpurun_out/dd_overhead.err; echo dd5=$? >> gpurun_out/status_dd.txt
timeout 600 python tools/dd_overhead.py 3 2,4,8 > gpurun_out/dd_overhead_cfg3.json 2>> gpurun_out/dd_overhead.err; echo dd3=$? >> gpurun_out/status_dd.txt
