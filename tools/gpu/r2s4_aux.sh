# end-of-round records of the AMR adapt / repartition timings and the shock-capturing costs
timeout 600 python tools/amr_profile.py > gpurun_out/amr_timing_final.json 2> gpurun_out/amr_timing.err; echo amr=$? >> gpurun_out/status_aux.txt
timeout 900 python tools/sc_profile.py > gpurun_out/sc_profile_final.json 2> gpurun_out/sc_profile.err; echo sc=$? >> gpurun_out/status_aux.txt
