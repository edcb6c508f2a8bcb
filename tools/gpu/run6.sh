set -x
python tools/ab_kinds.py 5,3,5sc A B C 3 > gpurun_out/abk6.json 2> gpurun_out/abk6.err
