# ncu full capture (with source-level stall sampling) of one decode launch: tools/gpu_prof.sh <shape> <tag>
mkdir -p gpurun_out
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on --warp-sampling-interval 0 -k regex:k_decode -s 3 -c 1 -o gpurun_out/prof_$2 python tools/prof_decode.py $1 > gpurun_out/ncu_$2.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
