mkdir -p gpurun_out
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_decode -s 3 -c 1 -o gpurun_out/prof_decode5 python tools/prof_decode.py l70_gate > gpurun_out/ncu_full.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
