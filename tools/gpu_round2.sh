# Round-end style validation plus prefill ncu evidence.
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
bash tools/gpu_round.sh
timeout 600 ncu --set full --clock-control none -k regex:k_prefill2 -s 1 -c 1 -o gpurun_out/ncu_prefill_pair python tools/prof_kernels.py prefill > gpurun_out/ncu_prefill_pair.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
