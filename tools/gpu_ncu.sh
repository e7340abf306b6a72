mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode -s 2 -c 1 -o gpurun_out/ncu_decode python tools/prof_kernels.py decode > gpurun_out/ncu_decode.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_prefill -s 1 -c 1 -o gpurun_out/ncu_prefill python tools/prof_kernels.py prefill > gpurun_out/ncu_prefill.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_power -s 1 -c 1 -o gpurun_out/ncu_power python tools/prof_kernels.py power > gpurun_out/ncu_power.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_decode -c 128 --csv --log-file gpurun_out/launches_decode.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-shapes > gpurun_out/ncu_launches.log 2>&1
echo done >> gpurun_out/status.txt
