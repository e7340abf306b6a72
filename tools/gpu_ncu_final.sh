# ncu evidence for the final kernels: decode launch list (bench step) + full captures of
# the decode (70B gate), prefill pair (70B q stage 2) and power-iteration kernels.
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_decode -c 128 --csv --log-file gpurun_out/launches_decode.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-shapes --no-admm > gpurun_out/ncu_launches.log 2>&1; echo launches=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none -k regex:k_decode -s 3 -c 1 -o gpurun_out/ncu_decode_final python tools/prof_kernels.py decode > gpurun_out/ncu_d.log 2>&1; echo decode=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none -k regex:k_prefill2 -s 1 -c 1 -o gpurun_out/ncu_prefill_final python tools/prof_kernels.py prefill > gpurun_out/ncu_p.log 2>&1; echo prefill=$? >> gpurun_out/status.txt
timeout 900 ncu --set full --clock-control none -k regex:k_power_stream -s 1 -c 1 -o gpurun_out/ncu_power_final python tools/prof_kernels.py power > gpurun_out/ncu_w.log 2>&1; echo power=$? >> gpurun_out/status.txt
