# ncu evidence for the decode kernel: launch list of one bench step + one full capture per shape.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_decode -c 128 --csv --log-file gpurun_out/launches_decode.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-shapes > gpurun_out/ncu_launches.log 2>&1
echo launches=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode -s 3 -c 1 -o gpurun_out/ncu_decode_l70gate python tools/prof_decode.py l70_gate > gpurun_out/ncu_decode.log 2>&1
echo full=$? >> gpurun_out/status.txt
