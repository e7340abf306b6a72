# decode kernel: parity tests, bench, launch list, one full ncu capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_forward.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_decode.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_decode -c 256 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-shapes > gpurun_out/ncu_bench.log 2>&1; echo ncu_list=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode -s 1 -c 2 -o gpurun_out/prof_decode python tools/prof_decode.py l70_gate > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$? >> gpurun_out/status.txt
