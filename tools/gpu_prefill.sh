mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_forward.py -k "prefill or gemm" -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_prefill.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_prefill.log 2>&1; echo bench=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_prefill -s 1 -c 1 -o gpurun_out/ncu_prefill2 python tools/prof_kernels.py prefill > gpurun_out/ncu_prefill2.log 2>&1
