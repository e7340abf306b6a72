mkdir -p gpurun_out
timeout 300 python tools/trace_decode.py l7_q l70_gate l70_down > gpurun_out/trace.log 2>&1; echo trace=$? >> gpurun_out/status.txt
timeout 600 python -m pytest tests/test_gpu_decode.py -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_decode.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status.txt
