mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_admm.py -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_admm.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
for sz in "1024 1024 1.0" "4096 4096 1.0"; do timeout 900 python tools/admm_time.py $sz >> gpurun_out/admm_time.log 2>&1; done
echo admm=$? >> gpurun_out/status.txt
