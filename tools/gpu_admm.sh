mkdir -p gpurun_out
for sz in "512 512 1.0" "1024 1024 1.0" "2048 2048 1.0"; do timeout 900 python tools/admm_time.py $sz >> gpurun_out/admm_time.log 2>&1; done
timeout 1500 python tools/admm_time.py 4096 4096 1.0 >> gpurun_out/admm_time.log 2>&1
echo done >> gpurun_out/status.txt
