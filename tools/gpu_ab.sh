mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_w16.log 2>&1
cp paper_2602_06694_b200/libnqb_w8.so paper_2602_06694_b200/libnqb.so
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_w8.log 2>&1
timeout 300 python tools/trace_decode.py l7_q l70_gate > gpurun_out/trace_w8.log 2>&1
echo done >> gpurun_out/status.txt
