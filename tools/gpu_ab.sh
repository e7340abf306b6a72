mkdir -p gpurun_out
for d in 0 1 2 3; do
  echo "=== NQB_DEC_DBG=$d" >> gpurun_out/trace_dbg.log
  NQB_DEC_DBG=$d timeout 300 python tools/trace_decode.py l7_q >> gpurun_out/trace_dbg.log 2>&1
done
echo done >> gpurun_out/status.txt
