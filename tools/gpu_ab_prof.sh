# A/B of libnqb_a.so vs libnqb_b.so on the decode passes (gpu_pass_libab.sh) with
# the pass knobs from the environment; PROF=1 adds an ncu capture of the b pass.
export NQB_PASS_SPLIT=${NQB_PASS_SPLIT:-4} NQB_PASS_ITEM_SLABS=${NQB_PASS_ITEM_SLABS:-4}
bash tools/gpu_pass_libab.sh
cp paper_2602_06694_b200/libnqb_b.so paper_2602_06694_b200/libnqb.so
if [ -n "$PROF" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode_pass -s 2 -c 1 -o gpurun_out/prof_pass_$PROF python tools/prof_pass.py > gpurun_out/ncu_pass.log 2>&1; echo ncu=$?
fi
if [ -n "$BUSY" ]; then timeout 300 python tools/pass_busy.py --model 7b --blocks 16 2>&1 | grep -v Warn | grep -v nanmed; fi
cat gpurun_out/ab.log
