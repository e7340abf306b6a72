# A/B of the SVD power iteration's L2-resident share (NQB_POWER_L2_MB) on a 4096^2 matrix
mkdir -p gpurun_out
for mb in 0 60 80 100; do
  echo "== L2_MB=$mb" >> gpurun_out/l2ab.txt
  NQB_POWER_L2_MB=$mb NQB_POWER_PROF=1 timeout 300 python tools/power_prof.py 4096 4096 3 2>&1 | tail -4 >> gpurun_out/l2ab.txt
done
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p)" >> gpurun_out/l2ab.txt 2>&1
echo done >> gpurun_out/status.txt
