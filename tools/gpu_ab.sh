# A/B two builds of the library on the bench: libnqb_a.so vs libnqb_b.so (copied over libnqb.so in turn);
# extra env for the b runs in $AB_ENV_B
mkdir -p gpurun_out
cp paper_2602_06694_b200/libnqb.so /tmp/libnqb_keep.so
for v in a b a b; do
  cp paper_2602_06694_b200/libnqb_$v.so paper_2602_06694_b200/libnqb.so
  if [ $v = b ]; then E="$AB_ENV_B"; else E=""; fi
  env $E timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-admm > gpurun_out/bench_$v.log 2>&1
  echo "== $v $E" >> gpurun_out/ab.txt
  python tools/show_bench.py gpurun_out/bench_$v.log 2>/dev/null | head -8 >> gpurun_out/ab.txt
done
cp /tmp/libnqb_keep.so paper_2602_06694_b200/libnqb.so
echo done >> gpurun_out/status.txt
