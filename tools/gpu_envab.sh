# A/B of one library under two environments: $AB_ENV_A vs $AB_ENV_B (bench, twice each)
mkdir -p gpurun_out
for v in a b a b; do
  if [ $v = b ]; then E="$AB_ENV_B"; else E="$AB_ENV_A"; fi
  env $E timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-admm > gpurun_out/bench_$v.log 2>&1
  echo "== $v $E" >> gpurun_out/ab.txt
  python tools/show_bench.py gpurun_out/bench_$v.log 2>/dev/null | head -8 >> gpurun_out/ab.txt
done
echo done >> gpurun_out/status.txt
