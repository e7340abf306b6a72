# A/B of decode-pass knobs: tools/gpu_pass_ab.sh "ENV=.. ENV=.." "..."   (AB_MODELS=7b,70b)
mkdir -p gpurun_out; : > gpurun_out/ab.log
for cfg in "$@"; do
  echo "== $cfg" >> gpurun_out/ab.log
  env $cfg timeout 300 python tools/pass_probe.py --models ${AB_MODELS:-7b} --no-graph --reps 10 > gpurun_out/ab_one.log 2>&1
  grep -v '^{' gpurun_out/ab_one.log | tail -3 >> gpurun_out/ab.log
  grep '^{' gpurun_out/ab_one.log | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print(d['model'], d['pass'])" >> gpurun_out/ab.log 2>&1
done
