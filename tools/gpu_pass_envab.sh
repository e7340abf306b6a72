# A/B of decode-pass environment settings on one library: AB_ENV_A vs AB_ENV_B,
# alternating three times on the 7B and 70B passes.
for v in A B A B A B; do
  if [ $v = A ]; then e="$AB_ENV_A"; else e="$AB_ENV_B"; fi
  echo "== $v ($e)"
  env $e timeout 300 python tools/pass_probe.py --models ${MODELS:-7b,70b} --no-graph --reps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print(d['model'], round(d['pass']['gbs'],1))"
done
