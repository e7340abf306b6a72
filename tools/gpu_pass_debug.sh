# Decode-pass skeleton rates: NQB_PASS_DEBUG bits (1 skip MMA, 2 skip quantise,
# 8 skip publish/outputs, 32 no weight copies) on the 7B / 70B passes.
export NQB_PASS_SPLIT=${NQB_PASS_SPLIT:-4} NQB_PASS_ITEM_SLABS=${NQB_PASS_ITEM_SLABS:-4}
for d in ${DEBUGS:-0 1 33 2 8 11}; do
  echo "== debug=$d"
  NQB_PASS_DEBUG=$d timeout 300 python tools/pass_probe.py --models ${MODELS:-7b,70b} --no-graph --reps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print(d['model'], round(d['pass']['gbs'],1), round(d['pass']['us'],1))"
done
