# Ring split / wave size grid on the tuned decode passes (7B, 70B): RING1_PCT:WAVE_DIV pairs from $GRID.
for t in ${GRID:-0:1 40:1 45:1 0:2 40:2}; do
  IFS=: read r d <<< "$t"
  printf "ring1=%s div1=%s: " $r $d
  NQB_PASS_RING1_PCT=$r NQB_PASS_WAVE_DIV=$d timeout 300 python tools/pass_probe.py --models ${MODELS:-7b,70b} --no-graph --reps 10 2>/dev/null | python -c "
import json,sys
print(' '.join('%s %.1f' % (d['model'], d['pass']['gbs']) for d in map(json.loads, sys.stdin)))"
done
