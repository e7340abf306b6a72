for a in 0 1 2 4; do echo "== ahead=$a"; NQB_PASS_L2_AHEAD=$a timeout 300 python tools/pass_probe.py --models 7b,70b --no-graph --reps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print(d['model'], round(d['pass']['gbs'],1), round(d['pass']['us'],1))"; done
