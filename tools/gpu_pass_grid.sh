# Grid of decode-pass settings: MODEL:SPLIT:RING1_PCT[:PLAN_SLABS] from $GRID (empty = default).
for t in $GRID; do
  IFS=: read m s r ps <<< "$t"
  printf "%s split=%s ring1=%s plan_slabs=%s: " $m $s $r $ps
  NQB_PASS_PLAN_SLABS=$ps NQB_PASS_SPLIT=$s NQB_PASS_RING1_PCT=$r NQB_PASS_VERBOSE=1 timeout 300 python tools/pass_probe.py --models $m --no-graph --reps 10 2>/tmp/v.txt | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print(round(d['pass']['gbs'],1))"
  grep "nqb pass: K" /tmp/v.txt | sed 's/.*partitions=/   partitions=/'
done
