# A/B of decode-pass knobs: SM partitions (NQB_PASS_SPLIT), work-item slabs
# (NQB_PASS_ITEM_SLABS), stage-1 warps (NQB_PASS_WARPS1) on the 7B / 70B passes,
# then the consumer phase split (tools/pass_busy.py) of the 7B pass.
if [ -n "$TESTS" ]; then timeout 600 python -m pytest tests/test_gpu_pass.py -x -q -m gpu 2>&1 | tail -15; fi
for s in ${SPLITS:-1 2 4}; do
  for it in ${ITEMS:-6}; do
    for w in ${WARPS:-0}; do
      echo "== split=$s items=$it warps1=$w"
      NQB_PASS_ITEM_SLABS=$it NQB_PASS_WARPS1=$w NQB_PASS_VERBOSE=1 NQB_PASS_SPLIT=$s timeout 300 python tools/pass_probe.py --models ${MODELS:-7b,70b} --no-graph 2>&1 | grep -v "^$" | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['model'], 'GB/s %.0f frac %.3f' % (d['pass']['gbs'], d['pass']['frac']))
    else:
        print(l.rstrip())"
    done
  done
done
for s in ${BUSY_SPLITS:-}; do
  for m in ${BUSY_MODELS:-7b}; do
    NQB_PASS_SPLIT=$s timeout 300 python tools/pass_busy.py --model $m --blocks ${BUSY_BLOCKS:-8} 2>&1 | grep -v Warning | grep -v nanmedian
  done
done
