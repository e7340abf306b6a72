mkdir -p gpurun_out; : > gpurun_out/ab.log
cp paper_2602_06694_b200/libnqb.so /tmp/libnqb_keep.so
for v in a b a b a b; do
  cp paper_2602_06694_b200/libnqb_$v.so paper_2602_06694_b200/libnqb.so
  echo "== $v" >> gpurun_out/ab.log
  timeout 300 python tools/pass_probe.py --models 7b,70b --no-graph --reps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print(d['model'], round(d['pass']['gbs'],1))" >> gpurun_out/ab.log 2>&1
done
cp /tmp/libnqb_keep.so paper_2602_06694_b200/libnqb.so
