import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    ro = d.get("roofline") or {}
    sh = (d.get("extra") or {}).get("per_shape_single_layer", {})
    print(f, round(d["value"], 1), "frac", round(ro.get("frac", 0), 4), "us/launch",
          round(ro.get("us_per_launch", 0), 2), "e2e", round((d.get("e2e") or {}).get("value", 0), 1))
    for k, v in sh.items():
        print(f"   {k:16s} {v['us']:8.2f} us  {v['gbs']:8.1f} GB/s  frac {v['frac']:.3f}")
    for k, v in (d.get("extra") or {}).get("prefill_tcgen05", {}).items():
        print(f"   prefill {k:22s} {v['ms']:8.3f} ms  {v['tflops']:7.1f} TFLOP/s  frac {v['frac_of_bf16_peak']:.3f}")
