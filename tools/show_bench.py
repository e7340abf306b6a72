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
    for k, v in (d.get("extra") or {}).get("bitrate_sweep_l13_decode", {}).items():
        print(f"   sweep {k:18s} r={v['r']:5d} {v['us']:8.2f} us  {v['gbs']:8.1f} GB/s  frac {v['frac']:.3f}")
    ad = (d.get("extra") or {}).get("admm_init")
    if ad:
        print(f"   admm_init {ad['matrices']} x {ad['shape']} @{ad['bpw']}: {ad['seconds_max_rank']:.1f} s, "
              f"{ad['matrices_per_s']:.4f} matrices/s, err {ad['rel_error']}")
