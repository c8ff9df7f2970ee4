import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    r = d["roofline"]; c = d["config"]
    print(f, f"value {d['value']:.0f} ms/step {d['ms_per_step']:.4f} ufi_mix {c.get('ufi_mix')} dom {r['kernel'][-22:]} {r['kernel_us']:.2f}us plan {c['plan']} e2e {d['e2e']['value']:.0f} multi {d.get('multistream',{}).get('value',0):.0f} plan_s {d['plan_seconds']:.1f}")
    if "baselines" in d:
        b = d["baselines"]; print("   geo cusparse %.3f cublas %.3f tf32 %.3f csr %s" % (b["geomean_speedup_vs_cusparse"], b["geomean_speedup_vs_cublas"], b["geomean_speedup_vs_cublas_tf32"], b["geomean_speedup_vs_csr_walk"]))
