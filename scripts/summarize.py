import json, sys, glob, os
for f in sorted(glob.glob(os.path.join(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out", "bench_c*.json"))):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    r = d["roofline"]
    print(os.path.basename(f), "MPix/s=%.0f ms/step=%.4f pass_frac=%s filter_frac=%.3f pass_ms=%s clk=%s" % (
        d["value"], d["ms_per_step"], r["frac"] and round(r["frac"], 3), r["filter_frac"], r["pass_ms"] and round(r["pass_ms"], 4), d["clocks"]["sm_mhz"]))
    kk = d.get("kernels_instrumented") or d.get("kernels") or {}
    print("   ", {k: (round(v.get("ms_per_step_instrumented", v.get("ms_per_step", 0)), 4), round(v["share"], 2)) for k, v in kk.items()})
    if d.get("e2e"): print("    e2e %.0f MPix/s %.3f ms" % (d["e2e"]["value"], d["e2e"]["ms_per_step"]))
    if d.get("cpu_baseline"): print("    cpu", d["cpu_baseline"])
