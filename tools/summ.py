import json, sys
d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench.json"))
print("value %.1f TOPS  step %.1f us  speedup %.3f  bf16 %.1f us  gemm_frac %.3f" % (
    d["value"], d["ms_per_step"] * 1e3, d["speedup_vs_bf16_cublas"], d["bf16_cublas_ms_per_step"] * 1e3,
    d["gemm_int8_peak_frac"]))
for k, v in d["kernels"].items():
    print("  %-16s %6.1f us  %s" % (k, v["avg_us"], {a: round(b, 3) for a, b in v.items() if a.startswith("frac")}))
print("roofline", {k: d["roofline"][k] for k in ("kernel", "bound", "frac")}, "clocks", d["clocks"], "e2e", d.get("e2e", {}) and round(d["e2e"]["value"], 1))
