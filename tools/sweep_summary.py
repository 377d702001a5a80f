"""One line per gpurun_out/<tag>sweep_*.json: step us, cuBLAS us, speedup, kernel us."""
import glob, json, sys
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for f in sorted(glob.glob(f"gpurun_out/{tag}sweep_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "FAILED", e); continue
    ks = {k: round(v["us_per_step"], 1) for k, v in d["kernels"].items()}
    print(f"{f.split('sweep_')[1][:-5]:34s} {d['ms_per_step']*1e3:8.1f} us  bf16 {d['bf16_cublas_ms_per_step']*1e3:7.1f}  x{d['speedup_vs_bf16_cublas']:.3f}  {ks}")
