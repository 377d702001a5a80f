"""Summarise ncu outputs into profiles/ (run on the CPU box, no GPU needed).

    python tools/ncu_summary.py r01 [config]

reads gpurun_out/<R>_launches.csv (gpu__time_duration per launch) and
gpurun_out/<R>_full.ncu-rep (--set full), writes
profiles/<R>_launches.md, profiles/<R>_ncu_full.md and updates
profiles/traffic.json[config][kernel] = DRAM bytes (read + write) per launch.
"""
import csv
import io
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import short_kernel_name  # noqa: E402

NCU = "/usr/local/cuda/bin/ncu"


def short(name):
    return short_kernel_name(name) or name.split("(")[0][:48]


def launches(r):
    path = os.path.join(ROOT, "gpurun_out", f"{r}_launches.csv")
    rows = list(csv.reader(open(path)))
    hi = [i for i, x in enumerate(rows) if "Kernel Name" in x][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = {}
    order = []
    for x in rows[hi + 1:]:
        nm = x[ki]
        mine = ("i4::" in nm or "nvjet" in nm or short_kernel_name(nm) is not None)
        if not mine:
            continue
        v = float(x[vi].replace(",", ""))
        unit = x[ui]
        us = v / 1000.0 if unit == "ns" else (v if unit == "us" else v * 1000.0)
        key = "cuBLAS bf16: " + nm[:40] if "nvjet" in nm else short(nm)
        if key not in per:
            order.append(key)
        per.setdefault(key, []).append(us)
    ours = [k for k in order if not k.startswith("cuBLAS")]
    if STEP:                                   # a one-step capture (tools/stack_step.py): totals per kernel
        tot = sum(sum(per[k]) for k in ours)
        lines = [f"# {r}: ncu launch list of ONE step of {CONFIG} (`--metrics gpu__time_duration.sum --clock-control none`)",
                 "", "Command: `ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none "
                 f"python tools/stack_step.py {CONFIG}` (the bench step: every forward, then every backward in "
                 "reverse layer order, PDL on, eager launches).  Per-launch times under ncu are cold-cache and "
                 "serialised: compare SHARES with the bench's CUPTI breakdown, not absolutes.", "",
                 "| kernel | launches | total us | median us | share of the step |", "|---|---|---|---|---|"]
        for k in ours:
            lines.append(f"| {k} | {len(per[k])} | {sum(per[k]):.1f} | {statistics.median(per[k]):.1f} | "
                         f"{sum(per[k]) / tot:.3f} |")
        lines.append(f"| **sum of our kernels per step** | | **{tot:.1f}** | | 1.000 |")
        return "\n".join(lines) + "\n", {k: sum(per[k]) for k in ours}
    tot = sum(statistics.median(per[k]) for k in ours)
    lines = [f"# {r}: ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`)", "",
             f"Command: `ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 3 "
             f"--warmup 1 --no-cpu-baseline --no-e2e --config {CONFIG}` (fwd + bwd).  Per-launch times under ncu are "
             "cold-cache and serialised: compare SHARES with the bench's CUPTI breakdown, not absolutes.", "",
             "| kernel | launches | median us | share of our step |", "|---|---|---|---|"]
    for k in order:
        med = statistics.median(per[k])
        share = f"{med / tot:.3f}" if k in ours else "-"
        lines.append(f"| {k} | {len(per[k])} | {med:.1f} | {share} |")
    lines.append(f"| **sum of our kernels per step** | | **{tot:.1f}** | 1.000 |")
    return "\n".join(lines) + "\n", {k: statistics.median(per[k]) for k in ours}


WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_%",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_%",
    "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed": "int8_tensor_%",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_%",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}


def full(r):
    rep = os.path.join(ROOT, "gpurun_out", f"{r}_full.ncu-rep")
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    ni = h.index("Kernel Name")
    res = []
    for x in rows[2:]:
        d = {"kernel": short(x[ni])}
        for m, key in WANT.items():
            if m in h:
                i = h.index(m)
                try:
                    v = float(x[i].replace(",", ""))
                except ValueError:
                    continue
                d[key] = v * UNIT_SCALE.get(units[i], 1)
        res.append(d)
    cmd = (f"ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:\"grad_split|"
           f"gemm_i8|hadamard_quant|lss_sampler|compact\" -s 213 -c 12 python tools/stack_step.py {CONFIG}` "
           "(one layer's three backwards, in backward order FFN-down, FFN-up, QKV, inside the one-step run)"
           if STEP else
           f"ncu --set full --clock-control none --import-source on -k regex:\"grad_split|gemm_i8|hadamard_quant|"
           f"lss_sampler|compact\" -s 7 -c 7 python bench.py --steps 1 --warmup 1 --config {CONFIG} ...` "
           "(tools/profile_round.sh)")
    lines = [f"# {r}: ncu --set full (one launch each, cold cache, --clock-control none)", "",
             "Command: `" + cmd + ".  DRAM write bytes stay in L2 within one replayed launch.", "",
             "| kernel | us | DRAM read MB | DRAM write MB | DRAM % | L2 % | INT8 tensor % | issue active % | warps active % | regs | grid x block |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for d in res:
        lines.append("| {kernel} | {du:.1f} | {dr:.2f} | {dw:.2f} | {dp:.1f} | {lp:.1f} | {tp} | {ia:.1f} | {wa:.1f} | {rg:.0f} | {gr:.0f} x {bl:.0f} |".format(
            kernel=d["kernel"], du=d.get("duration", 0), dr=d.get("dram_read", 0) / 1e6, dw=d.get("dram_write", 0) / 1e6,
            dp=d.get("dram_%", 0), lp=d.get("l2_%", 0),
            tp=f"{d['int8_tensor_%']:.1f}" if d.get("int8_tensor_%") else "-",
            ia=d.get("issue_active_%", 0), wa=d.get("warps_active_%", 0), rg=d.get("regs", 0),
            gr=d.get("grid", 0), bl=d.get("block", 0)))
    return "\n".join(lines) + "\n", res


CONFIG = sys.argv[2] if len(sys.argv) > 2 else "cfg2_bert_base_ffn1"
STEP = "--step" in sys.argv


def main():
    r = sys.argv[1] if len(sys.argv) > 1 else "r01"
    config = CONFIG
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    md, _ = launches(r)
    open(os.path.join(ROOT, "profiles", f"{r}_launches.md"), "w").write(md)
    if not os.path.exists(os.path.join(ROOT, "gpurun_out", f"{r}_full.ncu-rep")):
        print(open(os.path.join(ROOT, "profiles", f"{r}_launches.md")).read())
        return
    md, res = full(r)
    open(os.path.join(ROOT, "profiles", f"{r}_ncu_full.md"), "w").write(md)
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    t = traffic.setdefault(config, {})
    for d in res:
        if "dram_read" in d:
            t[d["kernel"]] = int(d["dram_read"] + d.get("dram_write", 0))
    traffic["_note"] = ("DRAM bytes (read + write) per launch from one ncu --set full capture "
                        f"({r}); cold cache, so it includes the compulsory input reads")
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
    print(open(os.path.join(ROOT, "profiles", f"{r}_launches.md")).read())
    print(md)


if __name__ == "__main__":
    main()
