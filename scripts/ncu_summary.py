#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, on the CPU box).

  python scripts/ncu_summary.py launches <launches.csv> <out.md>
  python scripts/ncu_summary.py full <prof.ncu-rep> <out.md> [--traffic profiles/ncu_traffic.json]

`launches`: the --metrics gpu__time_duration.sum launch list of one bench step
(cold-cache, serialised): per-kernel launches, time and share of the step.
`full`: per-launch key metrics of a --set full capture: duration, SM clock,
tensor-pipe activity, DRAM bytes, L2 hit rate.  The GEMM launches are mapped
to the step's row names by their order within one exit.
"""

import csv
import io
import json
import re
import subprocess
import sys
from collections import OrderedDict

# order of gemm_kernel launches within one MLP exit (api.cu; ds_mode recompute;
# no a12_du GEMM since the gain identity, A28)
MLP_GEMM_ORDER = ["a2_gateup_swiglu", "a3_down_resid", "a5_vocab_ce_stats", "a7_ds_recompute",
                  "a8_dz", "a9_dw_out", "a11_dm_swiglu_bwd", "a11_dw_down", "a12_dw_gateup"]


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "").replace("ee::", "")
    return name


def launches(path, out):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(txt)))
    agg = OrderedDict()
    total = 0.0
    gemm_idx = 0
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"])
        k = short(r["Kernel Name"])
        if k.startswith(("gemm_kernel", "gemm2_kernel")):
            k = f"{k} [{MLP_GEMM_ORDER[gemm_idx % len(MLP_GEMM_ORDER)]}]"
            gemm_idx += 1
        ours = not k.startswith("at::") and "elementwise" not in k and "distribution" not in k
        d = agg.setdefault(k, {"n": 0, "ns": 0.0, "ours": ours})
        d["n"] += 1
        d["ns"] += ns
    step = {k: v for k, v in agg.items() if v["ours"] and not k.startswith(("copy_cast", "fill", "random"))}
    total = sum(v["ns"] for v in step.values())
    lines = [f"# ncu launch list summary: `{path}`", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` over "
             "`bench.py --quick --steps 1 --warmup 0` (init + one 70B step). Per-launch times are "
             "cold-cache and serialised: compare shares, not absolutes.", "",
             "| kernel | launches | total ms | ms/launch | share of step |", "|---|---|---|---|---|"]
    for k, v in sorted(step.items(), key=lambda kv: -kv[1]["ns"]):
        lines.append(f"| {k} | {v['n']} | {v['ns']/1e6:.3f} | {v['ns']/v['n']/1e6:.3f} | "
                     f"{v['ns']/total:.4f} |")
    lines += ["", f"Step total (our kernels, excluding init): {total/1e6:.1f} ms", "",
              "Other launches (torch input generation / init): " +
              ", ".join(f"{k} x{v['n']}" for k, v in agg.items() if k not in step)]
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


METRICS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "launch__shared_mem_per_block_dynamic"]


def full(path, out, traffic_out=None):
    r = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    hdr, units = rows[0], rows[1]
    col = {m: hdr.index(m) for m in METRICS if m in hdr}
    kcol = hdr.index("Kernel Name")
    lines = [f"# ncu --set full summary: `{path}`", "",
             "| # | kernel | step row | ms | SM GHz | tensor pipe % | DRAM read GB | DRAM write GB | "
             "L2 hit % | L2 thru % | regs | grid |", "|" + "---|" * 12]
    traffic = {}
    gi = 0
    for i, row in enumerate(rows[2:]):
        k = short(row[kcol])
        tag = ""
        if k.startswith(("gemm_kernel", "gemm2_kernel")):
            tag = MLP_GEMM_ORDER[gi % len(MLP_GEMM_ORDER)]
            gi += 1

        def g(m, scale=1.0):
            if m not in col:
                return float("nan")
            v = row[col[m]].replace(",", "")
            try:
                return float(v) * scale
            except ValueError:
                return float("nan")
        ms = g("gpu__time_duration.sum")
        u = units[col["gpu__time_duration.sum"]]
        ms = ms / 1e6 if u == "ns" else (ms / 1e3 if u == "us" else ms)
        ghz = g("sm__cycles_elapsed.avg.per_second")
        dr, dw = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
        ur, uw = units[col["dram__bytes_read.sum"]], units[col["dram__bytes_write.sum"]]
        sc = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}
        dr *= sc.get(ur, 1.0)
        dw *= sc.get(uw, 1.0)
        if tag:
            traffic.setdefault(tag, (dr + dw) * 1e9)
        lines.append(f"| {i} | {k} | {tag} | {ms:.3f} | {ghz:.3f} | "
                     f"{g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
                     f"{dr:.2f} | {dw:.2f} | {g('lts__t_sector_hit_rate.pct'):.1f} | "
                     f"{g('lts__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{g('launch__registers_per_thread'):.0f} | {g('launch__grid_size'):.0f} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_out:
        old = {}
        try:
            old = json.load(open(traffic_out))
        except Exception:
            pass
        old.update(traffic)
        json.dump(old, open(traffic_out, "w"), indent=1)


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    t = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    (launches if mode == "launches" else full)(src, dst, *([t] if mode == "full" else []))
