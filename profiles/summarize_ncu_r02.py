"""Summarise the round-2 ncu captures (profiles/run_ncu_r02.sh output in gpurun_out/ncu_r02) into
profiles/r02_ncu_summary.md and profiles/traffic.json (per-launch DRAM bytes of every kernel group,
stamped with the git sha of the capture).

    python profiles/summarize_ncu_r02.py [capture_dir] [git_sha]
"""

import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from bench import Model, laplace3d_nnz  # noqa: E402

D = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "gpurun_out" / "ncu_r02"
SHA = sys.argv[2] if len(sys.argv) > 2 else subprocess.run(["git", "-C", str(ROOT), "rev-parse", "--short=12", "HEAD"],
                                                          capture_output=True, text=True).stdout.strip()
PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
    else 6543.1

n, nl, nu = laplace3d_nnz(256, 256, 256)
mod = Model(n, nl, nu)
mst = Model(n, nl, nu, stencil=True)  # stencil-encoded triangles: 32 B of lane masks per slice
V = mod.V

UNIT = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "byte": 1.0, "Kbyte": 1e3,
        "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9}


def fnum(v, u):
    return float(v.replace(",", "")) * UNIT.get(u, 1.0)


# ---- A: every launch of the region (duration, DRAM bytes)
rows = list(csv.reader(open(D / "region_metrics.csv")))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hi]
ci = {h: i for i, h in enumerate(hdr)}
launches = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) < len(hdr):
        continue
    key = (int(r[ci["ID"]]), r[ci["Kernel Name"]])
    launches.setdefault(key, {})[r[ci["Metric Name"]]] = fnum(r[ci["Metric Value"]], r[ci["Metric Unit"]])


def short(k):
    return k.split("(")[0].replace("void ", "").replace("rs::", "")


groups = collections.OrderedDict()
for (i, k), m in launches.items():
    g = groups.setdefault(short(k), {"launches": 0, "s": 0.0, "rd": 0.0, "wr": 0.0, "l2": 0.0})
    g["launches"] += 1
    g["s"] += m["gpu__time_duration.sum"]
    g["rd"] += m["dram__bytes_read.sum"]
    g["wr"] += m["dram__bytes_write.sum"]
    g["l2"] += 32.0 * m.get("lts__t_sectors.sum", 0.0)

# algorithmic bytes per launch (SURVEY §8(d) per-row figures x rows; 256^3)
ML = mod.ML
MS = mst.ML
model = {
    "k_st_resid<double, 1, 3, double, 0>": ("stencil GS2 pass 0: rd = (b - Ax)/d", MS + mst.MU + 4 * V),
    "k_st_resid<double, 1, 3, double, 1>": ("stencil GS2 pass 0 + fused ||r||^2 partials (smoother)",
                                            MS + mst.MU + 4 * V),
    "k_st_inner<double, 2, 0, 3, double>": ("stencil GS2 inner step, last, x += w g", MS + 3 * V),
    "k_st_resid<double, 2, 3, double, 0>": ("stencil JR sweep", MS + mst.MU + 4 * V),
    "k_st_resid<double, 0, 3, double, 0>": ("stencil SpMV y = Ax", mst.spmv()),
    "k_st_inner<double, 1, 0, 3, double>": ("stencil precond inner step, z = w g", MS + 2 * V),
    "k_st_inner<float, 1, 0, 3, double>": ("stencil fp32 precond inner, z = (double)(w g)", MS + V // 2 + V),
    "k_st_prec1<double, double, double, 0, 3>": ("stencil zero-start GS2(1,1,1) preconditioner, one pass",
                                                 MS + 3 * V),
    "k_st_prec1<float, double, double, 0, 3>": ("stencil fp32-inside-fp64 GS2(1,1,1) preconditioner, one pass",
                                                MS + 2 * V + V // 2),
    "k_st_mt<double, 3>": ("stencil MT-GS colour pass (all rows' b, d, x read: colours interleave; the colour's x "
                           "written)", MS + mst.MU + 3 * V + V // 2),
    "k_resid_tma<double, 1>": ("explicit GS2 pass 0 (TMA col/val)", ML + mod.MU + 4 * V),
    "k_resid_tma<double, 2>": ("explicit JR sweep (TMA col/val)", ML + mod.MU + 4 * V),
    "k_resid_tma<double, 0>": ("explicit SpMV (TMA col/val)", mod.spmv()),
    "k_resid<double, 1, 0>": ("GS2 pass 0: r = b - Ax, rd = r/d", ML + mod.MU + 4 * V),
    "k_resid<double, 1, 1>": ("GS2 pass 0 + fused ||r||^2 (smoother)", ML + mod.MU + 4 * V),
    "k_resid<double, 2, 0>": ("JR sweep: x' = x + w(b - Ax)/d", ML + mod.MU + 4 * V),
    "k_resid<double, 0, 0>": ("SpMV y = Ax", mod.spmv()),
    "k_inner<double, 1, 0>": ("GS2 inner step, last, x += w g", ML + 3 * V),
    "k_inner<double, 2, 0>": ("precond inner step, z = w g", ML + 2 * V),
    "k_scale_rd_f64x2": ("precond pass: rd = r/d", 3 * V),
    "k_scale_rd_f32x2": ("fp32 precond: rd = (float)r/d", V + V // 2 + V // 2),
    "k_inner_out_nr<float, double, 0, 2, 0>": ("fp32 precond inner, z = (double)(w g)",
                                               8 * nl + 4 * (n + 1) + V // 2 + V),
    "k_mt_color<double>": ("MT-GS colour pass (2 colours / sweep)", (ML + mod.MU + 3 * V) / 2),
    "k_spmv_red<1>": ("||b - Ax||^2, nothing stored", ML + mod.MU + 3 * V),
    "k_cgs<0, 1, 0, 1>": ("DCGS2 dual dots + coefficients (k = 1..60)", None),
    "k_cgs<1, 0, 1, 1>": ("DCGS2 update (k = 1..60)", None),
}
traffic = {"git_sha": SHA, "capture": "profiles/run_ncu_r02.sh A (ncu --metrics, --clock-control none, cold L2 per launch)",
           "grid": "laplace3d 256^3"}
lines = ["# ncu summary, round 2 (HEAD " + SHA + ")", "",
         "Captures: `profiles/run_ncu_r02.sh` on one B200 (`--clock-control none`; every launch replayed "
         "cold-cache and serialised, so absolute times are the kernel alone at full clock, not the "
         "power-capped in-cycle times of bench.py). Workload: `profiles/ncu_kernels.py` (laplace3d "
         "256^3: the sweep table once -- stencil-encoded triangles, then the streaming passes again on the "
         "explicit SELL-32 slots -- then one GMRES(60) cycle). Algorithmic bytes: SURVEY §8(d) per-row "
         "figures x rows; stencil-encoded triangles: the 32-B lane-mask row of each 32-row slice instead of "
         "the split-CSR bytes (uniform-width explicit slices read no slice pointers: 4(n+1) B per triangle "
         "less). L2 slice traffic = 32 B x lts__t_sectors (hits, misses and writes).", "",
         f"Roofline denominator: {PEAK} GB/s (MEASURED_PEAKS.json, copy).", "",
         "| kernel | computes | launches | avg us | DRAM read+write per launch (GB) | algorithmic (GB) | "
         "DRAM / algorithmic | achieved GB/s (DRAM) | frac | L2 slice traffic (GB) | L2 TB/s |",
         "|---|---|---|---|---|---|---|---|---|---|---|"]
for name, g in groups.items():
    if name not in model:
        continue
    what, alg = model[name]
    cnt = g["launches"]
    t = g["s"] / cnt
    dram = (g["rd"] + g["wr"]) / cnt
    if alg is None:  # DCGS2: sum over k of the per-k figures
        alg_tot = sum(mod.dcgs_dots(k) if "0, 1, 0, 1" in name else mod.dcgs_update(k) for k in range(1, cnt + 1))
        alg = alg_tot / cnt
    gbs = dram / t / 1e9
    l2 = g["l2"] / cnt
    lines.append(f"| `{name}` | {what} | {cnt} | {t * 1e6:.1f} | {dram / 1e9:.4f} | {alg / 1e9:.4f} | "
                 f"{dram / alg:.3f} | {gbs:.0f} | {gbs / PEAK:.3f} | {l2 / 1e9:.3f} | {l2 / t / 1e12:.1f} |")
    traffic[name] = {"launches": cnt, "avg_us": round(t * 1e6, 2), "dram_read": g["rd"] / cnt,
                     "dram_write": g["wr"] / cnt, "model_bytes": alg, "l2_bytes": l2}
# bench.py kernel groups (roofline.traffic): the DCGS2 groups
for grp, name in (("dcgs_dots", "k_cgs<0, 1, 0, 1>"), ("dcgs_update", "k_cgs<1, 0, 1, 1>"),
                  ("spmv", "k_st_resid<double, 0, 3, double, 0>"), ("precond", "k_st_prec1<double, double, double, 0, 3>")):
    if name in traffic:
        traffic[grp] = dict(traffic[name], kernel=name, capture=traffic["capture"])
lv = groups.get("k_mt_color_pdl<double>")
cta = groups.get("k_gs_levels_cta<double, 0>")
if lv:
    tot = lv["rd"] + lv["wr"] + (cta["rd"] + cta["wr"] if cta else 0)
    alg = ML + mod.MU + 3 * V
    lines += ["", f"Level-scheduled GS (one forward sweep): {lv['launches']} per-level launches "
                  f"(`k_mt_color_pdl`) + {cta['launches'] if cta else 0} single-CTA runs; DRAM "
                  f"{tot / 1e9:.2f} GB vs {alg / 1e9:.2f} GB algorithmic ({tot / alg:.1f}x: b, d and x are "
                  f"gathered by row id, one 32-B sector per 8-B value, along each level's anti-diagonal "
                  f"plane); serialised time {(lv['s'] + (cta['s'] if cta else 0)) * 1e3:.2f} ms (in the bench, "
                  f"PDL-chained: ~3.2 ms)."]

# ---- B / C: full-set sections of the key kernels
for f, title in (("sweeps.raw.csv", "sweep-phase kernels"), ("dcgs_skip60.raw.csv", "DCGS2 at k = 31"),
                 ("dcgs_skip118.raw.csv", "DCGS2 at k = 60")):
    p = D / f
    if not p.exists():
        continue
    rows = list(csv.reader(open(p)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ci = {h: i for i, h in enumerate(hdr)}
    cols = [("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
            ("lts__t_sector_hit_rate.pct", "L2 hit %"),
            ("launch__registers_per_thread", "regs"),
            ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "long-sb stall / issue")]
    cols = [(c, t) for c, t in cols if c in ci]
    lines += ["", f"## {title} (`--set full`)", "",
              "| kernel | us | " + " | ".join(t for _, t in cols) + " |", "|---|---|" + "---|" * len(cols)]
    seen = collections.Counter()
    for r in data:
        k = short(r[ci["Kernel Name"]])
        seen[k] += 1
        if seen[k] > 2:
            continue
        t = fnum(r[ci["gpu__time_duration.sum"]], units[ci["gpu__time_duration.sum"]]) * 1e6
        lines.append(f"| `{k}` | {t:.1f} | " + " | ".join(r[ci[c]] for c, _ in cols) + " |")

(ROOT / "profiles" / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
(ROOT / "profiles" / "r02_ncu_summary.md").write_text("\n".join(lines) + "\n")
print("\n".join(lines))
