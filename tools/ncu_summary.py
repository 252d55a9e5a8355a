"""Summarise ncu outputs into profiles/ (run here, after gpurun brought them back).

    python tools/ncu_summary.py --launches gpurun_out/launches.csv \
        --rep gpurun_out/prof.ncu-rep --tag r1 [--bench gpurun_out/bench.log]

Writes profiles/<tag>_launches.md (per-kernel share of the launch list),
profiles/<tag>_ncu_full.md (key counters per captured launch) and merges the
per-launch DRAM bytes into profiles/ncu_summary.json (read by bench.py for
roofline.traffic).
"""
import argparse
import csv
import json
import subprocess
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"
UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
FAMILY = {"k_ex0_eval": "exh0", "k_lu0_probe": "local0", "k_lu0_finish": "local0", "k_moments": "local1"}


def short(name):
    base = name.split("(")[0]
    return base.split("::")[-1].strip() or name[:40]


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        us = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        k = short(r[ki])
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list ({tag}): `{path}`", "",
             "`gpu__time_duration.sum`, `--clock-control none`; per-launch times are cold-cache and",
             "serialised, so compare SHARES with the bench's phase split, not absolutes.", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {n} | {us / 1e3:.3f} | {100 * us / tot:.2f}% |")
    lines.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot / 1e3:.3f} | 100% |")
    (PROF / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
    return agg


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "sm__cycles_active.avg",
        "gpc__cycles_elapsed.max", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def full(rep, tag):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for w in WANT:
            if w in h:
                d[w] = (r[h.index(w)], units[h.index(w)])
        res.append(d)
    lines = [f"# ncu --set full ({tag}): `{rep}`", ""]
    for d in res:
        lines.append(f"## `{d['kernel']}`")
        lines += [f"- {k}: {v[0]} {v[1]}" for k, v in d.items() if k != "kernel"]
        lines.append("")
    (PROF / f"{tag}_ncu_full.md").write_text("\n".join(lines))
    return res


def to_bytes(v):
    val, unit = v
    val = float(val.replace(",", ""))
    return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--tag", required=True)
    ap.add_argument("--log2d", type=int, default=None, help="grid size of the captured run (for traffic)")
    args = ap.parse_args()
    PROF.mkdir(exist_ok=True)
    summ_path = PROF / "ncu_summary.json"
    summ = json.loads(summ_path.read_text()) if summ_path.exists() else {}
    if args.launches:
        agg = launches(args.launches, args.tag)
        summ.setdefault("launch_share", {})[args.tag] = {
            k: round(v[1] / sum(x[1] for x in agg.values()), 5) for k, v in agg.items()}
    for rep in args.rep:
        for d in full(rep, args.tag + "_" + Path(rep).stem):
            fam = FAMILY.get(d["kernel"].split("<")[0])
            if fam and args.log2d and "dram__bytes_read.sum" in d:
                b = to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"])
                if b == b:  # skip NaN captures
                    summ.setdefault(f"dram_bytes_per_launch_2p{args.log2d}", {})[fam] = b
                    summ.setdefault(f"dram_source_2p{args.log2d}", {})[fam] = f"{rep} ({args.tag})"
    summ_path.write_text(json.dumps(summ, indent=1) + "\n")
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
