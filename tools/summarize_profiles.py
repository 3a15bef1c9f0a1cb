"""Summaries for profiles/: launch-list shares and --set full metrics.

    python tools/summarize_profiles.py <tag> <outtag>
reads gpurun_out/<tag>_launches_*.csv, gpurun_out/<tag>_*_full.ncu-rep,
gpurun_out/<tag>_bench_*.json; writes profiles/<outtag>_*."""
import csv
import io
import json
import re
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

tag, out = sys.argv[1], sys.argv[2]
G = Path("gpurun_out")
P = Path("profiles")
P.mkdir(exist_ok=True)


def short(name):
    m = re.search(r"(\w+_kernel)", name)
    return m.group(1) if m else name[:40]


lines = []
for f in sorted(G.glob(f"{tag}_launches_*.csv")):
    wl = f.stem.split("_launches_")[1]
    shutil.copy(f, P / f"{out}_launches_{wl}.csv")
    txt = f.read_text().splitlines()
    body = [l for l in txt if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(body))))
    h = rows[0]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(d["Kernel Name"])
        if not k.endswith("_kernel") or "distribution" in d["Kernel Name"] or "at::" in d["Kernel Name"]:
            continue
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"]) / 1e3  # ns -> us
    tot = sum(v[1] for v in agg.values())
    lines.append(f"## Launch list `{out}_launches_{wl}.csv` (ncu gpu__time_duration, cold, serialised)\n")
    lines.append("| kernel | launches | total us | share of library time |")
    lines.append("|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
    lines.append("")

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 inst %"),
        ("launch__registers_per_thread", "regs"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__occupancy_limit_shared_mem", "CTA/SM (smem)")]
for rep in sorted(G.glob(f"{tag}_*_full.ncu-rep")):
    wl = rep.stem[len(tag) + 1:-len("_full")]
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    lines.append(f"## `ncu --set full` ({wl}, one launch each; `{out}_ncu_full_{wl}.txt`)\n")
    lines.append("| kernel | " + " | ".join(n for _, n in KEYS) + " |")
    lines.append("|---" * (len(KEYS) + 1) + "|")
    for r in rows[2:]:
        d = dict(zip(h, r))
        cells = []
        for k, _ in KEYS:
            if k in h:
                cells.append(f"{d.get(k, '')} {u[h.index(k)]}".strip())
            else:
                cells.append("-")
        lines.append(f"| {short(d['Kernel Name'])} | " + " | ".join(cells) + " |")
    lines.append("")
    det = subprocess.run(["ncu", "-i", str(rep), "--page", "details"], capture_output=True,
                         text=True).stdout
    (P / f"{out}_ncu_full_{wl}.txt").write_text(det)

# text exports made on the GPU box (tools/ncu_full.sh): details pages and per-launch DRAM bytes
for f in sorted(G.glob(f"{tag}_ncu_full_*.txt")):
    shutil.copy(f, P / f.name.replace(tag, out, 1))
for f in sorted(G.glob(f"{tag}_ncu_dram_*.csv")):
    shutil.copy(f, P / f.name.replace(tag, out, 1))
    rows = list(csv.reader(open(f)))
    if len(rows) < 3:
        continue
    h, un = rows[0], dict(zip(rows[0], rows[1]))
    wl = f.stem.split("_ncu_dram_")[1]
    lines.append(f"## DRAM traffic per launch (`{f.name.replace(tag, out, 1)}`, ncu --set full, {wl})\n")
    lines.append(f"| kernel | grid | DRAM read {un['dram__bytes_read.sum']} | DRAM write "
                 f"{un['dram__bytes_write.sum']} | duration {un['gpu__time_duration.sum']} |")
    lines.append("|---|---|---|---|---|")
    for r in rows[2:]:
        d = dict(zip(h, r))
        lines.append(f"| {short(d['Kernel Name'])} | {d['Grid Size']} | {float(d['dram__bytes_read.sum']):.3f} | "
                     f"{float(d['dram__bytes_write.sum']):.3f} | {float(d['gpu__time_duration.sum']):.3f} |")
    lines.append("")

benches = []
for f in sorted(G.glob(f"{tag}_bench_*.json")):
    wl = f.stem.split("_bench_")[1]
    L = [l for l in f.read_text().splitlines() if l.startswith("{")]
    if not L:
        continue
    shutil.copy(f, P / f"{out}_bench_{wl}.json")
    d = json.loads(L[-1])
    e = d.get("e2e") or {}
    rf = d.get("roofline") or {}
    cb = d.get("cpu_baseline") or {}
    benches.append(f"| {wl} | {d['ms_per_step']:.3f} | {d['value']:.4g} | {e.get('ms_per_step', 0):.2f} | "
                   f"{e.get('value', 0):.4g} | {cb.get('value', 0):.4g} ({cb.get('cores')} cores) | "
                   f"{rf.get('kernel', '-')} {rf.get('frac', 0):.3f} |")
hdr = [f"# Profiles {out} (1x B200; bench lines, ncu launch lists, ncu --set full exports)\n",
       "| workload | ms/step (device) | points/s | e2e ms/step | e2e points/s | CPU oracle points/s | roofline kernel, frac |",
       "|---|---|---|---|---|---|---|"] + benches + [""]
(P / f"{out}_summary.md").write_text("\n".join(hdr + lines) + "\n")
print("\n".join(hdr + lines))
