"""Summarise ncu outputs brought back in gpurun_out/ into committed files under profiles/ (run here, no GPU).

    python tools/ncu_summary.py --tag r1 --launches gpurun_out/r1_launches.csv \
        --rep stream=gpurun_out/r1_stream.ncu-rep --rep select=gpurun_out/r1_select.ncu-rep [--config cfg3]

Writes profiles/<tag>_launches.md (per-kernel launch list: count, mean/min/max device time, share of the step) and
profiles/<tag>_ncu_<name>.md (key metrics of each --set full capture), and merges the per-launch DRAM traffic of the
dominant kernel into profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import statistics
import subprocess
from collections import OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PROF = ROOT / "profiles"
OURS = ("tetris::",)
# with an ncu -k filter the names come without their namespace: accept the library's kernel names as such
OUR_KERNELS = ("select1_kernel", "select_kernel", "gselect_kernel", "persist_stream_kernel", "finalize_kernel",
               "persist_greedy_kernel", "greedy_rowmap_kernel", "greedy_kernel", "compact_kernel", "pre_accept_kernel",
               "accept_kernel", "sample_kernel", "uniform_windows_kernel", "sim_step_kernel")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak (ncu nominal)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_dim_x", "cluster x"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "instructions"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long scoreboard"),
]


def launches(path: Path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", ""))
        unit = r[ui]
        us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        out.append((r[ki], us))
    return out


def short(name: str) -> str:
    return name.split("(")[0].replace("void ", "")


def launch_table(path: Path, tag: str) -> str:
    ls = [(short(n), us) for n, us in launches(path)
          if any(o in n for o in OURS) or short(n).split("<")[0] in OUR_KERNELS]
    # drop the first quarter (warm-up / set-up launches) when there are many
    groups: "OrderedDict[str, list]" = OrderedDict()
    for n, us in ls:
        groups.setdefault(n, []).append(us)
    tot = sum(statistics.mean(v) for v in groups.values())
    lines = [f"# {tag}: launch list (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
             f"Source: `{path.name}` (cold-cache, serialised replays: compare shares, not absolutes).", "",
             "| kernel | launches | mean µs | min µs | max µs | share of per-step sum |",
             "|---|---|---|---|---|---|"]
    for n, v in groups.items():
        m = statistics.mean(v)
        lines.append(f"| `{n}` | {len(v)} | {m:.2f} | {min(v):.2f} | {max(v):.2f} | {m / tot:.1%} |")
    lines += ["", f"Sum of per-kernel means (one of each): {tot:.1f} µs.", "", "Last launches in order:", "",
              "```"] + [f"{n:60s} {us:9.2f} us" for n, us in ls[-12:]] + ["```", ""]
    return "\n".join(lines)


def raw_metrics(rep: Path):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    units = rows[1]
    recs = []
    for r in rows[2:]:
        rec = {"Kernel Name": r[h.index("Kernel Name")]}
        for key, _ in KEYS:
            if key in h:
                i = h.index(key)
                rec[key] = (r[i], units[i])
        recs.append(rec)
    return recs


def to_bytes(v, unit):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def rep_table(rep: Path, name: str, tag: str):
    recs = raw_metrics(rep)
    lines = [f"# {tag}: ncu --set full of `{short(recs[0]['Kernel Name'])}`", "",
             f"Source: `{rep.name}` (`ncu --set full --clock-control none --import-source on`), {len(recs)} launches.",
             "", "| metric | " + " | ".join(f"launch {i}" for i in range(len(recs))) + " |",
             "|---|" + "---|" * len(recs)]
    for key, label in KEYS:
        if key not in recs[0]:
            continue
        vals = [f"{r[key][0]} {r[key][1]}".strip() for r in recs]
        lines.append(f"| {label} (`{key}`) | " + " | ".join(vals) + " |")
    traffic = [to_bytes(*r["dram__bytes_read.sum"]) + to_bytes(*r["dram__bytes_write.sum"]) for r in recs]
    dur = [float(r["gpu__time_duration.sum"][0].replace(",", "")) for r in recs]
    dunit = recs[0]["gpu__time_duration.sum"][1]
    dur_s = [d * {"usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3}.get(dunit, 1e-6) for d in dur]
    bw = [t / s / 1e9 for t, s in zip(traffic, dur_s)]
    lines += ["", f"DRAM traffic per launch (read+write): {statistics.mean(traffic) / 1e6:.1f} MB; "
                  f"traffic / duration = {statistics.mean(bw):.0f} GB/s.", ""]
    return "\n".join(lines), statistics.mean(traffic)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[], help="name=path.ncu-rep")
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--dominant", default="stream", help="--rep name whose traffic goes to ncu_traffic.json")
    a = ap.parse_args()
    PROF.mkdir(exist_ok=True)
    if a.launches:
        (PROF / f"{a.tag}_launches.md").write_text(launch_table(Path(a.launches), a.tag))
    tj = PROF / "ncu_traffic.json"
    traffic = json.loads(tj.read_text()) if tj.exists() else {}
    for spec in a.rep:
        name, path = spec.split("=", 1)
        md, tr = rep_table(Path(path), name, a.tag)
        (PROF / f"{a.tag}_ncu_{name}.md").write_text(md)
        if name == a.dominant:
            traffic[a.config] = tr
    tj.write_text(json.dumps(traffic, indent=1) + "\n")


if __name__ == "__main__":
    main()
