#!/usr/bin/env python
"""Summarise ncu evidence from gpurun_out/ into profiles/ (tracked).

  python tools/ncu_summarize.py ROUND TAG [TAG ...]

For each TAG reads gpurun_out/launches_TAG.csv (every launch, device time,
cold-cache and serialised) and gpurun_out/prof_TAG.ncu-rep (one --set full
capture of the PFAC kernel), writes profiles/rROUND_TAG.md and records the
per-launch DRAM traffic of the captured kernel in profiles/ncu_summary.json
(bench.py reads `traffic` from there).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "kernel duration"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads per warp instruction (divergence)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem load wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem store bank conflicts"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def launches(tag):
    path = os.path.join(OUT, f"launches_{tag}.csv")
    agg = collections.OrderedDict()
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = d.get("Metric Unit", "ns")
        v = float(d["Metric Value"].replace(",", ""))
        v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        name = d["Kernel Name"].split("(")[0]
        agg.setdefault(name, []).append(v)
    return agg


def full(tag):
    path = os.path.join(OUT, f"prof_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        m = {k: (d.get(k), units[hdr.index(k)] if k in hdr else "") for k, _ in METRICS}
        out.append((d["Kernel Name"], m))
    return out


def to_bytes(v, unit):
    v = float(str(v).replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    rnd, tags = sys.argv[1], sys.argv[2:]
    os.makedirs(PROF, exist_ok=True)
    summ_path = os.path.join(PROF, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    for tag in tags:
        lines = [f"# ncu evidence r{rnd} `{tag}`", ""]
        log = os.path.join(OUT, f"launches_{tag}.log")
        if os.path.exists(log):
            cmd = open(log).read().strip().splitlines()
            jl = [l for l in cmd if l.startswith("{")]
            if jl:
                cfg = json.loads(jl[-1])["config"]
                lines += [f"Workload: {cfg.get('workload')}", ""]
        lines += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`)", "",
                  "Cold-cache, serialised per-launch times: compare shares, not absolutes.", "",
                  "| kernel | launches | mean µs | share of listed time |", "|---|---|---|---|"]
        la = launches(tag)
        # drop the one-off corpus generator from the share (not part of a step)
        step = {k: v for k, v in la.items() if "gen_syslog" not in k and "gen_payload" not in k}
        tot = sum(sum(v) for v in step.values()) or 1
        for k, v in sorted(la.items(), key=lambda kv: -sum(kv[1])):
            share = f"{100 * sum(v) / tot:.1f}%" if k in step else "setup (untimed)"
            lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {share} |")
        lines += ["", "## Full capture of the dominant kernel (`ncu --set full --clock-control none`)", ""]
        for name, m in full(tag):
            lines += [f"Kernel: `{name[:160]}`", "", "| metric | value | unit | meaning |", "|---|---|---|---|"]
            for k, desc in METRICS:
                v, u = m[k]
                if v is not None:
                    lines.append(f"| `{k}` | {v} | {u} | {desc} |")
            rd = to_bytes(*m["dram__bytes_read.sum"]) if m["dram__bytes_read.sum"][0] else None
            wr = to_bytes(*m["dram__bytes_write.sum"]) if m["dram__bytes_write.sum"][0] else None
            key = name.split("(")[0].split("<")[0].replace("void ", "").strip().split("::")[-1]
            if rd is not None:
                summ.setdefault(key, {})[tag] = {"dram_bytes_per_launch": int(rd + (wr or 0)), "round": int(rnd),
                                                 "duration": m["gpu__time_duration.sum"][0] + " " +
                                                 m["gpu__time_duration.sum"][1]}
                summ[key]["dram_bytes_per_launch"] = int(rd + (wr or 0))
            lines.append("")
        with open(os.path.join(PROF, f"r{int(rnd):02d}_{tag}.md"), "w") as f:
            f.write("\n".join(lines) + "\n")
        print("wrote", f"profiles/r{int(rnd):02d}_{tag}.md")
    with open(summ_path, "w") as f:
        json.dump(summ, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
