#!/usr/bin/env python
"""Per-source-line instruction / stall attribution of an ncu report (reads here, no GPU).
  python tools/ncu_lines.py gpurun_out/prof_q1000.ncu-rep [bytes] [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; nbytes = float(sys.argv[2]) if len(sys.argv) > 2 else 2e9; top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw))); hdr = rows[0]
d = dict(zip(hdr, rows[2]))
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "launch__registers_per_thread"]
for k in keys: print(f"{k:60s} {d.get(k)}")
stalls = sorted(((float(v), k) for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") and v), reverse=True)[:8]
print("stalls/issue:", ", ".join(f"{k[34:-23]}={v:.2f}" for v, k in stalls))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
out = []; fname = None; hdr = None
for r in csv.reader(io.StringIO(src)):
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]
    if len(r) > 5 and r[0] == "Line No": hdr = r; continue
    if hdr and len(r) > 8 and r[0] != "" and r[2] == "-":
        out.append((int(r[7] or 0), int(r[4] or 0), fname, r[0], r[1][:80]))
tot = sum(o[0] for o in out); ts = sum(o[1] for o in out) or 1
it = nbytes / 512
print(f"total warp-inst {tot} = {tot/it:.1f} per 512B")
for o in sorted(out, key=lambda x: -x[0])[:top]:
    print(f"{o[0]/it:7.2f}/512B {o[1]/ts*100:5.1f}%stall {o[2]}:{o[3]:5s} {o[4]}")
# shared-memory wavefronts per source line (actual vs ideal): what bounds an smem-bound kernel
wf = []
for r in csv.reader(io.StringIO(src)):
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]
    if len(r) > 20 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            a, i = float(r[19] or 0), float(r[20] or 0)
        except ValueError:
            continue
        if a: wf.append((a, i, fname, r[0], r[1][:70]))
ta = sum(w[0] for w in wf) or 1
print(f"shared wavefronts {ta:.0f} = {ta/it:.1f} per 512B")
for w in sorted(wf, key=lambda x: -x[0])[:16]:
    print(f"{w[0]/it:7.2f}/512B (ideal {w[1]/it:6.2f}) {w[2]}:{w[3]:5s} {w[4]}")
