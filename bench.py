#!/usr/bin/env python
"""PFAC log-scan throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--impl glop|reference] [--config pfac|kmp]

Workload (configs[2] / configs[3] of BASELINE.json): synthetic RFC 5424 syslog,
8e9 bytes per GPU (weak scaling; 64e9 at 8 GPUs), 1,000 8-byte patterns
(half reference random_rules, half incident vocabulary), prefix L = 8.
A step = one pass of the hot path over the GPU's shard: device PFAC scan +
ordering + stage-2 verify + per-pattern counts, through the fused device
pipeline (glop_run_pfac_pipeline_device: one host wait per step), plus the
NCCL count all-reduce and alert gather at N > 1.
`value` has the text already in HBM; `e2e` goes through the public pipeline
call with the text in pinned HOST memory (H2D + scan + verify + D2H of alerts
inside the timed region).  The 8 GB shard is larger than L2, so no flush.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PFAC log-scan Gbps at 1/2/4/8 B200 vs pattern count; % of HBM roofline"
KMP_METRIC = "KMP log-scan Gbps (single pattern 'Failed password'), 1 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["glop", "reference"], default="glop")
    ap.add_argument("--config", choices=["pfac", "kmp", "dpi"], default="pfac",
                    help="pfac: configs[2]/[3] syslog; kmp: configs[1]; dpi: configs[4] packet payloads")
    ap.add_argument("--bytes-per-gpu", type=float, default=None,
                    help="default 8e9 (pfac), 1e9 (kmp), 4e9 (dpi: 32 GB over 8 GPUs)")
    ap.add_argument("--patterns", type=int, default=None, help="default 1000 (pfac), 10000 (dpi)")
    ap.add_argument("--prefix-len", type=int, default=8)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--rules-seed", type=int, default=606)
    ap.add_argument("--kernel", choices=["auto", "filtered", "direct"], default="auto")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0 = same as --steps")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the Gbps-vs-pattern-count sweep (pfac, N=1)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU-baseline work")
    ap.add_argument("--no-parity", action="store_true", help="skip the full-size result digests")
    ap.add_argument("--exchange", choices=["p2p", "nccl"], default="p2p",
                    help="N>1: the alert gather / count exchange over CUDA IPC + copy engines (p2p, peer.py) "
                         "or NCCL collectives")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the configs[0]/[1]/[4] sub-blocks of the default line")
    a = ap.parse_args()
    if a.bytes_per_gpu is None:
        a.bytes_per_gpu = {"pfac": 8e9, "kmp": 1e9, "dpi": 4e9}[a.config]
    if a.patterns is None:
        a.patterns = 10000 if a.config == "dpi" else 1000
    return a


def workload_rules(args, glop):
    """The config's pattern set (bytes) and text generators (host, device)."""
    if args.config == "dpi":
        pats = glop.gen_dpi_rules(args.patterns, args.rules_seed, 8, 24)
        return pats, glop.gen_payload_host, "gen_payload_device"
    pats, _ = glop.gen_rules(args.patterns, args.rules_seed)
    return pats, glop.gen_syslog_host, "gen_syslog_device"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kind: str, tag: str):
    """dram bytes (read + write) per launch of the dominant kernel from the
    committed ncu summary (profiles/ncu_summary.json, written by
    tools/ncu_summarize.py from one `ncu --set full` capture of this
    workload), or None when no capture of this workload is committed."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            s = json.load(f)
        return s.get(kind, {}).get(tag, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def settle(self, work, timeout=3.0):
        """Run untimed `work` until nvidia-smi is producing samples (it takes a
        moment to start), so the timed region that follows is sampled."""
        t0 = time.perf_counter()
        while self.proc and not self.rows and time.perf_counter() - t0 < timeout:
            work()

    def hold(self, work, min_samples=5, timeout=3.0):
        """After a short timed region: keep the same load running (untimed)
        until a few samples under it exist."""
        t0 = time.perf_counter()
        n0 = len(self.rows)
        while self.proc and len(self.rows) - n0 < min_samples and time.perf_counter() - t0 < timeout:
            work()

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 8 for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def cpu_baseline_pfac(text_host, pats, L, target_s):
    """The reference pfac_scan + verify_hits (oracle/_ref, all host threads)
    on a bounded sample of the same workload; falls back to the C port."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as O

    ref = O.ref()
    kind = "reference" if ref is not None else "port"
    timer = O.ref_time_pfac if ref is not None else (lambda t, p, l, w, r: O.port_time_pfac(t, p, l, w, r))
    probe = min(len(text_host), 64 << 20)
    secs, _ = timer(text_host[:probe], pats, L, 0, 1)
    per_byte = max(secs[0], 1e-6) / probe
    runs = 3
    sample = int(min(len(text_host), max(probe, target_s / runs / per_byte)))
    secs, na = timer(text_host[:sample], pats, L, 1, runs)
    mean = statistics.mean(secs)
    cores = int(ref.ref_default_workers()) if ref is not None else 1
    return {"value": round(8 * sample / mean / 1e9, 3), "unit": "Gbps", "cores": cores, "kind": kind,
            "cpu_model": O.cpu_model(),
            "sample": f"first {sample} bytes of the GPU-0 shard, same {len(pats)} rules, L={L}; pfac_scan + "
                      f"verify_hits, {runs} timed runs after 1 warm-up, mean {mean:.3f} s/run, "
                      f"{'workers=hardware_concurrency' if kind == 'reference' else 'single thread'}"}


# --------------------------------------------------------------------- reference arm
# Sub-configurations carried by the default (configs[2]) line besides its
# headline: BASELINE.json configs[0], [1] and configs[4]'s per-GPU shard.
SUB_CONFIGS = [
    {"config": "configs[0]", "kind": "pfac", "corpus": "syslog", "bytes": 256_000_000, "patterns": 10,
     "workload": "PFAC, 10 patterns (8-byte prefixes), 256 MB synthetic RFC 5424 syslog"},
    {"config": "configs[1]", "kind": "kmp", "corpus": "syslog", "bytes": 1_000_000_000, "patterns": 1,
     "workload": "KMP single pattern 'Failed password' over 1 GB synthetic syslog"},
    {"config": "configs[4]", "kind": "pfac", "corpus": "payload", "bytes": 4_000_000_000, "patterns": 10000,
     "workload": "DPI: PFAC, 10,000 Snort-style contents (8..24 B) over one GPU's 4 GB payload shard "
                 "(32 GB over 8 GPUs)"},
]
KMP_PATTERN = b"Failed password"


def ref_rules(args, O, corpus=None, k=None):
    """The config's pattern set and host text generator, from oracle/_ref (the
    reference arm never maps libglop.so)."""
    corpus = corpus or ("payload" if args.config == "dpi" else "syslog")
    k = k or args.patterns
    if corpus == "payload":
        return O.ref_gen_dpi_rules(k, args.rules_seed, 8, 24), O.ref_gen_payload
    return O.ref_gen_rules(k, args.rules_seed), O.ref_gen_syslog


def ref_parity_pfac(O, text, own, pats, L):
    """Digest of the reference pfac_scan + verify_hits over text (starts
    < own reported, the shard ownership rule of scan.hpp:230-232)."""
    from paper_1704_02278_b200.parity import digest

    if O.ref() is not None:
        hits, alerts = O.ref_pfac_verify(text, pats, L, compact=True, workers=0)
    else:
        hits, alerts = O.pfac_verify(text, pats, L)
    hits, alerts = hits[hits["offset"] < own], alerts[alerts["offset"] < own]
    return digest(hits, alerts, len(pats))


def ref_parity_kmp(O, text):
    from paper_1704_02278_b200.parity import offsets_digest

    offs, cmp_ = O.kmp_search(text, KMP_PATTERN) if O.ref() is None else ref_kmp(O, text)
    return offsets_digest(offs, cmp_)


def ref_kmp(O, text):
    import ctypes as C

    import numpy as np

    r = O.ref()
    op, no, rc = C.c_void_p(), C.c_uint64(), C.c_uint64()
    pa = np.frombuffer(KMP_PATTERN, np.uint8).copy()
    r.ref_kmp_search(text.ctypes.data_as(O.u8p), len(text), pa.ctypes.data_as(O.u8p), len(pa), C.byref(op),
                     C.byref(no), C.byref(rc))
    return O._take(op, no.value, np.uint64, r.ref_free), rc.value


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ffi as O

    from paper_1704_02278_b200.shards import plan_shards  # pure Python

    ref = O.ref()
    kind = "reference" if ref is not None else "port"
    budget = 120.0  # seconds for warmup + steps
    S = int(args.bytes_per_gpu)
    if args.config == "kmp":
        p = KMP_PATTERN
        probe = O.ref_gen_syslog(64 << 20, args.seed)
        secs, _ = (O.ref_time_kmp(probe, p, 0, 1) if ref is not None else ([time.perf_counter()], 0))
        per_byte = max(secs[0], 1e-6) / probe.size
        sample = int(min(S, max(probe.size, budget / (args.warmup + args.steps) / per_byte)))
        full = O.ref_gen_syslog(S, args.seed)
        text = full[:sample]
        secs, nm = O.ref_time_kmp(text, p, args.warmup, args.steps)
        cores, metric = 1, KMP_METRIC
        config = {"workload": "configs[1]: KMP single pattern 'Failed password' over 1 GB synthetic syslog",
                  "bytes_per_gpu": S, "l2": "inputs larger than L2"}
        desc = f"kmp_multi (kmp.hpp:74) single-threaded by design on the first {sample} bytes"
        parity = ref_parity_kmp(O, full) if not args.no_parity else None
    else:
        pats, gen_host = ref_rules(args, O)
        probe = gen_host(64 << 20, args.seed)
        timer = O.ref_time_pfac if ref is not None else (lambda t, q, l, w, r: O.port_time_pfac(t, q, l, w, r))
        secs, _ = timer(probe, pats, args.prefix_len, 0, 1)
        per_byte = max(secs[0], 1e-6) / probe.size
        sample = int(min(S, max(probe.size, budget / (args.warmup + args.steps) / per_byte)))
        halo = max(len(q) for q in pats) - 1
        sh = plan_shards(S * args.gpus, args.gpus, max(halo, args.prefix_len - 1))[0]
        full = gen_host(sh.read, args.seed)  # rank 0's shard (the whole text at N = 1)
        text = full[:sample]
        secs, na = timer(text, pats, args.prefix_len, args.warmup, args.steps)
        cores = int(ref.ref_default_workers()) if ref is not None else 1
        metric = METRIC
        config = workload_config(args, args.gpus)
        desc = (f"reference pfac_scan + verify_hits (oracle/_ref built from /root/reference), workers={cores}, "
                f"on the first {sample} bytes of the same corpus and rules")
        parity = ref_parity_pfac(O, full, sh.own, pats, args.prefix_len) if not args.no_parity else None
    del full, text
    mean = statistics.mean(secs)
    value = 8 * sample / mean / 1e9
    line = {"impl": "reference", "metric": metric, "value": round(value, 3), "unit": "Gbps", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(mean * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic RFC 5424 syslog (csrc/corpus.h)" if args.config != "dpi" else
                    "synthetic packet payloads (csrc/payload.h)", "config": config,
            "cpu_baseline": {"value": round(value, 3), "unit": "Gbps", "cores": cores, "kind": kind, "sample": desc,
                             "sample_bytes": sample, "cpu_model": O.cpu_model()},
            "e2e": {"value": round(value, 3), "unit": "Gbps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if parity is not None:
        parity["scope"] = f"rank 0's shard: starts [0, {S}) of the config's text, full size (untimed)"
        line["parity"] = parity
    if args.config == "pfac" and not args.no_configs and not args.no_parity:
        line["configs"] = [dict(c0, parity=ref_sub_parity(args, O, c0)) for c0 in
                           ({"config": c["config"], "workload": c["workload"], "bytes": c["bytes"]}
                            for c in SUB_CONFIGS)]
    print(json.dumps(line), flush=True)
    return 0


def ref_sub_parity(args, O, cfg):
    c = next(x for x in SUB_CONFIGS if x["config"] == cfg["config"])
    gen = O.ref_gen_payload if c["corpus"] == "payload" else O.ref_gen_syslog
    text = gen(c["bytes"], args.seed)
    if c["kind"] == "kmp":
        return ref_parity_kmp(O, text)
    pats, _ = ref_rules(args, O, c["corpus"], c["patterns"])
    return ref_parity_pfac(O, text, c["bytes"], pats, args.prefix_len)


def workload_config(args, world):
    if args.config == "dpi":
        what = ("configs[4] DPI mode: PFAC, %d Snort-style contents (8..24 bytes; 8-byte prefixes + stage-2 "
                "verify), %g GB synthetic packet payloads per GPU" % (args.patterns, args.bytes_per_gpu / 1e9))
    else:
        what = ("configs[2]/[3]: PFAC, %d patterns (8-byte prefixes), %g GB synthetic RFC 5424 syslog per GPU"
                % (args.patterns, args.bytes_per_gpu / 1e9))
    return {"workload": what,
            "bytes_per_gpu": int(args.bytes_per_gpu), "total_bytes": int(args.bytes_per_gpu) * world,
            "patterns": args.patterns, "prefix_len": args.prefix_len, "corpus_seed": args.seed,
            "rules_seed": args.rules_seed, "kernel": args.kernel,
            "parallelism": f"shard{world} (contiguous log shards, 7-byte halo)",
            "l2": ("inputs larger than L2 (%g GB per GPU vs 126 MB L2), no flush needed" % (args.bytes_per_gpu / 1e9)
                   if args.bytes_per_gpu > 1e9 else "small run: inputs may be L2-resident (not a bench number)")}


# --------------------------------------------------------------------- glop arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1704_02278_b200 import glop
    from paper_1704_02278_b200.shards import gather_alerts_to_root, plan_shards

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.config == "pfac":
        return bench_group(args)  # one process driving N GPUs through the C ABI's device group
    # GLOP_BENCH_ONE_GPU=1: functional check of the N>1 path on a one-GPU box
    # (all ranks on cuda:0, gloo instead of NCCL); never used for numbers.
    one_gpu = os.environ.get("GLOP_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ctx = glop.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream)
    S = int(args.bytes_per_gpu)
    total = S * world
    kernel = {"auto": glop.PFAC_AUTO, "filtered": glop.PFAC_FILTERED, "direct": glop.PFAC_DIRECT}[args.kernel]

    if args.config == "kmp":
        return bench_kmp(args, ctx, stream, rank, world, local, barrier, max_over_ranks)

    pats, _, gen_dev = workload_rules(args, glop)
    trie = ctx.upload(glop.build_failureless_trie(pats, args.prefix_len))
    rules = ctx.upload_rules(pats, args.prefix_len)
    info = trie.info
    halo = max(info.max_depth, max(len(p) for p in pats)) - 1
    sh = plan_shards(total, world, halo)[rank]
    d_text = torch.empty(sh.read + 64, dtype=torch.uint8, device="cuda")
    getattr(ctx, gen_dev)(d_text.data_ptr(), sh.read, args.seed, begin=sh.lo)
    ctx.synchronize()
    cap = max(1 << 20, S // 256)
    d_hits = torch.empty(cap * 16, dtype=torch.uint8, device="cuda")
    d_alerts = torch.empty(cap * 16, dtype=torch.uint8, device="cuda")
    d_counts = torch.zeros(args.patterns, dtype=torch.int64, device="cuda")

    def step():
        if kernel == glop.PFAC_AUTO:  # the fused device pipeline: one host wait per step
            nh, na = ctx.run_pfac_pipeline_device(trie, rules, d_text.data_ptr(), sh.read, d_alerts.data_ptr(), cap,
                                                  d_counts.data_ptr(), own=sh.own, base=sh.lo)
        else:
            with torch.cuda.stream(stream):
                d_counts.zero_()
            nh = ctx.pfac_scan_device(trie, d_text.data_ptr(), sh.read, d_hits.data_ptr(), cap, own=sh.own,
                                      base=sh.lo, kernel=kernel)
            na = ctx.verify_hits_device(rules, d_text.data_ptr(), sh.read, d_hits.data_ptr(), nh,
                                        d_alerts.data_ptr(), d_counts.data_ptr(), base=sh.lo)
        if world > 1:  # the one exchange: count all-reduce + alert gather to rank 0 (NCCL over NVLink)
            with torch.cuda.stream(stream):
                dist.all_reduce(d_counts)
                gather_alerts_to_root(d_alerts.view(-1, 16), na, root=0)
        return nh, na

    # N = 1: steps are submitted back to back (glop_run_pfac_pipeline_device_async,
    # each step's status lands in a pinned ticket) and checked after the
    # closing synchronize -- the host never idles the GPU between steps.
    pipelined = world == 1 and kernel == glop.PFAC_AUTO
    n_tickets = max(args.steps, 8)
    tickets = ctx.host_alloc(glop.TICKET_BYTES * n_tickets) if pipelined else None

    def submit(i):
        ctx.run_pfac_pipeline_device_async(trie, rules, d_text.data_ptr(), sh.read, d_alerts.data_ptr(), cap,
                                           d_counts.data_ptr(), tickets + glop.TICKET_BYTES * (i % n_tickets),
                                           own=sh.own, base=sh.lo)

    def results(count):
        return [glop.ticket_result(tickets + glop.TICKET_BYTES * i) for i in range(count)]

    # N > 1: the exchange of step i (count all-reduce + alert gather to rank
    # 0, NCCL) runs on its own stream while step i+1's scan runs on the
    # library stream: alerts / counts double-buffered, one ticket each.
    overlapped = world > 1 and kernel == glop.PFAC_AUTO
    p2p = None
    if overlapped:
        comm = torch.cuda.Stream()
        ev_done = [torch.cuda.Event(), torch.cuda.Event()]
        ev_freed = [torch.cuda.Event(), torch.cuda.Event()]
        xtickets = ctx.host_alloc(glop.TICKET_BYTES * 2)
        xres = [None, None]
        if args.exchange == "p2p":
            # CUDA IPC + copy engines (peer.py): the pipeline writes straight into
            # the exchange buffers; the root pulls them beside the next scan
            from paper_1704_02278_b200.peer import PeerExchange

            gloo = None if dist.get_backend() == "gloo" else dist.new_group(backend="gloo")
            p2p = PeerExchange(ctx, rank, world, args.patterns, cap, group=gloo)
            a_ptrs, c_ptrs = p2p.alerts, p2p.counts_buf
        else:
            a_bufs = [d_alerts, torch.empty_like(d_alerts)]
            c_bufs = [d_counts, torch.zeros_like(d_counts)]
            a_ptrs, c_ptrs = [t.data_ptr() for t in a_bufs], [t.data_ptr() for t in c_bufs]

        def exchange(i):
            b = i & 1
            ev_done[b].synchronize()  # step i's scan is done (step i+1's is running)
            xres[b] = glop.ticket_result(xtickets + glop.TICKET_BYTES * b)
            if p2p is not None:
                p2p.exchange(b, xres[b][1], ctx.stream, ev_done[b])
                return
            with torch.cuda.stream(comm):
                comm.wait_event(ev_done[b])
                dist.all_reduce(c_bufs[b])
                gather_alerts_to_root(a_bufs[b].view(-1, 16), xres[b][1], root=0)
                ev_freed[b].record(comm)

        def run_overlapped(nsteps):
            for i in range(nsteps):
                b = i & 1
                if p2p is None:
                    stream.wait_event(ev_freed[b])  # buffer b's previous exchange has finished
                ctx.run_pfac_pipeline_device_async(trie, rules, d_text.data_ptr(), sh.read, a_ptrs[b], cap, c_ptrs[b],
                                                   xtickets + glop.TICKET_BYTES * b, own=sh.own, base=sh.lo)
                ev_done[b].record(stream)
                if i:
                    exchange(i - 1)
            if nsteps:
                exchange(nsteps - 1)
                if p2p is None:
                    stream.wait_event(ev_freed[(nsteps - 1) & 1])
                elif rank == 0:  # the last exchange's copies are inside the timed region
                    stream.wait_stream(p2p.comm)
            return xres[(nsteps - 1) & 1]

    for _ in range(max(args.warmup, 3)):
        nh, na = step()
    ctx.synchronize()
    sampler = ClockSampler(local)
    with sampler:
        # (ranks must not run different numbers of collective steps: at N > 1
        # the settle wait is idle)
        sampler.settle((lambda: (step(), ctx.synchronize())) if world == 1 else (lambda: time.sleep(0.02)))
        barrier()
        l0 = ctx.launches
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        kms = []
        if overlapped:
            nh, na = run_overlapped(args.steps)
        for i in range(args.steps if not overlapped else 0):
            if pipelined:
                submit(i)
            else:
                nh, na = step()
                kms.append(ctx.last_kernel_ms())
        ev1.record(stream)
        ctx.synchronize()
        barrier()
        launches = ctx.launches - l0
        if pipelined:  # every step's result, checked now (GLOP_EAGAIN would raise: the step needs the sync path)
            got = results(min(args.steps, n_tickets))
            assert len(set(got)) == 1, f"steps disagree: {set(got)}"
            nh, na = got[-1]
        if pipelined or overlapped:
            for _ in range(args.steps):  # the dominant kernel's own device time, per launch
                ctx.run_pfac_pipeline_device(trie, rules, d_text.data_ptr(), sh.read, d_alerts.data_ptr(), cap,
                                             d_counts.data_ptr(), own=sh.own, base=sh.lo)
                kms.append(ctx.last_kernel_ms())
            if overlapped and p2p is None:  # the counts of the last exchanged step, for the results block
                d_counts.copy_(c_bufs[(args.steps - 1) & 1])
        if world == 1:
            sampler.hold(lambda: (step(), ctx.synchronize()))
        ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
        kernel_ms = max_over_ranks(statistics.mean(kms))
        total_alerts = int(d_counts.sum().item())
        gathered = None
        if p2p is not None:  # the root's gathered result of the last exchanged step (rank order)
            got = p2p.gathered((args.steps - 1) & 1)
            if got is not None:
                from paper_1704_02278_b200.parity import alerts16

                import hashlib

                g_alerts, g_counts = got
                total_alerts = int(g_counts.sum())
                gathered = {"alerts": int(len(g_alerts)), "alerts16_sha": hashlib.sha256(
                    np.ascontiguousarray(alerts16(g_alerts)).tobytes()).hexdigest(),
                            "counts_sha": hashlib.sha256(g_counts.astype("<u8").tobytes()).hexdigest()}
            dist.barrier(group=p2p.group)
            p2p.close()

        e2e = None
        if not args.no_e2e:
            e2e = run_e2e(args, ctx, trie, rules, d_text, sh, world, barrier, max_over_ranks, torch, dist)
            if world == 1 and args.config != "kmp":
                e2e["dropin"] = run_e2e_dropin(args, glop, d_text, sh, pats)
    clocks = sampler.summary()

    value = 8 * total / (ms / 1e3) / 1e9
    peak, peak_src = peaks()
    achieved = sh.own / (kernel_ms / 1e3) / 1e9  # GB/s of the dominant kernel
    kname = "pfac8_kernel" if info.min_depth >= 8 and args.kernel == "auto" else "pfac_warp_kernel"
    tag = "dpi" if args.config == "dpi" else f"k{args.patterns}"
    traffic = ncu_traffic(kname, tag) if args.bytes_per_gpu == {"dpi": 4e9}.get(args.config, 8e9) else None
    line = {"metric": METRIC, "value": round(value, 2), "unit": "Gbps", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": ("synthetic packet payloads generated on device (csrc/payload.h), seeded" if args.config == "dpi"
                     else "synthetic RFC 5424 syslog generated on device (csrc/corpus.h), seeded"),
            "config": workload_config(args, world),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                         "kernel": kname, "kernel_ms": round(kernel_ms, 4),
                         "algorithmic_bytes_per_launch": sh.own,
                         "step_share": round(kernel_ms / ms, 3)},
            "gpu_launches": launches, "clocks": clocks,
            "results": {"stage1_hits_per_gpu_step": int(nh), "alerts_per_step": total_alerts,
                        **({"exchange": args.exchange, "gathered": gathered} if world > 1 else {}),
                        "trie": {"states": info.state_count, "classes": info.classes, "q": info.q,
                                 "stride": info.stride, "table_bytes": int(info.table_bytes),
                                 "table_in_smem": bool(info.table_in_smem)}}}
    if e2e is not None:
        line["e2e"] = e2e
    if not args.no_parity:  # rank 0's full-size result, for the driver to compare with the reference arm
        from paper_1704_02278_b200.parity import digest

        nh, na = ctx.run_pfac_pipeline_device(trie, rules, d_text.data_ptr(), sh.read, d_alerts.data_ptr(), cap,
                                              d_counts.data_ptr(), own=sh.own, base=sh.lo, d_hits=d_hits.data_ptr(),
                                              hit_cap=cap)
        hits = d_hits[: nh * 16].cpu().numpy().view(glop.HIT_DTYPE)
        alerts = d_alerts[: na * 16].cpu().numpy().view(glop.ALERT_DTYPE)
        line["parity"] = dict(digest(hits, alerts, args.patterns),
                              scope=f"rank 0's shard: starts [0, {S}) of the config's text, full size (untimed)")
    if world == 1 and args.config == "pfac" and not args.no_sweep:
        line["pattern_sweep"] = pattern_sweep(args, ctx, glop, d_text, sh, d_hits, cap, peak)
    if rank == 0 and world == 1 and not args.no_cpu:
        sample = min(sh.own, 2 << 30)
        host = d_text[:sample].cpu().numpy()
        line["cpu_baseline"] = cpu_baseline_pfac(host, pats, args.prefix_len, args.cpu_seconds)
    if world == 1 and args.config == "pfac" and not args.no_configs:  # (overwrites d_text: after every use of it)
        line["configs"] = [sub_config(args, ctx, glop, stream, c, d_text, d_hits, d_alerts, cap, peak)
                           for c in SUB_CONFIGS]
    if tickets:
        ctx.host_free(tickets)
    if overlapped:
        ctx.host_free(xtickets)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def pattern_sweep(args, ctx, glop, d_text, sh, d_hits, cap, peak):
    """The metric's "vs pattern count" axis: the PFAC scan of the same
    resident shard for 10 / 100 / 1,000 / 10,000 rules (same generator, same
    seed), mean kernel time of 5 launches after 2 warm-ups."""
    out = []
    for k in (10, 100, 1000, 10000):
        pats, vocab = glop.gen_rules(k, args.rules_seed)
        trie = ctx.upload(glop.build_failureless_trie(pats, args.prefix_len))
        kms = []
        for i in range(7):
            nh = ctx.pfac_scan_device(trie, d_text.data_ptr(), sh.read, d_hits.data_ptr(), cap, own=sh.own, base=sh.lo)
            if i >= 2:
                kms.append(ctx.last_kernel_ms())
        ms = statistics.mean(kms)
        gbs = sh.own / (ms / 1e3) / 1e9
        out.append({"patterns": k, "kernel_ms": round(ms, 4), "gbps": round(8 * gbs, 1), "hbm_frac": round(gbs / peak, 4),
                    "hits": int(nh), "vocab_rules": int(vocab.sum()), "trie_states": trie.info.state_count})
    return out


def sub_config(args, ctx, glop, stream, c, d_text, d_hits, d_alerts, cap, peak):
    """One of BASELINE.json's other configs on this GPU, device-resident:
    3 warm-ups + min(steps, 10) timed steps (CUDA events on the library
    stream), the dominant kernel's mean time, and the full-size result digest."""
    import torch

    from paper_1704_02278_b200.parity import digest, offsets_digest

    n = c["bytes"]
    gen = ctx.gen_payload_device if c["corpus"] == "payload" else ctx.gen_syslog_device
    gen(d_text.data_ptr(), n, args.seed)
    ctx.synchronize()
    steps = max(1, min(args.steps, 10))
    if c["kind"] == "kmp":
        kcap = min(cap * 2, 1 << 24)

        def step():
            return ctx.kmp_search_device(KMP_PATTERN, d_text.data_ptr(), n, d_hits.data_ptr(), kcap)
        kname = "kmp3_kernel"
    else:
        pats = glop.gen_dpi_rules(c["patterns"], args.rules_seed, 8, 24) if c["corpus"] == "payload" else \
            glop.gen_rules(c["patterns"], args.rules_seed)[0]
        trie = ctx.upload(glop.build_failureless_trie(pats, args.prefix_len))
        rules = ctx.upload_rules(pats, args.prefix_len)
        d_counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")

        def step():
            return ctx.run_pfac_pipeline_device(trie, rules, d_text.data_ptr(), n, d_alerts.data_ptr(), cap,
                                                d_counts.data_ptr())
        kname = "pfac8_kernel" if trie.info.min_depth >= 8 else "pfac_warp_kernel"
    for _ in range(3):
        r = step()
    ctx.synchronize()
    # as the headline: steps submitted back to back, tickets checked after
    tickets = ctx.host_alloc(glop.TICKET_BYTES * steps)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    kms = []
    for i in range(steps):
        if c["kind"] == "kmp":
            ctx.kmp_search_device_async(KMP_PATTERN, d_text.data_ptr(), n, d_hits.data_ptr(), kcap,
                                        tickets + glop.TICKET_BYTES * i)
        else:
            ctx.run_pfac_pipeline_device_async(trie, rules, d_text.data_ptr(), n, d_alerts.data_ptr(), cap,
                                               d_counts.data_ptr(), tickets + glop.TICKET_BYTES * i)
    ev1.record(stream)
    ctx.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    res = glop.kmp_ticket_result if c["kind"] == "kmp" else glop.ticket_result
    got = {res(tickets + glop.TICKET_BYTES * i) for i in range(steps)}
    ctx.host_free(tickets)
    assert len(got) == 1, got
    for _ in range(steps):
        r = step()
        kms.append(ctx.last_kernel_ms())
    kernel_ms = statistics.mean(kms)
    gbs = n / (kernel_ms / 1e3) / 1e9
    out = {"config": c["config"], "workload": c["workload"], "bytes": n, "steps": steps, "kernel": kname,
           "kernel_ms": round(kernel_ms, 4), "ms_per_step": round(ms, 4), "gbps": round(8 * n / (ms / 1e3) / 1e9, 1),
           "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                        "frac": round(gbs / peak, 4)}}
    if not args.no_parity:
        if c["kind"] == "kmp":
            nm, cmp_ = r
            out["parity"] = offsets_digest(d_hits[: nm * 8].cpu().numpy().view("<u8"), cmp_)
        else:
            nh, na = ctx.run_pfac_pipeline_device(trie, rules, d_text.data_ptr(), n, d_alerts.data_ptr(), cap,
                                                  d_counts.data_ptr(), d_hits=d_hits.data_ptr(), hit_cap=cap)
            out["parity"] = digest(d_hits[: nh * 16].cpu().numpy().view(glop.HIT_DTYPE),
                                   d_alerts[: na * 16].cpu().numpy().view(glop.ALERT_DTYPE), len(pats))
    return out


def run_e2e(args, ctx, trie, rules, d_text, sh, world, barrier, max_over_ranks, torch, dist):
    """Same metric through the public pipeline call with the shard in pinned
    host memory: H2D copy + scan + verify + D2H alerts/counts every step."""
    try:  # pinned host copy of the shard; every rank must have one before going on
        host, why = ctx.host_alloc(sh.read), ""
    except Exception as e:  # noqa: BLE001 -- reported, not fatal
        host, why = None, f"pinned host allocation of {sh.read} bytes failed: {e}"
    if world > 1:
        ok = torch.tensor([0.0 if host is None else 1.0], dtype=torch.float64, device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 0 and host is not None:
            ctx.host_free(host)
            host, why = None, why or "another rank could not pin its shard"
    if host is None:
        return {"unavailable": why}
    try:
        ctx.memcpy(host, d_text.data_ptr(), sh.read, 2)
        ctx.synchronize()
        steps = args.e2e_steps or args.steps
        alerts, counts, s1 = ctx.run_pfac_pipeline(trie, rules, host, sh.read, False, own=sh.own, base=sh.lo)
        barrier()
        t0 = time.perf_counter()
        d2h = 0
        for _ in range(steps):
            alerts, counts, s1 = ctx.run_pfac_pipeline(trie, rules, host, sh.read, False, own=sh.own, base=sh.lo)
            if world > 1:
                c = torch.from_numpy(counts.astype("int64")).cuda()
                dist.all_reduce(c)
            d2h = alerts.nbytes + counts.nbytes
        barrier()
        dt = max_over_ranks((time.perf_counter() - t0) / steps)
    finally:
        ctx.host_free(host)
    return {"value": round(8 * sh.own * world / dt / 1e9, 2), "unit": "Gbps", "h2d_bytes_per_step": sh.read,
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(dt * 1e3, 3),
            "api": "glop_run_pfac_pipeline_shard (pinned host text)"}


def run_e2e_dropin(args, glop, d_text, sh, pats):
    """The reference caller's path: logtrawl::run_engine_scan (the drop-in
    C++ header API, pfac_compact engine, the reference default) on the text in
    PAGEABLE host memory, as a std::string would hold it -- upload, scan,
    verify and the alert report back, per call, wall-clock."""
    try:
        eng = glop.Engine(pats)
    except ImportError as e:
        return {"unavailable": str(e)}
    host = d_text[: sh.read].cpu().numpy()  # pageable
    eng.run(host.ctypes.data, sh.read)  # warm-up: builds + uploads the cached trie / rules
    steps = max(1, min(args.e2e_steps or args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(steps):
        alerts, _, s1 = eng.run(host.ctypes.data, sh.read)
    dt = (time.perf_counter() - t0) / steps
    eng.close()
    return {"value": round(8 * sh.own / dt / 1e9, 2), "unit": "Gbps", "h2d_bytes_per_step": sh.read,
            "d2h_bytes_per_step": int(alerts.nbytes), "ms_per_step": round(dt * 1e3, 3), "steps": steps,
            "api": "logtrawl::run_engine_scan (include/logtrawl/pipeline.hpp, pfac_compact) via libglop_engine.so, "
                   "text in pageable host memory"}


def bench_group(args):
    """`python bench.py --gpus N` without torchrun: one process drives N GPUs
    through libglop's device group -- per-member contexts scanning their
    halo'd shard (glop_run_pfac_pipeline_device) concurrently from host
    threads, device-timed with CUDA events on each member's stream, max over
    members; e2e through glop_group_run_pfac_pipeline on pinned host text.
    GLOP_BENCH_DEVICES="0,0" runs the N-way split on one GPU (functional
    check, not a number)."""
    import threading as th

    import numpy as np
    import torch

    from paper_1704_02278_b200 import glop
    from paper_1704_02278_b200.shards import plan_shards

    devs = [int(x) for x in os.environ.get("GLOP_BENCH_DEVICES", ",".join(map(str, range(args.gpus)))).split(",")]
    N = len(devs)
    S = int(args.bytes_per_gpu)
    total = S * N
    pats, _, gen_dev = workload_rules(args, glop)
    ctxs = [glop.Context(d) for d in devs]
    tries = [c.upload(glop.build_failureless_trie(pats, args.prefix_len)) for c in ctxs]
    rules = [c.upload_rules(pats, args.prefix_len) for c in ctxs]
    halo = max(tries[0].info.max_depth, max(len(p) for p in pats)) - 1
    shards = plan_shards(total, N, halo)
    cap = max(1 << 20, S // 256)
    bufs = []
    for c, d, sh in zip(ctxs, devs, shards):
        with torch.cuda.device(d):
            t = torch.empty(sh.read + 64, dtype=torch.uint8, device=f"cuda:{d}")
            a = torch.empty(cap * 16, dtype=torch.uint8, device=f"cuda:{d}")
            k = torch.zeros(len(pats), dtype=torch.int64, device=f"cuda:{d}")
        getattr(c, gen_dev)(t.data_ptr(), sh.read, args.seed, begin=sh.lo)
        bufs.append((t, a, k))
    for c in ctxs:
        c.synchronize()
    res = [None] * N

    def member(g, steps):
        c, (t, a, k), sh = ctxs[g], bufs[g], shards[g]
        with torch.cuda.device(devs[g]):
            s0 = torch.cuda.ExternalStream(c.stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s0)
            for _ in range(steps):
                r = c.run_pfac_pipeline_device(tries[g], rules[g], t.data_ptr(), sh.read, a.data_ptr(), cap,
                                               k.data_ptr(), own=sh.own, base=sh.lo)
            e1.record(s0)
            c.synchronize()
            res[g] = (e0.elapsed_time(e1) / max(steps, 1), r)

    def run(steps):
        ts = [th.Thread(target=member, args=(g, steps)) for g in range(N)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()

    run(max(args.warmup, 3))
    sampler = ClockSampler(devs[0])
    with sampler:
        sampler.settle(lambda: run(1))
        run(args.steps)
        sampler.hold(lambda: run(1))
    ms = max(r[0] for r in res)
    nh = sum(r[1][0] for r in res)
    na = sum(r[1][1] for r in res)
    peak, peak_src = peaks()
    line = {"metric": METRIC, "value": round(8 * total / (ms / 1e3) / 1e9, 2), "unit": "Gbps", "n_gpus": N,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic RFC 5424 syslog generated on device (csrc/corpus.h), seeded",
            "config": dict(workload_config(args, N), parallelism=f"group{N} (one process, libglop device group)",
                           devices=devs),
            "roofline": {"bound": "hbm", "achieved": round(total / (ms / 1e3) / 1e9, 1), "peak": peak * N,
                         "unit": "GB/s", "frac": round(total / (ms / 1e3) / 1e9 / (peak * N), 4),
                         "traffic": None, "peak_source": peak_src + f" x {N} GPUs", "kernel": "pfac8_kernel (step)"},
            "clocks": sampler.summary(),
            "results": {"stage1_hits_per_step": int(nh), "alerts_per_step": int(na)}}
    if not args.no_e2e:
        g = glop.Group(devs)
        gt, gr = g.upload(glop.build_failureless_trie(pats, args.prefix_len)), g.upload_rules(pats, args.prefix_len)
        try:
            host = np.empty(total, dtype=np.uint8)
            for (t, _, _), sh in zip(bufs, shards):
                host[sh.lo:sh.lo + sh.own] = t[:sh.own].cpu().numpy()
            g.run_pfac_pipeline(gt, gr, host)
            t0 = time.perf_counter()
            steps = max(1, min(args.e2e_steps or args.steps, 5))
            for _ in range(steps):
                alerts, counts, s1, _, _ = g.run_pfac_pipeline(gt, gr, host)
            dt = (time.perf_counter() - t0) / steps
            line["e2e"] = {"value": round(8 * total / dt / 1e9, 2), "unit": "Gbps", "h2d_bytes_per_step": total,
                           "d2h_bytes_per_step": int(alerts.nbytes + counts.nbytes), "ms_per_step": round(dt * 1e3, 3),
                           "api": "glop_group_run_pfac_pipeline (pageable host text)"}
        except MemoryError as e:
            line["e2e"] = {"unavailable": f"host copy of {total} bytes: {e}"}
    print(json.dumps(line), flush=True)
    return 0


def bench_kmp(args, ctx, stream, rank, world, local, barrier, max_over_ranks):
    import torch

    from paper_1704_02278_b200 import glop

    S = int(args.bytes_per_gpu)
    p = b"Failed password"
    d_text = torch.empty(S + 64, dtype=torch.uint8, device="cuda")
    ctx.gen_syslog_device(d_text.data_ptr(), S, args.seed, begin=rank * S)
    ctx.synchronize()
    cap = 1 << 24
    d_out = torch.empty(cap * 8, dtype=torch.uint8, device="cuda")
    for _ in range(max(args.warmup, 3)):
        nm, cmp_ = ctx.kmp_search_device(p, d_text.data_ptr(), S, d_out.data_ptr(), cap, base=rank * S)
    sampler = ClockSampler(local)
    kmp_step = lambda: ctx.kmp_search_device(p, d_text.data_ptr(), S, d_out.data_ptr(), cap, base=rank * S)  # noqa: E731
    with sampler:
        sampler.settle(kmp_step if world == 1 else (lambda: time.sleep(0.02)))
        barrier()
        l0 = ctx.launches
        tickets = ctx.host_alloc(glop.TICKET_BYTES * args.steps)  # steps submitted back to back
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for i in range(args.steps):
            ctx.kmp_search_device_async(p, d_text.data_ptr(), S, d_out.data_ptr(), cap,
                                        tickets + glop.TICKET_BYTES * i, base=rank * S)
        ev1.record(stream)
        ctx.synchronize()
        barrier()
        launches = ctx.launches - l0
        got = {glop.kmp_ticket_result(tickets + glop.TICKET_BYTES * i) for i in range(args.steps)}
        ctx.host_free(tickets)
        assert len(got) == 1, got
        nm, cmp_ = got.pop()
        kms = []
        for _ in range(args.steps):  # the kernel's own device time, per launch
            kmp_step()
            kms.append(ctx.last_kernel_ms())
        if world == 1:
            sampler.hold(kmp_step)
        ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
        kernel_ms = max_over_ranks(statistics.mean(kms))
    peak, peak_src = peaks()
    achieved = S / (kernel_ms / 1e3) / 1e9
    line = {"metric": KMP_METRIC, "value": round(8 * S * world / (ms / 1e3) / 1e9, 2), "unit": "Gbps",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic RFC 5424 syslog generated on device", "config": {
                "workload": "configs[1]: KMP single pattern 'Failed password' over 1 GB synthetic syslog",
                "bytes_per_gpu": S, "l2": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": ncu_traffic("kmp3_kernel", "kmp"),
                         "peak_source": peak_src, "kernel": "kmp3_kernel", "kernel_ms": round(kernel_ms, 4)},
            "gpu_launches": launches, "clocks": sampler.summary(), "results": {"matches": int(nm),
                                                                              "comparisons": int(cmp_)}}
    if rank == 0 and world == 1 and not args.no_cpu:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import oracle_ffi as O

        sample = min(S, 256 << 20)
        host = d_text[:sample].cpu().numpy()
        if O.ref() is not None:
            secs, _ = O.ref_time_kmp(host, p, 1, 3)
            line["cpu_baseline"] = {"value": round(8 * sample / statistics.mean(secs) / 1e9, 3), "unit": "Gbps",
                                    "cores": 1, "kind": "reference", "cpu_model": O.cpu_model(),
                                    "sample": f"kmp_multi on the first {sample} bytes, single thread by design"}
            # context: the reference's multi-core pfac_scan + verify_hits with k=1
            psecs, _ = O.ref_time_pfac(host, [p], 8, 1, 3)
            line["cpu_baseline"]["pfac_k1_multicore"] = {
                "value": round(8 * sample / statistics.mean(psecs) / 1e9, 3), "unit": "Gbps",
                "cores": int(O.ref().ref_default_workers()),
                "sample": f"pfac_scan + verify_hits, the one pattern, L=8, same {sample} bytes"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
