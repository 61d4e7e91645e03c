"""The sharded bench path with the CUDA-IPC / copy-engine exchange
(paper_1704_02278_b200/peer.py) under torchrun: two ranks (both on cuda:0
here -- GLOP_BENCH_ONE_GPU=1; one per GPU on a multi-GPU box) scan their
halo'd shards, the root pulls the peer's alerts and counts from the peer's
buffers each step, and the gathered rank-order result of the last step must
equal the reference over the whole text.  Run on the B200: pytest -m gpu."""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle_ffi as O
from paper_1704_02278_b200 import glop
from paper_1704_02278_b200.parity import alerts16

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_exchange_gathers_reference(world):
    S = 40_000_000
    env = dict(os.environ, GLOP_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world), os.path.join(ROOT, "bench.py"),
           "--gpus", str(world), "--steps", "4", "--warmup", "3", "--bytes-per-gpu", str(S), "--no-e2e",
           "--no-parity", "--exchange", "p2p"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    got = line["results"]["gathered"]
    assert line["results"]["exchange"] == "p2p" and got is not None
    pats, _ = glop.gen_rules(1000, 606)
    text = glop.gen_syslog_host(S * world, 1)
    if O.ref() is not None:
        _, ref = O.ref_pfac_verify(text, pats, 8, compact=True, workers=0)
    else:
        _, ref = O.pfac_verify(text, pats, 8)
    assert got["alerts"] == len(ref)
    assert got["alerts16_sha"] == hashlib.sha256(np.ascontiguousarray(alerts16(ref)).tobytes()).hexdigest()
    counts = np.bincount(ref["rule_id"].astype(np.int64), minlength=len(pats)).astype("<u8")
    assert got["counts_sha"] == hashlib.sha256(counts.tobytes()).hexdigest()
