"""SPMD runtime (one process per device) on the GPU box: module replication,
cross-process KV moves under a shrinking batch, asynchronous replication,
layer migration with KV and eviction -- greedy tokens equal to the fp32 oracle
at every step (tests/spmd_worker.py).  The box has one GPU, so every rank runs
on cuda:0: the host-staged transport (gloo) and the NCCL transport (each rank
its own NCCL_HOSTID, i.e. NCCL's network path) both carry the exchanges."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world: int, mode: str) -> dict:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "tests" / "spmd_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={**os.environ, "SPMD_MODE": mode, "WORKER_SAME_GPU": "1"})
    assert out.returncode == 0, out.stderr[-4000:]
    return json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])


@pytest.mark.parametrize("world,mode", [(2, "host"), (3, "host"), (2, "nccl")])
def test_spmd_scaling_ops_match_oracle(world, mode):
    rec = _run(world, mode)
    r0 = rec["ranks"][0]
    assert r0["n_mismatch"] == 0, r0["mismatches"]
    assert r0["tokens_checked"] == 15 * 4 + 12 * 7
    # layer 2 over `world` ranks: 15 -> split_batch(15, world), then 12 sequences
    share = [15 // world + (1 if j >= world - 15 % world else 0) for j in range(world)]
    assert [c for _, _, c in r0["routing_before"]] == share
    assert [d for d, _, _ in r0["routing_before"]] == list(range(world))
    assert sum(c for _, _, c in r0["routing_after"]) == 12
    assert r0["layer4_digests"][0] == r0["layer4_digests"][1]  # replicated block byte-identical across processes
    assert r0["placement"] == [[0], [0] + list(range(2, world)), [1], [0, 1]]
    # migrate layer 3 with KV: the receiver measured the layer block + the live KV prefixes
    r1 = rec["ranks"][1]
    assert r1["migrate"]["weight_bytes"] == 1_704_960
    assert r1["migrate"]["kv_bytes"] > 0
    assert all(r["transport_messages"] > 0 for r in rec["ranks"])
