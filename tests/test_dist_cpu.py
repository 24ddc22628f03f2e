"""Multi-process plumbing on CPU (gloo, world_size 2-3).

* ``bench.py`` under ``torch.distributed.run`` with two ranks: the reference
  arm runs on rank 0 only and prints exactly one JSON line; the rendezvous
  uses 127.0.0.1.
* The SPMD runtime's host side (``spmd.py``): lockstep broadcasts / votes,
  host messages and transfer batching through the ``cb_xfer_fn`` pointer.
* ``dist.ReplicaGroup``'s scatter / gather by ``split_batch``.
The device side of the N>1 path needs GPUs and is exercised on the box
(tests/test_spmd_gpu.py, tests/test_dist_gpu.py).
"""
from __future__ import annotations

import json
import socket
import subprocess
import sys

from conftest import ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_torchrun_reference_arm_rank0_only():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--batch", "2", "--prompt", "8"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["n_gpus"] == 2 and rec["value"] > 0
    assert rec["e2e"]["h2d_bytes_per_step"] == 0 and rec["cpu_baseline"]["kind"] == "port"


def test_gloo_barrier_world2():
    """The barrier/max-over-ranks pattern bench.py relies on, with gloo."""
    code = r'''
import os, torch, torch.distributed as dist
dist.init_process_group("gloo")
r = dist.get_rank()
t = torch.tensor([float(r + 1)])
dist.all_reduce(t, op=dist.ReduceOp.MAX)
dist.barrier()
if r == 0:
    print("MAX", t.item())
dist.destroy_process_group()
'''
    script = ROOT / "build" / "gloo_probe.py"
    script.parent.mkdir(exist_ok=True)
    script.write_text(code)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(script)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "MAX 2.0" in out.stdout


def _torchrun(script, nproc, env=None):
    import os
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(script)]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                          env={**os.environ, **(env or {})})


def test_replica_group_world2_matches_unreplicated():
    """One process per replica (gloo, world 2): scatter of the batch by
    split_batch (15 -> [7, 8]), each rank serves its share, the
    gather returns greedy tokens identical to one unreplicated pass."""
    out = _torchrun(ROOT / "tests" / "dist_replica_worker.py", 2)
    assert out.returncode == 0, out.stderr[-3000:]
    rec = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert rec["equal"] and rec["shares"] == [7, 8] and rec["world"] == 2


def test_replica_group_world3_uneven_shares():
    """Uneven split with an empty-remainder edge: 5 requests over 3 ranks -> [1, 2, 2]."""
    out = _torchrun(ROOT / "tests" / "dist_replica_worker.py", 3, {"N_REQ": "5"})
    assert out.returncode == 0, out.stderr[-3000:]
    rec = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert rec["equal"] and rec["shares"] == [1, 2, 2]


def test_spmd_host_plumbing_world2():
    """The SPMD runtime's host side over gloo (tests/spmd_host_worker.py):
    lockstep broadcast / all-gather, host messages through the cb_xfer_fn
    function pointer, transfer batching and error return."""
    out = _torchrun(ROOT / "tests" / "spmd_host_worker.py", 2)
    assert out.returncode == 0, out.stderr[-3000:]
    rec = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert rec["rank_of_device"] == [0, 0, 1, 1]
    assert rec["bcast"] == [5, 6, 7, 101]
    assert rec["allgather"] == [[0, 3], [1, 13]]
    assert rec["host_rc"] == 0 and rec["host_equal"]
    assert rec["host_counted"] == [1, 64 + 9 * 4]
    assert rec["flush_before_end"] == 0
    assert rec["flushed"] == [[0, [[True, 1, 0x1000, 256], [False, 1, 0x2000, 128]]], [1, [[True, 1, 0x3000, 64]]]]
    assert rec["err_rc"] == 1 and rec["err_kept"]
