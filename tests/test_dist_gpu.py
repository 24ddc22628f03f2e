"""One process per replica on the GPU: bench.py's N>1 path (dist.ReplicaGroup)
under torchrun with world size 2.  The box has one GPU and NCCL refuses two
ranks on one device, so BENCH_SAME_GPU=1 puts both ranks on cuda:0 with gloo
collectives -- the executor path per rank is the real one (7B shape)."""
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


@pytest.mark.parametrize("transport", ["host", "nccl"])
def test_bench_spmd_world2_same_gpu(transport):
    """bench.py's N>1 path (config 3, SPMD: hot layers 1..28 replicated on the
    second rank, cold layers + head on rank 0, continuous-batching window with
    cross-rank KV moves) with both ranks on cuda:0: host-staged transport, and
    the NCCL transport the multi-GPU run uses (each rank its own NCCL host)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "1", "--batch", "8", "--prompt", "16", "--churn-steps", "3"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                         env={**os.environ, "BENCH_SAME_GPU": "1", "BENCH_TRANSPORT": transport})
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["config"]["batch"] == 16 and rec["value"] > 0
    assert rec["config"]["replicated_layers"] == 28
    assert rec["gpu_launches"] > 0 and rec["scaling"] == "weak"
    assert rec["roofline"]["frac"] > 0 and rec["roofline"]["bound"] in ("hbm", "tensor")
    assert rec["migrate"]["bytes"] == 404_766_720 and rec["migrate"]["gbps"] > 0
    assert rec["continuous_batching"]["transport_messages"] > 0


def test_replica_group_world2_gpu_executors_match_oracle():
    """Two processes, each a real libcocob200 executor (tiny model, confident
    head) serving its split_batch share; gathered greedy tokens == the
    unreplicated fp32 oracle."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "tests" / "dist_replica_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={**os.environ, "WORKER_GPU": "1"})
    assert out.returncode == 0, out.stderr[-3000:]
    rec = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert rec["equal"] and rec["shares"] == [7, 8]
