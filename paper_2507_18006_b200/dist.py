"""One process per GPU: ranks holding a replica of every decoder layer.

The reference placement where every layer has a replica on every device
(``PlacementState.with_replica`` for all layers / devices, domain.py:414-421)
is ONE replicated run covering the whole model: ``split_batch(bs, p)``
(ops.py:151-158) hands replica j the contiguous sequence range j of the live
batch, and the only data exchanges are the scatter at the run's start and the
gather at its end (``_comm_units`` prices exactly one boundary
pair per run, _kernels.py:41-51).  ``ReplicaGroup`` is that run executed by N
processes, one per GPU, each driving a single-GPU ``Executor`` that holds the
full model:

* scatter -- rank 0 (the original device, home of the request router) owns
  the batch; it broadcasts the step's metadata and every rank keeps its
  ``split_batch`` share (rank order = replica order, the original first);
* each rank runs the pass over its share on its own GPU;
* gather -- the sampled tokens come back to rank 0 in batch order.

The collectives run over ``torch.distributed``: NCCL on the GPU box (the
messages are a few KB of int32 per step, latency-bound), gloo in the CPU tests.

This is the light mode for the one placement where every rank holds the whole
model and sequences never change rank.  The general multi-GPU path is the SPMD
runtime (``spmd.py``): partial (hot-layer) replication, layer / sub-module
migration and KV following re-split sequences across processes, which is what
``bench.py --gpus N`` runs.  Here a re-split that would move a sequence to
another rank (the batch shrank) raises and names that path.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

from .ops import split_batch

PHASE_PREFILL, PHASE_DECODE = 0, 1


class ReplicaGroup:
    """Scatter / pass / gather of one replicated run across the process group."""

    def __init__(self, dist, executor, device: str | None = None):
        self.dist = dist
        self.ex = executor
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        backend = dist.get_backend()
        self.device = device or ("cuda" if backend == "nccl" else "cpu")
        self.owner: dict[int, int] = {}  # global slot -> rank holding its KV
        self.local: dict[int, int] = {}  # global slot -> this rank's executor slot
        self.free = list(range(getattr(getattr(executor, "cfg", None), "max_slots", 1 << 20) - 1, -1, -1))
        self.last_shares: list[int] = []

    # ------------------------------------------------------------ collectives
    def _bcast_i64(self, arr: np.ndarray | None, n: int):
        import torch

        t = torch.empty(n, dtype=torch.int64, device=self.device)
        if self.rank == 0:
            t.copy_(torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int64)))
        self.dist.broadcast(t, 0)
        return t.cpu().numpy()

    def scatter(self, phase: int | None = None, slots: Sequence[int] | None = None,
                tokens: Sequence[int] | None = None, lens: Sequence[int] | None = None):
        """Rank 0 passes the whole batch; every rank returns its share
        (phase, slots, tokens, lens, first sequence index)."""
        if self.rank == 0:
            slots = np.asarray(slots, dtype=np.int64)
            tokens = np.asarray(tokens, dtype=np.int64)
            lens = np.asarray(lens if lens is not None else np.ones(len(slots)), dtype=np.int64)
            head = np.array([phase, len(slots), len(tokens)], dtype=np.int64)
        else:
            head = None
        phase, bs, nt = (int(v) for v in self._bcast_i64(head, 3))
        body = np.concatenate([slots, tokens, lens]) if self.rank == 0 else None
        body = self._bcast_i64(body, 2 * bs + nt)
        slots, tokens, lens = body[:bs], body[bs:bs + nt], body[bs + nt:]
        shares = split_batch(bs, self.world)
        self.last_shares = shares
        s0 = sum(shares[:self.rank])
        s1 = s0 + shares[self.rank]
        tok_off = np.concatenate([[0], np.cumsum(lens)]) if phase == PHASE_PREFILL else np.arange(bs + 1)
        for j, r in enumerate(np.repeat(np.arange(self.world), shares)):
            g = int(slots[j])
            if phase == PHASE_PREFILL:
                self.owner[g] = int(r)
            elif self.owner.get(g, r) != r:
                raise NotImplementedError(
                    f"slot {g} would move from rank {self.owner[g]} to rank {r}: cross-process KV moves are "
                    "not done by the replica-group mode; use spmd.SpmdExecutor, which moves KV across ranks")
        mine = []
        for g in slots[s0:s1]:
            g = int(g)
            if g not in self.local:
                if phase != PHASE_PREFILL:
                    raise KeyError(f"slot {g} was never prefilled on rank {self.rank}")
                self.local[g] = self.free.pop()
            mine.append(self.local[g])
        return (phase, np.asarray(mine, dtype=np.int32), tokens[tok_off[s0]:tok_off[s1]].astype(np.int32),
                lens[s0:s1].astype(np.int32), s0)

    def gather(self, local_next: np.ndarray) -> np.ndarray | None:
        """Sampled tokens of every share, back on rank 0 in batch order."""
        import torch

        shares = self.last_shares
        m = max(shares) if shares else 0
        buf = torch.full((m,), -1, dtype=torch.int64, device=self.device)
        buf[:len(local_next)] = torch.from_numpy(np.asarray(local_next, dtype=np.int64))
        parts = [torch.empty(m, dtype=torch.int64, device=self.device) for _ in range(self.world)]
        self.dist.all_gather(parts, buf)
        if self.rank != 0:
            return None
        return np.concatenate([p.cpu().numpy()[:n] for p, n in zip(parts, shares)]).astype(np.int32)

    # ------------------------------------------------------------ one step
    def step(self, phase: int | None = None, slots=None, tokens=None, lens=None):
        """scatter -> local pass -> gather.  Returns (next tokens on rank 0 or
        None, this rank's device ms)."""
        ph, s, t, l, _ = self.scatter(phase, slots, tokens, lens)
        if len(s) == 0:
            nxt, ms = np.empty(0, np.int32), 0.0
        elif ph == PHASE_PREFILL:
            nxt, _, ms = self.ex.prefill(s, t, l)
        else:
            nxt, _, ms = self.ex.decode(s, t)
        return self.gather(nxt), ms

    def release(self, slots: Sequence[int]) -> None:
        """Every rank calls this with the same global slots (finished requests)."""
        gone = []
        for g in slots:
            g = int(g)
            self.owner.pop(g, None)
            if g in self.local:
                loc = self.local.pop(g)
                gone.append(loc)
                self.free.append(loc)
        if gone and hasattr(self.ex, "release_slots"):
            self.ex.release_slots(np.asarray(gone, dtype=np.int32))
