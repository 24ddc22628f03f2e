"""One process per GPU: module-level scaling across processes (SPMD).

The reference serves one instance whose decoder layers (and their replicas)
live on several devices of one box (PlacementState, domain.py:306-459); a
replicated run scatters the batch rows to the replicas and gathers them back
(``_comm_units``, _kernels.py:41-51), a migration moves a layer
block (+ KV) between devices (ops.py:199-258).  Here every GPU is driven by its
own process, and every process runs the SAME program:

* ``SpmdRuntime`` -- the global list of logical devices, device j owned by rank
  ``rank_of_device[j]`` (``cb_runtime_create_spmd``).  Each rank allocates and
  computes only for its own devices and keeps the registry / KV-ownership
  bookkeeping of all of them, so every rank knows every exchange.
* ``Transport`` -- the ``cb_xfer_fn`` the runtime calls for each byte range that
  crosses a process boundary, in the same global order on every rank:
  activation rows at replica-run boundaries, KV prefixes following their
  sequence when ``split_batch`` re-assigns it; and host messages: the CUDA
  IPC handle of a layer block being replicated / migrated or of a KV block a
  scaling op moves, which the destination's rank maps and pulls with its own
  copy engines over NVLink (not through the collective library).  ``mode="nccl"``: zero-copy views of
  the library's device buffers, ``batch_isend_irecv`` on the stream the library
  names (NCCL over NVLink; one communicator per channel: per-step exchanges on
  the compute streams, op transfers on the copy streams).  ``mode="host"``:
  staged through host memory over gloo (CPU tests / several ranks on one GPU).
* ``SpmdGroup`` -- the lockstep of the host programs: rank 0 (the router's home,
  ``Engine._dispatch_arrivals``, sim.py:628-629) broadcasts each step's inputs
  and the sampled tokens over a gloo group, so every rank takes the same
  decisions; a scaling op is issued on every rank, the ranks agree on its
  outcome (the destination's reservation may fail: InfeasibleOpError
  everywhere) and only then start the transfer (``cb_op_start``).
* ``SpmdExecutor`` -- ``Executor`` with those rules (``load_layer`` on other
  ranks' devices registers the copy without bytes; ``issue`` / ``apply`` agree
  first).
"""
from __future__ import annotations

import ctypes as C
import traceback
import weakref
from typing import Mapping, Sequence

import numpy as np

from . import _lib
from . import ops as O
from .domain import ClusterSpec, ModuleCatalog, Replica
from .executor import Executor, ExecutorConfig, OpMeasurement, Runtime


class _DevBuf:
    """Zero-copy CUDA-array-interface view of a library-owned device buffer."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


class Transport:
    """``cb_xfer_fn`` over torch.distributed (see the module docstring)."""

    GROUP_BEGIN, GROUP_END = 2, 3

    HOST_SEND, HOST_RECV = 4, 5

    def __init__(self, dist, mode: str, device_index: int, groups: Sequence, host_group=None):
        import torch

        if mode not in ("nccl", "host"):
            raise ValueError("transport mode must be 'nccl' or 'host'")
        self.dist = dist
        self.torch = torch
        self.mode = mode
        self.device_index = device_index
        self.groups = list(groups)  # one per channel
        self.host_group = host_group  # gloo: host messages (CUDA IPC handles of layer blocks)
        self._batch: dict[int, list | None] = {0: None, 1: None}
        self.error: BaseException | None = None
        self.messages = 0
        self.bytes = 0
        self.cfn = _lib.XFER_FN(self._cb)  # kept alive as long as the transport
        if mode == "nccl":  # eager communicator init: every rank of each group takes part
            t = torch.zeros(1, device=f"cuda:{device_index}")
            for g in self.groups:
                dist.all_reduce(t, group=g)
            torch.cuda.synchronize(device_index)

    # called from libcocob200 (the ctypes callback re-enters Python)
    def _cb(self, ctx, channel, send, peer, ptr, nbytes, stream) -> int:
        try:
            if send == self.GROUP_BEGIN:
                self._batch[channel] = []
                return 0
            if send == self.GROUP_END:
                ops, self._batch[channel] = self._batch[channel] or [], None
                self._flush(channel, ops)
                return 0
            if send in (self.HOST_SEND, self.HOST_RECV):
                self._host_msg(send == self.HOST_SEND, int(peer), int(ptr), int(nbytes))
                return 0
            item = (bool(send), int(peer), int(ptr or 0), int(nbytes), int(stream or 0))
            self.messages += 1
            self.bytes += int(nbytes)
            if self._batch[channel] is not None:
                self._batch[channel].append(item)
            else:
                self._flush(channel, [item])
            return 0
        except BaseException as e:  # never unwind through C
            self.error = e
            traceback.print_exc()
            return 1

    def _host_msg(self, send: bool, peer: int, ptr: int, n: int) -> None:
        torch = self.torch
        if send:
            buf = torch.frombuffer(bytearray(C.string_at(ptr, n)), dtype=torch.uint8)
            self.dist.send(buf, peer, group=self.host_group)
        else:
            buf = torch.empty(n, dtype=torch.uint8)
            self.dist.recv(buf, peer, group=self.host_group)
            C.memmove(ptr, buf.data_ptr(), n)
        self.messages += 1
        self.bytes += n

    def _flush(self, channel: int, ops: list) -> None:
        if not ops:
            return
        if self.mode == "nccl":
            self._flush_nccl(channel, ops)
        else:
            self._flush_host(channel, ops)

    def _view(self, ptr: int, n: int):
        return self.torch.as_tensor(_DevBuf(ptr, n), device=f"cuda:{self.device_index}")

    def _flush_nccl(self, channel: int, ops: list) -> None:
        torch, dist = self.torch, self.dist
        g = self.groups[channel]
        i = 0
        while i < len(ops):  # runs of ops on one stream -> one NCCL group each
            j = i
            while j < len(ops) and ops[j][4] == ops[i][4]:
                j += 1
            p2p = [dist.P2POp(dist.isend if s else dist.irecv, self._view(ptr, n), peer, g)
                   for s, peer, ptr, n, _ in ops[i:j]]
            with torch.cuda.stream(torch.cuda.ExternalStream(ops[i][4], device=f"cuda:{self.device_index}")):
                for w in dist.batch_isend_irecv(p2p):
                    w.wait()  # NCCL: the stream waits, not the host
            i = j

    def _flush_host(self, channel: int, ops: list) -> None:
        torch, dist = self.torch, self.dist
        g = self.groups[channel]
        dev = f"cuda:{self.device_index}"
        pending = []
        for s, peer, ptr, n, st in ops:
            stream = torch.cuda.ExternalStream(st, device=dev)
            if s:
                stream.synchronize()
                host = self._view(ptr, n).cpu()
                pending.append((dist.isend(host, peer, group=g), host))
            else:
                host = torch.empty(n, dtype=torch.uint8)
                dist.recv(host, peer, group=g)
                with torch.cuda.stream(stream):
                    self._view(ptr, n).copy_(host)
                stream.synchronize()
        for w, _ in pending:
            w.wait()


class SpmdGroup:
    """Host lockstep of the SPMD ranks (gloo group; rank 0 is the router's home)."""

    def __init__(self, dist, meta_group=None):
        self.dist = dist
        self.group = meta_group
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()

    def bcast(self, arr: np.ndarray | None, src: int = 0) -> np.ndarray:
        """int64 array from `src` to every rank (length first)."""
        import torch

        n = torch.tensor([len(arr) if self.rank == src else 0], dtype=torch.int64)
        self.dist.broadcast(n, src, group=self.group)
        t = torch.empty(int(n.item()), dtype=torch.int64)
        if self.rank == src:
            t.copy_(torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int64)))
        self.dist.broadcast(t, src, group=self.group)
        return t.numpy()

    def allgather(self, vals: Sequence[int]) -> np.ndarray:
        """[world, len(vals)] int64 of every rank's values."""
        import torch

        t = torch.tensor(list(vals), dtype=torch.int64)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return torch.stack(out).numpy()

    def barrier(self) -> None:
        self.dist.barrier(group=self.group)


class SpmdRuntime(Runtime):
    """cb_runtime_create_spmd: the global device list, this rank's devices on one GPU."""

    def __init__(self, rank_of_device: Sequence[int], rank: int, cuda_ordinal: int, transport: Transport):
        self.lib = _lib.load()
        self.transport = transport
        self.rank = rank
        self.rank_of_device = list(rank_of_device)
        self.ordinals = [cuda_ordinal if r == rank else -1 for r in self.rank_of_device]
        arr = (C.c_int32 * len(self.rank_of_device))(*self.rank_of_device)
        h = C.c_void_p()
        _lib.check(self.lib.cb_runtime_create_spmd(len(arr), arr, rank, cuda_ordinal, transport.cfn, None,
                                                   C.byref(h)), "cb_runtime_create_spmd")
        self.handle = h
        self._models = weakref.WeakSet()

    def is_local(self, dev: int) -> bool:
        return self.rank_of_device[dev] == self.rank


class SpmdExecutor(Executor):
    """``Executor`` on an SPMD runtime: every rank makes the same calls."""

    def __init__(self, runtime: SpmdRuntime, cfg: ExecutorConfig, group: SpmdGroup, home_device: int = 0,
                 seed: int = 0):
        super().__init__(runtime, cfg, home_device=home_device, seed=seed)
        self.group = group
        self.home_rank = runtime.rank_of_device[home_device]

    # ---------------------------------------------------------------- weights
    def load_layer(self, layer: int, device: int, w) -> None:
        if self.rt.is_local(device):
            return super().load_layer(layer, device, w)
        _lib.check(self.lib.cb_layer_load(self.handle, layer, device, None), "cb_layer_load")
        self._rows[layer - 1] = (Replica(device, True),)

    def load_head(self, embed, final_norm, lm_head) -> None:
        if self.rt.is_local(self.home):
            return super().load_head(embed, final_norm, lm_head)
        _lib.check(self.lib.cb_head_load(self.handle, None, None, None), "cb_head_load")

    # ---------------------------------------------------------------- scaling ops
    def issue(self, op, catalog: ModuleCatalog, cluster: ClusterSpec, cost_model: O.OpCostModel = O.DEFAULT_COST_MODEL,
              extra_used_mb: Mapping[int, float] | None = None,
              kv_mb_by_layer: Mapping[int, float] | None = None) -> int:
        """Registry apply (identical on every rank), reservation on the
        destination's rank, agreement, then the transfer (send on the source's
        rank, receive on the destination's) while serving continues."""
        base = self._pending_placement if self._pending else self.placement
        new_p, _ = O.apply(base, op, catalog, cluster, cost_model, extra_used_mb, kv_mb_by_layer)
        oid, sf = C.c_int64(), C.c_uint64()
        if isinstance(op, O.ReplicateLayer):
            rc = self.lib.cb_issue_replicate_layer(self.handle, op.layer, op.dst_device, C.byref(oid), C.byref(sf))
        elif isinstance(op, O.MigrateLayer):
            rc = self.lib.cb_issue_migrate_layer(self.handle, op.layer, op.dst_device, int(op.with_kv), C.byref(oid),
                                                 C.byref(sf))
        elif isinstance(op, O.MigrateSubModule):
            rc = self.lib.cb_issue_migrate_submodule(self.handle, op.layer, _lib.KIND_IDS[op.kind.value],
                                                     op.dst_device, C.byref(oid), C.byref(sf))
        elif isinstance(op, O.EvictReplica):
            rc = self.lib.cb_issue_evict_replica(self.handle, op.layer, op.device, C.byref(oid))
        else:
            raise O.OpError(f"unknown op {op!r}")
        mine = _lib.last_error() if rc else ""
        votes = self.group.allgather([rc, sf.value, oid.value])
        ids = set(int(v) for v in votes[:, 2])
        if len(ids) != 1:
            raise RuntimeError(f"SPMD op ids diverged: {sorted(ids)}")
        worst = int(votes[:, 0].min())
        if worst != _lib.CB_OK:
            if rc == _lib.CB_OK:
                _lib.check(self.lib.cb_op_abort(self.handle, oid.value), "cb_op_abort")
            who = int(np.argmin(votes[:, 0]))
            _lib.raise_status(worst, f"issue {type(op).__name__} (rank {who}){': ' + mine if mine else ''}",
                              int(votes[:, 1].max()))
        _lib.check(self.lib.cb_op_start(self.handle, oid.value), "cb_op_start")
        self._pending.append((op, oid.value))
        self._pending_placement = new_p
        return oid.value

    def commit(self, wait: bool = False):
        """Every rank's part of every pending op finishes before any rank
        switches: a layer block is pulled by the destination's rank straight
        from the source's memory (CUDA IPC), and a migration frees the source
        block at the switch."""
        for _, oid in self._pending:
            _lib.check(self.lib.cb_op_wait(self.handle, oid, None), "cb_op_wait")
        if self._pending:
            self.group.barrier()
        return super().commit(wait)

    def apply(self, op, catalog: ModuleCatalog, cluster: ClusterSpec, cost_model: O.OpCostModel = O.DEFAULT_COST_MODEL,
              extra_used_mb: Mapping[int, float] | None = None,
              kv_mb_by_layer: Mapping[int, float] | None = None):
        """Synchronous form: issue, commit and wait (this rank's side of the copy)."""
        if self._pending:
            raise O.OpError("scaling ops are pending: commit() or abort() them first")
        _, analytic = O.apply(self.placement, op, catalog, cluster, cost_model, extra_used_mb, kv_mb_by_layer)
        self.issue(op, catalog, cluster, cost_model, extra_used_mb, kv_mb_by_layer)
        self.commit(wait=True)
        m: OpMeasurement = self.op_log[-1]
        return self.placement, O.TransitionCost(m.device_ms / 1e3, analytic.transient_memory_mb)

    # ---------------------------------------------------------------- lockstep passes
    def _lockstep(self, phase, slots, tokens, lens, want_logits):
        g = self.group
        head = np.array([len(slots), len(tokens)], dtype=np.int64) if g.rank == 0 else None
        bs, nt = (int(v) for v in g.bcast(head))
        body = np.concatenate([slots, tokens, lens if lens is not None else []]) if g.rank == 0 else None
        body = g.bcast(body)
        slots, tokens = body[:bs].astype(np.int32), body[bs:bs + nt].astype(np.int32)
        lens = body[bs + nt:].astype(np.int32) if phase == _lib.PHASE_PREFILL else None
        nxt, logits, ms = Executor._pass(self, phase, slots, tokens, lens, want_logits and g.rank == self.home_rank)
        nxt = g.bcast(nxt if g.rank == self.home_rank else None, src=self.home_rank).astype(np.int32)
        return nxt, logits, ms

    def prefill(self, slots, tokens, prompt_lens, want_logits: bool = False):
        """Every rank calls this; rank 0's arguments are the ones used."""
        return self._lockstep(_lib.PHASE_PREFILL, slots, tokens, prompt_lens, want_logits)

    def decode(self, slots, tokens, want_logits: bool = False):
        return self._lockstep(_lib.PHASE_DECODE, slots, tokens, None, want_logits)

    def release_slots(self, slots) -> None:
        body = self.group.bcast(np.asarray(slots) if self.group.rank == 0 else None)
        super().release_slots(body.astype(np.int32))


def init_spmd(dist, rank: int, world: int, cuda_ordinal: int, mode: str = "nccl",
              devices_per_rank: int = 1) -> tuple[SpmdGroup, Transport, list[int]]:
    """Process groups of the SPMD runtime: a gloo group for the host lockstep and
    one transport group per channel.  Returns (group, transport, rank_of_device)."""
    backend = "nccl" if mode == "nccl" else "gloo"
    meta = dist.new_group(backend="gloo")
    chans = [dist.new_group(backend=backend) for _ in range(2)]
    host = dist.new_group(backend="gloo")
    transport = Transport(dist, mode, cuda_ordinal, chans, host_group=host)
    rank_of_device = [r for r in range(world) for _ in range(devices_per_rank)]
    return SpmdGroup(dist, meta), transport, rank_of_device
