"""B200 executor: the physical side of the registry, operator and step hook.

``Executor`` owns one ``cb_model`` in libcocob200 (weights, per-replica KV
cache, activation workspaces on every logical device) and keeps the Python
registry (``PlacementState``) and the device plan in lock-step:

* ``apply(op, ...)`` = reference ``ops.apply`` (feasibility against the
  cluster spec, placement edit) followed by the physical op -- the layer
  block / KV bytes moved peer-to-peer by the copy engine (NVLink on a
  multi-GPU box).  The Table-2 lookup of the reference (ops.py:90-148) is
  replaced by the measured copy time; the op log records bytes and GB/s.
* ``step_batch(batch, phase)`` = reference ``step_batch`` (sim.py:269-300)
  executed for real: prefill of fresh requests / one decode step, rows routed
  to each layer's replicas with ``split_batch`` (ops.py:151-158).

One host thread drives all logical devices (the reference's single-writer
rule).  Logical devices map to CUDA ordinals; several may
share one GPU, which is how the multi-device paths are exercised on a
single B200.
"""
from __future__ import annotations

import ctypes as C
import time
import weakref
from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

from . import _lib
from . import ops as O
from .domain import ClusterSpec, ModuleCatalog, ModuleKind, PlacementState, Replica
from .sim import Request, StepOutcome


@dataclass(frozen=True)
class ExecutorConfig:
    """Geometry + capacities of one served model instance."""

    n_layers: int
    d_model: int
    d_ff: int
    n_heads: int
    n_kv_heads: int | None = None  # None = MHA (the reference's accounting); < n_heads = GQA extension
    vocab: int = 32000
    max_slots: int = 64
    max_ctx: int = 512
    max_tokens: int = 8192
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5

    def desc(self) -> _lib.ModelDesc:
        return _lib.ModelDesc(self.n_layers, self.d_model, self.d_ff, self.n_heads,
                              self.n_kv_heads or self.n_heads, self.vocab, self.max_slots, self.max_ctx,
                              self.max_tokens, self.rope_theta, self.norm_eps)


class Runtime:
    """Logical devices bound to CUDA ordinals (cb_runtime)."""

    def __init__(self, cuda_ordinals: Sequence[int] = (0,)):
        self.lib = _lib.load()
        self.ordinals = list(cuda_ordinals)
        arr = (C.c_int32 * len(self.ordinals))(*self.ordinals)
        h = C.c_void_p()
        _lib.check(self.lib.cb_runtime_create(len(self.ordinals), arr, C.byref(h)), "cb_runtime_create")
        self.handle = h
        self._models = weakref.WeakSet()  # executors on this runtime: closed before it

    @property
    def n_devices(self) -> int:
        return len(self.ordinals)

    def device_info(self, dev: int) -> dict:
        sms, free, total = C.c_int32(), C.c_uint64(), C.c_uint64()
        _lib.check(self.lib.cb_device_info(self.handle, dev, C.byref(sms), C.byref(free), C.byref(total)))
        return {"num_sms": sms.value, "free_bytes": free.value, "total_bytes": total.value}

    COPY_SINGLE, COPY_CHUNKED, COPY_SM = 0, 1, 2

    def set_copy_mode(self, mode: int, chunk_bytes: int = 0) -> None:
        """Transfer engine of the scaling ops (cb_set_copy_mode): COPY_SINGLE = one
        cudaMemcpyPeerAsync, COPY_CHUNKED = chunks alternating over two copy
        engines (default, 64 MB), COPY_SM = an SM kernel on the source GPU pushing
        16-byte stores into the destination."""
        _lib.check(self.lib.cb_set_copy_mode(self.handle, int(mode), int(chunk_bytes)), "cb_set_copy_mode")

    def close(self) -> None:
        if self.handle:
            for ex in list(self._models):  # a model must never outlive its runtime
                ex.close()
            self.lib.cb_runtime_destroy(self.handle)
            self.handle = None


@dataclass
class OpMeasurement:
    """What one physical scaling op moved and how fast (device-timed)."""

    op: object
    weight_bytes: int
    kv_bytes: int
    device_ms: float
    copy_ms: float | None = None      # asynchronous ops: transfer (overlapped with serving)
    catchup_ms: float | None = None   # asynchronous ops: KV appended meanwhile, copied at the commit
    catchup_bytes: int | None = None

    @property
    def gbps(self) -> float:
        return (self.weight_bytes + self.kv_bytes) / (self.device_ms * 1e6) if self.device_ms > 0 else 0.0


@dataclass
class _Slots:
    free: list = field(default_factory=list)


class Executor:
    """One model instance served on B200 logical devices."""

    def __init__(self, runtime: Runtime, cfg: ExecutorConfig, home_device: int = 0, seed: int = 0):
        self.rt = runtime
        self.lib = runtime.lib
        self.cfg = cfg
        self.home = home_device
        self.seed = seed
        h = C.c_void_p()
        desc = cfg.desc()
        _lib.check(self.lib.cb_model_create(runtime.handle, C.byref(desc), home_device, C.byref(h)), "cb_model_create")
        self.handle = h
        runtime._models.add(self)
        self._rows: list = [None] * cfg.n_layers  # registry rows as layers get loaded
        self._overrides: list = []
        self._slots = list(range(cfg.max_slots - 1, -1, -1))
        self.op_log: list[OpMeasurement] = []
        self._pending: list[tuple[object, int]] = []  # issued, uncommitted ops (op, op_id)
        self._pending_placement: PlacementState | None = None
        self._unresolved: list[tuple[object, int]] = []  # committed ops whose timings are not read yet
        self.last_step_ms = 0.0
        self.kv_offload_fraction = 0.0

    # ------------------------------------------------------------ weights
    def load_layer(self, layer: int, device: int, w) -> None:
        """Load bf16 (uint16) weights; the first copy of a layer is its original."""
        arrs = {k: np.ascontiguousarray(getattr(w, k), dtype=np.uint16) for k in
                ("attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")}
        c = self.cfg
        hd = c.d_model // c.n_heads
        kvd = (c.n_kv_heads or c.n_heads) * hd
        want = {"attn_norm": (c.d_model,), "wq": (c.n_heads * hd, c.d_model), "wk": (kvd, c.d_model),
                "wv": (kvd, c.d_model), "wo": (c.d_model, c.n_heads * hd), "ffn_norm": (c.d_model,),
                "w_gate": (c.d_ff, c.d_model), "w_up": (c.d_ff, c.d_model), "w_down": (c.d_model, c.d_ff)}
        for k, shape in want.items():  # the C side reads exactly these extents from the host pointers
            if arrs[k].shape != shape:
                raise O.OpError(f"layer {layer} {k}: shape {arrs[k].shape}, expected {shape} (PyTorch [out, in])")
        lw = _lib.LayerWeights(*[a.ctypes.data for a in arrs.values()])
        _lib.check(self.lib.cb_layer_load(self.handle, layer, device, C.byref(lw)), "cb_layer_load")
        self._rows[layer - 1] = (Replica(device, True),)

    def init_layer_random(self, layer: int, device: int, std: float = 0.02) -> None:
        _lib.check(self.lib.cb_layer_init_random(self.handle, layer, device, self.seed, std), "cb_layer_init_random")
        self._rows[layer - 1] = (Replica(device, True),)

    def load_head(self, embed: np.ndarray, final_norm: np.ndarray, lm_head: np.ndarray) -> None:
        e, f, h = (np.ascontiguousarray(a, dtype=np.uint16) for a in (embed, final_norm, lm_head))
        c = self.cfg
        for name, a, shape in (("embed", e, (c.vocab, c.d_model)), ("final_norm", f, (c.d_model,)),
                               ("lm_head", h, (c.vocab, c.d_model))):
            if a.shape != shape:
                raise O.OpError(f"{name}: shape {a.shape}, expected {shape}")
        _lib.check(self.lib.cb_head_load(self.handle, e.ctypes.data, f.ctypes.data, h.ctypes.data), "cb_head_load")

    def init_head_random(self, std: float = 0.02) -> None:
        _lib.check(self.lib.cb_head_init_random(self.handle, self.seed, std), "cb_head_init_random")

    def load_model(self, weights, device_of_layer=None) -> None:
        """Load oracle-format ModelWeights; layer li goes to device_of_layer(li)."""
        pick = device_of_layer if callable(device_of_layer) else (lambda li: self.home if device_of_layer is None
                                                                  else device_of_layer)
        self.load_head(weights.embed, weights.final_norm, weights.lm_head)
        for li, lw in enumerate(weights.layers, 1):
            self.load_layer(li, pick(li), lw)

    # ------------------------------------------------------------ registry mirror
    @property
    def placement(self) -> PlacementState:
        if any(r is None for r in self._rows):
            raise RuntimeError("not every decoder layer is loaded")
        return PlacementState(tuple(self._rows), tuple(self._overrides))

    def _set_placement(self, p: PlacementState) -> None:
        self._rows = list(p.replicas)
        self._overrides = list(p.overrides)

    def device_plan(self) -> tuple[list[int], list[int], list[int]]:
        """(layer_ptr, replica devices in CSR order, KV device per layer) as the device sees it."""
        n = self.cfg.n_layers
        cap = n * max(1, self.rt.n_devices)
        ptr = (C.c_int64 * (n + 1))()
        devs = (C.c_int32 * cap)()
        kv = (C.c_int32 * n)()
        _lib.check(self.lib.cb_get_placement(self.handle, ptr, devs, cap, kv))
        return list(ptr), list(devs)[: ptr[n]], list(kv)

    def check_plan(self) -> None:
        """Registry and device plan must agree (replica order and KV residency)."""
        p = self.placement
        ptr, devs, kv = self.device_plan()
        want_devs = [r.device_id for row in p.replicas for r in row]
        want_ptr = [0]
        for row in p.replicas:
            want_ptr.append(want_ptr[-1] + len(row))
        want_kv = [p.kv_device(li) for li in range(1, p.n_layers + 1)]
        if (ptr, devs, kv) != (want_ptr, want_devs, want_kv):
            raise RuntimeError(f"device plan {ptr, devs, kv} != registry {want_ptr, want_devs, want_kv}")

    # ------------------------------------------------------------ scaling ops
    def apply(self, op, catalog: ModuleCatalog, cluster: ClusterSpec, cost_model: O.OpCostModel = O.DEFAULT_COST_MODEL,
              extra_used_mb: Mapping[int, float] | None = None,
              kv_mb_by_layer: Mapping[int, float] | None = None) -> tuple[PlacementState, O.TransitionCost]:
        """Registry apply (reference semantics, errors and placement) + physical move,
        synchronously (issue, commit and wait at once; use ``issue`` / ``commit``
        to keep serving while the bytes move).

        Returns the new placement and a TransitionCost whose time is the
        measured copy time; the analytic cost of the reference is
        ``ops.apply(...)[1]``."""
        if self._pending:
            raise O.OpError("scaling ops are pending: commit() or abort() them first")
        new_p, analytic = O.apply(self.placement, op, catalog, cluster, cost_model, extra_used_mb, kv_mb_by_layer)
        st = _lib.OpStats()
        if isinstance(op, O.ReplicateLayer):
            rc = self.lib.cb_replicate_layer(self.handle, op.layer, op.dst_device, C.byref(st))
        elif isinstance(op, O.MigrateLayer):
            rc = self.lib.cb_migrate_layer(self.handle, op.layer, op.dst_device, int(op.with_kv), C.byref(st))
        elif isinstance(op, O.MigrateSubModule):
            rc = self.lib.cb_migrate_submodule(self.handle, op.layer, _lib.KIND_IDS[op.kind.value], op.dst_device,
                                               C.byref(st))
        elif isinstance(op, O.EvictReplica):
            rc = self.lib.cb_evict_replica(self.handle, op.layer, op.device, C.byref(st))
        else:
            raise O.OpError(f"unknown op {op!r}")
        _lib.check(rc, type(op).__name__, st.shortfall_bytes)
        self._set_placement(new_p)
        self.check_plan()
        m = OpMeasurement(op, st.weight_bytes, st.kv_bytes, st.device_ms)
        self.op_log.append(m)
        return new_p, O.TransitionCost(st.device_ms / 1e3, analytic.transient_memory_mb)

    # ------------------------------------------------------------ asynchronous scaling ops (A17)
    def issue(self, op, catalog: ModuleCatalog, cluster: ClusterSpec, cost_model: O.OpCostModel = O.DEFAULT_COST_MODEL,
              extra_used_mb: Mapping[int, float] | None = None,
              kv_mb_by_layer: Mapping[int, float] | None = None) -> int:
        """Start a scaling op without stopping service (the reference's
        transition, sim.py:396-403 / 812-841): the registry ``apply`` runs on the
        placement after every op issued so far (errors as ``ops.apply``), the
        destination memory is reserved now, the bytes move on the copy streams
        while ``step_batch`` keeps serving the committed placement, and
        ``commit()`` switches every issued op at a step boundary
        (sim.py:614-622).  Returns the op id."""
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
        _lib.check(rc, "issue " + type(op).__name__, sf.value)
        self._pending.append((op, oid.value))
        self._pending_placement = new_p
        return oid.value

    @property
    def pending_ops(self) -> list:
        return [op for op, _ in self._pending]

    def ops_done(self) -> bool:
        """Every issued op's transfer has finished (non-blocking)."""
        done = C.c_int32()
        for _, oid in self._pending:
            _lib.check(self.lib.cb_op_poll(self.handle, oid, C.byref(done)))
            if not done.value:
                return False
        return True

    def commit(self, wait: bool = False) -> PlacementState:
        """Switch every issued op at this step boundary (no host wait: the next
        step is stream-ordered after the transfers and the KV catch-up).  The
        measured times are read after the next step (``op_log``), or now with
        ``wait`` (blocks until the copies finished)."""
        if not self._pending:
            return self.placement
        n = C.c_int32()
        _lib.check(self.lib.cb_commit(self.handle, -1, C.byref(n)), "cb_commit")
        self._set_placement(self._pending_placement)
        self._unresolved.extend(self._pending)
        self._pending, self._pending_placement = [], None
        self.check_plan()
        if wait:
            self._resolve_ops()
        return self.placement

    def abort(self) -> None:
        """Release every uncommitted op's reservation; the executor is exactly as before."""
        if self._pending:
            _lib.check(self.lib.cb_op_abort(self.handle, -1), "cb_op_abort")
        self._pending, self._pending_placement = [], None

    def op_stats(self, op_id: int, wait: bool = True) -> dict:
        st = _lib.OpStats()
        if wait:
            _lib.check(self.lib.cb_op_wait(self.handle, op_id, C.byref(st)))
        else:
            done = C.c_int32()
            _lib.check(self.lib.cb_op_poll(self.handle, op_id, C.byref(done)))
            if not done.value:
                return {"done": False}
            _lib.check(self.lib.cb_op_wait(self.handle, op_id, C.byref(st)))
        return {f: getattr(st, f) for f, _ in _lib.OpStats._fields_}

    def _resolve_ops(self) -> None:
        for op, oid in self._unresolved:
            st = self.op_stats(oid)
            m = OpMeasurement(op, st["weight_bytes"], st["kv_bytes"], st["device_ms"])
            m.copy_ms, m.catchup_ms, m.catchup_bytes = st["copy_ms"], st["catchup_ms"], st["catchup_bytes"]
            self.op_log.append(m)
        self._unresolved = []

    def mem_usage(self, device: int) -> dict:
        """Bytes the executor holds on a logical device (+ allocatable bytes)."""
        ms = _lib.MemStats()
        _lib.check(self.lib.cb_mem_usage(self.handle, device, C.byref(ms)))
        return {f: getattr(ms, f) for f, _ in _lib.MemStats._fields_}

    # ------------------------------------------------------------ KV slots
    def acquire_slot(self) -> int:
        if not self._slots:
            raise RuntimeError("no free KV slot (max_slots reached)")
        return self._slots.pop()

    def release(self, requests: Sequence[Request]) -> None:
        slots = [r.slot for r in requests if r.slot is not None]
        if slots:
            arr = np.asarray(slots, dtype=np.int32)
            _lib.check(self.lib.cb_release_slots(self.handle, len(arr), _lib.i32(arr)))
            self._slots.extend(reversed(slots))
        for r in requests:
            r.slot = None

    def release_slots(self, slots: np.ndarray) -> None:
        """Free KV slots by id (callers that manage their own slot ids, e.g. dist.ReplicaGroup)."""
        arr = np.ascontiguousarray(slots, dtype=np.int32)
        _lib.check(self.lib.cb_release_slots(self.handle, len(arr), _lib.i32(arr)))

    def release_all(self) -> None:
        """Free every KV slot (end of a benchmark phase)."""
        arr = np.arange(self.cfg.max_slots, dtype=np.int32)
        _lib.check(self.lib.cb_release_slots(self.handle, len(arr), _lib.i32(arr)))
        self._slots = list(range(self.cfg.max_slots - 1, -1, -1))

    # ------------------------------------------------------------ passes
    def prefill(self, slots: np.ndarray, tokens: np.ndarray, prompt_lens: np.ndarray,
                want_logits: bool = False) -> tuple[np.ndarray, np.ndarray | None, float]:
        return self._pass(_lib.PHASE_PREFILL, slots, tokens, prompt_lens, want_logits)

    def decode(self, slots: np.ndarray, tokens: np.ndarray,
               want_logits: bool = False) -> tuple[np.ndarray, np.ndarray | None, float]:
        return self._pass(_lib.PHASE_DECODE, slots, tokens, None, want_logits)

    def _pass(self, phase, slots, tokens, lens, want_logits):
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        bs = len(slots)
        nxt = np.empty(bs, dtype=np.int32)
        logits = np.empty((bs, self.cfg.vocab), dtype=np.float32) if want_logits else None
        ms = C.c_float()
        lp = None
        if lens is not None:
            lens = np.ascontiguousarray(lens, dtype=np.int32)
            lp = _lib.i32(lens)
        rc = self.lib.cb_step(self.handle, phase, bs, _lib.i32(slots), _lib.i32(tokens), lp, _lib.i32(nxt),
                              _lib.f32(logits) if logits is not None else None, C.byref(ms))
        _lib.check(rc, "cb_step")
        self.last_step_ms = ms.value
        if self._unresolved:  # committed ops ran before this step: their timings are final
            self._resolve_ops()
        return nxt, logits, ms.value

    def synthetic_prompt(self, req: Request) -> np.ndarray:
        rng = np.random.default_rng((self.seed, req.id))
        return rng.integers(0, self.cfg.vocab, req.prompt_len, dtype=np.int64).astype(np.int32)

    def step_batch(self, batch: Sequence[Request], phase: str) -> StepOutcome:
        """The reference's executor hook, run on the GPUs (sim.py:269-300).

        prefill: every request in ``batch`` must be fresh; its prompt is
        processed in one pass and its first token sampled.  decode: one token
        for every request (its last output token is the input)."""
        if not batch:
            return StepOutcome(0.0, 0)
        if phase == "prefill":
            for r in batch:
                if r.slot is None:
                    r.slot = self.acquire_slot()
                if r.prompt_tokens is None:
                    r.prompt_tokens = self.synthetic_prompt(r)
            slots = np.array([r.slot for r in batch], dtype=np.int32)
            toks = np.concatenate([np.asarray(r.prompt_tokens, dtype=np.int32) for r in batch])
            lens = np.array([r.prompt_len for r in batch], dtype=np.int32)
            nxt, _, ms = self.prefill(slots, toks, lens)
            for r, t in zip(batch, nxt):
                r.output_tokens.append(int(t))
            return StepOutcome(ms / 1e3, int(lens.sum()), nxt)
        if phase == "decode":
            slots = np.array([r.slot for r in batch], dtype=np.int32)
            toks = np.array([r.output_tokens[-1] for r in batch], dtype=np.int32)
            nxt, _, ms = self.decode(slots, toks)
            for r, t in zip(batch, nxt):
                r.output_tokens.append(int(t))
            return StepOutcome(ms / 1e3, len(batch), nxt)
        raise ValueError(f"unknown phase {phase!r}")

    # ------------------------------------------------------------ Phase-3 KV offload
    def set_kv_offload(self, fraction: float) -> list[OpMeasurement]:
        """Offload a fraction of the KV cache off-device (the reference's Phase-3
        ``PerformanceReduction.new_offload_fraction``, autoscaler.py:568-583).

        The reference scales every layer's KV by (1 - f) (sim.py:500-505); the
        physical unit here is a layer's KV block, so layers 1..round(f * n_layers)
        keep their KV in mapped pinned host memory (attention reads it in place)
        and the rest return to HBM.  Returns the per-layer move measurements."""
        if not 0.0 <= fraction <= 1.0:
            raise ValueError("offload fraction must be in [0, 1]")
        n_off = int(round(fraction * self.cfg.n_layers))
        self.kv_offload_fraction = fraction
        out = []
        for li in range(1, self.cfg.n_layers + 1):
            want = li <= n_off
            if want == self.kv_offloaded(li):
                continue
            st = _lib.OpStats()
            _lib.check(self.lib.cb_kv_offload(self.handle, li, int(want), C.byref(st)), "cb_kv_offload")
            out.append(OpMeasurement(("kv_offload" if want else "kv_reload", li), 0, st.kv_bytes, st.device_ms))
        return out

    def kv_offloaded(self, layer: int) -> bool:
        v = C.c_int32()
        _lib.check(self.lib.cb_kv_offloaded(self.handle, layer, C.byref(v)))
        return bool(v.value)

    # ------------------------------------------------------------ profiling
    def profile(self, enable: bool) -> None:
        """Start (and reset) / stop per-launch CUDA-event timing inside cb_step."""
        _lib.check(self.lib.cb_profile(self.handle, int(enable)))

    def profile_read(self) -> dict:
        out = {}
        for i, name in enumerate(_lib.KCLASSES):
            k = _lib.KStat()
            _lib.check(self.lib.cb_profile_read(self.handle, i, C.byref(k)))
            out[name] = {"launches": k.launches, "ms": k.ms, "bytes": k.bytes, "flops": k.flops}
        return out

    # ------------------------------------------------------------ readback
    def module_bytes(self, kind: str | ModuleKind) -> int:
        k = kind.value if isinstance(kind, ModuleKind) else kind
        return int(self.lib.cb_module_bytes(self.handle, _lib.KIND_IDS[k]))

    def read_module(self, layer: int, device: int, kind: str | ModuleKind) -> np.ndarray:
        k = kind.value if isinstance(kind, ModuleKind) else kind
        n = self.module_bytes(k)
        out = np.empty(n // 2, dtype=np.uint16)
        _lib.check(self.lib.cb_module_read(self.handle, layer, device, _lib.KIND_IDS[k], out.ctypes.data, n),
                   "cb_module_read")
        return out

    def read_kv(self, layer: int, slot: int) -> tuple[np.ndarray, int]:
        ln = C.c_int32()
        _lib.check(self.lib.cb_slot_len(self.handle, slot, C.byref(ln)))
        n = ln.value * self.module_bytes("kv_cache")
        out = np.empty(n // 2, dtype=np.uint16)
        dev = C.c_int32()
        _lib.check(self.lib.cb_kv_read(self.handle, layer, slot, out.ctypes.data, n, C.byref(dev)), "cb_kv_read")
        return out, dev.value

    def last_routing(self, layer: int) -> list[tuple[int, int, int]]:
        """(device, first sequence, count) per replica of `layer` in the last step:
        split_batch counts over the step's sticky routing order (cb_step)."""
        cap = max(1, self.rt.n_devices)
        d, s, c, p = (C.c_int32 * cap)(), (C.c_int32 * cap)(), (C.c_int32 * cap)(), C.c_int32()
        _lib.check(self.lib.cb_last_routing(self.handle, layer, d, s, c, cap, C.byref(p)))
        return [(d[j], s[j], c[j]) for j in range(p.value)]

    def close(self) -> None:
        if getattr(self, "handle", None):
            self._pending, self._pending_placement = [], None
            self.lib.cb_model_destroy(self.handle)  # releases uncommitted reservations
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
