"""The reference auto-scaler driving the B200 data path.

The north star keeps the control plane as the reference's: this module runs
the *unmodified* ``modscale.autoscaler.controller_step`` (autoscaler.py:611-687,
Alg. 1 scale-up / Alg. 2 scale-down) on a view of the live executor, and
commits the ops it emits through the executor's asynchronous scaling ops --
the reference's registry semantics plus the physical NVLink/HBM copies.
Types are converted at the seam (frozen dataclasses with identical fields on
both sides).

What the controller sees (the reference Engine's ``_usage_by_device`` /
``_pressure_view``, sim.py:507-525, 740-762): the catalog accounting of the
placement (static module MB + resident KV tokens) plus, as
``extra_memory_mb``, the device memory the executor really holds that no
module explains -- activation / GEMM / attention workspaces (``cb_mem_usage``)
-- "foreign load" in the reference's words.  ``ServingEngine`` checks OOM
against exactly the same sum.  Physical overcommit the catalog cannot see
(a replica's KV block) surfaces as CB_ENOMEM when the op reserves its memory,
and the decision is then aborted whole.

How a decision is committed (the reference's transition, sim.py:396-403,
614-622, 812-841): ``issue`` starts every op (destination memory reserved
now); if any op fails -- registry infeasibility or a physical CB_ENOMEM --
the ops already issued are aborted and the executor is exactly as before
(``batch_apply``'s transactionality, ops.py:263-296).  The instance keeps
serving its old placement; ``commit_transition`` switches placement, batch
cap (Phase 3 ``new_bs``) and KV offload together at a step boundary once the
copies finished.  ``AutoscaleHook`` runs that loop inside ``ServingEngine``.

Dependency: the reference package ``modscale`` (autoscaler.py and its speedup
model), installed offline into ``baseline/_ref`` or, in the build container,
at ``/root/reference/pkg/src``.  It is appended to ``sys.path`` (never ahead
of anything else); without it ``load_reference()`` returns None.
"""
from __future__ import annotations

import importlib
import os
import sys
from dataclasses import dataclass, field
from pathlib import Path
from typing import Sequence

from . import domain as D
from . import ops as O

_ROOT = Path(__file__).resolve().parent.parent
_CANDIDATES = (_ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def load_reference():
    """Import the reference package ``modscale`` (or return None)."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")  # never write into the reference tree
    if "modscale" in sys.modules:
        return sys.modules["modscale"]
    for cand in _CANDIDATES:
        if (cand / "modscale" / "__init__.py").exists():
            if str(cand) not in sys.path:
                sys.path.append(str(cand))
            prev = sys.dont_write_bytecode
            sys.dont_write_bytecode = True
            try:
                return importlib.import_module("modscale")
            finally:
                sys.dont_write_bytecode = prev
    return None


# ------------------------------------------------------------------ type seam
def to_ref_placement(ms, p: D.PlacementState):
    rows = tuple(tuple(ms.Replica(r.device_id, r.is_original) for r in row) for row in p.replicas)
    ovr = tuple((li, ms.ModuleKind(k.value), dev) for li, k, dev in p.overrides)
    return ms.PlacementState(rows, ovr)


def from_ref_placement(rp) -> D.PlacementState:
    rows = tuple(tuple(D.Replica(r.device_id, r.is_original) for r in row) for row in rp.replicas)
    ovr = tuple((li, D.ModuleKind(k.value), dev) for li, k, dev in rp.overrides)
    return D.PlacementState(rows, ovr)


def to_ref_cluster(ms, c: D.ClusterSpec):
    return ms.ClusterSpec(tuple(ms.DeviceSpec(d.id, d.compute_gflops, d.memory_mb) for d in c.devices),
                          c.bandwidth_mbps)


def to_ref_catalog(ms, cat: D.ModuleCatalog):
    return ms.ModuleCatalog(**{k: getattr(cat, k) for k in cat.__dataclass_fields__})


def to_ref_model(ms, m: D.ModelSpec):
    return ms.ModelSpec(m.n_layers, m.d_model, m.d_ff, m.n_heads, m.dtype_bytes)


def from_ref_op(op):
    """Reference op dataclass -> ours (PerformanceReduction is returned as-is)."""
    name = type(op).__name__
    if name == "ReplicateLayer":
        return O.ReplicateLayer(op.layer, op.dst_device)
    if name == "MigrateLayer":
        return O.MigrateLayer(op.layer, op.dst_device, op.with_kv)
    if name == "MigrateSubModule":
        return O.MigrateSubModule(op.layer, D.ModuleKind(op.kind.value), op.dst_device)
    if name == "EvictReplica":
        return O.EvictReplica(op.layer, op.device)
    return op


_SCALING_OPS = (O.ReplicateLayer, O.MigrateLayer, O.MigrateSubModule, O.EvictReplica)


@dataclass
class Transition:
    """An issued decision waiting for its switch (reference ``_Transition``, sim.py:396-403)."""

    trigger: str
    ops: list                         # our scaling ops, issued in order
    placement: D.PlacementState       # the decision's placement (checked at the switch)
    bs: int | None                    # Phase-3 batch cap applied at the switch (None = unchanged)
    offload_fraction: float | None    # Phase-3 KV offload applied at the switch
    reserved_mb: dict = field(default_factory=dict)  # analytic reservation (sim.py:817-831)
    issued_s: float = 0.0


class ReferenceController:
    """One executor instance under the reference controller.

    ``decide`` evaluates ``controller_step`` on the live state (no side
    effects); ``issue`` / ``ready`` / ``commit_transition`` carry a decision
    out while serving continues; ``commit`` does all three at once."""

    def __init__(self, executor, cluster: D.ClusterSpec, model: D.ModelSpec, catalog: D.ModuleCatalog,
                 cfg=None, params=None, ms=None):
        self.ms = ms or load_reference()
        if self.ms is None:
            raise RuntimeError("reference modscale package not available (see control.py: Dependency)")
        from modscale import autoscaler as A  # noqa: WPS433 (reference control plane, kept as-is)

        self.A = A
        self.ex = executor
        self.cluster, self.model, self.catalog = cluster, model, catalog
        self.r_cluster = to_ref_cluster(self.ms, cluster)
        self.r_model = to_ref_model(self.ms, model)
        self.r_catalog = to_ref_catalog(self.ms, catalog)
        self.cfg = cfg or A.ControllerConfig()
        self.params = params or self.ms.SpeedupParams()
        self.log: list = []
        self.pending: Transition | None = None
        self.bs_cap: int | None = None  # batch cap of the last switch (AutoscaleHook applies it)

    # ------------------------------------------------------------ what the controller sees
    def foreign_mb(self) -> dict[int, float]:
        """Device memory no module accounts for: the executor's workspaces (MB
        per cluster device; 0 for registry-only stand-ins)."""
        return workspace_mb(self.ex, [d.id for d in self.cluster.devices])

    def _modeled_mb(self, placement: D.PlacementState, kv_tokens: float, offload: float) -> dict[int, float]:
        """The catalog's accounting of this placement (static + resident KV), per device."""
        usage = D.device_usage(placement, self.catalog)
        kv_count = D.kv_resident_layer_count(placement)
        kv_mb = kv_tokens * self.catalog.kv_bytes_per_token_per_layer / 1e6 * (1.0 - offload)
        return {d.id: (usage[d.id].memory_mb if d.id in usage else 0.0) + kv_count.get(d.id, 0) * kv_mb
                for d in self.cluster.devices}

    def view(self, bs: int, kv_tokens: float = 0.0, violation_rate: float = 0.0, busy: dict | None = None,
             mean_prompt_len: float = 0.0, mean_gen_len: float = 0.0, offload_fraction: float = 0.0,
             extra_memory_mb: dict | None = None):
        ms, A = self.ms, self.A
        placement = self.ex.placement
        if extra_memory_mb is None:
            extra_memory_mb = self.foreign_mb()
        pv = A.PressureView(cluster=self.r_cluster, model=self.r_model, catalog=self.r_catalog,
                            violation_rate=violation_rate, busy_fraction=busy or {}, kv_tokens=kv_tokens,
                            active_batch=bs, mean_prompt_len=mean_prompt_len, mean_gen_len=mean_gen_len,
                            extra_memory_mb=dict(extra_memory_mb))
        rp = to_ref_placement(ms, placement)
        return A.InstanceView(instance_id=0, placement=rp, bs=bs, offload_fraction=offload_fraction, view=pv)

    def usage_by_device(self, iv) -> dict:
        """Aggregate per-device usage the reference passes to controller_step
        (sim.py:516-525): this instance's modeled memory + its foreign load."""
        ms = self.ms
        static = ms.device_usage(iv.placement, self.r_catalog)
        out = {}
        for d in self.r_cluster.devices:
            mem = iv.view.current_memory_mb(iv.placement, d.id, iv.offload_fraction)
            comp = static[d.id].compute_gflops if d.id in static else 0.0
            out[d.id] = ms.DeviceUsage(mem, comp)
        return out

    def decide(self, bs: int, **kw):
        iv = self.view(bs, **kw)
        return self.A.controller_step([iv], self.r_cluster, self.r_model, self.r_catalog, self.cfg, self.params,
                                      self.usage_by_device(iv))

    # ------------------------------------------------------------ carrying a decision out
    def issue(self, decision, kv_mb_by_layer: dict | None = None, now_s: float = 0.0,
              kv_tokens: float = 0.0, offload_fraction: float = 0.0) -> Transition:
        """Start every op of the decision (transactional: on the first failure
        the issued ops are aborted and the error re-raised)."""
        if self.pending is not None:
            raise O.OpError("a transition is already pending (the controller skips busy instances, sim.py:765)")
        # Phase-3 PerformanceReduction ops carry no bytes: their new_bs / new_offload_fraction
        # are the decision's bs / offload_fraction, applied at the switch (sim.py:620)
        ops = [op for op in (from_ref_op(getattr(p, "op", p)) for p in decision.ops) if isinstance(op, _SCALING_OPS)]
        bs, off = decision.bs, decision.offload_fraction
        before = self.ex.placement
        try:
            for op in ops:
                self.ex.issue(op, self.catalog, self.cluster, kv_mb_by_layer=kv_mb_by_layer)
        except Exception:
            self.ex.abort()
            raise
        want = from_ref_placement(decision.placement) if decision.placement is not None else before
        tr = Transition(decision.trigger, ops, want, bs, off,
                        self._reservation_mb(before, want, kv_tokens, offload_fraction), now_s)
        self.pending = tr
        return tr

    def _reservation_mb(self, old: D.PlacementState, new: D.PlacementState, kv_tokens: float,
                        offload: float) -> dict:
        """Destination memory held from decision to switch (sim.py:817-831)."""
        a, b = self._modeled_mb(old, kv_tokens, offload), self._modeled_mb(new, kv_tokens, offload)
        return {d: b[d] - a[d] for d in b if b[d] - a[d] > 0}

    def ready(self) -> bool:
        return self.pending is not None and self.ex.ops_done()

    def commit_transition(self, wait: bool = False) -> Transition:
        """Switch at this step boundary: placement (all ops at once), then the
        Phase-3 KV offload; returns the transition (its ``bs`` is the caller's
        new batch cap, sim.py:620)."""
        tr = self.pending
        if tr is None:
            raise O.OpError("no pending transition")
        self.ex.commit(wait=wait) if _accepts_wait(self.ex) else self.ex.commit()
        if tr.offload_fraction is not None and tr.offload_fraction != getattr(self.ex, "kv_offload_fraction", 0.0):
            self.ex.set_kv_offload(tr.offload_fraction)
        p = self.ex.placement
        if tr.placement.replicas != p.replicas or set(tr.placement.overrides) != set(p.overrides):
            raise RuntimeError("executor placement diverged from the reference controller's decision")
        self.pending = None
        if tr.bs is not None:
            self.bs_cap = tr.bs
        self.log.append((tr.trigger, len(tr.ops)))
        return tr

    def commit(self, decision, kv_mb_by_layer: dict | None = None) -> list:
        """Issue + switch at once (callers between steps); returns [(op, measured cost)]."""
        tr = self.issue(decision, kv_mb_by_layer)
        n0 = len(getattr(self.ex, "op_log", []))
        self.commit_transition(wait=True)
        log = getattr(self.ex, "op_log", [])[n0:]
        return [(m.op, O.TransitionCost(m.device_ms / 1e3, 0.0)) for m in log] if log else \
            [(op, O.TransitionCost(0.0, 0.0)) for op in tr.ops]


def workspace_mb(ex, devices) -> dict[int, float]:
    out = {d: 0.0 for d in devices}
    if hasattr(ex, "mem_usage"):
        n_dev = getattr(getattr(ex, "rt", None), "n_devices", 0)
        for d in devices:
            if d < n_dev:
                out[d] = ex.mem_usage(d)["workspace_bytes"] / 1e6
    return out


def _accepts_wait(ex) -> bool:
    import inspect

    try:
        return "wait" in inspect.signature(ex.commit).parameters
    except (TypeError, ValueError):
        return False


class AutoscaleHook:
    """``ServingEngine.on_step`` hook: the reference Engine's controller loop
    (``_controller_tick`` every ``interval_s``, ``_commit_transitions`` at step
    boundaries, sim.py:614-622, 764-841) on the live executor.

    Pressure inputs follow the reference monitor: violation rate of the
    completions in the last ``window_s`` against ``slo_latency_s``; busy
    fraction of the home device from the step log; resident KV tokens and the
    batch from the instance."""

    def __init__(self, controller: ReferenceController, instance, interval_s: float = 1.0,
                 window_s: float = 5.0, slo_latency_s: float | None = None, prompt_len: float = 0.0,
                 gen_len: float = 0.0):
        self.ctl = controller
        self.inst = instance
        self.interval_s = interval_s
        self.window_s = window_s
        self.slo = slo_latency_s if slo_latency_s is not None else getattr(controller.cfg, "slo_latency_s", 1e9)
        self.prompt_len, self.gen_len = prompt_len, gen_len
        self.next_tick = interval_s
        self.decisions: list = []  # (t_s, trigger, n_ops, bs_after)
        self.switches: list = []   # (t_s, trigger, n_ops, issued_s)

    def __call__(self, eng, t_s: float) -> None:
        ctl, inst = self.ctl, self.inst
        if ctl.pending is not None and ctl.ready():
            tr = ctl.commit_transition()
            if tr.bs is not None:
                inst.max_batch_size = max(1, int(tr.bs))
            inst.offload_fraction = getattr(ctl.ex, "kv_offload_fraction", 0.0)
            inst.reserved_mb = {}
            self.switches.append((t_s, tr.trigger, len(tr.ops), tr.issued_s))
        if t_s < self.next_tick or ctl.pending is not None:
            return
        self.next_tick = t_s + self.interval_s
        recent = [r for r in eng.completed if r.completion_s is not None and r.completion_s >= t_s - self.window_s]
        viol = sum(1 for r in recent if r.failed or r.completion_s - r.arrival_s > self.slo) / len(recent) \
            if recent else 0.0
        busy = eng.busy_fraction(t_s, self.window_s)
        dec = ctl.decide(bs=inst.max_batch_size, kv_tokens=float(inst.resident_tokens), violation_rate=viol,
                         busy=busy, mean_prompt_len=self.prompt_len, mean_gen_len=self.gen_len,
                         offload_fraction=inst.offload_fraction)
        if dec.trigger == "none":
            return
        kv_layer_mb = inst.resident_tokens * ctl.catalog.kv_bytes_per_token_per_layer / 1e6
        try:
            tr = ctl.issue(dec, kv_mb_by_layer={li: kv_layer_mb for li in range(1, ctl.model.n_layers + 1)},
                           now_s=t_s, kv_tokens=float(inst.resident_tokens), offload_fraction=inst.offload_fraction)
        except (O.OpError, D.DomainError) as e:  # infeasible on the real devices: nothing was changed
            self.decisions.append((t_s, dec.trigger, 0, None, f"aborted: {e}"[:200]))
            return
        inst.reserved_mb = tr.reserved_mb
        self.decisions.append((t_s, dec.trigger, len(tr.ops), tr.bs, "issued"))


def apply_reference_ops(ms, placement: D.PlacementState, ref_ops: Sequence, catalog: D.ModuleCatalog,
                        cluster: D.ClusterSpec, kv_mb_by_layer: dict | None = None) -> D.PlacementState:
    """Registry-only replay of a reference op stream through our ``apply``."""
    p = placement
    for phased in ref_ops:
        op = from_ref_op(getattr(phased, "op", phased))
        if isinstance(op, _SCALING_OPS):
            p, _ = O.apply(p, op, catalog, cluster, kv_mb_by_layer=kv_mb_by_layer)
    return p
