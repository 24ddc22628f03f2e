"""The reference auto-scaler driving the B200 data path.

The north star keeps the control plane as the reference's: this module runs
the *unmodified* ``modscale.autoscaler.controller_step`` (autoscaler.py:611-687,
Alg. 1 scale-up / Alg. 2 scale-down) on a view of the live executor, and
commits the ops it emits through ``Executor.apply`` -- the reference's
registry semantics plus the physical NVLink/HBM copies.  Types are converted
at the seam (frozen dataclasses with identical fields on both sides).

``modscale`` is imported from ``baseline/_ref`` (the offline pip install of
the reference) or, in the build container, from ``/root/reference/pkg/src``;
when neither exists, ``load_reference()`` returns None and callers skip.
"""
from __future__ import annotations

import importlib
import os
import sys
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
            sys.path.insert(0, str(cand))
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


class ReferenceController:
    """One executor instance under the reference controller.

    ``decide`` evaluates ``controller_step`` on the registry state (no side
    effects); ``commit`` applies the decision's ops physically, in order, at a
    step boundary (the reference's atomic switch, sim.py:614-622)."""

    def __init__(self, executor, cluster: D.ClusterSpec, model: D.ModelSpec, catalog: D.ModuleCatalog,
                 cfg=None, params=None, ms=None):
        self.ms = ms or load_reference()
        if self.ms is None:
            raise RuntimeError("reference modscale package not available")
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
        self.bs_cap: int | None = None  # last Phase-3 batch cap decided

    def view(self, bs: int, kv_tokens: float = 0.0, violation_rate: float = 0.0, busy: dict | None = None,
             mean_prompt_len: float = 0.0, mean_gen_len: float = 0.0, offload_fraction: float = 0.0):
        ms, A = self.ms, self.A
        pv = A.PressureView(cluster=self.r_cluster, model=self.r_model, catalog=self.r_catalog,
                            violation_rate=violation_rate, busy_fraction=busy or {}, kv_tokens=kv_tokens,
                            active_batch=bs, mean_prompt_len=mean_prompt_len, mean_gen_len=mean_gen_len)
        rp = to_ref_placement(ms, self.ex.placement)
        return A.InstanceView(instance_id=0, placement=rp, bs=bs, offload_fraction=offload_fraction, view=pv)

    def decide(self, bs: int, **kw):
        iv = self.view(bs, **kw)
        usage = self.ms.device_usage(iv.placement, self.r_catalog)
        full = {d.id: usage.get(d.id, self.ms.DeviceUsage()) for d in self.r_cluster.devices}
        return self.A.controller_step([iv], self.r_cluster, self.r_model, self.r_catalog, self.cfg, self.params, full)

    def commit(self, decision, kv_mb_by_layer: dict | None = None) -> list:
        """Apply the decision's scaling ops physically; returns [(op, measured cost)]."""
        done = []
        for phased in decision.ops:
            op = from_ref_op(phased.op)
            if type(op).__name__ == "PerformanceReduction":
                # Phase 3: the batch cap is the serving loop's (``self.bs_cap``); the
                # KV offload fraction is applied physically (host-resident KV blocks)
                self.bs_cap = op.new_bs
                if op.new_offload_fraction != self.ex.kv_offload_fraction:
                    self.ex.set_kv_offload(op.new_offload_fraction)
                continue
            if not isinstance(op, (O.ReplicateLayer, O.MigrateLayer, O.MigrateSubModule, O.EvictReplica)):
                continue
            _, cost = self.ex.apply(op, self.catalog, self.cluster, kv_mb_by_layer=kv_mb_by_layer)
            done.append((op, cost))
        if decision.placement is not None:
            want = from_ref_placement(decision.placement)
            if want.replicas != self.ex.placement.replicas or set(want.overrides) != set(self.ex.placement.overrides):
                raise RuntimeError("executor placement diverged from the reference controller's decision")
        self.log.append((decision.trigger, len(done)))
        return done


def apply_reference_ops(ms, placement: D.PlacementState, ref_ops: Sequence, catalog: D.ModuleCatalog,
                        cluster: D.ClusterSpec, kv_mb_by_layer: dict | None = None) -> D.PlacementState:
    """Registry-only replay of a reference op stream through our ``apply``."""
    p = placement
    for phased in ref_ops:
        op = from_ref_op(getattr(phased, "op", phased))
        if isinstance(op, (O.ReplicateLayer, O.MigrateLayer, O.MigrateSubModule, O.EvictReplica)):
            p, _ = O.apply(p, op, catalog, cluster, kv_mb_by_layer=kv_mb_by_layer)
    return p
