"""The reference auto-scaler (unmodified) driving the drop-in registry (CPU).

``controller_step`` of the reference emits op streams (Alg. 1 scale-up,
Alg. 2 scale-down); replaying them through our ``apply`` must give exactly
the placement the reference decided.  The physical commit of such a decision
runs on the GPU in tests/test_control_gpu.py.
"""
from __future__ import annotations

import pytest

from paper_2507_18006_b200 import domain as D
from paper_2507_18006_b200 import ops as O
from paper_2507_18006_b200.control import (ReferenceController, apply_reference_ops, from_ref_placement,
                                           load_reference, to_ref_placement)

ms = load_reference()
pytestmark = pytest.mark.skipif(ms is None, reason="reference modscale not importable")


class RegistryOnlyExecutor:
    """Stand-in with the Executor's registry / op surface (no device)."""

    def __init__(self, placement):
        self.placement = placement
        self._pending, self._next = [], None

    def issue(self, op, catalog, cluster, kv_mb_by_layer=None):
        base = self._next if self._pending else self.placement
        self._next, _ = O.apply(base, op, catalog, cluster, kv_mb_by_layer=kv_mb_by_layer)
        self._pending.append(op)

    def ops_done(self):
        return True

    def commit(self):
        if self._pending:
            self.placement = self._next
        self._pending = []

    def abort(self):
        self._pending = []


def test_placement_roundtrip():
    p = D.PlacementState.sequential(6, 0).with_replica(2, 1).with_override(4, D.ModuleKind.KV_CACHE, 3)
    assert from_ref_placement(to_ref_placement(ms, p)) == p


def test_scale_up_7b_on_b200_box_matches_reference():
    """7B on an 8x B200 cluster spec: the reference scale-up replicates every
    layer on every device (SURVEY §7 hard part 7: P = [8]*32, 224 ops)."""
    model = D.ModelSpec(32, 4096, 11008, 32)
    cat = D.ModuleCatalog.from_model(model)
    cluster = D.ClusterSpec.b200(8)
    ex = RegistryOnlyExecutor(D.PlacementState.sequential(32, 0))
    ctl = ReferenceController(ex, cluster, model, cat, ms=ms)
    dec = ctl.decide(bs=16)
    assert dec.trigger == "scale_up"
    ref_final = from_ref_placement(dec.placement)
    ours = apply_reference_ops(ms, D.PlacementState.sequential(32, 0), dec.ops, cat, cluster)
    assert ours == ref_final
    ctl.commit(dec)
    assert ex.placement == ref_final
    assert ex.placement.p_vector() == (8,) * 32
    assert len(dec.ops) == 224


def test_scale_down_kv_migration_matches_reference():
    """Memory pressure on device 0 (13B, small devices): the reference's
    Alg. 2 picks KV / layer migrations; our registry reproduces its placement."""
    model = D.ModelSpec(40, 5120, 13824, 40)
    cat = D.ModuleCatalog.from_model(model)
    cluster = D.ClusterSpec.uniform([D.DeviceSpec(0, 312000.0, 30000.0), D.DeviceSpec(1, 312000.0, 40960.0)],
                                    25000.0, 200000.0)
    ex = RegistryOnlyExecutor(D.PlacementState.sequential(40, 0))
    ctl = ReferenceController(ex, cluster, model, cat, ms=ms)
    dec = ctl.decide(bs=16, kv_tokens=4000.0, mean_prompt_len=128, mean_gen_len=256)
    assert dec.trigger == "scale_down"
    kv_mb = {li: 4000.0 * cat.kv_bytes_per_token_per_layer / 1e6 for li in range(1, 41)}
    ours = apply_reference_ops(ms, D.PlacementState.sequential(40, 0), dec.ops, cat, cluster, kv_mb)
    assert ours == from_ref_placement(dec.placement)
    kinds = {type(p.op).__name__ for p in dec.ops}
    assert kinds & {"MigrateSubModule", "MigrateLayer", "PerformanceReduction"}
