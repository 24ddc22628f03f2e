"""OOM detection / crash / requeue and the controller loop in the serving
engine (CPU, registry-level fake executor on a virtual clock).

Mirrors the reference's ``oom_scenario`` (tests/test_sim.py:229-271): two 13B
layers (Table-1 catalog, 605 MB each) on a device of 1214 MB, four requests of
prompt 8 / gen 32 admitted together, one decode step every 201 ms.  The KV of
the resident tokens (0.04096 MB per token over the two layers) crosses the
capacity on the 17th decode commit: 1210 + (32 + 4k) * 0.04096 > 1214 => k = 17.

* without a controller the instance crashes there, every request is requeued
  once, crashes again and fails (4 failed, 0 completed) -- sim.py:670-707;
* with the reference controller (``control.AutoscaleHook`` running the
  unmodified ``controller_step``) the projected OOM triggers a scale-down whose
  KV-cache migration to device 1 is issued while serving and switched at a step
  boundary -- no OOM, all 4 complete;
* a Phase-3 decision's batch cap is applied to the instance at the switch.
"""
from __future__ import annotations

import pytest

from paper_2507_18006_b200 import domain as D
from paper_2507_18006_b200 import ops as O
from paper_2507_18006_b200.control import AutoscaleHook, ReferenceController, load_reference
from paper_2507_18006_b200.serving import InstanceState, ServingEngine
from paper_2507_18006_b200.sim import Request, StepOutcome

ms = load_reference()


class FakeClock:
    def __init__(self):
        self.t = 0.0

    def __call__(self):
        return self.t

    def sleep(self, dt):
        self.t += dt


class RegistryExecutor:
    """The Executor's registry / op / step surface without a device: steps
    advance the virtual clock; issue / commit / abort follow Executor's rules
    (ops.apply chained over the issued ops; the switch at commit)."""

    def __init__(self, clock, placement, step_s=0.201, kv_offload_fraction=0.0):
        self.clock, self.placement, self.step_s = clock, placement, step_s
        self.kv_offload_fraction = kv_offload_fraction
        self.calls, self.released, self.op_log = [], [], []
        self._pending, self._pending_p = [], None

    def step_batch(self, batch, phase):
        self.calls.append((phase, [r.id for r in batch]))
        self.clock.t += self.step_s
        kv = sum(r.prompt_len for r in batch) if phase == "prefill" else len(batch)
        return StepOutcome(self.step_s, kv)

    def release(self, reqs):
        self.released.extend(r.id for r in reqs)

    def issue(self, op, catalog, cluster, cost_model=O.DEFAULT_COST_MODEL, extra_used_mb=None, kv_mb_by_layer=None):
        base = self._pending_p if self._pending else self.placement
        self._pending_p, _ = O.apply(base, op, catalog, cluster, cost_model, extra_used_mb, kv_mb_by_layer)
        self._pending.append(op)
        return len(self._pending)

    def ops_done(self):
        return True

    def commit(self):
        if self._pending:
            self.placement = self._pending_p
            self.op_log.extend(self._pending)
        self._pending, self._pending_p = [], None
        return self.placement

    def abort(self):
        self._pending, self._pending_p = [], None

    def set_kv_offload(self, f):
        self.kv_offload_fraction = f


def _scenario(controller: bool, clock=None):
    clock = clock or FakeClock()
    devices = [D.DeviceSpec(0, 312000.0, 1214.0), D.DeviceSpec(1, 312000.0, 40960.0)]
    cluster = D.ClusterSpec.uniform(devices, 25000.0, 200000.0)
    model = D.ModelSpec(2, 5120, 13824, 40)
    cat = D.ModuleCatalog()  # Table-1 13B catalog (605 MB layers)
    ex = RegistryExecutor(clock, D.PlacementState.sequential(2, 0))
    inst = InstanceState(0, ex, max_batch_size=4)
    eng = ServingEngine([inst], clock=clock, sleep=clock.sleep, cluster=cluster, catalog=cat, oom_restart_s=1.0)
    hook = None
    if controller:
        ctl = ReferenceController(ex, cluster, model, cat, ms=ms,
                                  cfg=ms.autoscaler.ControllerConfig(compute_pressure=1.01))
        hook = AutoscaleHook(ctl, inst, interval_s=1.0, prompt_len=8, gen_len=32)
        eng.on_step = hook
    reqs = [Request(i, 0.0, 8, 32) for i in range(4)]
    return eng, ex, inst, hook, reqs


def test_memory_accounting_follows_the_reference():
    eng, ex, inst, _, _ = _scenario(False)
    assert eng.device_memory_mb(0) == pytest.approx(1210.0)
    inst.resident_tokens = 32 + 4 * 16
    assert eng.device_memory_mb(0) == pytest.approx(1210 + 96 * 0.04096)
    assert eng.device_memory_mb(0) <= 1214.0
    inst.resident_tokens += 4
    assert eng.device_memory_mb(0) > 1214.0


def test_oom_at_the_17th_decode_then_requeued_once_then_failed():
    eng, ex, inst, _, reqs = _scenario(False)
    res = eng.run(reqs)
    first = res.oom_events[0]
    # prefill at t=0 (201 ms) + 17 decode steps of 201 ms: the crossing is at the 17th decode commit
    assert first[1] == 0 and first[0] == pytest.approx(0.201 * 18)
    assert ex.calls[:2] == [("prefill", [0, 1, 2, 3]), ("decode", [0, 1, 2, 3])]
    assert sum(1 for c in ex.calls if c[0] == "decode") == 2 * 17
    assert len(res.oom_events) >= 2
    s = res.summary()
    assert (s["completed"], s["failed"]) == (0, 4)
    assert all(r.failed and r.requeued for r in res.failed)
    # a requeued request kept its queue position (reversed appendleft, sim.py:697-707)
    prefills = [c for c in ex.calls if c[0] == "prefill"]
    assert prefills[1] == ("prefill", [0, 1, 2, 3])
    assert sorted(ex.released) == [0, 0, 1, 1, 2, 2, 3, 3]


@pytest.mark.skipif(ms is None, reason="reference modscale not importable")
def test_controller_prevents_oom_by_kv_migration():
    eng, ex, inst, hook, reqs = _scenario(True)
    res = eng.run(reqs)
    s = res.summary()
    assert (s["oom_events"], s["failed"], s["completed"]) == (0, 0, 4)
    kv_moves = [op for op in ex.op_log if isinstance(op, O.MigrateSubModule) and op.kind is D.ModuleKind.KV_CACHE]
    assert kv_moves, ex.op_log
    assert hook.switches and hook.switches[0][1] == "scale_down"
    assert ex.placement.kv_device(kv_moves[0].layer) == 1


@pytest.mark.skipif(ms is None, reason="reference modscale not importable")
def test_phase3_batch_cap_applied_at_the_switch():
    """A decision carrying a smaller bs (Phase 3, autoscaler.py:568-583) caps
    the instance's admission from the switch on (sim.py:620)."""
    clock = FakeClock()
    eng, ex, inst, hook, _ = _scenario(True, clock)

    class Decision:  # the controller's decision shape (autoscaler.py:598-608)
        trigger = "scale_down"
        ops = ()
        placement = None
        bs = 2
        offload_fraction = 0.5

    ctl = hook.ctl
    tr = ctl.issue(Decision())
    assert tr.bs == 2 and inst.max_batch_size == 4
    hook(eng, 0.0)  # step boundary: ops done -> switch
    assert inst.max_batch_size == 2 and ex.kv_offload_fraction == 0.5 and ctl.pending is None
    reqs = [Request(i, 0.0, 8, 2) for i in range(4)]
    eng.on_step = None
    res = eng.run(reqs)
    assert res.summary()["completed"] == 4
    assert all(len(ids) <= 2 for _, ids in ex.calls)


@pytest.mark.skipif(ms is None, reason="reference modscale not importable")
def test_infeasible_decision_is_aborted_whole():
    """A decision whose k-th op is infeasible leaves the executor untouched."""
    clock = FakeClock()
    eng, ex, inst, hook, _ = _scenario(True, clock)
    before = ex.placement

    class Phased:
        def __init__(self, op):
            self.op = op

    class Decision:
        trigger = "scale_up"
        ops = (Phased(ms.ops.ReplicateLayer(1, 1)), Phased(ms.ops.ReplicateLayer(1, 1)))
        placement = None
        bs = 4
        offload_fraction = 0.0

    with pytest.raises((O.OpError, D.DomainError)):
        hook.ctl.issue(Decision())
    assert ex.placement == before and not ex._pending and hook.ctl.pending is None
