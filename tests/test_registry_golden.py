"""Registry / router / operator parity with the reference (CPU).

Every expected value here was produced by the reference package ``modscale``
itself (oracle/gen_golden.py -> tests/golden/modscale_golden.json), so the
drop-in's routing, batch splits, placement transitions, byte catalog and op
costs are compared bit-exactly (==, no tolerance) against the reference.
The hand values of the reference's own unit tests are repeated explicitly
(tests/test_ops.py:27-46, 209-227 of the reference).
"""
from __future__ import annotations

import json

import numpy as np
import pytest
from hypothesis import given, strategies as st

from conftest import GOLDEN
from paper_2507_18006_b200 import domain as D
from paper_2507_18006_b200 import ops as O
from paper_2507_18006_b200 import sim as S

G = json.loads((GOLDEN / "modscale_golden.json").read_text())


def _placement(spec) -> D.PlacementState:
    home = spec["home"]
    p = D.PlacementState.sequential(spec["n"], (lambda li: home[li - 1]) if isinstance(home, list) else home)
    for li, dev in spec.get("replicas", []):
        p = p.with_replica(li, dev)
    for li, kind, dev in spec.get("overrides", []):
        p = p.with_override(li, D.ModuleKind(kind), dev)
    return p


def _pjson(p: D.PlacementState):
    return {"replicas": [[[r.device_id, bool(r.is_original)] for r in row] for row in p.replicas],
            "overrides": [[li, k.value, dev] for li, k, dev in p.overrides]}


# ------------------------------------------------------------------ split_batch
def test_split_batch_reference_hand_values():
    assert O.split_batch(15, 2) == [7, 8]
    assert O.split_batch(8, 1) == [8]
    assert O.split_batch(10, 4) == [2, 2, 3, 3]
    assert O.split_batch(0, 3) == [0, 0, 0]
    with pytest.raises(O.OpError):
        O.split_batch(-1, 2)
    with pytest.raises(O.OpError):
        O.split_batch(3, 0)


def test_split_batch_golden():
    for bs, p, want in G["split_batch"]:
        assert O.split_batch(bs, p) == want, (bs, p)


def test_native_split_batch_matches_golden():
    """The executor's row router (cb_split_batch in libcocob200) obeys the same rule."""
    from paper_2507_18006_b200 import _lib

    lib = _lib.load()
    for bs, p, want in G["split_batch"]:
        out = np.zeros(p, np.int32)
        assert lib.cb_split_batch(bs, p, _lib.i32(out)) == 0
        assert out.tolist() == want, (bs, p)
    assert lib.cb_split_batch(-1, 2, _lib.i32(np.zeros(2, np.int32))) == _lib.CB_EINVAL


@given(st.integers(0, 500), st.integers(1, 40))
def test_split_batch_properties(bs, p):
    parts = O.split_batch(bs, p)
    assert len(parts) == p and sum(parts) == bs
    assert max(parts) - min(parts) <= 1 and parts == sorted(parts)


# ------------------------------------------------------------------ placements
@pytest.mark.parametrize("case", G["placements"], ids=lambda c: json.dumps(c["spec"])[:40])
def test_placement_golden(case):
    p = _placement(case["spec"])
    assert _pjson(p) == case["placement"]
    assert list(p.p_vector()) == case["p_vector"]
    assert [p.kv_device(li) for li in range(1, p.n_layers + 1)] == case["kv_device"]
    for dev, runs in case["replica_runs"].items():
        assert O.replica_runs(p, int(dev)) == runs
    cluster = D.ClusterSpec.uniform([D.DeviceSpec(i, 312000.0, 40960.0) for i in range(8)], 25000.0, 200000.0)
    arr = S.build_step_arrays(p, cluster)
    assert arr.layer_ptr.tolist() == case["layer_ptr"]
    assert arr.caps.tolist() == case["caps"]
    assert arr.run_min_p.tolist() == case["run_min_p"]
    assert arr.run_bw.tolist() == case["run_bw"]
    assert list(arr.busy_devices) == case["busy_devices"]
    assert {str(k): v for k, v in arr.kv_layer_count.items()} == case["kv_layer_count"]
    usage = D.device_usage(p, D.ModuleCatalog(), kv_tokens={0: 1234.0, 1: 77.0})
    assert {str(k): [u.memory_mb, u.compute_gflops] for k, u in usage.items()} == case["device_usage"]


def test_replica_runs_reference_hand_values():
    p = D.PlacementState.sequential(8, 0)
    for li in (3, 4, 7):
        p = p.with_replica(li, 1)
    assert O.replica_runs(p, 1) == [[3, 4], [7]]
    assert O.replica_runs(p, 0) == []


def test_placement_edit_errors():
    p = D.PlacementState.sequential(3, 0).with_replica(1, 1)
    with pytest.raises(D.DomainError):
        p.with_replica(1, 1)
    with pytest.raises(D.DomainError):
        p.without_replica(1, 0)
    with pytest.raises(D.DomainError):
        p.with_override(1, D.ModuleKind.KV_CACHE, 2)  # replicated layers carry no overrides
    with pytest.raises(D.DomainError):
        p.with_original_device(1, 2, keep_kv_on_source=True)
    q = D.PlacementState.sequential(2, 0).with_original_device(2, 1, keep_kv_on_source=True)
    assert q.kv_device(2) == 0 and q.original_device(2) == 1


# ------------------------------------------------------------------ router
@pytest.mark.parametrize("case", G["schedule"], ids=lambda c: f"seed{c['seed']}")
def test_schedule_golden(case):
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(case["seed"])))
    views = [tuple(v) for v in case["views"]]
    assert [S.schedule(views, rng) for _ in range(len(case["picks"]))] == case["picks"]


def test_schedule_errors():
    with pytest.raises(S.SimError):
        S.schedule([], np.random.default_rng(0))


# ------------------------------------------------------------------ catalog
@pytest.mark.parametrize("name,geom", [("tiny", (4, 256, 768, 4)), ("7b", (32, 4096, 11008, 32)),
                                       ("13b", (40, 5120, 13824, 40)), ("70b", (80, 8192, 28672, 64))])
def test_catalog_from_model_golden(name, geom):
    c = D.ModuleCatalog.from_model(D.ModelSpec(*geom))
    assert {k: getattr(c, k) for k in c.__dataclass_fields__} == G["catalogs"][name]


def test_catalog_layer_bytes_match_survey():
    # layer bytes per config
    for geom, want in [((4, 256, 768, 4), 1704960), ((32, 4096, 11008, 32), 404766720),
                       ((40, 5120, 13824, 40), 634408960), ((80, 8192, 28672, 64), 1946189824)]:
        assert round(D.ModuleCatalog.from_model(D.ModelSpec(*geom)).decoder_layer_mb * 1e6) == want


# ------------------------------------------------------------------ operator
def _op(d):
    d = dict(d)
    t = d.pop("type")
    if "kind" in d:
        d["kind"] = D.ModuleKind(d["kind"])
    return getattr(O, t)(**d)


@pytest.mark.parametrize("scen", G["apply"], ids=lambda s: s["name"])
def test_apply_golden(scen):
    cat = D.ModuleCatalog(**scen["catalog"])
    cl = scen["cluster"]
    cluster = D.ClusterSpec(tuple(D.DeviceSpec(*d) for d in cl["devices"]), tuple(tuple(r) for r in cl["bandwidth"]))
    kv = {int(k): v for k, v in scen["kv_mb"].items()}
    p = _placement(scen["base"])
    for opd, res in zip(scen["ops"], scen["results"]):
        op = _op(opd)
        if res["ok"]:
            p2, cost = O.apply(p, op, cat, cluster, kv_mb_by_layer=kv)
            assert _pjson(p2) == res["placement"], opd
            assert cost.time_s == res["time_s"] and cost.transient_memory_mb == res["mem_mb"], opd
            p = p2
        else:
            with pytest.raises(getattr(O, res["error"])) as exc:
                O.apply(p, op, cat, cluster, kv_mb_by_layer=kv)
            if res["shortfall_mb"] is not None:
                assert exc.value.shortfall_mb == res["shortfall_mb"]


@pytest.mark.parametrize("case", G["batch_apply"], ids=lambda c: c["mode"])
def test_batch_apply_golden(case):
    big = D.ClusterSpec.uniform([D.DeviceSpec(0, 1.0, 50000.0), D.DeviceSpec(1, 1.0, 50000.0)], 1.0, 10.0)
    ops = [_op(o) for o in case["ops"]]
    p2, total, per = O.batch_apply(D.PlacementState.sequential(12, 0), ops, D.ModuleCatalog(), big,
                                   kv_mb_by_layer={i: 10.0 * i for i in range(1, 13)}, cost_mode=case["mode"])
    assert _pjson(p2) == case["placement"]
    assert [total.time_s, total.transient_memory_mb] == case["total"]
    assert [[c.time_s, c.transient_memory_mb] for c in per] == case["per_op"]


def test_batch_apply_transactional():
    clus = D.ClusterSpec.uniform([D.DeviceSpec(0, 1.0, 10000.0), D.DeviceSpec(1, 1.0, 700.0)], 1.0, 10.0)
    p = D.PlacementState.sequential(3, 0)
    with pytest.raises(O.BatchApplyError) as exc:
        O.batch_apply(p, [O.ReplicateLayer(1, 1), O.ReplicateLayer(2, 1)], D.ModuleCatalog(), clus)
    assert exc.value.index == G["batch_apply_failure_index"]


def test_cost_model_anchors_exact():
    m = O.OpCostModel()
    for layers, repl, migr, mem in O.DEFAULT_ANCHORS:
        assert m.replication_time_s(layers) == repl
        assert m.migration_time_s(layers) == migr
        assert m.transient_memory_mb(layers) == mem
    assert m.replication_time_s(50) == pytest.approx(0.8938 + 10 * (0.8938 - 0.4947) / 10)
