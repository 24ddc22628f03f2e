"""Run artefacts in the reference schema (outputs.py:20-104): written by
telemetry.write_run, read back by the REFERENCE's own readers."""
from __future__ import annotations

import pytest

from paper_2507_18006_b200 import domain as D
from paper_2507_18006_b200 import ops as O
from paper_2507_18006_b200 import telemetry as T
from paper_2507_18006_b200.control import load_reference
from paper_2507_18006_b200.executor import OpMeasurement
from paper_2507_18006_b200.sim import Request

ms = load_reference()


def _run():
    reqs = []
    for i in range(6):
        r = Request(i, 0.2 * i, 16, 4)
        r.completion_s = 0.2 * i + 0.5 + 0.01 * i
        r.generated = 4
        reqs.append(r)
    steps = [(0.0, "prefill", 0, 3, 0.004, 0.005), (0.01, "decode", 0, 3, 0.002, 0.003),
             (1.1, "decode", 0, 2, 0.002, 0.003)]
    log = [OpMeasurement(O.ReplicateLayer(2, 1), 404766720, 0, 0.45),
           OpMeasurement(O.MigrateSubModule(3, D.ModuleKind.FFN_PROJ_GATE, 1), 90177536, 0, 0.12),
           OpMeasurement(O.MigrateLayer(4, 1, True), 404766720, 1638400, 0.5),
           OpMeasurement(("kv_offload", 1), 0, 1638400, 0.3)]
    trace = T.trace_rows(reqs, steps, window_s=1.0, devices=(0, 1))
    ops = T.op_rows(log, ticks_ms=[100, 200, 300, 400], src_devices=[0, 0, 0, 0])
    summ = T.summary(trace, ops, reqs, seed=7, duration_s=2.0, final_placements={"0": [1, 2, 1, 1]})
    return trace, ops, summ


def test_rows_follow_reference_fields():
    trace, ops, summ = _run()
    assert [r["kind"] for r in ops] == ["replicate_layer", "migrate_submodule", "migrate_layer", "kv_offload"]
    assert ops[1]["detail"].startswith("ffn_proj_gate;weight_bytes=90177536")
    assert ops[2]["detail"].startswith("with_kv;")
    assert abs(ops[0]["time_s"] - 0.45e-3) < 1e-12 and ops[0]["transient_mb"] == 404.76672
    assert sum(r["completions"] for r in trace) == 6 and summ["n_scaling_ops"] == 4
    assert summ["completed"] == 6 and summ["schema_version"] == "1.0"


@pytest.mark.skipif(ms is None, reason="reference modscale not importable")
@pytest.mark.parametrize("fmt", ["csv", "json"])
def test_reference_readers_accept_b200_run(tmp_path, fmt):
    from modscale import outputs as RO

    trace, ops, summ = _run()
    T.write_run(tmp_path, trace, ops, [], summ, fmt=fmt)
    back = RO.read_rows(tmp_path / f"ops.{fmt}")
    assert [r["kind"] for r in back] == [r["kind"] for r in ops]
    assert [str(r["layer"]) for r in back] == [str(r["layer"]) for r in ops]
    tr = RO.read_rows(tmp_path / f"trace.{fmt}")
    assert len(tr) == len(trace)
    s = RO.read_summary(tmp_path / "summary.json")
    assert s["n_scaling_ops"] == 4 and s["final_placements"] == {"0": [1, 2, 1, 1]}
    assert RO.OP_FIELDS == T.OP_FIELDS and RO.DECISION_FIELDS == T.DECISION_FIELDS
