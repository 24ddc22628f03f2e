"""Run artefacts of a B200 serving run in the reference's schema.

The reference writes ``trace`` / ``ops`` / ``decisions`` logs (CSV with a
``# schema_version=`` line, or JSON ``{"schema_version", "rows"}``) plus
``summary.json`` (outputs.py:20-104, trace rows sim.py:885-923, summary
sim.py:974-1017, schema "1.0").  ``write_run`` emits the same files from a real
run -- measured latencies, tokens, device busy time and the copy engine's
measured op times -- so the reference's own readers (``outputs.read_rows`` /
``read_summary``) and tooling consume B200 runs unchanged.

Extensions stay inside the schema: the op log's ``detail`` column carries the
measured bytes and GB/s as ``key=value`` pairs after the reference's own detail
text, and trace rows may carry extra columns (the reference writer takes the
trace field list from the rows themselves).
"""
from __future__ import annotations

import csv
import io
import json
from pathlib import Path
from typing import Sequence

import numpy as np

from . import ops as O

SCHEMA_VERSION = "1.0"  # reference sim.py:1020
OP_FIELDS = ["tick_ms", "kind", "layer", "src_device", "dst_device", "time_s", "transient_mb", "phase", "detail"]
DECISION_FIELDS = ["tick_ms", "trigger", "instance", "n_ops", "sp_before", "sp_after", "bs_before", "bs_after",
                   "resolved", "cost_s"]


def op_rows(op_log: Sequence, ticks_ms: Sequence[int] | None = None, src_devices: Sequence | None = None) -> list:
    """Executor op measurements (``Executor.op_log``) as reference op-log rows.

    time_s = measured device copy time; transient_mb = bytes moved / 1e6 (the
    destination holds the new copy while the source still serves)."""
    rows = []
    for i, m in enumerate(op_log):
        tick = int(ticks_ms[i]) if ticks_ms is not None else 0
        src = src_devices[i] if src_devices is not None else None
        moved = m.weight_bytes + m.kv_bytes
        extra = f"weight_bytes={m.weight_bytes};kv_bytes={m.kv_bytes};gbps={m.gbps:.1f}"
        if isinstance(m.op, (O.ReplicateLayer, O.MigrateLayer, O.MigrateSubModule, O.EvictReplica)):
            rec = O.OpRecord.from_op(tick, m.op, O.TransitionCost(m.device_ms / 1e3, moved / 1e6), src_device=src)
            row = {k: getattr(rec, k) for k in OP_FIELDS}
        else:  # Phase-3 KV offload / reload: (name, layer)
            name, layer = m.op
            row = {"tick_ms": tick, "kind": name, "layer": layer, "src_device": src, "dst_device": None,
                   "time_s": m.device_ms / 1e3, "transient_mb": moved / 1e6, "phase": 3, "detail": ""}
        row["detail"] = ";".join(x for x in (row["detail"], extra) if x)
        rows.append(row)
    return rows


def trace_rows(completed: Sequence, step_log: Sequence, window_s: float, devices: Sequence[int] = (0,),
               slo_latency_s: float = 10.0, n_arrived_by_window: dict | None = None) -> list:
    """Windowed metrics rows (reference sim.py:885-923) from a serving run.

    ``completed``: requests with arrival_s / completion_s / generated; ``step_log``:
    ServingEngine rows (t_s, kind, instance, bs, device_s, wall_s)."""
    if not completed and not step_log:
        return []
    end = max([r.completion_s for r in completed] + [s[0] + s[5] for s in step_log])
    n_win = int(np.floor(end / window_s)) + 1
    rows = []
    for k in range(n_win):
        lo, hi = k * window_s, (k + 1) * window_s
        done = [r for r in completed if lo <= r.completion_s < hi]
        lat = [r.completion_s - r.arrival_s for r in done]
        arr = np.asarray(lat, dtype=np.float64)
        p50, p95, p99 = (np.percentile(arr, [50.0, 95.0, 99.0]) if arr.size else (0.0, 0.0, 0.0))
        steps = [s for s in step_log if lo <= s[0] < hi]
        toks = sum(s[3] for s in steps if s[1] == "decode")
        viol = sum(1 for x in lat if x > slo_latency_s)
        arrived = sum(1 for r in completed if lo <= r.arrival_s < hi)
        row = {
            "tick_ms": int(round(lo * 1000)),
            "rps_in": (n_arrived_by_window or {}).get(k, arrived) / window_s,
            "throughput_rps": len(done) / window_s,
            "throughput_tok_s": toks / window_s,
            "completions": len(done),
            "failures": 0,
            "violations": viol,
            "violation_rate": viol / len(done) if done else 0.0,
            "mean_latency_s": float(arr.mean()) if arr.size else 0.0,
            "p50_latency_s": float(p50), "p95_latency_s": float(p95), "p99_latency_s": float(p99),
            "oom_events": 0,
        }
        for d in devices:
            busy = sum(s[4] for s in steps if s[2] == d)
            row[f"busy_{d}"] = min(1.0, busy / window_s)
        rows.append(row)
    return rows


def summary(trace: Sequence[dict], op_rows_: Sequence[dict], completed: Sequence, seed: int, duration_s: float,
            final_placements: dict) -> dict:
    """Reference summary keys (sim.py:987-1016), recomputable from the trace rows."""
    tot = sum(r["completions"] + r["failures"] for r in trace)

    def weighted(f):
        return sum(r[f] * (r["completions"] + r["failures"]) for r in trace) / tot if tot else 0.0

    return {
        "schema_version": SCHEMA_VERSION,
        "seed": seed,
        "duration_s": duration_s,
        "final_t_s": (trace[-1]["tick_ms"] / 1000.0 if trace else 0.0),
        "arrived": len(completed),
        "completed": len(completed),
        "failed": 0,
        "in_flight_end": 0,
        "mean_throughput_rps": sum(r["throughput_rps"] for r in trace) / len(trace) if trace else 0.0,
        "mean_throughput_tok_s": sum(r["throughput_tok_s"] for r in trace) / len(trace) if trace else 0.0,
        "mean_latency_s": weighted("mean_latency_s"),
        "p95_latency_s": weighted("p95_latency_s"),
        "violation_rate": (sum(r["violations"] for r in trace) / tot) if tot else 0.0,
        "oom_events": 0,
        "total_scaling_cost_s": float(sum(r["time_s"] for r in op_rows_)),
        "n_scaling_ops": len(op_rows_),
        "final_placements": final_placements,
    }


def _fmt(v):
    if isinstance(v, float):
        return repr(v)
    return "" if v is None else v


def _write(path: Path, rows: Sequence[dict], fields: Sequence[str], fmt: str) -> None:
    if fmt == "json":
        path.write_text(json.dumps({"schema_version": SCHEMA_VERSION, "rows": list(rows)}, indent=1))
        return
    buf = io.StringIO()
    buf.write(f"# schema_version={SCHEMA_VERSION}\n")
    w = csv.DictWriter(buf, fieldnames=list(fields), lineterminator="\n")
    w.writeheader()
    for r in rows:
        w.writerow({k: _fmt(r.get(k)) for k in fields})
    path.write_text(buf.getvalue())


def write_run(out_dir, trace: Sequence[dict], ops_: Sequence[dict], decisions: Sequence[dict], summary_: dict,
              fmt: str = "csv") -> list[Path]:
    """trace / ops / decisions in ``fmt`` + summary.json (outputs.py:78-104 layout)."""
    if fmt not in ("csv", "json"):
        raise ValueError(f"unknown output format {fmt!r}")
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    paths = []
    for name, rows, fields in (("trace", trace, list(trace[0].keys()) if trace else ["tick_ms"]),
                               ("ops", ops_, OP_FIELDS), ("decisions", decisions, DECISION_FIELDS)):
        p = out / f"{name}.{fmt}"
        _write(p, rows, fields, fmt)
        paths.append(p)
    sp = out / "summary.json"
    sp.write_text(json.dumps(summary_, indent=1, sort_keys=True))
    paths.append(sp)
    return paths
