"""BASELINE config 4: Llama-2-13B shape, decoder-layer migration mid-serving.

Weights + KV move between logical devices while a decode batch is in flight
(MigrateLayer with_kv=True, ops.py:213-228), single ops and a batched 10-layer
transfer (Table 2's k-layer rows).  On one B200 the two
logical devices share the GPU, so the copy runs D2D over HBM; with N GPUs the
same call moves the bytes over NVLink.  Decode keeps running between the ops
and its step time is reported before / during / after.

    python scripts/config4_migration.py [--batch 32] [--layers 10] [--out gpurun_out/config4.json]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2507_18006_b200 import domain as D  # noqa: E402
from paper_2507_18006_b200 import ops as O  # noqa: E402
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--layers", type=int, default=10)
    ap.add_argument("--ordinals", default="0,0")
    ap.add_argument("--out", default="gpurun_out/config4.json")
    args = ap.parse_args()
    ordinals = [int(x) for x in args.ordinals.split(",")]
    from _oracle_check import check

    def scenario(ex, cat, cluster, step):  # migrations with KV mid-decode: one synchronous, one asynchronous
        if step == 2:
            ex.apply(O.MigrateLayer(1, 1, with_kv=True), cat, cluster)
        if step == 3:
            ex.issue(O.MigrateLayer(2, 1, with_kv=True), cat, cluster)  # copies run while step 3 decodes
        if step == 4:
            ex.commit(wait=True)

    parity = check(dict(d_model=5120, d_ff=13824, n_heads=40), 2, 24, 48, 6, scenario, release={3: [5, 6]})
    rt = Runtime(ordinals)
    geom = dict(n_layers=40, d_model=5120, d_ff=13824, n_heads=40)
    ex = Executor(rt, ExecutorConfig(**geom, vocab=32000, max_slots=args.batch, max_ctx=args.prompt + 96,
                                     max_tokens=args.batch * args.prompt), seed=3)
    ex.init_head_random(0.02)
    for li in range(1, 41):
        ex.init_layer_random(li, 0, 0.02)
    model = D.ModelSpec(**geom)
    cat = D.ModuleCatalog.from_model(model)
    cluster = D.ClusterSpec.b200(len(ordinals))
    rng = np.random.default_rng(0)
    slots = np.arange(args.batch, dtype=np.int32)
    nxt, _, prefill_ms = ex.prefill(slots, rng.integers(0, 32000, args.batch * args.prompt).astype(np.int32),
                                    np.full(args.batch, args.prompt, np.int32))

    def decode(n):
        nonlocal nxt
        ms = []
        for _ in range(n):
            nxt, _, m = ex.decode(slots, nxt)
            ms.append(m)
        return float(np.median(ms))

    step_before = decode(8)
    singles = []
    for li in (1, 2):  # single-layer migrations with KV, decode in between
        ex.apply(O.MigrateLayer(li, 1, with_kv=True), cat, cluster)
        m = ex.op_log[-1]
        singles.append({"layer": li, "weight_bytes": m.weight_bytes, "kv_bytes": m.kv_bytes, "ms": m.device_ms,
                        "gbps": m.gbps})
        decode(2)
    # batched k-layer transfer (Table 2 rows), decode continues afterwards
    t0 = time.perf_counter()
    batch_ops = [O.MigrateLayer(li, 1, with_kv=True) for li in range(3, 3 + args.layers)]
    wb = kb = 0
    dev_ms = 0.0
    for op in batch_ops:
        ex.apply(op, cat, cluster)
        m = ex.op_log[-1]
        wb += m.weight_bytes
        kb += m.kv_bytes
        dev_ms += m.device_ms
    wall_ms = (time.perf_counter() - t0) * 1e3
    step_after = decode(8)
    analytic = O.batch_apply(D.PlacementState.sequential(40, 0), batch_ops, cat, D.ClusterSpec.b200(2))[1]
    res = {
        "config": "config 4: Llama-2-13B shape, migration mid-serving (weights + KV)",
        "parity": parity,
        "logical_devices": ordinals,
        "path": "same-GPU D2D (HBM)" if len(set(ordinals)) == 1 else "NVLink P2P",
        "batch": args.batch, "ctx_at_migration": args.prompt + 10,
        "layer_bytes": ex.module_bytes("decoder_layer"),
        "catalog_layer_bytes": round(cat.decoder_layer_mb * 1e6),
        "single_layer_migrations": singles,
        f"batched_{args.layers}_layers": {"weight_bytes": wb, "kv_bytes": kb, "device_ms": dev_ms, "wall_ms": wall_ms,
                                          "gbps": (wb + kb) / (dev_ms * 1e6)},
        "paper_table2_a100_s": {"migrate_1_layer": 0.2492, "migrate_10_layers": 0.3181},
        "reference_analytic_cost_s": analytic.time_s,
        "decode_step_ms": {"before": step_before, "after": step_after},
        "prefill_ms": prefill_ms,
        "placement_after": list(ex.placement.p_vector())[:12],
        "kv_device_after": [ex.placement.kv_device(li) for li in range(1, 13)],
    }
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(res, indent=1))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
