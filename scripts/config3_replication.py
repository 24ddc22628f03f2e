"""BASELINE config 3 (single-GPU form): Llama-2-7B shape with hot decoder layers
replicated across logical devices, under a bursty synthetic arrival trace.

The reference auto-scaler (unmodified ``controller_step``, via control.py) is
consulted every ``--eval-s`` seconds of the serving run and its scale-up /
scale-down ops are committed physically between steps.  On one B200 all
logical devices share the GPU, so replication adds no compute: this run
measures that the replicated data path (row split per layer, scatter/gather
at run boundaries, per-replica KV that follows its rows) serves correctly
under load and what it costs.  On an 8-GPU box the replicas are separate
GPUs and the same run scales.

    python scripts/config3_replication.py [--devices 2] [--hot 16] [--out gpurun_out/config3.json]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2507_18006_b200 import domain as D  # noqa: E402
from paper_2507_18006_b200 import ops as O  # noqa: E402
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime  # noqa: E402
from paper_2507_18006_b200.serving import InstanceState, ServingEngine, bursty_trace  # noqa: E402


def run(n_dev: int, hot: int, duration: float, batch: int, seed: int = 7) -> dict:
    rt = Runtime([0] * n_dev)
    ex = Executor(rt, ExecutorConfig(32, 4096, 11008, 32, vocab=32000, max_slots=batch, max_ctx=128 + 64 + 8,
                                     max_tokens=batch * 128), seed=1)
    ex.init_head_random(0.02)
    for li in range(1, 33):
        ex.init_layer_random(li, 0, 0.02)
    cat = D.ModuleCatalog.from_model(D.ModelSpec(32, 4096, 11008, 32))
    cluster = D.ClusterSpec.b200(n_dev)
    op_ms = []
    for li in range(1, hot + 1):  # hot layers replicated on every other logical device
        for dv in range(1, n_dev):
            ex.apply(O.ReplicateLayer(li, dv), cat, cluster)
            op_ms.append(ex.op_log[-1].device_ms)
    reqs = bursty_trace(5.0, 50.0, 4.0, 2.0, duration, 128, 64, seed)
    eng = ServingEngine([InstanceState(0, ex, batch)], seed=seed)
    res = eng.run(reqs)
    s = res.summary()
    s.update({"devices": n_dev, "hot_layers_replicated": hot, "p_vector": list(ex.placement.p_vector()),
              "replicate_op_ms_mean": sum(op_ms) / len(op_ms) if op_ms else 0.0,
              "routing_layer1": ex.last_routing(1) if hot else None})
    ex.close()
    rt.close()
    return s


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--devices", type=int, default=2)
    ap.add_argument("--hot", type=int, default=16)
    ap.add_argument("--duration", type=float, default=12.0)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--out", default="gpurun_out/config3.json")
    args = ap.parse_args()
    from _oracle_check import check

    def scenario(ex, cat, cluster, step):  # the hot layer replicated on every other device before serving
        if step == 0:
            for dv in range(1, args.devices):
                ex.apply(O.ReplicateLayer(1, dv), cat, cluster)

    parity = check(dict(d_model=4096, d_ff=11008, n_heads=32), args.devices, 48, 64, 6, scenario,
                   release={2: [0, 7, 30], 4: [11, 12, 13, 47]})
    base = run(1, 0, args.duration, args.batch)
    repl = run(args.devices, args.hot, args.duration, args.batch)
    res = {"config": "config 3: Llama-2-7B, hot layers replicated, bursty trace (5 rps 4 s / 50 rps 2 s)",
           "note": "logical devices share one B200: replication adds no compute here; shows correctness + overhead",
           "parity": parity, "baseline_no_replication": base, "replicated": repl}
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(res, indent=1))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
