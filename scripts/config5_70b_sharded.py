"""BASELINE config 5 (single-GPU form): Llama-2-70B shape, layers sharded over
8 logical devices (10 per device, PlacementState.sequential(80, (i-1)//10)),
GQA with 8 KV heads (the real 70B; the reference's MHA accounting is noted).

On one B200 the 8 logical devices share the GPU: activation hops at the 7
device boundaries are D2D copies; on an 8-GPU box they are NVLink P2P copies.
Reports decode tokens/s and the per-layer byte contract.

    python scripts/config5_70b_sharded.py [--batch 16] [--out gpurun_out/config5.json]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2507_18006_b200 import domain as D  # noqa: E402
from paper_2507_18006_b200 import ops as O  # noqa: E402
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--ordinals", default="0,0,0,0,0,0,0,0")
    ap.add_argument("--out", default="gpurun_out/config5.json")
    args = ap.parse_args()
    ordinals = [int(x) for x in args.ordinals.split(",")]
    from _oracle_check import check

    def scenario(ex, cat, cluster, step):  # sharded layers + the controller's projection migration
        if step == 2:
            ex.apply(O.MigrateSubModule(2, D.ModuleKind.FFN_PROJ_GATE, 0), cat, cluster)

    parity = check(dict(d_model=8192, d_ff=28672, n_heads=64, n_kv_heads=8), 2, 8, 32, 5, scenario,
                   device_of_layer=lambda li: li - 1)
    rt = Runtime(ordinals)
    cfg = ExecutorConfig(n_layers=80, d_model=8192, d_ff=28672, n_heads=64, n_kv_heads=8, vocab=32000,
                         max_slots=args.batch, max_ctx=args.prompt + args.steps + 8,
                         max_tokens=args.batch * args.prompt)
    ex = Executor(rt, cfg, home_device=0, seed=5)
    ex.init_head_random(0.01)
    per = 80 // len(ordinals)
    for li in range(1, 81):
        ex.init_layer_random(li, (li - 1) // per, 0.01)
    p = ex.placement
    rng = np.random.default_rng(0)
    slots = np.arange(args.batch, dtype=np.int32)
    nxt, _, prefill_ms = ex.prefill(slots, rng.integers(0, 32000, args.batch * args.prompt).astype(np.int32),
                                    np.full(args.batch, args.prompt, np.int32))
    ms = []
    for _ in range(args.steps):
        nxt, _, m = ex.decode(slots, nxt)
        ms.append(m)
    step = float(np.median(ms[2:]))
    layer_bytes = ex.module_bytes("decoder_layer")
    weight_bytes = 80 * layer_bytes + 2 * 32000 * 8192 * 2
    mha = D.ModuleCatalog.from_model(D.ModelSpec(80, 8192, 28672, 64))
    res = {
        "config": "config 5: Llama-2-70B shape (GQA 8 KV heads), 80 layers sharded 10 per logical device",
        "parity": parity,
        "logical_devices": ordinals, "batch": args.batch, "prompt": args.prompt,
        "original_layers_per_device": {d: len(p.original_layers_on(d)) for d in range(len(ordinals))},
        "decode_ms_per_step": step, "tokens_per_s": args.batch / step * 1e3, "prefill_ms": prefill_ms,
        "layer_bytes_gqa": layer_bytes, "layer_bytes_reference_mha_accounting": round(mha.decoder_layer_mb * 1e6),
        "weight_stream_gbps": weight_bytes / (step * 1e6),
        "note": "one physical B200: the 7 device-boundary hops are D2D copies; NVLink P2P with N GPUs",
    }
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(res, indent=1))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
