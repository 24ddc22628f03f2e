"""Config 2 open loop: Llama-2-7B shape (random-init bf16 weights) on one B200,
Poisson arrivals at rps 3 / 10 / 30 / 50,
prompt 128, gen 256, continuous batching with batch cap 256 through the
serving engine (reference Engine semantics, sim.py:624-736).  Per-request
latency = completion - arrival (sim.py:663-664), p50 / p99 by np.percentile,
tok/s = generated tokens / wall window.  Each window's arrivals span --window
seconds; the run drains every request.

    python scripts/serving_sweep.py [--rps 3,10,30,50] [--window 8] [--out gpurun_out/serving_sweep.json]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--rps", default="3,10,30,50")
    ap.add_argument("--window", type=float, default=8.0)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--out", default="gpurun_out/serving_sweep.json")
    args = ap.parse_args()
    rt = Runtime([0])
    cfg = ExecutorConfig(**bench.LLAMA2_7B, max_slots=args.batch, max_ctx=128 + 256 + 8,
                         max_tokens=64 * 128)
    ex = Executor(rt, cfg, home_device=0, seed=7)
    ex.init_head_random(std=0.02)
    for li in range(1, cfg.n_layers + 1):
        ex.init_layer_random(li, 0, std=0.02)
    sargs = argparse.Namespace(serve_s=args.window, prompt=128, serve_gen=256, telemetry="")
    rows = []
    for rps in (float(v) for v in args.rps.split(",")):
        s = bench.serving_window(ex, sargs, args.batch, rps)
        rows.append(s)
        print(json.dumps({k: s[k] for k in s if k != "what"}), flush=True)
    ex.close()
    rt.close()
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps({"config": "config 2 open loop: Llama-2-7B shape, bf16, 1 x B200, "
                                                    "prompt 128, gen 256, batch cap %d" % args.batch,
                                          "windows": rows}, indent=1))


if __name__ == "__main__":
    main()
