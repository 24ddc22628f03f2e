"""Worker for tests/test_dist_cpu.py::test_replica_group_*: one process per
(simulated) GPU, gloo backend.  Each rank serves its split_batch share of the
config-1 requests with a CPU stand-in executor (the fp32 oracle -- test
infrastructure, standing in for the per-GPU Executor); rank 0 checks that the
gathered greedy tokens equal one unreplicated oracle run over the whole batch."""
import json
import os
import sys

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.cpu_llama import TINY, OracleModel, greedy_generate, init_weights  # noqa: E402
from oracle.gen_golden import CONFIG1_SEED, config1_prompts  # noqa: E402
from paper_2507_18006_b200.dist import PHASE_DECODE, PHASE_PREFILL, ReplicaGroup  # noqa: E402


class OracleExecutor:
    """Executor-shaped CPU stand-in: prefill/decode(slots, tokens[, lens]) -> (next, logits, ms)."""

    class cfg:  # noqa: N801
        max_slots = 16

    def __init__(self, w):
        self.m = OracleModel(TINY, w, 64)

    def prefill(self, slots, tokens, lens):
        lg = self.m.forward(list(slots), tokens, list(lens))
        return lg.argmax(-1).astype(np.int32), lg, 0.0

    def decode(self, slots, tokens):
        lg = self.m.forward(list(slots), tokens, None)
        return lg.argmax(-1).astype(np.int32), lg, 0.0

    def release_slots(self, slots):
        self.m.release(list(slots))


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    w = init_weights(TINY, CONFIG1_SEED, head="permuted_tied")
    prompts = config1_prompts()[:int(os.environ.get("N_REQ", "15"))]
    n_new = 4
    if os.environ.get("WORKER_GPU") == "1":  # the real per-GPU executor (both ranks share cuda:0 in tests)
        from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime

        rt = Runtime([0])
        ex = Executor(rt, ExecutorConfig(TINY.n_layers, TINY.d_model, TINY.d_ff, TINY.n_heads, vocab=TINY.vocab,
                                         max_slots=16, max_ctx=32, max_tokens=256))
        ex.load_model(w, device_of_layer=0)
    else:
        ex = OracleExecutor(w)
    g = ReplicaGroup(dist, ex)
    slots = np.arange(len(prompts))
    out = []
    nxt, _ = g.step(PHASE_PREFILL, slots, np.concatenate(prompts) if rank == 0 else None,
                    [len(p) for p in prompts] if rank == 0 else None)
    out.append(nxt)
    for _ in range(n_new - 1):
        nxt, _ = g.step(PHASE_DECODE, slots, out[-1] if rank == 0 else None)
        out.append(nxt)
    shares = g.last_shares
    g.release(slots)
    if rank == 0:
        ref, _ = greedy_generate(OracleModel(TINY, w, 64), prompts, n_new)
        got = np.stack(out, 1)
        print(json.dumps({"equal": bool(np.array_equal(got, ref)), "shares": shares, "world": world,
                          "tokens": got.tolist()}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
