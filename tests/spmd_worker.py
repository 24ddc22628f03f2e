"""Worker for tests/test_spmd_gpu.py: the SPMD runtime (one process per device)
under torchrun, on the config-1 tiny model (confident head).

Devices 0..world-1 belong to ranks 0..world-1 (WORKER_SAME_GPU=1: every rank
on cuda:0, as on the single-GPU test box).  Transport: SPMD_MODE=host (staged
through host memory over gloo) or nccl (NCCL; on one GPU each rank gets its own
NCCL_HOSTID so NCCL treats them as separate hosts).

Scenario (every rank runs it; rank 0 checks against the fp32 oracle):
 1. layers on device 0; ReplicateLayer(2 -> every other device) across processes;
 2. prefill 15 requests + 3 decode steps (layer 2's rows split over the ranks);
 3. the batch shrinks (3 requests finish): split_batch moves sequences between
    ranks, their KV prefixes follow over the transport; 3 decode steps;
 4. ReplicateLayer(4 -> device 1) issued asynchronously, one decode step while
    it is pending, commit, one decode step;
 5. MigrateLayer(3 -> device 1, with_kv): the layer block and its KV move;
 6. EvictReplica(2, device 1): KV rows it held move back to the original;
every step's greedy tokens must equal the oracle's for every live sequence;
the replicated layer-4 block must be byte-identical on both ranks."""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    mode = os.environ.get("SPMD_MODE", "host")
    same_gpu = os.environ.get("WORKER_SAME_GPU", "1") == "1"
    if mode == "nccl" and same_gpu:  # separate "hosts" for NCCL: it refuses two ranks on one GPU otherwise
        os.environ["NCCL_HOSTID"] = f"cocob200-rank{rank}"
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
        os.environ.setdefault("NCCL_IB_DISABLE", "1")
    import torch
    import torch.distributed as dist

    from oracle.cpu_llama import TINY, OracleModel, greedy_generate, init_weights
    from oracle.gen_golden import CONFIG1_SEED, config1_prompts
    from paper_2507_18006_b200 import domain as D
    from paper_2507_18006_b200 import ops as O
    from paper_2507_18006_b200.executor import ExecutorConfig
    from paper_2507_18006_b200.spmd import SpmdExecutor, SpmdRuntime, init_spmd

    ordinal = 0 if same_gpu else rank
    torch.cuda.set_device(ordinal)
    dist.init_process_group("gloo")
    group, transport, rank_of_device = init_spmd(dist, rank, world, ordinal, mode)
    rt = SpmdRuntime(rank_of_device, rank, ordinal, transport)
    w = init_weights(TINY, CONFIG1_SEED, head="permuted_tied")
    cfg = ExecutorConfig(TINY.n_layers, TINY.d_model, TINY.d_ff, TINY.n_heads, vocab=TINY.vocab, max_slots=16,
                         max_ctx=32, max_tokens=256)
    ex = SpmdExecutor(rt, cfg, group, home_device=0)
    ex.load_model(w, device_of_layer=0)
    cat = D.ModuleCatalog.from_model(D.ModelSpec(TINY.n_layers, TINY.d_model, TINY.d_ff, TINY.n_heads))
    cluster = D.ClusterSpec.b200(world)
    for dv in range(1, world):
        ex.apply(O.ReplicateLayer(2, dv), cat, cluster)

    prompts = config1_prompts()
    n_new = 11
    ref, _ = greedy_generate(OracleModel(TINY, w, 32), prompts, n_new) if rank == 0 else (None, None)
    live = list(range(len(prompts)))
    outs = {i: [] for i in live}
    mism = []

    def record(nxt, phase):
        for i, t in zip(live, nxt):
            outs[i].append(int(t))
            if rank == 0 and int(t) != int(ref[i, len(outs[i]) - 1]):
                mism.append((phase, i, len(outs[i]) - 1, int(t), int(ref[i, len(outs[i]) - 1])))

    def decode(phase):
        slots = np.array(live, dtype=np.int32)
        toks = np.array([outs[i][-1] for i in live], dtype=np.int32)
        nxt, _, _ = ex.decode(slots, toks)
        record(nxt, phase)

    nxt, _, _ = ex.prefill(np.array(live, np.int32), np.concatenate(prompts),
                           np.array([len(p) for p in prompts], np.int32))
    record(nxt, "prefill")
    for _ in range(3):
        decode("replicated")
    routing_before = ex.last_routing(2)
    gone = [0, 5, 9]
    ex.release_slots(np.array(gone, np.int32))
    live = [i for i in live if i not in gone]
    for _ in range(3):
        decode("shrunk")
    routing_after = ex.last_routing(2)
    ex.issue(O.ReplicateLayer(4, 1), cat, cluster)
    decode("pending-replicate")
    ex.commit()
    decode("after-replicate")
    ex.apply(O.MigrateLayer(3, 1, with_kv=True), cat, cluster)
    decode("after-migrate")
    ex.apply(O.EvictReplica(2, 1), cat, cluster)
    decode("after-evict")
    blk = ex.read_module(4, rank if rank <= 1 else 0, "decoder_layer") if rank <= 1 else None
    dig = int(hashlib.sha256(blk.tobytes()).hexdigest()[:15], 16) if blk is not None else -1
    digs = group.allgather([dig])[:, 0].tolist()
    mig = ex.op_log[-2]
    res = {"mismatches": mism[:10], "n_mismatch": len(mism), "tokens_checked": sum(len(v) for v in outs.values()),
           "routing_before": routing_before, "routing_after": routing_after,
           "layer4_digests": digs[:2], "placement": [[r.device_id for r in row] for row in ex.placement.replicas],
           "transport_messages": transport.messages, "transport_bytes": transport.bytes,
           "migrate": {"weight_bytes": mig.weight_bytes, "kv_bytes": mig.kv_bytes, "ms": mig.device_ms}}
    allres = [None] * world
    dist.all_gather_object(allres, res)
    if rank == 0:
        print(json.dumps({"world": world, "mode": mode, "ranks": allres}), flush=True)
    ex.close()
    rt.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
