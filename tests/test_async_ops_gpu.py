"""Asynchronous, serving-concurrent scaling ops (A17) on the GPU.

The reference keeps an instance serving on its pre-op placement while a
transition's bytes move and switches atomically at the commit (sim.py:396-403,
614-622, 812-841).  Here ``Executor.issue`` reserves the
destination memory and starts the copy, decode steps keep running on the old
placement (asserted through the device plan and the routing), and
``Executor.commit`` switches at a step boundary after copying the KV appended
since the issue.  Bars: tokens equal the fp32 oracle throughout, moved bytes
identical, reservations released by ``abort``.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle.cpu_llama import TINY, OracleModel, init_weights
from oracle.gen_golden import CONFIG1_SEED, config1_prompts
from paper_2507_18006_b200 import domain as D
from paper_2507_18006_b200 import ops as O
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime
from paper_2507_18006_b200.sim import Request

pytestmark = pytest.mark.gpu

LOGIT_TOL = 2e-2
N_REQ, PROMPT = 15, 16


@pytest.fixture(scope="module")
def confident():
    return init_weights(TINY, CONFIG1_SEED, head="permuted_tied")


@pytest.fixture(scope="module")
def runtime(cuda):
    rt = Runtime([0, 0, 0])
    yield rt
    rt.close()


def _cat_cl(n=3):
    return D.ModuleCatalog.from_model(D.ModelSpec(TINY.n_layers, TINY.d_model, TINY.d_ff, TINY.n_heads)), \
        D.ClusterSpec.b200(n)


def _setup(runtime, w):
    ex = Executor(runtime, ExecutorConfig(TINY.n_layers, TINY.d_model, TINY.d_ff, TINY.n_heads, vocab=TINY.vocab,
                                          max_slots=32, max_ctx=64, max_tokens=512))
    ex.load_model(w, device_of_layer=0)
    oracle = OracleModel(TINY, w, 64)
    prompts = config1_prompts()
    live = list(range(N_REQ))
    nxt, _, _ = ex.prefill(np.array(live, np.int32), np.concatenate(prompts), np.full(N_REQ, PROMPT, np.int32))
    oracle.forward(live, np.concatenate(prompts), [PROMPT] * N_REQ)
    return ex, oracle, live, dict(zip(live, nxt))


def _decode(ex, oracle, live, last):
    inp = np.array([last[s] for s in live], np.int32)
    nxt, lg, _ = ex.decode(np.array(live, np.int32), inp, want_logits=True)
    ref = oracle.forward(live, inp, None)
    assert np.array_equal(nxt, ref.argmax(-1))
    assert np.abs(lg - ref).max() <= LOGIT_TOL
    last.update(zip(live, nxt))


def test_migrate_with_kv_while_serving(runtime, confident):
    """MigrateLayer(3 -> dev 1, with KV) issued, 4 decode steps on the old
    placement (one request finishes and its slot is refilled by a new prompt,
    so its pre-copied KV is stale), commit, 4 more steps: tokens equal the
    oracle at every step; the migrated block and every slot's KV equal the
    source; the catch-up copied only the tokens appended since the issue
    (plus the refilled slot whole)."""
    ex, oracle, live, last = _setup(runtime, confident)
    cat, cl = _cat_cl()
    block = ex.read_module(3, 0, "decoder_layer")
    oid = ex.issue(O.MigrateLayer(3, 1, with_kv=True), cat, cl)
    assert ex.pending_ops and ex.placement.original_device(3) == 0
    for step in range(4):
        _decode(ex, oracle, live, last)
        ex.check_plan()
        assert ex.device_plan()[2][2] == 0  # layer 3's KV still served from device 0
        if step == 1:  # request 4 finishes; a fresh prompt takes its slot
            live.remove(4)
            ex.release([Request(4, 0.0, PROMPT, 1, slot=4)])
            oracle.release([4])
            p = np.arange(PROMPT, dtype=np.int32) * 7 % TINY.vocab
            nx, _, _ = ex.prefill(np.array([4], np.int32), p, np.array([PROMPT], np.int32))
            ref = oracle.forward([4], p, [PROMPT])
            assert nx[0] == ref.argmax(-1)[0]
            live.append(4)
            last[4] = nx[0]
    assert ex.ops_done()
    kv_src = {s: ex.read_kv(3, s) for s in live}
    assert all(dev == 0 for _, dev in kv_src.values())
    ex.commit()
    assert ex.placement.original_device(3) == 1 and ex.placement.kv_device(3) == 1
    for s in live:  # pre-copy + catch-up == the source's KV, byte for byte
        kv, dev = ex.read_kv(3, s)
        assert dev == 1 and np.array_equal(kv, kv_src[s][0]), s
    for _ in range(4):
        _decode(ex, oracle, live, last)
    m = ex.op_log[-1]
    assert m.weight_bytes == 1704960
    kvb = 2 * TINY.d_model * 2
    # pre-copy: 15 slots x 16 prompt tokens; catch-up: 14 slots x 4 new tokens + slot 4 whole (16 + 2)
    assert m.catchup_bytes == (14 * 4 + (PROMPT + 2)) * kvb, m.catchup_bytes
    assert m.kv_bytes == N_REQ * PROMPT * kvb + m.catchup_bytes
    assert np.array_equal(ex.read_module(3, 1, "decoder_layer"), block)
    ex.close()


def test_decision_of_mixed_ops_commits_atomically(runtime, confident):
    """Several ops issued back to back (replicate, KV sub-module migration,
    projection migration), serving in between, one commit: the registry
    switches only at the commit, each op's placement equals ops.apply chained,
    and tokens equal the oracle before and after."""
    ex, oracle, live, last = _setup(runtime, confident)
    cat, cl = _cat_cl()
    before = ex.placement
    ops = [O.ReplicateLayer(2, 1), O.ReplicateLayer(2, 2), O.MigrateSubModule(4, D.ModuleKind.KV_CACHE, 1),
           O.MigrateSubModule(1, D.ModuleKind.FFN_PROJ_DOWN, 2)]
    want = before
    for op in ops:
        ex.issue(op, cat, cl, kv_mb_by_layer={4: 0.5})
        want, _ = O.apply(want, op, cat, cl, kv_mb_by_layer={4: 0.5})
    with pytest.raises(O.OpError):  # one uncommitted op per layer; sync apply refused while ops are pending
        ex.apply(O.EvictReplica(2, 1), cat, cl)
    for _ in range(3):
        _decode(ex, oracle, live, last)
        assert ex.placement == before
        assert ex.last_routing(2) == [(0, 0, len(live))]
    ex.commit()
    assert ex.placement == want
    for _ in range(3):
        _decode(ex, oracle, live, last)
    assert [c for _, _, c in ex.last_routing(2)] == O.split_batch(len(live), 3)
    assert ex.read_kv(4, 0)[1] == 1
    # scale back down asynchronously: evict both replicas (their KV returns to the original at the commit)
    ex.issue(O.EvictReplica(2, 2), cat, cl)
    _decode(ex, oracle, live, last)
    ex.commit()
    ex.issue(O.EvictReplica(2, 1), cat, cl)
    _decode(ex, oracle, live, last)
    ex.commit()
    for _ in range(2):
        _decode(ex, oracle, live, last)
    assert ex.placement.p_vector() == (1, 1, 1, 1)
    assert all(ex.read_kv(2, s)[1] == 0 for s in live)
    ex.close()


def test_abort_releases_reservations(runtime, confident):
    ex, oracle, live, last = _setup(runtime, confident)
    cat, cl = _cat_cl()
    use0 = [ex.mem_usage(d) for d in range(3)]
    ex.issue(O.ReplicateLayer(1, 1), cat, cl)
    ex.issue(O.MigrateLayer(3, 2, with_kv=True), cat, cl)
    mid = ex.mem_usage(1)
    assert mid["reserved_bytes"] >= 1704960 and mid["weight_bytes"] >= use0[1]["weight_bytes"] + 1704960
    _decode(ex, oracle, live, last)
    ex.abort()
    after = [ex.mem_usage(d) for d in range(3)]
    for a, b in zip(use0, after):
        assert (a["weight_bytes"], a["kv_bytes"], b["reserved_bytes"]) == (b["weight_bytes"], b["kv_bytes"], 0)
    assert not ex.pending_ops and ex.placement.p_vector() == (1, 1, 1, 1)
    ex.check_plan()
    for _ in range(2):
        _decode(ex, oracle, live, last)
    ex.close()


def test_7b_layer_migration_with_kv_during_decode(runtime):
    """A Llama-2-7B-geometry layer (404,766,720 B) + its KV migrates while 8
    decode steps of a 64-sequence batch run (2 layers + lm_head, 128-token
    prompts): teacher-forced logits within 2e-2 of the fp32 oracle and
    confident greedy tokens identical at every step; the placement switches only
    at the commit; the step-time jitter while the copy is in flight is printed
    (PAPER.md:679 reports < 3 % / < 5 % interference)."""
    from oracle.cpu_llama import LlamaConfig
    from oracle.torch_llama import TorchOracle

    cfg = LlamaConfig(2, 4096, 11008, 32, 32, 32000)
    w = init_weights(cfg, seed=4)
    B, L = 64, 128
    ex = Executor(runtime, ExecutorConfig(2, 4096, 11008, 32, vocab=32000, max_slots=B, max_ctx=L + 24,
                                          max_tokens=B * L))
    ex.load_model(w, device_of_layer=0)
    ref = TorchOracle(cfg, w, max_ctx=L + 24, max_slots=B, device="cuda")
    rng = np.random.default_rng(2)
    prompts = rng.integers(0, 32000, B * L).astype(np.int32)
    slots = np.arange(B, dtype=np.int32)
    _, lg, _ = ex.prefill(slots, prompts, np.full(B, L, np.int32), want_logits=True)
    want = ref.forward(slots, prompts, [L] * B)
    cat = D.ModuleCatalog.from_model(D.ModelSpec(2, 4096, 11008, 32))
    cl = D.ClusterSpec.b200(3)

    def step():
        nonlocal lg, want
        err = np.abs(lg - want).max()
        assert err <= LOGIT_TOL, err
        srt = np.sort(want, 1)
        sure = (srt[:, -1] - srt[:, -2]) > 2 * LOGIT_TOL
        assert np.array_equal(lg.argmax(1)[sure], want.argmax(1)[sure])
        inp = want.argmax(1).astype(np.int32)
        _, lg, ms = ex.decode(slots, inp, want_logits=True)
        want = ref.forward(slots, inp, None)
        return ms

    base = [step() for _ in range(4)]
    ex.issue(O.MigrateLayer(2, 1, with_kv=True), cat, cl)
    during, inflight = [], []
    for _ in range(8):
        inflight.append(not ex.ops_done())
        during.append(step())
        assert ex.placement.original_device(2) == 0
    ex.commit()
    after = [step() for _ in range(4)]
    step()
    m = ex.op_log[-1]
    assert m.weight_bytes == 404766720 and ex.placement.kv_device(2) == 1
    # pre-copy at issue: 132 tokens per slot (prompt + 4 steps); catch-up at the commit: the 8 appended since
    assert (m.kv_bytes, m.catchup_bytes) == (B * (L + 12) * 16384, B * 8 * 16384)
    jitter = during[0] / np.median(base) - 1.0
    print(f"7B layer + KV migration: {m.weight_bytes + m.kv_bytes} B, copy {m.copy_ms:.3f} ms "
          f"({(m.weight_bytes + m.kv_bytes - m.catchup_bytes) / m.copy_ms / 1e6:.0f} GB/s, same-GPU D2D), "
          f"catch-up {m.catchup_bytes} B in {m.catchup_ms:.3f} ms; step ms base {np.median(base):.3f}, "
          f"first step during copy {during[0]:.3f} (jitter {100 * jitter:+.1f} %), after {np.median(after):.3f}")
    ex.close()
