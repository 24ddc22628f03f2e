"""The reference controller scaling a live B200 instance mid-serving.

Config-1 model (confident head) on two logical devices of one B200; the
unmodified reference ``controller_step`` decides a scale-up (Alg. 1) after the
prefill, the decision is committed physically between decode steps (layer
blocks copied, rows re-split, KV rows follow), and every decode step keeps
matching the CPU oracle.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle.cpu_llama import TINY, OracleModel, init_weights
from oracle.gen_golden import CONFIG1_SEED, config1_prompts
from paper_2507_18006_b200 import domain as D
from paper_2507_18006_b200.control import ReferenceController, load_reference
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime

ms = load_reference()
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(ms is None, reason="reference modscale not importable")]


def test_reference_scale_up_mid_serving(cuda):
    w = init_weights(TINY, CONFIG1_SEED, head="permuted_tied")
    prompts = config1_prompts()
    rt = Runtime([0, 0])
    ex = Executor(rt, ExecutorConfig(4, 256, 768, 4, vocab=1024, max_slots=32, max_ctx=64, max_tokens=512))
    ex.load_model(w, 0)
    model = D.ModelSpec(4, 256, 768, 4)
    cat = D.ModuleCatalog.from_model(model)
    cluster = D.ClusterSpec.b200(2)
    oracle = OracleModel(TINY, w, 64)
    live = list(range(15))
    slots = np.array(live, np.int32)
    nxt, _, _ = ex.prefill(slots, np.concatenate(prompts), np.full(15, 16, np.int32))
    oracle.forward(live, np.concatenate(prompts), [16] * 15)
    for step in range(8):
        if step == 2:
            ctl = ReferenceController(ex, cluster, model, cat, ms=ms)
            dec = ctl.decide(bs=15, kv_tokens=16 + step)
            assert dec.trigger == "scale_up"
            done = ctl.commit(dec)
            assert len(done) == 4 and ex.placement.p_vector() == (2, 2, 2, 2)
            assert all(m.weight_bytes == ex.module_bytes("decoder_layer") for m in ex.op_log[-4:])
        inp = nxt
        nxt, lg, _ = ex.decode(slots, inp, want_logits=True)
        ref = oracle.forward(live, inp, None)
        assert np.array_equal(nxt, ref.argmax(-1)), step
        assert np.abs(lg - ref).max() <= 2e-2
    assert ex.last_routing(3) == [(0, 0, 7), (1, 7, 8)]
    ex.close()
    rt.close()


def test_reference_compute_bound_scale_down_moves_projections(cuda):
    """Device 0 compute-bound (busy 0.99) with SLO violations: the reference's
    scale-down Phase 1 (autoscaler.py:505-583, filter_modules 407-419) emits
    MigrateSubModule ops for FFN projections; they are committed physically
    between decode steps and every step keeps matching the CPU oracle."""
    w = init_weights(TINY, CONFIG1_SEED, head="permuted_tied")
    prompts = config1_prompts()
    rt = Runtime([0, 0])
    ex = Executor(rt, ExecutorConfig(4, 256, 768, 4, vocab=1024, max_slots=32, max_ctx=64, max_tokens=512))
    ex.load_model(w, 0)
    model = D.ModelSpec(4, 256, 768, 4)
    cat = D.ModuleCatalog.from_model(model)
    cluster = D.ClusterSpec.b200(2)
    oracle = OracleModel(TINY, w, 64)
    live = list(range(15))
    slots = np.array(live, np.int32)
    nxt, _, _ = ex.prefill(slots, np.concatenate(prompts), np.full(15, 16, np.int32))
    oracle.forward(live, np.concatenate(prompts), [16] * 15)
    moved = []
    for step in range(6):
        if step == 2:
            ctl = ReferenceController(ex, cluster, model, cat, ms=ms)
            dec = ctl.decide(bs=15, kv_tokens=16 + step, violation_rate=0.5, busy={0: 0.99})
            assert dec.trigger == "scale_down"
            done = ctl.commit(dec)
            moved = [(op.layer, op.kind) for op, _ in done]
            assert moved and all(k in (D.ModuleKind.FFN_PROJ_GATE, D.ModuleKind.FFN_PROJ_UP,
                                       D.ModuleKind.FFN_PROJ_DOWN) for _, k in moved)
            assert all(ex.placement.override_device(li, k) == 1 for li, k in moved)
        inp = nxt
        nxt, lg, _ = ex.decode(slots, inp, want_logits=True)
        ref = oracle.forward(live, inp, None)
        assert np.array_equal(nxt, ref.argmax(-1)), step
        assert np.abs(lg - ref).max() <= 2e-2
    assert len(moved) == 4
    ex.close()
    rt.close()
