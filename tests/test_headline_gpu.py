"""Parity of the bench's exact configuration (BASELINE config 2) against the
fp32 oracle -- the plans the headline number is measured on, end to end.

The bench decodes Llama-2-7B geometry (d 4096, d_ff 11008, 32 heads, vocab
32000) at batch 256 after 128-token prompts.  Here the same executor
configuration (max_tokens / max_slots / max_ctx computed as bench.py does, so
prefill runs in 8192-row passes) runs 2 decoder layers + the lm_head with
oracle weights, prefill + 17 decode steps (attended context 129 .. 145), and
every step is teacher-forced against the fp32 oracle
(oracle/torch_llama.py on cuda, IEEE fp32 -- pinned on the CPU to the numpy
oracle, which is pinned to transformers):

* logits within the north star's 2e-2 max-abs at every step;
* greedy tokens identical wherever the oracle's top-2 margin exceeds 2x that.

At B = 256 the decode GEMMs run the token-major CTA-pair kernel (O / down
split over K in 4 parts) and RMSNorm is fused into the GEMM epilogues
(asserted from the plan); B = 1 / 16 / 64 / 128 are the bench's sweep points
(1-CTA kernel plans).  A replicated variant
splits layer 2 over two logical devices (split_batch(256, 2) = [128, 128]).
Reference semantics: sim.py:269-300 (prefill then decode), ops.py:151-158.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from oracle.cpu_llama import LlamaConfig, init_weights
from paper_2507_18006_b200 import domain as D
from paper_2507_18006_b200 import ops as O
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime


LOGIT_TOL = 2e-2
PROMPT, DECODE_STEPS = 128, 17
CFG = LlamaConfig(2, 4096, 11008, 32, 32, 32000)


@pytest.fixture(scope="module")
def weights():
    return init_weights(CFG, seed=21)


@pytest.fixture(scope="module")
def runtime(cuda):
    rt = Runtime([0, 0])
    yield rt
    rt.close()


def _bench_cfg(batch: int) -> ExecutorConfig:
    """bench.build_instance's geometry for this batch (max_tokens = 64 prompts per pass)."""
    return ExecutorConfig(n_layers=CFG.n_layers, d_model=CFG.d_model, d_ff=CFG.d_ff, n_heads=CFG.n_heads,
                          vocab=CFG.vocab, max_slots=batch, max_ctx=PROMPT + DECODE_STEPS + 8,
                          max_tokens=max(min(batch, 64) * PROMPT, 256))


def _plan(lib, N, K, T):
    names = ["tn", "pair", "box_rows", "csplit", "max_parts", "whole", "kd", "nw", "ksplit"]
    out = np.zeros(len(names), np.int32)
    assert lib.cbt_gemm_plan(N, K, T, 148, T, out.ctypes.data_as(C.c_void_p)) == 0
    return dict(zip(names, out.tolist()))


def _run(runtime, weights, batch, replicate_layer2=False):
    from oracle.torch_llama import TorchOracle

    cfg = _bench_cfg(batch)
    ex = Executor(runtime, cfg)
    ex.load_model(weights, device_of_layer=0)
    if replicate_layer2:
        cat = D.ModuleCatalog.from_model(D.ModelSpec(CFG.n_layers, CFG.d_model, CFG.d_ff, CFG.n_heads))
        ex.apply(O.ReplicateLayer(2, 1), cat, D.ClusterSpec.b200(2))
    ref = TorchOracle(CFG, weights, max_ctx=cfg.max_ctx, max_slots=batch, device="cuda")
    rng = np.random.default_rng(batch)
    prompts = rng.integers(0, CFG.vocab, batch * PROMPT).astype(np.int32)
    slots = np.arange(batch, dtype=np.int32)
    lens = np.full(batch, PROMPT, np.int32)
    replicas = {1: 2} if replicate_layer2 else None
    _, lg, _ = ex.prefill(slots, prompts, lens, want_logits=True)
    want = ref.forward(slots, prompts, lens, replicas)
    worst, checked, total = 0.0, 0, 0
    for step in range(DECODE_STEPS + 1):
        err = float(np.abs(lg - want).max())
        worst = max(worst, err)
        assert err <= LOGIT_TOL, (batch, step, err)
        srt = np.sort(want, axis=1)
        sure = (srt[:, -1] - srt[:, -2]) > 2 * LOGIT_TOL
        assert np.array_equal(lg.argmax(1)[sure], want.argmax(1)[sure]), (batch, step)
        checked += int(sure.sum())
        total += batch
        if step == DECODE_STEPS:
            break
        inp = want.argmax(1).astype(np.int32)  # teacher forcing: both consume the oracle's tokens
        _, lg, _ = ex.decode(slots, inp, want_logits=True)
        want = ref.forward(slots, inp, None, replicas)
    if replicate_layer2:
        q, r = divmod(batch, 2)
        assert ex.last_routing(2) == [(0, 0, q), (1, q, q + r)]
    ex.close()
    print(f"7B x2 layers, B={batch}{' (layer 2 replicated)' if replicate_layer2 else ''}: "
          f"max |logit - oracle| {worst:.4g} over prefill + {DECODE_STEPS} decode steps (ctx up to "
          f"{PROMPT + DECODE_STEPS}); {checked}/{total} confident decisions identical")
    assert checked >= total // 2
    return worst


def test_headline_plans(lib):
    """The plans the B = 256 case exercises (host-only choice, csrc/gemm.cu
    gemm_plan): QKV, gate/up and lm_head run the token-major CTA-pair kernel
    (wave-fitted nw-row weight tiles); O and down the same kernel with 256-row
    weight tiles split over K in 4 parts (parts exchanged through L2)."""
    for N, K in ((12288, 4096), (22016, 4096), (32000, 4096)):
        pl = _plan(lib, N, K, 256)
        assert pl["pair"] == 1 and pl["nw"] > 0 and pl["whole"] == 1 and pl["ksplit"] == 0, (N, K, pl)
    for N, K in ((4096, 4096), (4096, 11008)):
        pl = _plan(lib, N, K, 256)
        assert pl["pair"] == 1 and pl["ksplit"] == 4 and pl["nw"] == 256, (N, K, pl)
        pl = _plan(lib, N, K, 128)  # <= 128 rows: the 1-CTA kernel, cluster split-K
        assert pl["pair"] == 0 and pl["csplit"] == 4, (N, K, pl)
    assert _plan(lib, 12288, 4096, 64)["pair"] == 0


@pytest.mark.gpu
def test_headline_b256_matches_oracle(runtime, weights):
    _run(runtime, weights, 256)


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [1, 2, 16, 64, 128])
def test_sweep_batches_match_oracle(runtime, weights, batch):
    _run(runtime, weights, batch)


@pytest.mark.gpu
def test_headline_b256_replicated_layer_matches_oracle(runtime, weights):
    _run(runtime, weights, 256, replicate_layer2=True)
