"""Token / logit check of a config script's scenario against the fp32 oracle.

TEST INFRASTRUCTURE (imports oracle/): the config scripts measure on
random-init 7B / 13B / 70B models of 32-80 layers, which no CPU oracle can
follow.  This check rebuilds the same geometry with two decoder layers of
oracle weights, applies the same kind of placement and scaling ops through the
same executor API (``scenario(ex, cat, cluster, step)`` is called before every
decode step), and teacher-forces every step against oracle/torch_llama.py
(IEEE fp32 on cuda, pinned to the numpy oracle in tests/): logits within the
north star's 2e-2 max-abs, greedy tokens identical wherever the oracle's
top-2 margin exceeds 4e-2.  Raises AssertionError on a mismatch.
"""
from __future__ import annotations

import sys
from pathlib import Path
from typing import Callable

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from oracle.cpu_llama import LlamaConfig, init_weights  # noqa: E402
from oracle.torch_llama import TorchOracle  # noqa: E402
from paper_2507_18006_b200 import domain as D  # noqa: E402
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime  # noqa: E402

TOL = 2e-2


def check(geom: dict, n_dev: int, batch: int, prompt: int, steps: int,
          scenario: Callable | None = None, device_of_layer=0, release: dict | None = None) -> dict:
    """geom: d_model, d_ff, n_heads (+ n_kv_heads); 2 decoder layers, vocab 32000.
    release: {step: [sequence indices]} finished before that decode step."""
    H, Hkv = geom["n_heads"], geom.get("n_kv_heads") or geom["n_heads"]
    cfg_o = LlamaConfig(2, geom["d_model"], geom["d_ff"], H, Hkv, 32000)
    w = init_weights(cfg_o, seed=17)
    rt = Runtime([0] * n_dev)
    cfg = ExecutorConfig(n_layers=2, d_model=geom["d_model"], d_ff=geom["d_ff"], n_heads=H,
                         n_kv_heads=None if Hkv == H else Hkv, vocab=32000, max_slots=batch,
                         max_ctx=prompt + steps + 8, max_tokens=max(batch * prompt, 256))
    ex = Executor(rt, cfg)
    ex.load_model(w, device_of_layer=device_of_layer)
    cat = D.ModuleCatalog.from_model(D.ModelSpec(2, geom["d_model"], geom["d_ff"], H))
    cluster = D.ClusterSpec.b200(n_dev)
    ref = TorchOracle(cfg_o, w, max_ctx=cfg.max_ctx, max_slots=batch, device="cuda")
    rng = np.random.default_rng(23)
    live = list(range(batch))
    prompts = rng.integers(0, 32000, batch * prompt).astype(np.int32)
    if scenario:
        scenario(ex, cat, cluster, 0)
    _, lg, _ = ex.prefill(np.array(live, np.int32), prompts, np.full(batch, prompt, np.int32), want_logits=True)
    want = ref.forward(np.array(live, np.int32), prompts, np.full(batch, prompt, np.int32))
    worst, sure_n, same_n = 0.0, 0, 0
    for step in range(1, steps + 1):
        worst = max(worst, float(np.abs(lg - want).max()))
        srt = np.sort(want, axis=1)
        sure = (srt[:, -1] - srt[:, -2]) > 2 * TOL
        sure_n += int(sure.sum())
        same_n += int((lg.argmax(1)[sure] == want.argmax(1)[sure]).sum())
        nxt = dict(zip(live, want.argmax(1).astype(np.int32)))  # teacher forcing
        for q in (release or {}).get(step, []):
            live.remove(q)
            ex.release_slots(np.array([q], np.int32))
            ref.release([q])
        if scenario:
            scenario(ex, cat, cluster, step)
        slots = np.array(live, np.int32)
        inp = np.array([nxt[q] for q in live], np.int32)
        _, lg, _ = ex.decode(slots, inp, want_logits=True)
        want = ref.forward(slots, inp, None)
    worst = max(worst, float(np.abs(lg - want).max()))
    placement = [list(r.device_id for r in row) for row in ex.placement.replicas]
    ex.close()
    rt.close()
    del ref
    res = {"max_abs_logit_err": worst, "tol": TOL, "confident_decisions": sure_n, "identical": same_n,
           "pass": bool(worst <= TOL and same_n == sure_n), "placement_layers_1_2": placement,
           "what": f"2 layers of the same geometry with oracle weights, batch {batch}, prompt {prompt}, "
                   f"{steps} teacher-forced decode steps with the same placement / ops vs the fp32 oracle"}
    assert res["pass"], res
    return res
