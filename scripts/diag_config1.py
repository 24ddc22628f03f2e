"""Diagnostic: config-1 GPU logits vs the bf16-faithful and fp32 oracles, teacher-forced."""
import sys
import numpy as np
sys.path.insert(0, '.')
from oracle.cpu_llama import TINY, OracleModel, greedy_generate, init_weights, top2_margin
from oracle.gen_golden import CONFIG1_SEED, config1_prompts
from paper_2507_18006_b200 import ops as O, domain as D
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime

w = init_weights(TINY, CONFIG1_SEED)
prompts = config1_prompts()
rt = Runtime([0, 0])
for rep in (False, True):
    ex = Executor(rt, ExecutorConfig(4, 256, 768, 4, vocab=1024, max_slots=32, max_ctx=64, max_tokens=512))
    ex.load_model(w, 0)
    if rep:
        ex.apply(O.ReplicateLayer(2, 1), D.ModuleCatalog.from_model(D.ModelSpec(4, 256, 768, 4)), D.ClusterSpec.b200(2))
    fa = OracleModel(TINY, w, 64, bf16_acts=True)
    fp = OracleModel(TINY, w, 64)
    ref_toks, _ = greedy_generate(OracleModel(TINY, w, 64, bf16_acts=True), prompts, 32)
    slots = np.arange(15, dtype=np.int32)
    _, lg, _ = ex.prefill(slots, np.concatenate(prompts), np.full(15, 16, np.int32), True)
    la = fa.forward(list(range(15)), np.concatenate(prompts), [16] * 15)
    lp = fp.forward(list(range(15)), np.concatenate(prompts), [16] * 15)
    print("rep", rep, "step 0: dev faithful %.2e fp32 %.2e margin %.2e" % (np.abs(lg - la).max(), np.abs(lg - lp).max(), top2_margin(la)))
    worst = 0
    for s in range(1, 32):
        _, lg, _ = ex.decode(slots, ref_toks[:, s - 1], True)
        la = fa.forward(list(range(15)), ref_toks[:, s - 1], None)
        lp = fp.forward(list(range(15)), ref_toks[:, s - 1], None)
        dv = np.abs(lg - la).max(); worst = max(worst, dv)
        mism = (lg.argmax(-1) != la.argmax(-1)).sum()
        if s % 8 == 0 or mism:
            print(" step %d dev faithful %.2e fp32 %.2e margin %.2e argmax-mismatch %d" % (s, dv, np.abs(lg - lp).max(), top2_margin(la), mism))
    print("worst faithful dev", worst)
    ex.close()
