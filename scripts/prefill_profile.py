"""Prefill of B prompts of length L (7B shape): device ms and per-class split."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
L = int(sys.argv[2]) if len(sys.argv) > 2 else 128
rt = Runtime([0])
cfg = ExecutorConfig(32, 4096, 11008, 32, vocab=32000, max_slots=B, max_ctx=L + 8, max_tokens=max(8192, L))
ex = Executor(rt, cfg, home_device=0, seed=7)
ex.init_head_random(std=0.02)
for li in range(1, 33):
    ex.init_layer_random(li, 0, std=0.02)
rng = np.random.default_rng(0)
slots = np.arange(B, dtype=np.int32)
toks = rng.integers(0, 32000, B * L).astype(np.int32)
ex.prefill(slots, toks, np.full(B, L, np.int32))
ex.release_all()
_, _, ms = ex.prefill(slots, toks, np.full(B, L, np.int32))
ex.release_all()
ex.profile(True)
ex.prefill(slots, toks, np.full(B, L, np.int32))
p = ex.profile_read()
ex.profile(False)
print(f"prefill B={B} L={L}: {ms:.1f} ms device ({B * L / ms * 1e3:.0f} tok/s)")
for k, v in p.items():
    print(f"  {k:12s} launches {v['launches']:5d}  ms {v['ms']:8.2f}  TFLOP/s {v['flops'] / max(v['ms'], 1e-9) / 1e9:7.1f}")
