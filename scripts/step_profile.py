"""One 7B decode step for profiling: prefill, warm decode steps, then the
profiled step(s) bracketed by cudaProfilerStart/Stop (use ncu
--profile-from-start off).  Without ncu it prints device ms per step and the
per-class breakdown of the executor's live profile.

    python scripts/step_profile.py BATCH [STEPS] [CTX]   (CTX: attended context of the profiled step, default 131)"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
STEPS = int(sys.argv[2]) if len(sys.argv) > 2 else 1
CTX = int(sys.argv[3]) if len(sys.argv) > 3 else 131
rt = Runtime([0])
cfg = ExecutorConfig(32, 4096, 11008, 32, vocab=32000, max_slots=B, max_ctx=max(160, CTX + STEPS + 12),
                     max_tokens=max(min(B, 64) * 128, 256))
ex = Executor(rt, cfg, home_device=0, seed=7)
ex.init_head_random(std=0.02)
for li in range(1, 33):
    ex.init_layer_random(li, 0, std=0.02)
rng = np.random.default_rng(0)
slots = np.arange(B, dtype=np.int32)
nxt, _, _ = ex.prefill(slots, rng.integers(0, 32000, B * 128).astype(np.int32), np.full(B, 128, np.int32))
for _ in range(max(3, CTX - 128)):
    nxt, _, ms = ex.decode(slots, nxt)
ms_all, enq = [], []
from paper_2507_18006_b200 import _lib
lib = _lib.load()
torch.cuda.profiler.start()
for _ in range(STEPS):
    nxt, _, ms = ex.decode(slots, nxt)
    ms_all.append(ms)
    enq.append(lib.cbt_last_enqueue_ms())
torch.cuda.profiler.stop()
print(f"B={B}: decode step device ms {np.mean(ms_all):.3f} ({B / np.mean(ms_all) * 1e3:.0f} tok/s)"
      f"  host enqueue ms {np.mean(enq):.3f}")
ex.profile(True)
for _ in range(3):
    nxt, _, ms = ex.decode(slots, nxt)
p = ex.profile_read()
ex.profile(False)
for k, v in p.items():
    print(f"  {k:12s} launches/step {v['launches'] / 3:6.1f}  ms/step {v['ms'] / 3:7.3f}  "
          f"GB/s {v['bytes'] / max(v['ms'], 1e-9) / 1e6:7.0f}")
