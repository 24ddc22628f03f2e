"""Debug: synchronous scaling ops on fresh runtimes (one GPU, logical devices)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from oracle.cpu_llama import TINY, init_weights
from paper_2507_18006_b200 import domain as D
from paper_2507_18006_b200 import ops as O
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime

w = init_weights(TINY, 3)
cat = D.ModuleCatalog.from_model(D.ModelSpec(4, 256, 768, 4))
for rnd, ords in enumerate(([0, 0, 0], [0, 0], [0, 0])):
    rt = Runtime(ords)
    ex = Executor(rt, ExecutorConfig(4, 256, 768, 4, vocab=1024, max_slots=16, max_ctx=32, max_tokens=256))
    ex.load_model(w, device_of_layer=0)
    for op in (O.ReplicateLayer(2, 1), O.MigrateLayer(3, 1, with_kv=True), O.EvictReplica(2, 1)):
        try:
            ex.apply(op, cat, D.ClusterSpec.b200(len(ords)))
            print(rnd, op, "ok", ex.op_log[-1])
        except Exception as e:
            print(rnd, op, "FAIL", e)
    rt.close()
