"""The serving loop on the real executor: OOM crash / requeue / fail, and the
reference controller preventing the OOM by moving KV while serving (GPU).

Config-1 model (confident head) on two logical devices of one B200.  Device
0's capacity is set so that the resident KV of four requests crosses it on the
11th decode commit (the reference's ``oom_scenario`` shape, tests/test_sim.py:
229-271, scaled to the tiny model): capacity = catalog static MB of the 4
layers + the executor's workspaces + the KV of 64 + 4 * 10 tokens.

* no controller: the batch crashes there, is requeued once, crashes again and
  every request fails (sim.py:670-707), KV slots released each time;
* with ``AutoscaleHook`` (the unmodified reference ``controller_step``): the
  projected OOM triggers a scale-down whose KV-cache migrations to device 1 are
  issued while decoding continues and switched at a step boundary; no OOM, and
  every request's greedy tokens equal the fp32 oracle's.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle.cpu_llama import TINY, OracleModel, greedy_generate, init_weights
from oracle.gen_golden import CONFIG1_SEED, config1_prompts
from paper_2507_18006_b200 import domain as D
from paper_2507_18006_b200.control import AutoscaleHook, ReferenceController, load_reference
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime
from paper_2507_18006_b200.serving import InstanceState, ServingEngine
from paper_2507_18006_b200.sim import Request

ms = load_reference()
pytestmark = pytest.mark.gpu
N, PROMPT, GEN = 4, 16, 24


@pytest.fixture(scope="module")
def confident():
    return init_weights(TINY, CONFIG1_SEED, head="permuted_tied")


def _engine(w, controller: bool):
    rt = Runtime([0, 0])
    ex = Executor(rt, ExecutorConfig(4, 256, 768, 4, vocab=1024, max_slots=16, max_ctx=64, max_tokens=256))
    ex.load_model(w, 0)
    model = D.ModelSpec(4, 256, 768, 4)
    cat = D.ModuleCatalog.from_model(model)
    ws0 = ex.mem_usage(0)["workspace_bytes"] / 1e6
    kv_tok_mb = 4 * cat.kv_bytes_per_token_per_layer / 1e6
    cap0 = 4 * cat.decoder_layer_mb + ws0 + (N * PROMPT + 4 * 10) * kv_tok_mb + 1e-6
    cluster = D.ClusterSpec.uniform([D.DeviceSpec(0, 2.25e6, cap0), D.DeviceSpec(1, 2.25e6, 180000.0)], 900000.0,
                                    8e6)
    inst = InstanceState(0, ex, max_batch_size=N)
    eng = ServingEngine([inst], cluster=cluster, catalog=cat, oom_restart_s=0.05)
    hook = None
    if controller:
        ctl = ReferenceController(ex, cluster, model, cat, ms=ms,
                                  cfg=ms.autoscaler.ControllerConfig(compute_pressure=1.01))
        hook = AutoscaleHook(ctl, inst, interval_s=0.0, prompt_len=PROMPT, gen_len=GEN)
        eng.on_step = hook
    prompts = config1_prompts()[:N]
    reqs = [Request(i, 0.0, PROMPT, GEN, prompt_tokens=prompts[i]) for i in range(N)]
    return rt, ex, eng, hook, reqs, prompts


def test_oom_crash_requeue_then_fail_on_gpu(confident):
    rt, ex, eng, _, reqs, _ = _engine(confident, controller=False)
    res = eng.run(reqs)
    s = res.summary()
    assert s["oom_events"] >= 2 and (s["completed"], s["failed"]) == (0, N)
    assert all(r.requeued and r.failed for r in res.failed)
    decodes = [x for x in res.step_log if x[1] == "decode"]
    assert len(decodes) == 2 * 11  # the 11th decode commit crosses, twice
    ex.close()
    rt.close()


@pytest.mark.skipif(ms is None, reason="reference modscale not importable")
def test_controller_moves_kv_while_serving_and_prevents_oom(confident):
    rt, ex, eng, hook, reqs, prompts = _engine(confident, controller=True)
    res = eng.run(reqs)
    s = res.summary()
    assert (s["oom_events"], s["failed"], s["completed"]) == (0, 0, N), (s, hook.decisions)
    assert hook.switches and hook.switches[0][1] == "scale_down"
    moved = [li for li in range(1, 5) if ex.placement.kv_device(li) == 1]
    assert moved, ex.placement
    assert any(m.catchup_bytes is not None for m in ex.op_log)  # committed through the asynchronous path
    ref, _ = greedy_generate(OracleModel(TINY, confident, 64), prompts, GEN + 1)
    got = np.array([r.output_tokens for r in sorted(res.completed, key=lambda r: r.id)])
    assert np.array_equal(got, ref)
    ex.close()
    rt.close()
