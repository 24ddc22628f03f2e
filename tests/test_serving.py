"""Continuous-batching loop semantics (CPU, fake executor with a virtual clock).

The loop must follow the reference Engine (sim.py:624-736): FIFO admission up
to max_batch_size, prefill-only steps for fresh requests, decode steps over the
whole batch, in-order removal of finished requests, KV token accounting
(prefill deposits sum of prompts, decode +bs, completion frees prompt+generated).
"""
from __future__ import annotations

import numpy as np

from paper_2507_18006_b200.serving import InstanceState, ServingEngine, bursty_trace, poisson_arrivals
from paper_2507_18006_b200.sim import Request, StepOutcome


class FakeClock:
    def __init__(self):
        self.t = 0.0

    def __call__(self):
        return self.t

    def sleep(self, dt):
        self.t += dt


class FakeExecutor:
    """Advances a virtual clock by a fixed cost per step; records the calls."""

    def __init__(self, clock, prefill_s=0.02, decode_s=0.01):
        self.clock, self.prefill_s, self.decode_s = clock, prefill_s, decode_s
        self.calls, self.released = [], []

    def step_batch(self, batch, phase):
        self.calls.append((phase, [r.id for r in batch]))
        dur = self.prefill_s if phase == "prefill" else self.decode_s
        self.clock.t += dur
        kv = sum(r.prompt_len for r in batch) if phase == "prefill" else len(batch)
        return StepOutcome(dur, kv)

    def release(self, reqs):
        self.released.extend(r.id for r in reqs)


def _run(reqs, max_bs=4, **kw):
    clock = FakeClock()
    ex = FakeExecutor(clock, **kw)
    inst = InstanceState(0, ex, max_bs)
    eng = ServingEngine([inst], clock=clock, sleep=clock.sleep)
    res = eng.run(reqs)
    return ex, inst, res


def test_prefill_then_decode_fifo_and_completion():
    reqs = [Request(i, 0.0, 8 + i, 3) for i in range(6)]
    ex, inst, res = _run(reqs, max_bs=4)
    # first step: prefill of the 4 admitted requests only; then decode of the batch
    assert ex.calls[0] == ("prefill", [0, 1, 2, 3])
    assert ex.calls[1] == ("decode", [0, 1, 2, 3])
    # after 3 decodes requests 0..3 finish together, then 4, 5 are admitted and prefilled
    assert ex.calls[4] == ("prefill", [4, 5])
    assert [r.id for r in res.completed] == [0, 1, 2, 3, 4, 5]
    assert all(r.generated == r.gen_len for r in res.completed)
    assert sorted(ex.released) == list(range(6))
    assert inst.resident_tokens == 0  # all KV released
    assert res.generated_tokens == sum(r.gen_len for r in reqs)


def test_staggered_lengths_ordered_removal():
    reqs = [Request(0, 0.0, 4, 1), Request(1, 0.0, 4, 3), Request(2, 0.0, 4, 2)]
    ex, inst, res = _run(reqs, max_bs=3)
    assert [r.id for r in res.completed] == [0, 2, 1]
    decodes = [c for c in ex.calls if c[0] == "decode"]
    assert [len(ids) for _, ids in decodes] == [3, 2, 1]


def test_latency_is_completion_minus_arrival():
    reqs = [Request(0, 0.0, 4, 2), Request(1, 0.05, 4, 2)]
    _, _, res = _run(reqs, max_bs=1)
    lat = res.latencies_s
    assert np.all(lat > 0)
    s = res.summary()
    assert s["completed"] == 2 and s["p99_latency_s"] >= s["p50_latency_s"]


def test_arrival_generators_deterministic():
    a = poisson_arrivals(10.0, 5.0, 128, 16, seed=7)
    b = poisson_arrivals(10.0, 5.0, 128, 16, seed=7)
    assert [r.arrival_s for r in a] == [r.arrival_s for r in b]
    assert abs(len(a) / 5.0 - 10.0) < 5.0
    t = bursty_trace(5.0, 50.0, 10.0, 5.0, 60.0, 128, 16, seed=7)
    ts = np.array([r.arrival_s for r in t])
    assert np.all(np.diff(ts) >= 0) and ts.max() <= 60.0
    hi = ((ts % 15.0) >= 10.0).sum() / 5.0 / 4  # per-second rate inside the high phases
    lo = ((ts % 15.0) < 10.0).sum() / 10.0 / 4
    assert hi > 3 * lo
