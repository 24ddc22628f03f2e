"""Continuous-batching serving loop driving the B200 executor in real time.

Follows the reference Engine's per-instance semantics (sim.py:624-736) with
wall-clock time instead of simulated time:

* arrivals (``generate_arrivals``-compatible ``Request`` lists, or a trace)
  are routed to instances with ``schedule`` (sim.py:157-184) and queued FIFO;
* an idle instance admits from its queue up to ``max_batch_size``
  (sim.py:713-714); if any admitted request is not prefilled, the step is a
  prefill of only those requests (sim.py:717-725), otherwise one decode step
  of the whole batch (sim.py:726-732);
* completion (sim.py:637-668): prefill marks requests prefilled and deposits
  their prompt tokens in the KV accounting; decode adds one token per request,
  removes finished requests in batch order and releases their KV;
* per-request latency = completion - arrival; tok/s = generated tokens /
  wall window; p50/p99 with ``np.percentile`` (sim.py:333-338).

* out-of-memory (sim.py:670-707): after every step each device's memory --
  the catalog accounting of every instance's placement plus its resident KV
  and pending reservations (the reference's ``_device_memory_mb``) plus the
  executor's workspaces (``mem_usage``: memory no module explains, the same
  "foreign load" the controller sees) -- is checked against the ClusterSpec
  capacity (``detect_oom``); a step that fails to allocate device memory
  (CB_ENOMEM) is an OOM too.  The instances touching
  the device crash: their batch is dropped (KV released), each request is
  requeued at the queue head once and fails the second time, and the instance
  is unavailable for ``oom_restart_s``;
* scaling decisions are carried out by ``on_step`` hooks at step boundaries
  (control.AutoscaleHook: issue while serving, switch placement + batch cap +
  KV offload atomically when the copies are done, sim.py:614-622).
"""
from __future__ import annotations

import time
from collections import deque
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from . import domain as D
from . import ops as O
from .sim import Request, schedule


@dataclass
class InstanceState:
    """One served model instance (reference ``_Instance``, sim.py:405-426)."""

    id: int
    executor: object
    max_batch_size: int
    queue: deque = field(default_factory=deque)
    batch: list = field(default_factory=list)
    resident_tokens: int = 0  # per KV-holding layer
    speedup: float = 1.0
    busy_s: float = 0.0
    steps: dict = field(default_factory=lambda: {"prefill": 0, "decode": 0})
    offload_fraction: float = 0.0
    reserved_mb: dict = field(default_factory=dict)  # pending transition's reservation (sim.py:817-831)
    unavailable_until_s: float = 0.0                 # restarting after an OOM crash

    @property
    def depth(self) -> int:
        return len(self.queue) + len(self.batch)


@dataclass
class ServingResult:
    completed: list
    wall_s: float
    generated_tokens: int
    step_log: list  # (t_start_s, kind, instance, bs, device_s, wall_s)
    failed: list = field(default_factory=list)
    oom_events: list = field(default_factory=list)  # (t_s, device)

    @property
    def latencies_s(self) -> np.ndarray:
        return np.array([r.completion_s - r.arrival_s for r in self.completed], dtype=np.float64)

    def summary(self) -> dict:
        lat = self.latencies_s
        p50, p95, p99 = (np.percentile(lat, [50.0, 95.0, 99.0]) if lat.size else (0.0, 0.0, 0.0))
        dec = [s for s in self.step_log if s[1] == "decode"]
        return {
            "completed": len(self.completed),
            "failed": len(self.failed),
            "oom_events": len(self.oom_events),
            "generated_tokens": self.generated_tokens,
            "wall_s": self.wall_s,
            "throughput_tok_s": self.generated_tokens / self.wall_s if self.wall_s else 0.0,
            "p50_latency_s": float(p50), "p95_latency_s": float(p95), "p99_latency_s": float(p99),
            "mean_latency_s": float(lat.mean()) if lat.size else 0.0,
            "decode_steps": len(dec),
            "mean_decode_batch": float(np.mean([s[3] for s in dec])) if dec else 0.0,
            "device_busy_s": float(sum(s[4] for s in self.step_log)),
        }


class ServingEngine:
    """Single host thread, one or more instances, real time."""

    def __init__(self, instances: Sequence[InstanceState], seed: int = 0,
                 clock: Callable[[], float] = time.perf_counter, sleep: Callable[[float], None] = time.sleep,
                 cluster: D.ClusterSpec | None = None, catalog: D.ModuleCatalog | None = None,
                 oom_restart_s: float = 1.0):
        self.instances = sorted(instances, key=lambda i: i.id)
        self.cluster, self.catalog = cluster, catalog
        self.oom_restart_s = oom_restart_s
        self.failed: list = []
        self.oom_events: list = []
        self._oom_seen: set = set()
        ss = np.random.SeedSequence(seed)
        _, sched_seed = ss.spawn(2)  # same stream layout as the reference Engine (sim.py:441-443)
        self.sched_rng = np.random.Generator(np.random.PCG64(sched_seed))
        self.clock = clock
        self.sleep = sleep
        self.completed: list = []
        self.generated = 0
        self.step_log: list = []
        self.on_step: Callable | None = None  # hook(engine, t_s) at step boundaries (controller / commits)

    def _dispatch(self, req: Request) -> None:
        view = [(i.id, i.depth, i.speedup) for i in self.instances]
        target = schedule(view, self.sched_rng)
        req.instance = target
        next(i for i in self.instances if i.id == target).queue.append(req)

    # ------------------------------------------------------------ memory / OOM (sim.py:499-525, 670-707)
    def device_memory_mb(self, device_id: int) -> float:
        total = 0.0
        for inst in self.instances:
            ex = inst.executor
            placement = ex.placement
            if self.catalog is not None:
                usage = D.device_usage(placement, self.catalog)
                total += usage[device_id].memory_mb if device_id in usage else 0.0
                n_kv = D.kv_resident_layer_count(placement).get(device_id, 0)
                total += (inst.resident_tokens * self.catalog.kv_bytes_per_token_per_layer * n_kv / 1e6
                          * (1.0 - inst.offload_fraction))
            total += inst.reserved_mb.get(device_id, 0.0)
            if hasattr(ex, "mem_usage") and device_id < getattr(getattr(ex, "rt", None), "n_devices", 0):
                total += ex.mem_usage(device_id)["workspace_bytes"] / 1e6
        return total

    def _check_oom(self, t_s: float) -> None:
        if self.cluster is None:
            return
        for dev in self.cluster.devices:
            if self.device_memory_mb(dev.id) > dev.memory_mb:  # detect_oom (sim.py:303-305)
                self._oom(dev.id, t_s)

    def _oom(self, device_id: int, t_s: float) -> None:
        key = (round(t_s, 6), device_id)
        if key not in self._oom_seen:
            self._oom_seen.add(key)
            self.oom_events.append((t_s, device_id))
        for inst in self.instances:
            if inst.batch and device_id in inst.executor.placement.devices_used():
                self._crash(inst, t_s)

    def _crash(self, inst: InstanceState, t_s: float) -> None:
        """Drop the batch; requeue each request once at the queue head, fail it the second time."""
        victims = list(inst.batch)
        inst.batch = []
        inst.resident_tokens = 0
        inst.unavailable_until_s = t_s + self.oom_restart_s
        inst.executor.release(victims)
        for r in reversed(victims):
            r.generated = 0
            r.prefilled = False
            r.output_tokens = []
            if r.requeued:
                r.failed = True
                r.completion_s = t_s
                self.failed.append(r)
            else:
                r.requeued = True
                inst.queue.appendleft(r)

    def busy_fraction(self, t_s: float, window_s: float) -> dict:
        """Share of the last ``window_s`` each instance's devices spent in steps."""
        lo = max(0.0, t_s - window_s)
        span = max(1e-9, t_s - lo)
        out: dict = {}
        for t0, _, iid, _, _, wall in self.step_log:
            busy = max(0.0, min(t_s, t0 + wall) - max(lo, t0))
            if busy <= 0:
                continue
            inst = next(i for i in self.instances if i.id == iid)
            for dev in inst.executor.placement.devices_used():
                out[dev] = out.get(dev, 0.0) + busy / span
        return {d: min(1.0, v) for d, v in out.items()}

    def _step(self, inst: InstanceState, t_s: float) -> bool:
        if t_s < inst.unavailable_until_s:
            return False
        while len(inst.batch) < inst.max_batch_size and inst.queue:
            inst.batch.append(inst.queue.popleft())
        if not inst.batch:
            return False
        fresh = [r for r in inst.batch if not r.prefilled]
        kind = "prefill" if fresh else "decode"
        group = fresh if fresh else inst.batch
        w0 = self.clock()
        try:
            out = inst.executor.step_batch(group, kind)
        except O.InfeasibleOpError:  # the step could not allocate device memory: a physical OOM
            self._oom(inst.executor.placement.original_device(1), self.clock() - self.t0)
            return True
        wall = self.clock() - w0
        inst.busy_s += wall
        inst.steps[kind] += 1
        self.step_log.append((t_s, kind, inst.id, len(group), out.duration_s, wall))
        done_t = self.clock() - self.t0
        if kind == "prefill":
            for r in fresh:
                r.prefilled = True
            inst.resident_tokens += out.kv_tokens_delta
            self._check_oom(done_t)
            return True
        inst.resident_tokens += out.kv_tokens_delta
        self.generated += len(inst.batch)
        finished = []
        for r in inst.batch:
            r.generated += 1
            if r.generated >= r.gen_len:
                finished.append(r)
        for r in finished:
            inst.batch.remove(r)
            inst.resident_tokens -= r.prompt_len + r.generated
            r.completion_s = done_t
            self.completed.append(r)
        if finished:
            inst.executor.release(finished)
        self._check_oom(done_t)
        return True

    def run(self, arrivals: Sequence[Request], duration_s: float | None = None,
            drain: bool = True) -> ServingResult:
        """Serve ``arrivals``; stop when everything arrived and (if ``drain``)
        finished, or at ``duration_s`` without draining."""
        pending = deque(sorted(arrivals, key=lambda r: (r.arrival_s, r.id)))
        self.t0 = self.clock()
        while True:
            t = self.clock() - self.t0
            if duration_s is not None and not drain and t >= duration_s:
                break
            while pending and pending[0].arrival_s <= t:
                self._dispatch(pending.popleft())
            if self.on_step is not None:
                self.on_step(self, t)
            worked = False
            for inst in self.instances:
                worked |= self._step(inst, t)
            if worked:
                continue
            restarting = [i.unavailable_until_s for i in self.instances if i.queue and i.unavailable_until_s > t]
            if not pending and not restarting:
                break  # idle and nothing more will arrive
            nxt = min(([pending[0].arrival_s] if pending else []) + restarting)
            wait = nxt - (self.clock() - self.t0)
            if wait > 0:
                self.sleep(min(wait, 0.001))
        return ServingResult(self.completed, self.clock() - self.t0, self.generated, self.step_log, self.failed,
                             self.oom_events)


def poisson_arrivals(rps: float, duration_s: float, prompt_len: int, gen_len: int, seed: int) -> list:
    """Seeded Poisson arrivals, the reference's generator layout (sim.py:126-150)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed)))
    out, t = [], 0.0
    while rps > 0:
        t += rng.exponential(1.0 / rps)
        if t > duration_s:
            break
        out.append(Request(len(out), t, prompt_len, gen_len))
    return out


def bursty_trace(low_rps: float, high_rps: float, low_s: float, high_s: float, duration_s: float, prompt_len: int,
                 gen_len: int, seed: int) -> list:
    """Config 3's bursty trace: alternate low_s at low_rps and high_s at high_rps."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed)))
    out, t, phase_end, high = [], 0.0, low_s, False
    while t < duration_s:
        rate = high_rps if high else low_rps
        t += rng.exponential(1.0 / rate)
        while t > phase_end and phase_end < duration_s:
            t = phase_end + rng.exponential(1.0 / (low_rps if high else high_rps))
            high = not high
            phase_end += high_s if high else low_s
        if t <= duration_s:
            out.append(Request(len(out), t, prompt_len, gen_len))
    return out
