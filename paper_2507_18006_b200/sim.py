"""Serving-side seams of the data path: request router, step plan, step hook.

Drop-in for the parts of ``modscale.sim`` (reference ``sim.py``) on the
north-star path:

* ``schedule`` -- speedup-weighted shortest-queue router with seeded
  tie-breaking (sim.py:157-184); bit-exact including the RNG draws;
* ``StepArrays`` / ``build_step_arrays`` -- the placement flattened into the
  executor plan (sim.py:204-236);
* ``Request`` / ``StepOutcome`` / ``step_batch`` -- the executor hook
  (sim.py:261-300).  In the reference ``step_batch`` prices a pass with the
  analytic ``work_units``/``comm_units`` stand-ins; here it runs the pass on
  the B200s through ``Executor`` and returns the *measured* duration with the
  reference's KV accounting (prefill: sum of prompt lengths; decode: batch
  size).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import ops as _ops
from .domain import ClusterSpec, PlacementState, kv_resident_layer_count


class SimError(ValueError):
    pass


@dataclass
class Request:
    """One generation request (reference sim.py:96-113) plus its token stream."""

    id: int
    arrival_s: float
    prompt_len: int
    gen_len: int
    instance: int | None = None
    completion_s: float | None = None
    failed: bool = False
    requeued: bool = False
    generated: int = 0
    prefilled: bool = False
    prompt_tokens: np.ndarray | None = None  # int32 [prompt_len]; synthetic if None
    output_tokens: list = field(default_factory=list)
    slot: int | None = None  # KV slot held while in a batch

    @property
    def arrival_ms(self) -> int:
        return int(round(self.arrival_s * 1000))


def schedule(queue_depths: Sequence[tuple[int, int, float]], rng: np.random.Generator) -> int:
    """Instance for one request: minimum depth/speedup; exact ties are broken by
    a draw proportional to speedup over the tied instances in id order."""
    if not queue_depths:
        raise SimError("no instances registered")
    ranked = sorted(((depth / spd, iid, spd) for iid, depth, spd in queue_depths), key=lambda e: (e[0], e[1]))
    tied = [(iid, spd) for score, iid, spd in ranked if score == ranked[0][0]]
    if len(tied) == 1:
        return tied[0][0]
    x = rng.random() * sum(spd for _, spd in tied)
    acc = 0.0
    for iid, spd in tied:
        acc += spd
        if x < acc:
            return iid
    return tied[-1][0]


_EMPTY_I8 = np.empty(0, dtype=np.int64)
_EMPTY_F8 = np.empty(0, dtype=np.float64)


@dataclass(frozen=True)
class StepArrays:
    """Placement flattened for the executor (reference sim.py:204-213).

    ``layer_ptr``/CSR replica order is also what ``cb_get_placement`` reports
    back from the device, so registry and device plan can be compared."""

    layer_ptr: np.ndarray
    caps: np.ndarray
    run_min_p: np.ndarray
    run_bw: np.ndarray
    busy_devices: tuple[int, ...]
    kv_layer_count: dict[int, int]


def build_step_arrays(placement: PlacementState, cluster: ClusterSpec) -> StepArrays:
    ptr, caps = [0], []
    for li in range(1, placement.n_layers + 1):
        caps.extend(cluster.device(r.device_id).compute_gflops for r in placement.replicas_of(li))
        ptr.append(len(caps))
    run_p: list[int] = []
    run_bw: list[float] = []
    for dev in sorted({r.device_id for row in placement.replicas for r in row}):
        for run in _ops.replica_runs(placement, dev):
            run_p.append(min(len(placement.replicas_of(li)) for li in run))
            run_bw.append(cluster.bandwidth(placement.original_device(run[0]), dev))
    return StepArrays(
        layer_ptr=np.asarray(ptr, dtype=np.int64),
        caps=np.asarray(caps, dtype=np.float64) if caps else _EMPTY_F8,
        run_min_p=np.asarray(run_p, dtype=np.int64) if run_p else _EMPTY_I8,
        run_bw=np.asarray(run_bw, dtype=np.float64) if run_bw else _EMPTY_F8,
        busy_devices=tuple(sorted(placement.devices_used())),
        kv_layer_count=kv_resident_layer_count(placement),
    )


@dataclass(frozen=True)
class StepOutcome:
    """One batch pass: duration and KV growth per KV-resident layer (sim.py:261-266)."""

    duration_s: float
    kv_tokens_delta: int
    next_tokens: np.ndarray | None = None  # greedy token per request (B200 executor only)


def step_batch(arrays: StepArrays | None, d_model: int, batch: Sequence[Request], phase: str, calibration=None,
               delta=None, offload_fraction: float = 0.0, offload_multiplier: float = 2.0, *,
               executor) -> StepOutcome:
    """Executor hook (reference sim.py:269-300) running the pass on the B200s.

    The analytic arguments (calibration, delta, offload) are accepted for
    signature compatibility; the duration is measured, not modelled."""
    if not batch:
        return StepOutcome(0.0, 0)
    if phase not in ("prefill", "decode"):
        raise SimError(f"unknown phase {phase!r}")
    return executor.step_batch(batch, phase)
