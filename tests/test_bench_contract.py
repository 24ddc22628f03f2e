"""bench.py's JSON contract pieces that run without a GPU: both arms report the
same workload config, and the roofline object reports the dominant kernel
class of the step (largest profiled share), picks the binding roof per launch
(bytes / HBM peak vs FLOPs / sustained tensor peak) and attributes the timed
step by the profiled class shares."""
from __future__ import annotations

import argparse

import pytest

import bench


def _args(**kw):
    base = dict(batch=256, prompt=128, gen=256, steps=20, warmup=5)
    base.update(kw)
    return argparse.Namespace(**base)


def test_both_arms_report_the_same_config():
    a = _args()
    ours = bench.headline_config(a, 1)
    assert ours["batch"] == 256 and ours["prompt_len"] == 128 and ours["gen_len"] == 256
    assert ours["ctx_at_mid_step"] == 128 + 256 // 2  # the reference arm's CPU context
    assert bench.headline_config(a, 1) == ours


PEAKS = {"hbm_gbs": 6500.0, "bf16_tflops": 1650.0, "bf16_tflops_sustained": 1400.0, "src": "test"}


def _prof(gemm_bytes, gemm_flops, gemm_ms, launches=129, steps=2, attn_ms=None):
    return {"gemm": {"launches": launches * steps, "ms": gemm_ms, "bytes": gemm_bytes, "flops": gemm_flops},
            "attention": {"launches": 32 * steps, "ms": gemm_ms * 0.9 if attn_ms is None else attn_ms,
                          "bytes": 1e9, "flops": 0.0},
            "elementwise": {"launches": 2 * steps, "ms": 0.01, "bytes": 1e6, "flops": 0.0},
            "copy": {"launches": 0, "ms": 0.0, "bytes": 0.0, "flops": 0.0}}


def test_roofline_tensor_bound_at_high_intensity():
    # 232 FLOP per byte (B = 256 decode): above the ridge 1400e12 / 6500e9 = 215
    prof = _prof(gemm_bytes=1e9, gemm_flops=232e9, gemm_ms=0.5)
    r = bench.step_roofline(prof, [1.0, 1.0], PEAKS, None, step_ms=0.8)
    assert r["class"] == "gemm" and r["bound"] == "tensor" and r["unit"] == "TFLOP/s"
    assert r["achieved"] == pytest.approx(232e9 / (0.5 * 1e9))
    assert r["frac"] == pytest.approx(r["achieved"] / 1400.0)
    # in-step attribution: 0.8 ms/step x (0.5 / 2.0 share) over 129 launches per step
    ms_l = 0.8 * (0.5 / 2.0) / 129
    assert r["in_step"]["ms_per_launch"] == pytest.approx(ms_l)
    assert r["in_step"]["frac"] == pytest.approx((232e9 / 258) / (ms_l * 1e9) / 1400.0)


def test_roofline_hbm_bound_at_low_intensity():
    prof = _prof(gemm_bytes=1e9, gemm_flops=2e9, gemm_ms=0.2)  # batch 1: 2 FLOP per byte
    r = bench.step_roofline(prof, [0.5, 0.5], PEAKS)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert r["achieved"] == pytest.approx(1e9 / (0.2 * 1e6))
    assert r["in_step"] is None  # no timed step given


def test_roofline_reports_the_dominant_class():
    """At long contexts the KV read dominates the step: the top-level roofline
    is the attention's (HBM-bound), the GEMMs stay under ``classes``."""
    prof = _prof(gemm_bytes=1e9, gemm_flops=232e9, gemm_ms=0.5, attn_ms=0.7)
    ncu = {"gemm_dram_bytes_per_launch": 1.1e8, "attention_dram_bytes_per_launch": 1.09e9,
           "attention_algorithmic_bytes_per_launch": 1.078e9}
    r = bench.step_roofline(prof, [1.2, 1.2], PEAKS, ncu, step_ms=1.0)
    assert r["class"] == "attention" and r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert r["achieved"] == pytest.approx(1e9 / (0.7 * 1e6))
    assert r["traffic"] == 1.09e9 and r["traffic_capture_algorithmic_bytes"] == 1.078e9
    assert r["classes"]["gemm"]["bound"] == "tensor" and r["classes"]["gemm"]["traffic"] == 1.1e8
    assert r["in_step"] is None and r["classes"]["gemm"]["in_step"]["frac"] > 0
    assert r["step_share"]["attention"] > r["step_share"]["gemm"]
