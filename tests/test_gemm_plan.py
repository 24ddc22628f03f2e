"""GEMM plan choice (host-only, no GPU): the replica-invariance rule the row
router relies on (csrc/gemm.cu gemm_plan; ops.py:151-158 split_batch).

A replica's micro-batch (a split_batch share of the pass) must run the kernel
kind and work split the unreplicated pass would, so its rows come out bit for
bit identical: everything but the token-tile bucket depends on (N, K) and the
rows of the whole pass (kind_T), never on the micro-batch size."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_2507_18006_b200 import ops

SHAPES = [(12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008), (32000, 4096), (1536, 512), (384, 256)]
FIELDS = ["tn", "pair", "box_rows", "csplit", "max_parts", "whole", "kd", "nw", "ksplit"]


def _plan(lib, N, K, T, kind_T, sms=148):
    out = np.zeros(len(FIELDS), np.int32)
    assert lib.cbt_gemm_plan(N, K, T, sms, kind_T, out.ctypes.data_as(C.c_void_p)) == 0
    return dict(zip(FIELDS, out.tolist()))


@pytest.mark.parametrize("N,K", SHAPES)
@pytest.mark.parametrize("bs", [1, 7, 15, 64, 100, 128, 129, 200, 256])
def test_replica_share_runs_the_unreplicated_split(lib, N, K, bs):
    full = _plan(lib, N, K, bs, bs)
    for p in (2, 3, 4, 8):
        for share in ops.split_batch(bs, p):
            if share == 0:
                continue
            sub = _plan(lib, N, K, share, bs)
            for f in ("pair", "csplit", "max_parts", "whole", "kd", "nw", "ksplit"):
                assert sub[f] == full[f], (N, K, bs, p, share, f, sub, full)


@pytest.mark.parametrize("N,K", SHAPES)
def test_plan_fields_are_sane(lib, N, K):
    for T in (1, 16, 64, 128, 129, 256, 1024, 8192):
        pl = _plan(lib, N, K, T, T)
        assert pl["tn"] in (16, 32, 64, 128, 256)
        assert pl["csplit"] in (1, 2, 4, 8)
        if pl["pair"]:
            assert T > 128 and pl["box_rows"] == pl["tn"] // 2
            assert pl["nw"] == 0 or (128 <= pl["nw"] <= 256 and pl["nw"] % 32 == 0)
            if pl["ksplit"]:  # split-K token-major pairs: 64-column parts, one token tile
                assert pl["nw"] % (32 * pl["ksplit"]) == 0 and T <= 256 and (K // 64) % pl["ksplit"] == 0
        else:
            assert pl["box_rows"] == pl["tn"] and pl["tn"] >= min(T, 256) // 2
        if pl["csplit"] > 1:  # cluster split-K: every CTA of the cluster gets >= 1 k-block
            assert (K + 63) // 64 >= pl["csplit"]
