"""Per-CTA timeline of the token-major split-K pair GEMM (O / down at T > 128):
k-block landing times, then the L2 part exchange: tfull (own K part done),
parts stored (bulk stores of the other column parts done), parts arrived (counter wait over, loads issued), drained, end.
    python scripts/gemm_split_trace.py N K T [epi]"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2507_18006_b200 import _lib

lib = _lib.load()
N, K, T = (int(v) for v in sys.argv[1:4])
EPI = int(sys.argv[4]) if len(sys.argv) > 4 else 2
MODE = int(sys.argv[6]) if len(sys.argv) > 6 else 0
NCOP = max(1, -(-512 * 2**20 // (N * K * 2)))
wall = torch.randn(NCOP, N, K, device='cuda').to(torch.bfloat16)
w = wall[0]
lib.cbt_gemm_set_wcopies(NCOP, N * K * 2)
x = torch.randn(T, K, device='cuda').to(torch.bfloat16)
out = torch.zeros(T, N, device='cuda', dtype=torch.float32 if EPI in (1, 2) else torch.bfloat16)
ms = C.c_float()
assert lib.cbt_gemm_bench(C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), T, N, K, T, EPI,
                          C.c_void_p(out.data_ptr()), N, 20, MODE + 8000 if MODE >= 0 else MODE - 8000, C.byref(ms)) == 0
tr = np.zeros(148 * 512, dtype=np.uint64)
lib.cbt_gemm_trace(tr.ctypes.data_as(C.c_void_p), tr.size)
tr = (tr.reshape(148, 512) & np.uint64((1 << 62) - 1)).astype(np.int64)
valid = tr[:, 0] > 0
t0 = tr[valid, 0].min()
rel = np.where(tr > 0, (tr - t0) / 1000.0, np.nan)
print(f"N={N} K={K} T={T}: {ms.value * 1000:.1f} us/launch (untraced); {valid.sum()} CTAs traced")
rows = []
for c in np.nonzero(valid)[0]:
    mma = rel[c, 2:66]
    mma = mma[~np.isnan(mma)]
    ev = rel[c, 130:134]
    rows.append((rel[c, 0], mma[0] if len(mma) else np.nan, mma[-1] if len(mma) else np.nan, len(mma), *ev, rel[c, 1]))
a = np.array(rows)
names = ["start", "kb0 landed", "kb63 landed", "n kb traced", "tfull", "parts stored", "parts arrived", "drained", "end"]
for i, nme in enumerate(names):
    col = a[:, i]
    print(f"  {nme:12s} min {np.nanmin(col):7.2f}  median {np.nanmedian(col):7.2f}  max {np.nanmax(col):7.2f}")
nk = a[:, 3]
print(f"  ns per k-block (first {int(np.median(nk))} traced): {np.nanmedian((a[:, 2] - a[:, 1]) / np.maximum(1, nk - 1)) * 1000:.0f}")
# per k-block pipeline latencies (slots: 66+i W issue, 150+i X issue, 214+i W landed at the MMA
# warp, 2+i both landed, 278+i MMAs issued), CTAs that traced >= 16 k-blocks
S = int(sys.argv[5]) if len(sys.argv) > 5 else 8
st = {"W issue->W landed": [], "X issue->both landed": [], "W landed->both landed": [],
      "both landed->MMA issued": [], "MMA issued->next both landed": [], "X issue - W issue": []}
for c in np.nonzero(valid)[0]:
    wi, xi, wl, bl, mi = (rel[c, o:o + 64] for o in (66, 150, 214, 2, 278))
    n = int(np.sum(~np.isnan(bl)))
    if n < 16:
        continue
    for i in range(2, n - 1):
        st["W issue->W landed"].append(wl[i] - wi[i])
        st["X issue->both landed"].append(bl[i] - xi[i])
        st["W landed->both landed"].append(bl[i] - wl[i])
        st["both landed->MMA issued"].append(mi[i] - bl[i])
        st["MMA issued->next both landed"].append(bl[i + 1] - mi[i])
        st["X issue - W issue"].append(xi[i] - wi[i])
for k, v in st.items():
    v = np.array(v)
    v = v[~np.isnan(v)]
    if len(v):
        print(f"  {k:30s} median {np.median(v) * 1000:6.0f} ns  p10 {np.percentile(v, 10) * 1000:6.0f}  p90 {np.percentile(v, 90) * 1000:6.0f}")
