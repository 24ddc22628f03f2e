"""Per-CTA timeline of one GEMM launch (experiments, 1-CTA kernel):
slot 0 start, 1 epilogue end, 2.. MMA-warp time each k-block's operands landed,
66.. W-producer time each stage was free again, 130 + 5*seg: epilogue segment
events (tfull landed | TMEM drained | fixup decision | fixup done).
    python scripts/gemm_trace.py N K T mode"""
import ctypes as C, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2507_18006_b200 import _lib
lib = _lib.load()
N, K, T, mode = (int(v) for v in sys.argv[1:5])
EPI = int(sys.argv[6]) if len(sys.argv) > 6 else 0
NCOP = max(1, -(-512 * 2**20 // (N * K * 2)))  # >= 512 MB of weight copies: never L2-resident
wall = torch.randn(NCOP, N, K, device='cuda').to(torch.bfloat16)
w = wall[0]
lib.cbt_gemm_set_wcopies(NCOP, N * K * 2)
x = torch.randn(T, K, device='cuda').to(torch.bfloat16)
OC = N // 2 if EPI == 3 else N
out = torch.zeros(T, OC, device='cuda', dtype=torch.float32 if EPI in (1, 2) else torch.bfloat16)
ms = C.c_float()
assert lib.cbt_gemm_bench(C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), T, N, K, T, EPI,
                          C.c_void_p(out.data_ptr()), OC, 20, mode + 8000 if mode >= 0 else mode - 8000, C.byref(ms)) == 0
tr = np.zeros(148 * 512, dtype=np.uint64)
lib.cbt_gemm_trace(tr.ctypes.data_as(C.c_void_p), tr.size)
tr = tr.reshape(148, 512)
flags = tr >> np.uint64(62)
tr = (tr & np.uint64((1 << 62) - 1)).astype(np.int64)
valid = tr[:, 0] > 0
t0 = tr[valid, 0].min()
rel = np.where(tr > 0, (tr - t0) / 1000.0, np.nan)
print(f"N={N} K={K} T={T} mode={mode}: {ms.value*1000:.1f} us/launch (untraced)")
print(f"CTA end us: min {np.nanmin(rel[:, 1]):.2f} median {np.nanmedian(rel[:, 1]):.2f} max {np.nanmax(rel[:, 1]):.2f}")
for c in (0, 1, 2, 75, 147):
    if not valid[c]:
        continue
    mma = rel[c, 2:66]
    mma = mma[~np.isnan(mma)]
    free = rel[c, 66:130]
    nk = len(mma)
    print(f"CTA {c:3d}: start {rel[c,0]:.2f}  kb landed first {mma[0]:.2f} last {mma[-1]:.2f} ({nk} kb, "
          f"{(mma[-1]-mma[0])/max(1,nk-1)*1000:.0f} ns/kb)  end {rel[c,1]:.2f}")
    # stage round trip: unit i landed at the MMA warp -> its stage free again
    # (the W producer passed the empty wait for unit i + S)
    S = int(sys.argv[5]) if len(sys.argv) > 5 else 8
    lt = [free[i + S] - mma[i] for i in range(0, min(nk, 64) - S) if not np.isnan(free[i + S])]
    land = [mma[i + S] - free[i + S] for i in range(0, min(nk, 64) - S) if not np.isnan(free[i + S])]
    xiss = rel[c, 150:214]
    wl = rel[c, 214:278]
    wlat = [wl[i + S] - free[i + S] for i in range(0, min(nk, 64) - S)]
    xlat = [mma[i + S] - xiss[i + S] for i in range(0, min(nk, 64) - S)]
    xlag = [xiss[i + S] - free[i + S] for i in range(0, min(nk, 64) - S)]
    print(f"     W issue -> W landed median {np.nanmedian(wlat)*1000:.0f} ns; X issue -> both landed "
          f"{np.nanmedian(xlat)*1000:.0f} ns; X issue - W issue {np.nanmedian(xlag)*1000:.0f} ns")
    iss = rel[c, 278:342]
    print(f"     per kb: W-landed->both-landed {np.nanmedian(mma[:nk]-wl[:nk])*1000:.0f} ns, both-landed->issued "
          f"{np.nanmedian(iss[:nk]-mma[:nk])*1000:.0f} ns, issued->next W-landed {np.nanmedian(wl[1:nk]-iss[:nk-1])*1000:.0f} ns")
    print(f"     S={S}: landed -> stage free median {np.median(lt)*1000:.0f} ns; "
          f"load issued -> landed median {np.median(land)*1000:.0f} ns")
    if not np.isnan(rel[c, 140]):
        print(f"     cluster split-K: reduce start {rel[c,140]:.2f} reduce+emit done {rel[c,141]:.2f}; chunks (loaded, emitted):",
              " ".join(f"({rel[c,142+2*k]:.2f},{rel[c,143+2*k]:.2f})" for k in range(4)))
    for sg in range(4):
        ev = rel[c, 130 + 4 * sg: 134 + 4 * sg]
        if np.isnan(ev[0]):
            continue
        fl = flags[c, 130 + 4 * sg]
        dec = flags[c, 132 + 4 * sg]
        print(f"     seg {sg}: {'whole' if fl & 1 else 'part '} tfull {ev[0]:.2f} drained {ev[1]:.2f} "
              f"decision {ev[2]:.2f}{' FINISHER' if dec & 2 else ''}{' ring-idle' if dec & 1 else ''} done {ev[3]:.2f}")
        fx = rel[c, 130 + 4 * sg + 220: 130 + 4 * sg + 226]
        if not np.all(np.isnan(fx)):
            print("       fixup rounds (copy landed, summed):", " ".join(f"{v:.2f}" for v in fx if not np.isnan(v)))
