"""One launch of each 7B projection at T prefill rows (for ncu: DRAM bytes vs
algorithmic bytes, tensor-pipe share).  python scripts/prefill_gemm_once.py [T]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, '.')
from paper_2507_18006_b200 import _lib

lib = _lib.load()
T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
EPI = {"qkv": 0, "o": 2, "gu": 3, "down": 2, "head": 1}
for name, N, K in [("qkv", 12288, 4096), ("o", 4096, 4096), ("gu", 22016, 4096), ("down", 4096, 11008),
                   ("head", 32000, 4096)]:
    w = (torch.randn(N, K, device='cuda') * 0.02).to(torch.bfloat16)
    x = torch.randn(T, K, device='cuda').to(torch.bfloat16)
    epi = EPI[name]
    ocols, odt = (N // 2, torch.bfloat16) if epi == 3 else (N, torch.float32 if epi in (1, 2) else torch.bfloat16)
    out = torch.zeros(T, ocols, device='cuda', dtype=odt)
    torch.cuda.synchronize()
    st = lib.cbt_gemm(C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), T, N, K, T, 0, epi,
                      C.c_void_p(out.data_ptr()), ocols)
    torch.cuda.synchronize()
    alg = N * K * 2 + T * K * 2 + T * ocols * out.element_size() * (2 if epi == 2 else 1)
    print(f"{name} N={N} K={K} T={T} status={st} algorithmic_bytes={alg} flops={2.0 * N * K * T:.4g}")
