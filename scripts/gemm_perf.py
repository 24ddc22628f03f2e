"""Decode/prefill GEMM sweep on the 7B projection shapes (warm, CUDA-event timed)."""
import ctypes as C, sys, json
import torch
sys.path.insert(0, '.')
from paper_2507_18006_b200 import _lib
lib = _lib.load()
parts = [int(x) for x in (sys.argv[1].split(',') if len(sys.argv) > 1 else ['2'])]
Ts = [int(x) for x in (sys.argv[2].split(',') if len(sys.argv) > 2 else ['1', '16', '64', '128', '256', '2048', '8192'])]
for (name, N, K) in [("qkv", 12288, 4096), ("o", 4096, 4096), ("gu", 22016, 4096), ("down", 4096, 11008), ("head", 32000, 4096)]:
    w = torch.randn(N, K, device='cuda').to(torch.bfloat16)
    for T in Ts:
        x = torch.randn(T, K, device='cuda').to(torch.bfloat16)
        out = torch.empty(T, N, device='cuda', dtype=torch.bfloat16)
        res = []
        for mp in parts:
            ms = C.c_float()
            st = lib.cbt_gemm_bench(C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), T, N, K, T, 0,
                                    C.c_void_p(out.data_ptr()), N, 20, mp, C.byref(ms))
            assert st == 0
            gbs = (N * K * 2 + T * K * 2 + T * N * 2) / ms.value / 1e6
            res.append(f"mp{mp}: {ms.value*1000:6.1f}us {gbs:5.0f}GB/s {2*N*K*T/ms.value/1e9:6.1f}TF/s")
        print(f"{name:5s} T={T:5d} " + " | ".join(res), flush=True)
