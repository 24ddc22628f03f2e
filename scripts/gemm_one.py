"""Run one GEMM shape a few times (for `ncu -k regex:gemm -c 1 python scripts/gemm_one.py N K T`)."""
import ctypes as C, sys
import torch
sys.path.insert(0, '.')
from paper_2507_18006_b200 import _lib
lib = _lib.load()
N, K, T = (int(v) for v in sys.argv[1:4])
mp = int(sys.argv[4]) if len(sys.argv) > 4 else 0
w = torch.randn(N, K, device='cuda').to(torch.bfloat16)
x = torch.randn(T, K, device='cuda').to(torch.bfloat16)
out = torch.empty(T, N, device='cuda', dtype=torch.bfloat16)
ms = C.c_float()
assert lib.cbt_gemm_bench(C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), T, N, K, T, 0,
                          C.c_void_p(out.data_ptr()), N, 3, mp, C.byref(ms)) == 0
print(N, K, T, f"{ms.value*1000:.1f} us")
