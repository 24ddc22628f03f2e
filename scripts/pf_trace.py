"""Timeline of one prefill-attention CTA (the last query block of head 0: the
most key blocks): builds a separate copy of the library with -DPF_TRACE
(build/pftrace/), runs one launch (1 prompt of L tokens, 32 heads, hd 128)
and prints per key block when K / V loads were issued, S and PV issued,
and the softmax warp's phases, in SM clock cycles from the CTA's start.

    python scripts/pf_trace.py [L]"""
import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2507_18006_b200 import _build  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
out = ROOT / "build" / "pftrace"
out.mkdir(parents=True, exist_ok=True)
objs = []
for src in _build._sources():
    obj = out / (src.stem + ".o")
    extra = (["-DPF_TRACE"] + os.environ.get("PF_FLAGS", "").split()) if src.stem == "prefill_attention" else []
    subprocess.run([_build._nvcc(), *_build.ARCH, *_build.FLAGS, *extra, "-c", str(src), "-o", str(obj)], check=True)
    objs.append(str(obj))
lib_path = out / "libcocob200_pftrace.so"
subprocess.run([_build._nvcc(), *_build.ARCH, "-shared", "-o", str(lib_path), *objs], check=True)
lib = C.CDLL(str(lib_path))
H, Hkv, hd = 32, 32, 128
qkv = (torch.randn(L, (H + 2 * Hkv) * hd, device="cuda")).to(torch.bfloat16)
kv = (torch.randn(1, L + 8, 2, Hkv * hd, device="cuda")).to(torch.bfloat16)
out_t = torch.zeros(L, H * hd, dtype=torch.bfloat16, device="cuda")
blocks = torch.tensor([(b0, min(256, L - b0), 0, b0) for b0 in range(0, L, 256)], dtype=torch.int32, device="cuda")
tr = torch.zeros(12 * 32, dtype=torch.int64, device="cuda")
P = C.c_void_p
lib.cbt_prefill_attention.argtypes = [P, P, P, P] + [C.c_int32] * 7
for _ in range(3):
    assert lib.cbt_prefill_attention(qkv.data_ptr(), kv.data_ptr(), out_t.data_ptr(), blocks.data_ptr(),
                                     blocks.shape[0], L, H, Hkv, hd, L + 8, 1) == 0
lib.cbt_pf_trace_set.argtypes = [P]
assert lib.cbt_pf_trace_set(tr.data_ptr()) == 0
assert lib.cbt_prefill_attention(qkv.data_ptr(), kv.data_ptr(), out_t.data_ptr(), blocks.data_ptr(),
                                 blocks.shape[0], L, H, Hkv, hd, L + 8, 1) == 0
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(12, 32).astype(np.float64)
t0 = t[9, 0]
rel = np.where(t > 0, (t - t0), np.nan)  # SM clock cycles (clock64: one SM, one counter)
names = ["-", "-", "S_A issued", "S_B issued", "PV_A issued", "PV_B issued", "S_A ready@smx", "A exp done",
         "P_A arrive", "-", "S_B ready@smx", "P_B arrive"]
nkb = (L - 1) // 64 + 1
print(f"L={L}: CTA of the last 256-row query block (tiles A, B), {nkb} key blocks of 64; SM cycles from the CTA start; "
      f"end at {rel[9, 1]:.0f}")
print("j   " + " ".join(f"{n:>12s}" for n in names if n != "-"))
for j in range(min(nkb, 32)):
    print(f"{j:2d}  " + " ".join(f"{rel[k, j]:12.0f}" for k in range(12) if names[k] != "-"))
