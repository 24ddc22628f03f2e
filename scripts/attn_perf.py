"""Decode attention sweep: achieved HBM GB/s (K/V bytes read once) per shape."""
import ctypes as C, sys, time
import torch
sys.path.insert(0, '.')
from paper_2507_18006_b200 import _lib
lib = _lib.load()
P = lambda t: C.c_void_p(t.data_ptr())
SHAPES = [(64, 32, 32, 150), (64, 32, 32, 512), (128, 32, 32, 256), (256, 32, 32, 300),
          (16, 32, 32, 2048), (1, 32, 32, 4096), (64, 64, 8, 512)]
if len(sys.argv) > 1:  # T:ctx,T:ctx,... (MHA 32 heads)
    SHAPES = [(int(a), 32, 32, int(b)) for a, b in (x.split(':') for x in sys.argv[1].split(','))]
for (T, H, Hkv, ctx) in SHAPES:
    hd = 128
    qkv = torch.randn(T, (H + 2 * Hkv) * hd, device='cuda').to(torch.bfloat16)
    kv = torch.randn(T, ctx + 2, 2, Hkv * hd, device='cuda').to(torch.bfloat16)
    out = torch.empty(T, H * hd, device='cuda', dtype=torch.bfloat16)
    slot = torch.arange(T, dtype=torch.int32, device='cuda')
    pos = torch.full((T,), ctx - 1, dtype=torch.int32, device='cuda')
    msv = C.c_float()
    assert lib.cbt_attention_bench(P(qkv), P(kv), P(out), P(slot), P(pos), T, H, Hkv, hd, ctx + 2, ctx, 20,
                                   C.byref(msv)) == 0
    ms = msv.value
    by = T * ctx * 2 * Hkv * hd * 2
    print(f"T={T:4d} H={H} Hkv={Hkv} ctx={ctx:5d}: {ms*1000:7.1f} us  {by/ms/1e6:6.0f} GB/s", flush=True)
