"""TMA HBM streaming with a concurrent MMA warp (smem contention probe)."""
import ctypes as C, sys
import torch
sys.path.insert(0, '.')
from paper_2507_18006_b200 import _lib
lib = _lib.load()
big = torch.empty(8 << 30, dtype=torch.uint8, device='cuda')
rows = (8 << 30) // 128
for (box, stages) in ((128, 8), (128, 4)):
    for mma_n in (0, 16, 64, 256):
        for grid in (96, 148):
            iters = 400
            ms = C.c_float()
            st = lib.cbt_tma_probe(C.c_void_p(big.data_ptr()), rows, box, stages, grid, iters, 1, 1, mma_n, C.byref(ms))
            assert st == 0, st
            tb = grid * iters * box * 128 / (ms.value * 1e-3) / 1e12
            print(f"HBM box {box}x128B stages {stages} grid {grid} concurrent MMA N={mma_n:3d}: {tb:5.2f} TB/s "
                  f"({tb*1e12/grid/1e9:5.1f} GB/s per CTA)", flush=True)
