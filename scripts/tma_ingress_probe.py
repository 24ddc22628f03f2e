"""Per-SM L2 -> SM ingress: TMA box loads from an L2-resident region by
grids of 16..148 CTAs (one per SM).  Flat GB/s per CTA as the grid grows =
the SM's port is the limit; falling = the chip-wide L2 output is."""
import ctypes as C, sys
import torch
sys.path.insert(0, '.')
from paper_2507_18006_b200 import _lib
lib = _lib.load()
big = torch.empty(1 << 30, dtype=torch.uint8, device='cuda')
for region_mb in (16, 64):
    rows = region_mb * (1 << 20) // 128
    for grid in (16, 32, 64, 96, 128, 148):
        for (box, kd, stages, nw) in ((128, 2, 2, 2), (128, 1, 4, 2)):
            ms = C.c_float()
            iters = 2000
            st = lib.cbt_tma_probe(C.c_void_p(big.data_ptr()), rows, box, stages, grid, iters, kd, nw, 0, C.byref(ms))
            assert st == 0, st
            gbs = grid * nw * iters * box * 128 * kd / (ms.value * 1e-3) / 1e9
            print(f"L2 region {region_mb:3d} MB grid {grid:3d} box {box}x{kd}x128B stages {stages} warps {nw}: "
                  f"{gbs / 1e3:6.2f} TB/s total, {gbs / grid:6.1f} GB/s per SM", flush=True)
