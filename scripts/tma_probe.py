"""TMA fill-rate probe: chip-wide bytes/s of TMA box loads from L2-resident and
HBM-resident regions, by box size (rows x k-slices), ring depth, issuing warps
and CTA count.  Per iteration each CTA moves box_rows * 128 * kd bytes per warp."""
import ctypes as C, sys
import torch
sys.path.insert(0, '.')
from paper_2507_18006_b200 import _lib
lib = _lib.load()
big = torch.empty(8 << 30, dtype=torch.uint8, device='cuda')  # 8 GiB (HBM)
cases = []
for region_mb in ([int(a) for a in sys.argv[1].split(',')] if len(sys.argv) > 1 else (32, 1024)):
    for (box, kd, stages, nw, grid) in [(128, 1, 8, 1, 148), (256, 1, 4, 1, 148), (128, 1, 4, 2, 148),
                                        (128, 2, 4, 1, 148), (128, 1, 2, 4, 148),
                                        (256, 1, 2, 2, 148), (256, 1, 1, 4, 148)]:
        rows = region_mb * (1 << 20) // 128
        iters = 3000 if region_mb <= 64 else 400
        iters = max(200, iters // kd)
        ms = C.c_float()
        st = lib.cbt_tma_probe(C.c_void_p(big.data_ptr()), rows, box, stages, grid, iters, kd, nw, 0, C.byref(ms))
        assert st == 0, (st, box, kd, stages, nw)
        tb = grid * nw * iters * box * 128 * kd / (ms.value * 1e-3) / 1e12
        print(f"region {region_mb:5d}MB box {box:3d}x{kd}x128B ({box*kd*128//1024:3d}KB) stages {stages:2d} warps {nw} "
              f"grid {grid}: {tb:6.2f} TB/s ({tb * 1e12 / 1.965e9 / 148:5.1f} B/clk/SM)", flush=True)
