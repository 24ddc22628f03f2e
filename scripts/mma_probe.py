"""tcgen05.mma (kind::f16, 128 x N x 16, both operands in smem) cycles per instruction."""
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_2507_18006_b200 import _lib
lib = _lib.load()
import torch  # noqa: F401  (context)
for N in (16, 64, 128, 256):
    for grid in (1, 148):
        for kstep in (0, 1):
            v = C.c_double()
            assert lib.cbt_mma_probe(N, 4096, grid, kstep, C.byref(v)) == 0
            print(f"N={N:3d} grid={grid:3d} kstep={kstep}: {v.value:7.1f} clk/MMA  (formula {128*N/256:.0f})", flush=True)
