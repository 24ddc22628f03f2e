"""Decode/prefill GEMM sweep on the 7B projection shapes (warm, CUDA-event timed).

    python scripts/gemm_perf.py [modes] [Ts]
modes: comma list of cbt_gemm_bench knobs: 0 = the plan gemm_plan picks,
201 = CTA-pair 256-token tiles, 202 = CTA-pair 128-token tiles, 203 = 1-CTA."""
import ctypes as C, sys, json
import torch
sys.path.insert(0, '.')
from paper_2507_18006_b200 import _lib
lib = _lib.load()
parts = [int(x) for x in (sys.argv[1].split(',') if len(sys.argv) > 1 else ['0'])]
Ts = [int(x) for x in (sys.argv[2].split(',') if len(sys.argv) > 2 else ['1', '16', '64', '128', '256', '2048', '8192'])]
rows = []
REAL_EPI = "--real-epi" in sys.argv
if REAL_EPI:
    sys.argv.remove("--real-epi")
NORM = "--norm" in sys.argv  # fused RMSNorm epilogues (consumer: qkv / gu / head, producer: o / down)
if NORM:
    sys.argv.remove("--norm")
# the decode step's epilogues: qkv bf16, o / down += fp32 residual, gate/up SwiGLU, lm_head fp32 logits
EPI = {"qkv": 0, "o": 2, "gu": 3, "down": 2, "head": 1}
for (name, N, K) in [("qkv", 12288, 4096), ("o", 4096, 4096), ("gu", 22016, 4096), ("down", 4096, 11008), ("head", 32000, 4096)]:
    NCOP = max(1, -(-512 * 2**20 // (N * K * 2)))  # >= 512 MB of weight copies: never L2-resident
    wall = torch.randn(NCOP, N, K, device='cuda').to(torch.bfloat16)
    w = wall[0]
    lib.cbt_gemm_set_wcopies(NCOP, N * K * 2)
    # tile-major copy [N/128][K/64][128][64] for modes with the 4000 bit (w_tiled)
    wt = wall.view(NCOP, N // 128, 128, K // 64, 64).permute(0, 1, 3, 2, 4).contiguous()[0]
    for T in Ts:
        x = torch.randn(T, K, device='cuda').to(torch.bfloat16)
        epi = EPI[name] if REAL_EPI else 0
        ocols, odt = (N // 2, torch.bfloat16) if epi == 3 else (N, torch.float32 if epi in (1, 2) else torch.bfloat16)
        out = torch.zeros(T, ocols, device='cuda', dtype=odt)
        if NORM:
            if epi == 2:
                hbuf = torch.zeros(T, N, device='cuda', dtype=torch.bfloat16)
                gam = torch.ones(N, device='cuda', dtype=torch.bfloat16)
                sso = torch.zeros(T, N // 32, device='cuda')
                lib.cbt_gemm_set_norm(None, hbuf.data_ptr(), gam.data_ptr(), sso.data_ptr(), N // 32, N, C.c_float(1e-5))
            else:
                ssi = torch.ones(T, K // 32, device='cuda')
                lib.cbt_gemm_set_norm(ssi.data_ptr(), None, None, None, K // 32, K, C.c_float(1e-5))
        res = []
        for mp in parts:
            ms = C.c_float()
            wp = wt if (mp // 1000) & 4 else w
            st = lib.cbt_gemm_bench(C.c_void_p(wp.data_ptr()), C.c_void_p(x.data_ptr()), T, N, K, T, epi,
                                    C.c_void_p(out.data_ptr()), ocols, 20, mp, C.byref(ms))
            assert st == 0
            gbs = (N * K * 2 + T * K * 2 + T * N * 2) / ms.value / 1e6
            tf = 2 * N * K * T / ms.value / 1e9
            res.append(f"m{mp}: {ms.value*1000:6.1f}us {gbs:5.0f}GB/s {tf:6.1f}TF/s")
            rows.append({"shape": name, "N": N, "K": K, "T": T, "mode": mp, "us": ms.value * 1000, "gbs": gbs, "tflops": tf})
        lib.cbt_gemm_set_norm(None, None, None, None, 0, 0, C.c_float(0))
        print(f"{name:5s} T={T:5d} " + " | ".join(res), flush=True)
if len(sys.argv) > 3:
    json.dump(rows, open(sys.argv[3], "w"), indent=1)
