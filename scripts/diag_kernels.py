"""Per-kernel agreement with the bf16-faithful oracle's rounding (ulp counts)."""
import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, '.')
from oracle.cpu_llama import bf16_round, rmsnorm, rope_table, apply_rope, attention_rows, silu, to_bf16_bits, from_bf16_bits
from paper_2507_18006_b200 import _lib
lib = _lib.load()
P = lambda t: C.c_void_p(t.data_ptr())
def tb(a): return torch.from_numpy(to_bf16_bits(a).view(np.int16)).view(torch.bfloat16).cuda()
def nb(t): return from_bf16_bits(t.cpu().view(torch.int16).numpy().view(np.uint16))
def ulps(a, b):
    ua = a.astype(np.float32).view(np.int32); ub = b.astype(np.float32).view(np.int32)
    d = np.abs((ua >> 16).astype(np.int64) - (ub >> 16).astype(np.int64))
    return (d > 0).mean(), d.max()
rng = np.random.default_rng(0)
T, d = 15, 256
x = rng.standard_normal((T, d)).astype(np.float32) * 2
g = from_bf16_bits(to_bf16_bits(1 + 0.1 * rng.standard_normal(d).astype(np.float32)))
xt = torch.from_numpy(x).cuda(); y = torch.empty(T, d, dtype=torch.bfloat16, device='cuda')
lib.cbt_rmsnorm(P(xt), P(tb(g)), P(y), T, d, C.c_float(1e-5))
print("rmsnorm frac!=, maxulp", ulps(nb(y), bf16_round(rmsnorm(x, g, 1e-5))))
h = bf16_round(rmsnorm(x, g, 1e-5))
W = from_bf16_bits(to_bf16_bits(rng.standard_normal((768, d)).astype(np.float32) / 16))
out = torch.zeros(T, 768, dtype=torch.bfloat16, device='cuda')
lib.cbt_gemm(P(tb(W)), P(tb(h)), T, 768, d, T, 0, 0, P(out), 768)
print("gemm bf16 frac!=, maxulp", ulps(nb(out), bf16_round(h @ W.T)))
out32 = torch.zeros(T, 768, dtype=torch.float32, device='cuda')
lib.cbt_gemm(P(tb(W)), P(tb(h)), T, 768, d, T, 0, 1, P(out32), 768)
ref = (h.astype(np.float64) @ W.T.astype(np.float64))
print("gemm f32 max rel err", np.abs(out32.cpu().numpy() - ref).max() / np.abs(ref).max(), "numpy f32 err", np.abs(h @ W.T - ref).max() / np.abs(ref).max())
# swiglu
Wg = W[:384]; Wu = W[384:]
Wi = np.stack([Wg, Wu], 1).reshape(768, d)
act = torch.zeros(T, 384, dtype=torch.bfloat16, device='cuda')
lib.cbt_gemm(P(tb(Wi)), P(tb(h)), T, 768, d, T, 0, 3, P(act), 384)
print("swiglu frac!=, maxulp", ulps(nb(act), bf16_round(silu(h @ Wg.T) * (h @ Wu.T))))
# rope
H, hd = 4, 64
qkv = bf16_round(rng.standard_normal((T, 3 * H * hd)).astype(np.float32))
qt = tb(qkv); kv = torch.zeros(16, 64, 2, H * hd, dtype=torch.bfloat16, device='cuda')
pos = np.arange(T).astype(np.int32); slot = np.zeros(T, np.int32)
lib.cbt_rope_kv(P(qt), P(kv), P(torch.from_numpy(slot).cuda()), P(torch.from_numpy(pos).cuda()), T, H, H, hd, 64, C.c_float(1e4))
cos, sin = rope_table(64, hd, 1e4)
qr = bf16_round(apply_rope(qkv[:, :H*hd].reshape(T, H, hd), pos, cos, sin)).reshape(T, -1)
kr = bf16_round(apply_rope(qkv[:, H*hd:2*H*hd].reshape(T, H, hd), pos, cos, sin)).reshape(T, -1)
print("rope q frac!=, maxulp", ulps(nb(qt)[:, :H*hd], qr))
print("rope k frac!=, maxulp", ulps(nb(kv[0, :T, 0]), kr))
# attention (prefill causal) on the roped values
att = torch.zeros(T, H * hd, dtype=torch.bfloat16, device='cuda')
lib.cbt_attention(P(qt), P(kv), P(att), P(torch.from_numpy(slot).cuda()), P(torch.from_numpy(pos).cuda()), T, H, H, hd, 64)
kc = nb(kv[0, :, 0]).reshape(64, H, hd); vc = nb(kv[0, :, 1]).reshape(64, H, hd)
ref = attention_rows(qr.reshape(T, H, hd), np.stack([kc] * T), np.stack([vc] * T), pos + 1).reshape(T, -1)
print("attn frac!=, maxulp", ulps(nb(att), bf16_round(ref)), "max abs", np.abs(nb(att) - ref).max())

# ---- whole-model ablations: 1 layer, zeroed parts
from oracle.cpu_llama import TINY, OracleModel, init_weights, LlamaConfig
from oracle.gen_golden import config1_prompts
from paper_2507_18006_b200.executor import Executor, ExecutorConfig, Runtime
import dataclasses
rt = Runtime([0])
prompts = config1_prompts()
for nl in (1, 2, 4):
    cfg = dataclasses.replace(TINY, n_layers=nl)
    for abl in ("none", "no_attn", "no_ffn"):
        w = init_weights(cfg, 3)
        for L in w.layers:
            if abl == "no_attn": L.wo[:] = 0
            if abl == "no_ffn": L.w_down[:] = 0
        ex = Executor(rt, ExecutorConfig(nl, 256, 768, 4, vocab=1024, max_slots=16, max_ctx=64, max_tokens=512))
        ex.load_model(w, 0)
        slots = np.arange(15, dtype=np.int32)
        _, lg, _ = ex.prefill(slots, np.concatenate(prompts), np.full(15, 16, np.int32), True)
        fa = OracleModel(cfg, w, 64, bf16_acts=True).forward(list(range(15)), np.concatenate(prompts), [16] * 15)
        fp = OracleModel(cfg, w, 64).forward(list(range(15)), np.concatenate(prompts), [16] * 15)
        print(f"layers={nl} {abl:8s} gpu-faithful {np.abs(lg-fa).max():.2e} gpu-fp32 {np.abs(lg-fp).max():.2e} faithful-fp32 {np.abs(fa-fp).max():.2e}")
        ex.close()
