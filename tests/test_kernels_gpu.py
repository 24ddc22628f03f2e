"""Kernel-level parity on the B200: each CUDA kernel vs an fp32/fp64 reference.

Floating-point kernels (GEMM epilogues, RMSNorm, RoPE, attention) are checked
against CPU float64/fp32 math on the same bf16 inputs, with the tolerance in
each test; integer results (argmax) are exact.  Determinism and the
row-split invariance the replica router relies on are checked bit-exactly.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _bf16(torch, shape, scale=1.0, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.randn(*shape, generator=g) * scale).to(torch.bfloat16)


def _gemm(lib, torch, w, x, T, row_off, epi, out, ldo):
    st = lib.cbt_gemm(_ptr(w), _ptr(x), x.shape[0], w.shape[0], w.shape[1], T, row_off, epi, _ptr(out), ldo)
    assert st == 0, st
    torch.cuda.synchronize()


@pytest.mark.parametrize("N,K,T", [(384, 256, 1), (384, 256, 5), (256, 512, 16), (384, 256, 17), (512, 256, 64),
                                   (256, 256, 100), (384, 320, 256), (256, 256, 300), (128, 128, 600),
                                   (200, 256, 33)])
def test_gemm_bf16_out(lib, cuda, N, K, T):
    torch = cuda
    w = _bf16(torch, (N, K), 0.05, 1).cuda()
    x = _bf16(torch, (T + 8, K), 1.0, 2).cuda()
    out = torch.zeros(T + 8, N, dtype=torch.bfloat16, device="cuda")
    _gemm(lib, torch, w, x, T, 0, 0, out, N)
    ref = x[:T].double().cpu() @ w.double().cpu().T
    got = out[:T].double().cpu()
    err = (got - ref).abs().max().item()
    assert err <= 1e-2 * ref.abs().max().item() + 1e-3, err
    assert out[T:].abs().max().item() == 0.0  # no stores past T


@pytest.mark.parametrize("N,K,T,row_off", [(4096, 4096, 64, 0), (12288, 4096, 16, 3), (4096, 11008, 64, 0),
                                           (22016, 4096, 8, 0), (1024, 4096, 1, 5), (12288, 4096, 200, 0),
                                           (32000, 4096, 128, 2), (4096, 11008, 256, 0), (22016, 4096, 1000, 0),
                                           (4096, 4096, 2100, 7), (12288, 4096, 100, 0), (22016, 4096, 77, 3)])
def test_gemm_f32_7b_shapes(lib, cuda, N, K, T, row_off):
    """7B projection shapes (QKV / O / down / gate+up): stream-K splits across SMs."""
    torch = cuda
    w = _bf16(torch, (N, K), 0.02, 3).cuda()
    x = _bf16(torch, (T + row_off, K), 1.0, 4).cuda()
    out = torch.zeros(T + row_off, N, dtype=torch.float32, device="cuda")
    _gemm(lib, torch, w, x, T, row_off, 1, out, N)
    ref = x[row_off:].double().cpu() @ w.double().cpu().T
    got = out[row_off:].double().cpu()
    err = (got - ref).abs().max().item()
    assert err <= 2e-5 * K ** 0.5 * ref.abs().max().item() + 1e-4, err
    if row_off:
        assert out[:row_off].abs().max().item() == 0.0  # rows before row_off untouched


@pytest.mark.parametrize("N,K,T,row_off,epi", [(22016, 4096, 8192, 0, 1), (4096, 11008, 3000, 5, 2),
                                               (12288, 4096, 4321, 0, 0), (4096, 4096, 1900, 3, 1)])
def test_gemm_prefill_rastered(lib, cuda, N, K, T, row_off, epi):
    """Prefill-size launches (token-major pair kernel, several token tiles,
    rastered tile order incl. a ragged last group), checked on the GPU against
    an fp32 torch matmul (TF32 off)."""
    torch = cuda
    torch.backends.cuda.matmul.allow_tf32 = False
    w = _bf16(torch, (N, K), 0.02, 21).cuda()
    x = _bf16(torch, (T + row_off, K), 1.0, 22).cuda()
    dt = torch.bfloat16 if epi == 0 else torch.float32
    base = torch.randn(T + row_off, N, dtype=torch.float32, device="cuda").to(dt)
    out = base.clone()
    _gemm(lib, torch, w, x, T, row_off, epi, out, N)
    ref = x[row_off:].float() @ w.float().T
    if epi == 2:
        ref = ref + base[row_off:].float()
    err = (out[row_off:].float() - ref).abs().max().item()
    tol = (1e-2 if epi == 0 else 2e-5 * K ** 0.5) * ref.abs().max().item() + 1e-3
    assert err <= tol, (err, tol)
    if row_off:
        assert torch.equal(out[:row_off], base[:row_off])


@pytest.mark.parametrize("N,K,T", [(256, 512, 24), (512, 1024, 200), (4096, 4096, 256), (768, 512, 700)])
def test_gemm_residual_epilogue(lib, cuda, N, K, T):
    """+= epilogue on the 1-CTA (T <= 128) and CTA-pair (T > 128) kernels, incl. stream-K fixups."""
    torch = cuda
    w = _bf16(torch, (N, K), 0.05, 5).cuda()
    x = _bf16(torch, (T, K), 1.0, 6).cuda()
    base = torch.randn(T, N, dtype=torch.float32, device="cuda")
    out = base.clone()
    _gemm(lib, torch, w, x, T, 0, 2, out, N)
    ref = base.double().cpu() + x.double().cpu() @ w.double().cpu().T
    assert (out.double().cpu() - ref).abs().max().item() < 2e-6 * K ** 0.5 * ref.abs().max().item() + 1e-4


@pytest.mark.parametrize("F,K,T", [(384, 256, 19), (11008, 4096, 256), (640, 512, 150)])
def test_gemm_swiglu_epilogue(lib, cuda, F, K, T):
    torch = cuda
    gate = _bf16(torch, (F, K), 0.06, 7)
    up = _bf16(torch, (F, K), 0.06, 8)
    w = torch.stack([gate, up], dim=1).reshape(2 * F, K).contiguous().cuda()  # row 2j gate_j, 2j+1 up_j
    x = _bf16(torch, (T, K), 1.0, 9).cuda()
    out = torch.zeros(T, F, dtype=torch.bfloat16, device="cuda")
    _gemm(lib, torch, w, x, T, 0, 3, out, F)
    xd = x.double().cpu()
    g = xd @ gate.double().T
    u = xd @ up.double().T
    ref = g / (1 + torch.exp(-g)) * u
    err = (out.double().cpu() - ref).abs().max().item()
    assert err <= 1e-2 * ref.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("N,K", [(4096, 4096), (12288, 4096), (22016, 4096)])
def test_gemm_deterministic_and_row_split_invariant(lib, cuda, N, K):
    """Bit-identical reruns, and rows give the same bits whether computed as one
    batch of 15 or as the 7 + 8 replica micro-batches split_batch produces
    (cluster split-K, multicast and stream-K plans)."""
    torch = cuda
    w = _bf16(torch, (N, K), 0.02, 10).cuda()
    x = _bf16(torch, (15, K), 1.0, 11).cuda()
    a = torch.zeros(15, N, dtype=torch.float32, device="cuda")
    b = torch.zeros_like(a)
    c = torch.zeros_like(a)
    _gemm(lib, torch, w, x, 15, 0, 1, a, N)
    _gemm(lib, torch, w, x, 15, 0, 1, b, N)
    _gemm(lib, torch, w, x, 7, 0, 1, c, N)
    _gemm(lib, torch, w, x, 8, 7, 1, c, N)
    assert torch.equal(a, b)
    assert torch.equal(a, c)


def _set_norm(lib, ssq_in=None, h_out=None, gamma=None, ssq_out=None, d=0, eps=1e-5):
    P = lambda t: None if t is None else t.data_ptr()
    assert lib.cbt_gemm_set_norm(P(ssq_in), P(h_out), P(gamma), P(ssq_out), d // 32, d, C.c_float(eps)) == 0


@pytest.mark.parametrize("epi,N,K,T,row_off", [(0, 12288, 4096, 64, 0), (0, 384, 256, 1, 3), (3, 22016, 4096, 256, 0),
                                               (3, 640, 512, 37, 2), (1, 32000, 4096, 128, 0), (1, 256, 256, 200, 0),
                                               (0, 12288, 4096, 256, 0)])
def test_gemm_fused_norm_consumer(lib, cuda, epi, N, K, T, row_off):
    """Fused RMSNorm, consumer side: X rows are h' = bf16(x * gamma), the
    epilogue scales each token row by rsqrt(sum(ssq partials) / d + eps) before
    its op (bf16 store, SwiGLU, fp32 logits) == GEMM of RMSNorm(x) (fp64 ref)."""
    torch = cuda
    rows = T + row_off
    x = torch.randn(rows, K, dtype=torch.float32) * 2
    gamma = (torch.rand(K) * 0.5 + 0.75).to(torch.bfloat16)
    hp = (x * gamma.float()).to(torch.bfloat16)
    ssq = (x * x).view(rows, K // 32, 32).sum(-1).contiguous()
    w = _bf16(torch, (N, K), 0.03, 21)
    ocols = N // 2 if epi == 3 else N
    odt = torch.float32 if epi == 1 else torch.bfloat16
    out = torch.zeros(rows, ocols, dtype=odt, device="cuda")
    ssq_d = ssq.cuda()
    _set_norm(lib, ssq_in=ssq_d, d=K)
    try:
        _gemm(lib, torch, w.cuda(), hp.cuda(), T, row_off, epi, out, ocols)
    finally:
        _set_norm(lib)
    xd = x.double()[row_off:]
    hn = xd / torch.sqrt((xd * xd).mean(-1, keepdim=True) + 1e-5) * gamma.double()
    y = hn @ w.double().T
    if epi == 3:
        g, u = y[:, 0::2], y[:, 1::2]
        y = g / (1 + torch.exp(-g)) * u
    got = out[row_off:].double().cpu()
    err = (got - y).abs().max().item()
    assert err <= 1.5e-2 * y.abs().max().item() + 1e-3, err
    if row_off:
        assert out[:row_off].abs().max().item() == 0.0


@pytest.mark.parametrize("N,K,T", [(4096, 4096, 64), (4096, 11008, 256), (4096, 4096, 1), (4096, 4096, 130),
                                   (512, 256, 19)])
def test_gemm_fused_norm_producer(lib, cuda, N, K, T):
    """Fused RMSNorm, producer side (residual epilogue): x += proj as before,
    plus h' = bf16(x_new * gamma) bit-exactly and per-32-feature sums of x_new^2."""
    torch = cuda
    w = _bf16(torch, (N, K), 0.03, 22).cuda()
    a = _bf16(torch, (T, K), 1.0, 23).cuda()
    base = torch.randn(T, N, dtype=torch.float32, device="cuda")
    x = base.clone()
    gamma = (torch.rand(N) * 0.5 + 0.75).to(torch.bfloat16).cuda()
    h = torch.zeros(T, N, dtype=torch.bfloat16, device="cuda")
    ssq = torch.zeros(T, N // 32, dtype=torch.float32, device="cuda")
    _set_norm(lib, h_out=h, gamma=gamma, ssq_out=ssq, d=N)
    try:
        _gemm(lib, torch, w, a, T, 0, 2, x, N)
    finally:
        _set_norm(lib)
    ref = base.double().cpu() + a.double().cpu() @ w.double().cpu().T
    assert (x.double().cpu() - ref).abs().max().item() < 2e-6 * K ** 0.5 * ref.abs().max().item() + 1e-4
    assert torch.equal(h, (x * gamma.float()).to(torch.bfloat16))
    ssq_ref = (x.double() ** 2).view(T, N // 32, 32).sum(-1)
    assert torch.allclose(ssq.double(), ssq_ref, rtol=1e-5, atol=1e-5)


def test_gemm_fused_norm_rejects_multi_tile(lib, cuda):
    """The row-scale table holds one token tile: T > 256 with ssq_in is refused."""
    torch = cuda
    K, N, T = 256, 256, 300
    ssq = torch.ones(T, K // 32, device="cuda")
    w = _bf16(torch, (N, K), 0.03, 24).cuda()
    x = _bf16(torch, (T, K), 1.0, 25).cuda()
    out = torch.zeros(T, N, dtype=torch.bfloat16, device="cuda")
    _set_norm(lib, ssq_in=ssq, d=K)
    try:
        st = lib.cbt_gemm(_ptr(w), _ptr(x), T, N, K, T, 0, 0, _ptr(out), N)
    finally:
        _set_norm(lib)
    assert st != 0


def test_rmsnorm(lib, cuda):
    torch = cuda
    T, d = 37, 4096
    x = torch.randn(T, d, dtype=torch.float32, device="cuda") * 3
    g = _bf16(torch, (d,), 0.1, 12).add(1.0).to(torch.bfloat16).cuda()
    y = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    assert lib.cbt_rmsnorm(_ptr(x), _ptr(g), _ptr(y), T, d, C.c_float(1e-5)) == 0
    xd = x.double().cpu()
    ref = xd / torch.sqrt((xd * xd).mean(-1, keepdim=True) + 1e-5) * g.double().cpu()
    err = (y.double().cpu() - ref).abs().max().item()
    assert err <= 8e-3 * ref.abs().max().item(), err


def _rope_ref(x, pos, theta):
    hd = x.shape[-1]
    half = hd // 2
    inv = np.power(float(theta), -2.0 * np.arange(half) / hd)
    ang = pos[:, None].astype(np.float64) * inv[None, :]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], -1)


@pytest.mark.parametrize("H,Hkv,hd", [(4, 4, 64), (32, 32, 128), (8, 2, 128)])
def test_rope_kv_append(lib, cuda, H, Hkv, hd):
    torch = cuda
    T, max_ctx, slots = 6, 40, 4
    qkv = _bf16(torch, (T, (H + 2 * Hkv) * hd), 1.0, 13).cuda()
    kv = torch.zeros(slots, max_ctx, 2, Hkv * hd, dtype=torch.bfloat16, device="cuda")
    row_slot = torch.tensor([0, 1, 3, 2, 1, 0], dtype=torch.int32, device="cuda")
    row_pos = torch.tensor([0, 5, 39, 7, 6, 1], dtype=torch.int32, device="cuda")
    orig = qkv.double().cpu().numpy()
    assert lib.cbt_rope_kv(_ptr(qkv), _ptr(kv), _ptr(row_slot), _ptr(row_pos), T, H, Hkv, hd, max_ctx,
                           C.c_float(10000.0)) == 0
    pos = row_pos.cpu().numpy()
    q_ref = _rope_ref(orig[:, : H * hd].reshape(T, H, hd), pos, 1e4)
    k_ref = _rope_ref(orig[:, H * hd:(H + Hkv) * hd].reshape(T, Hkv, hd), pos, 1e4)
    v_ref = orig[:, (H + Hkv) * hd:]
    q_got = qkv[:, : H * hd].double().cpu().numpy().reshape(T, H, hd)
    assert np.abs(q_got - q_ref).max() <= 1.6e-2
    kvc = kv.double().cpu().numpy()
    for t in range(T):
        s, p = int(row_slot[t]), int(pos[t])
        assert np.abs(kvc[s, p, 0].reshape(Hkv, hd) - k_ref[t]).max() <= 1.6e-2
        assert np.array_equal(kvc[s, p, 1], v_ref[t])  # v is copied bit-exactly


@pytest.mark.parametrize("H,Hkv,hd,lens", [(4, 4, 64, [1, 16, 17, 63]), (32, 32, 128, [300, 1, 128, 2000]),
                                           (8, 2, 128, [5, 700]), (32, 32, 128, [4096]), (16, 2, 128, [33, 260]),
                                           (64, 8, 128, [129, 7, 1000]), (8, 4, 64, [70, 3])])
def test_attention(lib, cuda, H, Hkv, hd, lens):
    torch = cuda
    T = len(lens)
    max_ctx = max(lens) + 3
    qkv = _bf16(torch, (T, (H + 2 * Hkv) * hd), 1.0, 14).cuda()
    kv = _bf16(torch, (T, max_ctx, 2, Hkv * hd), 1.0, 15).cuda()
    out = torch.zeros(T, H * hd, dtype=torch.bfloat16, device="cuda")
    row_slot = torch.arange(T, dtype=torch.int32, device="cuda")
    row_pos = torch.tensor([L - 1 for L in lens], dtype=torch.int32, device="cuda")
    assert lib.cbt_attention(_ptr(qkv), _ptr(kv), _ptr(out), _ptr(row_slot), _ptr(row_pos), T, H, Hkv, hd,
                             max_ctx) == 0
    q = qkv[:, : H * hd].double().cpu().numpy().reshape(T, H, hd)
    kvn = kv.double().cpu().numpy()
    g = H // Hkv
    for t, L in enumerate(lens):
        k = np.repeat(kvn[t, :L, 0].reshape(L, Hkv, hd), g, axis=1)
        v = np.repeat(kvn[t, :L, 1].reshape(L, Hkv, hd), g, axis=1)
        s = np.einsum("hd,lhd->hl", q[t], k) / np.sqrt(hd)
        p = np.exp(s - s.max(-1, keepdims=True))
        p /= p.sum(-1, keepdims=True)
        ref = np.einsum("hl,lhd->hd", p, v).reshape(-1)
        got = out[t].double().cpu().numpy()
        assert np.abs(got - ref).max() <= 1e-2 * max(1.0, np.abs(ref).max()), (t, np.abs(got - ref).max())


def test_argmax_ties_lowest_index(lib, cuda):
    torch = cuda
    T, V = 5, 32000
    logits = torch.randn(T, V, dtype=torch.float32, device="cuda")
    logits[1, 100] = 50.0
    logits[1, 20000] = 50.0  # tie -> lowest index
    logits[2, V - 1] = 60.0
    out = torch.empty(T, dtype=torch.int32, device="cuda")
    assert lib.cbt_argmax(_ptr(logits), _ptr(out), T, V) == 0
    ref = logits.cpu().numpy().argmax(-1)
    assert out.cpu().numpy().tolist() == ref.tolist()
    assert int(out[1]) == 100


@pytest.mark.parametrize("H,Hkv,hd,lens", [(4, 4, 64, [1, 16, 17, 40]), (32, 32, 128, [300, 1, 129, 900]),
                                           (8, 2, 128, [5, 700])])
def test_fused_decode_attention_bit_identical(lib, cuda, H, Hkv, hd, lens):
    """Decode path: RoPE + KV append fused into attention == rope_kv kernel then
    attention, bit for bit (output and appended cache row)."""
    torch = cuda
    T = len(lens)
    max_ctx = max(lens) + 2
    qkv = _bf16(torch, (T, (H + 2 * Hkv) * hd), 1.0, 21).cuda()
    kv = _bf16(torch, (T, max_ctx, 2, Hkv * hd), 1.0, 22).cuda()
    row_slot = torch.arange(T, dtype=torch.int32, device="cuda")
    row_pos = torch.tensor([L - 1 for L in lens], dtype=torch.int32, device="cuda")
    q1, kv1 = qkv.clone(), kv.clone()
    out1 = torch.zeros(T, H * hd, dtype=torch.bfloat16, device="cuda")
    assert lib.cbt_rope_kv(_ptr(q1), _ptr(kv1), _ptr(row_slot), _ptr(row_pos), T, H, Hkv, hd, max_ctx,
                           C.c_float(1e4)) == 0
    assert lib.cbt_attention(_ptr(q1), _ptr(kv1), _ptr(out1), _ptr(row_slot), _ptr(row_pos), T, H, Hkv, hd,
                             max_ctx) == 0
    q2, kv2 = qkv.clone(), kv.clone()
    out2 = torch.zeros_like(out1)
    assert lib.cbt_attention_fused(_ptr(q2), _ptr(kv2), _ptr(out2), _ptr(row_slot), _ptr(row_pos), T, H, Hkv, hd,
                                   max_ctx, C.c_float(1e4)) == 0
    assert torch.equal(out1, out2)
    assert torch.equal(kv1, kv2)


@pytest.mark.parametrize("N,K", [(4096, 4096), (12288, 4096), (4096, 11008)])
def test_gemm_pair_kernel_row_count_invariant(lib, cuda, N, K):
    """CTA-pair regime (129..256 rows): the stream-K split depends on (N, K)
    only, so the first 140 rows of a 256-row launch equal a 140-row launch bit
    for bit, and reruns are bit-identical."""
    torch = cuda
    w = _bf16(torch, (N, K), 0.02, 12).cuda()
    x = _bf16(torch, (256, K), 1.0, 13).cuda()
    a = torch.zeros(256, N, dtype=torch.float32, device="cuda")
    b = torch.zeros_like(a)
    c = torch.zeros_like(a)
    _gemm(lib, torch, w, x, 256, 0, 1, a, N)
    _gemm(lib, torch, w, x, 256, 0, 1, b, N)
    _gemm(lib, torch, w, x, 140, 0, 1, c, N)
    assert torch.equal(a, b)
    assert torch.equal(a[:140], c[:140])
    ref = x.double().cpu() @ w.double().cpu().T
    assert (a.double().cpu() - ref).abs().max().item() <= 2e-5 * K ** 0.5 * ref.abs().max().item() + 1e-4


@pytest.mark.parametrize("H,Hkv,hd,lens", [(4, 4, 64, [1, 63, 64, 65, 128, 129]), (32, 32, 128, [200, 7, 130]),
                                           (8, 2, 128, [129, 64, 256]), (64, 8, 128, [300]),
                                           (4, 4, 128, [1000, 128, 255])])
def test_prefill_attention_causal(lib, cuda, H, Hkv, hd, lens):
    """tcgen05 causal prefill attention (TMA-fed Q/K/V, S and O in TMEM, softmax
    warps one row per thread) vs a float64 causal softmax reference: every row
    of every prompt, 256-row blocks (two 128-row tiles) incl. ragged tails and
    single-tile blocks, multi-block prompts
    (lazy O rescaling in TMEM), GQA, head dims 64/128.  The cache holds NaN
    past each prompt (stale / uninitialised bytes must not leak into rows)."""
    torch = cuda
    T = sum(lens)
    max_ctx = max(lens) + 132
    qkv = _bf16(torch, (T, (H + 2 * Hkv) * hd), 1.0, 31).cuda()
    kv = _bf16(torch, (len(lens), max_ctx, 2, Hkv * hd), 1.0, 32).cuda()
    for sl, L in enumerate(lens):
        kv[sl, L:] = float("nan")
    out = torch.zeros(T, H * hd, dtype=torch.bfloat16, device="cuda")
    blocks, row = [], 0
    for sl, L in enumerate(lens):
        for b0 in range(0, L, 256):
            blocks.append((row + b0, min(256, L - b0), sl, b0))
        row += L
    bl = torch.tensor(blocks, dtype=torch.int32, device="cuda")
    assert lib.cbt_prefill_attention(_ptr(qkv), _ptr(kv), _ptr(out), _ptr(bl), len(blocks), T, H, Hkv, hd,
                                     max_ctx, len(lens)) == 0
    torch.cuda.synchronize()
    q = qkv[:, : H * hd].double().cpu().numpy().reshape(T, H, hd)
    kvn = kv.double().cpu().numpy()
    g = H // Hkv
    row = 0
    for sl, L in enumerate(lens):
        k = np.repeat(kvn[sl, :L, 0].reshape(L, Hkv, hd), g, axis=1)
        v = np.repeat(kvn[sl, :L, 1].reshape(L, Hkv, hd), g, axis=1)
        s = np.einsum("thd,lhd->htl", q[row:row + L], k) / np.sqrt(hd)
        s = np.where(np.tril(np.ones((L, L), bool))[None], s, -np.inf)
        p = np.exp(s - s.max(-1, keepdims=True))
        p /= p.sum(-1, keepdims=True)
        ref = np.einsum("htl,lhd->thd", p, v).reshape(L, -1)
        got = out[row:row + L].double().cpu().numpy()
        assert np.isfinite(got).all(), sl
        assert np.abs(got - ref).max() <= 2e-2 * max(1.0, np.abs(ref).max()), (sl, np.abs(got - ref).max())
        row += L


@pytest.mark.parametrize("T,H,Hkv,lens", [(64, 32, 32, None), (48, 32, 8, [1, 31, 32, 33, 64, 100, 128]),
                                         (40, 32, 32, [1, 31, 32, 33, 200]), (2, 32, 32, [300, 1000]),
                                         (3, 32, 8, [500, 129, 33]), (1, 32, 32, [4096]),
                                         (4, 64, 8, [700, 130, 33, 1]), (40, 64, 8, [1, 32, 64, 100, 128])])
def test_tma_decode_attention_matches_load_kernel(lib, cuda, T, H, Hkv, lens):
    """The TMA-fed decode attention (32-position K / V boxes) against the
    16-byte-load kernel on the same inputs: output and appended cache row
    bit-identical where the load kernel also takes 4 positions per step (MHA
    with >= 8 waves of CTAs), within bf16 rounding otherwise (GQA, few rows
    with long contexts split over whole boxes and merged by the last split);
    cache rows past each sequence poisoned with NaN (a box may cover them)
    never reach the output."""
    torch = cuda
    hd = 128
    if lens is None:
        g = torch.Generator().manual_seed(T)
        lens = torch.randint(1, 300, (T,), generator=g).tolist()
    lens = (lens * (T // len(lens) + 1))[:T]
    max_ctx = max(lens) + 40
    qkv = _bf16(torch, (T, (H + 2 * Hkv) * hd), 1.0, 41).cuda()
    kv = _bf16(torch, (T, max_ctx, 2, Hkv * hd), 1.0, 42)
    for i, L in enumerate(lens):
        kv[i, L:] = float("nan")  # stale rows past the sequence (the current position is written by the kernel)
    kv = kv.cuda()
    row_slot = torch.arange(T, dtype=torch.int32, device="cuda")
    row_pos = torch.tensor([L - 1 for L in lens], dtype=torch.int32, device="cuda")
    outs, kvs = [], []
    for slots in (0, T):
        q_, kv_ = qkv.clone(), kv.clone()
        out = torch.zeros(T, H * hd, dtype=torch.bfloat16, device="cuda")
        assert lib.cbt_attention_set_kv_slots(slots) == 0
        try:
            assert lib.cbt_attention_fused(_ptr(q_), _ptr(kv_), _ptr(out), _ptr(row_slot), _ptr(row_pos), T, H, Hkv,
                                           hd, max_ctx, C.c_float(1e4)) == 0
        finally:
            lib.cbt_attention_set_kv_slots(0)
        outs.append(out)
        kvs.append(kv_)
    assert torch.isfinite(outs[1].float()).all()
    assert torch.equal(kvs[0].nan_to_num(7.0), kvs[1].nan_to_num(7.0))  # the appended rows
    if Hkv == H and T * Hkv >= 8 * 148:
        assert torch.equal(outs[0], outs[1])
    else:
        assert (outs[0].float() - outs[1].float()).abs().max().item() <= 2e-2
