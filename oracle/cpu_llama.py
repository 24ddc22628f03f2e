"""CPU fp32 oracle for the decoder-layer data path.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker or the timed
CPU baseline -- never on the product path.

Why a restatement: the reference (CoCoServe's `modscale`) has no forward pass,
weights or tokenizer; SURVEY.md §8(c).  This oracle
restates the LLaMA decoder the paper serves (PAPER.md:117 layer composition:
Q/K/V/O projections + RMSNorm + SwiGLU FFN) with exactly the parameter
inventory the reference's byte catalog counts (ModuleCatalog.from_model,
domain.py:241-264: q,k,v,o = d x d; gate, up, down = d x d_ff; two norm
vectors; KV = 2*d per token per layer), the prefill-then-decode phases and KV
token accounting of the serving engine (sim.py:269-300, 637-668), and the
replica row split (ops.py:151-158; "a batch of 15 splits into 7 + 8").

Parity pin: tests/golden/tiny_llama_hf.npz holds logits/tokens produced by
`transformers.LlamaForCausalLM` (fp32, CPU) on the same weights
(oracle/gen_golden.py); tests check this oracle against it.

Numerics: fp32 math over bf16-valued weights (the weights ARE bf16 -- the
model is defined by its bf16 parameters; activations stay fp32 here).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


# ------------------------------------------------------------------ bf16 helpers
def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (round-to-nearest-even) and return as fp32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns (uint16), round-to-nearest-even."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# ------------------------------------------------------------------ config / weights
@dataclass(frozen=True)
class LlamaConfig:
    n_layers: int = 4
    d_model: int = 256
    d_ff: int = 768
    n_heads: int = 4
    n_kv_heads: int = 4
    vocab: int = 1024
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads


TINY = LlamaConfig()  # 4L, d=256, H=4, d_ff=768, vocab=1024
LLAMA2_7B = LlamaConfig(32, 4096, 11008, 32, 32, 32000)
LLAMA2_13B = LlamaConfig(40, 5120, 13824, 40, 40, 32000)


@dataclass
class LayerWeights:
    """bf16 bit patterns (uint16), PyTorch Linear layout [out, in]."""

    attn_norm: np.ndarray
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    ffn_norm: np.ndarray
    w_gate: np.ndarray
    w_up: np.ndarray
    w_down: np.ndarray

    def f32(self) -> dict:
        return {k: from_bf16_bits(v) for k, v in self.__dict__.items()}


@dataclass
class ModelWeights:
    embed: np.ndarray       # [vocab, d] bf16 bits
    final_norm: np.ndarray  # [d]
    lm_head: np.ndarray     # [vocab, d]
    layers: list = field(default_factory=list)


def init_weights(cfg: LlamaConfig, seed: int = 0, w_std: float | None = None, head_std: float | None = None,
                 n_layers: int | None = None, head: str = "random") -> ModelWeights:
    """Seeded normal init (bf16-rounded).  Defaults: O(1) hidden states and a
    logit std of ~0.6, small enough that a bf16 pipeline stays within the
    north star's 2e-2 max-abs logit tolerance of this fp32 oracle."""
    rng = np.random.default_rng(seed)
    d, ff, hd = cfg.d_model, cfg.d_ff, cfg.head_dim
    w_std = w_std if w_std is not None else 1.0 / np.sqrt(d)
    head_std = head_std if head_std is not None else 0.6 / np.sqrt(d)

    def mat(rows, cols, std):
        return to_bf16_bits(rng.standard_normal((rows, cols), dtype=np.float32) * std)

    def vec(n):
        return to_bf16_bits(1.0 + 0.1 * rng.standard_normal(n, dtype=np.float32))

    layers = []
    for _ in range(cfg.n_layers if n_layers is None else n_layers):
        layers.append(LayerWeights(
            attn_norm=vec(d),
            wq=mat(cfg.n_heads * hd, d, w_std),
            wk=mat(cfg.n_kv_heads * hd, d, w_std),
            wv=mat(cfg.n_kv_heads * hd, d, w_std),
            wo=mat(d, cfg.n_heads * hd, w_std),
            ffn_norm=vec(d),
            w_gate=mat(ff, d, w_std),
            w_up=mat(ff, d, w_std),
            w_down=mat(d, ff, 1.0 / np.sqrt(ff)),
        ))
    w = ModelWeights(
        embed=to_bf16_bits(rng.standard_normal((cfg.vocab, d), dtype=np.float32)),
        final_norm=vec(d),
        lm_head=mat(cfg.vocab, d, head_std),
        layers=layers,
    )
    if head == "permuted_tied":
        # "confident" head: lm_head[pi(t)] = e(t) / 128, so the next token's logit
        # stands ~1.6 above the rest (min top-2 margin 0.43 over the 480 config-1
        # decisions, >> the 2e-2 tolerance): greedy identity is then a property of
        # the numerics, not of luck at near-ties.
        perm = np.random.default_rng(seed + 1000).permutation(cfg.vocab)
        head_w = np.empty((cfg.vocab, d), dtype=np.float32)
        head_w[perm] = from_bf16_bits(w.embed) / 128.0
        w.lm_head = to_bf16_bits(head_w)
    elif head != "random":
        raise ValueError(head)
    return w


# ------------------------------------------------------------------ primitive ops
def rmsnorm(x: np.ndarray, gamma: np.ndarray, eps: float) -> np.ndarray:
    x = x.astype(np.float32)
    var = np.mean(x * x, axis=-1, keepdims=True)
    return (x / np.sqrt(var + np.float32(eps))) * gamma


def rope_table(max_ctx: int, hd: int, theta: float) -> tuple[np.ndarray, np.ndarray]:
    """cos/sin [max_ctx, hd/2]: angle(p, i) = p * theta^(-2i/hd), float64 -> fp32."""
    i = np.arange(hd // 2, dtype=np.float64)
    inv = np.power(np.float64(theta), -2.0 * i / hd)
    ang = np.arange(max_ctx, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def apply_rope(x: np.ndarray, pos: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """Rotate-half RoPE.  x: [T, heads, hd], pos: [T]."""
    half = x.shape[-1] // 2
    c = cos[pos][:, None, :]
    s = sin[pos][:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def attention_rows(q: np.ndarray, k_cache: np.ndarray, v_cache: np.ndarray, lens: np.ndarray) -> np.ndarray:
    """q: [T, H, hd]; k/v_cache: [T, ctx, Hkv, hd] per row; row t sees [0, lens[t])."""
    T, H, hd = q.shape
    Hkv = k_cache.shape[2]
    g = H // Hkv
    out = np.zeros((T, H, hd), dtype=np.float32)
    scale = np.float32(1.0 / np.sqrt(hd))
    for t in range(T):
        L = int(lens[t])
        k = np.repeat(k_cache[t, :L], g, axis=1)  # [L, H, hd]
        v = np.repeat(v_cache[t, :L], g, axis=1)
        s = np.einsum("hd,lhd->hl", q[t], k) * scale
        s = s - s.max(axis=-1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(axis=-1, keepdims=True)
        out[t] = np.einsum("hl,lhd->hd", p, v)
    return out


# ------------------------------------------------------------------ model with KV cache
class OracleModel:
    """fp32 LLaMA with a per-sequence KV cache (one cache per layer per slot).

    ``bf16_acts=True`` is a *diagnostic* variant: still fp32 math, but the
    activations are rounded to bf16 where the B200 path stores them in bf16
    (GEMM operands h/att/act, q/k/v, attention output, final h).  It is not
    bit-faithful to the GPU -- attention amplifies single-ulp rounding flips
    chaotically -- so parity tests use the plain fp32 oracle with the 2e-2
    logit tolerance.
    """

    def __init__(self, cfg: LlamaConfig, weights: ModelWeights, max_ctx: int = 512, bf16_acts: bool = False):
        self.cfg = cfg
        self.r = bf16_round if bf16_acts else (lambda a: a)
        self.w = weights
        self.embed = from_bf16_bits(weights.embed)
        self.final_norm = from_bf16_bits(weights.final_norm)
        self.lm_head = from_bf16_bits(weights.lm_head)
        self.layers = [lw.f32() for lw in weights.layers]
        self.cos, self.sin = rope_table(max_ctx, cfg.head_dim, cfg.rope_theta)
        self.kv: dict[int, list] = {}  # slot -> per layer [k (ctx,Hkv,hd), v]
        self.lens: dict[int, int] = {}

    def layer_forward(self, li: int, x: np.ndarray, slots: list[int], pos: np.ndarray) -> np.ndarray:
        """One decoder layer over rows x [T, d] (row t belongs to slots[t] at pos[t]).

        KV for each row is appended to its slot before attention (causal)."""
        cfg, W = self.cfg, self.layers[li]
        H, Hkv, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
        T = x.shape[0]
        r = self.r
        h = r(rmsnorm(x, W["attn_norm"], cfg.norm_eps))
        q = r(h @ W["wq"].T).reshape(T, H, hd)
        k = r(h @ W["wk"].T).reshape(T, Hkv, hd)
        v = r(h @ W["wv"].T).reshape(T, Hkv, hd)
        q = r(apply_rope(q, pos, self.cos, self.sin))
        k = r(apply_rope(k, pos, self.cos, self.sin))
        for t in range(T):
            kc, vc = self.kv[slots[t]][li]
            kc[pos[t]] = k[t]
            vc[pos[t]] = v[t]
        ctx = int(pos.max()) + 1
        kk = np.stack([self.kv[s][li][0][:ctx] for s in slots])
        vv = np.stack([self.kv[s][li][1][:ctx] for s in slots])
        att = r(attention_rows(q, kk, vv, pos + 1).reshape(T, H * hd))
        x = x + att @ W["wo"].T
        h = r(rmsnorm(x, W["ffn_norm"], cfg.norm_eps))
        a = r(silu(h @ W["w_gate"].T) * (h @ W["w_up"].T))
        return x + a @ W["w_down"].T

    def _ensure_slot(self, slot: int) -> None:
        if slot not in self.kv:
            cfg = self.cfg
            shape = (self.cos.shape[0], cfg.n_kv_heads, cfg.head_dim)
            self.kv[slot] = [[np.zeros(shape, np.float32), np.zeros(shape, np.float32)] for _ in self.layers]
            self.lens[slot] = 0

    def forward(self, slots: list[int], tokens: np.ndarray, prompt_lens: list[int] | None,
                replicas: dict[int, int] | None = None) -> np.ndarray:
        """One pass.  prompt_lens given -> prefill (concatenated prompts); else decode.

        ``replicas`` maps layer index -> p: the layer's rows are split with
        split_batch over sequences and each replica's micro-batch runs
        separately, then results are concatenated (replication is row-DP, so
        this must equal the unreplicated pass -- a property the tests check).
        Returns logits [n_seq, vocab] of each sequence's last row."""
        for s in slots:
            self._ensure_slot(s)
        n = len(slots)
        if prompt_lens is None:
            lens = [1] * n
            pos = np.array([self.lens[s] for s in slots], dtype=np.int64)
        else:
            lens = list(prompt_lens)
            pos = np.concatenate([np.arange(L) for L in lens]).astype(np.int64)
        row_slots = [s for s, L in zip(slots, lens) for _ in range(L)]
        seq_row = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        x = self.embed[tokens].astype(np.float32)
        for li in range(len(self.layers)):
            p = (replicas or {}).get(li, 1)
            q_, r_ = divmod(n, p)
            shares = [q_] * (p - r_) + [q_ + 1] * r_
            parts, s0 = [], 0
            for sh in shares:
                if sh:
                    r0, r1 = seq_row[s0], seq_row[s0 + sh]
                    parts.append(self.layer_forward(li, x[r0:r1], row_slots[r0:r1], pos[r0:r1]))
                s0 += sh
            x = np.concatenate(parts, axis=0)
        for s, L in zip(slots, lens):
            self.lens[s] += L
        last = x[seq_row[1:] - 1]
        h = self.r(rmsnorm(last, self.final_norm, self.cfg.norm_eps))
        return h @ self.lm_head.T

    def release(self, slots: list[int]) -> None:
        for s in slots:
            self.kv.pop(s, None)
            self.lens.pop(s, None)


def greedy_generate(model: OracleModel, prompts: list[np.ndarray], n_new: int,
                    replicas: dict[int, int] | None = None) -> tuple[np.ndarray, list[np.ndarray]]:
    """Prefill all prompts, then n_new-1 decode steps.  Returns tokens [n, n_new]
    and the per-step logits list."""
    slots = list(range(len(prompts)))
    logits = model.forward(slots, np.concatenate(prompts), [len(p) for p in prompts], replicas)
    out, all_logits = [logits.argmax(-1)], [logits]
    for _ in range(n_new - 1):
        logits = model.forward(slots, out[-1], None, replicas)
        out.append(logits.argmax(-1))
        all_logits.append(logits)
    return np.stack(out, axis=1), all_logits


def top2_margin(logits: np.ndarray) -> float:
    s = np.sort(logits, axis=-1)
    return float((s[..., -1] - s[..., -2]).min())
