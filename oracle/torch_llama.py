"""fp32 LLaMA oracle in torch, device-agnostic.  TEST INFRASTRUCTURE ONLY.

Same contract as ``oracle.cpu_llama.OracleModel`` (same math, same weights,
same ``forward(slots, tokens, prompt_lens, replicas)`` API), written with
batched torch ops so that headline-sized cases -- Llama-2-7B geometry, 256
sequences, 128-token prompts, 16+ decode steps -- finish in seconds.  It runs
on the CPU in the CPU test suite, where it is pinned to the numpy oracle (which
is pinned to ``transformers.LlamaForCausalLM``), and on ``cuda`` in the GPU
parity tests as the plain PyTorch fp32 reference of the floating-point path
(TF32 disabled, so every matmul is IEEE fp32).

Only tests/ may import this module; it is never on the product path.

Algorithm (what the numpy oracle restates): PAPER.md:117 layer
composition (RMSNorm -> Q/K/V -> rotate-half RoPE -> causal attention -> O +
residual -> RMSNorm -> SwiGLU gate/up -> down + residual), the parameter
inventory of ModuleCatalog.from_model (domain.py:241-264), prefill-then-decode
phases with KV appended per token (sim.py:269-300), and the replica row split
of split_batch (ops.py:151-158).
"""
from __future__ import annotations

import numpy as np
import torch

from .cpu_llama import LlamaConfig, ModelWeights, from_bf16_bits, rope_table


def _t(a: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(device)


class TorchOracle:
    """fp32 LLaMA with a slot-indexed KV cache [slot, ctx, Hkv, hd] per layer."""

    def __init__(self, cfg: LlamaConfig, weights: ModelWeights, max_ctx: int, max_slots: int,
                 device: str | torch.device = "cpu"):
        if torch.device(device).type == "cuda":
            torch.backends.cuda.matmul.allow_tf32 = False  # IEEE fp32 products
            torch.backends.cudnn.allow_tf32 = False
        self.cfg, self.dev = cfg, torch.device(device)
        self.embed = _t(from_bf16_bits(weights.embed), self.dev)
        self.final_norm = _t(from_bf16_bits(weights.final_norm), self.dev)
        self.lm_head = _t(from_bf16_bits(weights.lm_head), self.dev)
        self.layers = [{k: _t(v, self.dev) for k, v in lw.f32().items()} for lw in weights.layers]
        cos, sin = rope_table(max_ctx, cfg.head_dim, cfg.rope_theta)  # float64 angles -> fp32, as the oracle
        self.cos, self.sin = _t(cos, self.dev), _t(sin, self.dev)
        shape = (max_slots, max_ctx, cfg.n_kv_heads, cfg.head_dim)
        self.k = [torch.zeros(shape, device=self.dev) for _ in self.layers]
        self.v = [torch.zeros(shape, device=self.dev) for _ in self.layers]
        self.lens = np.zeros(max_slots, dtype=np.int64)

    # ---------------------------------------------------------------- pieces
    def _rmsnorm(self, x: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
        return x / torch.sqrt((x * x).mean(-1, keepdim=True) + self.cfg.norm_eps) * g

    def _rope(self, x: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        half = x.shape[-1] // 2
        c, s = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        x1, x2 = x[..., :half], x[..., half:]
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)

    def _attend(self, li: int, q: torch.Tensor, slot: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        """Row t attends to its slot's cached positions [0, pos[t]] (causal)."""
        cfg = self.cfg
        T, H, hd = q.shape
        Hkv = cfg.n_kv_heads
        g = H // Hkv
        ctx = int(pos.max().item()) + 1
        scale = 1.0 / float(np.sqrt(hd))
        out = torch.empty_like(q)
        chunk = max(1, (1 << 27) // max(1, ctx * Hkv * hd))  # bound the gathered K/V to ~0.5 GB each
        ar = torch.arange(ctx, device=self.dev)
        for a in range(0, T, chunk):
            b = min(T, a + chunk)
            kk = self.k[li][slot[a:b], :ctx]  # [t, ctx, Hkv, hd]
            vv = self.v[li][slot[a:b], :ctx]
            qq = q[a:b].view(b - a, Hkv, g, hd)
            s = torch.einsum("tkgd,tckd->tkgc", qq, kk) * scale
            s = s.masked_fill((ar[None, :] > pos[a:b, None])[:, None, None, :], float("-inf"))
            p = torch.softmax(s, dim=-1)
            out[a:b] = torch.einsum("tkgc,tckd->tkgd", p, vv).reshape(b - a, H, hd)
        return out

    def layer_forward(self, li: int, x: torch.Tensor, slot: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        cfg, W = self.cfg, self.layers[li]
        T = x.shape[0]
        H, Hkv, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
        h = self._rmsnorm(x, W["attn_norm"])
        q = self._rope((h @ W["wq"].T).view(T, H, hd), pos)
        k = self._rope((h @ W["wk"].T).view(T, Hkv, hd), pos)
        v = (h @ W["wv"].T).view(T, Hkv, hd)
        self.k[li][slot, pos] = k
        self.v[li][slot, pos] = v
        att = self._attend(li, q, slot, pos).reshape(T, H * hd)
        x = x + att @ W["wo"].T
        h = self._rmsnorm(x, W["ffn_norm"])
        gt = h @ W["w_gate"].T
        a = gt / (1.0 + torch.exp(-gt)) * (h @ W["w_up"].T)
        return x + a @ W["w_down"].T

    # ---------------------------------------------------------------- one pass
    @torch.no_grad()
    def forward(self, slots, tokens, prompt_lens=None, replicas: dict[int, int] | None = None) -> np.ndarray:
        """One pass (prefill when prompt_lens is given, else one decode token per
        sequence); returns fp32 logits [n_seq, vocab] of each sequence's last row.
        ``replicas`` = {layer index: p}: each replica's split_batch share of the
        sequences runs separately (row-DP; equals the unreplicated pass)."""
        slots = [int(s) for s in slots]
        n = len(slots)
        lens = [1] * n if prompt_lens is None else [int(L) for L in prompt_lens]
        if prompt_lens is None:
            pos_np = np.array([self.lens[s] for s in slots], dtype=np.int64)
        else:
            pos_np = np.concatenate([np.arange(L) for L in lens]).astype(np.int64)
        seq_row = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        slot = torch.from_numpy(np.repeat(np.array(slots, dtype=np.int64), lens)).to(self.dev)
        pos = torch.from_numpy(pos_np).to(self.dev)
        x = self.embed[torch.from_numpy(np.asarray(tokens, dtype=np.int64)).to(self.dev)]
        for li in range(len(self.layers)):
            p = (replicas or {}).get(li, 1)
            q_, r_ = divmod(n, p)
            shares = [q_] * (p - r_) + [q_ + 1] * r_
            parts, s0 = [], 0
            for sh in shares:
                if sh:
                    r0, r1 = int(seq_row[s0]), int(seq_row[s0 + sh])
                    parts.append(self.layer_forward(li, x[r0:r1], slot[r0:r1], pos[r0:r1]))
                s0 += sh
            x = torch.cat(parts, 0)
        for s, L in zip(slots, lens):
            self.lens[s] += L
        last = x[torch.from_numpy(seq_row[1:] - 1).to(self.dev)]
        h = self._rmsnorm(last, self.final_norm)
        return (h @ self.lm_head.T).cpu().numpy()

    def release(self, slots) -> None:
        for s in slots:
            self.lens[int(s)] = 0
