// Warp-shuffle attention over the contiguous per-replica slot KV cache.
//
// Cache layout per (layer, device): [slot][max_ctx][2 (k,v)][Hkv * hd] bf16, so
// one token's K and V rows are adjacent and one slot's live KV is the single
// contiguous prefix [0, len) -- the byte run the reference prices as
// `kv_bytes_per_token_per_layer` = 2*d*b (domain.py:263) and that a KV
// migration moves (ops.py:230-251).
//
// Row-parallel: CTA = (row, kv head, context split).  A group of hd/8 lanes owns
// one position (16 bytes per lane = one 128-bit load of K and of V), a warp
// covers 32/(hd/8) positions per step, 4 warps stride the context.  Scores use
// exp2 with q pre-scaled by log2(e)/sqrt(hd); online softmax in fp32; the
// partial states are merged across lane groups (shuffles), warps (smem) and --
// for short batches with long context -- across context splits (a second
// combine kernel).  Decode attention is HBM-bound: every K/V byte is read once.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace cb {

static constexpr int kAttnWarps = 4;
static constexpr int kUnroll = 4;

// positions in flight per lane group per step: fewer for wide GQA groups so the
// per-head q / accumulator registers fit
template <int GQ>
struct AttnUnroll {
  static constexpr int value = GQ >= 4 ? 2 : 4;
};

template <int HD, int GQ, int U>
__global__ void __launch_bounds__(kAttnWarps * 32)
    attn_kernel(const AttnArgs a, int nsplit, int chunk) {
  pdl_trigger();
  pdl_wait();
  constexpr int G = HD / 8;  // lanes per position
  constexpr int P = 32 / G;  // positions per warp step
  const int row = a.row_off + blockIdx.x;
  const int hk = blockIdx.y;
  const int split = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lg = lane % G, pg = lane / G;
  const int slot = a.row_slot[row];
  const int len = a.row_pos[row] + 1;
  const int p_begin = split * chunk;
  const int p_end = min(len, p_begin + chunk);
  const float qscale = a.scale * 1.4426950408889634f;
  const size_t kvd = size_t(a.Hkv) * HD;
  const size_t pos_stride = 2 * kvd;
  const uint16_t* kbase = a.kv + (size_t)slot * a.max_ctx * pos_stride + (size_t)hk * HD + lg * 8;
  const size_t qkv_ld = size_t(a.H + 2 * a.Hkv) * HD;
  const int cur = len - 1;  // position of this row's own token

  __shared__ float sm_state[kAttnWarps][GQ][G][10];

  if (a.rope != nullptr && warp == 0 && p_begin <= cur && cur < p_end) {
    // Fused decode path: the CTA whose context split holds the newest position
    // appends this row's rotated k and raw v for kv head hk to the cache.
    uint16_t* kc = const_cast<uint16_t*>(a.kv) + ((size_t)slot * a.max_ctx + cur) * pos_stride + (size_t)hk * HD;
    const uint16_t* ksrc = a.qkv + row * qkv_ld + (size_t)(a.H + hk) * HD;
    const uint16_t* vsrc = ksrc + (size_t)a.Hkv * HD;
    constexpr int half = HD / 2, cph = half / 8;
    const float2* rp = a.rope + (size_t)cur * half;
    if (lane < cph) {
      const int i0 = lane * 8;
      const uint4 x = *reinterpret_cast<const uint4*>(ksrc + i0);
      const uint4 y = *reinterpret_cast<const uint4*>(ksrc + i0 + half);
      const float x1[8] = {bf16_lo(x.x), bf16_hi(x.x), bf16_lo(x.y), bf16_hi(x.y),
                           bf16_lo(x.z), bf16_hi(x.z), bf16_lo(x.w), bf16_hi(x.w)};
      const float x2[8] = {bf16_lo(y.x), bf16_hi(y.x), bf16_lo(y.y), bf16_hi(y.y),
                           bf16_lo(y.z), bf16_hi(y.z), bf16_lo(y.w), bf16_hi(y.w)};
      float o1[8], o2[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float2 cs = rp[i0 + j];
        o1[j] = x1[j] * cs.x - x2[j] * cs.y;
        o2[j] = x2[j] * cs.x + x1[j] * cs.y;
      }
      uint4 r1, r2;
      r1.x = pack_bf16x2(o1[0], o1[1]); r1.y = pack_bf16x2(o1[2], o1[3]);
      r1.z = pack_bf16x2(o1[4], o1[5]); r1.w = pack_bf16x2(o1[6], o1[7]);
      r2.x = pack_bf16x2(o2[0], o2[1]); r2.y = pack_bf16x2(o2[2], o2[3]);
      r2.z = pack_bf16x2(o2[4], o2[5]); r2.w = pack_bf16x2(o2[6], o2[7]);
      *reinterpret_cast<uint4*>(kc + i0) = r1;
      *reinterpret_cast<uint4*>(kc + i0 + half) = r2;
    }
    if (lane < HD / 8)
      reinterpret_cast<uint4*>(kc + kvd)[lane] = reinterpret_cast<const uint4*>(vsrc)[lane];
  }
  if (a.rope != nullptr) __syncthreads();  // the appended row is read back by the loop below

  // q of every head of this KV group: this lane's 8 elements of each
  float q[GQ][8];
#pragma unroll
  for (int g = 0; g < GQ; ++g) {
    const int qh = hk * GQ + g;
    const uint4 qv = *reinterpret_cast<const uint4*>(a.qkv + row * qkv_ld + (size_t)qh * HD + lg * 8);
    q[g][0] = bf16_lo(qv.x); q[g][1] = bf16_hi(qv.x); q[g][2] = bf16_lo(qv.y); q[g][3] = bf16_hi(qv.y);
    q[g][4] = bf16_lo(qv.z); q[g][5] = bf16_hi(qv.z); q[g][6] = bf16_lo(qv.w); q[g][7] = bf16_hi(qv.w);
    if (a.rope != nullptr) {
      // rotate-half RoPE of q in registers: the partner chunk lives G/2 lanes away;
      // rounded to bf16 exactly like the stand-alone rope_kv kernel
      const int hl = lg % (G / 2);
      const bool first = lg < G / 2;
      const float2* rp = a.rope + (size_t)cur * (HD / 2) + hl * 8;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float other = __shfl_xor_sync(0xffffffffu, q[g][i], G / 2);
        const float2 cs = rp[i];
        const float r = first ? q[g][i] * cs.x - other * cs.y : q[g][i] * cs.x + other * cs.y;
        q[g][i] = bf16_to_f(f_to_bf16(r));
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) q[g][i] *= qscale;
  }
  float m[GQ], l[GQ], acc[GQ][8];
#pragma unroll
  for (int g = 0; g < GQ; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[g][i] = 0.f;
  }

  // every K/V row of the group is read once for all GQ heads
  for (int p0 = p_begin + warp * P; p0 < p_end; p0 += kAttnWarps * P * U) {
    uint4 kk[U], vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int pos = p0 + u * kAttnWarps * P + pg;
      if (pos < p_end) {
        const uint16_t* kp = kbase + (size_t)pos * pos_stride;
        // coherent loads: the fused path appended this row's K/V in this kernel
        kk[u] = *reinterpret_cast<const uint4*>(kp);
        vv[u] = *reinterpret_cast<const uint4*>(kp + kvd);
      } else {
        kk[u] = make_uint4(0, 0, 0, 0);
        vv[u] = make_uint4(0, 0, 0, 0);
      }
    }
    float kf[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      kf[u][0] = bf16_lo(kk[u].x); kf[u][1] = bf16_hi(kk[u].x); kf[u][2] = bf16_lo(kk[u].y);
      kf[u][3] = bf16_hi(kk[u].y); kf[u][4] = bf16_lo(kk[u].z); kf[u][5] = bf16_hi(kk[u].z);
      kf[u][6] = bf16_lo(kk[u].w); kf[u][7] = bf16_hi(kk[u].w);
    }
#pragma unroll
    for (int g = 0; g < GQ; ++g) {
      float s[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float t = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) t += q[g][i] * kf[u][i];
        s[u] = t;
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < U; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
      // one online-softmax update for the U positions
      float mx = m[g];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (p0 + u * kAttnWarps * P + pg >= p_end) s[u] = -INFINITY;
        mx = fmaxf(mx, s[u]);
      }
      if (mx != -INFINITY) {
        const float cf = exp2f(m[g] - mx);  // m == -inf -> 0
        l[g] *= cf;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[g][i] *= cf;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float p = exp2f(s[u] - mx);  // invalid positions: exp2(-inf) = 0
          l[g] += p;
          acc[g][0] += p * bf16_lo(vv[u].x);
          acc[g][1] += p * bf16_hi(vv[u].x);
          acc[g][2] += p * bf16_lo(vv[u].y);
          acc[g][3] += p * bf16_hi(vv[u].y);
          acc[g][4] += p * bf16_lo(vv[u].z);
          acc[g][5] += p * bf16_hi(vv[u].z);
          acc[g][6] += p * bf16_lo(vv[u].w);
          acc[g][7] += p * bf16_hi(vv[u].w);
        }
        m[g] = mx;
      }
    }
  }
#pragma unroll
  for (int g = 0; g < GQ; ++g) {
    // merge the P position groups of this warp (lanes with equal lg)
#pragma unroll
    for (int o = G; o < 32; o <<= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m[g], o);
      const float ol = __shfl_xor_sync(0xffffffffu, l[g], o);
      float oacc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) oacc[i] = __shfl_xor_sync(0xffffffffu, acc[g][i], o);
      const float mn = fmaxf(m[g], om);
      const float c1 = (m[g] == -INFINITY) ? 0.f : exp2f(m[g] - mn);
      const float c2 = (om == -INFINITY) ? 0.f : exp2f(om - mn);
      l[g] = l[g] * c1 + ol * c2;
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[g][i] = acc[g][i] * c1 + oacc[i] * c2;
      m[g] = mn;
    }
    if (pg == 0) {
      sm_state[warp][g][lg][0] = m[g];
      sm_state[warp][g][lg][1] = l[g];
#pragma unroll
      for (int i = 0; i < 8; ++i) sm_state[warp][g][lg][2 + i] = acc[g][i];
    }
  }
  __syncthreads();
  // warp w finalises heads g = w, w + 4, ... (lanes < G)
  for (int g = warp; g < GQ; g += kAttnWarps) {
    if (lane >= G) continue;
    const int qh = hk * GQ + g;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, sm_state[w][g][lane][0]);
    float L = 0.f, o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) {
      const float mw = sm_state[w][g][lane][0];
      const float cw = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
      L += sm_state[w][g][lane][1] * cw;
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] += sm_state[w][g][lane][2 + i] * cw;
    }
    if (nsplit == 1) {
      const float inv = 1.f / L;
      uint4 ov;
      ov.x = pack_bf16x2(o[0] * inv, o[1] * inv);
      ov.y = pack_bf16x2(o[2] * inv, o[3] * inv);
      ov.z = pack_bf16x2(o[4] * inv, o[5] * inv);
      ov.w = pack_bf16x2(o[6] * inv, o[7] * inv);
      *reinterpret_cast<uint4*>(a.out + (size_t)row * a.H * HD + (size_t)qh * HD + lane * 8) = ov;
    } else {
      // partial state: [(row_local * H + qh) * nsplit + split] -> (m, l, acc[HD])
      const size_t idx = ((size_t)blockIdx.x * a.H + qh) * nsplit + split;
      float* st = a.ws + idx * (HD + 2);
      if (lane == 0) {
        st[0] = M;
        st[1] = L;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) st[2 + lane * 8 + i] = o[i];
    }
  }
}

template <int HD>
__global__ void attn_combine_kernel(const AttnArgs a, int nsplit) {
  pdl_trigger();
  pdl_wait();
  const int rl = blockIdx.x, qh = blockIdx.y, i = threadIdx.x;
  const float* st = a.ws + ((size_t)rl * a.H + qh) * nsplit * (HD + 2);
  float M = -INFINITY;
  for (int s = 0; s < nsplit; ++s) M = fmaxf(M, st[s * (HD + 2)]);
  float L = 0.f, o = 0.f;
  for (int s = 0; s < nsplit; ++s) {
    const float ms = st[s * (HD + 2)];
    const float c = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
    L += st[s * (HD + 2) + 1] * c;
    o += st[s * (HD + 2) + 2 + i] * c;
  }
  const int row = a.row_off + rl;
  a.out[(size_t)row * a.H * HD + (size_t)qh * HD + i] = f_to_bf16(o / L);
}

template <int HD, int GQ>
static cudaError_t attention_launch_t(const AttnArgs& a, dim3 grid, int nsplit, int chunk, cudaStream_t st) {
  if (GQ == 1) {
    // positions in flight per lane group (tunable for experiments: CB_ATTN_UNROLL=2|4|8)
    static const int u = [] {
      const char* e = getenv("CB_ATTN_UNROLL");
      return e ? atoi(e) : 4;
    }();
    if (u == 2) return launch_pdl(attn_kernel<HD, GQ, 2>, grid, dim3(kAttnWarps * 32), 0, st, a, nsplit, chunk);
    if (u == 8) return launch_pdl(attn_kernel<HD, GQ, 8>, grid, dim3(kAttnWarps * 32), 0, st, a, nsplit, chunk);
  }
  return launch_pdl(attn_kernel<HD, GQ, AttnUnroll<GQ>::value>, grid, dim3(kAttnWarps * 32), 0, st, a, nsplit,
                    chunk);
}

template <int HD>
static cudaError_t attention_hd(const AttnArgs& a, int num_sms, cudaStream_t st) {
  const int gq = a.H / a.Hkv;
  int nsplit = 1;
  const long long ctas = (long long)a.T * a.Hkv;
  if (ctas < 2LL * num_sms && a.max_len > 256) {
    nsplit = int((2LL * num_sms + ctas - 1) / ctas);
    nsplit = min(nsplit, (a.max_len + 255) / 256);
    nsplit = min(nsplit, 32);
    while (nsplit > 1 && (size_t)a.T * a.H * nsplit * (HD + 2) > a.ws_floats) --nsplit;
  }
  const int chunk = (a.max_len + nsplit - 1) / nsplit;
  dim3 grid(a.T, a.Hkv, nsplit);
  cudaError_t e;
  switch (gq) {
    case 1: e = attention_launch_t<HD, 1>(a, grid, nsplit, chunk, st); break;
    case 2: e = attention_launch_t<HD, 2>(a, grid, nsplit, chunk, st); break;
    case 4: e = attention_launch_t<HD, 4>(a, grid, nsplit, chunk, st); break;
    case 8: e = attention_launch_t<HD, 8>(a, grid, nsplit, chunk, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess || nsplit == 1) return e;
  return launch_pdl(attn_combine_kernel<HD>, dim3(a.T, a.H), dim3(HD), 0, st, a, nsplit);
}

cudaError_t attention_launch(const AttnArgs& a, int num_sms, cudaStream_t st) {
  if (a.T <= 0) return cudaSuccess;
  switch (a.hd) {
    case 64: return attention_hd<64>(a, num_sms, st);
    case 128: return attention_hd<128>(a, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace cb
