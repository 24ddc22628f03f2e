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

// CTA = (row, kv head, context split), 4 warps.  Lane group j (hd/8 lanes,
// 16 bytes of a K/V row each) owns q-head  j % gq  of the KV group and the
// positions  p == j / gq  (mod  n_groups / gq).  For MHA (gq = 1) the groups
// split the positions 8 (hd 128) ways; for GQA the groups of one warp read the
// same K/V addresses (one transaction) for different q-heads, so every K/V
// byte is fetched once for the whole head group.
template <int HD, int U>
__global__ void __launch_bounds__(kAttnWarps * 32)
    attn_kernel(const AttnArgs a, int nsplit, int chunk, int gq, int head_major) {
  pdl_trigger();
  pdl_wait();
  constexpr int G = HD / 8;               // lanes per group
  constexpr int P = 32 / G;               // groups per warp
  constexpr int NG = kAttnWarps * P;      // groups per CTA
  // head-major grids launch the kv heads of one row back to back, so the CTAs
  // running together read the whole contiguous [k | v] rows of their positions
  const int rl = head_major ? blockIdx.y : blockIdx.x;
  const int row = a.row_off + rl;
  const int hk = head_major ? blockIdx.x : blockIdx.y;
  const int split = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lg = lane % G, pg = lane / G;
  const int grp = warp * P + pg;
  const int head = grp % gq, phase = grp / gq, nph = NG / gq;
  const int qh = hk * gq + head;
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

  __shared__ float sm_state[NG][G][10];

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

  float q[8];
  {
    const uint4 qv = *reinterpret_cast<const uint4*>(a.qkv + row * qkv_ld + (size_t)qh * HD + lg * 8);
    q[0] = bf16_lo(qv.x); q[1] = bf16_hi(qv.x); q[2] = bf16_lo(qv.y); q[3] = bf16_hi(qv.y);
    q[4] = bf16_lo(qv.z); q[5] = bf16_hi(qv.z); q[6] = bf16_lo(qv.w); q[7] = bf16_hi(qv.w);
    if (a.rope != nullptr) {
      // rotate-half RoPE of q in registers: the partner chunk lives G/2 lanes away;
      // rounded to bf16 exactly like the stand-alone rope_kv kernel
      const int hl = lg % (G / 2);
      const bool first = lg < G / 2;
      const float2* rp = a.rope + (size_t)cur * (HD / 2) + hl * 8;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float other = __shfl_xor_sync(0xffffffffu, q[i], G / 2);
        const float2 cs = rp[i];
        const float r = first ? q[i] * cs.x - other * cs.y : q[i] * cs.x + other * cs.y;
        q[i] = bf16_to_f(f_to_bf16(r));
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] *= qscale;
  }
  float m = -INFINITY, l = 0.f, acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;

  // the loop trip count is uniform within a warp (groups of a warp share the
  // phase when gq >= P; for gq < P they differ by < nph, handled by predication)
  const int wphase = (warp * P) / gq;
  for (int pb = p_begin + wphase; pb < p_end; pb += nph * U) {
    uint4 kk[U], vv[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int pos = pb + (phase - wphase) + u * nph;
      ok[u] = pos < p_end;
      if (ok[u]) {
        const uint16_t* kp = kbase + (size_t)pos * pos_stride;
        // coherent loads: the fused path appended this row's K/V in this kernel
        kk[u] = *reinterpret_cast<const uint4*>(kp);
        vv[u] = *reinterpret_cast<const uint4*>(kp + kvd);
      } else {
        kk[u] = make_uint4(0, 0, 0, 0);
        vv[u] = make_uint4(0, 0, 0, 0);
      }
    }
    float s[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      s[u] = q[0] * bf16_lo(kk[u].x) + q[1] * bf16_hi(kk[u].x) + q[2] * bf16_lo(kk[u].y) +
             q[3] * bf16_hi(kk[u].y) + q[4] * bf16_lo(kk[u].z) + q[5] * bf16_hi(kk[u].z) +
             q[6] * bf16_lo(kk[u].w) + q[7] * bf16_hi(kk[u].w);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < U; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
    float mx = m;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!ok[u]) s[u] = -INFINITY;
      mx = fmaxf(mx, s[u]);
    }
    if (mx != -INFINITY) {
      const float cf = exp2f(m - mx);  // m == -inf -> 0
      l *= cf;
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] *= cf;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float p = exp2f(s[u] - mx);  // invalid positions: exp2(-inf) = 0
        l += p;
        acc[0] += p * bf16_lo(vv[u].x);
        acc[1] += p * bf16_hi(vv[u].x);
        acc[2] += p * bf16_lo(vv[u].y);
        acc[3] += p * bf16_hi(vv[u].y);
        acc[4] += p * bf16_lo(vv[u].z);
        acc[5] += p * bf16_hi(vv[u].z);
        acc[6] += p * bf16_lo(vv[u].w);
        acc[7] += p * bf16_hi(vv[u].w);
      }
      m = mx;
    }
  }
  sm_state[grp][lg][0] = m;
  sm_state[grp][lg][1] = l;
#pragma unroll
  for (int i = 0; i < 8; ++i) sm_state[grp][lg][2 + i] = acc[i];
  __syncthreads();
  // group j < gq finalises head j over its nph phases (groups j, j+gq, ...)
  if (grp < gq) {
    float M = -INFINITY;
    for (int f = 0; f < nph; ++f) M = fmaxf(M, sm_state[grp + f * gq][lg][0]);
    float L = 0.f, o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int f = 0; f < nph; ++f) {
      const float* stt = sm_state[grp + f * gq][lg];
      const float cw = (stt[0] == -INFINITY) ? 0.f : exp2f(stt[0] - M);
      L += stt[1] * cw;
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] += stt[2 + i] * cw;
    }
    if (nsplit == 1) {
      const float inv = 1.f / L;
      uint4 ov;
      ov.x = pack_bf16x2(o[0] * inv, o[1] * inv);
      ov.y = pack_bf16x2(o[2] * inv, o[3] * inv);
      ov.z = pack_bf16x2(o[4] * inv, o[5] * inv);
      ov.w = pack_bf16x2(o[6] * inv, o[7] * inv);
      *reinterpret_cast<uint4*>(a.out + (size_t)row * a.H * HD + (size_t)qh * HD + lg * 8) = ov;
    } else {
      // partial state: [(row_local * H + qh) * nsplit + split] -> (m, l, acc[HD])
      const size_t idx = ((size_t)rl * a.H + qh) * nsplit + split;
      float* st = a.ws + idx * (HD + 2);
      if (lg == 0) {
        st[0] = M;
        st[1] = L;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) st[2 + lg * 8 + i] = o[i];
    }
  }
}

// ---------------------------------------------------------------------------
// attn2: same CTA = (kv head, row, context split) grid, re-mapped for decode:
//  * every lane group (hd/8 lanes, 16 bytes of a K/V row each) owns whole
//    positions and computes ALL gq q-heads of the KV group against them, so a
//    K/V byte is read once per KV head for MHA and GQA alike (the old mapping
//    re-read the context per q-head group under GQA);
//  * the fused decode path keeps the row's own (rotated) k / v in registers and
//    substitutes them at position `cur` inside the loop -- same arithmetic
//    order as reading them back, but without the append -> __syncthreads ->
//    reload round trip before the first K/V load;
//  * groups merge by shuffles inside a warp, then across the 4 warps in smem.
template <int HD, int GQ, int U>
__global__ void __launch_bounds__(kAttnWarps * 32)
    attn2_kernel(const AttnArgs a, int nsplit, int chunk) {
  pdl_trigger();
  if (a.prefetch_pos > 0) {
    // The cached K/V before the newest position were written by earlier steps
    // (and the row metadata by the step's H2D copy): pull this CTA's share of
    // them towards L2 while the kernel producing q (the QKV GEMM) finishes.
    // 4 threads per position: K and V rows of this kv head, 2 x 128 B lines each.
    const int row = a.row_off + int(blockIdx.y);
    const int cur = a.row_pos[row];
    const int p0 = int(blockIdx.z) * chunk, p1 = min(cur, p0 + min(chunk, a.prefetch_pos));
    const size_t kvd = size_t(a.Hkv) * HD, pos_stride = 2 * kvd;
    const uint16_t* kb = a.kv + (size_t)a.row_slot[row] * a.max_ctx * pos_stride + (size_t)blockIdx.x * HD;
    const int part = threadIdx.x & 3;
    for (int p = p0 + int(threadIdx.x >> 2); p < p1; p += int(blockDim.x >> 2))
      prefetch_l2(kb + (size_t)p * pos_stride + (part >> 1) * kvd + (part & 1) * 64);
  }
  pdl_wait();
  constexpr int G = HD / 8;           // lanes per group
  constexpr int P = 32 / G;           // groups per warp
  constexpr int NG = kAttnWarps * P;  // groups per CTA
  extern __shared__ float sm2[];      // [kAttnWarps][GQ][G][10]
  const int hk = blockIdx.x, rl = blockIdx.y, split = blockIdx.z;
  const int row = a.row_off + rl;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lg = lane % G, pg = lane / G;
  const int grp = warp * P + pg;
  const int slot = a.row_slot[row];
  const int len = a.row_pos[row] + 1;
  const int cur = len - 1;
  const int p_begin = split * chunk;
  const int p_end = min(len, p_begin + chunk);
  const float qscale = a.scale * 1.4426950408889634f;
  const size_t kvd = size_t(a.Hkv) * HD;
  const size_t pos_stride = 2 * kvd;
  const uint16_t* kbase = a.kv + (size_t)slot * a.max_ctx * pos_stride + (size_t)hk * HD + lg * 8;
  const size_t qkv_ld = size_t(a.H + 2 * a.Hkv) * HD;
  const uint16_t* qrow = a.qkv + row * qkv_ld;
  const bool fused = a.rope != nullptr;
  const int hl = lg % (G / 2);
  const bool first_half = lg < G / 2;
  const float2* rp = fused ? a.rope + (size_t)cur * (HD / 2) + hl * 8 : nullptr;

  // rotate-half RoPE of 8 consecutive dims held by this lane (partner G/2 lanes away), bf16-rounded
  auto rope8 = [&](float (&x)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float other = __shfl_xor_sync(0xffffffffu, x[i], G / 2);
      const float2 cs = rp[i];
      const float r = first_half ? x[i] * cs.x - other * cs.y : x[i] * cs.x + other * cs.y;
      x[i] = bf16_to_f(f_to_bf16(r));
    }
  };
  auto load8 = [&](const uint16_t* src, float (&x)[8]) {
    const uint4 v = *reinterpret_cast<const uint4*>(src);
    x[0] = bf16_lo(v.x); x[1] = bf16_hi(v.x); x[2] = bf16_lo(v.y); x[3] = bf16_hi(v.y);
    x[4] = bf16_lo(v.z); x[5] = bf16_hi(v.z); x[6] = bf16_lo(v.w); x[7] = bf16_hi(v.w);
  };

  float q[GQ][8];
#pragma unroll
  for (int h = 0; h < GQ; ++h) {
    load8(qrow + (size_t)(hk * GQ + h) * HD + lg * 8, q[h]);
    if (fused) rope8(q[h]);
#pragma unroll
    for (int i = 0; i < 8; ++i) q[h][i] *= qscale;
  }
  // fused decode: this row's own k (rotated) and v, substituted at position cur
  uint4 kc = make_uint4(0, 0, 0, 0), vc = make_uint4(0, 0, 0, 0);
  const bool have_cur = fused && p_begin <= cur && cur < p_end;
  if (have_cur) {
    float k8[8];
    load8(qrow + (size_t)(a.H + hk) * HD + lg * 8, k8);
    rope8(k8);
    kc.x = pack_bf16x2(k8[0], k8[1]); kc.y = pack_bf16x2(k8[2], k8[3]);
    kc.z = pack_bf16x2(k8[4], k8[5]); kc.w = pack_bf16x2(k8[6], k8[7]);
    vc = *reinterpret_cast<const uint4*>(qrow + (size_t)(a.H + a.Hkv + hk) * HD + lg * 8);
    if (grp == 0) {  // append (rotated k, raw v) to the cache for the next steps
      uint16_t* kcp = const_cast<uint16_t*>(kbase) + (size_t)cur * pos_stride;
      *reinterpret_cast<uint4*>(kcp) = kc;
      *reinterpret_cast<uint4*>(kcp + kvd) = vc;
    }
  }

  float m[GQ], l[GQ], acc[GQ][8];
#pragma unroll
  for (int h = 0; h < GQ; ++h) {
    m[h] = -INFINITY;
    l[h] = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[h][i] = 0.f;
  }
  // warp-uniform trip count: a warp's groups start at grp = warp*P .. warp*P+P-1
  const int wbase = p_begin + warp * P;
  for (int pb = wbase; pb < p_end; pb += NG * U) {
    uint4 kk[U], vv[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int pos = pb + pg + u * NG;
      ok[u] = pos < p_end;
      if (ok[u] && fused && pos == cur) {
        kk[u] = kc;
        vv[u] = vc;
      } else if (ok[u]) {
        const uint16_t* kp = kbase + (size_t)pos * pos_stride;
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
    for (int h = 0; h < GQ; ++h) {
      float s[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        s[u] = q[h][0] * kf[u][0] + q[h][1] * kf[u][1] + q[h][2] * kf[u][2] + q[h][3] * kf[u][3] +
               q[h][4] * kf[u][4] + q[h][5] * kf[u][5] + q[h][6] * kf[u][6] + q[h][7] * kf[u][7];
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < U; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
      float mx = m[h];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!ok[u]) s[u] = -INFINITY;
        mx = fmaxf(mx, s[u]);
      }
      if (mx != -INFINITY) {
        const float cf = exp2f(m[h] - mx);
        l[h] *= cf;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[h][i] *= cf;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float pr = exp2f(s[u] - mx);
          l[h] += pr;
          acc[h][0] += pr * bf16_lo(vv[u].x);
          acc[h][1] += pr * bf16_hi(vv[u].x);
          acc[h][2] += pr * bf16_lo(vv[u].y);
          acc[h][3] += pr * bf16_hi(vv[u].y);
          acc[h][4] += pr * bf16_lo(vv[u].z);
          acc[h][5] += pr * bf16_hi(vv[u].z);
          acc[h][6] += pr * bf16_lo(vv[u].w);
          acc[h][7] += pr * bf16_hi(vv[u].w);
        }
        m[h] = mx;
      }
    }
  }
  // merge the P groups of a warp (lanes lg, lg+G, ...) with shuffles
#pragma unroll
  for (int h = 0; h < GQ; ++h) {
#pragma unroll
    for (int o = G; o < 32; o <<= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m[h], o);
      const float l2 = __shfl_xor_sync(0xffffffffu, l[h], o);
      const float M = fmaxf(m[h], m2);
      const float c1 = (m[h] == -INFINITY) ? 0.f : exp2f(m[h] - M);
      const float c2 = (m2 == -INFINITY) ? 0.f : exp2f(m2 - M);
      l[h] = l[h] * c1 + l2 * c2;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float a2 = __shfl_xor_sync(0xffffffffu, acc[h][i], o);
        acc[h][i] = acc[h][i] * c1 + a2 * c2;
      }
      m[h] = M;
    }
  }
  if (pg == 0) {
#pragma unroll
    for (int h = 0; h < GQ; ++h) {
      float* st = sm2 + ((warp * GQ + h) * G + lg) * 10;
      st[0] = m[h];
      st[1] = l[h];
#pragma unroll
      for (int i = 0; i < 8; ++i) st[2 + i] = acc[h][i];
    }
  }
  __syncthreads();
  // warp w finalises heads h = w, w + 4, ... over the 4 warps' states (lanes < G)
  if (pg == 0) {
    for (int h = warp; h < GQ; h += kAttnWarps) {
      float M = -INFINITY;
#pragma unroll
      for (int f = 0; f < kAttnWarps; ++f) M = fmaxf(M, sm2[((f * GQ + h) * G + lg) * 10]);
      float L = 0.f, o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int f = 0; f < kAttnWarps; ++f) {
        const float* stt = sm2 + ((f * GQ + h) * G + lg) * 10;
        const float cw = (stt[0] == -INFINITY) ? 0.f : exp2f(stt[0] - M);
        L += stt[1] * cw;
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] += stt[2 + i] * cw;
      }
      const int qh = hk * GQ + h;
      if (nsplit == 1) {
        const float inv = 1.f / L;
        uint4 ov;
        ov.x = pack_bf16x2(o[0] * inv, o[1] * inv);
        ov.y = pack_bf16x2(o[2] * inv, o[3] * inv);
        ov.z = pack_bf16x2(o[4] * inv, o[5] * inv);
        ov.w = pack_bf16x2(o[6] * inv, o[7] * inv);
        *reinterpret_cast<uint4*>(a.out + (size_t)row * a.H * HD + (size_t)qh * HD + lg * 8) = ov;
      } else {
        const size_t idx = ((size_t)rl * a.H + qh) * nsplit + split;
        float* st = a.ws + idx * (HD + 2);
        if (lg == 0) {
          st[0] = M;
          st[1] = L;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) st[2 + lg * 8 + i] = o[i];
      }
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

template <int HD>
static cudaError_t attention_hd(const AttnArgs& a_in, int num_sms, cudaStream_t st) {
  // positions per CTA warmed into L2 before the PDL wait (0 = none)
  static const int prefetch_pos = [] {
    const char* e = getenv("CB_ATTN_PREFETCH_POS");
    return e ? atoi(e) : 64;
  }();
  AttnArgs a = a_in;
  a.prefetch_pos = prefetch_pos;
  const int gq = a.H / a.Hkv;
  constexpr int NG = kAttnWarps * (32 / (HD / 8));
  if (gq < 1 || NG % gq != 0) return cudaErrorInvalidValue;
  int nsplit = 1;
  const long long ctas = (long long)a.T * a.Hkv;
  // enough CTAs to keep HBM busy: MHA needs 2 waves; a GQA CTA carries gq
  // heads' work, so aim for 8 waves of CTAs there
  const long long want = (gq > 1 ? 8LL : 2LL) * num_sms;
  const int min_chunk = gq > 1 ? 128 : 256;
  if (ctas < want && a.max_len > min_chunk) {
    nsplit = int((want + ctas - 1) / ctas);
    nsplit = min(nsplit, (a.max_len + min_chunk - 1) / min_chunk);
    nsplit = min(nsplit, 32);
    while (nsplit > 1 && (size_t)a.T * a.H * nsplit * (HD + 2) > a.ws_floats) --nsplit;
  }
  const int chunk = (a.max_len + nsplit - 1) / nsplit;
  static const int head_major = [] {
    const char* e = getenv("CB_ATTN_HEAD_MAJOR");
    return e ? atoi(e) : 1;
  }();
  const dim3 grid = head_major ? dim3(a.Hkv, a.T, nsplit) : dim3(a.T, a.Hkv, nsplit);
  // positions in flight per lane group: 4 when there are enough CTAs to fill
  // the GPU (measured best for decode batches), 8 for few long rows
  static const int forced = [] {
    const char* e = getenv("CB_ATTN_UNROLL");
    return e ? atoi(e) : 0;
  }();
  const long long total = ctas * nsplit;
  const int u = forced ? forced : (gq == 1 && total >= 8LL * num_sms ? 4 : 8);
  static const int v2 = [] {
    const char* e = getenv("CB_ATTN_V1");
    return e ? 0 : 1;
  }();
  cudaError_t e;
  if (v2) {
    const dim3 g2(a.Hkv, a.T, nsplit);
    const size_t sm = size_t(kAttnWarps) * gq * (HD / 8) * 10 * sizeof(float);
    switch (gq) {
      case 1: e = u == 8 ? launch_pdl(attn2_kernel<HD, 1, 8>, g2, dim3(kAttnWarps * 32), sm, st, a, nsplit, chunk)
                         : launch_pdl(attn2_kernel<HD, 1, 4>, g2, dim3(kAttnWarps * 32), sm, st, a, nsplit, chunk);
        break;
      case 2: e = launch_pdl(attn2_kernel<HD, 2, 4>, g2, dim3(kAttnWarps * 32), sm, st, a, nsplit, chunk); break;
      case 4: e = launch_pdl(attn2_kernel<HD, 4, 4>, g2, dim3(kAttnWarps * 32), sm, st, a, nsplit, chunk); break;
      case 8: e = launch_pdl(attn2_kernel<HD, 8, 2>, g2, dim3(kAttnWarps * 32), sm, st, a, nsplit, chunk); break;
      default: e = cudaErrorInvalidValue;
    }
  } else {
    e = u == 8 ? launch_pdl(attn_kernel<HD, 8>, grid, dim3(kAttnWarps * 32), 0, st, a, nsplit, chunk, gq, head_major)
               : launch_pdl(attn_kernel<HD, 4>, grid, dim3(kAttnWarps * 32), 0, st, a, nsplit, chunk, gq, head_major);
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
