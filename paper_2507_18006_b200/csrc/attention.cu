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
// for short batches with long context -- across context splits (the last
// split CTA of a (row, kv head) to arrive merges the partials, in split
// order).  Decode attention is HBM-bound: every K/V byte is read once.
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "kernels.h"

namespace cb {

static constexpr int kAttnWarps = 4;

// ---------------------------------------------------------------------------
// attn2: CTA = (kv head, row, context split) (head-major grid), 4 warps:
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
    const int ks = a.kv_map ? a.kv_map[a.row_slot[row]] : a.row_slot[row];
    const uint16_t* kb = a.kv + (size_t)ks * a.max_ctx * pos_stride + (size_t)blockIdx.x * HD;
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
  const int slot = a.kv_map ? a.kv_map[a.row_slot[row]] : a.row_slot[row];  // index in this KV block
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
  if (nsplit > 1) {
    // the last split CTA of (row, kv head) merges every split's partial state
    // (fixed split order: deterministic whatever the arrival order)
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      int* cnt = a.counters + (size_t)rl * a.Hkv + hk;
      s_last = atomicAdd(cnt, 1) == nsplit - 1;
      if (s_last) *cnt = 0;  // every split arrived: ready for the next launch
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      const int row = a.row_off + rl;
      for (int idx = threadIdx.x; idx < GQ * HD; idx += kAttnWarps * 32) {
        const int h = idx / HD, i = idx % HD;
        const int qh = hk * GQ + h;
        const float* st = a.ws + ((size_t)rl * a.H + qh) * nsplit * (HD + 2);
        float M = -INFINITY;
        for (int s = 0; s < nsplit; ++s) M = fmaxf(M, __ldcg(st + s * (HD + 2)));
        float L = 0.f, o = 0.f;
        for (int s = 0; s < nsplit; ++s) {
          const float ms = __ldcg(st + s * (HD + 2));
          const float c = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
          L += __ldcg(st + s * (HD + 2) + 1) * c;
          o += __ldcg(st + s * (HD + 2) + 2 + i) * c;
        }
        a.out[(size_t)row * a.H * HD + (size_t)qh * HD + i] = f_to_bf16(o / L);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// attn_tma: the same CTA, lane-group mapping and arithmetic as attn2 (hd 128,
// KV block in device memory; context splits on whole boxes, merged by the
// last split CTA as in attn2), with K and V fed by TMA:
// boxes of 32 cached positions x one head's 128 dims (8 KB each) from the
// [slot * max_ctx + pos][k | v] view of the block, four K+V stages per CTA
// (64 KB: three CTAs per SM; 2 x 64 positions, 3 x 64 and 8 x 32 measured
// slower, profiles/r02_attn_tma_ab.txt), the first ones issued before
// griddepcontrol.wait (cached positions < cur were written by earlier steps;
// the row's own k / v are substituted at `cur` as in attn2).  Bulk tensor
// loads read HBM at ~7 TB/s where 16-byte loads top out near 6.2
// (profiles/r02_read_bw.txt).  A group's positions and their order (chunks of
// U = 4) are attn2's, so the arithmetic matches attn2 with u = 4.
constexpr int kTmaPos = 32;
constexpr int kTmaStages = 4;

template <int GQ, int U>
__global__ void __launch_bounds__(kAttnWarps * 32)
    attn_tma_kernel(const __grid_constant__ CUtensorMap tkv, const AttnArgs a, int nsplit, int chunk) {
  constexpr int HD = 128;
  constexpr int G = HD / 8;           // lanes per group
  constexpr int P = 32 / G;           // groups per warp
  constexpr int NG = kAttnWarps * P;  // groups per CTA
  constexpr uint32_t kBoxBytes = kTmaPos * HD * 2;
  extern __shared__ __align__(1024) uint8_t smt[];
  uint16_t* ring = reinterpret_cast<uint16_t*>(smt);  // [stage][K | V][kTmaPos][HD]
  uint64_t* full = reinterpret_cast<uint64_t*>(smt + kTmaStages * 2 * kBoxBytes);
  uint64_t* empty = full + kTmaStages;
  float* sm2 = reinterpret_cast<float*>(empty + kTmaStages);  // [kAttnWarps][GQ][G][10]
  pdl_trigger();
  const int hk = blockIdx.x, rl = blockIdx.y, split = blockIdx.z;
  const int row = a.row_off + rl;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lg = lane % G, pg = lane / G;
  const int grp = warp * P + pg;
  const int slot = a.kv_map ? a.kv_map[a.row_slot[row]] : a.row_slot[row];
  const int len = a.row_pos[row] + 1;
  const int cur = len - 1;
  // this split's positions [p_begin, p_end) (chunk: a multiple of kTmaPos)
  const int p_begin = split * chunk;
  const int p_end = min(len, p_begin + chunk);
  const int box0 = p_begin / kTmaPos;
  const int nbox = p_end > p_begin ? (p_end - p_begin + kTmaPos - 1) / kTmaPos : 0;
  const size_t kvd = size_t(a.Hkv) * HD;
  const int prow = slot * a.max_ctx;  // view row of position 0
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tkv);
    for (int i = 0; i < kTmaStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kAttnWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();  // every K / V byte is read once per step
  auto issue = [&](int b) {
    const int st = b % kTmaStages;
    uint16_t* kd = ring + size_t(st) * 2 * kTmaPos * HD;
    mbar_arrive_expect_tx(&full[st], 2 * kBoxBytes);
    tma_load_2d(&tkv, &full[st], kd, hk * HD, prow + (box0 + b) * kTmaPos, pol);
    tma_load_2d(&tkv, &full[st], kd + kTmaPos * HD, int(kvd) + hk * HD, prow + (box0 + b) * kTmaPos, pol);
  };
  if (threadIdx.x == 0)
    for (int b = 0; b < nbox && b < kTmaStages; ++b) issue(b);
  pdl_wait();

  const float qscale = a.scale * 1.4426950408889634f;
  const size_t pos_stride = 2 * kvd;
  const size_t qkv_ld = size_t(a.H + 2 * a.Hkv) * HD;
  const uint16_t* qrow = a.qkv + row * qkv_ld;
  const int hl = lg % (G / 2);
  const bool first_half = lg < G / 2;
  const float2* rp = a.rope + (size_t)cur * (HD / 2) + hl * 8;
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
    rope8(q[h]);
#pragma unroll
    for (int i = 0; i < 8; ++i) q[h][i] *= qscale;
  }
  uint4 kc = make_uint4(0, 0, 0, 0), vc = make_uint4(0, 0, 0, 0);
  if (p_begin <= cur && cur < p_end) {
    float k8[8];
    load8(qrow + (size_t)(a.H + hk) * HD + lg * 8, k8);
    rope8(k8);
    kc.x = pack_bf16x2(k8[0], k8[1]); kc.y = pack_bf16x2(k8[2], k8[3]);
    kc.z = pack_bf16x2(k8[4], k8[5]); kc.w = pack_bf16x2(k8[6], k8[7]);
    vc = *reinterpret_cast<const uint4*>(qrow + (size_t)(a.H + a.Hkv + hk) * HD + lg * 8);
    if (grp == 0) {  // append (rotated k, raw v) to the cache for the next steps
      uint16_t* kcp = const_cast<uint16_t*>(a.kv) + ((size_t)slot * a.max_ctx + cur) * pos_stride + hk * HD + lg * 8;
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
  for (int b = 0; b < nbox; ++b) {
    const int st = b % kTmaStages;
    mbar_wait(&full[st], uint32_t(b / kTmaStages) & 1u);
    const uint16_t* ks = ring + size_t(st) * 2 * kTmaPos * HD;
    const uint16_t* vs = ks + kTmaPos * HD;
    const int p0 = (box0 + b) * kTmaPos;
#pragma unroll
    for (int j0 = 0; j0 < kTmaPos / NG; j0 += U) {
      uint4 kk[U], vv[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = grp + (j0 + u) * NG;  // row of the box
        const int pos = p0 + r;
        ok[u] = pos < p_end;
        if (!ok[u]) {  // (stale or out-of-range rows may hold non-finite bytes: 0 * NaN)
          kk[u] = make_uint4(0, 0, 0, 0);
          vv[u] = make_uint4(0, 0, 0, 0);
        } else if (pos == cur) {
          kk[u] = kc;
          vv[u] = vc;
        } else {
          kk[u] = *reinterpret_cast<const uint4*>(ks + r * HD + lg * 8);
          vv[u] = *reinterpret_cast<const uint4*>(vs + r * HD + lg * 8);
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
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (threadIdx.x == 0 && b + kTmaStages < nbox) {
      mbar_wait(&empty[st], uint32_t(b / kTmaStages) & 1u);  // every warp read stage st
      issue(b + kTmaStages);
    }
  }
  // merge the P groups of a warp, then the warps (as attn2)
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
      float* stt = sm2 + ((warp * GQ + h) * G + lg) * 10;
      stt[0] = m[h];
      stt[1] = l[h];
#pragma unroll
      for (int i = 0; i < 8; ++i) stt[2 + i] = acc[h][i];
    }
  }
  __syncthreads();
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
        float* stt = a.ws + (((size_t)rl * a.H + qh) * nsplit + split) * (HD + 2);
        if (lg == 0) {
          stt[0] = M;
          stt[1] = L;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) stt[2 + lg * 8 + i] = o[i];
      }
    }
  }
  if (nsplit > 1) {  // the last split CTA of (row, kv head) merges, in split order (as attn2)
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      int* cnt = a.counters + (size_t)rl * a.Hkv + hk;
      s_last = atomicAdd(cnt, 1) == nsplit - 1;
      if (s_last) *cnt = 0;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      for (int idx = threadIdx.x; idx < GQ * HD; idx += kAttnWarps * 32) {
        const int h = idx / HD, i = idx % HD;
        const int qh = hk * GQ + h;
        const float* st = a.ws + ((size_t)rl * a.H + qh) * nsplit * (HD + 2);
        float M = -INFINITY;
        for (int sp = 0; sp < nsplit; ++sp) M = fmaxf(M, __ldcg(st + sp * (HD + 2)));
        float L = 0.f, o = 0.f;
        for (int sp = 0; sp < nsplit; ++sp) {
          const float ms = __ldcg(st + sp * (HD + 2));
          const float c = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
          L += __ldcg(st + sp * (HD + 2) + 1) * c;
          o += __ldcg(st + sp * (HD + 2) + 2 + i) * c;
        }
        a.out[(size_t)row * a.H * HD + (size_t)qh * HD + i] = f_to_bf16(o / L);
      }
    }
  }
}

// [slot * max_ctx + pos][2 * Hkv * 128] bf16 view of a device KV block, boxes
// of kTmaPos positions x one head's 128 dims (cached per block)
static bool kv_tma_map(const AttnArgs& a, CUtensorMap* out) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int>, CUtensorMap> cache;
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(static_cast<const void*>(a.kv), a.kv_slots, a.max_ctx, a.Hkv);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;  // (by value: the cache may be cleared by a later call)
    return true;
  }
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const uint64_t cols = uint64_t(2) * a.Hkv * 128;
  cuuint64_t dims[2] = {cols, uint64_t(a.kv_slots) * a.max_ctx};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {128, uint32_t(kTmaPos)};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMap m;
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(a.kv), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (cache.size() > 4096) cache.clear();
  cache[key] = m;
  *out = m;
  return true;
}

template <int GQ, int U = 4>
static cudaError_t launch_attn_tma(const CUtensorMap& tm, const AttnArgs& a, int nsplit, int chunk,
                                   cudaStream_t st) {
  const size_t smem = size_t(kTmaStages) * 2 * kTmaPos * 128 * 2 + 2 * kTmaStages * 8 +
                      size_t(kAttnWarps) * GQ * 16 * 10 * sizeof(float);
  static bool attr[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(attn_tma_kernel<GQ, U>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    attr[dev & 63] = true;
  }
  return launch_pdl(attn_tma_kernel<GQ, U>, dim3(a.Hkv, a.T, nsplit), dim3(kAttnWarps * 32), smem, st, tm, a,
                    nsplit, chunk);
}

template <int HD>
static cudaError_t attention_hd(const AttnArgs& a_in, int num_sms, cudaStream_t st) {
  // positions per CTA warmed into L2 before the PDL wait (-1.6% per B=256
  // step, profiles/r01_attn_prefetch_ab.txt)
  AttnArgs a = a_in;
  a.prefetch_pos = 64;
  const int gq = a.H / a.Hkv;
  constexpr int NG = kAttnWarps * (32 / (HD / 8));
  if (gq < 1 || NG % gq != 0) return cudaErrorInvalidValue;
  int nsplit = 1;
  // the split is decided from the rows of the whole pass (kind_T), so a
  // replica's share of the rows splits its contexts exactly like the
  // unreplicated pass (same summation order: replication stays bit-identical)
  const long long ctas = (long long)(a.kind_T > 0 ? a.kind_T : a.T) * a.Hkv;
  // enough CTAs to keep HBM busy: MHA needs 2 waves; a GQA CTA carries gq
  // heads' work, so aim for 8 waves of CTAs there.  The merge runs in the last
  // split CTA (no second launch), so short chunks only cost partial traffic.
  const long long want = (gq > 1 ? 8LL : 2LL) * num_sms;
  const int min_chunk = gq > 1 ? 128 : 64;
  if (ctas < want && a.max_len > min_chunk) {
    nsplit = int((want + ctas - 1) / ctas);
    nsplit = min(nsplit, (a.max_len + min_chunk - 1) / min_chunk);
    nsplit = min(nsplit, 32);
    while (nsplit > 1 && (size_t)a.T * a.H * nsplit * (HD + 2) > a.ws_floats) --nsplit;
    if (!a.counters) nsplit = 1;  // (the merge needs the arrival counters)
  }
  const int chunk = (a.max_len + nsplit - 1) / nsplit;
  // positions in flight per lane group: 4 when there are enough CTAs to fill
  // the GPU (measured best for decode batches), 8 for few long rows
  const long long total = ctas * nsplit;
  const int u = gq == 1 && total >= 8LL * num_sms ? 4 : 8;
  // hd 128, device-memory KV (kv_slots set by the runtime): the TMA-fed
  // kernel; the plan depends on kind_T and the block only, so replicas of a
  // layer run the same kernel as the unreplicated pass
  if (HD == 128 && a.rope && a.kv_slots > 0 && (gq == 1 || gq == 2 || gq == 4 || gq == 8)) {
    CUtensorMap tm;
    if (kv_tma_map(a, &tm)) {
      // context splits on whole boxes
      const int tchunk = (chunk + kTmaPos - 1) / kTmaPos * kTmaPos;
      const int tsplit = (a.max_len + tchunk - 1) / tchunk;
      switch (gq) {
        case 1: return launch_attn_tma<1>(tm, a, tsplit, tchunk, st);
        case 2: return launch_attn_tma<2>(tm, a, tsplit, tchunk, st);
        case 4: return launch_attn_tma<4>(tm, a, tsplit, tchunk, st);
        case 8: return launch_attn_tma<8, 2>(tm, a, tsplit, tchunk, st);  // (attn2's 2 positions per step at gq 8)
      }
    }
  }
  cudaError_t e;
  {
    const dim3 g2(a.Hkv, a.T, nsplit);  // head-major grid
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
  }
  return e;
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
