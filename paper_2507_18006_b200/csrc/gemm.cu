// tcgen05 / TMEM / TMA GEMM for the decoder-layer projections (sm_100a).
//
//   out[t, n] (op)= sum_k X[row_off + t, k] * W[n, k]        t < T, n < N
//
// W is a PyTorch-layout weight [N, K] (K contiguous), X the activation rows
// [rows, K].  Both are K-major, the native tcgen05 operand layout.  The MMA's
// M dimension is the weight rows (128 per CTA) and its N dimension the tokens
// ("swap-AB"), so a decode step with a handful of rows still drives the tensor
// pipe while the kernel streams the weight at HBM rate (decode
// GEMMs are HBM-bound, prefill GEMMs tensor-bound).
//
// Two kernels share the warp roles and the epilogue:
//  * gemm_tc_kernel<TN>  -- 1 CTA per 128 weight rows x TN tokens (T <= 128);
//  * gemm_tc2_kernel<TNP> -- CTA pair (tcgen05 cta_group::2): 256 weight rows x
//    TNP tokens per pair, each CTA stages 128 weight rows and TNP/2 token rows,
//    so the activation bytes read from L2 per weight byte halve (T > 128).
// Work split: persistent stream-K over (tile, k-block) units -- one contiguous
// range per CTA (pair), so every SM streams weight bytes for the whole launch --
// or, for few wide-K tiles, cluster split-K with a DSMEM reduction.  A tile
// split across CTAs is finished by the last CTA to arrive, summing the parts in
// fixed CTA order: deterministic, and for T <= one token tile the split points
// do not depend on T, so a row's result is identical whether it runs
// unreplicated or inside a replica's micro-batch (ops.py:151-158).
//
// Warp roles (224 threads): warp 0 = TMA producer of the weight ring (filled
// before griddepcontrol.wait: weights do not depend on the previous kernel),
// warp 1 = TMEM owner + MMA issuer (converged warp, elect.sync picks the issuing
// lane), warps 2..5 = epilogue (TMEM -> registers -> smem transpose -> 16-byte
// global stores), warp 6 = TMA producer of the activation ring.  TMEM
// accumulators are double buffered so a tile's epilogue overlaps the next
// tile's main loop.
//
// Stand-in replaced: reference `_kernels._work_units` (`_kernels.py:17-38`) and
// the per-module GEMM FLOPs of `ModuleCatalog.from_model` (`domain.py:241-264`).
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "kernels.h"

namespace cb {

static constexpr int kBM = 128;          // weight rows per CTA tile (UMMA M per CTA)
static constexpr int kBK = 64;           // k-block: 64 bf16 = one 128-byte swizzle row
static constexpr int kThreads1 = 224;    // TMA weights, MMA, 4 epilogue warps, TMA activations
static constexpr int kEpiThreads = 128;
static constexpr size_t kSmemBudget = 224 * 1024;  // of the 227 KB opt-in maximum
static constexpr int kTbRow = 36;  // transpose buffer row stride (floats): 32 + 4 pad -> conflict-free 16-byte reads
static constexpr int kChunkBytes = 16 * 32 * 4;  // one epilogue warp chunk: 16 tokens x 32 weight rows, fp32
// per epilogue warp: padded transpose buffer (register-store path) + 2 TMA staging chunks
// (staging first and the per-warp block a multiple of 1 KB: the swizzled
// staging boxes of the token-major epilogue need 512-byte alignment)
static constexpr int kEpiWarpBytes = ((2 * kChunkBytes + 16 * kTbRow * 4) + 1023) / 1024 * 1024;
static constexpr int kTbufBytes = 4 * kEpiWarpBytes;
static constexpr int kMaxStages = 16;
// after the transpose buffers: mbarriers (first 1 KB), then the fused-RMSNorm
// row-scale table (256 fp32, one per token row of the CTA's token tile)
static constexpr int kBarBytes = 2048;
static constexpr int kRtabOff = 1024;
static constexpr int kMaxNormRows = 256;

template <int WB, int XB>
struct RingCfg {
  static constexpr int kWBytes = WB;
  static constexpr int kXBytes = XB;
  static constexpr int kStageBytes = WB + XB;
  static constexpr int kStagesRaw = int((kSmemBudget - 1024 - kBarBytes - kTbufBytes) / kStageBytes);
  static constexpr int kStages = kStagesRaw > kMaxStages ? kMaxStages : kStagesRaw;
  static constexpr int kRingBytes = kStages * kStageBytes;
  // ring | transpose buffers | barriers
  static constexpr size_t kSmemBytes = size_t(kRingBytes) + kTbufBytes + 1024 /*align slack*/ + kBarBytes;
};
template <int TN, int KD = 1>
struct GemmCfg : RingCfg<kBM * kBK * 2 * KD, TN * kBK * 2 * KD> {
  // accumulators: [0, 2TN) double buffer for whole tiles, then (TN <= 128) two
  // retained partial tiles for cluster stream-K: [2TN, 3TN) first, [3TN, 4TN) last
  static constexpr uint32_t kAccCols = TN <= 128 ? 4 * TN : 2 * TN;
  static constexpr uint32_t kTmemCols = (kAccCols <= 32)    ? 32
                                        : (kAccCols <= 64)  ? 64
                                        : (kAccCols <= 128) ? 128
                                        : (kAccCols <= 256) ? 256
                                                            : 512;
};
template <int TNP, int KD = 1>
struct PairCfg : RingCfg<kBM * kBK * 2 * KD, (TNP / 2) * kBK * 2 * KD> {
  static constexpr uint32_t kTmemCols = 2 * TNP <= 256 ? 256 : 512;
};

struct StreamK {
  int units, grid, kb;
  CB_DEVICE int u0(int c) const { return int((long long)c * units / grid); }
  CB_DEVICE int cta_of(int u) const { return int(((long long)(u + 1) * grid - 1) / units); }
};

// ------------------------------------------------------------------ epilogue
// SwiGLU: silu(gate) * up.  Fast divide: an IEEE divide by the huge 1 + exp(-g)
// of a very negative gate takes the slow path (measured 3x slower epilogue);
// __fdividef returns the correct limit 0 there.  Every epilogue path uses this
// one function, so a row's bits do not depend on which path finished its tile.
CB_DEVICE float silu_mul(float g, float u) { return __fdividef(g, 1.0f + __expf(-g)) * u; }

// Scalar fallback (shapes whose outputs are not 16-byte aligned): 16 token
// columns of weight row n.
CB_DEVICE void emit16(const GemmArgs& a, int n, int row0, int ncols, const float (&v)[16]) {
  const int lane = threadIdx.x & 31;
  if (a.epi == EPI_SWIGLU) {
    // rows are interleaved gate/up pairs: even row = gate_j, odd row = up_j.
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float other = __shfl_xor_sync(0xffffffffu, v[i], 1);
      if (!(lane & 1) && n < a.N && i < ncols) {
        reinterpret_cast<uint16_t*>(a.out)[(size_t)(row0 + i) * a.ldo + (n >> 1)] = f_to_bf16(silu_mul(v[i], other));
      }
    }
    return;
  }
  if (n >= a.N) return;
  if (a.epi == EPI_BF16) {
    uint16_t* o = reinterpret_cast<uint16_t*>(a.out);
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < ncols) o[(size_t)(row0 + i) * a.ldo + n] = f_to_bf16(v[i]);
  } else if (a.epi == EPI_F32) {
    float* o = reinterpret_cast<float*>(a.out);
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < ncols) o[(size_t)(row0 + i) * a.ldo + n] = v[i];
  } else {  // EPI_RESID: fp32 residual stream += projection
    float* o = reinterpret_cast<float*>(a.out);
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < ncols) {
        size_t idx = (size_t)(row0 + i) * a.ldo + n;
        o[idx] = o[idx] + v[i];
      }
  }
}

// Scalar: weight rows n, n+1 (an interleaved gate/up pair for SwiGLU) of token `row`.
CB_DEVICE void emit_pair(const GemmArgs& a, int n, int row, float v0, float v1) {
  if (n >= a.N) return;
  const size_t base = (size_t)row * a.ldo;
  if (a.epi == EPI_SWIGLU) {
    reinterpret_cast<uint16_t*>(a.out)[base + (n >> 1)] = f_to_bf16(silu_mul(v0, v1));
  } else if (a.epi == EPI_BF16) {
    uint16_t* o = reinterpret_cast<uint16_t*>(a.out) + base + n;
    if (n + 1 < a.N) {
      *reinterpret_cast<uint32_t*>(o) = pack_bf16x2(v0, v1);
    } else {
      o[0] = f_to_bf16(v0);
    }
  } else if (a.epi == EPI_F32) {
    float* o = reinterpret_cast<float*>(a.out) + base + n;
    o[0] = v0;
    if (n + 1 < a.N) o[1] = v1;
  } else {
    float* o = reinterpret_cast<float*>(a.out) + base + n;
    o[0] += v0;
    if (n + 1 < a.N) o[1] += v1;
  }
}


// Vector: weight rows n0..n0+7 (n0 % 8 == 0) of token `row`, one 16-byte store
// (8-byte for SwiGLU, 2 x 16 bytes for fp32 outputs).  For EPI_RESID the
// caller passes the residual already loaded (res): loads of a batch are issued
// before its stores, since a store may alias a later load in the compiler's view.
CB_DEVICE float* out_f32(const GemmArgs& a, int n0, int row) {
  return reinterpret_cast<float*>(a.out) + (size_t)row * a.ldo + n0;
}
CB_DEVICE void emit8(const GemmArgs& a, int n0, int row, const float (&s)[8], const float4* res = nullptr) {
  if (n0 >= a.N) return;
  const size_t base = (size_t)row * a.ldo;
  if (a.epi == EPI_BF16) {
    uint4 o;
    o.x = pack_bf16x2(s[0], s[1]);
    o.y = pack_bf16x2(s[2], s[3]);
    o.z = pack_bf16x2(s[4], s[5]);
    o.w = pack_bf16x2(s[6], s[7]);
    *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(a.out) + base + n0) = o;
  } else if (a.epi == EPI_SWIGLU) {
    uint2 o;
    o.x = pack_bf16x2(silu_mul(s[0], s[1]), silu_mul(s[2], s[3]));
    o.y = pack_bf16x2(silu_mul(s[4], s[5]), silu_mul(s[6], s[7]));
    *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(a.out) + base + (n0 >> 1)) = o;
  } else {
    float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + base + n0);
    float4 x0 = make_float4(s[0], s[1], s[2], s[3]), x1 = make_float4(s[4], s[5], s[6], s[7]);
    if (a.epi == EPI_RESID) {
      const float4 y0 = res[0], y1 = res[1];
      x0 = make_float4(y0.x + x0.x, y0.y + x0.y, y0.z + x0.z, y0.w + x0.w);
      x1 = make_float4(y1.x + x1.x, y1.y + x1.y, y1.z + x1.z, y1.w + x1.w);
    }
    o[0] = x0;
    o[1] = x1;
  }
}

CB_DEVICE void load8(const float* src, float (&s)[8]) {
  const float4 x0 = *reinterpret_cast<const float4*>(src);
  const float4 x1 = *reinterpret_cast<const float4*>(src + 4);
  s[0] = x0.x; s[1] = x0.y; s[2] = x0.z; s[3] = x0.w;
  s[4] = x1.x; s[5] = x1.y; s[6] = x1.z; s[7] = x1.w;
}

// One warp's 32 weight rows (lane = row) x 16 token columns, transposed through
// the warp's smem buffer so every lane stores whole 16-byte runs of one token
// row: 2 store instructions per chunk instead of 16 scalar ones.
// Residual rows of one warp chunk in the fp32 store mapping: lane -> (token
// p*4 + lane/8, 4 features at (lane%8)*4).
CB_DEVICE void load_res(const GemmArgs& a, int nw0, int row, int nc, int lane, float4 (&res)[4]) {
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int i = p * 4 + (lane >> 3), f0 = (lane & 7) * 4;
    res[p] = (i < nc && nw0 + f0 < a.N) ? __ldcg(reinterpret_cast<const float4*>(out_f32(a, nw0 + f0, row + i)))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

CB_DEVICE void emit_warp_vec(const GemmArgs& a, float* tb, int nw0, int row, int nc, const float (&v)[16],
                             int lane, const float4* res_pre = nullptr, const uint2* g_pre = nullptr) {
  // fp32 outputs: residual loads issued first (or prefetched by the caller)
  float4 res[4];
  if (a.epi == EPI_RESID) {
    if (res_pre) {
#pragma unroll
      for (int p = 0; p < 4; ++p) res[p] = res_pre[p];
    } else {
      load_res(a, nw0, row, nc, lane, res);
    }
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) tb[i * kTbRow + lane] = v[i];
  __syncwarp();
  if (a.epi == EPI_SWIGLU) {
    const int i = lane >> 1, f0 = (lane & 1) * 16;
    if (i < nc) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float s[8];
        load8(tb + i * kTbRow + f0 + 8 * h, s);
        emit8(a, nw0 + f0 + 8 * h, row + i, s);
      }
    }
  } else if (a.epi == EPI_BF16) {
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int i = p * 8 + (lane >> 2), f0 = (lane & 3) * 8;
      if (i < nc) {
        float s[8];
        load8(tb + i * kTbRow + f0, s);
        emit8(a, nw0 + f0, row + i, s);
      }
    }
  } else {
    float ss[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int i = p * 4 + (lane >> 3), f0 = (lane & 7) * 4;
      ss[p] = 0.f;
      if (i < nc && nw0 + f0 < a.N) {
        float4 x = *reinterpret_cast<const float4*>(tb + i * kTbRow + f0);
        if (a.epi == EPI_RESID) x = make_float4(res[p].x + x.x, res[p].y + x.y, res[p].z + x.z, res[p].w + x.w);
        *reinterpret_cast<float4*>(out_f32(a, nw0 + f0, row + i)) = x;
        if (a.h_out) {  // fused RMSNorm producer: h' = bf16(x * gamma), partial sum of squares
          const uint2 g = g_pre ? *g_pre : *reinterpret_cast<const uint2*>(a.gamma_next + nw0 + f0);
          uint2 h;
          h.x = pack_bf16x2(x.x * bf16_lo(g.x), x.y * bf16_hi(g.x));
          h.y = pack_bf16x2(x.z * bf16_lo(g.y), x.w * bf16_hi(g.y));
          *reinterpret_cast<uint2*>(a.h_out + (size_t)(row + i) * a.ldo + nw0 + f0) = h;
          ss[p] = x.x * x.x + x.y * x.y + x.z * x.z + x.w * x.w;
        }
      }
    }
    if (a.h_out) {
      // the 8 lanes of token i hold its 32 features: xor tree (fixed order)
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        float t = ss[p];
        t += __shfl_xor_sync(0xffffffffu, t, 1);
        t += __shfl_xor_sync(0xffffffffu, t, 2);
        t += __shfl_xor_sync(0xffffffffu, t, 4);
        const int i = p * 4 + (lane >> 3);
        if ((lane & 7) == 0 && i < nc) a.ssq_out[(size_t)(row + i) * a.ssq_np + (nw0 >> 5)] = t;
      }
    }
  }
  __syncwarp();
}

// Per epilogue warp state: transpose buffer, two TMA staging chunks.
struct EpiWarp {
  float* tb;    // padded [16][kTbRow] fp32 (register-store path)
  uint8_t* st;  // 2 x kChunkBytes staging for TMA stores / bulk partial stores
  int sb;       // staging chunk to use next
  int q, lane;
  const float* rt;  // fused RMSNorm consumer: per-row scale table (index row - row_off), else null
  CB_DEVICE EpiWarp(uint8_t* base, int q_, int lane_, const float* rt_)
      : tb(reinterpret_cast<float*>(base + 2 * kChunkBytes)), st(base), sb(0), q(q_), lane(lane_), rt(rt_) {}
  // a staging chunk whose previous TMA store has finished reading it
  CB_DEVICE uint8_t* next_stage() {
    uint8_t* p = st + sb * kChunkBytes;
    if (lane == 0) bulk_wait_read<1>();
    __syncwarp();
    sb ^= 1;
    return p;
  }
  // 3-deep staging ring over the whole per-warp block (token-major epilogue:
  // the transpose buffer is unused there)
  CB_DEVICE uint8_t* next_stage3() {
    uint8_t* p = st + sb * kChunkBytes;
    if (lane == 0) bulk_wait_read<2>();
    __syncwarp();
    sb = sb == 2 ? 0 : sb + 1;
    return p;
  }
  CB_DEVICE void drain() {
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }
};
static_assert(3 * kChunkBytes <= kEpiWarpBytes, "token-major staging ring");
static constexpr int kTokEpiWarpBytes = 3 * kChunkBytes;  // token-major kernel: the staging ring only
static constexpr size_t kMaxDynSmem = 227 * 1024;         // sm_100 opt-in maximum per CTA

// Fused RMSNorm consumer: the epilogue warps turn the producer's per-row
// partial sums of squares into row scales rsqrt(mean(x^2) + eps), once per CTA
// (after griddepcontrol.wait: the partials belong to the previous kernel).
// Same summation order in every kernel, so a row's scale is bit-identical
// whichever kernel / plan consumes it.
CB_DEVICE const float* build_row_scales(const GemmArgs& a, uint8_t* bar_base, int et) {
  if (!a.ssq_in) return nullptr;
  float* rt = reinterpret_cast<float*>(bar_base + kRtabOff);
  const float inv_d = 1.0f / float(a.norm_d);
  const int w = et >> 5, l = et & 31, nv = a.ssq_np >> 2;
  // warp w: rows 64i + 16w + j (j < 16) -- 16 independent 16-byte loads in
  // flight per lane, lanes stride a row's partials, fixed xor-tree reduction
  for (int t0 = 16 * w; t0 < a.T; t0 += 64) {
    float s[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) s[j] = 0.f;
    for (int k = l; k - l < nv; k += 32) {  // one 16-byte load per row in flight at once
      float4 x[16];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        x[j] = (t0 + j < a.T && k < nv)
                   ? __ldcg(reinterpret_cast<const float4*>(a.ssq_in + (size_t)(a.row_off + t0 + j) * a.ssq_np) + k)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 16; ++j) s[j] += (x[j].x + x[j].y) + (x[j].z + x[j].w);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) s[j] += __shfl_xor_sync(0xffffffffu, s[j], o);
    }
    if (l < 16 && t0 + l < a.T) {
      float v = s[0];
#pragma unroll
      for (int j = 1; j < 16; ++j) v = (l == j) ? s[j] : v;
      rt[t0 + l] = rsqrtf(v * inv_d + a.norm_eps);
    }
  }
  named_bar_sync(1, kEpiThreads);
  return rt;
}

// the table build_row_scales filled (reduction passes after the main epilogue)
CB_DEVICE const float* row_scales(const GemmArgs& a, uint8_t* bar_base) {
  return a.ssq_in ? reinterpret_cast<const float*>(bar_base + kRtabOff) : nullptr;
}

// One warp chunk of output: weight rows nw0..nw0+31 (lane = row) x tokens
// row..row+nc-1 (register i = token).  Full chunks go through smem and one TMA
// store (EPI_RESID: TMA reduce-add = the fp32 residual +=) issued by lane 0 --
// the LSU never sees the output; a partial chunk (token tail) uses 16-byte
// register stores (or scalar ones for unaligned shapes).
CB_DEVICE void emit_chunk(const GemmArgs& a, const CUtensorMap* tmO, EpiWarp& e, int nw0, int row, int nc,
                          const float (&v_in)[16], const float4* res_pre = nullptr,
                          const uint2* g_pre = nullptr) {
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = e.rt ? v_in[i] * e.rt[row - a.row_off + i] : v_in[i];
  if (a.tma && nc == 16 && !a.h_out) {
    uint8_t* stg = e.next_stage();
    if (a.epi == EPI_SWIGLU) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float other = __shfl_xor_sync(0xffffffffu, v[i], 1);
        if (!(e.lane & 1)) reinterpret_cast<uint16_t*>(stg)[i * 16 + (e.lane >> 1)] = f_to_bf16(silu_mul(v[i], other));
      }
    } else if (a.epi == EPI_BF16) {
#pragma unroll
      for (int i = 0; i < 16; ++i) reinterpret_cast<uint16_t*>(stg)[i * 32 + e.lane] = f_to_bf16(v[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) reinterpret_cast<float*>(stg)[i * 32 + e.lane] = v[i];
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (e.lane == 0) {
      const int x = a.epi == EPI_SWIGLU ? (nw0 >> 1) : nw0;
      if (a.epi == EPI_RESID)
        tma_reduce_add_2d(tmO, stg, x, row);
      else
        tma_store_2d(tmO, stg, x, row);
      bulk_commit();
    }
    return;
  }
  if (a.vec)
    emit_warp_vec(a, e.tb, nw0, row, nc, v, e.lane, res_pre, g_pre);
  else
    emit16(a, nw0 + e.lane, row, nc, v);
}

// Partial tiles (stream-K / split-K): fp32, chunk-major [ncol/16][4 warps][16][32]
// so every warp chunk is one contiguous 2 KB block -- written with one bulk
// store from smem, summed by the finisher with one bulk load per part.
CB_DEVICE size_t part_chunk(int c0, int q) { return size_t((c0 >> 4) * 4 + q) * (kChunkBytes / 4); }

CB_DEVICE void write_part_chunk(EpiWarp& e, float* gdst, const float (&v)[16]) {
  uint8_t* stg = e.next_stage();
#pragma unroll
  for (int i = 0; i < 16; ++i) reinterpret_cast<float*>(stg)[i * 32 + e.lane] = v[i];
  fence_proxy_async_smem();
  __syncwarp();
  if (e.lane == 0) {
    bulk_s2g(gdst, stg, kChunkBytes);
    bulk_commit();
  }
}

// TMEM accumulator (this warp's 32 lanes) -> output (whole tile) or partial
// (global workspace, or -- cluster split-K -- this CTA's shared memory).
CB_DEVICE void epi_drain(const GemmArgs& a, const CUtensorMap* tmO, EpiWarp& e, uint32_t t_addr, int m0, int row0,
                         int ncols, bool whole, float* part, bool part_in_smem) {
  for (int c0 = 0; c0 < ncols; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(t_addr + uint32_t(c0), r);
    tmem_ld_wait();
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
    if (a.dbg & 16) continue;  // experiments: TMEM loads only
    if (whole) {
      emit_chunk(a, tmO, e, m0 + e.q * 32, row0 + c0, min(16, ncols - c0), v);
    } else if (part_in_smem) {
      float* pc = part + part_chunk(c0, e.q);
#pragma unroll
      for (int i = 0; i < 16; ++i) pc[i * 32 + e.lane] = v[i];
    } else {
      write_part_chunk(e, part + part_chunk(c0, e.q), v);
    }
  }
}

// Where the parts of a split tile live: CTA (or pair) cc's slot for `tile`.
struct PartMap {
  const float* ws;
  StreamK sk;
  int tile, cstride, coff, tn;
  CB_DEVICE const float* of(int cc) const {
    const int w = (sk.u0(cc) / sk.kb == tile) ? 0 : 1;  // slot 0 = the CTA's first segment
    return ws + ((size_t)(cc * cstride + coff) * 2 + w) * (size_t)(kBM * tn);
  }
};

// Stream-K fixup of one (tile, 128-row half): every CTA wrote its part; the
// last to arrive sums all parts in CTA order (deterministic, independent of
// who finishes) and emits the tile like a whole one.  When that CTA has
// finished its whole range (ring_idle) the parts are bulk-copied into its idle
// stage ring, one round per ring-full; otherwise they are read from L2.
CB_DEVICE void epi_fixup(const GemmArgs& a, const CUtensorMap* tmO, EpiWarp& e, int* counter, const PartMap& pm,
                         int c_first, int c_last, int m0, int row0, int ncols, bool ring_idle, uint8_t* ring,
                         uint32_t ring_bytes, uint64_t* fix_bar, uint32_t& fix_phase, int* bcast, int et,
                         unsigned long long* tr = nullptr) {
  const int nparts = c_last - c_first + 1;
  e.drain();  // this warp's bulk partial stores have landed
  fence_proxy_async_global();
  __threadfence();
  named_bar_sync(1, kEpiThreads);
  if (et == 0) {
    const int prev = atomicAdd(counter, 1);
    *bcast = (prev == nparts - 1) ? 1 : 0;
  }
  named_bar_sync(1, kEpiThreads);
  const bool finisher = *bcast != 0;
  if (tr) tr[2] = globaltimer_ns() | (finisher ? (1ull << 63) : 0) | (ring_idle ? (1ull << 62) : 0);
  if (finisher) {
    __threadfence();
    const int nchunks = (ncols + 15) >> 4;
    const uint32_t chunk4 = 4 * kChunkBytes;  // one 16-column chunk of all 4 warps of one part
    const int cap = int(ring_bytes / (uint32_t(nparts) * chunk4));
    if (ring_idle && cap >= 1) {
      for (int ch0 = 0; ch0 < nchunks; ch0 += cap) {
        const int nch = min(cap, nchunks - ch0);
        const uint32_t bytes = uint32_t(nch) * chunk4;
        if (et == 0) {
          fence_proxy_async_global();
          mbar_arrive_expect_tx(fix_bar, bytes * uint32_t(nparts));
          for (int p = 0; p < nparts; ++p)
            bulk_g2s(ring + p * bytes, pm.of(c_first + p) + part_chunk(ch0 * 16, 0), bytes, fix_bar);
        }
        mbar_wait(fix_bar, fix_phase);
        fix_phase ^= 1;
        for (int ch = ch0; ch < ch0 + nch; ++ch) {
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
          for (int p = 0; p < nparts; ++p) {
            const float* src = reinterpret_cast<const float*>(ring + p * bytes) + part_chunk((ch - ch0) * 16, e.q);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += src[i * 32 + e.lane];
          }
          emit_chunk(a, tmO, e, m0 + e.q * 32, row0 + ch * 16, min(16, ncols - ch * 16), v);
        }
        named_bar_sync(1, kEpiThreads);  // every read of this round is done before the next copy lands
        if (et == 0) fence_proxy_async_smem();
      }
    } else {
      for (int ch = 0; ch < nchunks; ++ch) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.f;
        for (int cc = c_first; cc <= c_last; ++cc) {
          const float* src = pm.of(cc) + part_chunk(ch * 16, e.q);
          float x[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) x[i] = __ldcg(src + i * 32 + e.lane);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += x[i];
        }
        emit_chunk(a, tmO, e, m0 + e.q * 32, row0 + ch * 16, min(16, ncols - ch * 16), v);
      }
    }
    if (et == 0) *counter = 0;
  }
  named_bar_sync(1, kEpiThreads);
  if (tr) tr[3] = globaltimer_ns();
}

// ------------------------------------------------------------------ 1-CTA kernel
// KD = k-blocks per stage: 2 -> one 3-D TMA box per operand and 8 MMAs per
// stage issue, halving the per-k-block cost of the MMA warp (waits, commits,
// descriptor moves) that bounds small-T decode GEMMs.
template <int TN, int KD>
__global__ void __launch_bounds__(kThreads1, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const __grid_constant__ CUtensorMap tmO, const GemmArgs a) {
  using Cfg = GemmCfg<TN, KD>;
  // ring depth chosen at launch (<= Cfg::kStages): a shallow ring lets two CTAs
  // -- this kernel's and the next kernel's (PDL) -- share an SM
  const int S = a.stages;                            // weight ring depth
  const int SX = a.xstages > 0 ? a.xstages : S;      // activation ring depth
  const int ring_bytes = S * Cfg::kWBytes + SX * Cfg::kXBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = smem + S * Cfg::kWBytes;
  uint8_t* epi_smem = smem + ring_bytes;  // 4 x kEpiWarpBytes
  // Two stage rings, weights and activations, each with its own depth and
  // full/empty barriers: the weight ring fills before the activations of the
  // previous kernel exist, and streams from HBM (~1.1 us away) while the
  // activations come from L2, so the weight ring gets the deeper share.
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + ring_bytes + kTbufBytes);  // weights landed
  uint64_t* empty_bar = full_bar + S;                                                     // weights consumed
  uint64_t* xfull_bar = empty_bar + S;                                                    // activations landed
  uint64_t* xempty_bar = xfull_bar + SX;                                                  // activations consumed
  uint64_t* tfull_bar = xempty_bar + SX;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* fix_bar = tempty_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fix_bar + 1);
  int* bcast = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_ttiles = a.n_ttiles;
  const int c = blockIdx.x;
  const StreamK sk{a.units, int(gridDim.x), a.kblocks};
  // Work range: stream-K slice of the (tile, k-block) space, or -- in cluster
  // split mode -- k-slice r of tile c / S (the cluster = the tile's S CTAs).
  const int csplit = a.cluster_split > 1 ? a.cluster_split : 1;
  int ubeg, uend;
  if (csplit > 1) {
    const int tile = c / csplit, r = c % csplit;
    ubeg = tile * sk.kb + (r * sk.kb) / csplit;
    uend = tile * sk.kb + ((r + 1) * sk.kb) / csplit;
  } else if (a.whole_tiles) {
    const int tiles = sk.units / sk.kb;
    ubeg = int((long long)c * tiles / sk.grid) * sk.kb;
    uend = int((long long)(c + 1) * tiles / sk.grid) * sk.kb;
  } else {
    ubeg = sk.u0(c);
    uend = sk.u0(c + 1);
  }

  float4 rp[4][4];  // epilogue warps, cluster split-K fused-norm producer: prefetched residual chunks
  uint2 gp = make_uint2(0u, 0u);  // ... and this lane's 4 gamma values

  pdl_trigger();  // the next kernel may start its own prologue / weight prefetch
  if (a.trace && threadIdx.x == 0) a.trace[(size_t)c * 512] = globaltimer_ns();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < SX; ++i) {
      mbar_init(&xfull_bar[i], 1);
      mbar_init(&xempty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], kEpiThreads);
    }
    mbar_init(fix_bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------- weight producer
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();  // weights stream through once
      int stage = 0;
      uint32_t phase = 0;
      for (int u = ubeg; u < uend; ++u) {
        const int tile = u / sk.kb, kb = u % sk.kb;
        const int mt = tile / n_ttiles;
        if (u - ubeg >= S) mbar_wait(&empty_bar[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full_bar[stage], Cfg::kWBytes);
        if (KD > 1)
          tma_load_3d(&tmW, &full_bar[stage], sW + stage * Cfg::kWBytes, 0, mt * kBM, kb * KD, pol_w);
        else if (a.w_tiled)
          tma_load_2d(&tmW, &full_bar[stage], sW + stage * Cfg::kWBytes, 0, (mt * sk.kb + kb) * kBM, pol_w);
        else
          tma_load_2d(&tmW, &full_bar[stage], sW + stage * Cfg::kWBytes, kb * kBK, mt * kBM, pol_w);
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 6) {
    // ---------------------------------------------------------- activation producer
    // Activations belong to the previous kernel: wait for it (programmatic
    // dependent launch) -- the weight ring above was filled without waiting.
    if (elect_one()) {
      const uint64_t pol_x = policy_evict_last();  // activations are re-read by every tile
      pdl_wait();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = ubeg; u < uend; ++u) {
        const int tile = u / sk.kb, kb = u % sk.kb;
        const int tt = tile % n_ttiles;
        mbar_wait(&xempty_bar[stage], phase ^ 1);
        mbar_arrive_expect_tx(&xfull_bar[stage], Cfg::kXBytes);
        if (KD > 1)
          tma_load_3d(&tmX, &xfull_bar[stage], sX + stage * Cfg::kXBytes, 0, a.row_off + tt * TN, kb * KD, pol_x);
        else
          tma_load_2d(&tmX, &xfull_bar[stage], sX + stage * Cfg::kXBytes, kb * kBK, a.row_off + tt * TN, pol_x);
        if (++stage == SX) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    // The whole warp runs this loop converged; elect.sync inside the issue
    // helper picks the lane that issues (and commits: a commit tracks the MMAs
    // of its own thread, and elect.sync of a converged warp is always lane 0).
    constexpr uint32_t idesc = make_idesc_bf16(kBM, TN);
    const uint64_t dw0 = make_sw128_desc(smem_u32(sW));
    const uint64_t dx0 = make_sw128_desc(smem_u32(sX));
    int stage = 0, xstage = 0;
    uint32_t phase = 0, xphase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = ubeg; u < uend;) {
      const int kb0 = u % sk.kb;
      const int kb1 = min(sk.kb, kb0 + (uend - u));
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + uint32_t(acc * TN);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        mbar_wait(&xfull_bar[xstage], xphase);
        tc_fence_after();
        const int i = u + (kb - kb0) - ubeg;
        if (a.trace && lane == 0 && i < 64) a.trace[(size_t)c * 512 + 2 + i] = globaltimer_ns();
        __syncwarp();
        if (a.dbg & 1) {  // experiments: no MMAs, release the stage at once
          if (lane == 0) {
            mbar_arrive(&empty_bar[stage]);
            mbar_arrive(&xempty_bar[xstage]);
          }
        } else {
          // descriptor start address += stage offset (>> 4 encoded, stays inside its 14-bit field)
          const uint64_t dw = dw0 + uint64_t((stage * Cfg::kWBytes) >> 4);
          const uint64_t dx = dx0 + uint64_t((xstage * Cfg::kXBytes) >> 4);
          if (KD > 1)  // second k-block: 128 weight rows / TN token rows x 128 B further
            umma_2kblock_elect(d_tmem, dw, dx, idesc, kb > kb0 ? 1u : 0u, &empty_bar[stage], &xempty_bar[xstage],
                               uint32_t(kBM * kBK * 2) >> 4, uint32_t(TN * kBK * 2) >> 4);
          else
            umma_kblock_elect(d_tmem, dw, dx, idesc, kb > kb0 ? 1u : 0u, &empty_bar[stage], &xempty_bar[xstage]);
        }
        if (a.trace && lane == 0 && i < 64) a.trace[(size_t)c * 512 + 278 + i] = globaltimer_ns();
        if (++stage == S) { stage = 0; phase ^= 1; }
        if (++xstage == SX) { xstage = 0; xphase ^= 1; }
      }
      __syncwarp();
      if (a.dbg & 1) {
        if (lane == 0) mbar_arrive(&tfull_bar[acc]);
      } else {
        umma_commit_elect(&tfull_bar[acc]);
      }
      u += kb1 - kb0;
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else {
    // ---------------------------------------------------------- epilogue
    pdl_wait();  // outputs / residual / stream-K workspace belong to the previous kernel until now
    if (csplit > 1 && a.epi == EPI_RESID && a.h_out) {
      // register-path residual epilogue of cluster split-K (fused-norm
      // producer): the residual of this warp's first 4 reduction chunks is
      // loaded now, while the main loop runs, and kept 4 chunks ahead later
      const int w = warp - 2, qpr = 4 / csplit, cstep = 4 / qpr;
      const int tile = c / csplit, mt = tile / n_ttiles, tt = tile % n_ttiles;
      const int qq = int(cluster_ctarank()) * qpr + (w % qpr);
      const int ncols_tile = min(TN, a.T - tt * TN), nchunks = (ncols_tile + 15) >> 4;
      gp = __ldg(reinterpret_cast<const uint2*>(a.gamma_next + mt * kBM + qq * 32 + (lane & 7) * 4));
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int ch = w / qpr + g * cstep;
        if (ch < nchunks)
          load_res(a, mt * kBM + qq * 32, a.row_off + tt * TN + ch * 16, min(16, ncols_tile - ch * 16), lane, rp[g]);
      }
    }
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int et = threadIdx.x - 64;  // 0..127
    EpiWarp e(epi_smem + q * kEpiWarpBytes, q, lane, build_row_scales(a, smem + ring_bytes + kTbufBytes, et));
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t fix_phase = 0;
    int seg_i = 0;
    for (int u = ubeg; u < uend;) {
      const int tile = u / sk.kb, kb0 = u % sk.kb;
      const int kb1 = min(sk.kb, kb0 + (uend - u));
      const int mt = tile / n_ttiles, tt = tile % n_ttiles;
      const int row0 = a.row_off + tt * TN;
      const int ncols = min(TN, a.T - tt * TN);
      const bool whole = (kb0 == 0 && kb1 == sk.kb);
      const bool last_seg = (u + (kb1 - kb0) == uend);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      unsigned long long* tr = (a.trace && et == 0 && seg_i < 4) ? a.trace + (size_t)c * 512 + 130 + 4 * seg_i : nullptr;
      ++seg_i;
      if (tr) tr[0] = globaltimer_ns() | (whole ? (1ull << 62) : 0);
      const uint32_t t_addr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * TN);
      // partials are column-major [col][128 rows]: slot 0 = the CTA's first segment
      float* part = csplit > 1 ? reinterpret_cast<float*>(sW)  // cluster mode: partial stays in smem
                               : a.ws + ((size_t)c * 2 + (u == ubeg ? 0 : 1)) * (size_t)(kBM * TN);
      if (!(a.dbg & 2)) epi_drain(a, &tmO, e, t_addr, mt * kBM, row0, ncols, whole, part, csplit > 1);
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      if (tr) tr[1] = globaltimer_ns();
      if (!whole && csplit == 1) {
        const PartMap pm{a.ws, sk, tile, 1, 0, TN};
        epi_fixup(a, &tmO, e, &a.counters[tile], pm, sk.cta_of(tile * sk.kb), sk.cta_of(tile * sk.kb + sk.kb - 1),
                  mt * kBM, row0, ncols, last_seg, smem, uint32_t(ring_bytes), fix_bar, fix_phase, bcast, et, tr);
      }
      u += kb1 - kb0;
    }
    e.drain();
    if (a.trace && et == 0) a.trace[(size_t)c * 512 + 1] = globaltimer_ns();
  }
  if (csplit > 1) {
    // Cluster split-K: every CTA of the cluster holds a partial [TN][128] in
    // its shared memory; CTA r reduces rows [r*128/S, (r+1)*128/S) across the
    // S partials through DSMEM in fixed rank order and runs the epilogue.
    const int tile = c / csplit;
    const int mt = tile / n_ttiles, tt = tile % n_ttiles;
    const int ncols_tile = min(TN, a.T - tt * TN);
    const bool epi_warp = warp >= 2 && warp < 6;
    if (uend == ubeg && epi_warp) {  // empty k-slice (kb < S): contribute zeros
      float* part = reinterpret_cast<float*>(sW);
      for (int i = threadIdx.x - 64; i < TN * kBM; i += kEpiThreads) part[i] = 0.f;
    }
    // CTA `rank` reduces its 128/csplit rows (qpr warp quarters) over the S
    // partials in fixed rank order; the 4 epilogue warps split the quarters
    // and the 16-column chunks, and emit like a whole tile.
    const uint32_t rank = cluster_ctarank();
    const int w = warp - 2;
    const int qpr = 4 / csplit;  // quarters per rank (csplit is 2 or 4)
    const int qq = int(rank) * qpr + (w % qpr);
    const int row0 = a.row_off + tt * TN;
    const int nchunks = (ncols_tile + 15) >> 4;
    const int cstep = 4 / qpr;
    const int nw0 = mt * kBM + qq * 32;
    const bool pre = epi_warp && a.epi == EPI_RESID && a.h_out != nullptr;  // rp holds the residual (see above)
    cluster_sync_all();
    if (epi_warp && !(a.dbg & 128)) {  // dbg 128 (experiments): skip the reduction
      EpiWarp e(epi_smem + w * kEpiWarpBytes, qq, lane, row_scales(a, smem + ring_bytes + kTbufBytes));
      const uint32_t base = smem_u32(sW);
      for (int ch = w / qpr; ch < nchunks; ch += cstep) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.f;
        const uint32_t off = base + uint32_t(part_chunk(ch * 16, qq) * 4 + lane * 4);
        for (int src = 0; src < csplit; ++src) {
          const uint32_t ra = dsmem_map(off, uint32_t(src));
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += dsmem_ld_f32(ra + uint32_t(i * 128));
        }
        emit_chunk(a, &tmO, e, nw0, row0 + ch * 16, min(16, ncols_tile - ch * 16), v, pre ? rp[0] : nullptr,
                   pre ? &gp : nullptr);
        if (pre) {
#pragma unroll
          for (int g = 0; g < 3; ++g)
#pragma unroll
            for (int p = 0; p < 4; ++p) rp[g][p] = rp[g + 1][p];
          const int chn = ch + 4 * cstep;
          if (chn < nchunks) load_res(a, nw0, row0 + chn * 16, min(16, ncols_tile - chn * 16), lane, rp[3]);
        }
      }
      e.drain();
    }
    cluster_sync_all();  // peers' shared memory stays alive until every read is done
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<Cfg::kTmemCols>(tmem_base);
}

// Token-major accumulator (swapped CTA-pair kernel): TMEM lane = token, column
// = weight row, so each lane owns one output row and stores 32 consecutive
// outputs per TMEM load -- no smem transpose, no shuffles.  The 4 epilogue
// warps of a CTA cover its 128 tokens; a tile's 256 weight rows are 8 loads.
// Swizzled staging row for a TMA store of a token-major box (SW64 / SW32 --
// the store's swizzle mode): 16-byte chunk c of box row r.  The XOR spreads the
// 8 lanes of a quarter-warp over 8 different 16-byte bank groups.
template <int RB, int M>
CB_DEVICE uint4* stg_chunk(uint8_t* stg, int r, int c) {
  const uint32_t o = uint32_t(r * RB + c * 16);
  return reinterpret_cast<uint4*>(stg + (o ^ (((o >> 7) & M) << 4)));
}

// Split-K pairs (xp != null): the tile's other K parts of these columns, in
// shared memory, block i (stride xstride floats) = K part i (i >= xme: part
// i + 1), each [32-column chunk][8 float4 groups][128 tokens][float4]; the
// column sum runs over the parts in K order, this CTA's own accumulator being
// part xme.
__device__ const float4 kNoRes[8] = {};

CB_DEVICE void epi_drain_tok(const GemmArgs& a, const CUtensorMap* tmO, EpiWarp& e, uint32_t t_addr, int n_base,
                             int nw, int row0, int tok0, int ncols, const float* xp = nullptr, int xs = 0,
                             int xme = 0, size_t xstride = 0, bool have_first = false,
                             const float4 (&res_first)[8] = kNoRes, const float4 (&res_second)[8] = kNoRes) {
  const int tok = tok0 + e.lane;  // tok0: first token of this warp
  const bool ok = tok < ncols;
  // full 32-token groups go out through swizzled staging + one TMA store per
  // box (the token-major map: 64-byte rows, 32 rows); a partial group and the
  // fused-norm producer store from registers
  const bool use_tma = a.tma && tok0 + 32 <= ncols && !(a.epi == EPI_RESID && a.h_out);
  const int row = row0 + tok;
  const float* rt = e.rt;
  const float sc = (rt && ok) ? rt[row - a.row_off] : 1.0f;
  if (!xp && use_tma && (a.epi == EPI_BF16 || a.epi == EPI_SWIGLU)) {
    // bf16 / SwiGLU boxes two chunks at a time: both TMEM loads behind one
    // wait, both staging slots behind one proxy fence, and the two chunks'
    // conversions independent (a lone epilogue warp per sub-partition is
    // latency-bound one chunk at a time, profiles/r02_gemm_epilogue_trace.txt)
    for (int c0 = 0; c0 < nw; c0 += 64) {
      const int n0 = n_base + c0;
      if (n0 >= a.N) break;
      const bool two = c0 + 32 < nw && n0 + 32 < a.N;
      uint32_t r[2][32];
      tmem_ld32(t_addr + uint32_t(c0), r[0]);
      if (two) tmem_ld32(t_addr + uint32_t(c0 + 32), r[1]);
      tmem_ld_wait();
      uint4 o[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = rt ? __uint_as_float(r[h][i]) * sc : __uint_as_float(r[h][i]);
        if (a.epi == EPI_BF16) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            o[h][c] = make_uint4(pack_bf16x2(v[8 * c], v[8 * c + 1]), pack_bf16x2(v[8 * c + 2], v[8 * c + 3]),
                                 pack_bf16x2(v[8 * c + 4], v[8 * c + 5]), pack_bf16x2(v[8 * c + 6], v[8 * c + 7]));
        } else {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const float* g = v + 16 * c;
            o[h][c] = make_uint4(pack_bf16x2(silu_mul(g[0], g[1]), silu_mul(g[2], g[3])),
                                 pack_bf16x2(silu_mul(g[4], g[5]), silu_mul(g[6], g[7])),
                                 pack_bf16x2(silu_mul(g[8], g[9]), silu_mul(g[10], g[11])),
                                 pack_bf16x2(silu_mul(g[12], g[13]), silu_mul(g[14], g[15])));
          }
        }
      }
      // slot of the first chunk: <= 2 older stores may still read theirs; the
      // second chunk's slot was read by the store two chunks back -> <= 1
      uint8_t* s0 = e.next_stage3();
      uint8_t* s1 = nullptr;
      if (two) {
        if (e.lane == 0) bulk_wait_read<1>();
        __syncwarp();
        s1 = e.st + e.sb * kChunkBytes;
        e.sb = e.sb == 2 ? 0 : e.sb + 1;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1 && !two) break;
        uint8_t* stg = h ? s1 : s0;
        if (a.epi == EPI_BF16) {
#pragma unroll
          for (int c = 0; c < 4; ++c) *stg_chunk<64, 3>(stg, e.lane, c) = o[h][c];
        } else {
#pragma unroll
          for (int c = 0; c < 2; ++c) *stg_chunk<32, 1>(stg, e.lane, c) = o[h][c];
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (e.lane == 0) {
        const int cn = a.epi == EPI_BF16 ? n0 : n0 >> 1;
        tma_store_2d(tmO, s0, cn, row0 + tok0);
        bulk_commit();
        if (two) {
          tma_store_2d(tmO, s1, a.epi == EPI_BF16 ? n0 + 32 : (n0 + 32) >> 1, row0 + tok0);
          bulk_commit();
        }
      }
    }
    return;
  }
  for (int c0 = 0; c0 < nw; c0 += 32) {
    const int n0 = n_base + c0;
    if (n0 >= a.N) break;  // N % 32 == 0 (launcher)
    float4 res[8];
    if (!use_tma && a.epi == EPI_RESID && ok) {  // residual loads in flight during the TMEM load
#pragma unroll
      for (int j = 0; j < 8; ++j)
        res[j] = (c0 == 0 && have_first)    ? res_first[j]
                 : (c0 == 32 && have_first) ? res_second[j]
                                            : __ldcg(reinterpret_cast<const float4*>(out_f32(a, n0 + 4 * j, row)));
    }
    uint32_t r[32];
    tmem_ld32(t_addr + uint32_t(c0), r);
    tmem_ld_wait();
    float v[32];
    if (xp) {
      const int lt = tok & 127;  // token row of this CTA
      float sum[32];
      for (int src = 0; src < xs; ++src) {
        if (src == xme) {
#pragma unroll
          for (int i = 0; i < 32; ++i) sum[i] = src == 0 ? __uint_as_float(r[i]) : sum[i] + __uint_as_float(r[i]);
          continue;
        }
        const float4* pp =
            reinterpret_cast<const float4*>(xp + (src - (src > xme)) * xstride) + size_t(c0 >> 5) * 8 * 128 + lt;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 p = pp[j * 128];
          const float px[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) sum[4 * j + i] = src == 0 ? px[i] : sum[4 * j + i] + px[i];
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(sum[i]);
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = rt ? __uint_as_float(r[i]) * sc : __uint_as_float(r[i]);
    if (use_tma) {
      if (a.epi == EPI_F32 || a.epi == EPI_RESID) {  // two 16-feature boxes (64-byte fp32 rows)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint8_t* stg = e.next_stage3();
#pragma unroll
          for (int c = 0; c < 4; ++c)
            *stg_chunk<64, 3>(stg, e.lane, c) =
                make_uint4(__float_as_uint(v[16 * h + 4 * c]), __float_as_uint(v[16 * h + 4 * c + 1]),
                           __float_as_uint(v[16 * h + 4 * c + 2]), __float_as_uint(v[16 * h + 4 * c + 3]));
          if (!(a.dbg & 64)) fence_proxy_async_smem();
          __syncwarp();
          if (e.lane == 0 && !(a.dbg & 32)) {
            if (a.epi == EPI_RESID)
              tma_reduce_add_2d(tmO, stg, n0 + 16 * h, row0 + tok0);
            else
              tma_store_2d(tmO, stg, n0 + 16 * h, row0 + tok0);
            bulk_commit();
          }
        }
      } else if (a.epi == EPI_BF16) {  // one box: 32 bf16 = 64-byte rows
        uint8_t* stg = e.next_stage3();
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *stg_chunk<64, 3>(stg, e.lane, c) =
              make_uint4(pack_bf16x2(v[8 * c], v[8 * c + 1]), pack_bf16x2(v[8 * c + 2], v[8 * c + 3]),
                         pack_bf16x2(v[8 * c + 4], v[8 * c + 5]), pack_bf16x2(v[8 * c + 6], v[8 * c + 7]));
        if (!(a.dbg & 64)) fence_proxy_async_smem();
        __syncwarp();
        if (e.lane == 0 && !(a.dbg & 32)) {
          tma_store_2d(tmO, stg, n0, row0 + tok0);
          bulk_commit();
        }
      } else {  // SwiGLU: 16 bf16 outputs = 32-byte rows
        uint8_t* stg = e.next_stage3();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float* g = v + 16 * c;
          *stg_chunk<32, 1>(stg, e.lane, c) = make_uint4(
              pack_bf16x2(silu_mul(g[0], g[1]), silu_mul(g[2], g[3])),
              pack_bf16x2(silu_mul(g[4], g[5]), silu_mul(g[6], g[7])),
              pack_bf16x2(silu_mul(g[8], g[9]), silu_mul(g[10], g[11])),
              pack_bf16x2(silu_mul(g[12], g[13]), silu_mul(g[14], g[15])));
        }
        if (!(a.dbg & 64)) fence_proxy_async_smem();
        __syncwarp();
        if (e.lane == 0 && !(a.dbg & 32)) {
          tma_store_2d(tmO, stg, n0 >> 1, row0 + tok0);
          bulk_commit();
        }
      }
      continue;
    }
    if (!ok) continue;
    const size_t base = (size_t)row * a.ldo;
    if (a.epi == EPI_BF16) {
      uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(a.out) + base + n0);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        o[j] = make_uint4(pack_bf16x2(v[8 * j], v[8 * j + 1]), pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                          pack_bf16x2(v[8 * j + 4], v[8 * j + 5]), pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
    } else if (a.epi == EPI_SWIGLU) {  // rows interleave gate / up: 16 outputs
      uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(a.out) + base + (n0 >> 1));
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float* g = v + 16 * j;
        o[j] = make_uint4(pack_bf16x2(silu_mul(g[0], g[1]), silu_mul(g[2], g[3])),
                          pack_bf16x2(silu_mul(g[4], g[5]), silu_mul(g[6], g[7])),
                          pack_bf16x2(silu_mul(g[8], g[9]), silu_mul(g[10], g[11])),
                          pack_bf16x2(silu_mul(g[12], g[13]), silu_mul(g[14], g[15])));
      }
    } else {
      float4* o = reinterpret_cast<float4*>(out_f32(a, n0, row));
      float4 x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        x[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        if (a.epi == EPI_RESID)
          x[j] = make_float4(res[j].x + x[j].x, res[j].y + x[j].y, res[j].z + x[j].z, res[j].w + x[j].w);
        o[j] = x[j];
      }
      if (a.epi == EPI_RESID && a.h_out) {  // fused-norm producer: h' and this 32-feature group's sum of squares
        const uint4* gm = reinterpret_cast<const uint4*>(a.gamma_next + n0);
        uint4* h = reinterpret_cast<uint4*>(a.h_out + base + n0);
        float ss = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 g = __ldg(gm + j);
          const float4 p = x[2 * j], q = x[2 * j + 1];
          h[j] = make_uint4(pack_bf16x2(p.x * bf16_lo(g.x), p.y * bf16_hi(g.x)),
                            pack_bf16x2(p.z * bf16_lo(g.y), p.w * bf16_hi(g.y)),
                            pack_bf16x2(q.x * bf16_lo(g.z), q.y * bf16_hi(g.z)),
                            pack_bf16x2(q.z * bf16_lo(g.w), q.w * bf16_hi(g.w)));
          ss += (p.x * p.x + p.y * p.y + p.z * p.z + p.w * p.w) + (q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
        }
        a.ssq_out[(size_t)row * a.ssq_np + (n0 >> 5)] = ss;
      }
    }
  }
}

// ------------------------------------------------------------------ CTA-pair kernel
// One MMA computes a 256 (weight rows) x TNP (tokens) tile across the two SMs of
// a cluster pair; each CTA stages its own 128 weight rows and TNP/2 token rows
// per k-block (both TMA loads complete on the leader's barriers).  At T = 256
// the 1-CTA kernel would re-read the activation tile once per 128 weight rows
// (L2 traffic 3x the weight bytes); the pair kernel once per 256 rows.  Same
// stream-K split (over pairs) and fixup as the 1-CTA kernel; each CTA finishes
// its own 128-row half.
//
// SWAP (TNP = 256, whole tiles only): the MMA operands trade places -- A = the
// 256 token rows (128 per CTA), B = the 256 weight rows (128 per CTA), the
// same smem tiles and TMA loads -- so the accumulator is token-major and the
// epilogue stores rows straight from TMEM (epi_drain_tok).  The transposing
// epilogue of the weight-major layout was 20% of a T = 256 launch.
template <int TNP, bool SWAP>
__global__ void __launch_bounds__(kThreads1, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                    const __grid_constant__ CUtensorMap tmO, const GemmArgs a) {
  using Cfg = PairCfg<TNP>;
  // Token-major (SWAP) launches size the ring at run time: weight stages of
  // exactly nw / 2 rows and 6 KB epilogue blocks (the token-major epilogue
  // only stages TMA stores) leave room for a deeper ring (launch_pair)
  constexpr bool kRt = SWAP;
  const int S = kRt ? a.stages : Cfg::kStages;
  const int SX = S;
  const int WBYTES = kRt ? (a.nw >> 1) * kBK * 2 : Cfg::kWBytes;
  constexpr int XBYTES = Cfg::kXBytes;
  const int ring_bytes = S * WBYTES + SX * XBYTES;
  const int tbuf_bytes = kRt ? 4 * kTokEpiWarpBytes : kTbufBytes;
  const int epi_stride = kRt ? kTokEpiWarpBytes : kEpiWarpBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = smem + S * WBYTES;
  uint8_t* epi_smem = smem + ring_bytes;  // 4 x epi_stride
  uint64_t* wfull_bar = reinterpret_cast<uint64_t*>(smem + ring_bytes + tbuf_bytes);  // leader: weights landed
  uint64_t* xfull_bar = wfull_bar + S;   // leader: both CTAs' tokens landed
  uint64_t* empty_bar = xfull_bar + SX;  // each CTA: stage consumed
  uint64_t* xempty_bar = empty_bar;      // (one ring: weights and tokens share the release)
  uint64_t* tfull_bar = empty_bar + S;   // each CTA: accumulator ready
  uint64_t* tempty_bar = tfull_bar + 2;  // leader: both epilogues drained
  uint64_t* fix_bar = tempty_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fix_bar + 1);
  int* bcast = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // Split-K (token-major, a.ksplit = s in {2, 4}): s pairs (clusters of 2,
  // consecutive) per tile, pair kh accumulating K part kh; the parts are
  // exchanged through L2 with per-(tile, column part) arrival counters and
  // each CTA finishes nw / s of the tile's columns.  All CTAs of the launch are
  // co-resident (<= one per SM, and the next kernel can only start once every
  // CTA here ran pdl_trigger), so waiting for the other parts cannot deadlock.
  const bool split = SWAP && a.ksplit > 1;
  const int ks = split ? a.ksplit : 1;
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank;                                   // rank inside the pair
  const int kh = split ? int(blockIdx.x >> 1) % ks : 0;          // K part of this pair
  const uint16_t pmask = uint16_t(3);
  const bool leader = rank == 0;
  const int pair = split ? int(blockIdx.x) / (2 * ks) : int(blockIdx.x >> 1);  // split: the tile
  const int n_tt = a.n_ttiles;
  const StreamK sk{a.units, int(gridDim.x) >> 1, a.kblocks};
  const int ptiles = sk.units / sk.kb;
  // Rastered whole tiles (token-major plans with several token tiles, i.e.
  // prefill): pair p takes tiles p, p + pairs, ... of an order that walks the
  // weight tiles inside groups of a.raster token tiles, so the tiles in flight
  // at any moment share a few weight tiles and a few token tiles (L2-resident)
  // instead of every pair streaming its own weight tile against all tokens.
  const bool rast = SWAP && a.raster > 0;
  const int n_mine = rast ? (pair < ptiles ? (ptiles - pair + sk.grid - 1) / sk.grid : 0) : 0;
  const int ubeg = split ? pair * sk.kb + (kh * sk.kb) / ks
                   : rast ? 0 : a.whole_tiles ? int((long long)pair * ptiles / sk.grid) * sk.kb : sk.u0(pair);
  const int uend = split ? pair * sk.kb + ((kh + 1) * sk.kb) / ks
                   : rast ? n_mine * sk.kb
                          : a.whole_tiles ? int((long long)(pair + 1) * ptiles / sk.grid) * sk.kb : sk.u0(pair + 1);
  const int c = blockIdx.x;
  auto tile_of = [&](int u, int& mt_o, int& tt_o) {
    const int t = u / sk.kb;
    if (!rast) {
      mt_o = t / n_tt;
      tt_o = t % n_tt;
      return;
    }
    const int g = pair + t * sk.grid, span = a.raster * a.n_mtiles;
    const int grp = g / span, r = g - grp * span, t0 = grp * a.raster;
    const int gw = min(a.raster, n_tt - t0);
    mt_o = r / gw;
    tt_o = t0 + r % gw;
  };

  pdl_trigger();
  if (a.trace && threadIdx.x == 0) a.trace[(size_t)c * 512] = globaltimer_ns();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int i = 0; i < S; ++i) {
      mbar_init(&wfull_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < SX; ++i) {
      mbar_init(&xfull_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 2 * kEpiThreads);  // both CTAs' epilogue threads report to the leader
    }
    mbar_init(fix_bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs exist before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------- weight producer
    if (elect_one()) {
      const uint64_t pol_w = n_tt > 1 ? policy_evict_last() : policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = ubeg; u < uend; ++u) {
        int mt, tt_unused;
        tile_of(u, mt, tt_unused);
        const int kb = u % sk.kb;
        if (u - ubeg >= S) mbar_wait(&empty_bar[stage], phase ^ 1);
        if (a.trace && u - ubeg < 64) a.trace[(size_t)c * 512 + 66 + (u - ubeg)] = globaltimer_ns();
        if (SWAP) {  // nw / 2 weight rows per CTA (box height of the launcher's map)
          if (leader) mbar_arrive_expect_tx(&wfull_bar[stage], uint32_t(a.nw) * kBK * 2);
          tma_load_2d_pair(&tmW, &wfull_bar[stage], sW + stage * WBYTES, kb * kBK, mt * a.nw + int(rank) * (a.nw >> 1),
                           pol_w);
          if (++stage == S) { stage = 0; phase ^= 1; }
          continue;
        }
        if (leader) mbar_arrive_expect_tx(&wfull_bar[stage], 2 * WBYTES);
        const int mt128 = mt * 2 + int(rank);
        if (a.w_tiled)
          tma_load_2d_pair(&tmW, &wfull_bar[stage], sW + stage * WBYTES, 0, (mt128 * sk.kb + kb) * kBM, pol_w);
        else
          tma_load_2d_pair(&tmW, &wfull_bar[stage], sW + stage * WBYTES, kb * kBK, mt128 * kBM, pol_w);
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 6) {
    // ---------------------------------------------------------- activation producer
    if (elect_one()) {
      const uint64_t pol_x = policy_evict_last();
      pdl_wait();  // activations belong to the previous kernel
      int stage = 0;
      uint32_t phase = 0;
      for (int u = ubeg; u < uend; ++u) {
        int mt_unused, tt;
        tile_of(u, mt_unused, tt);
        const int kb = u % sk.kb;
        mbar_wait(&xempty_bar[stage], phase ^ 1);
        if (a.trace && u - ubeg < 64) a.trace[(size_t)c * 512 + 150 + (u - ubeg)] = globaltimer_ns();
        if (leader) mbar_arrive_expect_tx(&xfull_bar[stage], 2 * XBYTES);
        tma_load_2d_pair(&tmX, &xfull_bar[stage], sX + stage * XBYTES, kb * kBK,
                         a.row_off + tt * TNP + int(rank) * (TNP / 2), pol_x);
        if (++stage == SX) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer (leader, converged warp)
    if (leader) {
      // token-major: M = 256 tokens (A = activations), N = nw weight rows (B)
      const uint32_t idesc = SWAP ? make_idesc_bf16(TNP, uint32_t(a.nw)) : make_idesc_bf16(2 * kBM, TNP);
      const uint64_t dw0 = make_sw128_desc(smem_u32(sW));
      const uint64_t dx0 = make_sw128_desc(smem_u32(sX));
      int stage = 0, xstage = 0;
      uint32_t phase = 0, xphase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = ubeg; u < uend;) {
        const int kb0 = u % sk.kb;
        const int kb1 = min(sk.kb, kb0 + (uend - u));
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(acc * TNP);
        for (int kb = kb0; kb < kb1; ++kb) {
          const int i = u + (kb - kb0) - ubeg;
          mbar_wait(&wfull_bar[stage], phase);
          if (a.trace && lane == 0 && i < 64) a.trace[(size_t)c * 512 + 214 + i] = globaltimer_ns();
          mbar_wait(&xfull_bar[xstage], xphase);
          tc_fence_after();
          if (a.trace && lane == 0 && i < 64) a.trace[(size_t)c * 512 + 2 + i] = globaltimer_ns();
          __syncwarp();
          const uint64_t dw = dw0 + uint64_t((stage * WBYTES) >> 4);
          const uint64_t dx = dx0 + uint64_t((xstage * XBYTES) >> 4);
          if (SWAP)
            umma_kblock_pair_elect(d_tmem, dx, dw, idesc, kb > kb0 ? 1u : 0u, &empty_bar[stage], pmask);
          else
            umma_kblock_pair_elect(d_tmem, dw, dx, idesc, kb > kb0 ? 1u : 0u, &empty_bar[stage]);
          if (a.trace && lane == 0 && i < 64) a.trace[(size_t)c * 512 + 278 + i] = globaltimer_ns();
          if (++stage == S) { stage = 0; phase ^= 1; }
          if (++xstage == SX) { xstage = 0; xphase ^= 1; }
        }
        __syncwarp();
        umma_commit_pair_elect(&tfull_bar[acc], pmask);
        u += kb1 - kb0;
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ---------------------------------------------------------- epilogue (both CTAs)
    pdl_wait();  // outputs / residual / stream-K workspace belong to the previous kernel until now
    const int q = warp & 3;
    const int et = threadIdx.x - 64;  // 0..127
    EpiWarp e(epi_smem + q * epi_stride, q, lane, build_row_scales(a, smem + ring_bytes + tbuf_bytes, et));
    const uint32_t tempty_leader0 = dsmem_map(smem_u32(&tempty_bar[0]), 0);
    const uint32_t tempty_leader1 = dsmem_map(smem_u32(&tempty_bar[1]), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t fix_phase = 0;
    int seg_i = 0;
    if (split) {
      // one segment per CTA (its K part of the tile), accumulator 0
      int mt, tt;
      tile_of(ubeg, mt, tt);
      const int row0 = a.row_off + tt * TNP;
      const int ncols = min(TNP, a.T - tt * TNP);
      const int w = a.nw / ks;  // columns this CTA finishes: [kh * w, (kh + 1) * w)
      const uint32_t t_addr = tmem_base + (uint32_t(q * 32) << 16);
      const size_t blk = size_t(kBM) * w;  // floats of one (destination, source) part block
      float* xb = a.ws + size_t(pair * 2 + int(rank)) * ks * ks * blk;  // [dst][src] part blocks of this CTA slot
      const int lt = q * 32 + lane;
      unsigned long long* tr = (a.trace && et == 0) ? a.trace + (size_t)c * 512 + 130 : nullptr;
      mbar_wait(&tfull_bar[0], 0);
      tc_fence_after();
      if (tr) tr[0] = globaltimer_ns();
      // my K part of the other column parts: TMEM -> the (idle) stage ring ->
      // bulk stores to L2; the other parts of my columns: bulk loads into the
      // ring behind them.  Blocks are [32-column chunk][8 float4 groups][128
      // tokens][float4] (consecutive lanes = consecutive 16 bytes).
      float* sout = reinterpret_cast<float*>(sW);
      float* sin = sout + size_t(ks - 1) * blk;
      int nb = 0;
      for (int dst = 0; dst < ks; ++dst) {
        if (dst == kh) continue;
        float4* pp = reinterpret_cast<float4*>(sout + size_t(nb) * blk) + lt;
        for (int c0 = 0; c0 < w; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(t_addr + uint32_t(dst * w + c0), r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            pp[((c0 >> 5) * 8 + j) * 128] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                                        __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
        }
        // each block leaves for L2 as soon as it is staged (its store overlaps
        // the staging of the next one)
        fence_proxy_async_smem();
        named_bar_sync(1, kEpiThreads);
        if (et == 0) {
          bulk_s2g(xb + (dst * ks + kh) * blk, sout + size_t(nb) * blk, uint32_t(blk * 4));
          bulk_commit();
        }
        ++nb;
      }
      int* cnt = a.counters + size_t(pair * 2 + int(rank)) * ks;
      if (et == 0) {
        bulk_wait<0>();
        if (tr) tr[1] = globaltimer_ns();
        fence_proxy_async_global();  // the async-proxy stores, then the generic release below
        __threadfence();
        for (int dst = 0; dst < ks; ++dst)
          if (dst != kh) atomicAdd(cnt + dst, 1);
        while (ld_acquire_gpu(cnt + kh) < ks - 1) __nanosleep(32);
        cnt[kh] = 0;  // (every other part arrived: reset for the next launch)
        fence_proxy_async_global();
        mbar_arrive_expect_tx(fix_bar, uint32_t((ks - 1) * blk * 4));
        nb = 0;
        for (int src = 0; src < ks; ++src)
          if (src != kh) bulk_g2s(sin + size_t(nb++) * blk, xb + (kh * ks + src) * blk, uint32_t(blk * 4), fix_bar);
        if (tr) tr[2] = globaltimer_ns();
      }
      // the residual rows of both 32-column chunks (this CTA alone updates
      // them) are loaded while the other parts are still arriving
      float4 res0[8], res1[8];
      const int tok = int(rank) * kBM + q * 32 + lane;
      const bool pre = a.epi == EPI_RESID && a.h_out && tok < ncols && w == 64;
      if (pre) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          res0[j] = __ldcg(reinterpret_cast<const float4*>(out_f32(a, mt * a.nw + kh * w + 4 * j, row0 + tok)));
          res1[j] = __ldcg(reinterpret_cast<const float4*>(out_f32(a, mt * a.nw + kh * w + 32 + 4 * j, row0 + tok)));
        }
      }
      mbar_wait(fix_bar, 0);
      epi_drain_tok(a, &tmO, e, t_addr + uint32_t(kh * w), mt * a.nw + kh * w, w, row0, int(rank) * kBM + q * 32,
                    ncols, sin, ks, kh, blk, pre, res0, res1);
      if (tr) tr[3] = globaltimer_ns();
    }
    for (int u = split ? uend : ubeg; u < uend;) {
      const int tile = u / sk.kb, kb0 = u % sk.kb;
      const int kb1 = min(sk.kb, kb0 + (uend - u));
      int mt, tt;
      tile_of(u, mt, tt);
      const int m0 = mt * 2 * kBM + int(rank) * kBM;  // this CTA's first weight row
      const int row0 = a.row_off + tt * TNP;
      const int ncols = min(TNP, a.T - tt * TNP);
      const bool whole = (kb0 == 0 && kb1 == sk.kb);
      const bool last_seg = (u + (kb1 - kb0) == uend);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      unsigned long long* tr = (a.trace && et == 0 && seg_i < 4) ? a.trace + (size_t)c * 512 + 130 + 4 * seg_i : nullptr;
      ++seg_i;
      if (tr) tr[0] = globaltimer_ns() | (whole ? (1ull << 62) : 0);
      const uint32_t t_addr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * TNP);
      float* part = a.ws + ((size_t)blockIdx.x * 2 + (u == ubeg ? 0 : 1)) * (size_t)(kBM * TNP);
      if (SWAP) {
        if (!whole) __trap();  // the launcher only swaps whole-tile plans
        if (!(a.dbg & 2))
          epi_drain_tok(a, &tmO, e, t_addr, mt * a.nw, a.nw, row0, int(rank) * kBM + q * 32, ncols);
      } else if (!(a.dbg & 2)) {
        epi_drain(a, &tmO, e, t_addr, m0, row0, ncols, whole, part, false);
      }
      tc_fence_before();
      mbar_arrive_remote(acc ? tempty_leader1 : tempty_leader0);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      if (tr) tr[1] = globaltimer_ns();
      if (!SWAP && !whole) {
        const PartMap pm{a.ws, sk, tile, 2, int(rank), TNP};
        epi_fixup(a, &tmO, e, &a.counters[2 * tile + int(rank)], pm, sk.cta_of(tile * sk.kb),
                  sk.cta_of(tile * sk.kb + sk.kb - 1), m0, row0, ncols, last_seg, smem, uint32_t(ring_bytes),
                  fix_bar, fix_phase, bcast, et, tr);
      }
      u += kb1 - kb0;
    }
    e.drain();
    if (a.trace && et == 0) a.trace[(size_t)c * 512 + 1] = globaltimer_ns();
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair<Cfg::kTmemCols>(tmem_base);
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static bool load_encode_fn() {
  if (g_encode) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || fn == nullptr)
    return false;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

int make_kmajor_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t k, uint64_t row_stride_elems,
                    uint32_t box_rows) {
  if (!load_encode_fn()) return -1;
  cuuint64_t dims[2] = {k, rows};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {uint32_t(kBK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

int make_out_map(CUtensorMap* map, const void* out, int epi, uint64_t rows, uint64_t cols, uint64_t ldo) {
  if (!load_encode_fn()) return -1;
  const bool f32 = epi == EPI_F32 || epi == EPI_RESID;
  const uint32_t esz = f32 ? 4 : 2;
  const uint32_t box_c = epi == EPI_SWIGLU ? 16 : 32;
  if ((reinterpret_cast<uintptr_t>(out) & 15) || (ldo * esz) % 16 || cols % box_c) return -3;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ldo * esz};
  cuuint32_t box[2] = {box_c, 16};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                        const_cast<void*>(out), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

// Token-major output boxes of the swapped pair kernel: 64-byte rows (16 fp32 /
// 32 bf16; SwiGLU 16 bf16 = 32 bytes) x 32 tokens, swizzled like the staging.
static int make_out_map_tok(CUtensorMap* map, const void* out, int epi, uint64_t rows, uint64_t cols, uint64_t ldo) {
  if (!load_encode_fn()) return -1;
  const bool f32 = epi == EPI_F32 || epi == EPI_RESID;
  const uint32_t esz = f32 ? 4 : 2;
  const uint32_t box_c = epi == EPI_SWIGLU ? 16 : 64 / esz;
  if ((reinterpret_cast<uintptr_t>(out) & 15) || (ldo * esz) % 16 || cols % box_c) return -3;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ldo * esz};
  cuuint32_t box[2] = {box_c, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                        const_cast<void*>(out), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        epi == EPI_SWIGLU ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

int make_kmajor_map3(CUtensorMap* map, const void* base, uint64_t rows, uint64_t k, uint64_t row_stride_elems,
                     uint32_t box_rows, uint32_t kd) {
  if (!load_encode_fn()) return -1;
  if (k % (uint64_t(kBK) * kd)) return -3;
  cuuint64_t dims[3] = {uint64_t(kBK), rows, k / kBK};
  cuuint64_t strides[2] = {row_stride_elems * 2, uint64_t(kBK) * 2};
  cuuint32_t box[3] = {uint32_t(kBK), box_rows, kd};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

int gemm_pick_tn(int T) {
  if (T <= 16) return 16;
  if (T <= 32) return 32;
  if (T <= 64) return 64;
  if (T <= 128) return 128;
  return 256;
}

// Work split of one launch.  Everything but the TN bucket depends on (N, K),
// the kernel kind and the tile count only, so within one kind a decode row's
// result does not depend on how many rows share the launch.
//   T <= 128: 1-CTA kernel (128 weight rows x TN tokens), stream-K or cluster
//             split-K -- HBM-bound weight streaming;
//   T  > 128: CTA-pair kernel (256 weight rows x 256 tokens per pair tile),
//             stream-K -- halves the activation re-reads from L2.
//
// Stream-K fixups (partials through L2, last arriver sums) cost several us per
// split tile at the end of a launch (measured), so a launch whose tiles fit in
// one wave runs one tile per CTA (pair) instead (max_parts = 1); stream-K is
// kept where tiles outnumber the SMs (gate/up, lm_head) or K is long enough to
// pay for the fixup (down projection on the pair kernel).
//
// kind_T = rows of the whole pass the launch belongs to: a replica's
// micro-batch (split_batch share) runs the kernel and split the unreplicated
// pass would run, so replication does not change a row's bits (T <= 256).
GemmPlan gemm_plan(int N, int K, int T, int num_sms, int kind_T) {
  GemmPlan p{};
  p.csplit = 1;
  p.max_parts = 0;
  if (kind_T < T) kind_T = T;
  const int kb = (K + kBK - 1) / kBK;
  const long long tiles = (N + kBM - 1) / kBM;  // 128-row weight tiles
  // 2 k-blocks per stage (3-D TMA boxes) for the 1-CTA kernel up to 128 rows
  // (measured against 1 k-block stages and against two co-resident shallow-ring
  // CTAs per SM, which starve the weight stream: 15-30% slower decode steps)
  const int kd2 = (K % (2 * kBK) == 0 && kind_T <= 128) ? 2 : 1;  // replica-invariant
  p.kd = 1;
  const int ks_nw = 256, ks_s = 4;
  if (kind_T > kPairMinT && kind_T <= 256 && N % ks_nw == 0 && K % (ks_s * kBK) == 0 &&
      (N / ks_nw) * 2 * ks_s <= num_sms && tiles * 10 < (long long)num_sms * 6) {
    // few wide-K tiles (O / down) with more than 128 rows: token-major CTA
    // pairs of 256 weight rows (the k-block loop runs at ~87% of the MMA rate,
    // scripts/gemm_split_trace.py), each tile's K quarters on four pairs, the
    // parts exchanged through L2 with arrival counters, each CTA finishing 64
    // columns.  T = 256: O 22.7 -> 21.7 us, down 33.6 -> 30.8 us alone, the
    // B = 256 decode step 8.1 -> 7.5 ms (profiles/r02_gemm_ksplit.txt).  Tried
    // and slower: 128-row pairs split in halves (K halves exchanged through
    // DSMEM or L2), 8-CTA clusters of the four pairs (two waves of clusters).
    p.pair = 1;
    p.tn = 256;
    p.box_rows = 128;
    p.nw = ks_nw;
    p.whole = 1;
    p.ksplit = ks_s;
    return p;
  }
  if (kind_T <= 256 && tiles * 10 < (long long)num_sms * 6) {
    // few wide-K tiles (O / down projections): 1-CTA kernel, cluster split-K
    // (DSMEM reduction) -- measured fastest up to 256 rows
    p.pair = 0;
    p.tn = gemm_pick_tn(T);
    p.kd = kd2;
    p.box_rows = p.tn;
    while (p.csplit < 4 && tiles * p.csplit * 2 <= num_sms && p.csplit * 2 <= kb) p.csplit *= 2;
    return p;
  }
  // (token-major pairs also win for QKV / gate/up alone from ~80 rows -- 5-11%
  // in gemm_perf -- but made the B=96/128 decode step 3-5% slower: the 1-CTA
  // QKV plan leaves 52 SMs free for the attention CTAs that start under PDL)
  if (kind_T > kPairMinT) {
    p.pair = 1;
    p.tn = 256;
    p.box_rows = p.tn / 2;
    const long long n_tt = (kind_T + p.tn - 1) / p.tn;
    const long long ptiles = (long long)((N + 2 * kBM - 1) / (2 * kBM)) * n_tt;
    if (ptiles <= num_sms / 2 && kb < 128) p.max_parts = 1;  // QKV: one wave of whole tiles
    if (ptiles > num_sms / 2) p.whole = 1;                   // gate/up, lm_head: whole tiles beat stream-K fixups
    // Token-major kernel: whole tiles of nw weight rows, nw picked so the
    // waves of pair tiles fit the SMs -- per-SM work of a wave ~ nw, so the
    // cost is waves * nw (12288 rows: 64 tiles of 192 = one wave on 74 pairs
    // instead of 48 tiles of 256 on 48 pairs); ties keep the larger tile.
    if (N % 32 == 0) {
      const long long pairs = num_sms / 2;
      long long best = -1;
      for (int nw = 256; nw >= 128; nw -= 32) {
        const long long t = (N + nw - 1) / nw * n_tt;
        const long long cost = (t + pairs - 1) / pairs * nw;
        if (best < 0 || cost < best) {
          best = cost;
          p.nw = nw;
        }
      }
      p.whole = 1;
      p.max_parts = 0;
      // (2 k-blocks per stage -- 3-D boxes, half the TMA issues per byte --
      // measured 5-15% slower at T = 192..8192: 64 KB stages leave a 3-deep ring)
    }
    return p;
  }
  p.pair = 0;
  p.tn = gemm_pick_tn(T);
  p.kd = kd2;
  if (tiles <= num_sms) p.max_parts = 1;             // QKV: one wave of whole tiles
  if (tiles * 2 >= (long long)num_sms * 3) p.whole = 1;  // lm_head (>= 1.5 waves): whole tiles
  p.box_rows = p.tn;
  // (a cluster stream-K variant -- clusters owning whole tiles, split tiles
  // reduced through DSMEM -- measured 5-15% slower on the 7B decode shapes)
  return p;
}

// 16-byte vector epilogue stores are legal: 8-row groups never straddle N, and
// every output row start is 16-byte aligned.
static int vec_ok(const GemmArgs& a) {
  const uintptr_t o = reinterpret_cast<uintptr_t>(a.out);
  if (a.N % 16 != 0 || (o & 15) != 0) return 0;
  if (a.epi == EPI_SWIGLU || a.epi == EPI_BF16) return (a.ldo % 8 == 0) ? 1 : 0;
  return (a.ldo % 4 == 0) ? 1 : 0;
}

template <int TN, int KD>
static cudaError_t launch_tn(const CUtensorMap& w, const CUtensorMap& x, const CUtensorMap& o, GemmArgs a,
                             const GemmPlan& plan, int num_sms, cudaStream_t st) {
  using Cfg = GemmCfg<TN, KD>;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<TN, KD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kMaxDynSmem));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(gemm_tc_kernel<TN, KD>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) cudaGetLastError();
    attr_set[dev & 63] = true;
  }
  a.n_ttiles = (a.T + TN - 1) / TN;
  a.n_mtiles = (a.N + kBM - 1) / kBM;
  a.kblocks = (a.K + kBK * KD - 1) / (kBK * KD);
  const int stages = Cfg::kStages;
  a.stages = stages;
  a.xstages = 0;
  size_t smem_bytes = size_t(stages) * Cfg::kStageBytes + kTbufBytes + 1024 + kBarBytes;
  // Decoupled depths: activations (L2, re-read by every tile) need a short
  // ring; the rest of the 227 KB goes to the weight ring (HBM, ~1.1 us away).
  // Measured: a win for 128-row token tiles (2-k-block stages: -1% per B=128
  // step); tiles <= 64 rows starve on 2-3 activation stages (consumed in ~0.2
  // us each), and the T=256 split-K launches, faster alone, made the B=256
  // step no faster -- both keep one shared depth.
  const int xs = (TN == 128 && KD == 2) ? 2 : 0;
  if (xs > 0) {
    const size_t fixed = size_t(kTbufBytes) + 1024 + kBarBytes;
    int ws = int((kMaxDynSmem - fixed - size_t(xs) * Cfg::kXBytes) / Cfg::kWBytes);
    if (ws > kMaxStages) ws = kMaxStages;
    const size_t ring = size_t(ws) * Cfg::kWBytes + size_t(xs) * Cfg::kXBytes;
    if (ws >= 2 && (plan.csplit <= 1 || ring >= size_t(TN) * kBM * 4)) {
      a.stages = ws;
      a.xstages = xs;
      smem_bytes = ring + fixed;
    }
  }
  a.vec = vec_ok(a);
  const long long tiles = (long long)a.n_mtiles * a.n_ttiles;
  a.cluster_split = plan.csplit;
  a.units = int(tiles * a.kblocks);
  a.whole_tiles = plan.whole;
  if (plan.csplit > 1)
    return launch_pdl_cluster(gemm_tc_kernel<TN, KD>, dim3(unsigned(tiles * plan.csplit)), dim3(kThreads1),
                              smem_bytes, st, unsigned(plan.csplit), w, x, o, a);
  // persistent stream-K: one CTA per SM, a tile spread over <= max_parts CTAs
  long long ctas = num_sms;
  if (ctas > a.units) ctas = a.units;
  const int mp = a.max_parts > 0 ? a.max_parts : plan.max_parts;
  if (mp > 0 && ctas > tiles * mp) ctas = tiles * mp;
  return launch_pdl(gemm_tc_kernel<TN, KD>, dim3(unsigned(ctas)), dim3(kThreads1), smem_bytes, st, w, x, o, a);
}

template <int TNP>
static cudaError_t launch_pair(const CUtensorMap& w, const CUtensorMap& x, const CUtensorMap& o, GemmArgs a,
                               const GemmPlan& plan, int num_sms, cudaStream_t st) {
  using Cfg = PairCfg<TNP>;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc2_kernel<TNP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(Cfg::kSmemBytes));
    if (e == cudaSuccess && TNP == 2 * kBM)  // runtime-sized ring: up to the opt-in maximum
      e = cudaFuncSetAttribute(gemm_tc2_kernel<TNP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(kMaxDynSmem));
    if (e != cudaSuccess) return e;
    attr_set[dev & 63] = true;
  }
  a.n_ttiles = (a.T + TNP - 1) / TNP;
  a.kblocks = (a.K + kBK - 1) / kBK;
  a.vec = vec_ok(a);
  // Token-major kernel (plan.nw): whole tiles of nw weight rows; the weight
  // map with nw / 2-row boxes and the token-major output map are built here
  // and cached (the runtime's weight and output buffers are long-lived).
  if (TNP == 2 * kBM && plan.nw > 0 && a.w_base && !a.w_tiled && a.N % 32 == 0 && a.vec) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, long long, long long, long long, int, int>, CUtensorMap> wcache;
    static std::map<std::tuple<const void*, int, long long, long long, int>, CUtensorMap> ocache;
    CUtensorMap wt;
    {
      std::lock_guard<std::mutex> lk(mu);
      const auto key = std::make_tuple(a.w_base, (long long)a.N, (long long)a.K, a.w_stride, plan.nw, 1);
      auto it = wcache.find(key);
      if (it == wcache.end()) {
        CUtensorMap m;
        if (make_kmajor_map(&m, a.w_base, uint64_t(a.N), uint64_t(a.K), uint64_t(a.w_stride), uint32_t(plan.nw / 2)))
          return cudaErrorInvalidValue;
        it = wcache.emplace(key, m).first;
      }
      wt = it->second;
    }
    a.nw = plan.nw;
    a.n_mtiles = (a.N + a.nw - 1) / a.nw;
    const long long tiles = (long long)a.n_mtiles * a.n_ttiles;
    a.units = int(tiles * a.kblocks);
    a.whole_tiles = 1;
    const long long pairs = std::min<long long>(num_sms / 2, tiles);
    // several token tiles (prefill): rastered tile order, 16 token tiles per
    // group, so the tiles in flight share a few weight and token tiles (8192
    // rows: QKV 703 -> 557 us, gate/up 1394 -> 1196, lm_head 2253 -> 1643;
    // groups of 4 / 8 / 16 within 3% of each other, profiles/r02_prefill_raster_ab.txt)
    a.raster = a.n_ttiles > 1 ? std::min(a.n_ttiles, 16) : 0;
    CUtensorMap ot;
    std::memset(&ot, 0, sizeof(ot));
    a.tma = 0;
    if (a.out_rows > 0) {
      const long long cols = a.epi == EPI_SWIGLU ? a.N / 2 : a.N;
      const auto key = std::make_tuple(static_cast<const void*>(a.out), a.epi, a.out_rows, a.ldo, int(cols));
      std::lock_guard<std::mutex> lk(mu);
      auto it = ocache.find(key);
      if (it == ocache.end()) {
        CUtensorMap m;
        if (make_out_map_tok(&m, a.out, a.epi, uint64_t(a.out_rows), uint64_t(cols), uint64_t(a.ldo)) == 0)
          it = ocache.emplace(key, m).first;
      }
      if (it != ocache.end()) {
        ot = it->second;
        a.tma = 1;
      }
    }
    a.ksplit = (plan.ksplit > 1 && a.n_ttiles == 1 && a.nw % (32 * plan.ksplit) == 0 &&
                size_t(a.n_mtiles) * 2 * plan.ksplit * plan.ksplit * kBM * (a.nw / plan.ksplit) <=
                    gemm_ws_floats(num_sms))
                   ? plan.ksplit
                   : 0;
    // ring of exactly-sized stages (nw / 2 weight rows + TNP / 2 token rows per
    // k-block) in whatever the 6 KB-per-warp epilogue and the barriers leave
    // (decoupled weight / token ring depths measured no better: the shared
    // 7-stage ring is balanced)
    const size_t budget = kMaxDynSmem;
    const size_t wbytes = size_t(plan.nw / 2) * kBK * 2;
    const size_t stage_bytes = wbytes + Cfg::kXBytes;
    const size_t fixed = size_t(4) * kTokEpiWarpBytes + 1024 + kBarBytes;
    int stages = int((budget - fixed) / stage_bytes);
    if (stages > kMaxStages) stages = kMaxStages;
    if (stages < 2) return cudaErrorInvalidValue;
    a.stages = stages;
    a.xstages = 0;
    const size_t smem = size_t(stages) * stage_bytes + fixed;
    if (a.ksplit > 1 && size_t(stages) * stage_bytes < size_t(2) * (a.ksplit - 1) * kBM * (a.nw / a.ksplit) * 4)
      a.ksplit = 0;  // the exchange blocks must fit the stage ring
    if (a.ksplit > 1) {  // ksplit pairs per tile, one K part each
      a.raster = 0;
      return launch_pdl_cluster(gemm_tc2_kernel<TNP, true>, dim3(unsigned(2 * a.ksplit * tiles)), dim3(kThreads1),
                                smem, st, 2u, wt, x, ot, a);
    }
    return launch_pdl_cluster(gemm_tc2_kernel<TNP, true>, dim3(unsigned(2 * pairs)), dim3(kThreads1), smem, st, 2u,
                              wt, x, ot, a);
  }
  a.n_mtiles = (a.N + 2 * kBM - 1) / (2 * kBM);
  const long long tiles = (long long)a.n_mtiles * a.n_ttiles;
  a.units = int(tiles * a.kblocks);
  a.whole_tiles = plan.whole;
  long long pairs = num_sms / 2;
  if (pairs > a.units) pairs = a.units;
  const int mp = a.max_parts > 0 ? a.max_parts : plan.max_parts;
  if (mp > 0 && pairs > tiles * mp) pairs = tiles * mp;
  return launch_pdl_cluster(gemm_tc2_kernel<TNP, false>, dim3(unsigned(2 * pairs)), dim3(kThreads1), Cfg::kSmemBytes,
                            st, 2u, w, x, o, a);
}

cudaError_t gemm_launch(const CUtensorMap& w, const CUtensorMap& x, const GemmArgs& a_in, const GemmPlan& plan,
                        int num_sms, cudaStream_t st, const CUtensorMap* out_map) {
  if (a_in.T <= 0 || a_in.N <= 0) return cudaSuccess;
  GemmArgs a = a_in;
  // fused RMSNorm: the row-scale table holds one token tile; the producer needs
  // the vector epilogue (whole 32-feature groups per warp, x in registers)
  if (a.ssq_in && (a.T > kMaxNormRows || a.ssq_np <= 0 || (a.ssq_np & 3) || a.norm_d <= 0))
    return cudaErrorInvalidValue;
  if (a.h_out && (a.epi != EPI_RESID || !a.gamma_next || !a.ssq_out || (a.N & 31) || a.ssq_np != a.N / 32 ||
                  !vec_ok(a) || (reinterpret_cast<uintptr_t>(a.h_out) & 7) ||
                  (reinterpret_cast<uintptr_t>(a.gamma_next) & 7)))
    return cudaErrorInvalidValue;
  CUtensorMap o;
  // TMA stores measured: a win for the fp32 outputs (residual reduce-add,
  // logits), neutral for bf16, 3x slower for the 32-byte SwiGLU boxes.  The
  // fused-norm producer needs x_new in registers: no reduce-add.
  if (out_map && (a.epi == EPI_F32 || (a.epi == EPI_RESID && !a.h_out))) {
    o = *out_map;
    a.tma = 1;
  } else {
    std::memset(&o, 0, sizeof(o));
    a.tma = 0;
  }
  if (plan.pair) {
    if (plan.tn == 128) return launch_pair<128>(w, x, o, a, plan, num_sms, st);
    if (plan.tn == 256) return launch_pair<256>(w, x, o, a, plan, num_sms, st);
    return cudaErrorInvalidValue;
  }
  if (plan.kd == 2) {
    switch (plan.tn) {
      case 16: return launch_tn<16, 2>(w, x, o, a, plan, num_sms, st);
      case 32: return launch_tn<32, 2>(w, x, o, a, plan, num_sms, st);
      case 64: return launch_tn<64, 2>(w, x, o, a, plan, num_sms, st);
      case 128: return launch_tn<128, 2>(w, x, o, a, plan, num_sms, st);
    }
    return cudaErrorInvalidValue;
  }
  switch (plan.tn) {
    case 16: return launch_tn<16, 1>(w, x, o, a, plan, num_sms, st);
    case 32: return launch_tn<32, 1>(w, x, o, a, plan, num_sms, st);
    case 64: return launch_tn<64, 1>(w, x, o, a, plan, num_sms, st);
    case 128: return launch_tn<128, 1>(w, x, o, a, plan, num_sms, st);
    case 256: return launch_tn<256, 1>(w, x, o, a, plan, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

size_t gemm_ws_floats(int num_sms) { return size_t(num_sms) * 2 * kBM * 256; }

}  // namespace cb
