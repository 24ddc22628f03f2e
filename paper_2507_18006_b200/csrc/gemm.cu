// tcgen05 / TMEM / TMA GEMM for the decoder-layer projections (sm_100a).
//
//   out[t, n] (op)= sum_k X[row_off + t, k] * W[n, k]        t < T, n < N
//
// W is a PyTorch-layout weight [N, K] (K contiguous), X the activation rows
// [rows, K].  Both are K-major, the native tcgen05 operand layout.  The MMA's
// M dimension is the weight rows (128 per tile) and its N dimension the tokens
// (TN = 16..256 per tile): "swap-AB", so a decode step with a handful of rows
// still drives the tensor pipe while the kernel streams the weight at HBM rate
// (decode GEMMs are HBM-bound, prefill GEMMs tensor-bound).
//
// Work split: persistent stream-K.  The (tile, k-block) unit space is cut into
// `grid` contiguous ranges, one per CTA (grid <= #SMs, one CTA per SM), so all
// SMs pull weight bytes for the whole launch regardless of N.  A tile split
// across CTAs is finished by the last CTA to arrive: every part writes an fp32
// partial to a (L2-resident) workspace and the finisher sums the parts in a
// fixed order -> deterministic, and for T <= 256 the split points do not depend
// on T, so a row's result is identical whether it runs unreplicated or inside
// a replica's micro-batch (reference batch split: ops.py:151-158).
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM owner + MMA
// issuer (one elected lane), warps 2..5 = epilogue (TMEM -> registers -> global,
// with the fused epilogue ops below).  TMEM accumulators are double buffered so
// the epilogue of one tile overlaps the main loop of the next.
//
// Stand-in replaced: reference `_kernels._work_units` (`_kernels.py:17-38`) and
// the per-module GEMM FLOPs of `ModuleCatalog.from_model` (`domain.py:241-264`).
#include "common.cuh"
#include "kernels.h"

namespace cb {

static constexpr int kBM = 128;          // weight rows per tile (UMMA M)
static constexpr int kBK = 64;           // k-block: 64 bf16 = one 128-byte swizzle row
static constexpr int kUmmaK = 16;        // K per tcgen05.mma (bf16)
static constexpr int kThreads = 192;
static constexpr int kEpiThreads = 128;
static constexpr size_t kSmemBudget = 200 * 1024;

template <int TN>
struct GemmCfg {
  static constexpr int kWBytes = kBM * kBK * 2;
  static constexpr int kXBytes = TN * kBK * 2;
  static constexpr int kStageBytes = kWBytes + kXBytes;
  static constexpr int kStagesRaw = int((kSmemBudget - 2048) / kStageBytes);
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr uint32_t kTmemCols = (2 * TN <= 32)    ? 32
                                        : (2 * TN <= 64)  ? 64
                                        : (2 * TN <= 128) ? 128
                                        : (2 * TN <= 256) ? 256
                                                          : 512;
  static constexpr size_t kSmemBytes = size_t(kStages) * kStageBytes + 1024 /*align slack*/ + 256;
};

struct StreamK {
  int units, grid, kb;
  CB_DEVICE int u0(int c) const { return int((long long)c * units / grid); }
  CB_DEVICE int cta_of(int u) const { return int(((long long)(u + 1) * grid - 1) / units); }
};

// Apply the fused epilogue to 16 consecutive token columns of one weight row.
CB_DEVICE void emit16(const GemmArgs& a, int n, int row0, int ncols, const float (&v)[16]) {
  const int lane = threadIdx.x & 31;
  if (a.epi == EPI_SWIGLU) {
    // rows are interleaved gate/up pairs: even row = gate_j, odd row = up_j.
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float other = __shfl_xor_sync(0xffffffffu, v[i], 1);
      if (!(lane & 1) && n < a.N && i < ncols) {
        float g = v[i];
        float s = g / (1.0f + __expf(-g));
        reinterpret_cast<uint16_t*>(a.out)[(size_t)(row0 + i) * a.ldo + (n >> 1)] = f_to_bf16(s * other);
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

// Epilogue of a (row pair, token column) of a finished tile: rows n, n+1 of
// the weight (an interleaved gate/up pair for SwiGLU).
CB_DEVICE void emit_pair(const GemmArgs& a, int n, int row, float v0, float v1) {
  if (n >= a.N) return;
  const size_t base = (size_t)row * a.ldo;
  if (a.epi == EPI_SWIGLU) {
    reinterpret_cast<uint16_t*>(a.out)[base + (n >> 1)] = f_to_bf16(v0 / (1.0f + __expf(-v0)) * v1);
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

template <int TN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const GemmArgs a) {
  using Cfg = GemmCfg<TN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = smem + S * Cfg::kWBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sX + S * Cfg::kXBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int* bcast = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_ttiles = a.n_ttiles;
  const StreamK sk{a.units, int(gridDim.x), a.kblocks};
  const int c = blockIdx.x;
  // Work range: stream-K slice of the (tile, k-block) space, or -- in cluster
  // split mode -- k-slice r of tile c / S (the cluster = the tile's S CTAs).
  const int csplit = a.cluster_split > 1 ? a.cluster_split : 1;
  int ubeg, uend;
  if (csplit > 1) {
    const int tile = c / csplit, r = c % csplit;
    ubeg = tile * sk.kb + (r * sk.kb) / csplit;
    uend = tile * sk.kb + ((r + 1) * sk.kb) / csplit;
  } else {
    ubeg = sk.u0(c);
    uend = sk.u0(c + 1);
  }

  pdl_trigger();  // the next kernel may start its own prologue / weight prefetch
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], kEpiThreads);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();  // weights stream through once
      const uint64_t pol_x = policy_evict_last();   // activations are re-read by every tile
      // Weights do not depend on the previous kernel: fill the first stages'
      // weight tiles before waiting on it (programmatic dependent launch).
      const int npre = min(S, uend - ubeg);
      for (int i = 0; i < npre; ++i) {
        const int u = ubeg + i, tile = u / sk.kb, kb = u % sk.kb;
        mbar_arrive_expect_tx(&full_bar[i], Cfg::kStageBytes);
        tma_load_2d(&tmW, &full_bar[i], sW + i * Cfg::kWBytes, kb * kBK, (tile / n_ttiles) * kBM, pol_w);
      }
      pdl_wait();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = ubeg; u < uend; ++u) {
        const int tile = u / sk.kb, kb = u % sk.kb;
        const int mt = tile / n_ttiles, tt = tile % n_ttiles;
        if (u - ubeg >= npre) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          tma_load_2d(&tmW, &full_bar[stage], sW + stage * Cfg::kWBytes, kb * kBK, mt * kBM, pol_w);
        }
        tma_load_2d(&tmX, &full_bar[stage], sX + stage * Cfg::kXBytes, kb * kBK, a.row_off + tt * TN, pol_x);
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = make_idesc_bf16(kBM, TN);
    int stage = 0;
    uint32_t phase = 0;
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
        tc_fence_after();
        if (lane == 0) {  // the same lane issues and commits (commit tracks its own MMAs)
          const uint64_t dw = make_sw128_desc(smem_u32(sW + stage * Cfg::kWBytes));
          const uint64_t dx = make_sw128_desc(smem_u32(sX + stage * Cfg::kXBytes));
#pragma unroll
          for (int k = 0; k < kBK / kUmmaK; ++k) {
            // +32 bytes per K=16 step inside the 128-byte swizzle row (>>4 encoded)
            umma_bf16(d_tmem, dw + uint64_t(2 * k), dx + uint64_t(2 * k), idesc,
                      (kb > kb0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) umma_commit(&tfull_bar[acc]);
      __syncwarp();
      u += kb1 - kb0;
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else {
    // ---------------------------------------------------------- epilogue
    pdl_wait();  // outputs / residual / stream-K workspace belong to the previous kernel until now
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row_in_tile = q * 32 + lane;
    const int et = threadIdx.x - 64;  // 0..127
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = ubeg; u < uend;) {
      const int tile = u / sk.kb, kb0 = u % sk.kb;
      const int kb1 = min(sk.kb, kb0 + (uend - u));
      const int mt = tile / n_ttiles, tt = tile % n_ttiles;
      const int n = mt * kBM + row_in_tile;
      const int row0 = a.row_off + tt * TN;
      const int ncols_tile = min(TN, a.T - tt * TN);
      const bool whole = (kb0 == 0 && kb1 == sk.kb);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_addr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * TN);
      // which workspace slot: 0 if this is the CTA's first segment, else 1
      const int which = (u == ubeg) ? 0 : 1;
      // partials are column-major [col][128 rows]: coalesced stores here and
      // coalesced row-pair loads in the fixup
      float* part = csplit > 1 ? reinterpret_cast<float*>(sW)  // cluster mode: partial stays in smem
                               : a.ws + ((size_t)c * 2 + which) * (size_t)(kBM * TN);
      for (int c0 = 0; c0 < ncols_tile; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(t_addr + uint32_t(c0), r);
        tmem_ld_wait();
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
        if (whole) {
          emit16(a, n, row0 + c0, min(16, ncols_tile - c0), v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) part[(size_t)(c0 + i) * kBM + row_in_tile] = v[i];
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;

      if (!whole && csplit == 1) {
        // stream-K fixup: the last CTA to deposit its part finishes the tile.
        const int c_first = sk.cta_of(tile * sk.kb);
        const int c_last = sk.cta_of(tile * sk.kb + sk.kb - 1);
        __threadfence();
        named_bar_sync(1, kEpiThreads);
        if (et == 0) {
          int prev = atomicAdd(&a.counters[tile], 1);
          *bcast = (prev == c_last - c_first) ? 1 : 0;
        }
        named_bar_sync(1, kEpiThreads);
        if (*bcast) {
          __threadfence();
          // work item = (row pair, token column); parts summed in fixed CTA
          // order (deterministic); 8 items per thread in flight per round trip.
          const int n_items = 64 * ncols_tile;
          for (int base = et; base < n_items; base += 8 * kEpiThreads) {
            float2 sum[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) sum[j] = make_float2(0.f, 0.f);
            for (int cc = c_first; cc <= c_last; ++cc) {
              const int w = (sk.u0(cc) / sk.kb == tile) ? 0 : 1;
              const float* p = a.ws + ((size_t)cc * 2 + w) * (size_t)(kBM * TN);
              float2 ld[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) ld[j] = make_float2(0.f, 0.f);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int it = base + j * kEpiThreads;
                if (it < n_items)
                  ld[j] = __ldcg(reinterpret_cast<const float2*>(p + (size_t)(it >> 6) * kBM + 2 * (it & 63)));
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                sum[j].x += ld[j].x;
                sum[j].y += ld[j].y;
              }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int it = base + j * kEpiThreads;
              if (it < n_items) emit_pair(a, mt * kBM + 2 * (it & 63), row0 + (it >> 6), sum[j].x, sum[j].y);
            }
          }
          if (et == 0) a.counters[tile] = 0;
        }
        named_bar_sync(1, kEpiThreads);
      }
      u += kb1 - kb0;
    }
  }
  if (csplit > 1) {
    // Cluster split-K: every CTA of the cluster holds a partial [TN][128] in
    // its shared memory; CTA r reduces rows [r*128/S, (r+1)*128/S) across the
    // S partials through DSMEM in fixed rank order and runs the epilogue.
    const int tile = c / csplit;
    const int mt = tile / n_ttiles, tt = tile % n_ttiles;
    const int ncols_tile = min(TN, a.T - tt * TN);
    if (uend == ubeg && warp >= 2) {  // empty k-slice (kb < S): contribute zeros
      float* part = reinterpret_cast<float*>(sW);
      for (int i = threadIdx.x - 64; i < TN * kBM; i += kEpiThreads) part[i] = 0.f;
    }
    cluster_sync_all();
    if (warp >= 2) {
      const int et = threadIdx.x - 64;
      const uint32_t rank = cluster_ctarank();
      const int rows_per = kBM / csplit, pairs = rows_per / 2;
      const int row_base = int(rank) * rows_per;
      const int row0 = a.row_off + tt * TN;
      const uint32_t base = smem_u32(sW);
      for (int it = et; it < pairs * ncols_tile; it += kEpiThreads) {
        const int col = it / pairs, row = row_base + 2 * (it % pairs);
        const uint32_t off = base + uint32_t((col * kBM + row) * 4);
        float2 sum = make_float2(0.f, 0.f);
        for (int src = 0; src < csplit; ++src) {
          const float2 v = dsmem_ld_f2(dsmem_map(off, uint32_t(src)));
          sum.x += v.x;
          sum.y += v.y;
        }
        emit_pair(a, mt * kBM + row, row0 + col, sum.x, sum.y);
      }
    }
    cluster_sync_all();  // peers' shared memory stays alive until every read is done
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<Cfg::kTmemCols>(tmem_base);
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

int gemm_pick_tn(int T) {
  if (T <= 16) return 16;
  if (T <= 32) return 32;
  if (T <= 64) return 64;
  if (T <= 128) return 128;
  return 256;
}

template <int TN>
static cudaError_t launch_tn(const CUtensorMap& w, const CUtensorMap& x, GemmArgs a, int num_sms,
                             cudaStream_t st) {
  using Cfg = GemmCfg<TN>;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<TN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(Cfg::kSmemBytes));
    if (e != cudaSuccess) return e;
    attr_set[dev & 63] = true;
  }
  a.n_ttiles = (a.T + TN - 1) / TN;
  a.n_mtiles = (a.N + kBM - 1) / kBM;
  a.kblocks = (a.K + kBK - 1) / kBK;
  const long long tiles0 = (long long)a.n_mtiles * a.n_ttiles;
  // Cluster split-K for few wide-K tiles (decode O / down projections): each
  // tile's K is cut over S CTAs of one cluster, partials reduced through DSMEM.
  int cs = a.cluster_split;
  if (cs == 0) {
    cs = 1;
    // depends on the tile count only (n_ttiles == 1 for every decode batch <= 256
    // rows), so a row's bits do not depend on how many rows share the launch
    if (a.n_ttiles == 1 && tiles0 * 10 < (long long)num_sms * 6) {
      while (cs < 8 && tiles0 * cs * 2 <= num_sms && cs * 2 <= a.kblocks) cs *= 2;
    }
  }
  a.cluster_split = cs;
  if (cs > 1) {
    a.units = int(tiles0 * a.kblocks);
    return launch_pdl_cluster(gemm_tc_kernel<TN>, dim3(unsigned(tiles0 * cs)), dim3(kThreads), Cfg::kSmemBytes, st,
                              unsigned(cs), w, x, a);
  }
  const long long tiles = (long long)a.n_mtiles * a.n_ttiles;
  long long units = tiles * a.kblocks;
  a.units = int(units);
  // HBM-bound weight streaming needs enough bytes in flight, not every SM:
  // cap the split so a tile is shared by <= ~max_parts CTAs (short fixups).
  long long grid = units < num_sms ? units : num_sms;
  // Split rule (depends only on the tile count and TN bucket, so for decode
  // batches in one bucket a row's bits do not depend on how many rows share
  // the launch): few tiles -> spread each over <= 4 CTAs so every SM streams
  // weights; many tiles or wide TN -> no split (the fixup would cost more).
  int max_parts = a.max_parts;
  if (max_parts <= 0) {
    if (TN > 64 || tiles * 10 >= (long long)num_sms * 6)
      max_parts = 1;
    else
      max_parts = int((num_sms + tiles - 1) / tiles) < 4 ? int((num_sms + tiles - 1) / tiles) : 4;
  }
  if (grid > tiles * max_parts) grid = tiles * max_parts;
  return launch_pdl(gemm_tc_kernel<TN>, dim3(unsigned(grid)), dim3(kThreads), Cfg::kSmemBytes, st, w, x, a);
}

cudaError_t gemm_launch(const CUtensorMap& w, const CUtensorMap& x, const GemmArgs& a, int tn, int num_sms,
                        cudaStream_t st) {
  if (a.T <= 0 || a.N <= 0) return cudaSuccess;
  switch (tn) {
    case 16: return launch_tn<16>(w, x, a, num_sms, st);
    case 32: return launch_tn<32>(w, x, a, num_sms, st);
    case 64: return launch_tn<64>(w, x, a, num_sms, st);
    case 128: return launch_tn<128>(w, x, a, num_sms, st);
    case 256: return launch_tn<256>(w, x, a, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

size_t gemm_ws_floats(int num_sms) { return size_t(num_sms) * 2 * kBM * 256; }

}  // namespace cb
