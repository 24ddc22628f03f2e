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
static constexpr int kThreads = 192;   // CTA-pair kernel: TMA, MMA, 4 epilogue warps
static constexpr int kThreads1 = 224;  // 1-CTA kernel: + a second producer warp for the activation ring
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
  static constexpr size_t kSmemBytes = size_t(kStages) * kStageBytes + 1024 /*align slack*/ + 512 /*barriers*/;
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
__global__ void __launch_bounds__(kThreads1, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const GemmArgs a) {
  using Cfg = GemmCfg<TN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = smem + S * Cfg::kWBytes;
  // Two stage rings with a shared index: weights (local TMA, its own barriers,
  // never coupled to other CTAs) and activations (possibly cluster multicast).
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sX + S * Cfg::kXBytes);  // weights landed
  uint64_t* empty_bar = full_bar + S;                                        // weights consumed
  uint64_t* xfull_bar = empty_bar + S;                                       // activations landed
  uint64_t* xempty_bar = xfull_bar + S;                                      // activations consumed (whole cluster)
  uint64_t* tfull_bar = xempty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int* bcast = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_ttiles = a.n_ttiles;
  const int c = blockIdx.x;
  // Multicast clusters (mc > 1): the mc CTAs of a cluster own mc neighbouring
  // weight tiles ("a group") and walk the group's k-blocks in lockstep; CTA r
  // loads 1/mc of each activation tile and multicasts it to the whole cluster,
  // so an activation k-block is read from L2 once per cluster.  Stream-K units
  // are (group, k-block) and are dealt out per cluster.
  const int mc = a.mcast > 1 ? a.mcast : 1;
  const int mrank = c % mc;
  const StreamK sk{a.units, int(gridDim.x) / mc, a.kblocks};
  const int cl = c / mc;
  // Work range: stream-K slice of the (group, k-block) space, or -- in cluster
  // split mode -- k-slice r of tile c / S (the cluster = the tile's S CTAs).
  const int csplit = a.cluster_split > 1 ? a.cluster_split : 1;
  int ubeg, uend;
  if (csplit > 1) {
    const int tile = c / csplit, r = c % csplit;
    ubeg = tile * sk.kb + (r * sk.kb) / csplit;
    uend = tile * sk.kb + ((r + 1) * sk.kb) / csplit;
  } else {
    ubeg = sk.u0(cl);
    uend = sk.u0(cl + 1);
  }
  const uint16_t mc_mask = uint16_t((1u << mc) - 1);

  pdl_trigger();  // the next kernel may start its own prologue / weight prefetch
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
      mbar_init(&xfull_bar[i], 1);
      mbar_init(&xempty_bar[i], mc);  // an activation slot is free once every CTA of the cluster consumed it
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], kEpiThreads);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  if (mc > 1)
    cluster_sync_all();  // peers' barriers exist before any multicast lands
  else
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
      (void)pol_x;
      int stage = 0;
      uint32_t phase = 0;
      for (int u = ubeg; u < uend; ++u) {
        const int tile = (u / sk.kb) * mc + mrank, kb = u % sk.kb;
        if (u - ubeg >= S) mbar_wait(&empty_bar[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full_bar[stage], Cfg::kWBytes);
        tma_load_2d(&tmW, &full_bar[stage], sW + stage * Cfg::kWBytes, kb * kBK, (tile / n_ttiles) * kBM, pol_w);
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 6) {
    // ---------------------------------------------------------- activation producer
    // Activations belong to the previous kernel: wait for it (programmatic
    // dependent launch) -- the weight ring above was filled without waiting.
    if (elect_one()) {
      const uint64_t pol_x = policy_evict_last();   // activations are re-read by every tile
      pdl_wait();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = ubeg; u < uend; ++u) {
        const int tile = (u / sk.kb) * mc + mrank, kb = u % sk.kb;
        const int tt = tile % n_ttiles;
        mbar_wait(&xempty_bar[stage], phase ^ 1);
        mbar_arrive_expect_tx(&xfull_bar[stage], Cfg::kXBytes);
        if (mc > 1)
          tma_load_2d_mc(&tmX, &xfull_bar[stage], sX + stage * Cfg::kXBytes + mrank * (Cfg::kXBytes / mc), kb * kBK,
                         a.row_off + tt * TN + mrank * (TN / mc), mc_mask, pol_x);
        else
          tma_load_2d(&tmX, &xfull_bar[stage], sX + stage * Cfg::kXBytes, kb * kBK, a.row_off + tt * TN, pol_x);
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
        mbar_wait(&xfull_bar[stage], phase);
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
          if (mc > 1)
            umma_commit_mc(&xempty_bar[stage], mc_mask);  // the slot's X slices came from every CTA
          else
            umma_commit(&xempty_bar[stage]);
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
      const int grp = u / sk.kb, kb0 = u % sk.kb;
      const int tile = grp * mc + mrank;
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
        const int c_first = sk.cta_of(grp * sk.kb);  // clusters sharing this group
        const int c_last = sk.cta_of(grp * sk.kb + sk.kb - 1);
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
              const int w = (sk.u0(cc) / sk.kb == grp) ? 0 : 1;
              const float* p = a.ws + ((size_t)(cc * mc + mrank) * 2 + w) * (size_t)(kBM * TN);
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
    const bool epi_warp = warp >= 2 && warp < 6;
    if (uend == ubeg && epi_warp) {  // empty k-slice (kb < S): contribute zeros
      float* part = reinterpret_cast<float*>(sW);
      for (int i = threadIdx.x - 64; i < TN * kBM; i += kEpiThreads) part[i] = 0.f;
    }
    cluster_sync_all();
    if (epi_warp) {
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
  if (mc > 1)
    cluster_sync_all();  // no CTA leaves while peers may still multicast into it / arrive on it
  else
    __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<Cfg::kTmemCols>(tmem_base);
}


// ---------------------------------------------------------------------------
// CTA-pair GEMM for prefill-sized batches (T > 256): one tcgen05.mma.cta_group::2
// computes a 256 (weight rows) x 256 (tokens) tile across the two SMs of a
// cluster pair.  Each CTA stages its own 128 weight rows and 128 token rows
// per k-block (both TMA loads signal the leader's barrier), so every byte of
// the B operand feeds twice the MMA work of the 1-CTA kernel -- the prefill
// GEMMs are L2-bandwidth / tensor bound, not HBM bound.  Persistent over pair
// tiles; accumulators double buffered in TMEM (2 x 256 columns per CTA).
static constexpr int kPairTN = 256;
static constexpr int kPairStageBytes = 2 * kBM * kBK * 2;  // 16 KB weights + 16 KB tokens per CTA
static constexpr int kPairStages = 6;
static constexpr size_t kPairSmemBytes = size_t(kPairStages) * kPairStageBytes + 1024 + 256;

__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                    const GemmArgs a) {
  constexpr int S = kPairStages;
  constexpr int HB = kBM * kBK * 2;  // one half-tile (128 rows x 64 k) in bytes
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = smem + S * HB;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sX + S * HB);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int n_mt = (a.N + 2 * kBM - 1) / (2 * kBM);
  const int n_tt = (a.T + kPairTN - 1) / kPairTN;
  const int n_tiles = n_mt * n_tt;
  const int kb_n = (a.K + kBK - 1) / kBK;

  pdl_trigger();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 2 * kEpiThreads);  // both CTAs' epilogue threads report to the leader
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs exist before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_last();  // a weight tile is reused by consecutive token tiles
      const uint64_t pol_x = policy_evict_last();
      pdl_wait();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = pair; tile < n_tiles; tile += npairs) {
        const int mt = tile / n_tt, tt = tile % n_tt;
        for (int kb = 0; kb < kb_n; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * kPairStageBytes);
          tma_load_2d_pair(&tmW, &full_bar[stage], sW + stage * HB, kb * kBK, mt * 2 * kBM + int(rank) * kBM, pol_w);
          tma_load_2d_pair(&tmX, &full_bar[stage], sX + stage * HB, kb * kBK,
                           a.row_off + tt * kPairTN + int(rank) * kBM, pol_x);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t idesc = make_idesc_bf16(2 * kBM, kPairTN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = pair; tile < n_tiles; tile += npairs) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(acc * kPairTN);
        for (int kb = 0; kb < kb_n; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint64_t dw = make_sw128_desc(smem_u32(sW + stage * HB));
            const uint64_t dx = make_sw128_desc(smem_u32(sX + stage * HB));
#pragma unroll
            for (int k = 0; k < kBK / kUmmaK; ++k)
              umma_bf16_pair(d_tmem, dw + uint64_t(2 * k), dx + uint64_t(2 * k), idesc, (kb > 0 || k > 0) ? 1u : 0u);
            umma_commit_pair(&empty_bar[stage]);  // frees the stage in both CTAs
          }
          __syncwarp();
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) umma_commit_pair(&tfull_bar[acc]);
        __syncwarp();
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    pdl_wait();
    const int q = warp & 3;
    const int row_in_tile = q * 32 + lane;
    const uint32_t tempty_leader0 = dsmem_map(smem_u32(&tempty_bar[0]), 0);
    const uint32_t tempty_leader1 = dsmem_map(smem_u32(&tempty_bar[1]), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = pair; tile < n_tiles; tile += npairs) {
      const int mt = tile / n_tt, tt = tile % n_tt;
      const int n = mt * 2 * kBM + int(rank) * kBM + row_in_tile;
      const int row0 = a.row_off + tt * kPairTN;
      const int ncols = min(kPairTN, a.T - tt * kPairTN);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_addr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * kPairTN);
      for (int c0 = 0; c0 < ncols; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(t_addr + uint32_t(c0), r);
        tmem_ld_wait();
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
        emit16(a, n, row0 + c0, min(16, ncols - c0), v);
      }
      tc_fence_before();
      mbar_arrive_remote(acc ? tempty_leader1 : tempty_leader0);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair<512>(tmem_base);
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
  if (T <= 256) return 256;
  return kPairTileMarker;  // CTA-pair kernel; its token box is 128 rows per CTA
}

// Work split of one launch.  Everything but the TN bucket depends on (N, K) and
// the tile count only, so for decode batches (T <= 256, one token tile) a row's
// result does not depend on how many rows share the launch.
GemmPlan gemm_plan(int N, int K, int T, int num_sms) {
  GemmPlan p{};
  p.tn = gemm_pick_tn(T);
  if (p.tn == kPairTileMarker) {
    p.box_rows = kBM;
    p.mcast = 1;
    p.csplit = 1;
    return p;
  }
  const long long tiles = (N + kBM - 1) / kBM;  // one token tile
  const int kb = (K + kBK - 1) / kBK;
  p.csplit = 1;
  p.mcast = 1;
  if (tiles * 10 < (long long)num_sms * 6) {
    // few wide-K tiles (O / down projections): cluster split-K
    while (p.csplit < 8 && tiles * p.csplit * 2 <= num_sms && p.csplit * 2 <= kb) p.csplit *= 2;
  }
  // (activation multicast across clusters -- a.mcast > 1 -- is implemented and
  // correct but measured no faster than plain loads on B200, so plans keep 1)
  p.box_rows = p.tn / p.mcast;
  return p;
}

// How many clusters of `cs` CTAs of this kernel can be resident at once (GPCs
// are not multiples of 4 SMs: clusters of 4 fit on 132 of the 148 SMs).
template <typename K>
static int max_active_clusters(K kernel, int cs, size_t smem, int threads) {
  static int cache[64][9] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& slot = cache[dev & 63][cs & 7];
  if (slot) return slot;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(cs));
  cfg.blockDim = dim3(unsigned(threads));
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(cs);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = 148 / cs;
  }
  slot = n;
  return n;
}

template <int TN>
static cudaError_t launch_tn(const CUtensorMap& w, const CUtensorMap& x, GemmArgs a, const GemmPlan& plan,
                             int num_sms, cudaStream_t st) {
  using Cfg = GemmCfg<TN>;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<TN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(Cfg::kSmemBytes));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(gemm_tc_kernel<TN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) cudaGetLastError();
    attr_set[dev & 63] = true;
  }
  a.n_ttiles = (a.T + TN - 1) / TN;
  a.n_mtiles = (a.N + kBM - 1) / kBM;
  a.kblocks = (a.K + kBK - 1) / kBK;
  const long long tiles = (long long)a.n_mtiles * a.n_ttiles;
  a.cluster_split = plan.csplit;
  a.mcast = plan.mcast;
  if (plan.csplit > 1) {
    a.units = int(tiles * a.kblocks);
    return launch_pdl_cluster(gemm_tc_kernel<TN>, dim3(unsigned(tiles * plan.csplit)), dim3(kThreads1),
                              Cfg::kSmemBytes, st, unsigned(plan.csplit), w, x, a);
  }
  const int mc = plan.mcast;
  const long long groups = (tiles + mc - 1) / mc;
  a.units = int(groups * a.kblocks);
  // persistent stream-K over clusters; a group is spread over <= max_parts clusters
  long long clusters = num_sms / mc;
  if (mc > 1) {
    const int resident = max_active_clusters(gemm_tc_kernel<TN>, mc, Cfg::kSmemBytes, kThreads1);
    if (clusters > resident) clusters = resident;  // one wave: no cluster waits for another to finish
  }
  if (clusters > a.units) clusters = a.units;
  const int max_parts = a.max_parts > 0 ? a.max_parts : 1;
  if (clusters > groups * max_parts) clusters = groups * max_parts;
  if (mc == 1)
    return launch_pdl(gemm_tc_kernel<TN>, dim3(unsigned(clusters)), dim3(kThreads1), Cfg::kSmemBytes, st, w, x, a);
  return launch_pdl_cluster(gemm_tc_kernel<TN>, dim3(unsigned(clusters * mc)), dim3(kThreads1), Cfg::kSmemBytes, st,
                            unsigned(mc), w, x, a);
}

static cudaError_t launch_pair(const CUtensorMap& w, const CUtensorMap& x, GemmArgs a, int num_sms, cudaStream_t st) {
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kPairSmemBytes));
    if (e != cudaSuccess) return e;
    attr_set[dev & 63] = true;
  }
  const long long tiles = (long long)((a.N + 2 * kBM - 1) / (2 * kBM)) * ((a.T + kPairTN - 1) / kPairTN);
  long long pairs = num_sms / 2;
  if (pairs > tiles) pairs = tiles;
  return launch_pdl_cluster(gemm_tc2_kernel, dim3(unsigned(2 * pairs)), dim3(kThreads), kPairSmemBytes, st, 2u,
                            w, x, a);
}

cudaError_t gemm_launch(const CUtensorMap& w, const CUtensorMap& x, const GemmArgs& a, const GemmPlan& plan,
                        int num_sms, cudaStream_t st) {
  if (a.T <= 0 || a.N <= 0) return cudaSuccess;
  switch (plan.tn) {
    case 16: return launch_tn<16>(w, x, a, plan, num_sms, st);
    case 32: return launch_tn<32>(w, x, a, plan, num_sms, st);
    case 64: return launch_tn<64>(w, x, a, plan, num_sms, st);
    case 128: return launch_tn<128>(w, x, a, plan, num_sms, st);
    case 256: return launch_tn<256>(w, x, a, plan, num_sms, st);
    case kPairTileMarker: return launch_pair(w, x, a, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

size_t gemm_ws_floats(int num_sms) { return size_t(num_sms) * 2 * kBM * 256; }

}  // namespace cb
