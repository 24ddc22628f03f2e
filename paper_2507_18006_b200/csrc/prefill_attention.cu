// Causal prefill attention on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Prefill rows of one sequence are contiguous in qkv and their K/V were just
// appended to the slot's cache (rope_kv_kernel).  CTA = (256-row query block of
// one sequence, q head) = two 128-row tiles A and B sharing the K / V blocks of
// 64 cached positions; 11 warps, warp-specialised:
//
//   warps 0, 10 TMA producers: Q of both tiles once, then K and V blocks
//               (SWIZZLE_128B boxes of 64 columns x 64 rows straight from the
//               [slot][pos][k|v] cache) into two 3-stage rings (K freed when
//               both S MMAs of a block retire, V when both PV MMAs do)
//   warp 1      MMA issuer (one elected lane of a converged warp, four MMAs per
//               asm block), per key block j: S_A(j), S_B(j) = Q K_j^T (M 128 x
//               N 64, K-major, double-buffered in TMEM per tile), then
//               PV_A(j-1), PV_B(j-1) (M 128 x N hd; P from TMEM, V MN-major:
//               the cache's [pos][hd] rows as they are)
//   warps 2..5  softmax of tile A, warps 6..9 of tile B: one thread per query
//               row (TMEM lane): S row -> registers (tcgen05.ld), causal mask
//               on diagonal blocks only, online softmax in the exp2 domain (one
//               FFMA + MUFU.EX2 per score) with lazy rescaling (O in TMEM is
//               rescaled with tcgen05.ld/st only when a row max grows by > 2^8),
//               P as bf16 pairs over the S columns just read (tcgen05.st): the
//               PV MMA's A operand straight from TMEM, as FlashAttention-4
//               does; finally O / l -> bf16 -> global.
//
// Ping-pong: while one tile's softmax runs, the tensor pipe executes the other
// tile's MMAs, and the two warpgroups take turns on each sub-partition's MUFU.
// TMEM: S_A[2 x 64] S_B[2 x 64] O_A[hd] O_B[hd] = 512 columns.  Smem (hd 128):
// Q 2 x 32 KB + K 3 x 16 KB + V 3 x 16 KB = 160 KB.  Positions
// past the sequence inside its last key block are masked in S, and their V
// rows are zeroed in smem before the PV MMAs (stale cache bytes could hold
// non-finite values; 0 * NaN would poison the row).  The tensor pipe is the
// limit now (scripts/pf_trace.py): with N = 64 the S MMAs read ~128 B/clk of
// operands from smem, and the PV MMAs with an MN-major B run ~2x their
// nominal time.
//
// Replaces the mma.sync (HMMA.16816) flash-attention forward of round 1.
#include "common.cuh"
#include "kernels.h"

#ifdef PF_TRACE  // timeline probe (scripts/pf_trace.py builds a separate library with it)
__device__ unsigned long long* g_pf_trace = nullptr;
#define PFT(slot, j)                                                                          \
  do {                                                                                        \
    if (g_pf_trace && blockIdx.y == 0 && blockIdx.x == gridDim.x - 1 && (j) < 32)             \
      g_pf_trace[(slot) * 32 + (j)] = clock64();                                       \
  } while (0)
extern "C" int cbt_pf_trace_set(unsigned long long* p) {
  return cudaMemcpyToSymbol(g_pf_trace, &p, sizeof(p)) == cudaSuccess ? 0 : -1;
}
#else
#define PFT(slot, j) \
  do {               \
  } while (0)
#endif

namespace cb {

static constexpr int kPfThreads = 352;  // 11 warps: K producer, MMA, 8 softmax, V producer


CB_DEVICE void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
CB_DEVICE float fast_exp2(float x) {  // ex2.approx.ftz: one MUFU.EX2, exp2(-inf) = 0
#ifdef PF_NOEXP  // probe only (wrong results): the softmax without its MUFU work
  return fmaf(x, 1e-30f, 0.5f);
#else
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#endif
}
// Four K=16 MMAs from one asm block (one elected lane of a converged warp):
// A advances 32 bytes per MMA (a K-major 128-byte-swizzled box), B by
// BSTEP (>> 4 encoded): 2 for a K-major box, 128 for an MN-major operand
// (16 rows of 128 bytes).  Per-MMA asm blocks cost ~120 clk of descriptor moves
// each (measured with scripts/pf_trace.py: 0.5 us for 8 MMAs).
template <int BSTEP>
CB_DEVICE void umma4_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.b32 q, %4, 0;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, %5;\n\tadd.s64 b2, %2, %6;\n\tadd.s64 b3, %2, %7;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "n"(BSTEP), "n"(2 * BSTEP), "n"(3 * BSTEP)
      : "memory");
}

// Four K=16 MMAs with A in tensor memory (M lanes x K/2 columns: two bf16 of
// a row per 32-bit column, so +8 columns per K=16 step) and B from smem.
template <int BSTEP>
CB_DEVICE void umma4_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t.reg .b32 a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "setp.ne.b32 q, %4, 0;\n\t"
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
      "add.s64 b1, %2, %5;\n\tadd.s64 b2, %2, %6;\n\tadd.s64 b3, %2, %7;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, q;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, 1;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, 1;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "n"(BSTEP), "n"(2 * BSTEP), "n"(3 * BSTEP)
      : "memory");
}
CB_DEVICE void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// non-blocking: has the phase with this parity completed?
CB_DEVICE bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
CB_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// MN-major operand (the contiguous dimension is N) in 128-byte-swizzled
// [k rows][64 n] boxes: SBO = 1024 B between 8-row k groups, LBO = bytes
// between consecutive 64-column n boxes.
CB_DEVICE uint64_t make_sw128_mn_desc(uint32_t smem_addr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= uint64_t((smem_addr & 0x3ffff) >> 4);
  d |= uint64_t((lbo_bytes >> 4) & 0x3fff) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

// ---------------------------------------------------------------------------
// CTA = (256-row query block of one sequence, q head) as
// two 128-row tiles A and B sharing the K / V blocks of 64 positions.  The
// MMA warp issues S_A(j), S_B(j), then PV_A(j-1), PV_B(j-1): while one tile's
// softmax warpgroup (4 warps, one thread per row) turns S into P, the tensor
// pipe runs the other tile's MMAs, and the two warpgroups take turns on each
// sub-partition's MUFU.  TMEM: S_A[2 x 64] S_B[2 x 64] O_A[hd] O_B[hd] (512
// columns); smem (hd 128): Q 2 x 32 KB + K 3 x 16 KB + V 3 x 16 KB + P 2 x 16 KB.
template <int HD>
struct PpCfg {
  static constexpr int kKeys = 64;                  // positions per K / V block
  static constexpr int kQBox = 128 * 128;           // [128 rows][64 bf16] swizzled box
  static constexpr int kKVBox = kKeys * 128;        // [64 keys][64 bf16]
  static constexpr int kQ = 2 * (HD / 64) * kQBox;  // two tiles
  static constexpr int kK = (HD / 64) * kKVBox;
  static constexpr int kV = kK;
  static constexpr int kStages = 3;
  static constexpr int kBars = 32 * 8;
  static constexpr int kSmem = 1024 + kQ + kStages * (kK + kV) + kBars;
};

template <int HD>
__global__ void __launch_bounds__(kPfThreads, 1)
    prefill_attn_pp_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mkv,
                           const AttnArgs a, const int4* __restrict__ blocks) {
  using C = PpCfg<HD>;
  constexpr int NR = HD / 64;
  constexpr int KB = C::kKeys;
  constexpr int ST = C::kStages;
  extern __shared__ uint8_t pf_raw[];
  uint8_t* sm = pf_raw + ((1024 - (smem_u32(pf_raw) & 1023)) & 1023);
  uint8_t* sQ = sm;                      // [tile][NR boxes]
  uint8_t* sK = sQ + C::kQ;              // [ST][NR boxes]
  uint8_t* sV = sK + ST * C::kK;         // [ST][NR boxes]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + ST * C::kV);
  uint64_t* bar_q = bars + 0;
  uint64_t* k_full = bars + 1;   // [3]
  uint64_t* k_empty = bars + 4;  // [3]
  uint64_t* v_full = bars + 7;   // [3]
  uint64_t* v_empty = bars + 10; // [3]
  uint64_t* s_full = bars + 13;  // [tile][2]
  uint64_t* s_free = bars + 17;  // [tile][2]
  uint64_t* p_full = bars + 21;  // [tile]
  uint64_t* o_done = bars + 23;  // [tile]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 25);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < ST; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(s_free + i, 128);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(p_full + t, 128);
      mbar_init(o_done + t, 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&mq);
    tma_prefetch_desc(&mkv);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // q rotated and K/V appended by rope_kv_kernel
  if (threadIdx.x == 0) PFT(9, 0);

  const int4 blk = blocks[blockIdx.x];  // (first row, rows <= 256, slot, first position)
  const int row0 = a.row_off + blk.x, rows = blk.y, p0 = blk.w;
  const int slot = a.kv_map ? a.kv_map[blk.z] : blk.z;  // index in this KV block
  const int qh = blockIdx.y;
  const int hk = qh / (a.H / a.Hkv);
  const int rows_a = min(rows, 128), rows_b = max(0, rows - 128);
  const int last_pos = p0 + rows - 1;
  const int nk_a = (p0 + rows_a - 1) / KB + 1, nk_b = rows_b > 0 ? (p0 + 128 + rows_b - 1) / KB + 1 : 0;
  const int nk = max(nk_a, nk_b);
  const int zt = nk_b == nk ? 1 : 0;  // the tile that zeroes the last block's V rows past the sequence

  if (warp == 0) {  // Q of both tiles, then K blocks
    if (elect_one()) {
      const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
      mbar_arrive_expect_tx(bar_q, C::kQ);
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int r = 0; r < NR; ++r)
          tma_load_2d(&mq, bar_q, sQ + (t * NR + r) * C::kQBox, qh * HD + r * 64, row0 + t * 128, pol_q);
      const int kv_row0 = slot * a.max_ctx;
      for (int j = 0; j < nk; ++j) {
        const int s = j % ST;
        if (j >= ST) mbar_wait(k_empty + s, ((j / ST) + 1) & 1);
        mbar_arrive_expect_tx(k_full + s, C::kK);
#pragma unroll
        for (int r = 0; r < NR; ++r)
          tma_load_2d(&mkv, k_full + s, sK + s * C::kK + r * C::kKVBox, hk * HD + r * 64, kv_row0 + j * KB, pol_kv);
      }
    }
    __syncwarp();
  } else if (warp == 10) {  // V blocks
    if (elect_one()) {
      const uint64_t pol_kv = policy_evict_last();
      const int kv_row0 = slot * a.max_ctx;
      for (int j = 0; j < nk; ++j) {
        const int s = j % ST;
        if (j >= ST) mbar_wait(v_empty + s, ((j / ST) + 1) & 1);
        mbar_arrive_expect_tx(v_full + s, C::kV);
#pragma unroll
        for (int r = 0; r < NR; ++r)
          tma_load_2d(&mkv, v_full + s, sV + s * C::kV + r * C::kKVBox, (a.Hkv + hk) * HD + r * 64,
                      kv_row0 + j * KB, pol_kv);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = make_idesc_bf16(128, KB);
    constexpr uint32_t idesc_o = make_idesc_bf16(128, HD) | (1u << 16);  // B (V) MN-major
    mbar_wait(bar_q, 0);
    for (int j = 0; j <= nk; ++j) {
      if (j < nk) {  // S_A(j), S_B(j)
        const int s = j % ST, b = j & 1;
        mbar_wait(k_full + s, (j / ST) & 1);
        const uint32_t k0 = smem_u32(sK + s * C::kK);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (j >= (t ? nk_b : nk_a)) continue;
          if (j >= 2) mbar_wait(s_free + t * 2 + b, ((j >> 1) + 1) & 1);
          tc_fence_after();
          const uint32_t q0 = smem_u32(sQ + t * NR * C::kQBox);
#pragma unroll
          for (int g = 0; g < NR; ++g)
            umma4_elect<2>(tmem + t * 128 + b * 64, make_sw128_desc(q0 + g * C::kQBox),
                           make_sw128_desc(k0 + g * C::kKVBox), idesc_s, g > 0);
          umma_commit_elect(s_full + t * 2 + b);
          if (lane == 0) PFT(2 + t, j);
        }
        umma_commit_elect(k_empty + s);
      }
      if (j >= 1) {  // PV_A(j-1), PV_B(j-1)
        const int jj = j - 1, s = jj % ST;
        mbar_wait(v_full + s, (jj / ST) & 1);
        if (jj == nk - 1) mbar_wait(p_full + zt, jj & 1);  // V rows past the sequence zeroed
        const uint32_t v0 = smem_u32(sV + s * C::kV);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (jj >= (t ? nk_b : nk_a)) continue;
          mbar_wait(p_full + t, jj & 1);
          tc_fence_after();
          // P(jj) lives in the first 32 columns of tile t's S buffer jj & 1
          umma4_ts_elect<128>(tmem + 256 + t * 128, tmem + t * 128 + (jj & 1) * 64,
                              make_sw128_mn_desc(v0, C::kKVBox), idesc_o, jj > 0 ? 1u : 0u);
          umma_commit_elect(o_done + t);
          if (lane == 0) PFT(4 + t, jj);
        }
        umma_commit_elect(v_empty + s);
      }
    }
    __syncwarp();
  } else {
    // softmax of tile t (warps 2-5: A, 6-9: B): thread = query row r = TMEM lane
    const int t = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = uint32_t(q4 * 32) << 16;
    const int pt = p0 + t * 128;  // the tile's first position
    const int nk_t = t ? nk_b : nk_a, rows_t = t ? rows_b : rows_a;
    const int qp = pt + r;
    const float sl2 = a.scale * 1.4426950408889634f;
    float m_used = -INFINITY, l = 0.f;
    const uint32_t tS = tmem + lane_off + t * 128, tO = tmem + lane_off + 256 + t * 128;
    for (int j = 0; j < nk_t; ++j) {
      const int b = j & 1;
      mbar_wait(s_full + t * 2 + b, (j >> 1) & 1);
      if (q4 == 0 && lane == 0) PFT(t ? 10 : 6, j);
      tc_fence_after();
      float v[KB];
      {
        uint32_t u0[32], u1[32];
        tmem_ld32(tS + b * 64, u0);
        tmem_ld32(tS + b * 64 + 32, u1);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          v[e] = __uint_as_float(u0[e]);
          v[32 + e] = __uint_as_float(u1[e]);
        }
      }
      tc_fence_before();
      mbar_arrive(s_free + t * 2 + b);
      const int kbase = j * KB;
      if (kbase + KB - 1 > pt) {  // (tile-uniform) causal mask on raw scores
#pragma unroll
        for (int c = 0; c < KB; ++c)
          if (kbase + c > qp) v[c] = -INFINITY;
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < KB; ++c) mx = fmaxf(mx, v[c]);
      mx *= sl2;  // row max in the scaled log2 domain
      float alpha = 1.f;
      bool need = false;
      if (j == 0) {
        m_used = mx;
      } else {
        need = mx > m_used + 8.f;
        if (need) {
          alpha = fast_exp2(m_used - mx);
          m_used = mx;
        }
      }
      float rs = 0.f;
      uint32_t pk[KB / 2];
#pragma unroll
      for (int e = 0; e < KB / 2; ++e) {
        const float e0 = fast_exp2(fmaf(v[2 * e], sl2, -m_used));
        const float e1 = fast_exp2(fmaf(v[2 * e + 1], sl2, -m_used));
        rs += e0 + e1;
        pk[e] = pack_bf16x2(e0, e1);
      }
      if (t == 0 && q4 == 0 && lane == 0) PFT(7, j);
      // P(j) as bf16 pairs over the S(j) columns just read: the A operand of PV(j)
      // (S(j+2) overwrites them only after PV(j): the tensor pipe runs in order)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t ph[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) ph[e] = pk[h * 16 + e];
        tmem_st16(tS + b * 64 + h * 16, ph);
      }
      if (j > 0) {
        // every PV completion is consumed in order (an mbarrier parity wait is only
        // valid one phase ahead); the lazy rescale needs PV(j-1) retired anyway
        mbar_wait(o_done + t, (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, need)) {
#pragma unroll
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t u[32];
            tmem_ld32(tO + c * 32, u);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) u[e] = __float_as_uint(__uint_as_float(u[e]) * alpha);
            tmem_st32(tO + c * 32, u);
          }
          tmem_st_wait();
        }
      }
      tmem_st_wait();
      l = l * alpha + rs;
      if (t == zt && j == nk - 1 && kbase + KB - 1 > last_pos) {
        // last block: V rows past the sequence's last position -> 0 (P is 0 there)
        const int s = j % ST;
        mbar_wait(v_full + s, (j / ST) & 1);
        if (r < KB && kbase + r > last_pos) {
          uint8_t* vrow = sV + s * C::kV + r * 128;
#pragma unroll
          for (int g = 0; g < NR; ++g)
#pragma unroll
            for (int ch = 0; ch < 8; ++ch)
              *reinterpret_cast<uint4*>(vrow + g * C::kKVBox + ch * 16) = make_uint4(0, 0, 0, 0);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full + t);
      if (q4 == 0 && lane == 0) PFT(t ? 11 : 8, j);
    }
    if (nk_t > 0) {
      mbar_wait(o_done + t, (nk_t - 1) & 1);
      tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      uint16_t* out = a.out + (size_t)(row0 + t * 128 + r) * a.H * HD + (size_t)qh * HD;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t u[32];
        tmem_ld32(tO + c * 32, u);
        tmem_ld_wait();
        if (r < rows_t) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint4 w;
            w.x = pack_bf16x2(__uint_as_float(u[8 * e + 0]) * inv, __uint_as_float(u[8 * e + 1]) * inv);
            w.y = pack_bf16x2(__uint_as_float(u[8 * e + 2]) * inv, __uint_as_float(u[8 * e + 3]) * inv);
            w.z = pack_bf16x2(__uint_as_float(u[8 * e + 4]) * inv, __uint_as_float(u[8 * e + 5]) * inv);
            w.w = pack_bf16x2(__uint_as_float(u[8 * e + 6]) * inv, __uint_as_float(u[8 * e + 7]) * inv);
            *reinterpret_cast<uint4*>(out + c * 32 + e * 8) = w;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) PFT(9, 1);
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <int HD>
static cudaError_t launch_hd(const AttnArgs& a, const int4* blocks, int nblocks, cudaStream_t st) {
  using C = PpCfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(prefill_attn_pp_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const uint64_t qkv_n = uint64_t(a.H + 2 * a.Hkv) * HD;
  const uint64_t kv_n = uint64_t(2 * a.Hkv) * HD;
  CUtensorMap mq, mkv;
  if (make_kmajor_map(&mq, a.qkv, uint64_t(a.qkv_rows), qkv_n, qkv_n, 128) != 0 ||
      make_kmajor_map(&mkv, a.kv, uint64_t(a.kv_slots) * a.max_ctx, kv_n, kv_n, C::kKeys) != 0)
    return cudaErrorInvalidValue;
  const dim3 grid(unsigned(nblocks), unsigned(a.H));
  return launch_pdl(prefill_attn_pp_kernel<HD>, grid, dim3(kPfThreads), size_t(C::kSmem), st, mq, mkv, a, blocks);
}

cudaError_t prefill_attention_launch(const AttnArgs& a, const int4* blocks, int nblocks, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  if (a.qkv_rows <= 0 || a.kv_slots <= 0) return cudaErrorInvalidValue;
  switch (a.hd) {
    case 64: return launch_hd<64>(a, blocks, nblocks, st);
    case 128: return launch_hd<128>(a, blocks, nblocks, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace cb
