// Causal prefill attention on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Prefill rows of one sequence are contiguous in qkv and their K/V were just
// appended to the slot's cache (rope_kv_kernel).  CTA = (128-row query block of
// one sequence, q head); 11 warps, warp-specialised:
//
//   warps 0, 10 TMA producers: the Q tile once, then K and V blocks of 128
//               cached positions (SWIZZLE_128B boxes of 64 columns x 128 rows
//               straight from the [slot][pos][k|v] cache) into a K ring
//               (freed when S_j retires, warp 0) and a 2-stage V ring
//               (freed when PV_j retires, warp 10)
//   warp 1      MMA issuer (one elected lane of a converged warp):
//               S_j = Q K_j^T   (M 128 x N 128 x K hd, both K-major) into one of
//                                two TMEM S buffers, issued one block ahead
//                                when K_j has landed (else after PV_{j-1});
//               O  += P_j V_j   (M 128 x N hd x K 128; P K-major from smem, V
//                                MN-major: the cache's [pos][hd] rows as is)
//   warps 2..9  softmax, two threads per query row (TMEM lane), one per half
//               of the block's columns: S half-row -> registers (tcgen05.ld),
//               causal mask, row max exchanged between the halves through
//               smem, online softmax in the exp2 domain (one FFMA + MUFU.EX2 per
//               score) with lazy rescaling (O in TMEM is rescaled with
//               tcgen05.ld/st only when a row max grows by > 2^8), P as bf16
//               into smem in the 128-byte-swizzled K-major layout the MMA
//               reads; finally O / l -> bf16 -> global.  Two warps per SM
//               sub-partition hide the MUFU / FFMA latencies one warp could not.
//
// TMEM: S double buffer (2 x 128 columns) + O (hd columns).  Smem (hd 128):
// Q 32 KB + 2 x K 32 KB + 2 x V 32 KB + P 32 KB = 192 KB (hd 64: 3 K stages).
// Positions past the sequence's last row inside the last key block are masked
// in S, and their V rows are zeroed in smem before the PV MMA (stale cache
// bytes could hold non-finite values; 0 * NaN would poison the row).
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

static constexpr int kPfRows = 128;  // query rows per CTA = UMMA M = TMEM lanes
static constexpr int kPfKeys = 128;  // cached positions per K/V block = UMMA N of S = UMMA K of PV
static constexpr int kPfThreads = 352;  // 11 warps: K producer, MMA, 8 softmax, V producer

template <int HD>
struct PfCfg {
  static constexpr int kRegion = kPfRows * 128;  // one [128 rows][64 bf16] swizzled box: 16 KB
  static constexpr int kQ = kPfRows * HD * 2;
  static constexpr int kK = kPfKeys * HD * 2;
  static constexpr int kV = kPfKeys * HD * 2;
  static constexpr int kP = kPfRows * kPfKeys * 2;
  static constexpr int kBars = 18 * 8 + 6 * 128 * 4;  // barriers + the softmax halves' max / sum exchange
  static constexpr int kKStages = HD == 64 ? 3 : 2, kVStages = 2;  // K is released after S, V after PV
  static constexpr int kSmem = 1024 + kQ + kKStages * kK + kVStages * kV + kP + kBars;
  static constexpr uint32_t kTmemCols = 512;  // S0 [0,128) S1 [128,256) O [256, 256 + HD)
};

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

template <int HD>
__global__ void __launch_bounds__(kPfThreads, 1)
    prefill_attn_tc_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mkv,
                           const AttnArgs a, const int4* __restrict__ blocks) {
  using C = PfCfg<HD>;
  constexpr int NR = HD / 64;  // 64-column boxes per Q / K / V tile
  extern __shared__ uint8_t pf_raw[];
  uint8_t* sm = pf_raw + ((1024 - (smem_u32(pf_raw) & 1023)) & 1023);
  uint8_t* sQ = sm;
  uint8_t* sK = sQ + C::kQ;                 // [kKStages]
  uint8_t* sV = sK + C::kKStages * C::kK;   // [2 stages]
  uint8_t* sP = sV + C::kVStages * C::kV;   // [2 boxes of 64 keys]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + C::kP);
  uint64_t* bar_q = bars + 0;
  uint64_t* k_full = bars + 1;   // [3]
  uint64_t* k_empty = bars + 4;  // [3]
  uint64_t* v_full = bars + 7;   // [2]
  uint64_t* v_empty = bars + 9;  // [2]
  uint64_t* s_full = bars + 11;  // [2]
  uint64_t* s_free = bars + 13;  // [2]
  uint64_t* p_full = bars + 15;
  uint64_t* o_done = bars + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < C::kKStages; ++i) {
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
      mbar_init(s_full + i, 1);
      mbar_init(s_free + i, 256);
    }
    mbar_init(p_full, 256);
    mbar_init(o_done, 1);
    fence_barrier_init();
    tma_prefetch_desc(&mq);
    tma_prefetch_desc(&mkv);
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // q rotated and K/V appended by rope_kv_kernel
  if (threadIdx.x == 0) PFT(9, 0);

  const int4 blk = blocks[blockIdx.x];  // (first row, rows, slot, first position)
  const int row0 = a.row_off + blk.x, nrows = blk.y, p0 = blk.w;
  const int slot = a.kv_map ? a.kv_map[blk.z] : blk.z;  // index in this KV block
  const int qh = blockIdx.y;
  const int hk = qh / (a.H / a.Hkv);
  const int last_pos = p0 + nrows - 1;
  const int nkb = last_pos / kPfKeys + 1;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
      mbar_arrive_expect_tx(bar_q, C::kQ);
#pragma unroll
      for (int r = 0; r < NR; ++r) tma_load_2d(&mq, bar_q, sQ + r * C::kRegion, qh * HD + r * 64, row0, pol_q);
      const int kv_row0 = slot * a.max_ctx;
      constexpr int KS = C::kKStages;
      auto load_k = [&](int j) {  // stage j % KS, free once S_{j-KS} retired
        const int s = j % KS;
        if (j >= KS) mbar_wait(k_empty + s, ((j / KS) + 1) & 1);
        mbar_arrive_expect_tx(k_full + s, C::kK);
#pragma unroll
        for (int r = 0; r < NR; ++r)
          tma_load_2d(&mkv, k_full + s, sK + s * C::kK + r * C::kRegion, hk * HD + r * 64, kv_row0 + j * kPfKeys,
                      pol_kv);
        PFT(0, j);
      };
      for (int j = 0; j < nkb; ++j) load_k(j);
    }
    __syncwarp();
  } else if (warp == 10) {  // V producer: its ring waits on PV, which must not hold back the K loads
    if (elect_one()) {
      const uint64_t pol_kv = policy_evict_last();
      const int kv_row0 = slot * a.max_ctx;
      for (int j = 0; j < nkb; ++j) {
        const int s = j & 1;
        if (j >= 2) mbar_wait(v_empty + s, ((j >> 1) + 1) & 1);
        mbar_arrive_expect_tx(v_full + s, C::kV);
#pragma unroll
        for (int r = 0; r < NR; ++r)
          tma_load_2d(&mkv, v_full + s, sV + s * C::kV + r * C::kRegion, (a.Hkv + hk) * HD + r * 64,
                      kv_row0 + j * kPfKeys, pol_kv);
        PFT(1, j);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = make_idesc_bf16(kPfRows, kPfKeys);
    constexpr uint32_t idesc_o = make_idesc_bf16(kPfRows, HD) | (1u << 16);  // B (V) MN-major
    const uint32_t tO = tmem + 256;
    mbar_wait(bar_q, 0);
    auto issue_s = [&](int j) {
      const int s = j & 1, ks = j % C::kKStages;
      mbar_wait(k_full + ks, (j / C::kKStages) & 1);
      if (j >= 2) mbar_wait(s_free + s, ((j >> 1) + 1) & 1);
      tc_fence_after();
      const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK + ks * C::kK);
#pragma unroll
      for (int g = 0; g < NR; ++g)  // 64 head dims (one box) per group of 4 MMAs
        umma4_elect<2>(tmem + s * 128, make_sw128_desc(q0 + g * C::kRegion), make_sw128_desc(k0 + g * C::kRegion),
                       idesc_s, g > 0);
      umma_commit_elect(s_full + s);
      umma_commit_elect(k_empty + ks);
      if (lane == 0) PFT(2, j);
    };
    issue_s(0);
    for (int j = 0; j < nkb; ++j) {
      const int s = j & 1;
      // S_{j+1} ahead of PV_j (the softmax of j+1 then starts as soon as j's is
      // done) -- unless K_{j+1} has not landed: PV_j must not wait on that load
      bool ahead = false;
      if (j + 1 < nkb) {
        const int n = j + 1;
        bool ok = mbar_test(k_full + n % C::kKStages, (n / C::kKStages) & 1) &&
                  (n < 2 || mbar_test(s_free + (n & 1), ((n >> 1) + 1) & 1));
        ahead = __shfl_sync(0xffffffffu, ok, 0);
        if (ahead) issue_s(n);
      }
      mbar_wait(p_full, j & 1);
      if (lane == 0) PFT(3, j);
      mbar_wait(v_full + s, (j >> 1) & 1);
      if (lane == 0) PFT(10, j);
      tc_fence_after();
      const uint32_t p0a = smem_u32(sP), v0 = smem_u32(sV + s * C::kV);
#pragma unroll
      for (int g = 0; g < kPfKeys / 64; ++g)  // 64 keys (one P box, 64 V rows) per group of 4 MMAs
        umma4_elect<128>(tO, make_sw128_desc(p0a + g * C::kRegion), make_sw128_mn_desc(v0 + g * 8192, C::kRegion),
                         idesc_o, (j > 0 || g > 0) ? 1u : 0u);
      if (lane == 0) PFT(11, j);
      umma_commit_elect(o_done);
      umma_commit_elect(v_empty + s);
      if (lane == 0) PFT(4, j);
      if (j + 1 < nkb && !ahead) issue_s(j + 1);
    }
    __syncwarp();
  } else if (warp >= 2 && warp <= 9) {
    // softmax: two warps per query row quarter (warp w may touch TMEM lanes
    // 32 (w % 4) ..); thread = (row r = TMEM lane, column half hh): 64 of the
    // block's 128 scores and hd / 2 of the O columns.  The two halves of a row
    // exchange their partial row max through smem each block (named barrier
    // of the quarter's 64 threads) and their partial sums at the end.
    constexpr int KH = kPfKeys / 2, OH = HD / 2;
    const int q4 = warp & 3, hh = (warp - 2) >> 2;
    const int r = q4 * 32 + lane;
    const uint32_t lane_off = uint32_t(q4 * 32) << 16;
    const int qp = p0 + r;
    const float sl2 = a.scale * 1.4426950408889634f;
    float m_used = -INFINITY, l = 0.f;
    uint8_t* prow = sP + hh * C::kRegion + r * 128;
    const int rsw = r & 7;
    float* red = reinterpret_cast<float*>(bars + 18);  // [2 blocks][2 halves][128 rows]
    for (int j = 0; j < nkb; ++j) {
      const int s = j & 1;
      mbar_wait(s_full + s, (j >> 1) & 1);
      if (warp == 2 && lane == 0) PFT(5, j);
      tc_fence_after();
      float v[KH];
      {
        uint32_t u0[32], u1[32];
        tmem_ld32(tmem + lane_off + s * 128 + hh * KH, u0);
        tmem_ld32(tmem + lane_off + s * 128 + hh * KH + 32, u1);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          v[e] = __uint_as_float(u0[e]);
          v[32 + e] = __uint_as_float(u1[e]);
        }
      }
      tc_fence_before();
      mbar_arrive(s_free + s);
      const int kbase = j * kPfKeys + hh * KH;
      if (j * kPfKeys + kPfKeys - 1 > p0) {  // (block-uniform) causal mask on raw scores
#pragma unroll
        for (int c = 0; c < KH; ++c)
          if (kbase + c > qp) v[c] = -INFINITY;
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < KH; ++c) mx = fmaxf(mx, v[c]);
      red[((j & 1) * 2 + hh) * 128 + r] = mx;
      named_bar_sync(1 + q4, 64);
      mx = fmaxf(mx, red[((j & 1) * 2 + (hh ^ 1)) * 128 + r]) * sl2;  // row max, scaled log2 domain
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
      // P = exp2(S - m) packed to bf16 in registers while PV_{j-1} may still run
      float rs = 0.f;
      uint32_t pk[KH / 2];
#pragma unroll
      for (int e = 0; e < KH / 2; ++e) {
        const float e0 = fast_exp2(fmaf(v[2 * e], sl2, -m_used));  // FFMA + MUFU.EX2 per score
        const float e1 = fast_exp2(fmaf(v[2 * e + 1], sl2, -m_used));
        rs += e0 + e1;
        pk[e] = pack_bf16x2(e0, e1);
      }
      if (warp == 2 && lane == 0) PFT(6, j);
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);  // PV_{j-1} retired: O is final for j-1 and P is free
        if (warp == 2 && lane == 0) PFT(7, j);
        tc_fence_after();
        if (__any_sync(0xffffffffu, need)) {  // lazy rescale: only when a row max grew by > 2^8
#pragma unroll
          for (int c = 0; c < OH / 32; ++c) {
            uint32_t u[32];
            tmem_ld32(tmem + lane_off + 256 + hh * OH + c * 32, u);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) u[e] = __float_as_uint(__uint_as_float(u[e]) * alpha);
            tmem_st32(tmem + lane_off + 256 + hh * OH + c * 32, u);
          }
          tmem_st_wait();
        }
      }
#pragma unroll
      for (int ch = 0; ch < KH / 8; ++ch) {  // 16-byte chunks of 8 keys, 128-byte swizzle
        uint8_t* dst = prow + ((ch ^ rsw) << 4);
        *reinterpret_cast<uint4*>(dst) = make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
      }
      l = l * alpha + rs;
      if (j * kPfKeys + kPfKeys - 1 > last_pos) {
        // last block: V rows past the sequence's last position -> 0 (P is 0 there)
        mbar_wait(v_full + s, (j >> 1) & 1);
        if (j * kPfKeys + r > last_pos) {
          uint8_t* vrow = sV + s * C::kV + r * 128;
#pragma unroll
          for (int b = 0; b < NR; ++b)
            if ((b & 1) == hh)
#pragma unroll
              for (int ch = 0; ch < 8; ++ch)
                *reinterpret_cast<uint4*>(vrow + b * C::kRegion + ch * 16) = make_uint4(0, 0, 0, 0);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
      if (warp == 2 && lane == 0) PFT(8, j);
    }
    red[(4 + hh) * 128 + r] = l;  // the two halves' row sums
    named_bar_sync(1 + q4, 64);
    l += red[(4 + (hh ^ 1)) * 128 + r];
    mbar_wait(o_done, (nkb - 1) & 1);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    uint16_t* out = a.out + (size_t)(row0 + r) * a.H * HD + (size_t)qh * HD + hh * OH;
#pragma unroll
    for (int c = 0; c < OH / 32; ++c) {
      uint32_t u[32];
      tmem_ld32(tmem + lane_off + 256 + hh * OH + c * 32, u);
      tmem_ld_wait();
      if (r < nrows) {
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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) PFT(9, 1);
  if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem);
}

template <int HD>
static cudaError_t launch_hd(const AttnArgs& a, const int4* blocks, int nblocks, cudaStream_t st) {
  using C = PfCfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(prefill_attn_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const uint64_t qkv_n = uint64_t(a.H + 2 * a.Hkv) * HD;
  const uint64_t kv_n = uint64_t(2 * a.Hkv) * HD;
  CUtensorMap mq, mkv;
  if (make_kmajor_map(&mq, a.qkv, uint64_t(a.qkv_rows), qkv_n, qkv_n, kPfRows) != 0 ||
      make_kmajor_map(&mkv, a.kv, uint64_t(a.kv_slots) * a.max_ctx, kv_n, kv_n, kPfKeys) != 0)
    return cudaErrorInvalidValue;
  const dim3 grid(unsigned(nblocks), unsigned(a.H));
  return launch_pdl(prefill_attn_tc_kernel<HD>, grid, dim3(kPfThreads), size_t(C::kSmem), st, mq, mkv, a, blocks);
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
