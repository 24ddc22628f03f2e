// Kernel-level test entry points (include/cocob200_testing.h).  Thin wrappers
// that build tensor maps / workspaces for caller-owned device buffers.
#include <cmath>
#include <cstring>
#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "../../include/cocob200.h"
#include "../../include/cocob200_testing.h"
#include "common.cuh"
#include "kernels.h"

namespace {

struct TestWs {
  float* gemm_ws = nullptr;
  int* cnt = nullptr;
  float* attn_ws = nullptr;
  size_t attn_floats = 0;
  int* attn_cnt = nullptr;
  int sms = 148;
};

std::map<int, TestWs> g_ws;
unsigned long long g_trace[148 * 512];
int g_wcopies = 1;          // experiments: rotate over this many weight copies ...
int64_t g_wcopy_stride = 0; // ... this many bytes apart (defeats L2 residency of the weight)

int ws_for_current(TestWs** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return CB_ECUDA;
  TestWs& w = g_ws[dev];
  if (!w.gemm_ws) {
    cudaDeviceGetAttribute(&w.sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaMalloc(&w.gemm_ws, cb::gemm_ws_floats(w.sms) * 4) != cudaSuccess) return CB_ECUDA;
    if (cudaMalloc(&w.cnt, size_t(cb::kGemmMaxTiles) * 4) != cudaSuccess) return CB_ECUDA;
    cudaMemset(w.cnt, 0, size_t(cb::kGemmMaxTiles) * 4);
    w.attn_floats = size_t(1) << 24;
    if (cudaMalloc(&w.attn_ws, w.attn_floats * 4) != cudaSuccess) return CB_ECUDA;
    if (cudaMalloc(&w.attn_cnt, size_t(1 << 16) * 4) != cudaSuccess) return CB_ECUDA;
    cudaMemset(w.attn_cnt, 0, size_t(1 << 16) * 4);
  }
  *out = &w;
  return CB_OK;
}

int finish(cudaError_t e) {
  if (e != cudaSuccess) return CB_ECUDA;
  return cudaDeviceSynchronize() == cudaSuccess ? CB_OK : CB_ECUDA;
}

// fused-RMSNorm fields applied to every cbt_gemm / cbt_gemm_bench launch (cbt_gemm_set_norm)
struct NormFields {
  const float* ssq_in = nullptr;
  uint16_t* h_out = nullptr;
  const uint16_t* gamma_next = nullptr;
  float* ssq_out = nullptr;
  int np = 0, d = 0;
  float eps = 0.f;
} g_norm;

void apply_norm(cb::GemmArgs& a) {
  a.ssq_in = g_norm.ssq_in;
  a.h_out = g_norm.h_out;
  a.gamma_next = g_norm.gamma_next;
  a.ssq_out = g_norm.ssq_out;
  a.ssq_np = g_norm.np;
  a.norm_d = g_norm.d;
  a.norm_eps = g_norm.eps;
}

int gemm_setup(const void* w, const void* x, int64_t x_rows, int N, int K, const cb::GemmPlan& plan,
               CUtensorMap* mw, CUtensorMap* mx) {
  if (plan.kd == 2) {  // 3-D views for the 2-k-block-per-stage kernel
    if (cb::make_kmajor_map3(mw, w, N, K, K, 128, 2) != 0) return CB_ECUDA;
    if (cb::make_kmajor_map3(mx, x, x_rows, K, K, plan.box_rows, 2) != 0) return CB_ECUDA;
    return CB_OK;
  }
  if (cb::make_kmajor_map(mw, w, N, K, K, 128) != 0) return CB_ECUDA;
  if (cb::make_kmajor_map(mx, x, x_rows, K, K, plan.box_rows) != 0) return CB_ECUDA;
  return CB_OK;
}

}  // namespace

extern "C" {

int cbt_gemm(const void* w, const void* x, int64_t x_rows, int32_t N, int32_t K, int32_t T, int32_t row_off,
             int32_t epi, void* out, int64_t ldo) {
  TestWs* ws;
  int r = ws_for_current(&ws);
  if (r) return r;
  const cb::GemmPlan plan = cb::gemm_plan(N, K, T, ws->sms);
  CUtensorMap mw, mx;
  if ((r = gemm_setup(w, x, x_rows, N, K, plan, &mw, &mx))) return r;
  cb::GemmArgs a{};
  a.N = N;
  a.K = K;
  a.T = T;
  a.row_off = row_off;
  a.epi = epi;
  a.ldo = ldo;
  a.out_rows = row_off + T;
  a.w_base = w;
  a.w_stride = K;
  a.out = out;
  a.ws = ws->gemm_ws;
  a.counters = ws->cnt;
  apply_norm(a);
  CUtensorMap mo;
  const uint64_t ocols = epi == cb::EPI_SWIGLU ? uint64_t(N) / 2 : uint64_t(N);
  const bool tma = cb::make_out_map(&mo, out, epi, uint64_t(row_off + T), ocols, uint64_t(ldo)) == 0;
  return finish(cb::gemm_launch(mw, mx, a, plan, ws->sms, 0, tma ? &mo : nullptr));
}

// The plan gemm_plan picks (host-only): tn, pair, box_rows, csplit, max_parts, whole, kd, nw, ksplit.
int cbt_gemm_plan(int32_t N, int32_t K, int32_t T, int32_t num_sms, int32_t kind_T, int32_t* out) {
  const cb::GemmPlan p = cb::gemm_plan(N, K, T, num_sms, kind_T);
  const int32_t v[9] = {p.tn, p.pair, p.box_rows, p.csplit, p.max_parts, p.whole, p.kd, p.nw, p.ksplit};
  for (int i = 0; i < 9; ++i) out[i] = v[i];
  return CB_OK;
}

int cbt_gemm_bench(const void* w, const void* x, int64_t x_rows, int32_t N, int32_t K, int32_t T, int32_t epi,
                   void* out, int64_t ldo, int32_t iters, int32_t max_parts, float* ms_per_launch) {
  TestWs* ws;
  int r = ws_for_current(&ws);
  if (r) return r;
  cb::GemmPlan plan = cb::gemm_plan(N, K, T, ws->sms);
  // knob + sign * 1000 * dbg bits (negative knobs keep their sign: -4 - 8000)
  const int dbg_bits = (max_parts < 0 ? -max_parts : max_parts) / 1000;
  max_parts = max_parts < 0 ? -((-max_parts) % 1000) : max_parts % 1000;
  // experiment knobs: 201 / 202 force the CTA-pair kernel (256 / 128-token
  // tiles), 203 forces the 1-CTA kernel, < 0 forces cluster split -max_parts,
  // 1..99 cap the stream-K parts per tile
  if (max_parts == 201 || max_parts == 202) {
    plan = cb::GemmPlan{max_parts == 201 ? 256 : 128, 1, max_parts == 201 ? 128 : 64, 1, 0};
  } else if (max_parts > 300 && max_parts <= 308) {  // token-major pair kernel, nw = 32 * (knob - 300)
    plan = cb::GemmPlan{256, 1, 128, 1, 0};
    plan.whole = 1;
    plan.nw = 32 * (max_parts - 300);
  } else if (max_parts == 352 || max_parts == 354 || max_parts == 362) {  // token-major pairs, K split
    plan = cb::GemmPlan{256, 1, 128, 1, 0};   // 35x: 256 weight rows, K split in 2 / 4; 362: 128 rows, split 2
    plan.whole = 1;
    plan.nw = max_parts == 362 ? 128 : 256;
    plan.ksplit = max_parts % 10;
  } else if (max_parts > 400 && max_parts <= 408) {  // 1-CTA kernel, 128-token tiles, cluster split (knob - 400)
    plan = cb::GemmPlan{128, 0, 128, max_parts - 400, 0};
  } else if (max_parts > 410 && max_parts <= 418) {  // 1-CTA kernel, 64-token tiles, cluster split (knob - 410)
    plan = cb::GemmPlan{64, 0, 64, max_parts - 410, 0};
  } else if (max_parts == 203 && plan.pair) {
    plan = cb::GemmPlan{cb::gemm_pick_tn(T), 0, cb::gemm_pick_tn(T), 1, 0};
  } else if (max_parts < 0) {  // 1-CTA kernel with cluster split -max_parts
    plan = cb::GemmPlan{cb::gemm_pick_tn(T), 0, cb::gemm_pick_tn(T), -max_parts, 0};
  } else if (max_parts > 0 && max_parts < 100 && !plan.pair) {
    plan.csplit = 1;
  } else if (max_parts == 99) {
    plan.max_parts = 0;  // experiments: force stream-K
  }
  if (dbg_bits & 4) plan.kd = 1;  // tile-major weight experiment uses 2-D maps
  if (dbg_bits & 512) plan.whole = 1, plan.max_parts = 0, plan.csplit = plan.pair ? 1 : plan.csplit;  // whole tiles
  if (dbg_bits & 1024) plan.whole = 0;                                                          // stream-K
  CUtensorMap mw, mx;
  if ((r = gemm_setup(w, x, x_rows, N, K, plan, &mw, &mx))) return r;
  const bool tiled = (dbg_bits & 4) != 0;  // w holds the tile-major layout
  std::vector<CUtensorMap> mws(std::max(1, g_wcopies));
  for (size_t i = 0; i < mws.size(); ++i) {
    const void* wi = static_cast<const uint8_t*>(w) + i * g_wcopy_stride;
    int e = tiled           ? cb::make_kmajor_map(&mws[i], wi, uint64_t(N) * (K / 64), 64, 64, 128)
            : plan.kd == 2 ? cb::make_kmajor_map3(&mws[i], wi, N, K, K, 128, 2)
                           : cb::make_kmajor_map(&mws[i], wi, N, K, K, 128);
    if (e != 0) return CB_ECUDA;
  }
  cb::GemmArgs a{};
  a.w_tiled = tiled ? 1 : 0;
  a.N = N;
  a.K = K;
  a.T = T;
  a.epi = epi;
  a.ldo = ldo;
  a.out_rows = T;
  a.w_base = tiled ? nullptr : w;  // (weight copies: the token-major map follows the first copy)
  a.w_stride = K;
  a.out = out;
  a.ws = ws->gemm_ws;
  a.counters = ws->cnt;
  a.max_parts = (max_parts > 0 && max_parts < 100) ? max_parts : 0;
  apply_norm(a);
  static unsigned long long* trace = nullptr;
  if (dbg_bits & 8) {  // experiments: per-CTA timeline of the last launch -> g_trace
    if (!trace) cudaMalloc(&trace, 148 * 512 * 8);
    cudaMemset(trace, 0, 148 * 512 * 8);
    a.trace = trace;
  }
  a.dbg = dbg_bits & ~(4 | 8 | 256 | 512 | 1024);  // experiments: knob + 1000 * dbg bits (4 = tile-major weight, 256 = no TMA store)
  CUtensorMap mo;
  const uint64_t ocols = epi == cb::EPI_SWIGLU ? uint64_t(N) / 2 : uint64_t(N);
  const CUtensorMap* pmo =
      (!(dbg_bits & 256) && cb::make_out_map(&mo, out, epi, uint64_t(T), ocols, uint64_t(ldo)) == 0) ? &mo : nullptr;
  // launch with weight copy i (the token-major plan builds its weight map from w_base)
  auto launch = [&](int i) {
    const size_t ci = size_t(i) % mws.size();
    if (!tiled) a.w_base = static_cast<const uint8_t*>(w) + ci * g_wcopy_stride;
    return cb::gemm_launch(mws[ci], mx, a, plan, ws->sms, 0, pmo);
  };
  for (int i = 0; i < 3; ++i) launch(i);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, 0);
  for (int i = 0; i < iters; ++i) launch(i);
  cudaEventRecord(e1, 0);
  if (cudaEventSynchronize(e1) != cudaSuccess) return CB_ECUDA;
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  *ms_per_launch = ms / iters;
  if (a.trace) {
    cudaMemset(trace, 0, 148 * 512 * 8);
    launch(iters);
    cudaDeviceSynchronize();
    cudaMemcpy(g_trace, trace, sizeof(g_trace), cudaMemcpyDeviceToHost);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return finish(cudaGetLastError());
}

int cbt_rmsnorm(const float* x, const uint16_t* gamma, uint16_t* y, int32_t T, int32_t d, float eps) {
  return finish(cb::rmsnorm_launch(x, gamma, y, T, d, eps, 0, 0));
}

}  // extern "C"

namespace {
float2* rope_table_dev(int max_ctx, int hd, float theta) {
  const int half = hd / 2;
  std::vector<float2> tab(size_t(max_ctx) * half);
  for (int p = 0; p < max_ctx; ++p)
    for (int i = 0; i < half; ++i) {
      const double ang = double(p) * std::pow(double(theta), -2.0 * i / double(hd));
      tab[size_t(p) * half + i] = make_float2(float(std::cos(ang)), float(std::sin(ang)));
    }
  float2* dtab = nullptr;
  if (cudaMalloc(&dtab, tab.size() * sizeof(float2)) != cudaSuccess) return nullptr;
  cudaMemcpy(dtab, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice);
  return dtab;
}
}  // namespace

// slots of the KV buffer the fused decode attention may view through TMA (0 = the
// 16-byte-load kernel; > 0 lets attention_launch pick the TMA-fed kernel)
static int g_attn_kv_slots = 0;
extern "C" int cbt_attention_set_kv_slots(int32_t n) {
  g_attn_kv_slots = n < 0 ? 0 : n;
  return CB_OK;
}

extern "C" int cbt_attention_fused(const uint16_t* qkv, uint16_t* kv, uint16_t* out, const int32_t* row_slot,
                                   const int32_t* row_pos, int32_t T, int32_t H, int32_t Hkv, int32_t hd,
                                   int32_t max_ctx, float theta) {
  TestWs* ws;
  int r = ws_for_current(&ws);
  if (r) return r;
  float2* dtab = rope_table_dev(max_ctx, hd, theta);
  if (!dtab) return CB_ECUDA;
  std::vector<int32_t> pos(T);
  cudaMemcpy(pos.data(), row_pos, size_t(T) * 4, cudaMemcpyDeviceToHost);
  int max_len = 0;
  for (int v : pos) max_len = std::max(max_len, v + 1);
  cb::AttnArgs a{};
  a.qkv = qkv;
  a.kv = kv;
  a.out = out;
  a.row_slot = row_slot;
  a.row_pos = row_pos;
  a.ws = ws->attn_ws;
  a.counters = ws->attn_cnt;
  a.ws_floats = ws->attn_floats;
  a.T = T;
  a.H = H;
  a.Hkv = Hkv;
  a.hd = hd;
  a.max_ctx = max_ctx;
  a.max_len = max_len;
  a.scale = 1.0f / std::sqrt(float(hd));
  a.rope = dtab;
  a.kv_slots = g_attn_kv_slots;
  r = finish(cb::attention_launch(a, ws->sms, 0));
  cudaFree(dtab);
  return r;
}

extern "C" {

int cbt_rope_kv(uint16_t* qkv, uint16_t* kv, const int32_t* row_slot, const int32_t* row_pos, int32_t T, int32_t H,
                int32_t Hkv, int32_t hd, int32_t max_ctx, float theta) {
  const int half = hd / 2;
  std::vector<float2> tab(size_t(max_ctx) * half);
  for (int p = 0; p < max_ctx; ++p)
    for (int i = 0; i < half; ++i) {
      const double ang = double(p) * std::pow(double(theta), -2.0 * i / double(hd));
      tab[size_t(p) * half + i] = make_float2(float(std::cos(ang)), float(std::sin(ang)));
    }
  float2* dtab = nullptr;
  if (cudaMalloc(&dtab, tab.size() * sizeof(float2)) != cudaSuccess) return CB_ECUDA;
  cudaMemcpy(dtab, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice);
  int r = finish(cb::rope_kv_launch(qkv, kv, nullptr, dtab, row_slot, row_pos, T, 0, H, Hkv, hd, max_ctx, 0));
  cudaFree(dtab);
  return r;
}

int cbt_attention(const uint16_t* qkv, const uint16_t* kv, uint16_t* out, const int32_t* row_slot,
                  const int32_t* row_pos, int32_t T, int32_t H, int32_t Hkv, int32_t hd, int32_t max_ctx) {
  TestWs* ws;
  int r = ws_for_current(&ws);
  if (r) return r;
  std::vector<int32_t> pos(T);
  cudaMemcpy(pos.data(), row_pos, size_t(T) * 4, cudaMemcpyDeviceToHost);
  int max_len = 0;
  for (int v : pos) max_len = std::max(max_len, v + 1);
  cb::AttnArgs a{};
  a.qkv = qkv;
  a.kv = kv;
  a.out = out;
  a.row_slot = row_slot;
  a.row_pos = row_pos;
  a.ws = ws->attn_ws;
  a.counters = ws->attn_cnt;
  a.ws_floats = ws->attn_floats;
  a.T = T;
  a.H = H;
  a.Hkv = Hkv;
  a.hd = hd;
  a.max_ctx = max_ctx;
  a.max_len = max_len;
  a.scale = 1.0f / std::sqrt(float(hd));
  return finish(cb::attention_launch(a, ws->sms, 0));
}

int cbt_attention_bench(const uint16_t* qkv, const uint16_t* kv, uint16_t* out, const int32_t* row_slot,
                        const int32_t* row_pos, int32_t T, int32_t H, int32_t Hkv, int32_t hd, int32_t max_ctx,
                        int32_t max_len, int32_t iters, float* ms_per_launch) {
  TestWs* ws;
  int r = ws_for_current(&ws);
  if (r) return r;
  cb::AttnArgs a{};
  a.qkv = qkv;
  a.kv = kv;
  a.out = out;
  a.row_slot = row_slot;
  a.row_pos = row_pos;
  a.ws = ws->attn_ws;
  a.counters = ws->attn_cnt;
  a.ws_floats = ws->attn_floats;
  a.T = T;
  a.H = H;
  a.Hkv = Hkv;
  a.hd = hd;
  a.max_ctx = max_ctx;
  a.max_len = max_len;
  a.scale = 1.0f / std::sqrt(float(hd));
  for (int i = 0; i < 3; ++i) cb::attention_launch(a, ws->sms, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, 0);
  for (int i = 0; i < iters; ++i) cb::attention_launch(a, ws->sms, 0);
  cudaEventRecord(e1, 0);
  if (cudaEventSynchronize(e1) != cudaSuccess) return CB_ECUDA;
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  *ms_per_launch = ms / iters;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return finish(cudaGetLastError());
}

int cbt_argmax(const float* logits, int32_t* out, int32_t T, int32_t V) {
  return finish(cb::argmax_launch(logits, out, T, V, 0));
}

}  // extern "C"

// ---------------------------------------------------------------------------
// TMA read-bandwidth probe (experiments only): every CTA streams `iters` boxes
// of box_rows x 64 bf16 through an S-stage smem ring (one thread issues, the
// same thread waits), from a rows x 64 K-major region.  Small regions stay in
// L2, large ones stream from HBM: the per-SM and chip-wide TMA fill rates the
// GEMM kernels are bounded by.
namespace {
// warp w (< nw) streams its own S-stage ring; kd > 1 = 3-D boxes of kd k-slices
template <int S>
__global__ void __launch_bounds__(128, 1) tma_probe_kernel(const __grid_constant__ CUtensorMap tm, int rows,
                                                           int box_rows, int kd, int nw, int iters, int mma_n) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int box_bytes = box_rows * 128 * kd;
  const int w = threadIdx.x >> 5;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + nw * S * box_bytes) + w * S;
  __shared__ volatile int done;
  __shared__ uint32_t tslot;
  __shared__ uint64_t mbar;
  if (mma_n > 0) {
    // warp 3: back-to-back 128 x mma_n x 16 MMAs on a separate smem region while warps < nw stream TMA
    if (threadIdx.x == 0) done = 0;
    if (w == 3) cb::tmem_alloc<256>(&tslot);
    cb::tc_fence_before();
    __syncthreads();
    cb::tc_fence_after();
    if (w == 3) {
      if ((threadIdx.x & 31) == 0) {
        cb::mbar_init(&mbar, 1);
        cb::fence_barrier_init();
        uint8_t* ops = smem + nw * S * box_bytes + 4096;
        ops = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ops) + 1023) & ~uintptr_t(1023));
        const uint64_t da = cb::make_sw128_desc(cb::smem_u32(ops));
        const uint64_t db = cb::make_sw128_desc(cb::smem_u32(ops + 16384));
        const uint32_t idesc = cb::make_idesc_bf16(128, uint32_t(mma_n));
        uint32_t ph = 0;
        while (!done) {
          for (int i = 0; i < 64; ++i) cb::umma_bf16(tslot, da + uint64_t(2 * (i & 3)), db + uint64_t(2 * (i & 3)), idesc, 1u);
          cb::umma_commit(&mbar);
          cb::mbar_wait(&mbar, ph);
          ph ^= 1;
        }
      }
      __syncwarp();
      cb::tc_fence_before();
      cb::tmem_dealloc<256>(tslot);
      return;
    }
  }
  if (w >= nw || (threadIdx.x & 31) != 0) return;
  uint8_t* ring = smem + w * S * box_bytes;
  for (int i = 0; i < S; ++i) cb::mbar_init(&bar[i], 1);
  cb::fence_barrier_init();
  const uint64_t pol = cb::policy_evict_first();
  const int nbox = rows / box_rows;
  int next = 0;
  auto issue = [&](int i) {
    const int s = i % S;
    const int b = int(((long long)(blockIdx.x * nw + w) * iters + i) % nbox);  // disjoint chunks (HBM) / wraps (L2)
    cb::mbar_arrive_expect_tx(&bar[s], box_bytes);
    if (kd == 1)
      cb::tma_load_2d(&tm, &bar[s], ring + s * box_bytes, 0, b * box_rows, pol);
    else
      cb::tma_load_3d(&tm, &bar[s], ring + s * box_bytes, 0, b * box_rows, 0, pol);
  };
  for (; next < S && next < iters; ++next) issue(next);
  for (int i = 0; i < iters; ++i) {
    cb::mbar_wait(&bar[i % S], (i / S) & 1);
    if (next < iters) issue(next++);
  }
  if (mma_n > 0 && w == 0) done = 1;
}

}

extern "C" int cbt_tma_probe(const void* buf, int64_t rows, int32_t box_rows, int32_t stages, int32_t grid,
                             int32_t iters, int32_t kd, int32_t nw, int32_t mma_n, float* ms_out) {
  CUtensorMap tm;
  // region viewed as [rows][kd * 64] bf16; a 3-D box = (64, box_rows, kd) lands as kd SW128 sub-tiles
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return CB_ECUDA;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const int64_t r = rows / kd;
  cuuint64_t dims[3] = {64, cuuint64_t(r), cuuint64_t(kd)};
  cuuint64_t strides[2] = {cuuint64_t(kd) * 128, 128};
  cuuint32_t box[3] = {64, uint32_t(box_rows), uint32_t(kd)};
  cuuint32_t estr[3] = {1, 1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, kd == 1 ? 2 : 3, const_cast<void*>(buf), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return CB_EINVAL;
  const size_t smem = size_t(nw) * stages * box_rows * 128 * kd + 1024 + 512 + (mma_n > 0 ? 4096 + 1024 + 49152 : 0);
  auto run = [&](auto kern) -> int {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    kern<<<grid, 128, smem>>>(tm, int(r), box_rows, kd, nw, iters, mma_n);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<grid, 128, smem>>>(tm, int(r), box_rows, kd, nw, iters, mma_n);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) return CB_ECUDA;
    cudaEventElapsedTime(ms_out, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return cudaGetLastError() == cudaSuccess ? CB_OK : CB_ECUDA;
  };
  switch (stages) {
    case 1: return run(tma_probe_kernel<1>);
    case 2: return run(tma_probe_kernel<2>);
    case 4: return run(tma_probe_kernel<4>);
    case 8: return run(tma_probe_kernel<8>);
    case 16: return run(tma_probe_kernel<16>);
  }
  return CB_EINVAL;
}

extern "C" int cbt_gemm_trace(unsigned long long* out, int32_t n) {
  if (n > 148 * 512) n = 148 * 512;
  std::memcpy(out, g_trace, size_t(n) * 8);
  return CB_OK;
}

extern "C" int cbt_gemm_set_norm(const float* ssq_in, uint16_t* h_out, const uint16_t* gamma_next, float* ssq_out,
                                 int32_t np, int32_t d, float eps) {
  g_norm.ssq_in = ssq_in;
  g_norm.h_out = h_out;
  g_norm.gamma_next = gamma_next;
  g_norm.ssq_out = ssq_out;
  g_norm.np = np;
  g_norm.d = d;
  g_norm.eps = eps;
  return CB_OK;
}

extern "C" int cbt_gemm_set_wcopies(int32_t n, int64_t stride_bytes) {
  g_wcopies = n < 1 ? 1 : n;
  g_wcopy_stride = stride_bytes;
  return CB_OK;
}

// ---------------------------------------------------------------------------
// tcgen05.mma issue-rate probe (experiments only): one CTA per SM issues `n`
// kind::f16 MMAs of 128 x N x 16 from shared memory (SW128 K-major operands,
// garbage data) into TMEM, then waits for completion; cycles per MMA.
namespace {
template <int N>
__global__ void __launch_bounds__(128, 1) mma_probe_kernel(int n, int kstep, unsigned long long* cyc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    cb::mbar_init(&bar, 1);
    cb::fence_barrier_init();
  }
  if (warp == 0) cb::tmem_alloc<256>(&tslot);
  cb::tc_fence_before();
  __syncthreads();
  cb::tc_fence_after();
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = cb::make_idesc_bf16(128, N);
    const uint64_t da = cb::make_sw128_desc(cb::smem_u32(smem));
    const uint64_t db = cb::make_sw128_desc(cb::smem_u32(smem + 16384));
    const unsigned long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      const int k = (i % 4) * kstep;
      cb::umma_bf16(tm, da + uint64_t(2 * k), db + uint64_t(2 * k), idesc, i > 0 ? 1u : 0u);
    }
    cb::umma_commit(&bar);
    cb::mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  cb::tc_fence_before();
  __syncthreads();
  cb::tc_fence_after();
  if (warp == 0) cb::tmem_dealloc<256>(tm);
}
}  // namespace

extern "C" int cbt_mma_probe(int32_t N, int32_t n, int32_t grid, int32_t kstep, double* cyc_per_mma) {
  unsigned long long* d = nullptr;
  cudaMalloc(&d, size_t(grid) * 8);
  const size_t smem = 16384 + 32768 + 1024;
  auto run = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    kern<<<grid, 128, smem>>>(n, kstep, d);
    kern<<<grid, 128, smem>>>(n, kstep, d);
  };
  switch (N) {
    case 16: run(mma_probe_kernel<16>); break;
    case 64: run(mma_probe_kernel<64>); break;
    case 128: run(mma_probe_kernel<128>); break;
    case 256: run(mma_probe_kernel<256>); break;
    default: cudaFree(d); return CB_EINVAL;
  }
  std::vector<unsigned long long> h(grid);
  if (cudaMemcpy(h.data(), d, size_t(grid) * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return CB_ECUDA;
  cudaFree(d);
  double s = 0;
  for (auto v : h) s += double(v);
  *cyc_per_mma = s / grid / n;
  return CB_OK;
}

// causal prefill attention: rows [0, T) of qkv hold consecutive prompts; blocks_dev
// = int4 (row, rows, slot, first position) per 256-row block; K/V already in kv
// ([n_slots][max_ctx][2][Hkv hd]).
extern "C" int cbt_prefill_attention(const uint16_t* qkv, const uint16_t* kv, uint16_t* out, const int32_t* blocks_dev,
                                     int32_t nblocks, int32_t T, int32_t H, int32_t Hkv, int32_t hd,
                                     int32_t max_ctx, int32_t n_slots) {
  cb::AttnArgs a{};
  a.qkv = qkv;
  a.kv = kv;
  a.out = out;
  a.T = T;
  a.H = H;
  a.Hkv = Hkv;
  a.hd = hd;
  a.max_ctx = max_ctx;
  a.qkv_rows = T;
  a.kv_slots = n_slots;
  a.scale = 1.0f / std::sqrt(float(hd));
  return finish(cb::prefill_attention_launch(a, reinterpret_cast<const int4*>(blocks_dev), nblocks, 0));
}
