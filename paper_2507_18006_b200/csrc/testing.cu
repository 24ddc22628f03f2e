// Kernel-level test entry points (include/cocob200_testing.h).  Thin wrappers
// that build tensor maps / workspaces for caller-owned device buffers.
#include <cmath>
#include <map>
#include <string>
#include <vector>

#include "../../include/cocob200.h"
#include "../../include/cocob200_testing.h"
#include "kernels.h"

namespace {

struct TestWs {
  float* gemm_ws = nullptr;
  int* cnt = nullptr;
  float* attn_ws = nullptr;
  size_t attn_floats = 0;
  int sms = 148;
};

std::map<int, TestWs> g_ws;

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
  }
  *out = &w;
  return CB_OK;
}

int finish(cudaError_t e) {
  if (e != cudaSuccess) return CB_ECUDA;
  return cudaDeviceSynchronize() == cudaSuccess ? CB_OK : CB_ECUDA;
}

int gemm_setup(const void* w, const void* x, int64_t x_rows, int N, int K, const cb::GemmPlan& plan,
               CUtensorMap* mw, CUtensorMap* mx) {
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
  a.out = out;
  a.ws = ws->gemm_ws;
  a.counters = ws->cnt;
  return finish(cb::gemm_launch(mw, mx, a, plan, ws->sms, 0));
}

int cbt_gemm_bench(const void* w, const void* x, int64_t x_rows, int32_t N, int32_t K, int32_t T, int32_t epi,
                   void* out, int64_t ldo, int32_t iters, int32_t max_parts, float* ms_per_launch) {
  TestWs* ws;
  int r = ws_for_current(&ws);
  if (r) return r;
  cb::GemmPlan plan = cb::gemm_plan(N, K, T, ws->sms);
  if (max_parts < 0 && plan.tn != cb::kPairTileMarker) {  // experiments: force cluster split -max_parts
    plan.csplit = -max_parts;
    plan.mcast = 1;
    plan.box_rows = plan.tn;
  } else if (max_parts == 100 && plan.tn != cb::kPairTileMarker) {  // experiments: no multicast
    plan.mcast = 1;
    plan.box_rows = plan.tn;
  }
  CUtensorMap mw, mx;
  if ((r = gemm_setup(w, x, x_rows, N, K, plan, &mw, &mx))) return r;
  cb::GemmArgs a{};
  a.N = N;
  a.K = K;
  a.T = T;
  a.epi = epi;
  a.ldo = ldo;
  a.out = out;
  a.ws = ws->gemm_ws;
  a.counters = ws->cnt;
  a.max_parts = (max_parts < 0 || max_parts == 100) ? 1 : max_parts;
  for (int i = 0; i < 3; ++i) cb::gemm_launch(mw, mx, a, plan, ws->sms, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, 0);
  for (int i = 0; i < iters; ++i) cb::gemm_launch(mw, mx, a, plan, ws->sms, 0);
  cudaEventRecord(e1, 0);
  if (cudaEventSynchronize(e1) != cudaSuccess) return CB_ECUDA;
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  *ms_per_launch = ms / iters;
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
  a.ws_floats = ws->attn_floats;
  a.T = T;
  a.H = H;
  a.Hkv = Hkv;
  a.hd = hd;
  a.max_ctx = max_ctx;
  a.max_len = max_len;
  a.scale = 1.0f / std::sqrt(float(hd));
  a.rope = dtab;
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
  int r = finish(cb::rope_kv_launch(qkv, kv, dtab, row_slot, row_pos, T, 0, H, Hkv, hd, max_ctx, 0));
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
