// Memory-bound kernels of the decoder-layer executor: embedding gather,
// RMSNorm, RoPE + KV append, argmax, deterministic init, segment copy.
//
// Each is HBM/L2-bound (SURVEY.md §8(d) "RMSNorm/RoPE, KV append: HBM"):
// 128-bit vector accesses, one warp per row so every row is read once.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace cb {

// ---------------------------------------------------------------- embedding
__global__ void embed_kernel(const uint16_t* __restrict__ table, const int32_t* __restrict__ tokens,
                             float* __restrict__ x, int T, int d, int row_off) {
  pdl_trigger();
  pdl_wait();
  const int warps = blockDim.x >> 5;
  const int t = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const uint4* src = reinterpret_cast<const uint4*>(table + (size_t)tokens[t] * d);
  float4* dst = reinterpret_cast<float4*>(x + (size_t)(row_off + t) * d);
  for (int i = lane; i < d / 8; i += 32) {
    uint4 v = __ldg(src + i);
    dst[2 * i] = make_float4(bf16_lo(v.x), bf16_hi(v.x), bf16_lo(v.y), bf16_hi(v.y));
    dst[2 * i + 1] = make_float4(bf16_lo(v.z), bf16_hi(v.z), bf16_lo(v.w), bf16_hi(v.w));
  }
}

cudaError_t embed_launch(const uint16_t* table, const int32_t* tokens, float* x, int T, int d, int row_off,
                         cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  return launch_pdl(embed_kernel, dim3((T + 3) / 4), dim3(128), 0, st, table, tokens, x, T, d, row_off);
}

// Embedding + the producer half of the fused RMSNorm of layer 0: besides x,
// h = bf16(x * gamma) and ssq[t][g] = sum of x^2 over features 32g..32g+31
// (the QKV GEMM scales its outputs by rsqrt(mean(x^2) + eps); kernels.h GemmArgs).
__global__ void embed_norm_kernel(const uint16_t* __restrict__ table, const int32_t* __restrict__ tokens,
                                  float* __restrict__ x, const uint16_t* __restrict__ gamma, uint16_t* __restrict__ h,
                                  float* __restrict__ ssq, int T, int d, int row_off) {
  pdl_trigger();
  pdl_wait();
  const int warps = blockDim.x >> 5;
  const int t = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const size_t row = size_t(row_off + t);
  const uint4* src = reinterpret_cast<const uint4*>(table + (size_t)tokens[t] * d);
  const uint4* g8 = reinterpret_cast<const uint4*>(gamma);
  float4* dst = reinterpret_cast<float4*>(x + row * d);
  uint4* hd = reinterpret_cast<uint4*>(h + row * d);
  const int np = d >> 5;
  for (int i = lane; i < d / 8; i += 32) {  // d % 256 == 0: every lane of the warp is active
    const uint4 v = __ldg(src + i), g = __ldg(g8 + i);
    const float e[8] = {bf16_lo(v.x), bf16_hi(v.x), bf16_lo(v.y), bf16_hi(v.y),
                        bf16_lo(v.z), bf16_hi(v.z), bf16_lo(v.w), bf16_hi(v.w)};
    dst[2 * i] = make_float4(e[0], e[1], e[2], e[3]);
    dst[2 * i + 1] = make_float4(e[4], e[5], e[6], e[7]);
    uint4 o;
    o.x = pack_bf16x2(e[0] * bf16_lo(g.x), e[1] * bf16_hi(g.x));
    o.y = pack_bf16x2(e[2] * bf16_lo(g.y), e[3] * bf16_hi(g.y));
    o.z = pack_bf16x2(e[4] * bf16_lo(g.z), e[5] * bf16_hi(g.z));
    o.w = pack_bf16x2(e[6] * bf16_lo(g.w), e[7] * bf16_hi(g.w));
    hd[i] = o;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += e[k] * e[k];
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if ((lane & 3) == 0) ssq[row * np + (i >> 2)] = s;
  }
}

cudaError_t embed_norm_launch(const uint16_t* table, const int32_t* tokens, float* x, const uint16_t* gamma,
                              uint16_t* h, float* ssq, int T, int d, int row_off, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  if (d % 256 != 0) return cudaErrorInvalidValue;
  return launch_pdl(embed_norm_kernel, dim3((T + 3) / 4), dim3(128), 0, st, table, tokens, x, gamma, h, ssq, T, d,
                    row_off);
}

// ---------------------------------------------------------------- SwiGLU combine
// act[r] = bf16(silu(gate[r]) * up[r]) in place over act, rows [row_off, row_off + T):
// the gate/up pair of a layer whose FFN_PROJ_GATE / FFN_PROJ_UP was migrated
// to another device (MigrateSubModule, ops.py:230-251) runs as two GEMMs, so the
// fused SwiGLU epilogue is replaced by this pass (same silu formula).
__global__ void swiglu_kernel(const uint16_t* __restrict__ gate, uint16_t* __restrict__ act, size_t n8) {
  pdl_trigger();
  pdl_wait();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 g = reinterpret_cast<const uint4*>(gate)[i];
    uint4 u = reinterpret_cast<uint4*>(act)[i];
    const uint32_t gw[4] = {g.x, g.y, g.z, g.w};
    uint32_t* uw = &u.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float g0 = bf16_lo(gw[j]), g1 = bf16_hi(gw[j]);
      const float u0 = bf16_lo(uw[j]), u1 = bf16_hi(uw[j]);
      uw[j] = pack_bf16x2(__fdividef(g0, 1.0f + __expf(-g0)) * u0, __fdividef(g1, 1.0f + __expf(-g1)) * u1);
    }
    reinterpret_cast<uint4*>(act)[i] = u;
  }
}

cudaError_t swiglu_launch(const uint16_t* gate, uint16_t* act, int T, int d_ff, int row_off, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  const size_t off = size_t(row_off) * d_ff;
  const size_t n8 = size_t(T) * d_ff / 8;
  const unsigned blocks = unsigned(std::min<size_t>((n8 + 255) / 256, 148 * 8));
  return launch_pdl(swiglu_kernel, dim3(blocks), dim3(256), 0, st, gate + off, act + off, n8);
}

// ---------------------------------------------------------------- RMSNorm
// reference composition: LLaMA decoder (norm vectors counted in
// ModuleCatalog.from_model, domain.py:259).  fp32 residual in, bf16 out.
// One CTA per row; the row is held in registers (<= 8 float4 per thread), so
// it is read once and every load of the row is in flight at the same time.
static constexpr int kNormVec = 8;

__global__ void rmsnorm_kernel(const float* __restrict__ x, const uint16_t* __restrict__ gamma,
                               uint16_t* __restrict__ y, int d, float eps, int row_off) {
  pdl_trigger();
  pdl_wait();
  const int row = row_off + blockIdx.x;
  const int n4 = d / 4;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)row * d);
  float4 v[kNormVec];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kNormVec; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < n4) {
      v[k] = xr[i];
      ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
    }
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float r = rsqrtf(red[0] / float(d) + eps);
  const uint2* g = reinterpret_cast<const uint2*>(gamma);
  uint2* yr = reinterpret_cast<uint2*>(y + (size_t)row * d);
#pragma unroll
  for (int k = 0; k < kNormVec; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < n4) {
      const uint2 gg = __ldg(g + i);
      uint2 o;
      o.x = pack_bf16x2(v[k].x * r * bf16_lo(gg.x), v[k].y * r * bf16_hi(gg.x));
      o.y = pack_bf16x2(v[k].z * r * bf16_lo(gg.y), v[k].w * r * bf16_hi(gg.y));
      yr[i] = o;
    }
  }
}

cudaError_t rmsnorm_launch(const float* x, const uint16_t* gamma, uint16_t* y, int T, int d, float eps,
                           int row_off, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  const int n4 = d / 4;
  int threads = ((n4 + kNormVec - 1) / kNormVec + 31) / 32 * 32;
  threads = threads < 32 ? 32 : threads;
  if (threads > 1024) return cudaErrorInvalidValue;
  return launch_pdl(rmsnorm_kernel, dim3(T), dim3(threads), 0, st, x, gamma, y, d, eps, row_off);
}

// ---------------------------------------------------------------- RoPE + KV append
// One CTA per row, 128-bit accesses.  A work item is 8 consecutive elements of
// one head's first half plus their rotation partners in the second half
// (rotate-half convention).  q is rotated in place; rotated k and raw v are
// appended at cache[slot][pos].
__global__ void rope_kv_kernel(uint16_t* __restrict__ qkv, uint16_t* __restrict__ kv,
                               const int32_t* __restrict__ kv_map, const float2* __restrict__ rope,
                               const int32_t* __restrict__ row_slot,
                               const int32_t* __restrict__ row_pos, int row_off, int H, int Hkv, int hd,
                               int max_ctx) {
  pdl_trigger();
  pdl_wait();
  const int row = row_off + blockIdx.x;
  const int slot = kv_map ? kv_map[row_slot[row]] : row_slot[row];  // index in this KV block
  const int pos = row_pos[row];
  const int half = hd / 2;
  const int cph = half / 8;  // 8-element chunks per half head
  const size_t qkv_ld = size_t(H + 2 * Hkv) * hd;
  uint16_t* q = qkv + (size_t)row * qkv_ld;
  uint16_t* k = q + size_t(H) * hd;
  const uint16_t* v = k + size_t(Hkv) * hd;
  const size_t kvd = size_t(Hkv) * hd;
  uint16_t* kc = kv + ((size_t)slot * max_ctx + pos) * 2 * kvd;
  uint16_t* vc = kc + kvd;
  const float2* rp = rope + (size_t)pos * half;
  const int nrot = (H + Hkv) * cph;
  const int nv = int(kvd / 8);
  for (int c = threadIdx.x; c < nrot + nv; c += blockDim.x) {
    if (c >= nrot) {  // v: straight copy into the cache
      reinterpret_cast<uint4*>(vc)[c - nrot] = reinterpret_cast<const uint4*>(v)[c - nrot];
      continue;
    }
    const int head = c / cph, i0 = (c % cph) * 8;
    const uint16_t* src = head < H ? q + (size_t)head * hd : k + (size_t)(head - H) * hd;
    const uint4 a = *reinterpret_cast<const uint4*>(src + i0);
    const uint4 b = *reinterpret_cast<const uint4*>(src + i0 + half);
    const float4* cs4 = reinterpret_cast<const float4*>(rp + i0);
    const float x1[8] = {bf16_lo(a.x), bf16_hi(a.x), bf16_lo(a.y), bf16_hi(a.y),
                         bf16_lo(a.z), bf16_hi(a.z), bf16_lo(a.w), bf16_hi(a.w)};
    const float x2[8] = {bf16_lo(b.x), bf16_hi(b.x), bf16_lo(b.y), bf16_hi(b.y),
                         bf16_lo(b.z), bf16_hi(b.z), bf16_lo(b.w), bf16_hi(b.w)};
    float o1[8], o2[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 cs = __ldg(cs4 + j);  // (cos, sin) of elements 2j and 2j+1
      o1[2 * j] = x1[2 * j] * cs.x - x2[2 * j] * cs.y;
      o2[2 * j] = x2[2 * j] * cs.x + x1[2 * j] * cs.y;
      o1[2 * j + 1] = x1[2 * j + 1] * cs.z - x2[2 * j + 1] * cs.w;
      o2[2 * j + 1] = x2[2 * j + 1] * cs.z + x1[2 * j + 1] * cs.w;
    }
    uint4 r1, r2;
    r1.x = pack_bf16x2(o1[0], o1[1]); r1.y = pack_bf16x2(o1[2], o1[3]);
    r1.z = pack_bf16x2(o1[4], o1[5]); r1.w = pack_bf16x2(o1[6], o1[7]);
    r2.x = pack_bf16x2(o2[0], o2[1]); r2.y = pack_bf16x2(o2[2], o2[3]);
    r2.z = pack_bf16x2(o2[4], o2[5]); r2.w = pack_bf16x2(o2[6], o2[7]);
    uint16_t* dst = head < H ? q + (size_t)head * hd : kc + (size_t)(head - H) * hd;
    *reinterpret_cast<uint4*>(dst + i0) = r1;
    *reinterpret_cast<uint4*>(dst + i0 + half) = r2;
  }
}

cudaError_t rope_kv_launch(uint16_t* qkv, uint16_t* kv, const int32_t* kv_map, const float2* rope,
                           const int32_t* row_slot, const int32_t* row_pos, int T, int row_off, int H, int Hkv, int hd,
                           int max_ctx, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  return launch_pdl(rope_kv_kernel, dim3(T), dim3(256), 0, st, qkv, kv, kv_map, rope, row_slot, row_pos, row_off, H,
                    Hkv, hd, max_ctx);
}

// ---------------------------------------------------------------- row gather
__global__ void gather_rows_kernel(const uint16_t* __restrict__ src, const int32_t* __restrict__ idx,
                                   uint16_t* __restrict__ dst, int d) {
  pdl_trigger();
  pdl_wait();
  const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)idx[blockIdx.x] * d);
  uint4* o = reinterpret_cast<uint4*>(dst + (size_t)blockIdx.x * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) o[i] = s[i];
}

cudaError_t gather_rows_launch(const uint16_t* src, const int32_t* idx, uint16_t* dst, int n, int d,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(gather_rows_kernel, dim3(n), dim3(128), 0, st, src, idx, dst, d);
}

// ---------------------------------------------------------------- argmax
__global__ void argmax_kernel(const float* __restrict__ logits, int32_t* __restrict__ out, int V) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  const float* row = logits + (size_t)t * V;
  float best = -INFINITY;
  int idx = 0x7fffffff;
  // 128-bit loads, all in flight at once; each thread scans ascending indices so
  // its first maximum is its lowest index
  if ((V & 3) == 0) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
    for (int i = threadIdx.x; i < V / 4; i += blockDim.x) {
      const float4 v = r4[i];
      if (v.x > best) { best = v.x; idx = 4 * i; }
      if (v.y > best) { best = v.y; idx = 4 * i + 1; }
      if (v.z > best) { best = v.z; idx = 4 * i + 2; }
      if (v.w > best) { best = v.w; idx = 4 * i + 3; }
    }
  } else {
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
      const float v = row[i];
      if (v > best) { best = v; idx = i; }
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > best || (ov == best && oi < idx)) { best = ov; idx = oi; }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[w] = best; si[w] = idx; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    best = lane < nw ? sv[lane] : -INFINITY;
    idx = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov > best || (ov == best && oi < idx)) { best = ov; idx = oi; }
    }
    if (lane == 0) out[t] = idx;
  }
}

cudaError_t argmax_launch(const float* logits, int32_t* out, int T, int V, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  return launch_pdl(argmax_kernel, dim3(T), dim3(1024), 0, st, logits, out, V);
}

// ---------------------------------------------------------------- init
CB_DEVICE uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void init_uniform_kernel(uint16_t* dst, size_t n, uint64_t seed, float a, float mean) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t h = splitmix64(seed ^ (i * 0xd1b54a32d192ed03ull));
    float u = float(h >> 40) * (1.0f / 16777216.0f);  // [0,1)
    dst[i] = f_to_bf16(mean + a * (2.f * u - 1.f));
  }
}

cudaError_t init_uniform_launch(uint16_t* dst, size_t n, uint64_t seed, float std, float mean, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  init_uniform_kernel<<<148 * 8, 256, 0, st>>>(dst, n, seed, std * 1.7320508f, mean);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- SM copy engine
// Transfer mode 2 of the scaling ops (cb_set_copy_mode): launched on the SOURCE
// GPU, 128-bit streaming loads and stores, 4-way unrolled; dst may be a peer
// pointer (NVLink writes need no round trip).
__global__ void __launch_bounds__(512) copy_bulk_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                          size_t n16) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    const uint4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
                d = __ldcs(src + i + 3 * stride);
    __stcs(dst + i, a);
    __stcs(dst + i + stride, b);
    __stcs(dst + i + 2 * stride, c);
    __stcs(dst + i + 3 * stride, d);
  }
  for (; i < n16; i += stride) __stcs(dst + i, __ldcs(src + i));
}

cudaError_t copy_bulk_launch(void* dst, const void* src, size_t bytes, int num_sms, cudaStream_t st) {
  if (bytes == 0) return cudaSuccess;
  const size_t n16 = bytes / 16;
  const int ctas = int(std::min<size_t>(size_t(num_sms) * 2, (n16 + 511) / 512));
  copy_bulk_kernel<<<ctas, 512, 0, st>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), n16);
  return cudaGetLastError();
}

}  // namespace cb
