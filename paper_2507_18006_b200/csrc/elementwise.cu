// Memory-bound kernels of the decoder-layer executor: embedding gather,
// RMSNorm, RoPE + KV append, argmax, deterministic init, segment copy.
//
// Each is HBM/L2-bound (SURVEY.md §8(d) "RMSNorm/RoPE, KV append: HBM"):
// 128-bit vector accesses, one warp per row so every row is read once.
#include "common.cuh"
#include "kernels.h"

namespace cb {

// ---------------------------------------------------------------- embedding
__global__ void embed_kernel(const uint16_t* __restrict__ table, const int32_t* __restrict__ tokens,
                             float* __restrict__ x, int T, int d, int row_off) {
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
  embed_kernel<<<(T + 3) / 4, 128, 0, st>>>(table, tokens, x, T, d, row_off);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- RMSNorm
// reference composition: LLaMA decoder (norm vectors counted in
// ModuleCatalog.from_model, domain.py:259).  fp32 residual in, bf16 out.
__global__ void rmsnorm_kernel(const float* __restrict__ x, const uint16_t* __restrict__ gamma,
                               uint16_t* __restrict__ y, int T, int d, float eps, int row_off) {
  const int warps = blockDim.x >> 5;
  const int t = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)(row_off + t) * d);
  float ss = 0.f;
  for (int i = lane; i < d / 4; i += 32) {
    float4 v = xr[i];
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / float(d) + eps);
  const uint2* g = reinterpret_cast<const uint2*>(gamma);
  uint2* yr = reinterpret_cast<uint2*>(y + (size_t)(row_off + t) * d);
  for (int i = lane; i < d / 4; i += 32) {
    float4 v = xr[i];
    uint2 gg = __ldg(g + i);
    uint2 o;
    o.x = pack_bf16x2(v.x * r * bf16_lo(gg.x), v.y * r * bf16_hi(gg.x));
    o.y = pack_bf16x2(v.z * r * bf16_lo(gg.y), v.w * r * bf16_hi(gg.y));
    yr[i] = o;
  }
}

cudaError_t rmsnorm_launch(const float* x, const uint16_t* gamma, uint16_t* y, int T, int d, float eps,
                           int row_off, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  rmsnorm_kernel<<<(T + 3) / 4, 128, 0, st>>>(x, gamma, y, T, d, eps, row_off);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- RoPE + KV append
// One CTA per row.  Thread j handles rotation pair j of a head: (i, i + hd/2)
// (rotate-half convention).  q is rotated in place; rotated k and raw v are
// appended at cache[slot][pos].
__global__ void rope_kv_kernel(uint16_t* __restrict__ qkv, uint16_t* __restrict__ kv,
                               const float2* __restrict__ rope, const int32_t* __restrict__ row_slot,
                               const int32_t* __restrict__ row_pos, int row_off, int H, int Hkv, int hd,
                               int max_ctx) {
  const int row = row_off + blockIdx.x;
  const int slot = row_slot[row];
  const int pos = row_pos[row];
  const int half = hd / 2;
  const size_t qkv_ld = size_t(H + 2 * Hkv) * hd;
  uint16_t* q = qkv + row * qkv_ld;
  uint16_t* k = q + size_t(H) * hd;
  const uint16_t* v = k + size_t(Hkv) * hd;
  const size_t kvd = size_t(Hkv) * hd;
  uint16_t* kc = kv + ((size_t)slot * max_ctx + pos) * 2 * kvd;
  uint16_t* vc = kc + kvd;
  const float2* rp = rope + (size_t)pos * half;
  const int npairs = (H + Hkv) * half;
  for (int j = threadIdx.x; j < npairs; j += blockDim.x) {
    const int head = j / half, i = j % half;
    const float2 cs = rp[i];
    uint16_t* base = (head < H) ? (q + (size_t)head * hd) : (k + (size_t)(head - H) * hd);
    const float x1 = bf16_to_f(base[i]), x2 = bf16_to_f(base[i + half]);
    const uint16_t o1 = f_to_bf16(x1 * cs.x - x2 * cs.y);
    const uint16_t o2 = f_to_bf16(x2 * cs.x + x1 * cs.y);
    if (head < H) {
      base[i] = o1;
      base[i + half] = o2;
    } else {
      const size_t off = (size_t)(head - H) * hd;
      kc[off + i] = o1;
      kc[off + i + half] = o2;
    }
  }
  for (int j = threadIdx.x; j < int(kvd / 8); j += blockDim.x)
    reinterpret_cast<uint4*>(vc)[j] = reinterpret_cast<const uint4*>(v)[j];
}

cudaError_t rope_kv_launch(uint16_t* qkv, uint16_t* kv, const float2* rope, const int32_t* row_slot,
                           const int32_t* row_pos, int T, int row_off, int H, int Hkv, int hd, int max_ctx,
                           cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  rope_kv_kernel<<<T, 256, 0, st>>>(qkv, kv, rope, row_slot, row_pos, row_off, H, Hkv, hd, max_ctx);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- row gather
__global__ void gather_rows_kernel(const uint16_t* __restrict__ src, const int32_t* __restrict__ idx,
                                   uint16_t* __restrict__ dst, int d) {
  const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)idx[blockIdx.x] * d);
  uint4* o = reinterpret_cast<uint4*>(dst + (size_t)blockIdx.x * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) o[i] = s[i];
}

cudaError_t gather_rows_launch(const uint16_t* src, const int32_t* idx, uint16_t* dst, int n, int d,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  gather_rows_kernel<<<n, 128, 0, st>>>(src, idx, dst, d);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- argmax
__global__ void argmax_kernel(const float* __restrict__ logits, int32_t* __restrict__ out, int V) {
  const int t = blockIdx.x;
  const float* row = logits + (size_t)t * V;
  float best = -INFINITY;
  int idx = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    float v = row[i];
    if (v > best) { best = v; idx = i; }  // strided ascending: first max per thread
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
  argmax_kernel<<<T, 512, 0, st>>>(logits, out, V);
  return cudaGetLastError();
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

// ---------------------------------------------------------------- segment copy
// One CTA per segment, 128-bit loads with 4-way unroll; src may live on a peer.
__global__ void copy_segments_kernel(const CopySeg* __restrict__ segs) {
  const CopySeg s = segs[blockIdx.y];
  const size_t n16 = s.bytes / 16;
  const uint4* src = reinterpret_cast<const uint4*>(s.src);
  uint4* dst = reinterpret_cast<uint4*>(s.dst);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

cudaError_t copy_segments_launch(const CopySeg* segs_dev, int nseg, cudaStream_t st) {
  if (nseg <= 0) return cudaSuccess;
  dim3 grid(8, nseg);
  copy_segments_kernel<<<grid, 256, 0, st>>>(segs_dev);
  return cudaGetLastError();
}

}  // namespace cb
