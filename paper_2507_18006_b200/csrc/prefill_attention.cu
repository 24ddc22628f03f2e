// Causal prefill attention on the tensor cores (flash-attention forward).
//
// Prefill rows of one sequence are contiguous in qkv and their K/V were just
// appended to the slot's cache (rope_kv_kernel), so a block of 64 consecutive
// query rows of one sequence attends to cache positions [0, p0 + 63] of its
// slot.  CTA = (q block, q head), 4 warps x 16 query rows.  Per 64-position
// K/V block: S = Q K^T and O += P V with mma.sync.m16n8k16 (bf16 in, fp32
// accumulate), online softmax in registers (exp2), causal mask on the diagonal
// block only.  K/V blocks are staged in shared memory with cp.async (double
// buffered, 16-byte chunks XOR-swizzled against bank conflicts) and read back
// with ldmatrix (.trans for V).  The decode path keeps attention.cu (one query
// row per sequence: HBM-bound, no tensor-core work to do).
//
// Replaces the row-parallel prefill use of attn_kernel: at 2048-token prompts
// that path ran at ~10 TFLOP/s and was 81% of the prefill time.
#include "common.cuh"
#include "kernels.h"

namespace cb {

static constexpr int kPfRows = 64;  // query rows per CTA (4 warps x 16)
static constexpr int kPfKeys = 64;  // key positions per block

CB_DEVICE void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
CB_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
CB_DEVICE void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

CB_DEVICE void ldmatrix_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
CB_DEVICE void ldmatrix_x4_trans(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
// D (16x8 fp32) += A (16x16 bf16, row) * B (16x8 bf16, col)
CB_DEVICE void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// row-major [rows][HD] bf16 tile in smem, 16-byte chunk c of row r at chunk c ^ (r & 7)
template <int HD>
CB_DEVICE uint16_t* swz(uint16_t* base, int r, int c) {
  return base + r * HD + ((c ^ (r & 7)) << 3);
}

template <int HD>
__global__ void __launch_bounds__(128) prefill_attn_kernel(const AttnArgs a, const int4* blocks) {
  pdl_trigger();
  pdl_wait();
  constexpr int CH = HD / 8;  // 16-byte chunks per row
  extern __shared__ __align__(128) uint8_t pf_smem[];
  uint16_t* sQ = reinterpret_cast<uint16_t*>(pf_smem);  // [64][HD]
  uint16_t* sK = sQ + kPfRows * HD;                     // [2][64][HD]
  uint16_t* sV = sK + 2 * kPfKeys * HD;                 // [2][64][HD]
  const int4 blk = blocks[blockIdx.x];                  // (first row, rows, slot, first position)
  const int row0 = a.row_off + blk.x, nrows = blk.y, slot = blk.z, p0 = blk.w;
  const int qh = blockIdx.y;
  const int gq = a.H / a.Hkv;
  const int hk = qh / gq;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const size_t qkv_ld = size_t(a.H + 2 * a.Hkv) * HD;
  const size_t kvd = size_t(a.Hkv) * HD;
  const uint16_t* kv_slot = a.kv + (size_t)slot * a.max_ctx * 2 * kvd + (size_t)hk * HD;

  // Q tile -> smem (rows beyond the block read row0 .. clamp: masked at the store)
  for (int i = threadIdx.x; i < kPfRows * CH; i += 128) {
    const int r = i / CH, c = i % CH;
    const int rr = min(r, nrows - 1);
    cp_async16(swz<HD>(sQ, r, c), a.qkv + (size_t)(row0 + rr) * qkv_ld + (size_t)qh * HD + c * 8);
  }
  const int last_pos = p0 + nrows - 1;
  const int nkb = last_pos / kPfKeys + 1;
  auto load_kv = [&](int kb, int buf) {
    uint16_t* dk = sK + buf * kPfKeys * HD;
    uint16_t* dv = sV + buf * kPfKeys * HD;
    for (int i = threadIdx.x; i < kPfKeys * CH; i += 128) {
      const int r = i / CH, c = i % CH;
      const int pos = min(kb * kPfKeys + r, last_pos);  // beyond the causal range: masked
      const uint16_t* src = kv_slot + (size_t)pos * 2 * kvd + c * 8;
      cp_async16(swz<HD>(dk, r, c), src);
      cp_async16(swz<HD>(dv, r, c), src + kvd);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  const float sl2 = a.scale * 1.4426950408889634f;
  float o[HD / 8][4];
#pragma unroll
  for (int j = 0; j < HD / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // rows g and g + 8 of this warp
  const int qr0 = warp * 16 + g;                            // local query rows of this thread
  const int qp0 = p0 + qr0, qp1 = qp0 + 8;                  // their positions
  uint32_t qa[HD / 16][4];
  bool q_loaded = false;

  for (int kb = 0; kb < nkb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nkb) {
      load_kv(kb + 1, buf ^ 1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (!q_loaded) {  // A fragments of this warp's 16 query rows, all k-chunks
#pragma unroll
      for (int kc = 0; kc < HD / 16; ++kc) {
        const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = kc * 2 + (lane >> 4);
        ldmatrix_x4(qa[kc], swz<HD>(sQ, r, c));
      }
      q_loaded = true;
    }
    const uint16_t* k_s = sK + buf * kPfKeys * HD;
    const uint16_t* v_s = sV + buf * kPfKeys * HD;
    // S = Q K^T for 64 key positions: 8 n-tiles of 8
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int kc = 0; kc < HD / 16; ++kc) {
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {  // n-tiles 2jp, 2jp+1 (positions 16jp .. 16jp+15)
        uint32_t b[4];
        const int r = jp * 16 + (lane & 7) + (lane >> 4) * 8;
        const int c = kc * 2 + ((lane >> 3) & 1);
        ldmatrix_x4(b, swz<HD>(const_cast<uint16_t*>(k_s), r, c));
        mma16816(s[2 * jp], qa[kc], b[0], b[1]);
        mma16816(s[2 * jp + 1], qa[kc], b[2], b[3]);
      }
    }
    // causal mask (diagonal block), scale, online softmax
    const int kbase = kb * kPfKeys;
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int kp = kbase + j * 8 + 2 * t;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        s[j][e] = (kp + e <= qp0) ? s[j][e] * sl2 : -INFINITY;
        s[j][2 + e] = (kp + e <= qp1) ? s[j][2 + e] * sl2 : -INFINITY;
        mx0 = fmaxf(mx0, s[j][e]);
        mx1 = fmaxf(mx1, s[j][2 + e]);
      }
    }
#pragma unroll
    for (int o2 = 1; o2 < 4; o2 <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o2));
    }
    const float c0 = (mx0 == -INFINITY) ? 1.f : exp2f(m0 - mx0);
    const float c1 = (mx1 == -INFINITY) ? 1.f : exp2f(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
    float rs0 = 0.f, rs1 = 0.f;
    uint32_t pa[4][4];  // P as A fragments: k-chunk kk covers n-tiles 2kk, 2kk+1
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float e0 = (m0 == -INFINITY) ? 0.f : exp2f(s[j][0] - m0);
      const float e1 = (m0 == -INFINITY) ? 0.f : exp2f(s[j][1] - m0);
      const float e2 = (m1 == -INFINITY) ? 0.f : exp2f(s[j][2] - m1);
      const float e3 = (m1 == -INFINITY) ? 0.f : exp2f(s[j][3] - m1);
      rs0 += e0 + e1;
      rs1 += e2 + e3;
      const int kk = j >> 1, hi = j & 1;
      pa[kk][hi * 2 + 0] = pack_bf16x2(e0, e1);
      pa[kk][hi * 2 + 1] = pack_bf16x2(e2, e3);
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) {
      o[j][0] *= c0;
      o[j][1] *= c0;
      o[j][2] *= c1;
      o[j][3] *= c1;
    }
    // O += P V: k = 64 positions (4 chunks of 16), n = HD dims
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int jd = 0; jd < HD / 16; ++jd) {  // dim tiles 2jd, 2jd+1
        uint32_t b[4];
        const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = jd * 2 + (lane >> 4);
        ldmatrix_x4_trans(b, swz<HD>(const_cast<uint16_t*>(v_s), r, c));
        mma16816(o[2 * jd], pa[kk], b[0], b[1]);
        mma16816(o[2 * jd + 1], pa[kk], b[2], b[3]);
      }
    }
    __syncthreads();  // the buffer is refilled two blocks later
  }
  // row sums across the quad, normalise, store
#pragma unroll
  for (int o2 = 1; o2 < 4; o2 <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, o2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o2);
  }
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
  uint16_t* out0 = a.out + (size_t)(row0 + qr0) * a.H * HD + (size_t)qh * HD;
  uint16_t* out1 = out0 + (size_t)8 * a.H * HD;
#pragma unroll
  for (int j = 0; j < HD / 8; ++j) {
    const int d = j * 8 + 2 * t;
    if (qr0 < nrows) *reinterpret_cast<uint32_t*>(out0 + d) = pack_bf16x2(o[j][0] * inv0, o[j][1] * inv0);
    if (qr0 + 8 < nrows) *reinterpret_cast<uint32_t*>(out1 + d) = pack_bf16x2(o[j][2] * inv1, o[j][3] * inv1);
  }
}

cudaError_t prefill_attention_launch(const AttnArgs& a, const int4* blocks, int nblocks, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  const dim3 grid(unsigned(nblocks), unsigned(a.H));
  switch (a.hd) {
    case 64: {
      const size_t smem = size_t(kPfRows + 4 * kPfKeys) * 64 * 2;
      return launch_pdl(prefill_attn_kernel<64>, grid, dim3(128), smem, st, a, blocks);
    }
    case 128: {
      const size_t smem = size_t(kPfRows + 4 * kPfKeys) * 128 * 2;
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(prefill_attn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        attr = true;
      }
      return launch_pdl(prefill_attn_kernel<128>, grid, dim3(128), smem, st, a, blocks);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace cb
