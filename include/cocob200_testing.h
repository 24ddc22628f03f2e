/*
 * cocob200 kernel-level test entry points.  NOT part of the drop-in boundary
 * (include/cocob200.h is); these let tests/ drive one kernel at a time on
 * caller-owned device buffers (torch tensors) and compare it with the CPU
 * oracle.  All calls run on the current CUDA device's default stream and
 * synchronize before returning.
 */
#ifndef COCOB200_TESTING_H
#define COCOB200_TESTING_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* out (op)= X[row_off:row_off+T] @ W^T; epi: 0 bf16, 1 fp32, 2 fp32 residual +=, 3 SwiGLU (interleaved rows) */
int cbt_gemm(const void* w, const void* x, int64_t x_rows, int32_t N, int32_t K, int32_t T, int32_t row_off,
             int32_t epi, void* out, int64_t ldo);
int cbt_rmsnorm(const float* x, const uint16_t* gamma, uint16_t* y, int32_t T, int32_t d, float eps);
int cbt_rope_kv(uint16_t* qkv, uint16_t* kv, const int32_t* row_slot, const int32_t* row_pos, int32_t T, int32_t H,
                int32_t Hkv, int32_t hd, int32_t max_ctx, float theta);
int cbt_attention(const uint16_t* qkv, const uint16_t* kv, uint16_t* out, const int32_t* row_slot,
                  const int32_t* row_pos, int32_t T, int32_t H, int32_t Hkv, int32_t hd, int32_t max_ctx);
/* decode path: RoPE of q/k + KV append fused into the attention kernel */
int cbt_attention_fused(const uint16_t* qkv, uint16_t* kv, uint16_t* out, const int32_t* row_slot,
                        const int32_t* row_pos, int32_t T, int32_t H, int32_t Hkv, int32_t hd, int32_t max_ctx,
                        float theta);
/* slots of the KV buffer cbt_attention_fused may view through TMA: 0 (default) = the 16-byte-load kernel,
   > 0 lets the launcher pick the TMA-fed decode kernel (one context split, hd 128) */
int cbt_attention_set_kv_slots(int32_t n);
/* ms per launch of `iters` back-to-back attention launches (max_len given, no host sync inside) */
int cbt_attention_bench(const uint16_t* qkv, const uint16_t* kv, uint16_t* out, const int32_t* row_slot,
                        const int32_t* row_pos, int32_t T, int32_t H, int32_t Hkv, int32_t hd, int32_t max_ctx,
                        int32_t max_len, int32_t iters, float* ms_per_launch);
int cbt_argmax(const float* logits, int32_t* out, int32_t T, int32_t V);
/* causal tcgen05 prefill attention: blocks_dev = int4 (row, rows <= 256, slot, first position) per block;
   the KV cache holds n_slots x max_ctx positions */
int cbt_prefill_attention(const uint16_t* qkv, const uint16_t* kv, uint16_t* out, const int32_t* blocks_dev,
                          int32_t nblocks, int32_t T, int32_t H, int32_t Hkv, int32_t hd, int32_t max_ctx,
                          int32_t n_slots);
/* wall-clock of `iters` back-to-back GEMM launches measured with CUDA events, ms per launch */
// gemm_plan's choice for an (N, K, T) launch (host only): out[11] = tn, pair, box_rows, csplit,
// max_parts, whole, kd, corun, cstream, nclusters, nw.
int cbt_gemm_plan(int32_t N, int32_t K, int32_t T, int32_t num_sms, int32_t kind_T, int32_t* out);
int cbt_gemm_bench(const void* w, const void* x, int64_t x_rows, int32_t N, int32_t K, int32_t T, int32_t epi,
                   void* out, int64_t ldo, int32_t iters, int32_t max_parts, float* ms_per_launch);
/* cbt_gemm_bench rotates over n weight copies stride_bytes apart (weights larger than L2, as in a step) */
int cbt_gemm_set_wcopies(int32_t n, int64_t stride_bytes);
/* host milliseconds the runtime spent enqueuing its last forward pass (launch-overhead experiments) */
double cbt_last_enqueue_ms(void);
/* Fused-RMSNorm fields (GemmArgs ssq_in / h_out / gamma_next / ssq_out) for
 * every following cbt_gemm / cbt_gemm_bench launch; all null = plain GEMM. */
int cbt_gemm_set_norm(const float* ssq_in, uint16_t* h_out, const uint16_t* gamma_next, float* ssq_out, int32_t np,
                      int32_t d, float eps);
/* tcgen05.mma issue-rate probe: cycles per 128 x N x 16 bf16 MMA (smem operands), grid CTAs */
int cbt_mma_probe(int32_t N, int32_t n, int32_t grid, int32_t kstep, double* cyc_per_mma);
/* per-CTA timeline (globaltimer ns, 64 slots per CTA) of the last traced cbt_gemm_bench launch */
int cbt_gemm_trace(unsigned long long* out, int32_t n);
/* TMA read-bandwidth probe: `grid` CTAs, `nw` issuing warps each, stream `iters` boxes of
 * box_rows x (kd x 64) bf16 (kd > 1: 3-D boxes) through a `stages`-deep ring per warp; device ms */
int cbt_tma_probe(const void* buf, int64_t rows, int32_t box_rows, int32_t stages, int32_t grid, int32_t iters,
                  int32_t kd, int32_t nw, int32_t mma_n, float* ms_out);

#ifdef __cplusplus
}
#endif
#endif
