// Internal kernel launchers of libcocob200 (not part of the public C-ABI; see
// include/cocob200.h for that).  All launchers are asynchronous on `st`.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace cb {

// ---------------------------------------------------------------- GEMM
enum EpiKind : int {
  EPI_BF16 = 0,    // out bf16 [row][n]           = acc
  EPI_F32 = 1,     // out fp32 [row][n]           = acc          (lm_head logits)
  EPI_RESID = 2,   // out fp32 [row][n]          += acc          (residual stream)
  EPI_SWIGLU = 3,  // out bf16 [row][n/2] = silu(acc[2j]) * acc[2j+1]   (gate/up interleaved)
};

struct GemmArgs {
  int N;        // weight rows (output features; 2*d_ff for the fused gate/up)
  int K;        // reduction length
  int T;        // activation rows in this launch
  int row_off;  // first activation/output row
  int epi;      // EpiKind
  long long ldo;  // output row stride (elements)
  void* out;
  float* ws;      // stream-K partials, gemm_ws_floats(num_sms) floats
  int* counters;  // per-tile arrival counters, zero-initialised, >= n_tiles ints
  int max_parts;      // stream-K: max CTAs (pairs) per tile (0 = no cap)
  int cluster_split;  // set from the plan: >1 = tile split over a cluster, DSMEM reduce
  int w_tiled;        // 1 = weight stored tile-major [N/128][K/64][128][64] (each TMA box contiguous)
  unsigned long long* trace;  // experiments only: per-CTA event timestamps (globaltimer ns) when non-null
  int vec;            // set by the launcher: 16-byte vector epilogue stores are legal for out/N/ldo
  int tma;            // set by the launcher: an output tensor map was passed (TMA-store epilogue)
  int whole_tiles;    // set from the plan: CTA (pair) ranges rounded to whole tiles
  int stages;         // set by the launcher: pipeline ring depth (1-CTA kernel: the weight ring)
  int xstages;        // set by the launcher: activation ring depth (1-CTA kernel; 0 = stages)
  int dbg;            // experiments only: bit0 = skip the MMAs, bit1 = skip the epilogue
  // Fused RMSNorm (decode passes, T <= 256; SURVEY.md §8(a) rmsnorm):
  //  consumer (ssq_in != null): X rows are h' = bf16(x * gamma); output row t is
  //    scaled by rsqrt(sum_k ssq_in[t][k] / norm_d + norm_eps) before the epilogue op;
  //  producer (EPI_RESID, h_out != null): besides x += proj it writes
  //    h_out = bf16(x * gamma_next) and ssq_out[t][n / 32] = sum over the 32
  //    features n..n+31 of x^2 (fixed order: deterministic).
  const float* ssq_in;
  uint16_t* h_out;
  const uint16_t* gamma_next;
  float* ssq_out;
  int ssq_np;  // partials per row (= d / 32)
  long long out_rows;  // rows of the output tensor (TMA-store maps); 0 = unknown (register stores)
  const void* w_base;  // weight base / row stride (elements): token-major plans build their own weight map
  long long w_stride;
  int nw;              // set by the launcher: weight rows per pair tile of the token-major kernel
  int raster;          // set by the launcher: token tiles per raster group of the token-major kernel (0 = contiguous ranges)
  int ksplit;          // set by the launcher: token-major kernel split over K across a 4-CTA cluster (2 pairs)
  int norm_d;
  float norm_eps;
  // filled by the launcher
  int n_mtiles, n_ttiles, kblocks, units;
};

int make_kmajor_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t k, uint64_t row_stride_elems,
                    uint32_t box_rows);
// 3-D view (64, rows, k / 64) of the same operand: one box = box_rows x (kd x 64) in kd SW128 sub-tiles
int make_kmajor_map3(CUtensorMap* map, const void* base, uint64_t rows, uint64_t k, uint64_t row_stride_elems,
                     uint32_t box_rows, uint32_t kd);
// TN bucket of a 1-CTA launch (16..256).
int gemm_pick_tn(int T);
// Launches with more rows than this use the CTA-pair kernel (tunable for experiments).
constexpr int kPairMinT = 128;
struct GemmPlan {
  int tn;        // token tile: 16..256 (1-CTA) or the pair tile (128 / 256 tokens per pair)
  int pair;      // 1 = CTA-pair kernel (tcgen05 cta_group::2, 256 weight rows per tile)
  int box_rows;  // activation tensor-map box height this plan needs (pair: tn / 2)
  int csplit;    // cluster split-K size (1, 2, 4, 8)
  int max_parts; // stream-K: max CTAs (pairs) sharing a tile (0 = no cap; 1 = one tile per CTA, no fixups)
  int whole;     // 1 = persistent over whole tiles (contiguous tile ranges per CTA / pair, no fixups)
  int kd;        // k-blocks (64 wide) per pipeline stage: 2 = 3-D TMA maps (make_kmajor_map3), 1-CTA kernel only
  int nw;        // > 0: token-major CTA-pair kernel, whole tiles of nw weight rows (32..256, multiple of 32)
  int ksplit;    // token-major pair kernel: 2 = each tile's K halves on two pairs of a 4-CTA cluster
};
// kind_T: rows of the whole pass (>= T); selects the kernel and split so replica
// micro-batches compute exactly what the unreplicated pass would.
GemmPlan gemm_plan(int N, int K, int T, int num_sms, int kind_T = 0);
// out_map: TMA map of the output (make_out_map) or null -> register-store epilogue
cudaError_t gemm_launch(const CUtensorMap& w, const CUtensorMap& x, const GemmArgs& a, const GemmPlan& plan,
                        int num_sms, cudaStream_t st, const CUtensorMap* out_map = nullptr);
// Output tensor map for the TMA-store epilogue: `out` is [rows][ldo] (bf16, or fp32
// for EPI_F32 / EPI_RESID) holding `cols` output columns (N, or N/2 for SwiGLU);
// box = one epilogue warp chunk (16 tokens x 32 weight rows).  Returns 0 when the
// shape allows it (16-byte aligned base and pitch, cols a multiple of the box).
int make_out_map(CUtensorMap* map, const void* out, int epi, uint64_t rows, uint64_t cols, uint64_t ldo);
size_t gemm_ws_floats(int num_sms);
constexpr int kGemmMaxTiles = 1 << 16;

// ---------------------------------------------------------------- element-wise
// x[row_off + t, :] = fp32(table[tokens[t], :])
cudaError_t embed_launch(const uint16_t* table, const int32_t* tokens, float* x, int T, int d, int row_off,
                         cudaStream_t st);
// embed_launch + fused-RMSNorm producer outputs: h = bf16(x * gamma), ssq[t][g] =
// sum of x^2 over features 32g..32g+31 (d % 256 == 0)
cudaError_t embed_norm_launch(const uint16_t* table, const int32_t* tokens, float* x, const uint16_t* gamma,
                              uint16_t* h, float* ssq, int T, int d, int row_off, cudaStream_t st);
// y = bf16(x * rsqrt(mean(x^2) + eps) * gamma) for rows [row_off, row_off + T)
cudaError_t rmsnorm_launch(const float* x, const uint16_t* gamma, uint16_t* y, int T, int d, float eps,
                           int row_off, cudaStream_t st);
// In place RoPE of q,k inside qkv rows and append of (k, v) to the slot KV cache.
// qkv row = [q: H*hd | k: Hkv*hd | v: Hkv*hd]; cache = [index][max_ctx][2][Hkv*hd]
// with index = kv_map[slot] (a share-sized replica block's slot table) or slot (kv_map null).
cudaError_t rope_kv_launch(uint16_t* qkv, uint16_t* kv, const int32_t* kv_map, const float2* rope,
                           const int32_t* row_slot, const int32_t* row_pos, int T, int row_off, int H, int Hkv, int hd,
                           int max_ctx, cudaStream_t st);
// Row-parallel causal attention over the slot KV cache: row r attends to
// positions [0, row_pos[r]] of its slot.  Decode (one row per sequence) and
// prefill (one row per prompt token) share this kernel.
struct AttnArgs {
  const uint16_t* qkv;
  const uint16_t* kv;
  uint16_t* out;  // [row][H*hd]
  const int32_t* row_slot;
  const int32_t* kv_map;  // slot -> index in this KV block (null: the slot itself)
  const int32_t* row_pos;
  float* ws;       // split-context partials
  size_t ws_floats;
  int* counters;   // split-context arrivals per (row, kv head), zero between launches
  int kind_T;      // rows of the whole pass (the split decision; 0 = T): replicas split like the unreplicated pass
  const float2* rope;  // non-null: fused decode path (RoPE of q/k + KV append inside the kernel)
  int T, row_off, H, Hkv, hd, max_ctx, max_len;
  float scale;  // 1/sqrt(hd)
  int prefetch_pos;  // set by the launcher: cached positions per CTA prefetched to L2 before the PDL wait
  int qkv_rows;      // prefill: rows of the qkv buffer (TMA bounds)
  int kv_slots;      // slots of the KV block (TMA bounds: kv_slots * max_ctx positions); decode: 0 = host-mapped block
};
cudaError_t attention_launch(const AttnArgs& a, int num_sms, cudaStream_t st);

// act = bf16(silu(gate) * act) over rows [row_off, row_off + T) of [rows][d_ff] buffers (d_ff % 8 == 0)
cudaError_t swiglu_launch(const uint16_t* gate, uint16_t* act, int T, int d_ff, int row_off, cudaStream_t st);
// Causal prefill attention on the tcgen05 tensor cores: blocks[i] = (first row
// relative to a.row_off, rows (<= 256), slot, first position) of one sequence; q
// already rotated and the block's K/V already in the cache (rope_kv_launch).
// Grid (blocks, H); a.qkv_rows / a.kv_slots bound the TMA views.
cudaError_t prefill_attention_launch(const AttnArgs& a, const int4* blocks, int nblocks, cudaStream_t st);
// dst[i, :] = src[idx[i], :] (bf16 rows; prefill keeps only each sequence's last row)
cudaError_t gather_rows_launch(const uint16_t* src, const int32_t* idx, uint16_t* dst, int n, int d,
                               cudaStream_t st);
// logits [T][V] fp32 -> argmax index per row (ties -> lowest index)
cudaError_t argmax_launch(const float* logits, int32_t* out, int T, int V, cudaStream_t st);
// deterministic counter-based init: uniform with the given std, plus `mean`
cudaError_t init_uniform_launch(uint16_t* dst, size_t n, uint64_t seed, float std, float mean, cudaStream_t st);
// Contiguous copy by the SMs of the launching GPU (dst and/or src may be peer
// memory): 16-byte vectors, 4 in flight per thread.  bytes % 16 == 0, 16-byte aligned.
cudaError_t copy_bulk_launch(void* dst, const void* src, size_t bytes, int num_sms, cudaStream_t st);

}  // namespace cb
