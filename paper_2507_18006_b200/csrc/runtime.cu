// libcocob200 runtime: logical devices, the module registry of device buffers,
// the decoder-layer executor (cb_step), the replica router / batch splitter and
// the replication / migration copy engine.  Implements include/cocob200.h.
//
// Reference seams replaced (all Python in the reference, /root/reference/pkg):
//   cb_split_batch        <- ops.split_batch                  ops.py:151-158
//   cb_step               <- sim.step_batch / step_time_s     sim.py:239-300
//                            (+ _kernels.work_units/comm_units _kernels.py:17-51)
//   cb_replicate_layer    <- ops.apply(ReplicateLayer)        ops.py:199-211
//   cb_migrate_layer      <- ops.apply(MigrateLayer)          ops.py:213-228
//   cb_migrate_submodule  <- ops.apply(MigrateSubModule)      ops.py:230-251
//   cb_evict_replica      <- ops.apply(EvictReplica)          ops.py:253-258
//   cb_get_placement      <- sim.build_step_arrays            sim.py:216-236
//
// Executor data layout (per logical device that runs any layer rows):
//   x    fp32 [max_tokens][d]       residual stream (rows indexed globally)
//   h    bf16 [max_tokens][d]       RMSNorm output (GEMM B operand)
//   qkv  bf16 [max_tokens][(H+2Hkv)hd]
//   att  bf16 [max_tokens][H hd]
//   act  bf16 [max_tokens][d_ff]    SwiGLU output
// Layer copy = ONE contiguous block [wqkv | wo | w_gate/up interleaved | w_down
// | attn_norm | ffn_norm], so replication/migration of a layer is one
// peer-to-peer copy of exactly ModuleCatalog.decoder_layer_mb bytes (MHA).
// KV per (layer, device): [slot][max_ctx][2][Hkv hd] bf16.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/cocob200.h"
#include "kernels.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CB_CUDA(expr)                                                                    \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail(CB_ECUDA, std::string(#expr) + " failed: " + cudaGetErrorString(_e)); \
  } while (0)

#define CB_TRY(expr)          \
  do {                        \
    int _r = (expr);          \
    if (_r != CB_OK) return _r; \
  } while (0)

// Device memory categories (cb_mem_usage): what the executor really holds per
// logical device, for the controller's pressure view (autoscaler PressureView).
enum MemCat { MEM_WS = 0, MEM_WEIGHTS = 1, MEM_KV = 2, MEM_CATS = 3 };

struct DeviceCtx {
  int id = 0;
  int ordinal = 0;
  bool local = true;  // SPMD runtime: computed by this process (else: bookkeeping only, no streams / memory)
  int rank = 0;       // SPMD runtime: the process that owns this device
  int num_sms = 148;
  cudaStream_t compute = nullptr;
  cudaStream_t copy = nullptr;   // scaling-op transfers (main lane)
  cudaStream_t copy2 = nullptr;  // second copy lane: chunks of large transfers alternate between the two
  cudaStream_t alloc = nullptr;  // always idle: synchronous pool allocations never wait on a running copy
  std::vector<cudaEvent_t> ev_pool;  // dependency events (no timing)
  size_t ev_next = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;  // timing events
  std::map<void*, std::pair<size_t, int>> allocs;  // live allocations: bytes, MemCat
  size_t mem[MEM_CATS] = {0, 0, 0};
  bool ipc_weights = false;  // SPMD: weight blocks from cudaMalloc, exportable with CUDA IPC
  std::map<void*, bool> ipc_allocs;
  size_t reserved = 0;  // bytes held by pending (uncommitted) scaling ops
};

// activation tensor maps per box height (GEMM plans need 8..256-row boxes)
constexpr int kTnCount = 6;
constexpr int kTns[kTnCount] = {8, 16, 32, 64, 128, 256};
// A GEMM operand's TMA views: 2-D (64-wide k-blocks) and, when K allows, the
// 3-D view the 2-k-block-per-stage 1-CTA kernel loads with one box.
struct OpMap {
  CUtensorMap m2;
  CUtensorMap m3;
  bool has3 = false;
  const void* base = nullptr;  // operand base / row stride (elements): the GEMM launcher builds
  uint64_t stride = 0;         // the token-major kernel's weight boxes from these
};

int box_index(int rows) {
  for (int i = 0; i < kTnCount; ++i)
    if (kTns[i] == rows) return i;
  return kTnCount - 1;
}

}  // namespace

struct cb_runtime {
  std::vector<DeviceCtx> devs;
  bool spmd = false;               // one process per GPU (cb_runtime_create_spmd)
  int my_rank = 0;
  std::vector<int> ranks;          // the distinct ranks owning devices, ascending
  cb_xfer_fn xfer = nullptr;       // cross-process transport (host callback)
  void* xfer_ctx = nullptr;
  int grp_ch = -1;                 // an exchange group is open on this channel (XGroup) ...
  bool grp_live = false;           // ... and the transport has been told (first exchange seen)
  int copy_mode = 1;                  // transfer engine (cb_set_copy_mode)
  size_t copy_chunk = size_t(64) << 20;
};

namespace {

struct LayerCopy {
  int dev = -1;
  uint8_t* block = nullptr;
  OpMap m_qkv, m_o, m_gu, m_d;
};

// A sub-module moved off its layer by MigrateSubModule (ops.py:230-251): its
// weights in canonical [out, in] layout on `dev`.  Index = CB_* kind id
// (Q, K, V, O, SELF_ATTENTION = [wqkv | wo], GATE, UP, DOWN).
struct ModCopy {
  int dev = -1;
  uint8_t* buf = nullptr;
};
constexpr int kModKinds = CB_FFN_PROJ_DOWN + 1;

// One (layer, device) KV block: [cap][max_ctx][2][Hkv hd] bf16.  The layer's
// KV device keeps every slot at its own index (cap = max_slots, no table).  A
// replica's block is sized for its split_batch share -- cap = ceil(max_slots /
// p), the reference keeps KV only on the KV device (domain.py:380-383) -- and
// maps slot -> local index through a slot table (pinned host copy + device
// copy the attention kernels read), growing by an eighth when a re-split brings
// more sequences than it holds.  An index released during a step is reusable
// from the next step on (a copy on another stream may still read it).
struct KvBlock {
  uint16_t* p = nullptr;
  int cap = 0;                 // slots
  bool host = false;           // offloaded: mapped pinned host memory (Phase 3)
  bool table = false;          // share-sized, slot table in use
  int32_t* map_h = nullptr;    // slot -> local index (-1 = none); pinned, the authoritative copy
  int32_t* map_d = nullptr;    // device copy read by the kernels
  bool dirty = false;
  std::vector<int> free_idx, pending;
};

struct LayerState {
  std::vector<LayerCopy> reps;      // original first (Replica order, domain.py:306-317)
  int kv_override = -1;             // device holding KV when overridden, else -1
  std::map<int, KvBlock> kv;        // device -> KV block
  std::vector<int> owner;           // slot -> device holding that slot's KV (-1 none)
  ModCopy mod[kModKinds];           // projection / self-attention overrides
  bool proj_ov = false;             // any entry of mod[] in use
  std::vector<std::pair<int, int>> pend;  // uncommitted scaling ops on this layer: (OpKind, dst or module kind)
};

// An issued, not yet committed scaling op (A17: the reference's _Transition,
// sim.py:396-403).  Destination memory is reserved at issue (sim.py:812-841);
// the transfer runs on the destination's copy streams while the executor keeps
// serving on the pre-op placement; the commit switches at a step boundary
// (sim.py:614-622) after a catch-up copy of the KV appended since.
enum OpKind { OPK_REPLICATE = 0, OPK_MIGRATE = 1, OPK_PROJ = 2, OPK_KV = 3, OPK_EVICT = 4 };
struct PendingOp {
  int64_t id = 0;
  int kind = 0, layer = 0, dst = -1, with_kv = 0, mod_kind = -1;
  LayerCopy copy;  // replicate / migrate: the reserved destination block
  ModCopy mod;     // projection: the reserved destination buffer
  int kv_from = -1, kv_to = -1;  // KV transfer of the slots kv_from holds (pre-copied at issue when safe)
  bool kv_new = false;           // this op allocated kv_to's block (abort releases it)
  std::vector<int> snap_len, snap_epoch;  // per slot: prefix pre-copied at issue (-1 = none)
  int copy_dev = -1;             // device whose copy stream carries the transfer
  cudaEvent_t e0 = nullptr, e1 = nullptr;  // transfer start / end (copy stream)
  cudaEvent_t c0 = nullptr, c1 = nullptr;  // commit catch-up start / end (kv_to's compute stream)
  uint64_t weight_bytes = 0, kv_bytes = 0, catchup_bytes = 0;
  size_t reserved = 0;           // bytes reserved on dst (released from the pending count at commit / abort)
  bool committed = false;
  bool started = false;          // transfer enqueued (SPMD: cb_op_start, after every rank reserved)
  int ev_dev = -1;               // local device whose copy stream carries e0 / e1 (-1: no local part)
  // the transfer cb_op_start / the issue enqueues
  int src_dev = -1;
  const void* xsrc = nullptr;
  void* xdst = nullptr;
  size_t xbytes = 0;
  bool strided_gu = false;       // gate / up rows of the interleaved block (row pitch 2x)
  bool precopy = false;          // pre-copy the KV kv_from holds into kv_to
  void* ipc_base = nullptr;      // SPMD destination: the source block mapped with CUDA IPC (closed at commit / abort)
};

struct Workspace {
  bool ready = false;
  float* x = nullptr;
  uint16_t *h = nullptr, *hl = nullptr, *qkv = nullptr, *att = nullptr, *act = nullptr;
  uint16_t* gbuf = nullptr;  // [max_tokens][d_ff] gate output when gate / up run as separate GEMMs
  float* ssq = nullptr;      // fused RMSNorm: [max_tokens][d_model / 32] partial sums of x^2 of the rows in h
  float* logits = nullptr;
  int32_t* meta = nullptr;  // [tokens | row_slot | row_pos | gather]
  int32_t* next = nullptr;
  float* gemm_ws = nullptr;
  int* gemm_cnt = nullptr;
  float* attn_ws = nullptr;
  size_t attn_ws_floats = 0;
  int* attn_cnt = nullptr;  // split-context arrivals per (row, kv head)
  float2* rope = nullptr;
  OpMap map_h[kTnCount], map_hl[kTnCount], map_att[kTnCount], map_act[kTnCount];
  // TMA-store epilogue maps by (output base, epi, cols, ldo, rows), built on first use
  std::map<std::tuple<const void*, int, uint64_t, uint64_t, uint64_t>, CUtensorMap> out_maps;
};

struct Route {
  int dev, s0, cnt;
};

struct ProfRec {
  int dev, cls;
  cudaEvent_t e0, e1;
  double bytes, flops;
};

struct Prof {
  bool on = false;
  std::vector<ProfRec> pending;
  cb_kstat stats[4] = {};
  std::map<int, std::vector<cudaEvent_t>> pool;
  std::map<int, size_t> next;
};

struct Seg {
  int dev;      // logical device computing these rows
  int rep;      // replica index
  int r0, r1;   // row range
  int s0, s1;   // sequence range
};

}  // namespace

struct cb_model {
  cb_runtime* rt = nullptr;
  cb_model_desc d{};
  int home = 0;
  int hd = 0, qkv_n = 0, q_n = 0, kv_n = 0;
  size_t off_qkv = 0, off_o = 0, off_gu = 0, off_d = 0, off_an = 0, off_fn = 0, layer_bytes = 0;
  size_t kv_block_bytes = 0;
  std::vector<LayerState> layers;
  uint16_t *embed = nullptr, *final_norm = nullptr, *lm_head = nullptr;
  OpMap m_head;
  bool head_loaded = false;
  std::map<int, Workspace> ws;
  std::vector<int> slot_len;
  int32_t* pin_meta = nullptr;
  int32_t* pin_next = nullptr;
  std::vector<std::vector<Route>> last_routing;
  int cur_phase = 0;  // CB_PHASE_* of the pass in flight
  // Fused RMSNorm per layer boundary of the pass in flight: fin[li] = layer li's
  // attention-norm input arrives as h' = bf16(x * gamma) + row sums of squares
  // (produced by the previous layer's down projection, or the embedding), so
  // its QKV GEMM applies the row scales; fin[n_layers] = the same for the head.
  std::vector<char> fin;
  int cur_T = 0;  // rows of the pass in flight: per-step meta = [tokens | slot | pos] x T, then gather x bs
  int cur_bs = 0;  // sequences of the pass in flight
  std::vector<int> seq_blk;  // prefill: first q-block of each sequence (+ total), blocks follow the gather list
  Prof prof;
  std::vector<uint32_t> slot_epoch;  // bumped on release: a pre-copied KV prefix of an older occupant is stale
  std::map<int64_t, PendingOp> ops;  // issued scaling ops (pending, then committed records)
  int64_t next_op = 1;
  // SPMD: every layer's attention norm + the final norm on this process's GPU
  // (the fused-norm producers of a layer need the NEXT layer's norm vector,
  // which may live on another rank); filled by the first step (collective)
  uint16_t* norm_tab = nullptr;
  int norm_dev = -1;
  bool norm_ready = false;
};

namespace {

DeviceCtx& devctx(cb_model* m, int dev) { return m->rt->devs[dev]; }
bool is_local(cb_model* m, int dev) { return m->rt->devs[dev].local; }

int use(const DeviceCtx& d) {
  if (!d.local) return fail(CB_ESTATE, "internal: device " + std::to_string(d.id) + " belongs to rank " +
                                           std::to_string(d.rank));
  CB_CUDA(cudaSetDevice(d.ordinal));
  return CB_OK;
}

// SPMD: hand one byte range that crosses a process boundary to the host
// transport.  send: ptr (on local device `dev`) is ready on `st`, goes to the
// rank owning `peer`; recv: ptr is filled from that rank, ordered before later
// work on `st`.  Every rank reaches the same sequence of exchanges.
int xfer(cb_model* m, int channel, bool send, int dev, int peer, void* ptr, size_t bytes, cudaStream_t st) {
  cb_runtime* rt = m->rt;
  if (bytes == 0) return CB_OK;
  if (!rt->xfer) return fail(CB_ESTATE, "SPMD runtime without a transport");
  CB_TRY(use(devctx(m, dev)));
  if (rt->grp_ch == channel && !rt->grp_live) {  // open the transport's group lazily: empty groups cost nothing
    rt->grp_live = true;
    if (rt->xfer(rt->xfer_ctx, channel, 2, -1, nullptr, 0, nullptr) != 0) return fail(CB_ECOMM, "transport group failed");
  }
  const int r = rt->xfer(rt->xfer_ctx, channel, send ? 1 : 0, devctx(m, peer).rank, ptr, bytes, st);
  if (r != 0)
    return fail(CB_ECOMM, std::string("transport ") + (send ? "send to" : "recv from") + " rank " +
                              std::to_string(devctx(m, peer).rank) + " failed (" + std::to_string(r) + ")");
  return CB_OK;
}

// Byte range src_dev:sp -> dst_dev:dp across processes: the sender's part on
// s_st (a stream of src_dev), the receiver's on d_st (of dst_dev); a rank owning
// neither does nothing.  (Same-process moves keep their peer-copy paths.)
int xmove(cb_model* m, int channel, int src_dev, const void* sp, cudaStream_t s_st, int dst_dev, void* dp,
          cudaStream_t d_st, size_t bytes) {
  if (is_local(m, src_dev)) CB_TRY(xfer(m, channel, true, src_dev, dst_dev, const_cast<void*>(sp), bytes, s_st));
  if (is_local(m, dst_dev)) CB_TRY(xfer(m, channel, false, dst_dev, src_dev, dp, bytes, d_st));
  return CB_OK;
}
bool crosses(cb_model* m, int a, int b) { return m->rt->spmd && (!is_local(m, a) || !is_local(m, b)); }

// Group the exchanges between begin and end (an NCCL group on the transport):
// the transport may batch them into one launch (send = 2 / 3 markers).
struct XGroup {
  cb_model* m;
  int ch;
  bool on;
  XGroup(cb_model* m_, int ch_) : m(m_), ch(ch_), on(m_->rt->spmd && m_->rt->xfer && m_->rt->grp_ch < 0) {
    if (on) {
      m->rt->grp_ch = ch;
      m->rt->grp_live = false;
    }
  }
  int close() {
    if (!on) return CB_OK;
    on = false;
    cb_runtime* rt = m->rt;
    const bool live = rt->grp_live;
    rt->grp_ch = -1;
    rt->grp_live = false;
    if (live && rt->xfer(rt->xfer_ctx, ch, 3, -1, nullptr, 0, nullptr) != 0)
      return fail(CB_ECOMM, "transport group failed");
    return CB_OK;
  }
  ~XGroup() { close(); }
};

// dst stream waits for everything issued so far on src's compute stream
// (devices of other processes: ordered by the transport instead)
int depend(DeviceCtx& dst, DeviceCtx& src) {
  if (&dst == &src || !dst.local || !src.local) return CB_OK;
  CB_TRY(use(src));
  cudaEvent_t ev = src.ev_pool[src.ev_next++ % src.ev_pool.size()];
  CB_CUDA(cudaEventRecord(ev, src.compute));
  CB_TRY(use(dst));
  CB_CUDA(cudaStreamWaitEvent(dst.compute, ev, 0));
  return CB_OK;
}

// ---- live profiling: bracket one launch with timing events on its stream
cudaEvent_t prof_event(cb_model* m, int dev) {
  auto& pool = m->prof.pool[dev];
  size_t& nx = m->prof.next[dev];
  if (nx == pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    pool.push_back(e);
  }
  return pool[nx++];
}

struct ProfScope {
  cb_model* m;
  int dev, cls;
  double bytes, flops;
  cudaStream_t st;
  cudaEvent_t e0 = nullptr;
  ProfScope(cb_model* m_, int dev_, int cls_, cudaStream_t st_, double bytes_, double flops_ = 0.0)
      : m(m_), dev(dev_), cls(cls_), bytes(bytes_), flops(flops_), st(st_) {
    if (m->prof.on) {
      e0 = prof_event(m, dev);
      cudaEventRecord(e0, st);
    }
  }
  ~ProfScope() {
    if (!e0) return;
    cudaEvent_t e1 = prof_event(m, dev);
    cudaEventRecord(e1, st);
    m->prof.pending.push_back({dev, cls, e0, e1, bytes, flops});
  }
};

// fold the finished step's launch timings into the per-class totals
void prof_resolve(cb_model* m) {
  for (const ProfRec& r : m->prof.pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.e0, r.e1) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    cb_kstat& k = m->prof.stats[r.cls];
    k.launches += 1;
    k.ms += ms;
    k.bytes += r.bytes;
    k.flops += r.flops;
  }
  m->prof.pending.clear();
  for (auto& kv : m->prof.next) kv.second = 0;
}

// Device memory comes from each GPU's stream-ordered pool with an unbounded
// release threshold: a migrated / evicted layer block returns to the pool and
// the next replication reuses it without cudaMalloc / cudaFree (which unmap and
// synchronise the device -- hundreds of ms per op for 0.6 GB blocks).
//  - synchronous allocations (workspaces, loads) go through the device's idle
//    `alloc` stream, so they never wait on a scaling op's running copy;
//  - a scaling op's reservation is allocated on the destination's copy stream
//    without any host synchronisation (`st`): the op's copies run on that
//    stream and the commit orders the compute streams after them.
int dev_alloc(DeviceCtx& d, void** p, size_t bytes, uint64_t* shortfall = nullptr, int cat = MEM_WS,
              cudaStream_t st = nullptr) {
  CB_TRY(use(d));
  *p = nullptr;
  // SPMD weight and KV blocks: plain cudaMalloc, so another process can map them
  // (CUDA IPC) and pull a replicated / migrated layer or its KV with its copy engines
  const bool ipc = d.ipc_weights && (cat == MEM_WEIGHTS || cat == MEM_KV);
  cudaError_t e = ipc ? cudaMalloc(p, bytes) : cudaMallocAsync(p, bytes, st ? st : d.alloc);
  if (e == cudaSuccess && !st && !ipc) e = cudaStreamSynchronize(d.alloc);  // usable from every stream from here on
  if (e != cudaSuccess) {
    cudaGetLastError();
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    if (shortfall) *shortfall = bytes > free_b ? bytes - free_b : bytes;
    *p = nullptr;
    return fail(CB_ENOMEM, "device " + std::to_string(d.id) + " lacks memory for " + std::to_string(bytes) +
                               " bytes (" + cudaGetErrorString(e) + ")");
  }
  d.allocs[*p] = {bytes, cat};
  d.mem[cat] += bytes;
  if (ipc) d.ipc_allocs[*p] = true;
  return CB_OK;
}

// `dst_stream` (on dst) waits for everything issued so far on `src_stream` (on src)
int join(DeviceCtx& dst, cudaStream_t dst_stream, DeviceCtx& src, cudaStream_t src_stream) {
  if (dst_stream == src_stream || !dst.local || !src.local) return CB_OK;
  CB_TRY(use(src));
  cudaEvent_t ev = src.ev_pool[src.ev_next++ % src.ev_pool.size()];
  CB_CUDA(cudaEventRecord(ev, src_stream));
  CB_TRY(use(dst));
  CB_CUDA(cudaStreamWaitEvent(dst_stream, ev, 0));
  return CB_OK;
}

// Stream-ordered free, no host synchronisation: the owning device's compute
// stream first joins every stream of every logical device (any of them may
// still read the buffer: peer row pulls, KV moves, op copies), then returns the
// buffer to the pool.
void dev_free(cb_model* m, int dev, void* p) {
  if (!p || !is_local(m, dev)) return;
  DeviceCtx& d = devctx(m, dev);
  for (auto& o : m->rt->devs)
    if (o.local)
      for (cudaStream_t s : {o.compute, o.copy, o.copy2}) join(d, d.compute, o, s);
  cudaSetDevice(d.ordinal);
  if (d.ipc_allocs.erase(p)) {
    cudaStreamSynchronize(d.compute);  // (the joins above: every stream that may read it is done)
    cudaFree(p);
  } else {
    cudaFreeAsync(p, d.compute);
  }
  auto it = d.allocs.find(p);
  if (it != d.allocs.end()) {
    d.mem[it->second.second] -= it->second.first;
    d.allocs.erase(it);
  }
}

int check_layer(cb_model* m, int layer) {
  if (layer < 1 || layer > m->d.n_layers)
    return fail(CB_EINVAL, "unknown layer " + std::to_string(layer));
  return CB_OK;
}
int check_dev(cb_model* m, int dev) {
  if (dev < 0 || dev >= int(m->rt->devs.size()))
    return fail(CB_EINVAL, "unknown device " + std::to_string(dev));
  return CB_OK;
}

int make_map(OpMap* map, const void* base, uint64_t rows, uint64_t k, uint32_t box_rows) {
  map->base = base;
  map->stride = k;
  int r = cb::make_kmajor_map(&map->m2, base, rows, k, k, box_rows);
  if (r != 0) return fail(CB_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  map->has3 = box_rows <= 128 && k % 128 == 0 && cb::make_kmajor_map3(&map->m3, base, rows, k, k, box_rows, 2) == 0;
  return CB_OK;
}

int ensure_ws(cb_model* m, int dev) {
  if (!is_local(m, dev)) return CB_OK;  // another process's device
  Workspace& w = m->ws[dev];
  if (w.ready) return CB_OK;
  DeviceCtx& dc = devctx(m, dev);
  const cb_model_desc& d = m->d;
  const size_t T = d.max_tokens;
  CB_TRY(dev_alloc(dc, (void**)&w.x, T * d.d_model * 4));
  CB_TRY(dev_alloc(dc, (void**)&w.h, T * d.d_model * 2));
  CB_TRY(dev_alloc(dc, (void**)&w.ssq, T * (d.d_model / 32) * 4));
  CB_TRY(dev_alloc(dc, (void**)&w.hl, size_t(d.max_slots) * d.d_model * 2));
  CB_TRY(dev_alloc(dc, (void**)&w.qkv, T * m->qkv_n * 2));
  CB_TRY(dev_alloc(dc, (void**)&w.att, T * m->q_n * 2));
  CB_TRY(dev_alloc(dc, (void**)&w.act, T * d.d_ff * 2));
  CB_TRY(dev_alloc(dc, (void**)&w.meta, (3 * T + d.max_slots + 4 + 4 * (T / 64 + d.max_slots)) * 4));
  CB_TRY(dev_alloc(dc, (void**)&w.next, size_t(d.max_slots) * 4));
  const size_t gws = cb::gemm_ws_floats(dc.num_sms);
  CB_TRY(dev_alloc(dc, (void**)&w.gemm_ws, gws * 4));
  CB_TRY(dev_alloc(dc, (void**)&w.gemm_cnt, size_t(cb::kGemmMaxTiles) * 4));
  CB_CUDA(cudaMemset(w.gemm_cnt, 0, size_t(cb::kGemmMaxTiles) * 4));
  w.attn_ws_floats = size_t(4 * dc.num_sms) * 8 * (m->hd + 2) * 4;
  CB_TRY(dev_alloc(dc, (void**)&w.attn_ws, w.attn_ws_floats * 4));
  CB_TRY(dev_alloc(dc, (void**)&w.attn_cnt, size_t(std::max(d.max_tokens, d.max_slots)) * d.n_kv_heads * 4));
  CB_CUDA(cudaMemset(w.attn_cnt, 0, size_t(std::max(d.max_tokens, d.max_slots)) * d.n_kv_heads * 4));
  // RoPE table, rotate-half convention: angle(pos, i) = pos * theta^(-2i/hd)
  const int half = m->hd / 2;
  std::vector<float2> tab(size_t(d.max_ctx) * half);
  for (int p = 0; p < d.max_ctx; ++p)
    for (int i = 0; i < half; ++i) {
      const double inv = std::pow(double(d.rope_theta), -2.0 * i / double(m->hd));
      const double ang = double(p) * inv;
      tab[size_t(p) * half + i] = make_float2(float(std::cos(ang)), float(std::sin(ang)));
    }
  CB_TRY(dev_alloc(dc, (void**)&w.rope, tab.size() * sizeof(float2)));
  CB_CUDA(cudaMemcpy(w.rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
  if (dev == m->home) {
    CB_TRY(dev_alloc(dc, (void**)&w.logits, size_t(d.max_slots) * d.vocab * 4));
  }
  for (int i = 0; i < kTnCount; ++i) {
    CB_TRY(make_map(&w.map_h[i], w.h, T, d.d_model, kTns[i]));
    CB_TRY(make_map(&w.map_hl[i], w.hl, d.max_slots, d.d_model, kTns[i]));
    CB_TRY(make_map(&w.map_att[i], w.att, T, m->q_n, kTns[i]));
    CB_TRY(make_map(&w.map_act[i], w.act, T, d.d_ff, kTns[i]));
  }
  w.ready = true;
  return CB_OK;
}

int make_layer_maps(cb_model* m, LayerCopy& c) {
  const cb_model_desc& d = m->d;
  CB_TRY(make_map(&c.m_qkv, c.block + m->off_qkv, m->qkv_n, d.d_model, 128));
  CB_TRY(make_map(&c.m_o, c.block + m->off_o, d.d_model, m->q_n, 128));
  CB_TRY(make_map(&c.m_gu, c.block + m->off_gu, 2 * size_t(d.d_ff), d.d_model, 128));
  CB_TRY(make_map(&c.m_d, c.block + m->off_d, d.d_model, d.d_ff, 128));
  return CB_OK;
}

// st != null: stream-ordered reservation for a scaling op (no host sync);
// *created tells the caller whether this call allocated the block.
size_t kv_token_bytes(cb_model* m);
size_t kv_slot_bytes(cb_model* m) { return size_t(m->d.max_ctx) * kv_token_bytes(m); }
int kv_device(const LayerState& L);
void sync_all_devices(cb_model* m);

// Slots a new KV block on `dev` holds: every slot for an unreplicated layer's
// KV device; the split_batch share ceil(max_slots / p) on each device of a
// replicated layer (the original included: see kv_shrink_empty), p counting
// the replications still pending.
int kv_cap_for(cb_model* m, const LayerState& L, int dev) {
  const int ms = m->d.max_slots;
  if (L.reps.empty()) return ms;
  int p = int(L.reps.size());
  for (const auto& pk : L.pend) p += pk.first == OPK_REPLICATE ? 1 : 0;
  bool replica = false;
  for (const auto& c : L.reps) replica |= c.dev == dev;
  for (const auto& pk : L.pend) replica |= pk.first == OPK_REPLICATE && pk.second == dev;
  if (!replica || p <= 1) return ms;
  return std::min(ms, (ms + p - 1) / p);
}

int kv_alloc_bytes(cb_model* m, DeviceCtx& dc, bool host, size_t bytes, uint16_t** p, uint64_t* shortfall,
                   cudaStream_t st) {
  if (host) {
    CB_CUDA(cudaHostAlloc((void**)p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    return CB_OK;
  }
  return dev_alloc(dc, (void**)p, bytes, shortfall, MEM_KV, st);
}

// st != null: stream-ordered reservation for a scaling op (no host sync);
// *created tells the caller whether this call allocated the block.
int ensure_kv(cb_model* m, LayerState& L, int dev, uint64_t* shortfall = nullptr, cudaStream_t st = nullptr,
              bool* created = nullptr, int cap = 0) {
  if (created) *created = false;
  if (L.kv.count(dev) || !is_local(m, dev)) return CB_OK;
  const int ms = m->d.max_slots;
  if (cap <= 0) cap = kv_cap_for(m, L, dev);
  DeviceCtx& dc = devctx(m, dev);
  KvBlock b;
  b.cap = cap;
  CB_TRY(kv_alloc_bytes(m, dc, false, size_t(cap) * kv_slot_bytes(m), &b.p, shortfall, st));
  if (cap < ms) {
    b.table = true;
    CB_TRY(use(dc));
    if (cudaHostAlloc((void**)&b.map_h, size_t(ms) * 4, cudaHostAllocPortable) != cudaSuccess ||
        cudaMalloc((void**)&b.map_d, size_t(ms) * 4) != cudaSuccess) {
      cudaGetLastError();
      dev_free(m, dev, b.p);
      return fail(CB_ENOMEM, "KV slot table allocation failed");
    }
    for (int i = 0; i < ms; ++i) b.map_h[i] = -1;
    for (int i = cap - 1; i >= 0; --i) b.free_idx.push_back(i);
    b.dirty = true;
  }
  L.kv[dev] = b;
  if (created) *created = true;
  return CB_OK;
}

size_t kv_block_bytes_of(cb_model* m, const KvBlock& b) { return size_t(b.cap) * kv_slot_bytes(m); }

// Free a device's KV block (and its slot table).
void free_kv_block(cb_model* m, LayerState& L, int dev, KvBlock& b) {
  (void)L;
  if (b.host) {
    sync_all_devices(m);
    cudaFreeHost(b.p);
  } else {
    dev_free(m, dev, b.p);
  }
  if (b.table && is_local(m, dev)) {
    sync_all_devices(m);
    cudaFreeHost(b.map_h);
    cudaSetDevice(devctx(m, dev).ordinal);
    cudaFree(b.map_d);
  }
  b = KvBlock{};
}

// Local index of `slot` in a block (the slot itself without a table).
int kv_index(const KvBlock& b, int slot) { return b.table ? b.map_h[slot] : slot; }

// Grow a table block by an eighth (at least one slot): new block, the old one
// copied whole on the device's compute stream (every write into a block is
// issued on its device's compute stream), the old freed stream-ordered.
int kv_grow(cb_model* m, KvBlock& b, int dev) {
  DeviceCtx& dc = devctx(m, dev);
  const int ncap = std::min(m->d.max_slots, b.cap + std::max(1, b.cap / 8));
  uint16_t* np = nullptr;
  CB_TRY(kv_alloc_bytes(m, dc, b.host, size_t(ncap) * kv_slot_bytes(m), &np, nullptr, nullptr));
  CB_TRY(use(dc));
  CB_CUDA(cudaMemcpyAsync(np, b.p, kv_block_bytes_of(m, b), cudaMemcpyDefault, dc.compute));
  if (b.host) {
    sync_all_devices(m);
    cudaFreeHost(b.p);
  } else {
    dev_free(m, dev, b.p);
  }
  b.p = np;
  for (int i = ncap - 1; i >= b.cap; --i) b.free_idx.push_back(i);
  b.cap = ncap;
  return CB_OK;
}

// `slot`'s KV is (about to be) held by `dev`: give it a local index there.
int kv_assign(cb_model* m, LayerState& L, int dev, int slot) {
  auto it = L.kv.find(dev);
  if (it == L.kv.end() || !it->second.table) return CB_OK;
  KvBlock& b = it->second;
  if (b.map_h[slot] >= 0) return CB_OK;
  if (b.free_idx.empty()) {
    if (b.cap >= m->d.max_slots) return fail(CB_ESTATE, "KV slot table full");
    CB_TRY(kv_grow(m, b, dev));
  }
  b.map_h[slot] = b.free_idx.back();
  b.free_idx.pop_back();
  b.dirty = true;
  return CB_OK;
}

// Grow dev's table block (if any) until `need` more slots fit.  Called before a
// batch of copies into the block is queued: inside a transport group
// (SPMD) the copies run at the group's close, so the block must not be
// replaced while they are queued.
int kv_reserve(cb_model* m, LayerState& L, int dev, int need) {
  auto it = L.kv.find(dev);
  if (it == L.kv.end() || !it->second.table) return CB_OK;
  KvBlock& b = it->second;
  while (int(b.free_idx.size()) < need && b.cap < m->d.max_slots) CB_TRY(kv_grow(m, b, dev));
  return CB_OK;
}

// `slot`'s KV left `dev` (or the slot was released): its index becomes
// reusable at the next step.
void kv_unassign(LayerState& L, int dev, int slot) {
  auto it = L.kv.find(dev);
  if (it == L.kv.end() || !it->second.table) return;
  KvBlock& b = it->second;
  if (b.map_h[slot] < 0) return;
  b.pending.push_back(b.map_h[slot]);
  b.map_h[slot] = -1;
  b.dirty = true;
}

// the slot table the kernels of (layer, dev) read this step (null: identity)
int kv_table_for_launch(KvBlock& b, DeviceCtx& dc, cudaStream_t st, const int32_t** out, int n) {
  *out = nullptr;
  if (!b.table) return CB_OK;
  if (b.dirty) {
    CB_TRY(use(dc));
    CB_CUDA(cudaMemcpyAsync(b.map_d, b.map_h, size_t(n) * 4, cudaMemcpyHostToDevice, st));
    b.dirty = false;
  }
  *out = b.map_d;
  return CB_OK;
}

void drop_kv_if_unused(cb_model* m, LayerState& L, int dev) {
  auto it = L.kv.find(dev);
  if (it == L.kv.end()) return;
  for (int o : L.owner)
    if (o == dev) return;
  const bool attn_here =
      L.reps.size() > 1
          ? std::any_of(L.reps.begin(), L.reps.end(), [&](const LayerCopy& c) { return c.dev == dev; })
          : kv_device(L) == dev;
  if (attn_here) return;
  free_kv_block(m, L, dev, it->second);
  L.kv.erase(it);
}

// After a replication commits: a block of the layer that holds no live KV and
// more slots than the new share is dropped; it is re-created at its first use,
// sized for the share (a layer replicated before serving -- config 3 -- so
// never keeps a full block on its original).
void kv_shrink_empty(cb_model* m, LayerState& L) {
  for (auto it = L.kv.begin(); it != L.kv.end();) {
    const int dev = it->first;
    KvBlock& b = it->second;
    bool live = false;
    for (int slot = 0; slot < m->d.max_slots && !live; ++slot) live = L.owner[slot] == dev;
    if (!b.host && !live && b.cap > kv_cap_for(m, L, dev)) {
      free_kv_block(m, L, dev, b);
      it = L.kv.erase(it);
    } else {
      ++it;
    }
  }
}

// indices released during the previous step become reusable (cb_step entry:
// the previous step and every copy it issued have completed)
void kv_release_pending(cb_model* m) {
  for (auto& L : m->layers)
    for (auto& kv : L.kv) {
      KvBlock& b = kv.second;
      b.free_idx.insert(b.free_idx.end(), b.pending.begin(), b.pending.end());
      b.pending.clear();
    }
}

int kv_device(const LayerState& L) { return L.kv_override >= 0 ? L.kv_override : L.reps[0].dev; }

size_t kv_token_bytes(cb_model* m) { return size_t(2) * m->kv_n * 2; }
size_t kv_slot_offset(cb_model* m, int idx) { return size_t(idx) * m->d.max_ctx * m->kv_n * 2; }  // elements
// element offset of `slot`'s position p0 inside dev's block (null block: another rank's)
uint16_t* kv_ptr(cb_model* m, LayerState& L, int dev, int slot, int p0) {
  if (!is_local(m, dev)) return nullptr;
  KvBlock& b = L.kv.at(dev);
  const int idx = kv_index(b, slot);
  if (idx < 0) return nullptr;
  return b.p + kv_slot_offset(m, idx) + size_t(p0) * m->kv_n * 2;
}

// copy KV positions [p0, p1) of `slot` from src's block to dst's block (on
// st, a stream of dst; across processes: channel ch, the sender on src_st)
int kv_copy(cb_model* m, LayerState& L, int slot, int src, int dst, int p0, int p1, cudaStream_t st,
            uint64_t* bytes, int ch = 0, cudaStream_t src_st = nullptr) {
  if (p1 <= p0 || src == dst) return CB_OK;
  const size_t tb = kv_token_bytes(m);
  CB_TRY(kv_assign(m, L, dst, slot));
  uint16_t* sp = kv_ptr(m, L, src, slot, p0);
  uint16_t* dp = kv_ptr(m, L, dst, slot, p0);
  if ((is_local(m, src) && !sp) || (is_local(m, dst) && !dp)) return fail(CB_ESTATE, "KV slot has no index");
  if (crosses(m, src, dst)) {
    if (bytes) *bytes += size_t(p1 - p0) * tb;
    return xmove(m, ch, src, sp, src_st ? src_st : (is_local(m, src) ? devctx(m, src).compute : nullptr), dst, dp,
                 st, size_t(p1 - p0) * tb);
  }
  // cudaMemcpyDefault: either block may be offloaded to mapped pinned host memory
  CB_CUDA(cudaMemcpyAsync(dp, sp, size_t(p1 - p0) * tb, cudaMemcpyDefault, st));
  if (bytes) *bytes += size_t(p1 - p0) * tb;
  return CB_OK;
}

// copy the whole live KV prefix of `slot` (pulled on dst's stream)
int kv_move(cb_model* m, LayerState& L, int slot, int src, int dst, cudaStream_t st, uint64_t* bytes) {
  return kv_copy(m, L, slot, src, dst, 0, m->slot_len[slot], st, bytes);
}

// Fused RMSNorm hooks of one GEMM (kernels.h GemmArgs): consume = X rows are
// h' = bf16(x * gamma), outputs scaled by the rows' rsqrt(mean(x^2) + eps);
// gamma_next != null = EPI_RESID producer of h' / ssq for the next norm.
struct NormIO {
  bool consume = false;
  const uint16_t* gamma_next = nullptr;
};

int gemm(cb_model* m, int dev, const OpMap& w, const OpMap* xmaps, int N, int K, int T, int row_off, int epi,
         void* out, long long ldo, const NormIO& nio = NormIO{}) {
  DeviceCtx& dc = devctx(m, dev);
  Workspace& ws = m->ws[dev];
  cb::GemmPlan plan = cb::gemm_plan(N, K, T, dc.num_sms, m->cur_T);
  const OpMap& xm = xmaps[box_index(plan.box_rows)];
  if (plan.kd == 2 && !(w.has3 && xm.has3)) plan.kd = 1;
  cb::GemmArgs a{};
  a.N = N;
  a.K = K;
  a.T = T;
  a.row_off = row_off;
  a.epi = epi;
  a.ldo = ldo;
  a.out = out;
  a.out_rows = out == ws.logits ? m->d.max_slots : m->d.max_tokens;
  a.w_base = w.base;
  a.w_stride = (long long)w.stride;
  a.ws = ws.gemm_ws;
  a.counters = ws.gemm_cnt;
  if (nio.consume || nio.gamma_next) {
    a.ssq_np = m->d.d_model / 32;
    a.norm_d = m->d.d_model;
    a.norm_eps = m->d.norm_eps;
  }
  if (nio.consume) a.ssq_in = ws.ssq;
  if (nio.gamma_next) {
    a.h_out = ws.h;
    a.gamma_next = nio.gamma_next;
    a.ssq_out = ws.ssq;
  }
  const double out_b = (epi == cb::EPI_F32 || epi == cb::EPI_RESID) ? 4.0 : 2.0;
  const double out_n = epi == cb::EPI_SWIGLU ? N / 2.0 : double(N);
  const double bytes = double(N) * K * 2 + double(T) * K * 2 + double(T) * out_n * out_b +
                       (epi == cb::EPI_RESID ? double(T) * N * 4 : 0.0);
  // output map for the TMA-store epilogue (rows = the buffer's rows: a store box
  // never crosses the launch's last token row, partial chunks use register stores)
  const uint64_t ocols = epi == cb::EPI_SWIGLU ? uint64_t(N) / 2 : uint64_t(N);
  const uint64_t orows = out == ws.logits ? uint64_t(m->d.max_slots) : uint64_t(m->d.max_tokens);
  const auto key = std::make_tuple(static_cast<const void*>(out), epi, ocols, uint64_t(ldo), orows);
  const CUtensorMap* om = nullptr;
  auto it = ws.out_maps.find(key);
  if (it != ws.out_maps.end()) {
    om = &it->second;
  } else {
    CUtensorMap mo;
    if (cb::make_out_map(&mo, out, epi, orows, ocols, uint64_t(ldo)) == 0)
      om = &(ws.out_maps[key] = mo);
  }
  ProfScope ps(m, dev, CB_KCLASS_GEMM, dc.compute, bytes, 2.0 * N * K * T);
  CB_CUDA(cb::gemm_launch(plan.kd == 2 ? w.m3 : w.m2, plan.kd == 2 ? xm.m3 : xm.m2, a, plan, dc.num_sms, dc.compute,
                          om));
  return CB_OK;
}

// Move residual rows so that every row sits on the device of its new segment.
// with_norm: the next layer consumes fused-norm input (h' rows + sums of squares travel too)
int reshard_rows(cb_model* m, const std::vector<Seg>& from, const std::vector<Seg>& to, bool with_norm);
int reshard(cb_model* m, const std::vector<Seg>& from, const std::vector<Seg>& to, bool with_norm) {
  XGroup grp(m, 0);
  CB_TRY(reshard_rows(m, from, to, with_norm));
  return grp.close();
}

int reshard_rows(cb_model* m, const std::vector<Seg>& from, const std::vector<Seg>& to, bool with_norm) {
  const size_t row_bytes = size_t(m->d.d_model) * 4;
  for (const Seg& ns : to)
    for (const Seg& os : from) {
      const int a = std::max(ns.r0, os.r0), b = std::min(ns.r1, os.r1);
      if (a >= b || os.dev == ns.dev) continue;
      if (crosses(m, os.dev, ns.dev)) {
        // the reference's replica scatter / gather (_kernels.py:41-51) between processes:
        // residual rows (+ the next norm's input rows and sums of squares when fused)
        const int sd = os.dev, dd = ns.dev;
        const bool ls = is_local(m, sd), ld = is_local(m, dd);
        if (!ls && !ld) continue;
        cudaStream_t ss = ls ? devctx(m, sd).compute : nullptr, ds = ld ? devctx(m, dd).compute : nullptr;
        auto at = [&](int dv, bool loc, auto* base, size_t row) {
          return loc ? reinterpret_cast<uint8_t*>(base) + size_t(a) * row : nullptr;
        };
        const size_t xr = row_bytes, hr = size_t(m->d.d_model) * 2, qr = size_t(m->d.d_model / 32) * 4;
        ProfScope ps(m, ld ? dd : sd, CB_KCLASS_COPY, ld ? ds : ss, double(b - a) * row_bytes);
        CB_TRY(xmove(m, 0, sd, at(sd, ls, ls ? m->ws[sd].x : nullptr, xr), ss, dd,
                     at(dd, ld, ld ? m->ws[dd].x : nullptr, xr), ds, size_t(b - a) * xr));
        if (with_norm) {
          CB_TRY(xmove(m, 0, sd, at(sd, ls, ls ? m->ws[sd].h : nullptr, hr), ss, dd,
                       at(dd, ld, ld ? m->ws[dd].h : nullptr, hr), ds, size_t(b - a) * hr));
          CB_TRY(xmove(m, 0, sd, at(sd, ls, ls ? m->ws[sd].ssq : nullptr, qr), ss, dd,
                       at(dd, ld, ld ? m->ws[dd].ssq : nullptr, qr), ds, size_t(b - a) * qr));
        }
        continue;
      }
      DeviceCtx& dd = devctx(m, ns.dev);
      DeviceCtx& sd = devctx(m, os.dev);
      CB_TRY(depend(dd, sd));
      CB_TRY(use(dd));
      ProfScope ps(m, ns.dev, CB_KCLASS_COPY, dd.compute, double(b - a) * row_bytes);
      CB_CUDA(cudaMemcpyPeerAsync(m->ws[ns.dev].x + size_t(a) * m->d.d_model, dd.ordinal,
                                  m->ws[os.dev].x + size_t(a) * m->d.d_model, sd.ordinal,
                                  size_t(b - a) * row_bytes, dd.compute));
      if (with_norm) {  // the next layer's normalised input rows and their sums of squares travel too
        const size_t np = size_t(m->d.d_model / 32);
        CB_CUDA(cudaMemcpyPeerAsync(m->ws[ns.dev].h + size_t(a) * m->d.d_model, dd.ordinal,
                                    m->ws[os.dev].h + size_t(a) * m->d.d_model, sd.ordinal,
                                    size_t(b - a) * m->d.d_model * 2, dd.compute));
        CB_CUDA(cudaMemcpyPeerAsync(m->ws[ns.dev].ssq + size_t(a) * np, dd.ordinal, m->ws[os.dev].ssq + size_t(a) * np,
                                    sd.ordinal, size_t(b - a) * np * 4, dd.compute));
      }
    }
  return CB_OK;
}

// ---- sub-module (projection) overrides: where each projection's weights live
struct ProjView {
  int dev;
  const uint8_t* base;
  uint64_t row_stride;  // elements
  int rows, k;
  int col0;  // column offset inside the fused qkv output (Q, K, V)
};

size_t block_offset(cb_model* m, int kind) {
  const size_t dm = m->d.d_model;
  switch (kind) {
    case CB_ATTN_PROJ_Q: return m->off_qkv;
    case CB_ATTN_PROJ_K: return m->off_qkv + size_t(m->q_n) * dm * 2;
    case CB_ATTN_PROJ_V: return m->off_qkv + size_t(m->q_n + m->kv_n) * dm * 2;
    case CB_ATTN_PROJ_O: return m->off_o;
    case CB_SELF_ATTENTION: return m->off_qkv;
    case CB_FFN_PROJ_GATE: return m->off_gu;
    case CB_FFN_PROJ_UP: return m->off_gu + dm * 2;  // odd rows of the interleaved gate/up block
    case CB_FFN_PROJ_DOWN: return m->off_d;
  }
  return 0;
}

ProjView proj_view(cb_model* m, const LayerState& L, int kind) {
  const cb_model_desc& d = m->d;
  ProjView v{};
  v.col0 = 0;
  switch (kind) {
    case CB_ATTN_PROJ_Q: v.rows = m->q_n; v.k = d.d_model; break;
    case CB_ATTN_PROJ_K: v.rows = m->kv_n; v.k = d.d_model; v.col0 = m->q_n; break;
    case CB_ATTN_PROJ_V: v.rows = m->kv_n; v.k = d.d_model; v.col0 = m->q_n + m->kv_n; break;
    case CB_ATTN_PROJ_O: v.rows = d.d_model; v.k = m->q_n; break;
    case CB_FFN_PROJ_GATE:
    case CB_FFN_PROJ_UP: v.rows = d.d_ff; v.k = d.d_model; break;
    case CB_FFN_PROJ_DOWN: v.rows = d.d_model; v.k = d.d_ff; break;
  }
  const ModCopy& own = L.mod[kind];
  const ModCopy& sa = L.mod[CB_SELF_ATTENTION];
  if (own.dev >= 0) {
    v.dev = own.dev;
    v.base = own.buf;
    v.row_stride = uint64_t(v.k);
  } else if (kind <= CB_ATTN_PROJ_O && sa.dev >= 0) {
    v.dev = sa.dev;  // SELF_ATTENTION copy = block[off_qkv, off_o + |wo|)
    v.base = sa.buf + (block_offset(m, kind) - m->off_qkv);
    v.row_stride = uint64_t(v.k);
  } else {
    v.dev = L.reps[0].dev;
    v.base = L.reps[0].block + block_offset(m, kind);
    v.row_stride = uint64_t(v.k) * ((kind == CB_FFN_PROJ_GATE || kind == CB_FFN_PROJ_UP) ? 2 : 1);
  }
  return v;
}

int ensure_gbuf(cb_model* m, int dev) {
  Workspace& w = m->ws[dev];
  if (w.gbuf) return CB_OK;
  return dev_alloc(devctx(m, dev), (void**)&w.gbuf, size_t(m->d.max_tokens) * m->d.d_ff * 2);
}

// rows [r0, r0 + T) of a row-major buffer, device src -> dst (pulled on dst's stream)
int hop_rows(cb_model* m, int src, int dst, const void* sbase, void* dbase, size_t row_bytes, int r0, int T) {
  if (src == dst || T <= 0) return CB_OK;
  DeviceCtx& dd = devctx(m, dst);
  DeviceCtx& sd = devctx(m, src);
  CB_TRY(depend(dd, sd));
  CB_TRY(use(dd));
  ProfScope ps(m, dst, CB_KCLASS_COPY, dd.compute, double(T) * row_bytes);
  CB_CUDA(cudaMemcpyPeerAsync(static_cast<uint8_t*>(dbase) + size_t(r0) * row_bytes, dd.ordinal,
                              static_cast<const uint8_t*>(sbase) + size_t(r0) * row_bytes, sd.ordinal,
                              size_t(T) * row_bytes, dd.compute));
  return CB_OK;
}

// columns [c0, c0 + nc) (bf16) of rows [r0, r0 + T) of a [rows][pitch] buffer, src -> dst
int hop_cols(cb_model* m, int src, int dst, const uint16_t* sbase, uint16_t* dbase, int pitch, int c0, int nc, int r0,
             int T) {
  if (src == dst || T <= 0) return CB_OK;
  DeviceCtx& dd = devctx(m, dst);
  CB_TRY(depend(dd, devctx(m, src)));
  CB_TRY(use(dd));
  ProfScope ps(m, dst, CB_KCLASS_COPY, dd.compute, double(T) * nc * 2);
  const size_t off = size_t(r0) * pitch + c0;
  CB_CUDA(cudaMemcpy2DAsync(dbase + off, size_t(pitch) * 2, sbase + off, size_t(pitch) * 2, size_t(nc) * 2, T,
                            cudaMemcpyDefault, dd.compute));
  return CB_OK;
}

int proj_gemm(cb_model* m, const ProjView& v, const OpMap* xmaps, int T, int r0, int epi, void* out,
              long long ldo) {
  OpMap wm;
  CB_TRY(use(devctx(m, v.dev)));
  if (cb::make_kmajor_map(&wm.m2, v.base, uint64_t(v.rows), uint64_t(v.k), v.row_stride, 128) != 0)
    return fail(CB_ECUDA, "cuTensorMapEncodeTiled failed for a migrated projection");
  wm.base = v.base;
  wm.stride = v.row_stride;
  return gemm(m, v.dev, wm, xmaps, v.rows, v.k, T, r0, epi, out, ldo);
}

// RoPE + KV append + attention for the segment's rows: qkv on `dev` -> att on `dev`.
// Runs where the rows' KV lives: on the replica itself for a replicated layer,
// on the KV device (MigrateSubModule KV_CACHE / MigrateLayer without KV) otherwise.
int attention_part(cb_model* m, LayerState& L, const Seg& s, const std::vector<int>& seq_slot,
                   const std::vector<int>& row_pos) {
  const cb_model_desc& d = m->d;
  const int dev = s.dev;
  const int T = s.r1 - s.r0;
  DeviceCtx& dc = devctx(m, dev);
  Workspace& ws = m->ws[dev];
  const int ad = L.reps.size() > 1 ? dev : kv_device(L);
  DeviceCtx& ac = devctx(m, ad);
  CB_TRY(ensure_ws(m, ad));
  Workspace& wa = m->ws[ad];
  const size_t qkv_row = size_t(m->qkv_n) * 2, att_row = size_t(m->q_n) * 2;
  if (ad != dev) {
    CB_TRY(depend(ac, dc));
    CB_TRY(use(ac));
    CB_CUDA(cudaMemcpyPeerAsync(reinterpret_cast<uint8_t*>(wa.qkv) + s.r0 * qkv_row, ac.ordinal,
                                reinterpret_cast<uint8_t*>(ws.qkv) + s.r0 * qkv_row, dc.ordinal, T * qkv_row,
                                ac.compute));
  }
  CB_TRY(ensure_kv(m, L, ad));
  CB_TRY(use(ac));
  KvBlock& kvb = L.kv.at(ad);
  uint16_t* kv = kvb.p;
  const int32_t* kv_map = nullptr;  // slot -> local index in a share-sized replica block
  CB_TRY(kv_table_for_launch(kvb, ac, ac.compute, &kv_map, d.max_slots));
  const int32_t* row_slot = wa.meta + m->cur_T;
  const int32_t* rpos = wa.meta + 2 * m->cur_T;
  // decode rows are one per sequence: RoPE + KV append fuse into the attention kernel
  const bool fused = m->cur_phase == CB_PHASE_DECODE;
  if (!fused) {
    ProfScope ps(m, ad, CB_KCLASS_ELEMWISE, ac.compute, double(T) * m->qkv_n * 4);
    CB_CUDA(cb::rope_kv_launch(wa.qkv, kv, kv_map, wa.rope, row_slot, rpos, T, s.r0, d.n_heads, d.n_kv_heads,
                               m->hd, d.max_ctx, ac.compute));
  }
  if (!fused) {
    // prefill: causal tensor-core attention over the segment's sequences' 256-row blocks
    const int b0 = m->seq_blk[s.s0], b1 = m->seq_blk[s.s1];
    const int4* blocks = reinterpret_cast<const int4*>(wa.meta + ((3 * m->cur_T + m->cur_bs + 3) & ~3)) + b0;
    cb::AttnArgs pa{};
    pa.qkv = wa.qkv;
    pa.kv = kv;
    pa.out = wa.att;
    pa.T = T;
    pa.row_off = 0;  // block rows are absolute pass rows
    pa.H = d.n_heads;
    pa.Hkv = d.n_kv_heads;
    pa.hd = m->hd;
    pa.max_ctx = d.max_ctx;
    pa.qkv_rows = m->cur_T;
    pa.kv_slots = kvb.cap;
    pa.kv_map = kv_map;
    pa.scale = 1.0f / std::sqrt(float(m->hd));
    double flops = 0;  // QK^T + PV over the causal prefix of every row
    for (int r = s.r0; r < s.r1; ++r) flops += 4.0 * (row_pos[r] + 1) * m->q_n;
    ProfScope ps(m, ad, CB_KCLASS_ATTENTION, ac.compute, double(T) * m->q_n * 4, flops);
    CB_CUDA(cb::prefill_attention_launch(pa, blocks, b1 - b0, ac.compute));
    if (ad != dev) {
      CB_TRY(depend(dc, ac));
      CB_TRY(use(dc));
      CB_CUDA(cudaMemcpyPeerAsync(reinterpret_cast<uint8_t*>(ws.att) + s.r0 * att_row, dc.ordinal,
                                  reinterpret_cast<uint8_t*>(wa.att) + s.r0 * att_row, ac.ordinal, T * att_row,
                                  dc.compute));
    }
    return CB_OK;
  }
  int max_len = 0;
  double kv_tokens = 0;
  for (int r = s.r0; r < s.r1; ++r) {
    max_len = std::max(max_len, row_pos[r] + 1);
    kv_tokens += row_pos[r] + 1;
  }
  cb::AttnArgs aa{};
  aa.qkv = wa.qkv;
  aa.kv = kv;
  aa.out = wa.att;
  aa.row_slot = row_slot;
  aa.kv_map = kv_map;
  aa.row_pos = rpos;
  aa.ws = wa.attn_ws;
  aa.ws_floats = wa.attn_ws_floats;
  aa.counters = wa.attn_cnt;
  aa.kind_T = m->cur_T;  // the split decision follows the whole pass, not this replica's rows
  aa.kv_slots = kvb.host ? 0 : kvb.cap;  // device-memory block: the TMA-fed decode kernel may read it
  aa.T = T;
  aa.row_off = s.r0;
  aa.H = d.n_heads;
  aa.Hkv = d.n_kv_heads;
  aa.hd = m->hd;
  aa.max_ctx = d.max_ctx;
  aa.max_len = max_len;
  aa.scale = 1.0f / std::sqrt(float(m->hd));
  aa.rope = fused ? wa.rope : nullptr;
  {
    // algorithmic bytes: every attended K/V row once, q in, output out
    ProfScope ps(m, ad, CB_KCLASS_ATTENTION, ac.compute, kv_tokens * kv_token_bytes(m) + double(T) * m->q_n * 4,
                 kv_tokens * 4.0 * m->q_n);
    CB_CUDA(cb::attention_launch(aa, ac.num_sms, ac.compute));
  }
  if (ad != dev) {
    CB_TRY(depend(dc, ac));
    CB_TRY(use(dc));
    CB_CUDA(cudaMemcpyPeerAsync(reinterpret_cast<uint8_t*>(ws.att) + s.r0 * att_row, dc.ordinal,
                                reinterpret_cast<uint8_t*>(wa.att) + s.r0 * att_row, ac.ordinal, T * att_row,
                                dc.compute));
  }
  return CB_OK;
}

// KV rows follow their sequence (SURVEY §7 hard part 1, option B): before a
// segment runs, every slot of it whose KV prefix sits on another device moves
// to the device that attends it.  Called on every rank for every segment (the
// owner bookkeeping is replicated; a move between processes is an exchange).
int kv_follow(cb_model* m, LayerState& L, const Seg& s, const std::vector<int>& seq_slot) {
  const int ad = L.reps.size() > 1 ? s.dev : kv_device(L);
  const bool la = is_local(m, ad);
  if (la) {
    CB_TRY(ensure_kv(m, L, ad));
    const KvBlock& b = L.kv.at(ad);
    int need = 0;
    for (int q = s.s0; q < s.s1 && b.table; ++q) need += b.map_h[seq_slot[q]] < 0;
    CB_TRY(kv_reserve(m, L, ad, need));
  }
  for (int q = s.s0; q < s.s1; ++q) {
    const int slot = seq_slot[q];
    const int owner = L.owner[slot];
    if (owner >= 0 && owner != ad && m->slot_len[slot] > 0) {
      const double nb = double(m->slot_len[slot]) * kv_token_bytes(m);
      if (crosses(m, owner, ad)) {
        const bool lo = is_local(m, owner);
        if (la || lo) {
          const int pdev = la ? ad : owner;
          ProfScope ps(m, pdev, CB_KCLASS_COPY, devctx(m, pdev).compute, nb);
          CB_TRY(kv_move(m, L, slot, owner, ad, la ? devctx(m, ad).compute : nullptr, nullptr));
        } else {
          CB_TRY(kv_move(m, L, slot, owner, ad, nullptr, nullptr));  // bookkeeping only
        }
      } else {
        DeviceCtx& ac = devctx(m, ad);
        CB_TRY(depend(ac, devctx(m, owner)));
        CB_TRY(use(ac));
        ProfScope ps(m, ad, CB_KCLASS_COPY, ac.compute, nb);
        CB_TRY(kv_move(m, L, slot, owner, ad, ac.compute, nullptr));
      }
    }
    if (owner != ad && owner >= 0) kv_unassign(L, owner, slot);
    CB_TRY(kv_assign(m, L, ad, slot));
    L.owner[slot] = ad;
  }
  return CB_OK;
}

// A projection that runs on another device: its input rows hop there, the
// fp32 residual rows too for the += epilogues (O, down), and the output rows
// hop back -- the "module on another device" of PAPER.md:182-189.
int remote_resid_proj(cb_model* m, const ProjView& v, int dev, const uint16_t* in_local, size_t in_row_bytes,
                      uint16_t* in_remote, const OpMap* xmaps_remote, int T, int r0) {
  const size_t x_row = size_t(m->d.d_model) * 4;
  CB_TRY(hop_rows(m, dev, v.dev, in_local, in_remote, in_row_bytes, r0, T));
  CB_TRY(hop_rows(m, dev, v.dev, m->ws[dev].x, m->ws[v.dev].x, x_row, r0, T));
  CB_TRY(proj_gemm(m, v, xmaps_remote, T, r0, cb::EPI_RESID, m->ws[v.dev].x, m->d.d_model));
  return hop_rows(m, v.dev, dev, m->ws[v.dev].x, m->ws[dev].x, x_row, r0, T);
}

// Decoder layer with migrated projections (the layer is not replicated: the
// registry forbids overrides on replicated layers, domain.py:339-340).
int run_layer_overridden(cb_model* m, LayerState& L, const Seg& s, const std::vector<int>& seq_slot,
                         const std::vector<int>& row_pos) {
  const cb_model_desc& d = m->d;
  const LayerCopy& W = L.reps[s.rep];
  const int dev = s.dev;
  const int T = s.r1 - s.r0;
  DeviceCtx& dc = devctx(m, dev);
  Workspace& ws = m->ws[dev];
  const uint16_t* an = reinterpret_cast<const uint16_t*>(W.block + m->off_an);
  const uint16_t* fn = reinterpret_cast<const uint16_t*>(W.block + m->off_fn);
  const double norm_bytes = double(T) * d.d_model * 6 + d.d_model * 2.0;
  const size_t h_row = size_t(d.d_model) * 2;
  CB_TRY(use(dc));
  {
    ProfScope ps(m, dev, CB_KCLASS_ELEMWISE, dc.compute, norm_bytes);
    CB_CUDA(cb::rmsnorm_launch(ws.x, an, ws.h, T, d.d_model, d.norm_eps, s.r0, dc.compute));
  }
  // ---- Q, K, V: each projection where its weights live, into its column slice of qkv
  const bool qkv_moved = L.mod[CB_SELF_ATTENTION].dev >= 0 || L.mod[CB_ATTN_PROJ_Q].dev >= 0 ||
                         L.mod[CB_ATTN_PROJ_K].dev >= 0 || L.mod[CB_ATTN_PROJ_V].dev >= 0;
  if (!qkv_moved) {
    CB_TRY(gemm(m, dev, W.m_qkv, ws.map_h, m->qkv_n, d.d_model, T, s.r0, cb::EPI_BF16, ws.qkv, m->qkv_n));
  } else {
    std::vector<int> h_at{dev};
    for (int kind : {CB_ATTN_PROJ_Q, CB_ATTN_PROJ_K, CB_ATTN_PROJ_V}) {
      const ProjView v = proj_view(m, L, kind);
      CB_TRY(ensure_ws(m, v.dev));
      Workspace& we = m->ws[v.dev];
      if (std::find(h_at.begin(), h_at.end(), v.dev) == h_at.end()) {
        CB_TRY(hop_rows(m, dev, v.dev, ws.h, we.h, h_row, s.r0, T));
        h_at.push_back(v.dev);
      }
      CB_TRY(proj_gemm(m, v, we.map_h, T, s.r0, cb::EPI_BF16, we.qkv + v.col0, m->qkv_n));
      CB_TRY(hop_cols(m, v.dev, dev, we.qkv, ws.qkv, m->qkv_n, v.col0, v.rows, s.r0, T));
    }
  }
  CB_TRY(attention_part(m, L, s, seq_slot, row_pos));
  // ---- O (+= residual)
  {
    const ProjView v = proj_view(m, L, CB_ATTN_PROJ_O);
    if (v.dev == dev) {
      CB_TRY(proj_gemm(m, v, ws.map_att, T, s.r0, cb::EPI_RESID, ws.x, d.d_model));
    } else {
      CB_TRY(ensure_ws(m, v.dev));
      CB_TRY(remote_resid_proj(m, v, dev, ws.att, size_t(m->q_n) * 2, m->ws[v.dev].att, m->ws[v.dev].map_att, T,
                               s.r0));
    }
  }
  CB_TRY(use(dc));
  {
    ProfScope ps(m, dev, CB_KCLASS_ELEMWISE, dc.compute, norm_bytes);
    CB_CUDA(cb::rmsnorm_launch(ws.x, fn, ws.h, T, d.d_model, d.norm_eps, s.r0, dc.compute));
  }
  // ---- gate / up: fused SwiGLU GEMM unless one of them moved
  if (L.mod[CB_FFN_PROJ_GATE].dev < 0 && L.mod[CB_FFN_PROJ_UP].dev < 0) {
    CB_TRY(gemm(m, dev, W.m_gu, ws.map_h, 2 * d.d_ff, d.d_model, T, s.r0, cb::EPI_SWIGLU, ws.act, d.d_ff));
  } else {
    CB_TRY(ensure_gbuf(m, dev));
    std::vector<int> h_at{dev};
    for (int kind : {CB_FFN_PROJ_GATE, CB_FFN_PROJ_UP}) {
      const ProjView v = proj_view(m, L, kind);
      CB_TRY(ensure_ws(m, v.dev));
      CB_TRY(ensure_gbuf(m, v.dev));
      Workspace& we = m->ws[v.dev];
      if (std::find(h_at.begin(), h_at.end(), v.dev) == h_at.end()) {
        CB_TRY(hop_rows(m, dev, v.dev, ws.h, we.h, h_row, s.r0, T));
        h_at.push_back(v.dev);
      }
      uint16_t* out_e = kind == CB_FFN_PROJ_GATE ? we.gbuf : we.act;
      uint16_t* out_d = kind == CB_FFN_PROJ_GATE ? ws.gbuf : ws.act;
      CB_TRY(proj_gemm(m, v, we.map_h, T, s.r0, cb::EPI_BF16, out_e, d.d_ff));
      CB_TRY(hop_rows(m, v.dev, dev, out_e, out_d, size_t(d.d_ff) * 2, s.r0, T));
    }
    CB_TRY(use(dc));
    ProfScope ps(m, dev, CB_KCLASS_ELEMWISE, dc.compute, double(T) * d.d_ff * 6);
    CB_CUDA(cb::swiglu_launch(ws.gbuf, ws.act, T, d.d_ff, s.r0, dc.compute));
  }
  // ---- down (+= residual)
  {
    const ProjView v = proj_view(m, L, CB_FFN_PROJ_DOWN);
    if (v.dev == dev) {
      CB_TRY(proj_gemm(m, v, ws.map_act, T, s.r0, cb::EPI_RESID, ws.x, d.d_model));
    } else {
      CB_TRY(ensure_ws(m, v.dev));
      CB_TRY(remote_resid_proj(m, v, dev, ws.act, size_t(d.d_ff) * 2, m->ws[v.dev].act, m->ws[v.dev].map_act, T,
                               s.r0));
    }
  }
  return CB_OK;
}

// gamma_next: the norm that follows this layer (next layer's attention norm,
// or the final norm), readable from s.dev -- used when the pass fuses RMSNorm.
// fused_in: this layer's input arrives fused (fin[li]; the segment has <= 256
// rows, so the O -> gate/up norm fuses too); gamma_next != null: the next
// consumer is fused, so the down projection emits its h' and sums of squares.
int run_layer_segment(cb_model* m, LayerState& L, const Seg& s, const std::vector<int>& seq_slot,
                      const std::vector<int>& row_pos, bool fused_in, const uint16_t* gamma_next) {
  if (L.proj_ov) return run_layer_overridden(m, L, s, seq_slot, row_pos);
  const cb_model_desc& d = m->d;
  const LayerCopy& W = L.reps[s.rep];
  const int dev = s.dev;
  const int T = s.r1 - s.r0;
  DeviceCtx& dc = devctx(m, dev);
  Workspace& ws = m->ws[dev];
  CB_TRY(use(dc));
  const uint16_t* an = reinterpret_cast<const uint16_t*>(W.block + m->off_an);
  const uint16_t* fn = reinterpret_cast<const uint16_t*>(W.block + m->off_fn);
  const double norm_bytes = double(T) * d.d_model * 6 + d.d_model * 2.0;
  NormIO prod_next;
  prod_next.gamma_next = gamma_next;
  if (fused_in) {
    // RMSNorm folded into the GEMMs: the residual projections emit h' = bf16(x * gamma)
    // plus per-row sums of squares, the next projection scales its outputs by rsqrt(mean + eps)
    NormIO cons;
    cons.consume = true;
    NormIO prod_fn;
    prod_fn.gamma_next = fn;
    CB_TRY(gemm(m, dev, W.m_qkv, ws.map_h, m->qkv_n, d.d_model, T, s.r0, cb::EPI_BF16, ws.qkv, m->qkv_n, cons));
    CB_TRY(attention_part(m, L, s, seq_slot, row_pos));
    CB_TRY(use(dc));
    CB_TRY(gemm(m, dev, W.m_o, ws.map_att, d.d_model, m->q_n, T, s.r0, cb::EPI_RESID, ws.x, d.d_model, prod_fn));
    CB_TRY(gemm(m, dev, W.m_gu, ws.map_h, 2 * d.d_ff, d.d_model, T, s.r0, cb::EPI_SWIGLU, ws.act, d.d_ff, cons));
    CB_TRY(gemm(m, dev, W.m_d, ws.map_act, d.d_model, d.d_ff, T, s.r0, cb::EPI_RESID, ws.x, d.d_model, prod_next));
    return CB_OK;
  }
  {
    ProfScope ps(m, dev, CB_KCLASS_ELEMWISE, dc.compute, norm_bytes);
    CB_CUDA(cb::rmsnorm_launch(ws.x, an, ws.h, T, d.d_model, d.norm_eps, s.r0, dc.compute));
  }
  CB_TRY(gemm(m, dev, W.m_qkv, ws.map_h, m->qkv_n, d.d_model, T, s.r0, cb::EPI_BF16, ws.qkv, m->qkv_n));
  CB_TRY(attention_part(m, L, s, seq_slot, row_pos));
  CB_TRY(use(dc));
  CB_TRY(gemm(m, dev, W.m_o, ws.map_att, d.d_model, m->q_n, T, s.r0, cb::EPI_RESID, ws.x, d.d_model));
  {
    ProfScope ps(m, dev, CB_KCLASS_ELEMWISE, dc.compute, norm_bytes);
    CB_CUDA(cb::rmsnorm_launch(ws.x, fn, ws.h, T, d.d_model, d.norm_eps, s.r0, dc.compute));
  }
  CB_TRY(gemm(m, dev, W.m_gu, ws.map_h, 2 * d.d_ff, d.d_model, T, s.r0, cb::EPI_SWIGLU, ws.act, d.d_ff));
  CB_TRY(gemm(m, dev, W.m_d, ws.map_act, d.d_model, d.d_ff, T, s.r0, cb::EPI_RESID, ws.x, d.d_model, prod_next));
  return CB_OK;
}

// A norm vector (attention norm of layer li, or the final norm for li == n_layers)
// that kernels on logical device dev can read: a copy on the same physical GPU.
const uint16_t* norm_gamma_for(cb_model* m, int li, int dev) {
  if (m->rt->spmd) return m->norm_ready ? m->norm_tab + size_t(li) * m->d.d_model : nullptr;
  const int ord = devctx(m, dev).ordinal;
  if (li >= m->d.n_layers) return devctx(m, m->home).ordinal == ord ? m->final_norm : nullptr;
  for (const LayerCopy& c : m->layers[li].reps)
    if (devctx(m, c.dev).ordinal == ord) return reinterpret_cast<const uint16_t*>(c.block + m->off_an);
  return nullptr;
}

// SPMD: the norm table of this process (every layer's attention norm, then the
// final norm) -- each vector comes from the rank holding the layer's original
// (the final norm from the home rank); one collective, at the first step.
int build_norm_table(cb_model* m, int tdev) {
  const size_t dm = m->d.d_model;
  const int nl = m->d.n_layers;
  DeviceCtx& tc = devctx(m, tdev);
  if (!m->norm_tab) {
    CB_TRY(dev_alloc(tc, (void**)&m->norm_tab, size_t(nl + 1) * dm * 2, nullptr, MEM_WEIGHTS));
    m->norm_dev = tdev;
  }
  const int me = m->rt->my_rank;
  XGroup grp(m, 0);
  auto dev_of_rank = [&](int r) {
    for (const DeviceCtx& dc : m->rt->devs)
      if (dc.rank == r) return dc.id;
    return -1;
  };
  for (int li = 0; li <= nl; ++li) {
    const int src = li < nl ? m->layers[li].reps[0].dev : m->home;
    const int src_rank = devctx(m, src).rank;
    uint16_t* slot = m->norm_tab + size_t(li) * dm;
    CB_TRY(use(tc));
    if (src_rank == me) {
      const void* from = li < nl ? static_cast<const void*>(m->layers[li].reps[0].block + m->off_an)
                                 : static_cast<const void*>(m->final_norm);
      CB_CUDA(cudaMemcpyAsync(slot, from, dm * 2, cudaMemcpyDefault, tc.compute));
      for (int r : m->rt->ranks)
        if (r != me) CB_TRY(xfer(m, 0, true, tdev, dev_of_rank(r), slot, dm * 2, tc.compute));
    } else {
      CB_TRY(xfer(m, 0, false, tdev, src, slot, dm * 2, tc.compute));
    }
  }
  CB_TRY(grp.close());
  m->norm_ready = true;
  return CB_OK;
}

std::vector<int> split_batch_vec(int bs, int p) {
  std::vector<int> out(p);
  const int q = bs / p, r = bs % p;
  for (int j = 0; j < p; ++j) out[j] = (j >= p - r) ? q + 1 : q;
  return out;
}

// One pass over a group of sequences whose rows fit max_tokens.
double g_last_enqueue_ms = 0.0;  // experiments: host time to enqueue the last pass (cbt_last_enqueue_ms)

// One pass over sequences [g_off, g_off + bs) of a step of g_bs sequences (a
// prefill longer than max_tokens rows runs in several passes): each layer's
// rows are routed by split_batch over the WHOLE step (sim.py:717-725: one
// prefill of all fresh requests), so a sequence lands on the same replica as in
// the decode steps that follow and its KV does not move.
int step_pass(cb_model* m, int phase, int bs, const int32_t* slots, const int32_t* tokens, const int32_t* lens,
              int32_t* next_out, float* logits_out, float* ms_out, int g_off, int g_bs) {
  const auto enq0 = std::chrono::steady_clock::now();
  const cb_model_desc& d = m->d;
  const bool prefill = phase == CB_PHASE_PREFILL;
  std::vector<int> seq_row(bs + 1, 0);
  for (int i = 0; i < bs; ++i) seq_row[i + 1] = seq_row[i] + (prefill ? lens[i] : 1);
  const int T = seq_row[bs];
  std::vector<int> seq_slot(slots, slots + bs);
  std::vector<int> row_pos(T);
  int32_t* meta = m->pin_meta;
  m->cur_T = T;
  m->cur_phase = phase;
  for (int i = 0; i < bs; ++i)
    for (int r = seq_row[i]; r < seq_row[i + 1]; ++r) {
      const int pos = prefill ? r - seq_row[i] : m->slot_len[slots[i]];
      if (pos >= d.max_ctx) return fail(CB_EINVAL, "slot " + std::to_string(slots[i]) + " exceeds max_ctx");
      row_pos[r] = pos;
      meta[r] = tokens[r];
      meta[T + r] = slots[i];
      meta[2 * T + r] = pos;
    }
  for (int i = 0; i < bs; ++i) meta[3 * T + i] = seq_row[i + 1] - 1;
  // prefill: 256-row query blocks (two 128-row tiles) of every sequence for the tensor-core attention
  m->cur_bs = bs;
  m->seq_blk.assign(bs + 1, 0);
  int nblk = 0;
  const int blk_off = (3 * T + bs + 3) & ~3;  // int4-aligned
  if (prefill) {
    int32_t* blk = meta + blk_off;
    for (int i = 0; i < bs; ++i) {
      m->seq_blk[i] = nblk;
      const int len = seq_row[i + 1] - seq_row[i];
      for (int b0 = 0; b0 < len; b0 += 256, ++nblk) {
        blk[4 * nblk + 0] = seq_row[i] + b0;
        blk[4 * nblk + 1] = std::min(256, len - b0);
        blk[4 * nblk + 2] = slots[i];
        blk[4 * nblk + 3] = b0;
      }
    }
    m->seq_blk[bs] = nblk;
  }

  // participating devices (SPMD: only this process's; the rest is bookkeeping)
  std::vector<int> devs{m->home};
  for (auto& L : m->layers) {
    for (auto& c : L.reps) devs.push_back(c.dev);
    devs.push_back(kv_device(L));
    for (auto& mc : L.mod)
      if (mc.dev >= 0) devs.push_back(mc.dev);
  }
  std::sort(devs.begin(), devs.end());
  devs.erase(std::unique(devs.begin(), devs.end()), devs.end());
  devs.erase(std::remove_if(devs.begin(), devs.end(), [&](int dv) { return !is_local(m, dv); }), devs.end());
  const bool home_local = is_local(m, m->home);
  // the device whose compute stream times the pass and roots the metadata upload
  int tdev = m->home;
  if (!home_local) {
    tdev = -1;
    for (const DeviceCtx& dc : m->rt->devs)
      if (dc.local) {
        tdev = dc.id;
        break;
      }
    if (tdev < 0) return fail(CB_ESTATE, "no local device");
    if (std::find(devs.begin(), devs.end(), tdev) == devs.end()) devs.insert(devs.begin(), tdev);
  }
  DeviceCtx& hc = devctx(m, tdev);
  CB_TRY(ensure_ws(m, tdev));
  if (m->rt->spmd && !m->norm_ready) CB_TRY(build_norm_table(m, tdev));
  CB_TRY(use(hc));
  CB_CUDA(cudaEventRecord(hc.t0, hc.compute));
  const size_t meta_bytes = (size_t(blk_off) + 4 * size_t(nblk)) * 4;  // exactly what this pass needs
  for (int dv : devs) {
    CB_TRY(ensure_ws(m, dv));
    DeviceCtx& dc = devctx(m, dv);
    CB_TRY(depend(dc, hc));
    CB_TRY(use(dc));
    CB_CUDA(cudaMemcpyAsync(m->ws[dv].meta, meta, meta_bytes, cudaMemcpyHostToDevice, dc.compute));
  }
  // Fused RMSNorm, per layer boundary: a layer consumes fused input when every
  // segment of it has <= 256 rows (one GEMM token tile: the row-scale table),
  // neither it nor its producer carries migrated projections, and the norm
  // vector is readable where the producer runs.  Prefill keeps the separate norm
  // kernels (compute-bound GEMMs).  Decided from the placement and the batch
  // only: identical on every SPMD rank (it decides whether h' rows travel).
  const bool can_fuse = !prefill && d.d_model % 256 == 0;
  m->fin.assign(d.n_layers + 1, 0);
  for (int li = 0; li <= d.n_layers && can_fuse; ++li) {
    const int p = li < d.n_layers ? int(m->layers[li].reps.size()) : 1;
    const int max_share = (bs + p - 1) / p;  // decode: one row per sequence
    bool ok = max_share <= 256;
    if (li < d.n_layers && m->layers[li].proj_ov) ok = false;
    if (li > 0 && m->layers[li - 1].proj_ov) ok = false;
    // the producers (previous layer's copies, or the embedding on the home device) read the norm vector
    if (ok && li == 0) ok = !is_local(m, m->home) || norm_gamma_for(m, 0, m->home);
    if (ok && li > 0)
      for (const LayerCopy& c : m->layers[li - 1].reps)
        if (is_local(m, c.dev) && !norm_gamma_for(m, li, c.dev)) ok = false;
    m->fin[li] = ok;
  }
  Workspace& hw = m->ws[m->home];
  if (home_local) {
    CB_TRY(use(devctx(m, m->home)));
    ProfScope ps(m, m->home, CB_KCLASS_ELEMWISE, hc.compute, double(T) * d.d_model * 6);
    if (m->fin[0])
      CB_CUDA(cb::embed_norm_launch(m->embed, hw.meta, hw.x, norm_gamma_for(m, 0, m->home), hw.h, hw.ssq, T,
                                    d.d_model, 0, hc.compute));
    else
      CB_CUDA(cb::embed_launch(m->embed, hw.meta, hw.x, T, d.d_model, 0, hc.compute));
  }

  std::vector<Seg> layout{{m->home, 0, 0, T, 0, bs}};
  m->last_routing.assign(d.n_layers, {});
  for (int li = 0; li < d.n_layers; ++li) {
    LayerState& L = m->layers[li];
    const int p = int(L.reps.size());
    const std::vector<int> shares = split_batch_vec(g_bs, p);
    std::vector<Seg> segs;
    int g0 = 0;  // replica j's sequences: [g0, g0 + shares[j]) of the whole step
    for (int j = 0; j < p; ++j) {
      m->last_routing[li].push_back({L.reps[j].dev, g0, shares[j]});
      const int s0 = std::max(g0, g_off) - g_off, s1 = std::min(g0 + shares[j], g_off + bs) - g_off;
      if (s1 > s0) segs.push_back({L.reps[j].dev, j, seq_row[s0], seq_row[s1], s0, s1});
      g0 += shares[j];
    }
    CB_TRY(reshard(m, layout, segs, m->fin[li]));
    {
      XGroup grp(m, 0);
      for (const Seg& s : segs) CB_TRY(kv_follow(m, L, s, seq_slot));
      CB_TRY(grp.close());
    }
    for (const Seg& s : segs)
      if (is_local(m, s.dev))
        CB_TRY(run_layer_segment(m, L, s, seq_slot, row_pos, m->fin[li],
                                 m->fin[li + 1] ? norm_gamma_for(m, li + 1, s.dev) : nullptr));
    layout = segs;
  }
  std::vector<Seg> home_layout{{m->home, 0, 0, T, 0, bs}};
  CB_TRY(reshard(m, layout, home_layout, m->fin[d.n_layers]));
  // every device's trailing work joins the timing stream
  for (int dv : devs) CB_TRY(depend(hc, devctx(m, dv)));
  CB_TRY(use(hc));
  if (home_local) {
    if (!m->fin[d.n_layers]) {  // fused: the last layer's down projection already wrote h' for the final norm
      ProfScope ps(m, m->home, CB_KCLASS_ELEMWISE, hc.compute, double(T) * d.d_model * 6);
      CB_CUDA(cb::rmsnorm_launch(hw.x, m->final_norm, hw.h, T, d.d_model, d.norm_eps, 0, hc.compute));
    }
    const OpMap* xm = hw.map_h;
    if (prefill) {
      ProfScope ps(m, m->home, CB_KCLASS_ELEMWISE, hc.compute, double(bs) * d.d_model * 4);
      CB_CUDA(cb::gather_rows_launch(hw.h, hw.meta + 3 * T, hw.hl, bs, d.d_model, hc.compute));
      xm = hw.map_hl;
    }
    NormIO head_norm;
    head_norm.consume = m->fin[d.n_layers];
    CB_TRY(gemm(m, m->home, m->m_head, xm, d.vocab, d.d_model, bs, 0, cb::EPI_F32, hw.logits, d.vocab, head_norm));
    {
      ProfScope ps(m, m->home, CB_KCLASS_ELEMWISE, hc.compute, double(bs) * d.vocab * 4);
      CB_CUDA(cb::argmax_launch(hw.logits, hw.next, bs, d.vocab, hc.compute));
    }
  }
  CB_CUDA(cudaEventRecord(hc.t1, hc.compute));
  g_last_enqueue_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - enq0).count();
  if (home_local) {
    CB_CUDA(cudaMemcpyAsync(m->pin_next, hw.next, size_t(bs) * 4, cudaMemcpyDeviceToHost, hc.compute));
    if (logits_out)
      CB_CUDA(cudaMemcpyAsync(logits_out, hw.logits, size_t(bs) * d.vocab * 4, cudaMemcpyDeviceToHost, hc.compute));
  }
  CB_CUDA(cudaStreamSynchronize(hc.compute));
  if (m->prof.on) prof_resolve(m);
  float ms = 0.f;
  CB_CUDA(cudaEventElapsedTime(&ms, hc.t0, hc.t1));
  if (ms_out) *ms_out += ms;
  if (home_local)
    std::memcpy(next_out, m->pin_next, size_t(bs) * 4);
  else
    std::fill(next_out, next_out + bs, -1);  // the tokens are sampled on the home device's rank
  for (int i = 0; i < bs; ++i) m->slot_len[slots[i]] = prefill ? lens[i] : m->slot_len[slots[i]] + 1;
  return CB_OK;
}

int layer_offsets(cb_model* m) {
  const cb_model_desc& d = m->d;
  const size_t dm = d.d_model;
  m->off_qkv = 0;
  m->off_o = m->off_qkv + size_t(m->qkv_n) * dm * 2;
  m->off_gu = m->off_o + dm * size_t(m->q_n) * 2;
  m->off_d = m->off_gu + 2 * size_t(d.d_ff) * dm * 2;
  m->off_an = m->off_d + dm * size_t(d.d_ff) * 2;
  m->off_fn = m->off_an + dm * 2;
  m->layer_bytes = m->off_fn + dm * 2;
  return CB_OK;
}

// host-side validation shared by the weight loaders
int begin_layer_load(cb_model* m, int layer, int dev, LayerCopy& c) {
  CB_TRY(check_layer(m, layer));
  CB_TRY(check_dev(m, dev));
  LayerState& L = m->layers[layer - 1];
  if (!L.reps.empty()) return fail(CB_EINVAL, "layer " + std::to_string(layer) + " already loaded");
  c.dev = dev;
  if (!is_local(m, dev)) return CB_OK;  // SPMD: another rank holds the bytes
  CB_TRY(dev_alloc(devctx(m, dev), (void**)&c.block, m->layer_bytes, nullptr, MEM_WEIGHTS));
  return CB_OK;
}

int finish_layer_load(cb_model* m, int layer, LayerCopy& c) {
  LayerState& L = m->layers[layer - 1];
  if (c.block) CB_TRY(make_layer_maps(m, c));
  L.reps.push_back(c);
  m->norm_ready = false;
  L.owner.assign(m->d.max_slots, -1);
  CB_TRY(ensure_ws(m, c.dev));  // (the KV block is created at its first use, sized for the placement then)
  return CB_OK;
}

void sync_all(cb_model* m) {
  for (auto& dc : m->rt->devs) {
    if (!dc.local) continue;
    cudaSetDevice(dc.ordinal);
    cudaStreamSynchronize(dc.compute);
    cudaStreamSynchronize(dc.copy);
    cudaStreamSynchronize(dc.copy2);
  }
}
void sync_all_devices(cb_model* m) { sync_all(m); }

// ---- transfer engine of the scaling ops (NVLink 5 / NVSwitch between GPUs).
// copy_mode 1 (default): the transfer is cut into copy_chunk pieces that
// alternate between the destination's two copy lanes, so two copy engines move
// it; 0: one cudaMemcpyPeerAsync; 2: an SM kernel on the SOURCE GPU pushes
// 16-byte stores into the destination (NVLink writes need no round trip).
// Everything ends ordered on the destination's main copy stream.
int transfer(cb_model* m, int dst_dev, void* dst, int src_dev, const void* src, size_t bytes) {
  DeviceCtx& dc = devctx(m, dst_dev);
  DeviceCtx& sc = devctx(m, src_dev);
  const cb_runtime& rt = *m->rt;
  if (crosses(m, src_dev, dst_dev)) {
    // between processes: the source's copy lane (after its compute stream:
    // the block may be a layer the source still serves) sends, the
    // destination's copy lane receives (NCCL over NVLink via the host transport)
    if (sc.local) CB_TRY(join(sc, sc.copy, sc, sc.compute));
    return xmove(m, 1, src_dev, src, sc.local ? sc.copy : nullptr, dst_dev, dst, dc.local ? dc.copy : nullptr, bytes);
  }
  if (rt.copy_mode == 2 && bytes % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(src) % 16 == 0) {
    CB_TRY(join(sc, sc.copy, dc, dc.copy));
    CB_TRY(use(sc));
    CB_CUDA(cb::copy_bulk_launch(dst, src, bytes, sc.num_sms, sc.copy));
    return join(dc, dc.copy, sc, sc.copy);
  }
  CB_TRY(use(dc));
  const size_t chunk = std::max<size_t>(rt.copy_chunk, 1 << 20);
  if (rt.copy_mode == 0 || bytes <= chunk) {
    CB_CUDA(cudaMemcpyPeerAsync(dst, dc.ordinal, src, sc.ordinal, bytes, dc.copy));
    return CB_OK;
  }
  CB_TRY(join(dc, dc.copy2, dc, dc.copy));
  CB_TRY(use(dc));
  int lane = 0;
  for (size_t off = 0; off < bytes; off += chunk, lane ^= 1) {
    const size_t n = std::min(chunk, bytes - off);
    CB_CUDA(cudaMemcpyPeerAsync(static_cast<uint8_t*>(dst) + off, dc.ordinal, static_cast<const uint8_t*>(src) + off,
                                sc.ordinal, n, lane ? dc.copy2 : dc.copy));
  }
  return join(dc, dc.copy, dc, dc.copy2);
}

// ---- asynchronous scaling ops (A17) ----------------------------------------
// Which uncommitted ops may share a layer: a scale-up decision fans a layer out
// to many devices (replications to distinct devices), a compute-bound
// scale-down moves several projections of one layer (distinct, non-conflicting
// modules) and maybe its KV; a layer migration or an eviction stands alone.
int check_idle(const LayerState& L, int layer, int kind, int arg = -1) {
  auto attn_part = [](int mk) { return mk <= CB_ATTN_PROJ_O; };
  bool clash = false;
  for (const auto& pk : L.pend) {
    const int k = pk.first, a = pk.second;
    if (kind == OPK_MIGRATE || kind == OPK_EVICT || k == OPK_MIGRATE || k == OPK_EVICT) clash = true;
    else if (kind == OPK_REPLICATE) clash |= k != OPK_REPLICATE || a == arg;
    else if (k == OPK_REPLICATE) clash = true;
    else if (kind == OPK_KV) clash |= k == OPK_KV;
    else if (kind == OPK_PROJ && k == OPK_PROJ)
      clash |= a == arg || (arg == CB_SELF_ATTENTION && attn_part(a)) || (a == CB_SELF_ATTENTION && attn_part(arg));
  }
  if (clash)
    return fail(CB_ESTATE, "layer " + std::to_string(layer) + " has an uncommitted scaling op in the way");
  return CB_OK;
}

PendingOp new_op(cb_model* m, int kind, int layer, int dst, int copy_dev) {
  PendingOp op;
  op.kind = kind;
  op.layer = layer;
  op.dst = dst;
  op.copy_dev = copy_dev;
  op.snap_len.assign(m->d.max_slots, -1);
  op.snap_epoch.assign(m->d.max_slots, 0);
  return op;
}

// The local device whose copy stream carries this rank's part of an op's
// transfer (its e0 / e1 events): the destination, else (SPMD) the source.
int op_event_dev(cb_model* m, const PendingOp& op) {
  if (op.copy_dev >= 0 && is_local(m, op.copy_dev)) return op.copy_dev;
  if (op.src_dev >= 0 && is_local(m, op.src_dev)) return op.src_dev;
  if (op.kv_from >= 0 && is_local(m, op.kv_from)) return op.kv_from;
  return -1;
}

// open the transfer: ordered after every compute stream's work so far (the KV
// prefixes it may read were written by earlier steps)
int op_open(cb_model* m, PendingOp& op) {
  op.ev_dev = op_event_dev(m, op);
  if (op.ev_dev < 0) return CB_OK;  // SPMD: no part of this op runs on this rank
  DeviceCtx& dc = devctx(m, op.ev_dev);
  for (auto& o : m->rt->devs) CB_TRY(join(dc, dc.copy, o, o.compute));
  CB_TRY(use(dc));
  CB_CUDA(cudaEventCreate(&op.e0));
  CB_CUDA(cudaEventCreate(&op.e1));
  CB_CUDA(cudaEventRecord(op.e0, dc.copy));
  return CB_OK;
}

// register the op: id, layer lock, reservation count (its transfer starts now
// or, SPMD, at cb_op_start once every rank has reserved)
int op_register(cb_model* m, PendingOp& op, int64_t* id_out) {
  op.id = m->next_op++;
  LayerState& L = m->layers[op.layer - 1];
  L.pend.push_back({op.kind, op.kind == OPK_PROJ ? op.mod_kind : op.dst});
  if (op.dst >= 0) devctx(m, op.dst).reserved += op.reserved;
  m->ops[op.id] = op;
  if (id_out) *id_out = op.id;
  return CB_OK;
}

// Pre-copy of the live KV prefixes held by op.kv_from into op.kv_to's block,
// on the destination's copy stream.  KV is append-only: positions below a
// slot's length never change while its occupant lives, so the prefix stays
// valid and the commit copies only what was appended since (a slot released
// and refilled meanwhile has a new epoch and is copied whole).  Only used when
// nothing else writes kv_to's block for this layer while the op is pending.
int kv_ipc_pull(cb_model* m, PendingOp& op, LayerState& L, bool catchup, cudaStream_t dst_st, uint64_t* bytes);

int op_precopy_kv(cb_model* m, PendingOp& op, LayerState& L) {
  const bool lt = is_local(m, op.kv_to), lf = is_local(m, op.kv_from);
  if (crosses(m, op.kv_from, op.kv_to)) {  // between processes: a CUDA IPC pull (every rank keeps the snapshot)
    for (int slot = 0; slot < m->d.max_slots; ++slot) {
      if (L.owner[slot] != op.kv_from || m->slot_len[slot] <= 0) continue;
      op.snap_len[slot] = m->slot_len[slot];
      op.snap_epoch[slot] = int(m->slot_epoch[slot]);
    }
    return kv_ipc_pull(m, op, L, false, lt ? devctx(m, op.kv_to).copy : nullptr, &op.kv_bytes);
  }
  cudaStream_t dst_st = lt ? devctx(m, op.kv_to).copy : nullptr;
  cudaStream_t src_st = nullptr;
  if (crosses(m, op.kv_from, op.kv_to) && lf) {  // the sender orders its copy lane after its compute stream
    DeviceCtx& fc = devctx(m, op.kv_from);
    CB_TRY(join(fc, fc.copy, fc, fc.compute));
    src_st = fc.copy;
  }
  XGroup grp(m, 1);
  for (int slot = 0; slot < m->d.max_slots; ++slot) {
    if (L.owner[slot] != op.kv_from || m->slot_len[slot] <= 0) continue;
    CB_TRY(kv_copy(m, L, slot, op.kv_from, op.kv_to, 0, m->slot_len[slot], dst_st, &op.kv_bytes, 1, src_st));
    op.snap_len[slot] = m->slot_len[slot];
    op.snap_epoch[slot] = int(m->slot_epoch[slot]);
  }
  return grp.close();
}

// ---- between processes (SPMD): a layer block moves as a P2P copy-engine pull
// over NVLink, not through the collective library.  The source's rank exports
// the block (CUDA IPC handle, after its compute stream drained: every write into
// the block has landed) and sends the handle over the host transport; the
// destination's rank maps it and pulls it in chunks alternating over its two
// copy lanes.  Weight blocks are static while they serve, and the SPMD commit
// is preceded by a barrier of every rank's part, so the source block outlives
// the pull.  (KV pre-copies / catch-ups and per-step rows stay on the transport.)
struct IpcMsg {
  cudaIpcMemHandle_t h;
  uint64_t offset;
};

int host_msg(cb_model* m, bool send, int peer_rank, void* buf, size_t n) {
  cb_runtime* rt = m->rt;
  if (rt->xfer(rt->xfer_ctx, 2, send ? 4 : 5, peer_rank, buf, n, nullptr) != 0)
    return fail(CB_ECOMM, std::string("transport host message ") + (send ? "to" : "from") + " rank " +
                              std::to_string(peer_rank) + " failed");
  return CB_OK;
}

int ipc_pull(cb_model* m, PendingOp& op) {
  DeviceCtx& sc = devctx(m, op.src_dev);
  DeviceCtx& dc = devctx(m, op.dst);
  if (sc.local) {
    auto it = sc.allocs.upper_bound(const_cast<void*>(op.xsrc));
    if (it == sc.allocs.begin()) return fail(CB_ESTATE, "IPC source is not a tracked allocation");
    --it;
    if (!sc.ipc_allocs.count(it->first)) return fail(CB_ESTATE, "IPC source block is not exportable");
    CB_TRY(use(sc));
    CB_CUDA(cudaStreamSynchronize(sc.compute));
    IpcMsg msg{};
    CB_CUDA(cudaIpcGetMemHandle(&msg.h, it->first));
    msg.offset = uint64_t(static_cast<const uint8_t*>(op.xsrc) - static_cast<const uint8_t*>(it->first));
    CB_TRY(host_msg(m, true, dc.rank, &msg, sizeof msg));
  }
  if (dc.local) {
    IpcMsg msg{};
    CB_TRY(host_msg(m, false, sc.rank, &msg, sizeof msg));
    CB_TRY(use(dc));
    CB_CUDA(cudaIpcOpenMemHandle(&op.ipc_base, msg.h, cudaIpcMemLazyEnablePeerAccess));
    const uint8_t* src = static_cast<const uint8_t*>(op.ipc_base) + msg.offset;
    uint8_t* dst = static_cast<uint8_t*>(op.xdst);
    const size_t chunk = std::max<size_t>(m->rt->copy_chunk, 1 << 20);
    if (op.e0 && op.ev_dev == op.dst) CB_CUDA(cudaEventRecord(op.e0, dc.copy));  // time the pull, not the handshake
    CB_TRY(join(dc, dc.copy2, dc, dc.copy));
    int lane = 0;
    for (size_t off = 0; off < op.xbytes; off += chunk, lane ^= 1)
      CB_CUDA(cudaMemcpyAsync(dst + off, src + off, std::min(chunk, op.xbytes - off), cudaMemcpyDeviceToDevice,
                              lane ? dc.copy2 : dc.copy));
    CB_TRY(join(dc, dc.copy, dc, dc.copy2));
  }
  return CB_OK;
}

void ipc_close(PendingOp& op) {
  if (!op.ipc_base) return;
  if (op.e1) cudaEventSynchronize(op.e1);
  cudaIpcCloseMemHandle(op.ipc_base);
  op.ipc_base = nullptr;
}

// KV of a scaling op between processes (pre-copy at the start, catch-up at the
// commit): the source's rank drains its compute stream and sends its KV
// block's IPC handle with its slot table; the destination's rank maps the
// block, pulls each slot kv_from holds -- positions [0, len) for the pre-copy,
// [snapshot, len) for the catch-up -- with its copy engine on dst_st, waits,
// unmaps and acknowledges.  The source waits for the acknowledgement: its block
// may be regrown or freed right after.
int kv_ipc_pull(cb_model* m, PendingOp& op, LayerState& L, bool catchup, cudaStream_t dst_st, uint64_t* bytes) {
  DeviceCtx& fc = devctx(m, op.kv_from);
  DeviceCtx& tc = devctx(m, op.kv_to);
  const int ms = m->d.max_slots;
  // message: [has_block][IPC handle][slot -> index table]
  std::vector<uint8_t> msg(8 + sizeof(cudaIpcMemHandle_t) + size_t(ms) * 4, 0);
  int32_t* has = reinterpret_cast<int32_t*>(msg.data());
  cudaIpcMemHandle_t* hdl = reinterpret_cast<cudaIpcMemHandle_t*>(msg.data() + 8);
  int32_t* map = reinterpret_cast<int32_t*>(msg.data() + 8 + sizeof(cudaIpcMemHandle_t));
  uint8_t ack = 1;
  if (fc.local) {
    auto it = L.kv.find(op.kv_from);
    if (it != L.kv.end()) {  // (no block: the layer never held KV there)
      KvBlock& b = it->second;
      if (!fc.ipc_allocs.count(b.p)) return fail(CB_ESTATE, "KV block is not exportable");
      CB_TRY(use(fc));
      CB_CUDA(cudaStreamSynchronize(fc.compute));
      CB_CUDA(cudaIpcGetMemHandle(hdl, b.p));
      *has = 1;
      for (int slot = 0; slot < ms; ++slot) map[slot] = kv_index(b, slot);
    }
    CB_TRY(host_msg(m, true, tc.rank, msg.data(), msg.size()));
    CB_TRY(host_msg(m, false, tc.rank, &ack, 1));
  }
  if (tc.local) {
    CB_TRY(host_msg(m, false, fc.rank, msg.data(), msg.size()));
    if (!*has) return host_msg(m, true, fc.rank, &ack, 1);
    CB_TRY(use(tc));
    void* base = nullptr;
    CB_CUDA(cudaIpcOpenMemHandle(&base, *hdl, cudaIpcMemLazyEnablePeerAccess));
    const size_t tb = kv_token_bytes(m);
    for (int slot = 0; slot < ms; ++slot) {
      if (L.owner[slot] != op.kv_from) continue;
      const int len = m->slot_len[slot];
      int p0 = 0;
      if (catchup) {
        const bool fresh = op.snap_len[slot] >= 0 && op.snap_epoch[slot] == int(m->slot_epoch[slot]);
        p0 = fresh ? std::min(op.snap_len[slot], len) : 0;
      }
      if (len <= p0 || map[slot] < 0) continue;
      CB_TRY(kv_assign(m, L, op.kv_to, slot));
      uint16_t* dst = kv_ptr(m, L, op.kv_to, slot, p0);
      const uint16_t* src = static_cast<const uint16_t*>(base) + kv_slot_offset(m, map[slot]) + size_t(p0) * tb / 2;
      CB_CUDA(cudaMemcpyAsync(dst, src, size_t(len - p0) * tb, cudaMemcpyDeviceToDevice, dst_st));
      if (bytes) *bytes += size_t(len - p0) * tb;
    }
    CB_CUDA(cudaStreamSynchronize(dst_st));
    CB_CUDA(cudaIpcCloseMemHandle(base));
    CB_TRY(host_msg(m, true, fc.rank, &ack, 1));
  } else if (bytes) {  // (the byte count is bookkeeping on every rank)
    for (int slot = 0; slot < ms; ++slot) {
      if (L.owner[slot] != op.kv_from) continue;
      const int len = m->slot_len[slot];
      int p0 = 0;
      if (catchup) {
        const bool fresh = op.snap_len[slot] >= 0 && op.snap_epoch[slot] == int(m->slot_epoch[slot]);
        p0 = fresh ? std::min(op.snap_len[slot], len) : 0;
      }
      if (len > p0) *bytes += size_t(len - p0) * kv_token_bytes(m);
    }
  }
  return CB_OK;
}

// Enqueue an op's data movement: the weight transfer (+ KV pre-copy) on the
// copy streams; e1 marks this rank's part done.
int op_run(cb_model* m, PendingOp& op) {
  CB_TRY(op_open(m, op));
  if (op.xbytes) {
    if (op.strided_gu) {  // every other row of the interleaved gate/up block (single process)
      DeviceCtx& dc = devctx(m, op.dst);
      const size_t row = size_t(m->d.d_model) * 2;
      CB_TRY(use(dc));
      CB_CUDA(cudaMemcpy2DAsync(op.xdst, row, op.xsrc, 2 * row, row, m->d.d_ff, cudaMemcpyDefault, dc.copy));
    } else if (crosses(m, op.src_dev, op.dst)) {
      CB_TRY(ipc_pull(m, op));
    } else {
      CB_TRY(transfer(m, op.dst, op.xdst, op.src_dev, op.xsrc, op.xbytes));
    }
  }
  if (op.precopy) CB_TRY(op_precopy_kv(m, op, m->layers[op.layer - 1]));
  if (op.ev_dev >= 0) {
    DeviceCtx& dc = devctx(m, op.ev_dev);
    CB_TRY(use(dc));
    CB_CUDA(cudaEventRecord(op.e1, dc.copy));
  }
  op.started = true;
  return CB_OK;
}

// single process: the transfer starts at issue; SPMD: at cb_op_start
int op_issue(cb_model* m, PendingOp& op, int64_t* id_out) {
  if (!m->rt->spmd) CB_TRY(op_run(m, op));
  return op_register(m, op, id_out);
}

// At the commit: the rest of every slot op.kv_from still holds moves to
// op.kv_to on kv_to's compute stream (stream-ordered before the next step).
int op_catchup_kv(cb_model* m, PendingOp& op, LayerState& L) {
  const bool lt = is_local(m, op.kv_to), lf = is_local(m, op.kv_from);
  DeviceCtx& tc = devctx(m, op.kv_to);
  DeviceCtx& fc = devctx(m, op.kv_from);
  CB_TRY(join(tc, tc.compute, fc, fc.compute));
  if (lt) {
    CB_TRY(use(tc));
    CB_CUDA(cudaEventCreate(&op.c0));
    CB_CUDA(cudaEventCreate(&op.c1));
    CB_CUDA(cudaEventRecord(op.c0, tc.compute));
  }
  if (lt) {
    auto it = L.kv.find(op.kv_to);
    if (it != L.kv.end() && it->second.table) {
      int need = 0;
      for (int slot = 0; slot < m->d.max_slots; ++slot)
        need += L.owner[slot] == op.kv_from && it->second.map_h[slot] < 0;
      CB_TRY(kv_reserve(m, L, op.kv_to, need));
    }
  }
  const bool ipc = crosses(m, op.kv_from, op.kv_to);
  if (ipc) CB_TRY(kv_ipc_pull(m, op, L, true, lt ? tc.compute : nullptr, &op.catchup_bytes));
  XGroup grp(m, 0);
  for (int slot = 0; slot < m->d.max_slots; ++slot) {
    if (L.owner[slot] != op.kv_from) continue;
    const int len = m->slot_len[slot];
    const bool fresh = op.snap_len[slot] >= 0 && op.snap_epoch[slot] == int(m->slot_epoch[slot]);
    const int have = fresh ? std::min(op.snap_len[slot], len) : 0;
    if (!ipc)
      CB_TRY(kv_copy(m, L, slot, op.kv_from, op.kv_to, have, len, lt ? tc.compute : nullptr, &op.catchup_bytes, 0,
                     lf ? fc.compute : nullptr));
    CB_TRY(kv_assign(m, L, op.kv_to, slot));
    kv_unassign(L, op.kv_from, slot);
    L.owner[slot] = op.kv_to;
  }
  CB_TRY(grp.close());
  if (lt) CB_CUDA(cudaEventRecord(op.c1, tc.compute));
  return CB_OK;
}

void op_unlock(LayerState& L, const PendingOp& op) {
  const std::pair<int, int> key{op.kind, op.kind == OPK_PROJ ? op.mod_kind : op.dst};
  auto it = std::find(L.pend.begin(), L.pend.end(), key);
  if (it != L.pend.end()) L.pend.erase(it);
}

// release what an op reserved but never committed
void op_release_reservation(cb_model* m, PendingOp& op) {
  LayerState& L = m->layers[op.layer - 1];
  if (op.copy.block) dev_free(m, op.copy.dev, op.copy.block);
  if (op.mod.buf) dev_free(m, op.mod.dev, op.mod.buf);
  op.copy.block = nullptr;
  op.mod.buf = nullptr;
  if (op.kv_new && op.kv_to >= 0) {
    auto it = L.kv.find(op.kv_to);
    if (it != L.kv.end()) {
      free_kv_block(m, L, op.kv_to, it->second);
      L.kv.erase(it);
    }
  }
}

// reserve a layer block on dst (this rank's device only; others record the copy)
int reserve_block(cb_model* m, PendingOp& op, int dst, uint64_t* shortfall) {
  op.copy.dev = dst;
  if (!is_local(m, dst)) return CB_OK;
  DeviceCtx& dc = devctx(m, dst);
  return dev_alloc(dc, (void**)&op.copy.block, m->layer_bytes, shortfall, MEM_WEIGHTS, dc.copy);
}

// ReplicateLayer (ops.py:199-211): reserve + copy the layer block original -> dst.
int issue_replicate(cb_model* m, int layer, int dst, int64_t* id, uint64_t* shortfall) {
  CB_TRY(check_layer(m, layer));
  CB_TRY(check_dev(m, dst));
  LayerState& L = m->layers[layer - 1];
  if (L.reps.empty()) return fail(CB_ESTATE, "layer not loaded");
  CB_TRY(check_idle(L, layer, OPK_REPLICATE, dst));
  for (auto& c : L.reps)
    if (c.dev == dst)
      return fail(CB_EINVAL, "layer " + std::to_string(layer) + " already has a copy on device " + std::to_string(dst));
  if (L.kv_override >= 0 || L.proj_ov) return fail(CB_EINVAL, "layer carries overrides and cannot be replicated");
  PendingOp op = new_op(m, OPK_REPLICATE, layer, dst, dst);
  int r = reserve_block(m, op, dst, shortfall);
  if (r == CB_OK) {
    // the replica's KV block holds its split_batch share: ceil(max_slots / p) slots
    int p = int(L.reps.size()) + 1;
    for (const auto& pk : L.pend) p += pk.first == OPK_REPLICATE ? 1 : 0;
    const int cap = (m->d.max_slots + p - 1) / p;
    r = ensure_kv(m, L, dst, shortfall, is_local(m, dst) ? devctx(m, dst).copy : nullptr, &op.kv_new, cap);
    op.kv_to = dst;  // (no KV moves at issue: rows move with split_batch once serving)
  }
  if (r == CB_OK) r = ensure_ws(m, dst);
  if (r != CB_OK) {
    const std::string err = g_err;
    op_release_reservation(m, op);
    return fail(r, err);
  }
  op.reserved = m->layer_bytes + (op.kv_new ? kv_block_bytes_of(m, L.kv.at(dst)) : 0);
  op.src_dev = L.reps[0].dev;
  op.xsrc = L.reps[0].block;
  op.xdst = op.copy.block;
  op.xbytes = m->layer_bytes;
  op.weight_bytes = m->layer_bytes;
  return op_issue(m, op, id);
}

// MigrateLayer (ops.py:213-228): reserve + copy the original to dst; with_kv
// pre-copies the KV the layer's KV device holds (replica-held rows stay).
int issue_migrate(cb_model* m, int layer, int dst, int with_kv, int64_t* id, uint64_t* shortfall) {
  CB_TRY(check_layer(m, layer));
  CB_TRY(check_dev(m, dst));
  LayerState& L = m->layers[layer - 1];
  if (L.reps.empty()) return fail(CB_ESTATE, "layer not loaded");
  CB_TRY(check_idle(L, layer, OPK_MIGRATE));
  const int src = L.reps[0].dev;
  if (dst == src) return fail(CB_EINVAL, "layer original already on device " + std::to_string(dst));
  for (auto& c : L.reps)
    if (c.dev == dst) return fail(CB_EINVAL, "layer already has a copy on device " + std::to_string(dst));
  if (!with_kv && L.reps.size() > 1) return fail(CB_EINVAL, "cannot detach KV from a replicated layer");
  if (!with_kv && m->rt->spmd && devctx(m, src).rank != devctx(m, dst).rank)
    return fail(CB_ENOTSUP, "SPMD runtime: a layer's KV moves with it between processes (with_kv=1)");
  PendingOp op = new_op(m, OPK_MIGRATE, layer, dst, dst);
  op.with_kv = with_kv;
  op.kv_from = kv_device(L);
  int r = reserve_block(m, op, dst, shortfall);
  if (r == CB_OK && with_kv && op.kv_from != dst) {
    op.kv_to = dst;
    r = ensure_kv(m, L, dst, shortfall, is_local(m, dst) ? devctx(m, dst).copy : nullptr, &op.kv_new);
  }
  if (r == CB_OK) r = ensure_ws(m, dst);
  if (r != CB_OK) {
    const std::string err = g_err;
    op_release_reservation(m, op);
    return fail(r, err);
  }
  op.reserved = m->layer_bytes + (op.kv_new ? m->kv_block_bytes : 0);
  op.src_dev = src;
  op.xsrc = L.reps[0].block;
  op.xdst = op.copy.block;
  op.xbytes = m->layer_bytes;
  op.weight_bytes = m->layer_bytes;
  op.precopy = op.kv_to >= 0;  // dst serves nothing of this layer until the commit
  return op_issue(m, op, id);
}

// MigrateSubModule of a projection / SELF_ATTENTION (ops.py:230-251): reserve +
// copy the module's weights (canonical [out, in] layout) to dst; after the
// commit the layer runs that projection there with activation hops
// (run_layer_overridden).  The layer block keeps its bytes (one allocation);
// the registry does the reference's memory accounting (domain.py:481-535).
int issue_projection(cb_model* m, int layer, int kind, int dst, int64_t* id, uint64_t* shortfall) {
  LayerState& L = m->layers[layer - 1];
  if (L.reps.empty()) return fail(CB_ESTATE, "layer not loaded");
  if (m->rt->spmd) return fail(CB_ENOTSUP, "SPMD runtime: sub-module overrides need the single-process runtime");
  CB_TRY(check_idle(L, layer, OPK_PROJ, kind));
  if (L.reps.size() > 1) return fail(CB_EINVAL, "layer is replicated and cannot carry overrides");
  const bool attn_part = kind <= CB_ATTN_PROJ_O;
  if ((kind == CB_SELF_ATTENTION && (L.mod[0].dev >= 0 || L.mod[1].dev >= 0 || L.mod[2].dev >= 0 ||
                                     L.mod[3].dev >= 0)) ||
      (attn_part && L.mod[CB_SELF_ATTENTION].dev >= 0))
    return fail(CB_EINVAL, "projection override conflicts with a self_attention override (domain.py:298-303)");
  const uint64_t bytes = cb_module_bytes(m, kind);
  DeviceCtx& dc = devctx(m, dst);
  PendingOp op = new_op(m, OPK_PROJ, layer, dst, dst);
  op.mod_kind = kind;
  op.mod.dev = dst;
  int r = dev_alloc(dc, (void**)&op.mod.buf, bytes, shortfall, MEM_WEIGHTS, dc.copy);
  if (r == CB_OK) r = ensure_ws(m, dst);
  if (r != CB_OK) {
    const std::string err = g_err;
    op_release_reservation(m, op);
    return fail(r, err);
  }
  op.reserved = bytes;
  const ModCopy& mc = L.mod[kind];
  if (mc.dev >= 0) {  // moved once already: copy from the current override
    op.src_dev = mc.dev;
    op.xsrc = mc.buf;
  } else {
    op.src_dev = L.reps[0].dev;
    op.xsrc = L.reps[0].block + block_offset(m, kind);
    op.strided_gu = kind == CB_FFN_PROJ_GATE || kind == CB_FFN_PROJ_UP;
  }
  op.xdst = op.mod.buf;
  op.xbytes = bytes;
  op.weight_bytes = bytes;
  return op_issue(m, op, id);
}

// MigrateSubModule(KV_CACHE) (ops.py:230-251): the layer's KV moves to dst
// (pre-copied now, caught up at the commit); attention then runs there.
int issue_kv(cb_model* m, int layer, int dst, int64_t* id, uint64_t* shortfall) {
  LayerState& L = m->layers[layer - 1];
  if (L.reps.empty()) return fail(CB_ESTATE, "layer not loaded");
  if (m->rt->spmd) return fail(CB_ENOTSUP, "SPMD runtime: sub-module overrides need the single-process runtime");
  CB_TRY(check_idle(L, layer, OPK_KV));
  if (L.reps.size() > 1) return fail(CB_EINVAL, "layer is replicated and cannot carry overrides");
  DeviceCtx& dc = devctx(m, dst);
  PendingOp op = new_op(m, OPK_KV, layer, dst, dst);
  op.kv_from = kv_device(L);
  op.kv_to = dst;
  int r = ensure_kv(m, L, dst, shortfall, dc.copy, &op.kv_new);
  if (r == CB_OK) r = ensure_ws(m, dst);
  if (r != CB_OK) {
    const std::string err = g_err;
    op_release_reservation(m, op);
    return fail(r, err);
  }
  op.reserved = op.kv_new ? m->kv_block_bytes : 0;
  op.precopy = op.kv_from != dst;  // attention stays on kv_from until the commit
  return op_issue(m, op, id);
}

// EvictReplica (ops.py:253-258).  The original keeps serving its own rows
// while the op is pending, so the KV rows the replica holds move back at the
// commit (on the original's compute stream, before the next step).
int issue_evict(cb_model* m, int layer, int dev, int64_t* id) {
  CB_TRY(check_layer(m, layer));
  LayerState& L = m->layers[layer - 1];
  if (L.reps.empty()) return fail(CB_ESTATE, "layer not loaded");
  CB_TRY(check_idle(L, layer, OPK_EVICT));
  if (L.reps[0].dev == dev) return fail(CB_ENOREPLICA, "cannot evict the original replica");
  auto it = std::find_if(L.reps.begin() + 1, L.reps.end(), [&](const LayerCopy& c) { return c.dev == dev; });
  if (it == L.reps.end())
    return fail(CB_ENOREPLICA, "layer " + std::to_string(layer) + " has no replica on device " + std::to_string(dev));
  PendingOp op = new_op(m, OPK_EVICT, layer, -1, L.reps[0].dev);
  op.kv_from = dev;
  op.kv_to = L.reps[0].dev;
  return op_issue(m, op, id);
}

// Switch one op's placement at this step boundary.  No host synchronisation:
// every compute stream orders after the op's transfer, the KV catch-up runs on
// the new KV device's compute stream, replaced buffers are freed stream-ordered.
int op_commit(cb_model* m, PendingOp& op) {
  LayerState& L = m->layers[op.layer - 1];
  if (!op.started) return fail(CB_ESTATE, "op " + std::to_string(op.id) + " was never started (cb_op_start)");
  ipc_close(op);
  if (op.e1)
    for (auto& o : m->rt->devs) {
      if (!o.local) continue;
      CB_TRY(use(o));
      CB_CUDA(cudaStreamWaitEvent(o.compute, op.e1, 0));
    }
  switch (op.kind) {
    case OPK_REPLICATE:
      if (op.copy.block) CB_TRY(make_layer_maps(m, op.copy));
      L.reps.push_back(op.copy);
      break;
    case OPK_MIGRATE: {
      const int kv_src = op.kv_from;
      if (op.kv_to >= 0) CB_TRY(op_catchup_kv(m, op, L));
      if (op.copy.block) CB_TRY(make_layer_maps(m, op.copy));
      const LayerCopy old = L.reps[0];
      L.reps[0] = op.copy;
      dev_free(m, old.dev, old.block);
      L.kv_override = op.with_kv ? -1 : kv_src;  // without KV it stays resident where it was (domain.py:445-451)
      for (int dv : std::vector<int>{old.dev, kv_src}) drop_kv_if_unused(m, L, dv);
      break;
    }
    case OPK_PROJ: {
      const ModCopy old = L.mod[op.mod_kind];
      L.mod[op.mod_kind] = op.mod;
      if (old.dev >= 0) dev_free(m, old.dev, old.buf);
      L.proj_ov = false;
      for (const ModCopy& x : L.mod)
        if (x.dev >= 0) L.proj_ov = true;
      break;
    }
    case OPK_KV:
      if (op.kv_from != op.kv_to) CB_TRY(op_catchup_kv(m, op, L));
      L.kv_override = op.kv_to;
      drop_kv_if_unused(m, L, op.kv_from);
      break;
    case OPK_EVICT: {
      CB_TRY(op_catchup_kv(m, op, L));
      auto it = std::find_if(L.reps.begin() + 1, L.reps.end(), [&](const LayerCopy& c) { return c.dev == op.kv_from; });
      dev_free(m, it->dev, it->block);
      L.reps.erase(it);
      drop_kv_if_unused(m, L, op.kv_from);
      break;
    }
  }
  op.copy.block = nullptr;  // owned by the layer now
  op.mod.buf = nullptr;
  op_unlock(L, op);
  if (op.kind == OPK_REPLICATE) kv_shrink_empty(m, L);
  if (op.dst >= 0) devctx(m, op.dst).reserved -= op.reserved;
  op.committed = true;
  return CB_OK;
}

int op_abort(cb_model* m, PendingOp& op) {
  ipc_close(op);
  op_release_reservation(m, op);
  op_unlock(m->layers[op.layer - 1], op);
  if (op.dst >= 0) devctx(m, op.dst).reserved -= op.reserved;
  return CB_OK;
}

void op_destroy_events(PendingOp& op) {
  for (cudaEvent_t e : {op.e0, op.e1, op.c0, op.c1})
    if (e) cudaEventDestroy(e);
}

int op_stats(cb_model* m, PendingOp& op, cb_op_stats* st, bool wait) {
  if (wait) {
    if (!op.started) return fail(CB_ESTATE, "op " + std::to_string(op.id) + " was never started (cb_op_start)");
    if (op.e1) CB_CUDA(cudaEventSynchronize(op.e1));
    if (op.c1) CB_CUDA(cudaEventSynchronize(op.c1));
  }
  if (!st) return CB_OK;
  *st = cb_op_stats{};
  st->weight_bytes = op.weight_bytes;
  st->kv_bytes = op.kv_bytes + op.catchup_bytes;
  st->catchup_bytes = op.catchup_bytes;
  st->committed = op.committed ? 1 : 0;
  float ms = 0.f;
  st->done = op.started && (!op.e1 || cudaEventQuery(op.e1) == cudaSuccess) &&
             (!op.c1 || cudaEventQuery(op.c1) == cudaSuccess);
  cudaGetLastError();
  if (st->done) {
    if (op.e1) CB_CUDA(cudaEventElapsedTime(&ms, op.e0, op.e1));
    st->copy_ms = ms;
    if (op.c1) {
      float cm = 0.f;
      CB_CUDA(cudaEventElapsedTime(&cm, op.c0, op.c1));
      st->catchup_ms = cm;
    }
    st->device_ms = st->copy_ms + st->catchup_ms;
  }
  return CB_OK;
}

int kv_offload(cb_model* m, int layer, bool to_host, cb_op_stats* st) {
  LayerState& L = m->layers[layer - 1];
  if (L.reps.empty()) return fail(CB_ESTATE, "layer not loaded");
  if (m->rt->spmd) return fail(CB_ENOTSUP, "SPMD runtime: KV offload needs the single-process runtime");
  CB_TRY(check_idle(L, layer, OPK_MIGRATE));
  sync_all(m);  // Phase-3 relief (rare): a blocking move keeps the host-memory swap simple
  if (to_host && is_local(m, kv_device(L))) CB_TRY(ensure_kv(m, L, kv_device(L)));  // not used yet: offload it empty
  uint64_t moved = 0;
  float ms = 0.f;
  for (auto& kv : L.kv) {
    const int dev = kv.first;
    KvBlock& b = kv.second;
    if (b.host == to_host) continue;
    DeviceCtx& dc = devctx(m, dev);
    CB_TRY(use(dc));
    uint16_t* nb = nullptr;
    uint64_t shortfall = 0;
    int r = kv_alloc_bytes(m, dc, to_host, kv_block_bytes_of(m, b), &nb, &shortfall, nullptr);
    if (r != CB_OK) {
      if (st) st->shortfall_bytes = shortfall;
      return r;
    }
    CB_TRY(use(dc));
    CB_CUDA(cudaEventRecord(dc.t0, dc.copy));
    for (int slot = 0; slot < m->d.max_slots; ++slot) {  // live prefixes, same local indices
      if (L.owner[slot] != dev || m->slot_len[slot] <= 0 || kv_index(b, slot) < 0) continue;
      const size_t nbytes = size_t(m->slot_len[slot]) * kv_token_bytes(m);
      const size_t off = kv_slot_offset(m, kv_index(b, slot));
      CB_CUDA(cudaMemcpyAsync(nb + off, b.p + off, nbytes, cudaMemcpyDefault, dc.copy));
      moved += nbytes;
    }
    CB_CUDA(cudaEventRecord(dc.t1, dc.copy));
    CB_CUDA(cudaStreamSynchronize(dc.copy));
    float one = 0.f;
    CB_CUDA(cudaEventElapsedTime(&one, dc.t0, dc.t1));
    ms += one;
    if (b.host) {
      cudaFreeHost(b.p);
    } else {
      dev_free(m, dev, b.p);
    }
    b.p = nb;
    b.host = to_host;
  }
  if (st) {
    st->kv_bytes = moved;
    st->device_ms = ms;
  }
  return CB_OK;
}

}  // namespace

// ============================================================== C-ABI
namespace {
// Routing order of a step's sequences (SURVEY §7 hard part 1, option A: sticky
// assignment).  split_batch fixes how MANY sequences each replica of a layer
// serves (ops.py:151-158, bit-exact); which ones is the executor's choice.  In
// the first replicated layer's run, a sequence whose KV already lives on one of
// the replicas stays there while that replica's share has room (earliest in
// batch order first); the rest -- fresh prompts and the overflow of shrunken
// shares -- fill the replicas with room in replica order, in batch order.
// The step then runs on the sequences in that order (each replica's rows
// contiguous) and the outputs return in the caller's order.  Under continuous
// batching only the share changes move KV, not every shifted range boundary.
// Deterministic from the replicated owner bookkeeping: every SPMD rank derives
// the same order.
std::vector<int> routing_order(cb_model* m, int bs, const int32_t* slots) {
  std::vector<int> perm(bs);
  for (int i = 0; i < bs; ++i) perm[i] = i;
  const LayerState* L = nullptr;
  for (const auto& l : m->layers)
    if (l.reps.size() > 1) {
      L = &l;
      break;
    }
  if (!L || L->owner.empty()) return perm;
  const int p = int(L->reps.size());
  const std::vector<int> shares = split_batch_vec(bs, p);
  std::vector<std::vector<int>> groups(p);
  std::vector<int> pool;
  for (int i = 0; i < bs; ++i) {
    const int o = L->owner[slots[i]];
    int j = -1;
    for (int r = 0; r < p && o >= 0; ++r)
      if (L->reps[r].dev == o) j = r;
    if (j >= 0 && int(groups[j].size()) < shares[j]) {
      groups[j].push_back(i);
    } else {
      pool.push_back(i);
    }
  }
  size_t next = 0;
  for (int j = 0; j < p; ++j)
    while (int(groups[j].size()) < shares[j]) groups[j].push_back(pool[next++]);
  int k = 0;
  for (const auto& g : groups)
    for (int i : g) perm[k++] = i;
  return perm;
}

// cb_step on the sequences in the given order (each layer's replicas take
// contiguous split_batch ranges of it)
int step_ordered(cb_model* m, int32_t phase, int32_t bs, const int32_t* slots, const int32_t* tokens,
                 const int32_t* prompt_lens, int32_t* next_out, float* logits_out, float* ms_out) {
  if (!m) return fail(CB_EINVAL, "null model");
  if (ms_out) *ms_out = 0.f;
  if (bs == 0) return CB_OK;
  if (bs < 0 || bs > m->d.max_slots || !slots || !tokens || !next_out)
    return fail(CB_EINVAL, "bad batch arguments");
  if (phase != CB_PHASE_PREFILL && phase != CB_PHASE_DECODE) return fail(CB_EINVAL, "unknown phase");
  if (!m->head_loaded) return fail(CB_ESTATE, "embedding / lm_head not loaded");
  kv_release_pending(m);
  for (auto& L : m->layers)
    if (L.reps.empty()) return fail(CB_ESTATE, "a decoder layer is not loaded");
  std::vector<char> seen(m->d.max_slots, 0);
  for (int i = 0; i < bs; ++i) {
    if (slots[i] < 0 || slots[i] >= m->d.max_slots) return fail(CB_EINVAL, "slot out of range");
    if (seen[slots[i]]++) return fail(CB_EINVAL, "duplicate slot in batch");
    const int len = m->slot_len[slots[i]];
    if (phase == CB_PHASE_PREFILL && len != 0) return fail(CB_EINVAL, "prefill into a non-empty slot");
    if (phase == CB_PHASE_DECODE && len == 0) return fail(CB_EINVAL, "decode on an empty slot");
  }
  // token ids index the embedding table on the device: reject out-of-range ids
  // before any launch (an out-of-bounds gather would poison the context)
  auto bad_tokens = [&](long long n) {
    for (long long t = 0; t < n; ++t)
      if (tokens[t] < 0 || tokens[t] >= m->d.vocab) return true;
    return false;
  };
  if (phase == CB_PHASE_DECODE) {
    if (bad_tokens(bs)) return fail(CB_EINVAL, "token id out of range [0, vocab)");
    return step_pass(m, phase, bs, slots, tokens, nullptr, next_out, logits_out, ms_out, 0, bs);
  }
  if (!prompt_lens) return fail(CB_EINVAL, "prefill needs prompt_lens");
  {
    long long total = 0;
    for (int t = 0; t < bs; ++t) {
      if (prompt_lens[t] < 1 || prompt_lens[t] > m->d.max_ctx) return fail(CB_EINVAL, "bad prompt length");
      total += prompt_lens[t];
    }
    if (bad_tokens(total)) return fail(CB_EINVAL, "token id out of range [0, vocab)");
  }
  // prefill: group sequences so each pass fits max_tokens rows
  int i = 0, tok_off = 0;
  while (i < bs) {
    int j = i, rows = 0;
    while (j < bs && rows + prompt_lens[j] <= m->d.max_tokens) {
      if (prompt_lens[j] < 1 || prompt_lens[j] > m->d.max_ctx) return fail(CB_EINVAL, "bad prompt length");
      rows += prompt_lens[j++];
    }
    if (j == i) return fail(CB_EINVAL, "prompt longer than max_tokens");
    CB_TRY(step_pass(m, phase, j - i, slots + i, tokens + tok_off, prompt_lens + i, next_out + i,
                     logits_out ? logits_out + size_t(i) * m->d.vocab : nullptr, ms_out, i, bs));
    tok_off += rows;
    i = j;
  }
  return CB_OK;
}
}  // namespace

extern "C" {

int cb_abi_version(void) { return CB_ABI_VERSION; }
const char* cb_last_error(void) { return g_err.c_str(); }

int cb_split_batch(int32_t bs, int32_t p, int32_t* shares_out) {
  if (bs < 0) return fail(CB_EINVAL, "bs must be >= 0");
  if (p < 1) return fail(CB_EINVAL, "p must be >= 1");
  if (!shares_out) return fail(CB_EINVAL, "null output");
  const std::vector<int> v = split_batch_vec(bs, p);
  for (int j = 0; j < p; ++j) shares_out[j] = v[j];
  return CB_OK;
}

int cb_runtime_create(int32_t n_devices, const int32_t* ordinals, cb_runtime** out) {
  if (n_devices < 1 || !ordinals || !out) return fail(CB_EINVAL, "bad runtime arguments");
  int count = 0;
  CB_CUDA(cudaGetDeviceCount(&count));
  auto* rt = new cb_runtime();
  rt->devs.resize(n_devices);
  for (int i = 0; i < n_devices; ++i) {
    if (ordinals[i] < 0 || ordinals[i] >= count) {
      delete rt;
      return fail(CB_EINVAL, "CUDA ordinal " + std::to_string(ordinals[i]) + " not present");
    }
    DeviceCtx& dc = rt->devs[i];
    dc.id = i;
    dc.ordinal = ordinals[i];
    CB_CUDA(cudaSetDevice(dc.ordinal));
    int major = 0;
    CB_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dc.ordinal));
    if (major != 10) {
      delete rt;
      return fail(CB_ENOTSUP, "libcocob200 requires an sm_100 (B200) GPU");
    }
    CB_CUDA(cudaDeviceGetAttribute(&dc.num_sms, cudaDevAttrMultiProcessorCount, dc.ordinal));
    CB_CUDA(cudaStreamCreateWithFlags(&dc.compute, cudaStreamNonBlocking));
    CB_CUDA(cudaStreamCreateWithFlags(&dc.copy, cudaStreamNonBlocking));
    CB_CUDA(cudaStreamCreateWithFlags(&dc.copy2, cudaStreamNonBlocking));
    CB_CUDA(cudaStreamCreateWithFlags(&dc.alloc, cudaStreamNonBlocking));
    dc.ev_pool.resize(1024);
    for (auto& e : dc.ev_pool) CB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CB_CUDA(cudaEventCreate(&dc.t0));
    CB_CUDA(cudaEventCreate(&dc.t1));
  }
  // all-pairs peer access between distinct physical GPUs (NVLink via NVSwitch),
  // for plain allocations and for every device's memory pool
  for (auto& a : rt->devs) {
    cudaMemPool_t pool;
    CB_CUDA(cudaDeviceGetDefaultMemPool(&pool, a.ordinal));
    uint64_t keep = ~0ull;
    CB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    for (auto& b : rt->devs) {
      if (a.ordinal == b.ordinal) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, b.ordinal, a.ordinal);
      if (!can) continue;
      cudaSetDevice(b.ordinal);
      cudaError_t e = cudaDeviceEnablePeerAccess(a.ordinal, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      cudaMemAccessDesc acc{};
      acc.location.type = cudaMemLocationTypeDevice;
      acc.location.id = b.ordinal;  // b may read/write a's pool memory
      acc.flags = cudaMemAccessFlagsProtReadWrite;
      if (cudaMemPoolSetAccess(pool, &acc, 1) != cudaSuccess) cudaGetLastError();
    }
  }
  *out = rt;
  return CB_OK;
}

int cb_runtime_create_spmd(int32_t n_devices, const int32_t* rank_of_device, int32_t my_rank, int32_t my_ordinal,
                           cb_xfer_fn xfer_fn, void* xfer_ctx, cb_runtime** out) {
  if (n_devices < 1 || !rank_of_device || !out || !xfer_fn) return fail(CB_EINVAL, "bad runtime arguments");
  std::vector<int32_t> ords(n_devices, my_ordinal);
  int n_local = 0;
  for (int i = 0; i < n_devices; ++i) n_local += rank_of_device[i] == my_rank;
  if (n_local == 0) return fail(CB_EINVAL, "rank " + std::to_string(my_rank) + " owns no device");
  // the local devices get streams exactly as in the single-process runtime
  std::vector<int32_t> local_ords(n_local, my_ordinal);
  cb_runtime* base = nullptr;
  CB_TRY(cb_runtime_create(n_local, local_ords.data(), &base));
  auto* rt = new cb_runtime();
  rt->spmd = true;
  rt->my_rank = my_rank;
  rt->xfer = xfer_fn;
  rt->xfer_ctx = xfer_ctx;
  rt->devs.resize(n_devices);
  int k = 0;
  for (int i = 0; i < n_devices; ++i) {
    if (rank_of_device[i] == my_rank) {
      rt->devs[i] = base->devs[k++];
    } else {
      rt->devs[i].local = false;
      rt->devs[i].ordinal = -1;
    }
    rt->devs[i].id = i;
    rt->devs[i].rank = rank_of_device[i];
    rt->devs[i].ipc_weights = true;
    rt->ranks.push_back(rank_of_device[i]);
  }
  std::sort(rt->ranks.begin(), rt->ranks.end());
  rt->ranks.erase(std::unique(rt->ranks.begin(), rt->ranks.end()), rt->ranks.end());
  base->devs.clear();  // streams / events now owned by rt
  delete base;
  *out = rt;
  return CB_OK;
}

int cb_device_is_local(cb_runtime* rt, int32_t device, int32_t* local_out) {
  if (!rt || !local_out || device < 0 || device >= int(rt->devs.size())) return fail(CB_EINVAL, "unknown device");
  *local_out = rt->devs[device].local ? 1 : 0;
  return CB_OK;
}

int cb_runtime_destroy(cb_runtime* rt) {
  if (!rt) return CB_OK;
  for (auto& dc : rt->devs) {
    if (!dc.local) continue;
    cudaSetDevice(dc.ordinal);
    cudaStreamSynchronize(dc.compute);
    cudaStreamSynchronize(dc.copy);
    cudaStreamSynchronize(dc.copy2);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dc.ordinal) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    for (auto e : dc.ev_pool) cudaEventDestroy(e);
    cudaEventDestroy(dc.t0);
    cudaEventDestroy(dc.t1);
    cudaStreamDestroy(dc.compute);
    cudaStreamDestroy(dc.copy);
    cudaStreamDestroy(dc.copy2);
    cudaStreamDestroy(dc.alloc);
  }
  delete rt;
  return CB_OK;
}

int cb_device_info(cb_runtime* rt, int32_t device, int32_t* num_sms, uint64_t* free_bytes, uint64_t* total_bytes) {
  if (!rt || device < 0 || device >= int(rt->devs.size())) return fail(CB_EINVAL, "unknown device");
  DeviceCtx& dc = rt->devs[device];
  if (!dc.local) return fail(CB_EINVAL, "device " + std::to_string(device) + " belongs to rank " + std::to_string(dc.rank));
  CB_TRY(use(dc));
  size_t f = 0, t = 0;
  CB_CUDA(cudaMemGetInfo(&f, &t));
  if (num_sms) *num_sms = dc.num_sms;
  if (free_bytes) *free_bytes = f;
  if (total_bytes) *total_bytes = t;
  return CB_OK;
}

int cb_model_create(cb_runtime* rt, const cb_model_desc* desc, int32_t home, cb_model** out) {
  if (!rt || !desc || !out) return fail(CB_EINVAL, "null argument");
  const cb_model_desc& d = *desc;
  if (d.n_layers < 1 || d.d_model <= 0 || d.d_ff <= 0 || d.n_heads <= 0 || d.n_kv_heads <= 0)
    return fail(CB_EINVAL, "model dimensions must be > 0");
  if (d.d_model % d.n_heads != 0) return fail(CB_EINVAL, "d_model must be divisible by n_heads");
  if (d.n_heads % d.n_kv_heads != 0) return fail(CB_EINVAL, "n_heads must be divisible by n_kv_heads");
  const int hd = d.d_model / d.n_heads;
  if (hd != 64 && hd != 128) return fail(CB_ENOTSUP, "head_dim must be 64 or 128");
  if (d.d_model % 64 || d.d_ff % 64) return fail(CB_ENOTSUP, "d_model and d_ff must be multiples of 64");
  if (d.vocab < 1 || d.max_slots < 1 || d.max_ctx < 1 || d.max_tokens < d.max_slots)
    return fail(CB_EINVAL, "vocab/max_slots/max_ctx/max_tokens invalid");
  if (home < 0 || home >= int(rt->devs.size())) return fail(CB_EINVAL, "unknown home device");
  auto* m = new cb_model();
  m->rt = rt;
  m->d = d;
  m->home = home;
  m->hd = hd;
  m->q_n = d.n_heads * hd;
  m->kv_n = d.n_kv_heads * hd;
  m->qkv_n = m->q_n + 2 * m->kv_n;
  layer_offsets(m);
  m->kv_block_bytes = size_t(d.max_slots) * d.max_ctx * kv_token_bytes(m);
  m->layers.resize(d.n_layers);
  m->slot_len.assign(d.max_slots, 0);
  m->slot_epoch.assign(d.max_slots, 0);
  for (const DeviceCtx& dc : rt->devs)
    if (dc.local) {
      cudaSetDevice(dc.ordinal);
      break;
    }
  if (cudaMallocHost(&m->pin_meta, (3 * size_t(d.max_tokens) + d.max_slots + 4 +
                                    4 * (size_t(d.max_tokens) / 64 + d.max_slots)) * 4) != cudaSuccess ||
      cudaMallocHost(&m->pin_next, size_t(d.max_slots) * 4) != cudaSuccess) {
    delete m;
    return fail(CB_ECUDA, "pinned host allocation failed");
  }
  int r = ensure_ws(m, home);
  if (r != CB_OK) {
    cb_model_destroy(m);
    return r;
  }
  *out = m;
  return CB_OK;
}

int cb_model_destroy(cb_model* m) {
  if (!m) return CB_OK;
  sync_all(m);
  for (auto& kv : m->ops) {
    if (!kv.second.committed) op_abort(m, kv.second);
    op_destroy_events(kv.second);
  }
  m->ops.clear();
  sync_all(m);
  for (auto& L : m->layers) {
    for (auto& c : L.reps) dev_free(m, c.dev, c.block);
    for (auto& kv : L.kv) free_kv_block(m, L, kv.first, kv.second);
    for (auto& mc : L.mod) dev_free(m, mc.dev, mc.buf);
  }
  for (auto& kv : m->ws) {
    Workspace& w = kv.second;
    void* ptrs[] = {w.x, w.h, w.hl, w.qkv, w.att, w.act, w.gbuf, w.logits, w.meta, w.next, w.gemm_ws, w.gemm_cnt,
                    w.attn_ws, w.attn_cnt, w.rope};
    for (void* p : ptrs) dev_free(m, kv.first, p);
  }
  dev_free(m, m->home, m->embed);
  dev_free(m, m->home, m->final_norm);
  dev_free(m, m->home, m->lm_head);
  if (m->norm_tab) dev_free(m, m->norm_dev, m->norm_tab);
  for (auto& kv : m->prof.pool) {
    if (!is_local(m, kv.first)) continue;
    cudaSetDevice(devctx(m, kv.first).ordinal);
    for (auto e : kv.second) cudaEventDestroy(e);
  }
  if (m->pin_meta) cudaFreeHost(m->pin_meta);
  if (m->pin_next) cudaFreeHost(m->pin_next);
  delete m;
  return CB_OK;
}

uint64_t cb_module_bytes(cb_model* m, int32_t kind) {
  if (!m) return 0;
  const size_t dm = m->d.d_model, ff = m->d.d_ff;
  switch (kind) {
    case CB_ATTN_PROJ_Q: return size_t(m->q_n) * dm * 2;
    case CB_ATTN_PROJ_K:
    case CB_ATTN_PROJ_V: return size_t(m->kv_n) * dm * 2;
    case CB_ATTN_PROJ_O: return dm * size_t(m->q_n) * 2;
    case CB_SELF_ATTENTION: return (size_t(m->qkv_n) * dm + dm * size_t(m->q_n)) * 2;
    case CB_FFN_PROJ_GATE:
    case CB_FFN_PROJ_UP:
    case CB_FFN_PROJ_DOWN: return ff * dm * 2;
    case CB_DECODER_LAYER: return m->layer_bytes;
    case CB_KV_CACHE: return kv_token_bytes(m);
    case CB_ATTN_NORM:
    case CB_FFN_NORM: return dm * 2;
  }
  return 0;
}

int cb_layer_load(cb_model* m, int32_t layer, int32_t dev, const cb_layer_weights* w) {
  if (!m) return fail(CB_EINVAL, "null argument");
  CB_TRY(check_dev(m, dev));
  if (!w && is_local(m, dev)) return fail(CB_EINVAL, "null weights");
  LayerCopy c;
  CB_TRY(begin_layer_load(m, layer, dev, c));
  if (!c.block) return finish_layer_load(m, layer, c);  // SPMD: registry entry of another rank's copy
  const size_t dm = m->d.d_model, ff = m->d.d_ff;
  CB_CUDA(cudaMemcpy(c.block + m->off_qkv, w->wq, size_t(m->q_n) * dm * 2, cudaMemcpyHostToDevice));
  CB_CUDA(cudaMemcpy(c.block + m->off_qkv + size_t(m->q_n) * dm * 2, w->wk, size_t(m->kv_n) * dm * 2,
                     cudaMemcpyHostToDevice));
  CB_CUDA(cudaMemcpy(c.block + m->off_qkv + size_t(m->q_n + m->kv_n) * dm * 2, w->wv, size_t(m->kv_n) * dm * 2,
                     cudaMemcpyHostToDevice));
  CB_CUDA(cudaMemcpy(c.block + m->off_o, w->wo, dm * size_t(m->q_n) * 2, cudaMemcpyHostToDevice));
  // gate/up interleaved by row: row 2j = gate_j, row 2j+1 = up_j (SwiGLU epilogue pairs)
  CB_CUDA(cudaMemcpy2D(c.block + m->off_gu, 2 * dm * 2, w->w_gate, dm * 2, dm * 2, ff, cudaMemcpyHostToDevice));
  CB_CUDA(cudaMemcpy2D(c.block + m->off_gu + dm * 2, 2 * dm * 2, w->w_up, dm * 2, dm * 2, ff, cudaMemcpyHostToDevice));
  CB_CUDA(cudaMemcpy(c.block + m->off_d, w->w_down, dm * ff * 2, cudaMemcpyHostToDevice));
  CB_CUDA(cudaMemcpy(c.block + m->off_an, w->attn_norm, dm * 2, cudaMemcpyHostToDevice));
  CB_CUDA(cudaMemcpy(c.block + m->off_fn, w->ffn_norm, dm * 2, cudaMemcpyHostToDevice));
  return finish_layer_load(m, layer, c);
}

int cb_layer_init_random(cb_model* m, int32_t layer, int32_t dev, uint64_t seed, float std) {
  if (!m) return fail(CB_EINVAL, "null model");
  LayerCopy c;
  CB_TRY(begin_layer_load(m, layer, dev, c));
  if (!c.block) return finish_layer_load(m, layer, c);  // SPMD: registry entry of another rank's copy
  DeviceCtx& dc = devctx(m, dev);
  const size_t mat_elems = m->off_an / 2;
  const uint64_t s = seed * 1000003ull + uint64_t(layer);
  CB_CUDA(cb::init_uniform_launch(reinterpret_cast<uint16_t*>(c.block), mat_elems, s, std, 0.f, dc.compute));
  CB_CUDA(cb::init_uniform_launch(reinterpret_cast<uint16_t*>(c.block + m->off_an), 2 * size_t(m->d.d_model), s + 7,
                                  0.f, 1.f, dc.compute));
  CB_CUDA(cudaStreamSynchronize(dc.compute));
  return finish_layer_load(m, layer, c);
}

int cb_head_load(cb_model* m, const uint16_t* embed, const uint16_t* final_norm, const uint16_t* lm_head) {
  if (!m) return fail(CB_EINVAL, "null argument");
  if (!is_local(m, m->home)) {  // SPMD: the home device's rank holds the head
    m->head_loaded = true;
    return CB_OK;
  }
  if (!embed || !final_norm || !lm_head) return fail(CB_EINVAL, "null argument");
  DeviceCtx& dc = devctx(m, m->home);
  const size_t ve = size_t(m->d.vocab) * m->d.d_model * 2;
  if (!m->embed) {
    CB_TRY(dev_alloc(dc, (void**)&m->embed, ve, nullptr, MEM_WEIGHTS));
    CB_TRY(dev_alloc(dc, (void**)&m->lm_head, ve, nullptr, MEM_WEIGHTS));
    CB_TRY(dev_alloc(dc, (void**)&m->final_norm, size_t(m->d.d_model) * 2, nullptr, MEM_WEIGHTS));
  }
  CB_TRY(use(dc));
  CB_CUDA(cudaMemcpy(m->embed, embed, ve, cudaMemcpyHostToDevice));
  CB_CUDA(cudaMemcpy(m->lm_head, lm_head, ve, cudaMemcpyHostToDevice));
  CB_CUDA(cudaMemcpy(m->final_norm, final_norm, size_t(m->d.d_model) * 2, cudaMemcpyHostToDevice));
  CB_TRY(make_map(&m->m_head, m->lm_head, m->d.vocab, m->d.d_model, 128));
  m->head_loaded = true;
  return CB_OK;
}

int cb_head_init_random(cb_model* m, uint64_t seed, float std) {
  if (!m) return fail(CB_EINVAL, "null model");
  if (!is_local(m, m->home)) {
    m->head_loaded = true;
    return CB_OK;
  }
  DeviceCtx& dc = devctx(m, m->home);
  const size_t ve = size_t(m->d.vocab) * m->d.d_model;
  if (!m->embed) {
    CB_TRY(dev_alloc(dc, (void**)&m->embed, ve * 2, nullptr, MEM_WEIGHTS));
    CB_TRY(dev_alloc(dc, (void**)&m->lm_head, ve * 2, nullptr, MEM_WEIGHTS));
    CB_TRY(dev_alloc(dc, (void**)&m->final_norm, size_t(m->d.d_model) * 2, nullptr, MEM_WEIGHTS));
  }
  CB_TRY(use(dc));
  CB_CUDA(cb::init_uniform_launch(m->embed, ve, seed * 31 + 1, 1.0f, 0.f, dc.compute));
  CB_CUDA(cb::init_uniform_launch(m->lm_head, ve, seed * 31 + 2, std, 0.f, dc.compute));
  CB_CUDA(cb::init_uniform_launch(m->final_norm, m->d.d_model, seed * 31 + 3, 0.f, 1.f, dc.compute));
  CB_CUDA(cudaStreamSynchronize(dc.compute));
  CB_TRY(make_map(&m->m_head, m->lm_head, m->d.vocab, m->d.d_model, 128));
  m->head_loaded = true;
  return CB_OK;
}

int cb_module_read(cb_model* m, int32_t layer, int32_t dev, int32_t kind, void* dst, uint64_t nbytes) {
  if (!m || !dst) return fail(CB_EINVAL, "null argument");
  CB_TRY(check_layer(m, layer));
  LayerState& L = m->layers[layer - 1];
  const uint64_t want = cb_module_bytes(m, kind);
  if (kind == CB_KV_CACHE || want == 0) return fail(CB_EINVAL, "kind not readable here (use cb_kv_read)");
  if (nbytes != want) return fail(CB_EINVAL, "nbytes must be " + std::to_string(want));
  if (kind >= 0 && kind < kModKinds && L.mod[kind].dev >= 0 && L.mod[kind].dev == dev) {  // migrated sub-module
    sync_all(m);
    CB_TRY(use(devctx(m, dev)));
    CB_CUDA(cudaMemcpy(dst, L.mod[kind].buf, want, cudaMemcpyDeviceToHost));
    return CB_OK;
  }
  const LayerCopy* c = nullptr;
  for (auto& r : L.reps)
    if (r.dev == dev) c = &r;
  if (!c) return fail(CB_ENOREPLICA, "layer " + std::to_string(layer) + " has no copy on device " + std::to_string(dev));
  if (!c->block) return fail(CB_EINVAL, "device " + std::to_string(dev) + " belongs to another rank");
  CB_TRY(use(devctx(m, dev)));
  sync_all(m);
  const size_t dm = m->d.d_model, ff = m->d.d_ff;
  uint8_t* out = static_cast<uint8_t*>(dst);
  const uint8_t* b = c->block;
  switch (kind) {
    case CB_ATTN_PROJ_Q: CB_CUDA(cudaMemcpy(out, b + m->off_qkv, want, cudaMemcpyDeviceToHost)); break;
    case CB_ATTN_PROJ_K:
      CB_CUDA(cudaMemcpy(out, b + m->off_qkv + size_t(m->q_n) * dm * 2, want, cudaMemcpyDeviceToHost));
      break;
    case CB_ATTN_PROJ_V:
      CB_CUDA(cudaMemcpy(out, b + m->off_qkv + size_t(m->q_n + m->kv_n) * dm * 2, want, cudaMemcpyDeviceToHost));
      break;
    case CB_ATTN_PROJ_O: CB_CUDA(cudaMemcpy(out, b + m->off_o, want, cudaMemcpyDeviceToHost)); break;
    case CB_SELF_ATTENTION: CB_CUDA(cudaMemcpy(out, b + m->off_qkv, want, cudaMemcpyDeviceToHost)); break;
    case CB_FFN_PROJ_GATE:
      CB_CUDA(cudaMemcpy2D(out, dm * 2, b + m->off_gu, 2 * dm * 2, dm * 2, ff, cudaMemcpyDeviceToHost));
      break;
    case CB_FFN_PROJ_UP:
      CB_CUDA(cudaMemcpy2D(out, dm * 2, b + m->off_gu + dm * 2, 2 * dm * 2, dm * 2, ff, cudaMemcpyDeviceToHost));
      break;
    case CB_FFN_PROJ_DOWN: CB_CUDA(cudaMemcpy(out, b + m->off_d, want, cudaMemcpyDeviceToHost)); break;
    case CB_DECODER_LAYER: CB_CUDA(cudaMemcpy(out, b, want, cudaMemcpyDeviceToHost)); break;
    case CB_ATTN_NORM: CB_CUDA(cudaMemcpy(out, b + m->off_an, want, cudaMemcpyDeviceToHost)); break;
    case CB_FFN_NORM: CB_CUDA(cudaMemcpy(out, b + m->off_fn, want, cudaMemcpyDeviceToHost)); break;
    default: return fail(CB_EINVAL, "unknown kind");
  }
  return CB_OK;
}

int cb_kv_read(cb_model* m, int32_t layer, int32_t slot, void* dst, uint64_t nbytes, int32_t* dev_out) {
  if (!m || !dst) return fail(CB_EINVAL, "null argument");
  CB_TRY(check_layer(m, layer));
  if (slot < 0 || slot >= m->d.max_slots) return fail(CB_EINVAL, "unknown slot");
  LayerState& L = m->layers[layer - 1];
  const int owner = L.owner.empty() ? -1 : L.owner[slot];
  const uint64_t want = uint64_t(m->slot_len[slot]) * kv_token_bytes(m);
  if (owner < 0 || want == 0) return fail(CB_ESTATE, "slot holds no KV for this layer");
  if (nbytes != want) return fail(CB_EINVAL, "nbytes must be " + std::to_string(want));
  if (!is_local(m, owner)) return fail(CB_EINVAL, "the slot's KV lives on another rank's device " + std::to_string(owner));
  sync_all(m);
  CB_TRY(use(devctx(m, owner)));
  const uint16_t* src = kv_ptr(m, L, owner, slot, 0);
  if (!src) return fail(CB_ESTATE, "slot has no KV index on its owner");
  CB_CUDA(cudaMemcpy(dst, src, want, cudaMemcpyDefault));
  if (dev_out) *dev_out = owner;
  return CB_OK;
}

int cb_slot_len(cb_model* m, int32_t slot, int32_t* len_out) {
  if (!m || !len_out || slot < 0 || slot >= m->d.max_slots) return fail(CB_EINVAL, "bad slot");
  *len_out = m->slot_len[slot];
  return CB_OK;
}

int cb_get_placement(cb_model* m, int64_t* layer_ptr, int32_t* replica_dev, int32_t cap, int32_t* kv_dev) {
  if (!m || !layer_ptr || !replica_dev || !kv_dev) return fail(CB_EINVAL, "null argument");
  int64_t n = 0;
  layer_ptr[0] = 0;
  for (int li = 0; li < m->d.n_layers; ++li) {
    const LayerState& L = m->layers[li];
    for (const auto& c : L.reps) {
      if (n >= cap) return fail(CB_EINVAL, "replica_dev capacity too small");
      replica_dev[n++] = c.dev;
    }
    layer_ptr[li + 1] = n;
    kv_dev[li] = L.reps.empty() ? -1 : kv_device(L);
  }
  return CB_OK;
}


int cb_step(cb_model* m, int32_t phase, int32_t bs, const int32_t* slots, const int32_t* tokens,
            const int32_t* prompt_lens, int32_t* next_out, float* logits_out, float* ms_out) {
  if (!m) return fail(CB_EINVAL, "null model");
  if (bs <= 0 || bs > m->d.max_slots || !slots || !tokens || !next_out || (phase == CB_PHASE_PREFILL && !prompt_lens))
    return step_ordered(m, phase, bs, slots, tokens, prompt_lens, next_out, logits_out, ms_out);
  for (int i = 0; i < bs; ++i)
    if (slots[i] < 0 || slots[i] >= m->d.max_slots) return fail(CB_EINVAL, "slot out of range");
  const std::vector<int> perm = routing_order(m, bs, slots);
  bool ident = true;
  for (int i = 0; i < bs; ++i) ident &= perm[i] == i;
  if (ident) return step_ordered(m, phase, bs, slots, tokens, prompt_lens, next_out, logits_out, ms_out);
  std::vector<int32_t> ps(bs), pl, pt, pn(bs);
  for (int k = 0; k < bs; ++k) ps[k] = slots[perm[k]];
  if (phase == CB_PHASE_PREFILL) {
    std::vector<long long> off(bs + 1, 0);
    for (int i = 0; i < bs; ++i) off[i + 1] = off[i] + std::max(0, prompt_lens[i]);
    pl.resize(bs);
    for (int k = 0; k < bs; ++k) {
      pl[k] = prompt_lens[perm[k]];
      pt.insert(pt.end(), tokens + off[perm[k]], tokens + off[perm[k] + 1]);
    }
  } else {
    pt.resize(bs);
    for (int k = 0; k < bs; ++k) pt[k] = tokens[perm[k]];
  }
  std::vector<float> plog(logits_out ? size_t(bs) * m->d.vocab : 0);
  CB_TRY(step_ordered(m, phase, bs, ps.data(), pt.data(), pl.empty() ? nullptr : pl.data(), pn.data(),
                         logits_out ? plog.data() : nullptr, ms_out));
  for (int k = 0; k < bs; ++k) {
    next_out[perm[k]] = pn[k];
    if (logits_out)
      std::memcpy(logits_out + size_t(perm[k]) * m->d.vocab, plog.data() + size_t(k) * m->d.vocab,
                  size_t(m->d.vocab) * 4);
  }
  return CB_OK;
}

int cb_release_slots(cb_model* m, int32_t n, const int32_t* slots) {
  if (!m || (n > 0 && !slots)) return fail(CB_EINVAL, "null argument");
  for (int i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= m->d.max_slots) return fail(CB_EINVAL, "slot out of range");
    m->slot_len[slots[i]] = 0;
    m->slot_epoch[slots[i]] += 1;
    for (auto& L : m->layers)
      if (!L.owner.empty()) {
        if (L.owner[slots[i]] >= 0) kv_unassign(L, L.owner[slots[i]], slots[i]);
        L.owner[slots[i]] = -1;
      }
  }
  return CB_OK;
}

int cb_last_routing(cb_model* m, int32_t layer, int32_t* dev_out, int32_t* s0_out, int32_t* cnt_out, int32_t cap,
                    int32_t* p_out) {
  if (!m || !p_out) return fail(CB_EINVAL, "null argument");
  CB_TRY(check_layer(m, layer));
  if (m->last_routing.empty()) return fail(CB_ESTATE, "no step has run");
  const auto& r = m->last_routing[layer - 1];
  *p_out = int(r.size());
  if (int(r.size()) > cap) return fail(CB_EINVAL, "capacity too small");
  for (size_t j = 0; j < r.size(); ++j) {
    dev_out[j] = r[j].dev;
    s0_out[j] = r[j].s0;
    cnt_out[j] = r[j].cnt;
  }
  return CB_OK;
}

int cb_kv_offload(cb_model* m, int32_t layer, int32_t to_host, cb_op_stats* st) {
  if (!m) return fail(CB_EINVAL, "null model");
  if (st) *st = cb_op_stats{};
  CB_TRY(check_layer(m, layer));
  return kv_offload(m, layer, to_host != 0, st);
}

int cb_kv_offloaded(cb_model* m, int32_t layer, int32_t* out) {
  if (!m || !out) return fail(CB_EINVAL, "null argument");
  CB_TRY(check_layer(m, layer));
  const LayerState& L = m->layers[layer - 1];
  *out = 0;
  for (auto& kv : L.kv)
    if (kv.second.host) *out = 1;
  return CB_OK;
}

int cb_profile(cb_model* m, int32_t enable) {
  if (!m) return fail(CB_EINVAL, "null model");
  sync_all(m);
  prof_resolve(m);
  for (auto& k : m->prof.stats) k = cb_kstat{};
  m->prof.on = enable != 0;
  return CB_OK;
}

int cb_profile_read(cb_model* m, int32_t kclass, cb_kstat* out) {
  if (!m || !out || kclass < 0 || kclass > 3) return fail(CB_EINVAL, "bad profile query");
  *out = m->prof.stats[kclass];
  return CB_OK;
}

// ---- scaling ops: asynchronous issue / poll / wait / commit / abort (A17)
// SPMD: a failed issue still consumes its op id (the other ranks' issue of the
// same op may have succeeded and registered it under that id)
static int issued(cb_model* m, int r, int64_t* op_id) {
  if (r != CB_OK && m->rt->spmd) {
    *op_id = m->next_op++;
  }
  return r;
}

int cb_issue_replicate_layer(cb_model* m, int32_t layer, int32_t dst, int64_t* op_id, uint64_t* shortfall) {
  if (!m || !op_id) return fail(CB_EINVAL, "null argument");
  if (shortfall) *shortfall = 0;
  return issued(m, issue_replicate(m, layer, dst, op_id, shortfall), op_id);
}

int cb_issue_migrate_layer(cb_model* m, int32_t layer, int32_t dst, int32_t with_kv, int64_t* op_id,
                           uint64_t* shortfall) {
  if (!m || !op_id) return fail(CB_EINVAL, "null argument");
  if (shortfall) *shortfall = 0;
  return issued(m, issue_migrate(m, layer, dst, with_kv, op_id, shortfall), op_id);
}

int cb_issue_migrate_submodule(cb_model* m, int32_t layer, int32_t kind, int32_t dst, int64_t* op_id,
                               uint64_t* shortfall) {
  if (!m || !op_id) return fail(CB_EINVAL, "null argument");
  if (shortfall) *shortfall = 0;
  CB_TRY(check_layer(m, layer));
  CB_TRY(check_dev(m, dst));
  if (kind == CB_DECODER_LAYER) return fail(CB_EINVAL, "whole layers move via MigrateLayer");
  if (kind < 0 || kind > CB_KV_CACHE) return fail(CB_EINVAL, "unknown module kind");
  if (kind == CB_KV_CACHE) return issued(m, issue_kv(m, layer, dst, op_id, shortfall), op_id);
  return issued(m, issue_projection(m, layer, kind, dst, op_id, shortfall), op_id);
}

int cb_issue_evict_replica(cb_model* m, int32_t layer, int32_t device, int64_t* op_id) {
  if (!m || !op_id) return fail(CB_EINVAL, "null argument");
  return issued(m, issue_evict(m, layer, device, op_id), op_id);
}

int cb_op_start(cb_model* m, int64_t op_id) {
  if (!m) return fail(CB_EINVAL, "null model");
  auto it = m->ops.find(op_id);
  if (it == m->ops.end() || it->second.committed) return fail(CB_EINVAL, "op " + std::to_string(op_id) + " is not pending");
  if (it->second.started) return CB_OK;  // single-process ops start at issue
  return op_run(m, it->second);
}

int cb_op_poll(cb_model* m, int64_t op_id, int32_t* done) {
  if (!m || !done) return fail(CB_EINVAL, "null argument");
  auto it = m->ops.find(op_id);
  if (it == m->ops.end()) return fail(CB_EINVAL, "unknown op id " + std::to_string(op_id));
  cb_op_stats st{};
  CB_TRY(op_stats(m, it->second, &st, false));
  *done = st.done;
  return CB_OK;
}

int cb_op_wait(cb_model* m, int64_t op_id, cb_op_stats* st) {
  if (!m) return fail(CB_EINVAL, "null model");
  auto it = m->ops.find(op_id);
  if (it == m->ops.end()) return fail(CB_EINVAL, "unknown op id " + std::to_string(op_id));
  return op_stats(m, it->second, st, true);
}

int cb_commit(cb_model* m, int64_t op_id, int32_t* n_committed) {
  if (!m) return fail(CB_EINVAL, "null model");
  int n = 0;
  for (auto& kv : m->ops) {  // issue order
    PendingOp& op = kv.second;
    if (op.committed || (op_id >= 0 && kv.first != op_id)) continue;
    CB_TRY(op_commit(m, op));
    ++n;
  }
  if (op_id >= 0 && n == 0) return fail(CB_EINVAL, "op " + std::to_string(op_id) + " is not pending");
  if (n_committed) *n_committed = n;
  return CB_OK;
}

int cb_op_abort(cb_model* m, int64_t op_id) {
  if (!m) return fail(CB_EINVAL, "null model");
  std::vector<int64_t> ids;
  for (auto& kv : m->ops)
    if (!kv.second.committed && (op_id < 0 || kv.first == op_id)) ids.push_back(kv.first);
  if (op_id >= 0 && ids.empty()) return fail(CB_EINVAL, "op " + std::to_string(op_id) + " is not pending");
  for (auto it = ids.rbegin(); it != ids.rend(); ++it) {  // newest first
    PendingOp& op = m->ops[*it];
    CB_TRY(op_abort(m, op));
    op_destroy_events(op);
    m->ops.erase(*it);
  }
  return CB_OK;
}

int cb_pending_ops(cb_model* m, int32_t* n) {
  if (!m || !n) return fail(CB_EINVAL, "null argument");
  *n = 0;
  for (auto& kv : m->ops) *n += kv.second.committed ? 0 : 1;
  return CB_OK;
}

int cb_mem_usage(cb_model* m, int32_t device, cb_mem_stats* out) {
  if (!m || !out) return fail(CB_EINVAL, "null argument");
  CB_TRY(check_dev(m, device));
  DeviceCtx& dc = devctx(m, device);
  if (!dc.local) return fail(CB_EINVAL, "device " + std::to_string(device) + " belongs to rank " + std::to_string(dc.rank));
  *out = cb_mem_stats{};
  out->workspace_bytes = dc.mem[MEM_WS];
  out->weight_bytes = dc.mem[MEM_WEIGHTS];
  out->kv_bytes = dc.mem[MEM_KV];
  out->reserved_bytes = dc.reserved;
  CB_TRY(use(dc));
  size_t f = 0, t = 0;
  CB_CUDA(cudaMemGetInfo(&f, &t));
  cudaMemPool_t pool;
  CB_CUDA(cudaDeviceGetDefaultMemPool(&pool, dc.ordinal));
  uint64_t res = 0, used = 0;
  CB_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res));
  CB_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  // pool memory freed back to the pool (not to the driver) is still allocatable
  out->free_bytes = f + (res > used ? res - used : 0);
  out->total_bytes = t;
  return CB_OK;
}

int cb_set_copy_mode(cb_runtime* rt, int32_t mode, uint64_t chunk_bytes) {
  if (!rt || mode < 0 || mode > 2) return fail(CB_EINVAL, "copy mode must be 0 (one copy engine), 1 (two lanes) or 2 (SM push)");
  rt->copy_mode = mode;
  if (chunk_bytes) rt->copy_chunk = chunk_bytes;
  return CB_OK;
}

// ---- synchronous forms: issue + commit at once, then wait (data movement of
// ops.apply, ops.py:173-260, for callers between steps)
static int run_now(cb_model* m, int r, int64_t id, uint64_t shortfall, cb_op_stats* st) {
  if (r != CB_OK) {
    if (st) st->shortfall_bytes = shortfall;
    return r;
  }
  if (m->rt->spmd) {  // (validation passed, the reservation is held: undo it)
    auto it = m->ops.find(id);
    if (it != m->ops.end()) {
      op_abort(m, it->second);
      m->ops.erase(it);
    }
    return fail(CB_ENOTSUP, "SPMD runtime: use cb_issue_* + cb_op_start + cb_commit (every rank agrees first)");
  }
  auto it = m->ops.find(id);
  if (it == m->ops.end()) return fail(CB_ESTATE, "internal: issued op not registered");
  CB_TRY(op_commit(m, it->second));
  CB_TRY(op_stats(m, it->second, st, true));
  op_destroy_events(m->ops[id]);
  m->ops.erase(id);
  return CB_OK;
}

int cb_replicate_layer(cb_model* m, int32_t layer, int32_t dst, cb_op_stats* st) {
  if (!m) return fail(CB_EINVAL, "null model");
  if (st) *st = cb_op_stats{};
  int64_t id = 0;
  uint64_t sf = 0;
  const int r = issue_replicate(m, layer, dst, &id, &sf);  // (issue before reading id)
  return run_now(m, r, id, sf, st);
}

int cb_migrate_layer(cb_model* m, int32_t layer, int32_t dst, int32_t with_kv, cb_op_stats* st) {
  if (!m) return fail(CB_EINVAL, "null model");
  if (st) *st = cb_op_stats{};
  int64_t id = 0;
  uint64_t sf = 0;
  const int r = issue_migrate(m, layer, dst, with_kv, &id, &sf);
  return run_now(m, r, id, sf, st);
}

int cb_migrate_submodule(cb_model* m, int32_t layer, int32_t kind, int32_t dst, cb_op_stats* st) {
  if (!m) return fail(CB_EINVAL, "null model");
  if (st) *st = cb_op_stats{};
  int64_t id = 0;
  uint64_t sf = 0;
  const int r = cb_issue_migrate_submodule(m, layer, kind, dst, &id, &sf);
  return run_now(m, r, id, sf, st);
}

int cb_evict_replica(cb_model* m, int32_t layer, int32_t dev, cb_op_stats* st) {
  if (!m) return fail(CB_EINVAL, "null model");
  if (st) *st = cb_op_stats{};
  int64_t id = 0;
  const int r = issue_evict(m, layer, dev, &id);
  return run_now(m, r, id, 0, st);
}

// experiments: host milliseconds spent enqueuing the last forward pass
double cbt_last_enqueue_ms() { return g_last_enqueue_ms; }

}  // extern "C"
