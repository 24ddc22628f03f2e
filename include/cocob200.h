/*
 * cocob200 — C-ABI of the B200-native module-level scaling data path.
 *
 * The reference (arxiv 2507.18006 "CoCoServe", package `modscale`, mounted at
 * /root/reference) is pure Python and has no FFI: its data path is analytic
 * (SPEC.md:136,317).  Each entry point below is the native replacement of one
 * reference Python seam on the north-star path; the citation after each
 * declaration names the reference function it stands behind.  The Python
 * binding that a maintainer would add on the reference side is shown in
 * INTEGRATION.md (ctypes, the reference's own language).
 *
 * Conventions
 *  - Every function returns an int status: CB_OK (0) or a negative CB_E* code;
 *    cb_last_error() returns the message of the last failure on this thread.
 *  - Status mapping onto the reference's exception classes (ops.py:24-46):
 *      CB_EINVAL     -> OpError            (invalid op / placement edit)
 *      CB_ENOMEM     -> InfeasibleOpError  (shortfall in bytes via out-param)
 *      CB_ENOREPLICA -> MissingReplicaError
 *      CB_ECUDA / CB_ESTATE / CB_ENOTSUP -> RuntimeError
 *    Infeasibility is detected before any byte moves, which keeps
 *    batch_apply (ops.py:263-296) transactional.
 *  - Layers are 1-based, as in PlacementState (domain.py:306-459).  Devices
 *    are logical ids 0..n-1 of the runtime, each bound to a CUDA ordinal
 *    (several logical devices may share one physical GPU).
 *  - Host buffers are plain pointers; bf16 tensors are passed as uint16_t.
 *  - Thread-compatible, not thread-safe: one host thread drives the model
 *    ("placement mutation is single-writer").
 */
#ifndef COCOB200_H
#define COCOB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CB_ABI_VERSION 2

#define CB_OK 0
#define CB_EINVAL (-1)
#define CB_ENOMEM (-2)
#define CB_ENOREPLICA (-3)
#define CB_ECUDA (-4)
#define CB_ESTATE (-5)
#define CB_ENOTSUP (-6)
#define CB_ECOMM (-7) /* the multi-process transport failed (RuntimeError) */

/* ModuleKind ids, in the reference enum's declaration order (domain.py:23-36). */
#define CB_ATTN_PROJ_Q 0
#define CB_ATTN_PROJ_K 1
#define CB_ATTN_PROJ_V 2
#define CB_ATTN_PROJ_O 3
#define CB_SELF_ATTENTION 4
#define CB_FFN_PROJ_GATE 5
#define CB_FFN_PROJ_UP 6
#define CB_FFN_PROJ_DOWN 7
#define CB_DECODER_LAYER 8
#define CB_KV_CACHE 9
/* extra readable parts of a decoder layer (norm vectors, domain.py:259) */
#define CB_ATTN_NORM 10
#define CB_FFN_NORM 11

#define CB_PHASE_PREFILL 0
#define CB_PHASE_DECODE 1

typedef struct cb_runtime cb_runtime;
typedef struct cb_model cb_model;

typedef struct {
  int32_t n_layers;   /* ModelSpec.n_layers   (domain.py:173-191) */
  int32_t d_model;    /* ModelSpec.d_model */
  int32_t d_ff;       /* ModelSpec.d_ff */
  int32_t n_heads;    /* ModelSpec.n_heads */
  int32_t n_kv_heads; /* == n_heads for the reference's MHA accounting; < for GQA (extension) */
  int32_t vocab;      /* builder choice: the reference has no vocabulary */
  int32_t max_slots;  /* concurrent sequences (KV slots) */
  int32_t max_ctx;    /* KV positions per slot */
  int32_t max_tokens; /* activation rows per pass (prefill chunk) */
  float rope_theta;
  float norm_eps;
} cb_model_desc;

/* bf16 host tensors of one decoder layer, PyTorch Linear layout [out, in]. */
typedef struct {
  const uint16_t* attn_norm; /* [d] */
  const uint16_t* wq;        /* [H*hd, d] */
  const uint16_t* wk;        /* [Hkv*hd, d] */
  const uint16_t* wv;        /* [Hkv*hd, d] */
  const uint16_t* wo;        /* [d, H*hd] */
  const uint16_t* ffn_norm;  /* [d] */
  const uint16_t* w_gate;    /* [d_ff, d] */
  const uint16_t* w_up;      /* [d_ff, d] */
  const uint16_t* w_down;    /* [d, d_ff] */
} cb_layer_weights;

/* Data movement of one scaling op, measured with CUDA events: the transfer on
 * the destination's copy stream(s) and the commit's KV catch-up on the new KV
 * device's compute stream. */
typedef struct {
  uint64_t weight_bytes;    /* bytes of module weights moved */
  uint64_t kv_bytes;        /* bytes of KV moved (pre-copy + catch-up) */
  float device_ms;          /* copy_ms + catchup_ms */
  uint64_t shortfall_bytes; /* set on CB_ENOMEM */
  float copy_ms;            /* transfer start -> end (serving continues meanwhile) */
  float catchup_ms;         /* commit: KV appended since the pre-copy (or all of it for evict) */
  uint64_t catchup_bytes;
  int32_t done;             /* every copy of the op has finished */
  int32_t committed;        /* the placement switched */
} cb_op_stats;

/* What the executor really holds on one logical device (bytes). */
typedef struct {
  uint64_t weight_bytes;    /* layer blocks, migrated sub-modules, embedding / lm_head */
  uint64_t kv_bytes;        /* KV blocks */
  uint64_t workspace_bytes; /* activations, GEMM / attention workspaces */
  uint64_t reserved_bytes;  /* held by issued, uncommitted scaling ops (included above) */
  uint64_t free_bytes;      /* allocatable now: cudaMemGetInfo + the pool's cached free memory */
  uint64_t total_bytes;
} cb_mem_stats;

/* ---- library ---------------------------------------------------------- */
int cb_abi_version(void);
const char* cb_last_error(void);

/* Even integer batch split: the first p - (bs mod p) replicas get floor(bs/p),
 * the rest ceil.  Replaces ops.split_batch (ops.py:151-158); the executor uses
 * exactly this rule to route rows to replicas (and _kernels.py:29-33). */
int cb_split_batch(int32_t bs, int32_t p, int32_t* shares_out);

/* ---- runtime: logical devices --------------------------------------------
 * Replaces the simulated ClusterSpec device list (domain.py:74-170): each
 * logical device gets a compute stream, a copy stream and P2P access to every
 * other physical GPU (NVLink through NVSwitch on an HGX B200). */
int cb_runtime_create(int32_t n_devices, const int32_t* cuda_ordinals, cb_runtime** out);
/* Multi-process (SPMD) runtime: one process per GPU, every process holding the
 * SAME global list of logical devices; rank_of_device[i] names the process that
 * owns device i, and the devices of my_rank live on CUDA ordinal my_ordinal.
 * Every rank issues the same calls in the same order (loads, ops, steps, slot
 * releases -- the reference's single-writer control plane, SPEC.md:310-311,
 * replayed on each rank); each rank allocates and computes only for its own
 * devices, keeps the same registry / KV-ownership bookkeeping for all of them,
 * and hands every byte range that crosses a process boundary to `xfer`, in the
 * same global order on every rank.  send != 0: `bytes` at dev_ptr are ready on
 * `cuda_stream`, send them to peer_rank; send == 0: receive `bytes` from
 * peer_rank into dev_ptr, to be consumed on `cuda_stream` (stream-ordered, no
 * host synchronisation required).  channel 0 = per-step exchanges on compute
 * streams (activation rows at replica-run boundaries = the reference's
 * scatter/gather, _kernels.py:41-51; KV rows following their sequence; norm
 * vectors at the first step), channel 1 = scaling-op transfers on copy streams
 * (unused when both sides are on GPUs: layer blocks and the KV of scaling ops
 * move as CUDA IPC pulls, see below).  Markers: send == 2 / 3 open / close a group of
 * exchanges the transport may batch.  Host messages (channel 2): send == 4 sends
 * `bytes` of HOST memory at dev_ptr to peer_rank, send == 5 receives them, both
 * complete on return -- used for the CUDA IPC handle of a layer block or KV
 * block, which the destination's rank maps and pulls with its copy engines over
 * NVLink (weight and KV blocks of an SPMD runtime are cudaMalloc allocations,
 * exportable; the host
 * must not commit an op on any rank before every rank's part finished, e.g. a
 * barrier after cb_op_wait).  A non-zero return fails the call with CB_ECOMM.  The Python host implements it with torch.distributed (NCCL over
 * NVLink on a B200 box).  Not supported in this mode: projection / KV-cache
 * sub-module overrides and KV offload (single-process runtime only). */
typedef int (*cb_xfer_fn)(void* ctx, int32_t channel, int32_t send, int32_t peer_rank, void* dev_ptr,
                          uint64_t bytes, void* cuda_stream);
int cb_runtime_create_spmd(int32_t n_devices, const int32_t* rank_of_device, int32_t my_rank, int32_t my_ordinal,
                           cb_xfer_fn xfer, void* xfer_ctx, cb_runtime** out);
/* 1 if `device` is computed by this process. */
int cb_device_is_local(cb_runtime* rt, int32_t device, int32_t* local_out);
int cb_runtime_destroy(cb_runtime* rt);
int cb_device_info(cb_runtime* rt, int32_t device, int32_t* num_sms, uint64_t* free_bytes,
                   uint64_t* total_bytes);

/* ---- model: module registry of device buffers -----------------------------
 * The library owns every device buffer, keyed by (layer, ModuleKind, device). */
int cb_model_create(cb_runtime* rt, const cb_model_desc* desc, int32_t home_device, cb_model** out);
int cb_model_destroy(cb_model* m);
/* Bytes of one module copy (DECODER_LAYER = ModuleCatalog.decoder_layer_mb*1e6
 * for MHA shapes, domain.py:241-264; KV_CACHE = bytes per token per layer). */
uint64_t cb_module_bytes(cb_model* m, int32_t kind);

/* First load of a layer makes `device` its original (PlacementState.sequential,
 * domain.py:352-359).  Weights are copied; host buffers may be freed after. */
int cb_layer_load(cb_model* m, int32_t layer, int32_t device, const cb_layer_weights* w);
int cb_layer_init_random(cb_model* m, int32_t layer, int32_t device, uint64_t seed, float std);
int cb_head_load(cb_model* m, const uint16_t* embed, const uint16_t* final_norm, const uint16_t* lm_head);
int cb_head_init_random(cb_model* m, uint64_t seed, float std);

/* Byte readback of one module copy in canonical [out, in] layout (for byte
 * parity of replication/migration).  `kind` = CB_* module id; DECODER_LAYER
 * returns the raw contiguous layer block.  nbytes must equal the module size. */
int cb_module_read(cb_model* m, int32_t layer, int32_t device, int32_t kind, void* host_dst, uint64_t nbytes);
/* KV of one slot for one layer: [len][2][Hkv*hd] bf16 from the device holding it. */
int cb_kv_read(cb_model* m, int32_t layer, int32_t slot, void* host_dst, uint64_t nbytes, int32_t* device_out);
int cb_slot_len(cb_model* m, int32_t slot, int32_t* len_out);

/* Current executor plan = the registry as the device sees it: CSR replica list
 * (original first) like StepArrays.layer_ptr (sim.py:204-236) plus the KV
 * device per layer (PlacementState.kv_device, domain.py:380-383). */
int cb_get_placement(cb_model* m, int64_t* layer_ptr, int32_t* replica_dev, int32_t cap, int32_t* kv_dev);

/* ---- executor hook: replaces step_batch / step_time_s (sim.py:239-300) -----
 * One pass over `bs` sequences in admission order.  Prefill: tokens holds the
 * concatenated prompts (prompt_lens[i] each) and the slots must be empty.
 * Decode: one token per sequence, appended at the slot's current length.
 * Rows are routed to each layer's replicas with cb_split_batch counts over the
 * step's sequences in a sticky routing order (a sequence stays on the replica
 * holding its KV while that replica's share has room; fresh and overflow
 * sequences fill the rest in replica order), each replica taking a contiguous
 * range of that order; activations move between devices at placement changes,
 * and KV rows follow their sequence's replica.  Outputs are in the caller's order.
 * Outputs: greedy next token per sequence, optional fp32 logits [bs][vocab],
 * device time of the pass.  CB_EINVAL before any launch for: slots out of range
 * or repeated, token ids outside [0, vocab), prompt lengths outside
 * [1, max_ctx], prefill into a live slot, decode on an empty one, a sequence
 * reaching max_ctx. */
int cb_step(cb_model* m, int32_t phase, int32_t bs, const int32_t* slots, const int32_t* tokens,
            const int32_t* prompt_lens, int32_t* next_tokens_out, float* logits_out, float* device_ms_out);
int cb_release_slots(cb_model* m, int32_t n, const int32_t* slots);
/* Routing the last step used for `layer`: per replica (device, first sequence,
 * sequence count), the sequences counted in the step's routing order.  p_out =
 * number of replicas. */
int cb_last_routing(cb_model* m, int32_t layer, int32_t* dev_out, int32_t* seq_begin_out, int32_t* seq_count_out,
                    int32_t cap, int32_t* p_out);

/* ---- scaling operator data movement: apply() (ops.py:173-260) ------------- */
/* ReplicateLayer (ops.py:199-211): copy the layer block original -> dst. */
int cb_replicate_layer(cb_model* m, int32_t layer, int32_t dst, cb_op_stats* st);
/* MigrateLayer (ops.py:213-228): move the original to dst; with_kv moves the
 * layer's KV too, otherwise KV stays resident on its current device. */
int cb_migrate_layer(cb_model* m, int32_t layer, int32_t dst, int32_t with_kv, cb_op_stats* st);
/* MigrateSubModule (ops.py:230-251).  KV_CACHE moves the layer's KV rows (the
 * attention core then runs on that device); a projection kind (Q/K/V/O, GATE,
 * UP, DOWN) or SELF_ATTENTION copies the module's weights ([out, in] layout) to
 * dst, after which that projection's GEMM runs there with its input rows (and
 * the fp32 residual rows for O / DOWN) hopping to dst and its output rows back. */
int cb_migrate_submodule(cb_model* m, int32_t layer, int32_t kind, int32_t dst, cb_op_stats* st);
/* EvictReplica (ops.py:253-258): drop a non-original copy; KV rows it held move
 * back to the original first. */
int cb_evict_replica(cb_model* m, int32_t layer, int32_t device, cb_op_stats* st);
/* The four functions above are the synchronous forms (issue + commit + wait)
 * for callers between steps.  The serving path uses the asynchronous forms:
 *
 * Asynchronous, serving-concurrent scaling ops -- the reference's transition
 * (_Transition / _controller_tick / _commit_transitions, sim.py:396-403,
 * 812-841, 614-622; "the old placement keeps serving until the switch",
 * SPEC.md:531).  cb_issue_* validates (CB_EINVAL / CB_ENOREPLICA / CB_ESTATE
 * before anything moves), RESERVES the destination memory (CB_ENOMEM with the
 * shortfall, nothing reserved), enqueues the transfer on the destination's copy
 * streams and returns at once with an op id.  cb_step keeps running on the
 * pre-op placement meanwhile.  KV the op moves is pre-copied at issue and only
 * the tokens appended since are copied at the commit.  At most one uncommitted
 * op per layer (CB_ESTATE).  cb_commit switches the placement of one op
 * (op_id >= 0) or of every pending op in issue order (op_id = -1) at the step
 * boundary it is called at, without host synchronisation (the next step's
 * kernels are stream-ordered after the transfer).  cb_op_abort releases the
 * reservations of uncommitted ops (op_id = -1: all, newest first): a decision
 * whose k-th op fails leaves the executor exactly as before (batch_apply's
 * transactionality, ops.py:263-296). */
int cb_issue_replicate_layer(cb_model* m, int32_t layer, int32_t dst, int64_t* op_id, uint64_t* shortfall_bytes);
int cb_issue_migrate_layer(cb_model* m, int32_t layer, int32_t dst, int32_t with_kv, int64_t* op_id,
                           uint64_t* shortfall_bytes);
int cb_issue_migrate_submodule(cb_model* m, int32_t layer, int32_t kind, int32_t dst, int64_t* op_id,
                               uint64_t* shortfall_bytes);
int cb_issue_evict_replica(cb_model* m, int32_t layer, int32_t device, int64_t* op_id);
/* SPMD runtime only: cb_issue_* reserves on the destination's rank and
 * returns; every rank then agrees on the outcome (the host all-reduces the
 * status) and calls cb_op_start (all succeeded: the transfer is enqueued, send
 * on the source's rank, receive on the destination's) or cb_op_abort.  A rank
 * whose issue failed still consumes the op id, so ids stay aligned. */
int cb_op_start(cb_model* m, int64_t op_id);
int cb_op_poll(cb_model* m, int64_t op_id, int32_t* done); /* non-blocking */
int cb_op_wait(cb_model* m, int64_t op_id, cb_op_stats* st); /* blocks until the op's copies finished */
int cb_commit(cb_model* m, int64_t op_id, int32_t* n_committed);
int cb_op_abort(cb_model* m, int64_t op_id);
int cb_pending_ops(cb_model* m, int32_t* n);
/* Per-device memory the executor holds (the controller's usage view,
 * PressureView / _usage_by_device, sim.py:507-525). */
int cb_mem_usage(cb_model* m, int32_t device, cb_mem_stats* out);
/* Transfer engine of the scaling ops: 0 = one cudaMemcpyPeerAsync, 1 = chunks
 * alternating over two copy lanes (default, 64 MB chunks), 2 = SM kernel pushing
 * 16-byte stores from the source GPU.  chunk_bytes 0 keeps the current chunk. */
int cb_set_copy_mode(cb_runtime* rt, int32_t mode, uint64_t chunk_bytes);

/* Phase-3 KV offload (autoscaler.py:568-583 PerformanceReduction): move the
 * layer's KV blocks to (to_host=1) or back from (0) mapped pinned host memory.
 * Attention reads an offloaded block in place (zero-copy); kv_bytes = live KV moved. */
int cb_kv_offload(cb_model* m, int32_t layer, int32_t to_host, cb_op_stats* st);
int cb_kv_offloaded(cb_model* m, int32_t layer, int32_t* offloaded_out);

/* ---- live per-kernel profiling (evidence for the roofline numbers) ----------
 * When enabled, every launch of the executor is bracketed by CUDA events on the
 * stream it is launched on; after each step the elapsed times are added to
 * per-class totals together with the launch's ALGORITHMIC bytes and FLOPs
 * (weights + activations read/written; KV bytes actually attended). */
#define CB_KCLASS_GEMM 0      /* tcgen05 projections (QKV, O, gate/up, down, lm_head) */
#define CB_KCLASS_ATTENTION 1 /* KV-cache attention (+ split combine) */
#define CB_KCLASS_ELEMWISE 2  /* RMSNorm, RoPE+KV append, embedding, argmax, gather */
#define CB_KCLASS_COPY 3      /* activation reshard / KV row moves between devices */
typedef struct {
  uint32_t launches;
  float ms;     /* summed device time */
  double bytes; /* summed algorithmic bytes */
  double flops; /* summed algorithmic FLOPs */
} cb_kstat;
int cb_profile(cb_model* m, int32_t enable); /* enable=1 resets the counters */
int cb_profile_read(cb_model* m, int32_t kclass, cb_kstat* out);

#ifdef __cplusplus
}
#endif
#endif /* COCOB200_H */
