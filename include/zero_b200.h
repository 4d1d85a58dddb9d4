/*
 * zero_b200.h -- C ABI of the B200-native ZeRO-DP hot path (arXiv 1910.02054).
 *
 * The library implements one partitioned mixed-precision Adam step at ZeRO-DP
 * stage 0 (replicated DP baseline), 1 (P_os), 2 (P_os+g) or 3 (P_os+g+p):
 *   zero_reduce_grads  flatten/cast/prescale a gradient bucket and reduce-scatter it
 *                      so rank r holds only its 1/N_d partition (§5.2)
 *   zero_step          overflow check + global grad norm, fused partitioned Adam on
 *                      the owned shard with the 16-bit recast written straight into
 *                      the all-gather buffer, then the all-gather (§5.1)
 *   zero_gather_params stage 3: per-layer all-gather with prefetch before each
 *                      forward/backward use (§5.3 and §7.2.2)
 * Citations "P:n" are lines of the paper text; "c-k" are the readings
 * recorded in DESIGN.md §3 where the paper is silent.
 *
 * Conventions for every call:
 *  - Every function returns zero_status; nothing throws across the ABI.
 *  - Pointers documented as "device" are CUDA device (or UVA-mapped) addresses on
 *    the context's device; "host" pointers are ordinary CPU memory.
 *  - A context is used by one host thread.  All calls after zero_bind_buffers are
 *    asynchronous with respect to the host (stream-ordered on the caller's compute
 *    stream) unless stated otherwise.
 *  - ZERO_EINVAL: bad argument; no state was changed.
 *    ZERO_ESTATE: call-order violation (e.g. zero_step before every bucket of the
 *    step was reduced); no state was changed.
 *    ZERO_ECUDA / ZERO_ENCCL: a CUDA or NCCL error; the context is poisoned (sticky)
 *    and every later call except zero_last_error/zero_destroy returns the same code.
 *  - Gradient overflow is NOT an error: the step is skipped and reported (c-4).
 */
#ifndef ZERO_B200_H
#define ZERO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZERO_ABI_VERSION 3     /* 2: zero_config.mp_rank, zero_tensor.flags, zero_step_begin/end, zero_pa_*;
                                  3: zero_timing.ag_ms, R32 over NCCL, zero_wait (NCCL watchdog), zero_set_timing */
#define ZERO_MAX_RANKS 8      /* one NVL8 box */

typedef enum {
  ZERO_OK = 0,
  ZERO_EINVAL = 1,
  ZERO_ENOMEM = 2,
  ZERO_ECUDA = 3,
  ZERO_ENCCL = 4,
  ZERO_ESTATE = 5,
  ZERO_EUNSUPPORTED = 6,
  ZERO_ETIMEOUT = 7          /* zero_wait: work still running at the deadline (not sticky) */
} zero_status;

/* 16-bit model dtypes (fp16 params/grads, fp32 optimizer states). */
typedef enum { ZERO_FP16 = 0, ZERO_BF16 = 1, ZERO_FP32 = 2 } zero_dtype;

/* Reduced-gradient precision (reading c-2): R16 = fp32 sum in ascending rank,
 * rounded once to 16-bit (2 bytes/elem, the paper's 2Psi/N_d); R32 = the
 * same fp32 sum kept in fp32 (4 bytes/elem). */
typedef enum { ZERO_R16 = 0, ZERO_R32 = 1 } zero_reduce_mode;

/* How ranks exchange data.
 * LOCAL: n_d == 1, no collective ("N=1 degenerates").
 * NCCL:  one process per GPU; ncclReduceScatter / ncclAllGather / ncclAllReduce on a
 *        communicator borrowed from torch (ProcessGroupNCCL._comm_ptr()).
 * PEER:  ranks read/write each other's buffers through a peer-pointer table
 *        (pull reduce-scatter in fixed rank order; the Adam kernel stores the
 *        recast parameters into every rank's replica = fused all-gather).  The
 *        table is installed by zero_sim_group (N contexts on one device, one
 *        process: BASELINE config 1's "simulated ranks"). */
typedef enum { ZERO_TRANSPORT_LOCAL = 0, ZERO_TRANSPORT_NCCL = 1, ZERO_TRANSPORT_PEER = 2 } zero_transport;

/* ---------------------------------------------------------------------------
 * Parameter layout (reading c-7; "N_d equal partitions", P:366 buckets,
 * P:420-422 constant-size buffer C_B).
 * Tensors are listed in forward order with non-decreasing layer ids.  Tensor t
 * is placed in buckets that never span layers (nor MP-replicated and partitioned
 * tensors, see ZERO_TENSOR_MP_REPLICATED); every bucket is padded to a
 * multiple of N_d * align_elems; rank r owns the r-th 1/N_d slice of every
 * bucket, so each rank owns exactly psi_padded / N_d elements.
 * ------------------------------------------------------------------------- */
/* zero_tensor.flags: the tensor is replicated across a model-parallel group (e.g.
 * LayerNorm weights and row-parallel biases under Megatron tensor slicing):
 * its gradient-norm contribution counts only on MP rank 0 (zero_config.mp_rank), and
 * no bucket mixes replicated and MP-partitioned tensors (reading R-MP1). */
#define ZERO_TENSOR_MP_REPLICATED 1u

typedef struct {
  uint64_t numel;   /* elements of the tensor (0 allowed: the tensor is skipped) */
  uint32_t layer;   /* layer id, non-decreasing in forward order */
  uint32_t flags;   /* ZERO_TENSOR_MP_REPLICATED or 0 */
} zero_tensor;

typedef struct {
  uint32_t n_tensors;
  uint32_t align_elems;        /* A: power of two >= 1; 64 = 128 B of 16-bit */
  const zero_tensor* tensors;  /* host array of n_tensors, copied by the callee */
  uint64_t bucket_cap_elems;   /* C_B in elements; 0 = one bucket per layer */
} zero_layout_desc;

typedef struct {
  uint32_t layer;
  uint32_t n_pieces;
  uint32_t first_piece;        /* index into the piece array */
  uint32_t flags;              /* ZERO_TENSOR_MP_REPLICATED if its tensors are */
  uint64_t base;               /* global flat offset of the bucket */
  uint64_t size;               /* B_k: padded size, multiple of N_d * A */
  uint64_t shard_off;          /* offset of this bucket's slice in every rank's shard */
} zero_bucket;

typedef struct {
  uint32_t tensor;
  uint32_t bucket;
  uint64_t tensor_off;         /* first element of the tensor covered */
  uint64_t bucket_off;         /* position inside the bucket (A-aligned) */
  uint64_t count;
} zero_piece;

typedef struct {
  uint64_t psi;                /* true parameter count */
  uint64_t psi_padded;         /* Psi' = sum of B_k */
  uint64_t shard;              /* Psi' / N_d */
  uint32_t n_buckets;
  uint32_t n_pieces;
  uint32_t n_layers;           /* number of distinct layer ids that own buckets */
  uint32_t max_bucket;         /* max B_k (elements) -- fits in 32 bits only when
                                  C_B is set; 0xFFFFFFFF means "see buckets" */
} zero_layout_info;

/* Pure host function (no GPU needed).  Computes the layout of `desc` for `n_d`
 * ranks.  Fills *info; fills `buckets` / `pieces` (host arrays) when non-NULL
 * and their capacities (cap_buckets, cap_pieces) are large enough, else returns
 * ZERO_EINVAL after filling *info (call once with NULL arrays to size them).
 * Errors: ZERO_EINVAL for n_d < 1 or > ZERO_MAX_RANKS, A not a power of two,
 * 0 < C_B < N_d*A, decreasing layer ids, or a layout with no elements. */
zero_status zero_plan_layout(const zero_layout_desc* desc, int n_d, zero_layout_info* info,
                             zero_bucket* buckets, uint32_t cap_buckets,
                             zero_piece* pieces, uint32_t cap_pieces);

/* ---------------------------------------------------------------------------
 * Optimizer configuration (copied at zero_init).  Adam as read in c-3:
 *   g = G * inv (* clip);  m = b1*m + (1-b1)*g;  v = b2*v + ((1-b2)*g)*g;
 *   p = p - step * (m / (sqrt(v)*rsb2 + eps)),  step = lr/(1-b1^t), rsb2 = 1/sqrt(1-b2^t)
 * fp32, each op rounded to nearest, no FMA; inv = 1/(N_d * S * prescale).
 * ------------------------------------------------------------------------- */
typedef struct {
  float lr, beta1, beta2, eps;
  float weight_decay;          /* > 0: decoupled p -= lr*wd*p before the update */
  float max_grad_norm;         /* > 0: clip by max/(norm + 1e-6) when norm > max */
  zero_dtype param_dtype;      /* FP16 | BF16 */
  zero_dtype grad_dtype;       /* FP16 | BF16 (must equal param_dtype) | FP32 */
  zero_reduce_mode reduce_mode;
  int32_t dynamic_loss_scale;  /* 1: halve on overflow, double after scale_window good steps */
  float loss_scale;            /* initial S (power of two) */
  float min_loss_scale;
  uint32_t scale_window;
  float grad_prescale;         /* sigma, power of two applied in the flatten (default 1) */
  uint32_t prefetch_depth;     /* stage 3: layers gathered ahead of use (default 1) */
  uint32_t pool_buckets;       /* stages 2/3, N_d > 1: C_B staging slots (default 2) */
  uint32_t timing;             /* 1: record CUDA events around each phase (ZERO_Q_TIMING) */
  uint32_t mp_rank;            /* ZeRO x MP: this rank's index in its model-parallel group
                                  (0 without MP); MP-replicated tensors add to the
                                  gradient norm only on MP rank 0 (R-MP1) */
} zero_config;

/* Step record (32 bytes), written asynchronously by zero_step. */
typedef struct {
  uint64_t t;                  /* Adam step count after this step (unchanged if skipped) */
  uint32_t overflow;           /* 1: a non-finite reduced gradient -> step skipped */
  float loss_scale;            /* S used by this step */
  float clip;                  /* clip coefficient applied (1 = none) */
  uint32_t reserved;
  double grad_norm;            /* sqrt(sum (G*inv)^2) over all Psi' elements */
} zero_step_info;

/* ---------------------------------------------------------------------------
 * Context lifecycle
 * ------------------------------------------------------------------------- */
struct zero_ctx;

/* Create the context of rank `rank` of `n_d`.
 *  stage: 0 = replicated DP (all-reduce, every rank updates all Psi'),
 *         1 = P_os, 2 = P_os+g, 3 = P_os+g+p.
 *  K: optimizer bytes per parameter; must be 12 ("Mixed-precision Adam has K=12").
 *  transport: LOCAL requires n_d == 1 (n_d == 1 with PEER also becomes LOCAL);
 *  NCCL requires nccl_comm (an ncclComm_t of size n_d whose rank is `rank`, borrowed,
 *  never destroyed; n_d == 1 keeps the NCCL code path on a 1-rank communicator);
 *  PEER requires a later zero_sim_group (one process) or zero_peer_open (CUDA IPC).
 *  compute_stream: cudaStream_t (borrowed; NULL = legacy default stream).
 *  The current CUDA device is the context's device.  No device work happens here
 *  (the host layout and arena sizes are usable without a GPU); the context owns only
 *  host memory until zero_bind_buffers.
 *  Errors: ZERO_EINVAL (K != 12, stage not in 0..3, bad dtype combination,
 *  rank/n_d/transport mismatch, layout errors), ZERO_EUNSUPPORTED (stage 0 with R32;
 *  R32 over NCCL at stage 1), ZERO_ECUDA.
 *  R32 over NCCL (stages 2/3; also on a 1-rank communicator): each bucket is flattened
 *  into an fp32 pool slot holding the cast/prescaled 16-bit values widened, and
 *  reduce-scattered in fp32 (2x the 16-bit wire bytes), so no partial sum is rounded
 *  to 16-bit; the sum order is NCCL's (exact for N_d <= 2). */
zero_status zero_init(const zero_layout_desc* desc, int n_d, int rank, int stage, int K,
                      const zero_config* cfg, zero_transport transport, void* nccl_comm,
                      void* compute_stream, struct zero_ctx** out);

/* Bytes of each arena the caller must allocate (device memory, >= 256-B aligned).
 *  opt     12 * stride : fp32 master | momentum | variance, S_e elements each at
 *                     a stride of opt_stride_elems = S_e rounded up to 64
 *                     (S_e = Psi'/N_d; Psi' at stage 0)            -- K Psi / N_d
 *  p16     2 * Psi' (stages 0-2: full replica) or 2 * Psi'/N_d (stage 3 shard)
 *  grad    2 * Psi' (stages 0/1: flat gradient buffer, reduced in place) or
 *          pool_buckets * max B_k * 2 (stages 2/3 staging pool, NCCL/PEER); 0 otherwise
 *  gred    reduced-gradient shard: stages 2/3 R16 2*Psi'/N_d, R32 4*Psi'/N_d;
 *          stage 1 R32 4*Psi'/N_d; 0 otherwise
 *  gather  stage 3, NCCL/PEER: (prefetch_depth + 1) * max layer elements * 2
 *  scratch device state, norm slots, partial sums, segment table, signals (< 1 MB),
 *          plus 14 KB of per-CTA epilogue partials per bucket slot (e.g. 1.7 MB at 7.5B)
 * The grad/gred/gather/scratch arenas are the only transient buffers: nothing is
 * allocated during a step (M_D). */
typedef struct {
  uint64_t opt_bytes, p16_bytes, grad_bytes, gred_bytes, gather_bytes, scratch_bytes;
  uint64_t opt_stride_elems;   /* element offset of m (and 2x that of v) inside opt */
} zero_sizes;
zero_status zero_buffer_sizes(const struct zero_ctx* ctx, zero_sizes* out);

typedef struct {
  void *opt, *p16, *grad, *gred, *gather, *scratch;   /* device pointers, caller-owned */
} zero_buffers;
/* Bind the caller's arenas (NULL allowed where the size is 0) and zero them on the
 * compute stream.  The library never frees them. */
zero_status zero_bind_buffers(struct zero_ctx* ctx, const zero_buffers* bufs);

/* Link n contexts of one process and one device into a PEER group (BASELINE config
 * 1: N_d simulated ranks on one GPU).  ranks[r] must have rank r, transport PEER,
 * the same layout/stage/config/stream, and bound buffers.  The pull reduce-scatter
 * of bucket k is issued when the last rank has flattened k; zero_step of any rank
 * may run once every rank reduced every bucket of the step. */
zero_status zero_sim_group(struct zero_ctx* const* ranks, int n);

/* PEER across processes (one process per GPU, or several on one GPU): export this
 * rank's peer-visible arenas (grad, p16, scratch) as an opaque blob of CUDA IPC
 * handles + offsets; exchange the blobs (e.g. torch.distributed.all_gather_object)
 * and install all n_d of them, in rank order, with zero_peer_open.  Afterwards the
 * pull reduce-scatter reads peers' buckets over NVLink, the Adam kernel stores the
 * recast parameters into every peer's replica (fused all-gather), and device-side
 * release/acquire signals at system scope order the ranks (no host barrier).
 * As with NCCL, every rank must reduce the buckets of a step in the same order (the
 * pull reduce-scatter of bucket k waits for every rank's flatten of bucket k).
 * zero_peer_export with blob == NULL returns the blob size in *blob_bytes.
 * Errors: ZERO_ESTATE (not an unlinked, bound PEER context), ZERO_EINVAL (a blob of
 * another rank/layout/stage), ZERO_ECUDA (IPC failure; the arenas must come from
 * cudaMalloc-backed memory without expandable segments). */
zero_status zero_peer_export(struct zero_ctx* ctx, void* blob, size_t* blob_bytes);
zero_status zero_peer_open(struct zero_ctx* ctx, const void* const* blobs, size_t blob_bytes);

/* Initialise the model states from the full fp32 master weights: tensor_master[t]
 * is a device pointer to tensor t's numel fp32 values (every rank passes the same
 * values), or NULL to leave tensor t as it is -- so a large model can be loaded in
 * several calls with a bounded temporary (each call covers a subset of tensors).
 * Writes this rank's fp32 shard of the given tensors and their 16-bit parameters
 * (full replica at stages 0-2, own shard at stage 3); every call zeroes m and v and
 * resets t, S and the loss-scale state.  Pointers are borrowed until the call's
 * stream work completes. */
zero_status zero_load_master(struct zero_ctx* ctx, const void* const* tensor_master);

typedef struct {          /* loss-scale / Adam scalars (reading c-4) */
  double b1t, b2t;
  uint64_t t;
  float loss_scale;
  uint32_t good_steps;
} zero_device_state;

/* Checkpointing and resharding (P:357's partitions are per rank).
 * zero_export_state writes the elements THIS rank owns of every tensor's fp32
 * master / momentum / variance into the caller's per-tensor arrays (device pointers
 * to numel fp32 each; NULL = skip), leaving the other elements untouched -- the
 * union over ranks (e.g. a sum of zero-initialised arrays; at stage 0 any single
 * rank) is the whole optimizer state in tensor coordinates, independent of N_d,
 * bucketing and padding.  zero_import_state reads such arrays (the owned elements
 * only; a context of any N_d/stage/C_B), rewrites the 16-bit parameters from the
 * master, and, if st != NULL, sets the device scalars (t, beta^t, S, good steps; from
 * zero_query(ZERO_Q_STATE)).  Both are stream-ordered on the compute stream. */
zero_status zero_export_state(struct zero_ctx* ctx, void* const* master, void* const* m, void* const* v);
zero_status zero_import_state(struct zero_ctx* ctx, const void* const* master, const void* const* m,
                              const void* const* v, const zero_device_state* st);

/* Register per-tensor gradient pointers (device; dtype = grad_dtype; tensor t has
 * numel contiguous elements).  Used by zero_reduce_grads when it is passed NULL. */
zero_status zero_set_grad_ptrs(struct zero_ctx* ctx, const void* const* tensor_grads);

/* Bucket k's gradients are complete (backward hook, buckets in any order):
 * flatten/cast/prescale them into the bucket (M_D copy; "fuse all the
 * gradients into a single flattened buffer"), then reduce-scatter the bucket
 * so this rank holds the sum of its slice ("perform reduction on the entire
 * bucket at once") and the slice's overflow flag and norm partial.
 * tensor_grads: NULL (registered pointers) or an array of n_tensors device pointers.
 * The gradient buffers are read asynchronously (LOCAL/NCCL flatten on library
 * streams forked from the caller's stream) and are borrowed until zero_step is
 * enqueued; the caller's stream is ordered after them by zero_step.
 * Errors: ZERO_EINVAL (bad k, missing pointer), ZERO_ESTATE (k already reduced this step). */
zero_status zero_reduce_grads(struct zero_ctx* ctx, uint32_t bucket, const void* const* tensor_grads);

/* Finish the step: global overflow decision and grad norm (all-reduced), loss-scale
 * update, fused Adam on the owned shard writing the recast 16-bit parameters into
 * the all-gather buffer, then the all-gather (stages 1/2, "all-gather ... at
 * the end of each training step"; stage 0 updates everything locally; stage 3
 * keeps only the shard).  host_out (optional, pinned host memory for
 * asynchrony) receives the step record by the time the step's work completes (read it
 * after synchronizing the compute stream): UVA-mapped pinned memory (cudaHostAlloc /
 * torch pin_memory) is written directly by the decision kernel, other memory by a D2H
 * copy at the end of the step.  An overflow skips the update on the
 * device (t, m, v, master unchanged; the loss scale is halved when dynamic); the host
 * never waits.  The caller's compute stream is ordered after the step; with the
 * cross-process PEER transport the step ends with a device barrier, so every
 * replica is final before any rank's next forward.  Stage 3 copies gathered before
 * the step are invalidated (the next zero_gather_params gathers again).
 * Errors: ZERO_ESTATE if some bucket of the step was not reduced (or, in a
 * simulated group, not reduced by every rank; or the rank already stepped). */
zero_status zero_step(struct zero_ctx* ctx, zero_step_info* host_out);

/* ZeRO x MP (reading R-MP1): zero_step in two halves, so that the step
 * decision can span the model-parallel group as well as this data-parallel one.
 * zero_step_begin does everything zero_step does up to the decision: it joins the
 * reduce phase and writes this DP group's combined partial {sum of (G*inv)^2 over
 * the counted buckets, number of ranks with a non-finite gradient} (two doubles) to
 * the device address zero_query(ZERO_Q_DECISION) returns; the caller's compute
 * stream is ordered after the write.  The caller then SUM-all-reduces those 16 bytes
 * over its MP group on the compute stream (e.g. torch.distributed.all_reduce of a
 * float64 view), so every MP rank sees the global norm and the global overflow, and
 * calls zero_step_end, which makes the decision from the (all-reduced) partial and
 * finishes the step exactly as zero_step.  Without MP, zero_step_begin followed by
 * zero_step_end is zero_step.  Buckets of MP-replicated tensors
 * (ZERO_TENSOR_MP_REPLICATED) add to the norm only on MP rank 0 (zero_config.mp_rank).
 * Errors: as zero_step; ZERO_ESTATE for a begin without end or the reverse. */
zero_status zero_step_begin(struct zero_ctx* ctx);
zero_status zero_step_end(struct zero_ctx* ctx, zero_step_info* host_out);

/* Stage 3: make layer `layer`'s 16-bit parameters available (all-gather of its
 * buckets into a pool slot, "spread ... across the entire forward
 * propagation ... once again for the backward propagation in the reverse order")
 * and prefetch the next prefetch_depth layers in the current direction (ascending
 * after an ascending call, descending otherwise).  views_out (host array of
 * n_tensors entries, may be NULL) receives device pointers for the layer's tensors
 * (others untouched); valid until zero_release_params(layer).  The caller's stream
 * is ordered after the gather.  Errors: ZERO_ESTATE at stages 0-2 or when the pool
 * is exhausted by unreleased layers; ZERO_EINVAL for an unknown layer. */
zero_status zero_gather_params(struct zero_ctx* ctx, uint32_t layer, void** views_out);
zero_status zero_release_params(struct zero_ctx* ctx, uint32_t layer);

/* Stages 0-2 (and stage 3 at LOCAL): device pointer of tensor t's 16-bit parameters
 * in the replica (contiguous numel elements; rewritten by every zero_step).
 * Errors: ZERO_EINVAL (bad tensor / zero-size tensor), ZERO_ESTATE (not bound, or
 * stage 3 with a collective transport: use zero_gather_params). */
zero_status zero_param_view(const struct zero_ctx* ctx, uint32_t tensor, void** p16);

/* Synchronous queries (they synchronize the compute stream when device data is read). */
enum {
  ZERO_Q_LAYOUT = 0,      /* out: zero_layout_info */
  ZERO_Q_MEMORY = 1,      /* out: zero_memory */
  ZERO_Q_COMM = 2,        /* out: zero_comm_counters */
  ZERO_Q_STEP = 3,        /* out: zero_step_info of the last step (synchronizes) */
  ZERO_Q_BUCKETS = 4,     /* out: zero_bucket[n_buckets] */
  ZERO_Q_PIECES = 5,      /* out: zero_piece[n_pieces] */
  ZERO_Q_STATE = 6,       /* out: zero_device_state (synchronizes) */
  ZERO_Q_TIMING = 7,      /* out: zero_timing, accumulated since the last TIMING query
                             (synchronizes; needs cfg.timing = 1), then reset */
  ZERO_Q_DECISION = 8     /* out: void*, the device address of the 16-byte decision
                             partial {double sum_sq, double overflow} that
                             zero_step_begin writes (see zero_step_begin) */
};
typedef struct {          /* persistent model-state bytes on this rank (Fig. 1 categories) */
  uint64_t params16, grads16, optimizer, reduced_grad_extra, staging, gather_pool, scratch;
} zero_memory;
typedef struct {          /* elements this rank sent, cumulative (S:173 CommStats) */
  uint64_t reduce_scatter, all_gather, all_reduce, steps;
} zero_comm_counters;
typedef struct {          /* device time per phase, CUDA events on the launching stream */
  double reduce_ms;       /* first flatten of a step -> last reduce-scatter/epilogue issued */
  double adam_ms;         /* the fused Adam kernel (sum over steps) */
  double step_ms;         /* zero_step: decision + Adam + all-gather */
  double ag_ms;           /* the all-gather after the Adam kernel (NCCL transport; ~0 when the
                             all-gather is fused into the Adam kernel's stores, PEER) */
  uint64_t steps;         /* steps accumulated */
  uint64_t kernel_launches;  /* library kernels launched (all, cumulative, never reset) */
  uint64_t adam_launches;
} zero_timing;
zero_status zero_query(const struct zero_ctx* ctx, int what, void* out, size_t out_bytes);
/* Turn the per-phase CUDA events of ZERO_Q_TIMING on (1) or off (0) from the next step on
 * (zero_config.timing sets the initial state).  Host-only; ZERO_ESTATE inside a step (after
 * its first zero_reduce_grads). */
zero_status zero_set_timing(struct zero_ctx* ctx, int on);

/* Last error text of ctx (NULL: of the calling thread's last failed zero_init or
 * zero_plan_layout).  The string is owned by the library and valid until the next
 * call on the same context. */
const char* zero_last_error(const struct zero_ctx* ctx);

/* Failure detection (a transport failure is an error naming the rank, not a
 * hang).  Blocks the host until every piece of work the context has issued so far (the
 * caller's stream and the library's streams) has completed, or timeout_ms elapsed.
 * NCCL transport: while waiting (and at the start of every NCCL-issuing call) the
 * communicator's asynchronous error is polled (ncclCommGetAsyncError); on an error, or
 * at the deadline with work outstanding, the communicator is aborted (ncclCommAbort --
 * the only way to release a hung collective; the borrowed communicator must then be
 * treated as destroyed by its owner) and the context is poisoned with a sticky
 * ZERO_ENCCL whose text names this rank.  Other transports: ZERO_ETIMEOUT at the
 * deadline (not sticky; the cross-process PEER spin-waits also trap after 300 s).
 * Errors: ZERO_ESTATE (not bound), ZERO_ECUDA (a device error surfaced). */
zero_status zero_wait(struct zero_ctx* ctx, uint64_t timeout_ms);
/* Synchronize the context's streams, close IPC mappings, destroy the library's
 * streams and events and free the context.  The caller's arenas are not freed.
 * Destroying one member of a simulated group dissolves the group. */
void zero_destroy(struct zero_ctx* ctx);

/* ---------------------------------------------------------------------------
 * P_a / P_a+cpu: partitioned activation checkpoints over a model-parallel group
 * (ZeRO-R, §6.1; communication P:486-498 §8).  Under tensor-slicing MP
 * every MP rank holds a replicated copy of each layer's input activation; P_a keeps
 * only this rank's 1/N_m slice of the checkpoint after the layer's forward and
 * re-materializes the replicated copy with an all-gather right before the
 * recompute in backward.  P_a+cpu keeps the slice in pinned host memory
 * and brings it back before the gather (2x the slice over PCIe).
 * The gather is, element for element, the saved activation (oracle/activation.py).
 *
 * Partition (reading R-Pa1): one checkpoint has `numel` 16-bit elements, padded to
 * `padded` = a multiple of N_m * 8; rank r keeps [r*slice, (r+1)*slice), slice =
 * padded / N_m (16-byte granules).
 * Transports: LOCAL (n_m == 1), PEER (zero_pa_sim_group: N_m contexts on one device;
 * the gather pulls every peer's slice with 128-bit loads) and NCCL (one process per
 * GPU: in-place ncclAllGather into a staging buffer, then a copy out).
 * Arenas (zero_pa_info): device = n_layers * slice * 2 B (P_a) or one slice staging
 * slot (P_a+cpu, PEER) or + `padded` staging elements (NCCL); host = n_layers * slice
 * * 2 B of pinned memory (P_a+cpu only; caller-allocated, e.g. torch pin_memory).
 * All calls are stream-ordered on the context's stream; errors as for zero_ctx
 * (ZERO_EINVAL bad argument, ZERO_ESTATE call order, ZERO_ECUDA/ENCCL sticky).
 * ------------------------------------------------------------------------- */
struct zero_pa_ctx;
typedef struct {
  uint64_t numel, padded, slice;          /* elements per checkpoint / padded / per rank */
  uint64_t device_bytes, host_bytes;      /* arenas the caller allocates */
  uint32_t n_layers, n_m, rank, offload;
} zero_pa_info;
typedef struct {                          /* cumulative counters */
  uint64_t saved_elems;                   /* elements this rank kept (its slices) */
  uint64_t gathered_elems;                /* elements received from other MP ranks */
  uint64_t d2h_bytes, h2d_bytes;          /* P_a+cpu PCIe traffic */
} zero_pa_counters;

/* numel: elements of one checkpoint (b*s*h); n_layers checkpoints (one per layer).
 * dtype FP16 | BF16.  offload: 0 = P_a, 1 = P_a+cpu.  transport/nccl_comm/stream as
 * for zero_init.  Errors: ZERO_EINVAL (n_m outside 1..ZERO_MAX_RANKS, rank >= n_m,
 * numel == 0, n_layers == 0, dtype, LOCAL with n_m > 1, NCCL without a comm). */
zero_status zero_pa_init(int n_m, int rank, uint32_t n_layers, uint64_t numel, zero_dtype dtype, int offload,
                         zero_transport transport, void* nccl_comm, void* stream, struct zero_pa_ctx** out);
zero_status zero_pa_get_info(const struct zero_pa_ctx* ctx, zero_pa_info* out);
/* Bind the caller's arenas (device: >= 256-B aligned, device_bytes; host: pinned,
 * host_bytes, NULL when 0).  The library never frees them. */
zero_status zero_pa_bind(struct zero_pa_ctx* ctx, void* device_arena, void* host_arena);
/* Link n PEER contexts of one process and device (rank r at index r, same numel,
 * n_layers, dtype, offload, stream, all bound) into an MP group. */
zero_status zero_pa_sim_group(struct zero_pa_ctx* const* ranks, int n);
/* After layer `layer`'s forward: keep this rank's slice of the checkpoint `act`
 * (device pointer, numel elements; borrowed until the stream work completes) in the
 * device store, or copy it to the host store (P_a+cpu).  Re-saving a layer
 * overwrites it. */
zero_status zero_pa_save(struct zero_pa_ctx* ctx, uint32_t layer, const void* act);
/* P_a+cpu: bring this rank's slice of `layer` back into the device staging slot
 * (H2D), ahead of the gather; every rank of the group must prefetch a layer before
 * any rank gathers it.  P_a: no-op.  ZERO_ESTATE if the layer was never saved. */
zero_status zero_pa_prefetch(struct zero_pa_ctx* ctx, uint32_t layer);
/* Before the recompute: write the replicated checkpoint of `layer` (numel elements)
 * into act_out (device).  ZERO_ESTATE if some rank of the group has not saved (P_a)
 * or prefetched (P_a+cpu) the layer. */
zero_status zero_pa_gather(struct zero_pa_ctx* ctx, uint32_t layer, void* act_out);
zero_status zero_pa_get_counters(const struct zero_pa_ctx* ctx, zero_pa_counters* out);
const char* zero_pa_last_error(const struct zero_pa_ctx* ctx);
/* Synchronize the stream and free the context (not the arenas); dissolves its group. */
void zero_pa_destroy(struct zero_pa_ctx* ctx);
/* P:419 closed form: per-GPU bytes of one checkpointed b x s x h activation per layer,
 * divided by the MP degree (P_a) -- floor(layers*batch*seq*hidden*elem_bytes / n_m). */
uint64_t zero_pa_checkpoint_bytes(uint64_t layers, uint64_t batch, uint64_t seq, uint64_t hidden, int n_m,
                                  int elem_bytes);

/* Pure host functions (no GPU): the closed forms the runtime reports against. */
/* Fig. 1 / Table 1: per-device model-state bytes for stage 0..3 (floor). */
uint64_t zero_model_state_bytes(uint64_t psi, int K, int n_d, int stage);
/* Elements each rank sends per step: 2 Psi'(N-1)/N (stages 0-2), 3 Psi'(N-1)/N (stage 3). */
uint64_t zero_comm_elems_per_rank(uint64_t psi_padded, int n_d, int stage);
int zero_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ZERO_B200_H */
