// Host engine of the ZeRO-DP hot path: layout, arenas, stage schedule, stream/event
// plan and the C ABI declared in include/zero_b200.h.  Citations "P:n" are lines of
// the paper; "c-k" are the readings in DESIGN.md §3.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <dlfcn.h>
#include <chrono>
#include <cstring>
#include <thread>
#include <map>
#include <string>
#include <vector>

#include "zero_b200.h"
#include "zero_internal.h"

using namespace zero;

namespace {

thread_local std::string g_init_error;

// NVTX range for the host-side issue of each phase (visible in nsys; header-only NVTX3,
// a no-op unless a tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

int to_dt(zero_dtype d) { return d == ZERO_FP16 ? DT_F16 : d == ZERO_BF16 ? DT_BF16 : DT_F32; }
uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------------------
// Layout (reading c-7): written from the rule in DESIGN.md §3, independently of the
// oracle.  Q = N*A, cap = floor(C_B/Q)*Q; a bucket never spans layers; a tensor that
// does not fit at the next A-aligned position is split at cap; buckets padded to Q.
// ---------------------------------------------------------------------------
struct LayoutResult {
  std::vector<zero_bucket> buckets;
  std::vector<zero_piece> pieces;
  zero_layout_info info{};
  std::string error;
};

bool plan(const zero_layout_desc* d, int n_d, LayoutResult& out) {
  if (!d || (d->n_tensors > 0 && !d->tensors)) { out.error = "null layout descriptor"; return false; }
  if (n_d < 1 || n_d > ZERO_MAX_RANKS) { out.error = "n_d out of range 1..8"; return false; }
  const uint64_t A = d->align_elems;
  if (A == 0 || (A & (A - 1))) { out.error = "align_elems must be a power of two"; return false; }
  const uint64_t Q = (uint64_t)n_d * A;
  uint64_t cap = 0;  // 0 = unlimited
  if (d->bucket_cap_elems) {
    if (d->bucket_cap_elems < Q) { out.error = "bucket_cap_elems < N_d * align_elems"; return false; }
    cap = d->bucket_cap_elems / Q * Q;
  }
  for (uint32_t t = 1; t < d->n_tensors; ++t)
    if (d->tensors[t].layer < d->tensors[t - 1].layer) { out.error = "layer ids must be non-decreasing"; return false; }

  // a bucket never spans layers, nor MP-replicated and MP-partitioned tensors (R-MP1)
  struct Cur { uint32_t layer, flags; uint64_t used; std::vector<zero_piece> p; } cur{0, 0, 0, {}};
  bool have_layer = false;
  std::vector<Cur> closed;
  auto close = [&](uint32_t next_layer) {
    if (cur.used > 0) closed.push_back(cur);
    cur = Cur{next_layer, 0, 0, {}};
  };
  uint64_t psi = 0;
  for (uint32_t t = 0; t < d->n_tensors; ++t) {
    const uint64_t n = d->tensors[t].numel;
    const uint32_t L = d->tensors[t].layer;
    const uint32_t F = d->tensors[t].flags & ZERO_TENSOR_MP_REPLICATED;
    if (n == 0) continue;
    psi += n;
    if (!have_layer) { cur.layer = L; have_layer = true; }
    if (cur.used > 0 && (L != cur.layer || F != cur.flags)) close(L);
    if (cur.used == 0) { cur.layer = L; cur.flags = F; }
    uint64_t rem = n, toff = 0;
    while (rem > 0) {
      const uint64_t start = align_up(cur.used, A);
      if (cap && start >= cap) { close(L); cur.flags = F; continue; }
      const uint64_t room = cap ? cap - start : rem;
      const uint64_t take = std::min(rem, room);
      cur.p.push_back(zero_piece{t, 0, toff, start, take});
      cur.used = start + take;
      rem -= take;
      toff += take;
      if (rem > 0) { close(L); cur.flags = F; }
    }
  }
  close(0);
  if (psi == 0) { out.error = "layout has no elements"; return false; }

  uint64_t base = 0, shard_off = 0, maxb = 0;
  std::map<uint32_t, int> layers;
  for (size_t k = 0; k < closed.size(); ++k) {
    zero_bucket b{};
    b.layer = closed[k].layer;
    b.flags = closed[k].flags;
    b.size = align_up(closed[k].used, Q);
    b.base = base;
    b.shard_off = shard_off;
    b.first_piece = (uint32_t)out.pieces.size();
    b.n_pieces = (uint32_t)closed[k].p.size();
    for (auto p : closed[k].p) { p.bucket = (uint32_t)k; out.pieces.push_back(p); }
    out.buckets.push_back(b);
    base += b.size;
    shard_off += b.size / n_d;
    maxb = std::max(maxb, b.size);
    layers[b.layer] = 1;
  }
  out.info.psi = psi;
  out.info.psi_padded = base;
  out.info.shard = base / n_d;
  out.info.n_buckets = (uint32_t)out.buckets.size();
  out.info.n_pieces = (uint32_t)out.pieces.size();
  out.info.n_layers = (uint32_t)layers.size();
  out.info.max_bucket = maxb > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)maxb;
  return true;
}

}  // namespace

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct ZeroGroup;

#define CK0(expr)                                                                             \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) return c->fail(ZERO_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

struct LayerInfo {
  uint32_t layer;
  uint32_t k0, k1;          // buckets [k0, k1)
  uint64_t flat0, flat1;    // global flat range
};

struct GatherSlot {
  int layer = -1;           // layer held (-1 free)
  bool released = true;
  cudaEvent_t ready = nullptr, freed = nullptr;
  uint64_t lru = 0;
};

struct zero_ctx {
  // configuration
  int n_d = 1, rank = 0, stage = 1;
  zero_config cfg{};
  zero_transport transport = ZERO_TRANSPORT_LOCAL;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;       // caller's compute stream
  cudaStream_t comm_stream = nullptr;  // library stream for NCCL work
  bool own_comm_stream = false;
  int pdt = DT_BF16, gdt = DT_BF16;
  bool r32 = false;                    // reduced gradient kept in fp32 (R32 and N_d > 1, or NCCL)
  bool wide = false;                   // R32 over NCCL: buckets flattened to fp32 (the RS sums fp32)

  // layout
  std::vector<zero_tensor> tensors;
  std::vector<zero_bucket> buckets;
  std::vector<zero_piece> pieces;
  zero_layout_info info{};
  std::vector<LayerInfo> layers;
  std::map<uint32_t, int> layer_index;
  std::vector<std::vector<FlatPiece>> flat_tmpl;   // per bucket: data + zero pieces (src = tensor id)
  std::vector<std::vector<uint32_t>> flat_tensor;  // per bucket: tensor id per flat piece (UINT32_MAX = zero)
  std::vector<std::vector<uint64_t>> flat_toff;    // per bucket: tensor offset per flat piece
  std::vector<int> slot_base;                      // per bucket: first epilogue slot
  int n_slots = 0;
  std::vector<uint64_t> tensor_flat;               // tensor -> global flat offset of element 0
  uint64_t S_e = 0;                                // elements this rank updates
  uint64_t opt_stride = 0;                         // S_e rounded up to 64 (256-B aligned m, v)
  uint64_t max_layer = 0;
  uint32_t pool = 2;

  // arenas
  zero_sizes sizes{};
  zero_buffers bufs{};
  bool bound = false;
  float *p32 = nullptr, *m = nullptr, *v = nullptr;
  uint16_t* p16 = nullptr;
  uint16_t* grad = nullptr;
  void* gred = nullptr;
  uint16_t* gather = nullptr;
  DevState* st = nullptr;
  Slot* slots = nullptr;
  double* cta_sum = nullptr;                       // per-CTA epilogue partials per slot (flatten at N_d = 1,
                                                   // reduce-scatter at N_d > 1)
  uint32_t* cta_flag = nullptr;
  uint32_t* cta_grid = nullptr;
  bool flat_pdl = false;                           // ZERO_FLAT_PDL: one flatten stream, PDL-chained launches
  bool flat_cta_partials = true;                   // ZERO_FLAT_CTA_PARTIALS=0: last-CTA combine in each flatten
  bool rs_cta_partials = true;                     // ZERO_RS_CTA_PARTIALS=0: last-CTA combine in each reduce-scatter
  int rs_ctas = 4, rs_u = 0;                       // ZERO_RS_CTAS (CTAs per SM), ZERO_RS_U (0 = per-N default)
  int gather_grid = 0;                             // ZERO_GATHER_GRID: cap on a stage-3 layer gather's CTAs per
                                                   // source rank (0 = none; NVLink-bound, overlaps the forward)
  int rs_grid = 0;                                 // ZERO_RS_GRID: cap on the pull's CTAs per launch (0 = none;
                                                   // an NVLink-bound pull needs few SMs: the sweep knob for NVL8)
  int rs_pipe = 1;                                 // ZERO_RS_PIPE: 1 = software-pipelined pull (default), 0 = plain
  bool rs_multi = true;                            // ZERO_RS_MULTI=0: simulated ranks' pulls launched per rank
  // ZeRO x MP (R-MP1): per-slot norm weights (0 for MP-replicated buckets on MP rank > 0)
  double* slot_w = nullptr;
  std::vector<double> slot_w_host;
  bool use_slot_w = false;
  RankPartial* dp_partial = nullptr;               // zero_step_begin's data-parallel sum
  bool step_begun = false;
  int pend_ev = -1;
  GridPartials* part_compute = nullptr;
  GridPartials* part_flat[4] = {};                 // grid partials per flatten stream
  // LOCAL / NCCL: flattens of consecutive buckets alternate between two library streams
  // forked from the caller's stream, so one bucket's tail overlaps the next one's
  // start; they are joined into the step (zero_step) -- gradient buffers are
  // therefore borrowed until zero_step is enqueued.
  static constexpr int kMaxFlatStreams = 4;
  int n_flat_streams = 3;                          // ZERO_FLAT_STREAMS (1..4; 3 measured best)
  int n_flat_streams_req = 3;
  cudaStream_t flat_stream[kMaxFlatStreams] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[kMaxFlatStreams] = {};
  uint32_t flat_rr = 0;
  bool flat_used[kMaxFlatStreams] = {};
  GridPartials* part_comm = nullptr;
  RankPartial* my_partial = nullptr;
  RankPartial* gathered = nullptr;
  AdamSeg* segs = nullptr;
  std::vector<AdamSeg> segs_host;
  bool segs_aligned8 = true;                       // every segment offset/count % 8 == 0
  int sms = 148;
  int adam_variant = 21;                           // ZERO_ADAM_VARIANT (tuning; 21 = TMA in/out, 4096 x 2 stages)
  bool adam_variant_env = false;
  uint64_t adam_small = 1ull << 21;                // ZERO_ADAM_SMALL: shards up to this size use the
                                                   // register-staged 4-CTA/SM kernel (latency-bound sizes)
  int flat_vecs = 4, flat_ctas = 4;                // ZERO_FLAT_VECS / ZERO_FLAT_CTAS
  int flat_tma = 0;                                // ZERO_FLAT_TMA: 0 off, else the TMA variant

  // LOCAL: adjacent small buckets are flattened by one launch, issued at the next bucket that
  // does not join the run or at zero_step (the gradients are borrowed until zero_step anyway)
  int pend_lo = -1, pend_hi = -1;
  std::vector<std::pair<uint32_t, FlatPiece>> pend_pieces;  // (bucket, piece with its source resolved)
  uint64_t small_bucket = 1ull << 20;              // ZERO_SMALL_BUCKET (elements; 0 = never batch)
  bool step_small = false;                         // ZERO_STEP_SMALL=1: a small model's step as one cooperative
                                                   // launch (measured slower: 26 vs 24 us at 1M params, the two
                                                   // grid barriers cost more than the launch they save)
  int step_small_ctas = 0;                         // ZERO_STEP_SMALL_CTAS: grid cap of that launch (0 = occupancy)
  bool fused_pending = false;                      // this zero_step runs as one cooperative launch
  bool adam_pdl = false;                           // the Adam follows the whole-step flatten on its stream
  bool adam_pdl_ok = true;                         // ZERO_ADAM_PDL=0: never launch the Adam with PDL
  int step_small_grid = -1;                        // co-resident grid limit of that kernel (-1: not queried)

  // per-step tracking
  std::vector<uint8_t> reduced;
  uint32_t n_reduced = 0;
  std::vector<int> pool_pending;                   // per pool slot: bucket awaiting its RS (-1 none)
  std::vector<const void*> grad_ptrs;
  std::vector<cudaEvent_t> ev_pool_free;           // NCCL: RS of the slot's last bucket done
  cudaEvent_t ev_flat = nullptr, ev_step = nullptr;
  bool stepped_this_round = false;

  // stage 3
  // cross-process PEER: layer gathers run on their own stream (pipelined, spread
  // over the forward and backward), ordered by ev_params (the shards are final: after a
  // load or a step's end barrier) and each slot's freed event; the caller's stream waits
  // on the slot's ready event
  cudaStream_t gather_stream = nullptr;
  cudaEvent_t ev_params = nullptr, ev_gjoin = nullptr;
  std::vector<GatherSlot> gslots;
  std::vector<int> layer_slot;                     // layer index -> gather slot (-1)
  int last_layer = -1;
  int direction = +1;
  uint64_t lru_clock = 0;

  ZeroGroup* group = nullptr;
  zero_comm_counters counters{};

  // cross-process PEER (CUDA IPC) peer table
  bool ipc = false;
  uint16_t* peer_grad[ZERO_MAX_RANKS] = {};
  uint16_t* peer_p16[ZERO_MAX_RANKS] = {};
  char* peer_scratch[ZERO_MAX_RANKS] = {};
  std::vector<void*> ipc_mapped;                   // bases to cudaIpcCloseMemHandle
  std::vector<std::pair<int, uint64_t>> pool_last; // per pool slot: (bucket, epoch) of its last use
  size_t off_sig_flat = 0, off_sig_rs = 0, off_sig_part = 0, off_sig_adam = 0, off_gathered = 0;
  size_t off_sig_hello = 0, off_hello_result = 0;
  uint64_t epoch() const { return counters.steps + 1; }
  uint64_t* sig(int r, size_t off, size_t idx) const {  // signal slot in rank r's scratch
    return reinterpret_cast<uint64_t*>(peer_scratch[r] + off) + idx;
  }

  // phase timing (cfg.timing): one event set per step, reused from a pool
  struct StepEvents { cudaEvent_t r0 = nullptr, r1 = nullptr, a0 = nullptr, a1 = nullptr, g1 = nullptr, s1 = nullptr; };
  std::vector<StepEvents> ev_pool;
  size_t ev_used = 0;
  bool step_open = false;          // a reduce phase began (r0 recorded)
  uint64_t launches = 0, adam_launches = 0;
  zero_status timing_events(StepEvents** out);

  zero_status sticky = ZERO_OK;
  std::string err;
  const void* rec_host = nullptr;                  // the last zero_step host_out and its device alias
  void* rec_dev = nullptr;
  bool comm_aborted = false;                       // the NCCL watchdog aborted the communicator
  cudaEvent_t ev_wait[kMaxFlatStreams + 3] = {};   // zero_wait: one per stream the context uses

  zero_status fail(zero_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    err = buf;
    if (s == ZERO_ECUDA || s == ZERO_ENCCL) sticky = s;
    return s;
  }

  // destinations ------------------------------------------------------------
  uint64_t slice(uint32_t k) const { return buckets[k].size / n_d; }
  uint16_t* flat_dst(uint32_t k) const {       // where bucket k is flattened
    const zero_bucket& b = buckets[k];
    if (stage <= 1) return grad + b.base;
    if (transport == ZERO_TRANSPORT_LOCAL) return reinterpret_cast<uint16_t*>(gred) + b.shard_off;
    return grad + (uint64_t)(k % pool) * maxB;
  }
  void* flat_dst_any(uint32_t k) const {       // as flat_dst; fp32 pool slots for R32 over NCCL
    if (wide) return reinterpret_cast<float*>(grad) + (uint64_t)(k % pool) * maxB;
    return flat_dst(k);
  }
  // where bucket k's reduced slice (this rank's) lives
  void* rs_dst(uint32_t k) const {
    const zero_bucket& b = buckets[k];
    if (r32) return reinterpret_cast<float*>(gred) + b.shard_off;
    if (stage <= 1) return grad + b.base + (uint64_t)rank * slice(k);
    return reinterpret_cast<uint16_t*>(gred) + b.shard_off;
  }
  uint64_t maxB = 0;
};

zero_status zero_ctx::timing_events(StepEvents** out) {
  zero_ctx* c = this;
  if (ev_used == ev_pool.size()) {
    StepEvents e;
    CK0(cudaEventCreate(&e.r0));
    CK0(cudaEventCreate(&e.r1));
    CK0(cudaEventCreate(&e.a0));
    CK0(cudaEventCreate(&e.a1));
    CK0(cudaEventCreate(&e.g1));
    CK0(cudaEventCreate(&e.s1));
    ev_pool.push_back(e);
  }
  *out = &ev_pool[ev_used];
  return ZERO_OK;
}

// A PEER group of contexts sharing one device and one stream (config 1's simulated
// ranks).  Collective steps are issued once every member reached them.
struct ZeroGroup {
  int n = 0;
  zero_ctx* ranks[ZERO_MAX_RANKS] = {};
  std::vector<int> flat_count;   // per bucket: ranks that flattened it this step
  uint32_t reduced_buckets = 0;  // buckets whose pull reduce-scatter was issued
  int stepped = 0;               // ranks that ran zero_step this round
};

namespace {

#define CK(expr)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) return c->fail(ZERO_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)
#define NK(expr)                                                                              \
  do {                                                                                        \
    ncclResult_t r_ = (expr);                                                                 \
    if (r_ != ncclSuccess) return c->fail(ZERO_ENCCL, "%s: %s", #expr, ncclGetErrorString(r_)); \
  } while (0)
#define STICKY(c)                                  \
  do {                                             \
    if (!(c)) return ZERO_EINVAL;                  \
    if ((c)->sticky != ZERO_OK) return (c)->sticky; \
  } while (0)

ncclDataType_t nccl_dt(int dt) { return dt == DT_F16 ? ncclFloat16 : dt == DT_BF16 ? ncclBfloat16 : ncclFloat32; }

// NCCL failure handling ("transport failure -> protocol error with rank id"):
// a failed or hung collective is unblocked only by aborting its communicator, after which
// the context is poisoned with a sticky ZERO_ENCCL naming this rank
zero_status abort_comm(zero_ctx* c, const char* why) {
  if (c->comm && !c->comm_aborted) {
    ncclCommAbort(c->comm);
    c->comm_aborted = true;
  }
  return c->fail(ZERO_ENCCL, "rank %d of %d: %s; the communicator was aborted", c->rank, c->n_d, why);
}
// cheap host-side poll of the communicator's asynchronous error (every NCCL-issuing call)
zero_status poll_nccl(zero_ctx* c) {
  if (c->transport != ZERO_TRANSPORT_NCCL || !c->comm || c->comm_aborted) return ZERO_OK;
  ncclResult_t ae = ncclSuccess;
  const ncclResult_t r = ncclCommGetAsyncError(c->comm, &ae);
  if (r != ncclSuccess) ae = r;
  if (ae != ncclSuccess && ae != ncclInProgress) {
    char why[160];
    snprintf(why, sizeof(why), "asynchronous NCCL error: %s", ncclGetErrorString(ae));
    return abort_comm(c, why);
  }
  return ZERO_OK;
}

int grid_for(uint64_t work_items, int per_sm, int sms) {
  const uint64_t cap = (uint64_t)per_sm * sms;
  uint64_t g = work_items < cap ? work_items : cap;
  if (g < 1) g = 1;
  if (g > (uint64_t)kMaxGrid) g = kMaxGrid;
  return (int)g;
}

// the reduce-scatter's epilogue destination for bucket k (per-CTA partials or grid combine),
// its loads-in-flight knob and its grid
int rs_setup(const zero_ctx* c, uint32_t k, RSArgs& a, uint64_t sl) {
  const int slot = c->slot_base[k];
  if (c->rs_cta_partials) {
    a.cta_sum = c->cta_sum + (size_t)slot * kMaxGrid;
    a.cta_flag = c->cta_flag + (size_t)slot * kMaxGrid;
    a.cta_grid = c->cta_grid + slot;
  }
  a.u = c->rs_u;
  a.pipe = c->rs_pipe;
  const int g = grid_for((sl + 2047) / 2048, c->rs_ctas, c->sms);
  return c->rs_grid > 0 ? std::min(g, c->rs_grid) : g;   // grid-stride body: any grid is exact
}

DecideParams decide_params(const zero_ctx* c);

// the device-visible alias of the caller's pinned step record (UVA-mapped pinned memory), or
// NULL (pageable memory: the record is copied D2H at the end of the step instead)
void* mapped_record(zero_ctx* c, const void* host_out) {
  if (!host_out) return nullptr;
  if (host_out != c->rec_host) {
    cudaPointerAttributes at{};
    c->rec_dev = nullptr;
    if (cudaPointerGetAttributes(&at, host_out) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer)
      c->rec_dev = at.devicePointer;
    cudaGetLastError();   // a pageable pointer is not an error
    c->rec_host = host_out;
  }
  return c->rec_dev;
}

// the rank's {sum of squares, overflow} partial from the per-bucket epilogue results;
// *decided (N_d = 1, zero_step): the same launch also made the step's decision
cudaError_t issue_decide_local(zero_ctx* c, cudaStream_t s, bool* decided = nullptr, void* rec_dev = nullptr) {
  const bool cp = c->transport == ZERO_TRANSPORT_LOCAL ? c->flat_cta_partials : c->rs_cta_partials;
  const double* w = c->use_slot_w ? c->slot_w : nullptr;
  c->launches++;
  if (cp && c->n_slots <= kMaxGrid) {   // one CTA per slot, last CTA combines (part_compute is free here)
    DecideParams p = decide_params(c);
    p.rec_out = rec_dev;
    if (decided) *decided = true;
    return launch_decide_local_slots(c->n_slots, c->my_partial, s, w, c->cta_sum, c->cta_flag, c->cta_grid,
                                     c->part_compute, decided ? c->st : nullptr, decided ? &p : nullptr);
  }
  return launch_decide_local(c->slots, c->n_slots, c->my_partial, s, w, cp ? c->cta_sum : nullptr,
                             cp ? c->cta_flag : nullptr, cp ? c->cta_grid : nullptr);
}

// bytes of the scratch arena and the offsets inside it
struct ScratchLayout {
  size_t st, slots, part_compute, part_flat2, part_flat3, part_flat4, part_comm, my_partial, gathered, segs, sig_flat, sig_rs, sig_part, sig_adam,
      sig_hello, hello_result, cta_sum, cta_flag, cta_grid, slot_w, dp_partial, total;
};
// sig_flat[k][r] / sig_rs[k][r]: epoch at which rank r flattened / finished reducing bucket k
// sig_part[r] / sig_adam[r]: epoch at which rank r published its partial / finished Adam
// per-CTA epilogue partials for every slot (k_decide_local): the flatten's at N_d == 1,
// the reduce-scatter's (first slot of each bucket) at N_d > 1
ScratchLayout scratch_layout(int n_slots, size_t n_segs, size_t n_buckets) {
  ScratchLayout s{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
  s.st = take(sizeof(DevState));
  s.slots = take(sizeof(Slot) * (size_t)std::max(n_slots, 1));
  s.part_compute = take(sizeof(GridPartials));
  s.part_flat2 = take(sizeof(GridPartials));
  s.part_flat3 = take(sizeof(GridPartials));
  s.part_flat4 = take(sizeof(GridPartials));
  s.part_comm = take(sizeof(GridPartials));
  s.my_partial = take(sizeof(RankPartial));
  s.gathered = take(sizeof(RankPartial) * ZERO_MAX_RANKS);
  s.segs = take(sizeof(AdamSeg) * std::max<size_t>(n_segs, 1));
  s.sig_flat = take(sizeof(uint64_t) * ZERO_MAX_RANKS * std::max<size_t>(n_buckets, 1));
  s.sig_rs = take(sizeof(uint64_t) * ZERO_MAX_RANKS * std::max<size_t>(n_buckets, 1));
  s.sig_part = take(sizeof(uint64_t) * ZERO_MAX_RANKS);
  s.sig_adam = take(sizeof(uint64_t) * ZERO_MAX_RANKS);
  s.sig_hello = take(sizeof(uint64_t) * ZERO_MAX_RANKS);   // zero_peer_open's handshake
  s.hello_result = take(sizeof(uint32_t));
  const size_t ns = (size_t)std::max(n_slots, 1);
  s.cta_sum = take(sizeof(double) * kMaxGrid * ns);
  s.cta_flag = take(sizeof(uint32_t) * kMaxGrid * ns);
  s.cta_grid = take(sizeof(uint32_t) * ns);
  s.slot_w = take(sizeof(double) * (size_t)std::max(n_slots, 1));
  s.dp_partial = take(sizeof(RankPartial));
  s.total = o;
  return s;
}

zero_status create_flat_streams(zero_ctx* c) {
  if (c->n_flat_streams <= 1) return ZERO_OK;
  for (int i = 0; i < c->n_flat_streams; ++i) {
    if (c->flat_stream[i]) continue;
    CK(cudaStreamCreateWithFlags(&c->flat_stream[i], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->ev_join[i], cudaEventDisableTiming));
  }
  if (!c->ev_fork) CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  return ZERO_OK;
}

}  // namespace

extern "C" {

int zero_abi_version(void) { return ZERO_ABI_VERSION; }

zero_status zero_plan_layout(const zero_layout_desc* desc, int n_d, zero_layout_info* info, zero_bucket* buckets,
                             uint32_t cap_buckets, zero_piece* pieces, uint32_t cap_pieces) {
  LayoutResult r;
  if (!plan(desc, n_d, r)) { g_init_error = r.error; return ZERO_EINVAL; }
  if (info) *info = r.info;
  if (buckets) {
    if (cap_buckets < r.info.n_buckets) return ZERO_EINVAL;
    std::memcpy(buckets, r.buckets.data(), sizeof(zero_bucket) * r.buckets.size());
  }
  if (pieces) {
    if (cap_pieces < r.info.n_pieces) return ZERO_EINVAL;
    std::memcpy(pieces, r.pieces.data(), sizeof(zero_piece) * r.pieces.size());
  }
  return ZERO_OK;
}

uint64_t zero_model_state_bytes(uint64_t psi, int K, int n_d, int stage) {
  // Fig. 1 / P:360, P:369, P:397 -- exact in 128-bit, floored.
  using u128 = unsigned __int128;
  if (n_d < 1) return 0;
  const u128 p = psi, k = (u128)K, n = (u128)n_d;
  switch (stage) {
    case 0: return (uint64_t)((4 + k) * p);
    case 1: return (uint64_t)((4 * p * n + k * p) / n);
    case 2: return (uint64_t)((2 * p * n + (2 + k) * p) / n);
    case 3: return (uint64_t)(((4 + k) * p) / n);
    default: return 0;
  }
}

uint64_t zero_comm_elems_per_rank(uint64_t psi_padded, int n_d, int stage) {
  // P:445, P:473 (2 Psi) and P:476-478 (3 Psi) with the exact ring factor (N-1)/N.
  if (n_d < 1) return 0;
  const uint64_t one = psi_padded / (uint64_t)n_d * (uint64_t)(n_d - 1);
  return stage == 3 ? 3 * one : 2 * one;
}

zero_status zero_init(const zero_layout_desc* desc, int n_d, int rank, int stage, int K, const zero_config* cfg,
                      zero_transport transport, void* nccl_comm, void* compute_stream, zero_ctx** out) {
  g_init_error.clear();
  auto bad = [&](const char* why) { g_init_error = why; return ZERO_EINVAL; };
  if (!out || !cfg) return bad("null argument");
  *out = nullptr;
  if (K != 12) return bad("K must be 12 (mixed-precision Adam, P:266)");
  if (stage < 0 || stage > 3) return bad("stage must be 0..3");
  if (n_d < 1 || n_d > ZERO_MAX_RANKS || rank < 0 || rank >= n_d) return bad("rank/n_d out of range");
  if (cfg->param_dtype != ZERO_FP16 && cfg->param_dtype != ZERO_BF16) return bad("param_dtype must be FP16 or BF16");
  if (cfg->grad_dtype != cfg->param_dtype && cfg->grad_dtype != ZERO_FP32) return bad("grad_dtype must equal param_dtype or be FP32");
  if (cfg->reduce_mode != ZERO_R16 && cfg->reduce_mode != ZERO_R32) return bad("reduce_mode");
  if (!(cfg->lr > 0.f) || !(cfg->beta1 >= 0.f && cfg->beta1 < 1.f) || !(cfg->beta2 >= 0.f && cfg->beta2 < 1.f) ||
      !(cfg->eps > 0.f))
    return bad("Adam hyper-parameters out of range");
  if (!(cfg->loss_scale > 0.f) || !(cfg->grad_prescale > 0.f)) return bad("loss_scale and grad_prescale must be > 0");
  if (cfg->dynamic_loss_scale && (cfg->scale_window == 0 || !(cfg->min_loss_scale > 0.f)))
    return bad("dynamic loss scaling needs scale_window > 0 and min_loss_scale > 0");
  if (transport == ZERO_TRANSPORT_LOCAL && n_d != 1) return bad("LOCAL transport requires n_d == 1");
  if (transport == ZERO_TRANSPORT_NCCL && !nccl_comm) return bad("NCCL transport requires a communicator");
  if (transport != ZERO_TRANSPORT_LOCAL && transport != ZERO_TRANSPORT_NCCL && transport != ZERO_TRANSPORT_PEER)
    return bad("unknown transport");
  // R32 at N_d = 1 is R16 (one value rounded to 16-bit is itself), except on a 1-rank NCCL
  // communicator, which keeps the fp32 collective path so that it can be tested on one GPU
  const bool r32 = cfg->reduce_mode == ZERO_R32 && (n_d > 1 || transport == ZERO_TRANSPORT_NCCL);
  if (r32 && stage == 0) { g_init_error = "stage 0 supports R16 only"; return ZERO_EUNSUPPORTED; }
  if (r32 && transport == ZERO_TRANSPORT_NCCL && stage == 1) {
    g_init_error = "R32 over NCCL needs stage 2 or 3 (fp32 staging pool); stage 1 reduces in place in its 16-bit buffer";
    return ZERO_EUNSUPPORTED;
  }

  LayoutResult L;
  if (!plan(desc, n_d, L)) return bad(L.error.c_str());

  zero_ctx* c = new zero_ctx();
  c->n_d = n_d;
  c->rank = rank;
  c->stage = stage;
  c->cfg = *cfg;
  if (c->cfg.prefetch_depth == 0) c->cfg.prefetch_depth = 1;
  c->pool = c->cfg.pool_buckets ? c->cfg.pool_buckets : 2;
  // n_d == 1 degenerates to LOCAL, except NCCL with a real (1-rank) communicator, which
  // keeps the collective code path (used to test it on one GPU)
  c->transport = (n_d == 1 && transport != ZERO_TRANSPORT_NCCL) ? ZERO_TRANSPORT_LOCAL : transport;
  const bool coll = c->transport != ZERO_TRANSPORT_LOCAL;
  c->comm = reinterpret_cast<ncclComm_t>(nccl_comm);
  c->stream = reinterpret_cast<cudaStream_t>(compute_stream);
  c->pdt = to_dt(cfg->param_dtype);
  c->gdt = to_dt(cfg->grad_dtype);
  c->r32 = r32;
  c->wide = r32 && c->transport == ZERO_TRANSPORT_NCCL;
  c->tensors.assign(desc->tensors, desc->tensors + desc->n_tensors);
  c->buckets = L.buckets;
  c->pieces = L.pieces;
  c->info = L.info;
  for (auto& b : c->buckets) c->maxB = std::max(c->maxB, b.size);

  // tensor -> flat offset (split tensors are contiguous: split points are multiples of Q)
  c->tensor_flat.assign(c->tensors.size(), UINT64_MAX);
  for (auto& p : c->pieces)
    if (p.tensor_off == 0) c->tensor_flat[p.tensor] = c->buckets[p.bucket].base + p.bucket_off;

  // layers
  for (uint32_t k = 0; k < c->info.n_buckets; ++k) {
    const zero_bucket& b = c->buckets[k];
    auto it = c->layer_index.find(b.layer);
    if (it == c->layer_index.end()) {
      c->layer_index[b.layer] = (int)c->layers.size();
      c->layers.push_back(LayerInfo{b.layer, k, k + 1, b.base, b.base + b.size});
    } else {
      LayerInfo& li = c->layers[it->second];
      li.k1 = k + 1;
      li.flat1 = b.base + b.size;
    }
  }
  for (auto& li : c->layers) c->max_layer = std::max(c->max_layer, li.flat1 - li.flat0);

  // flatten templates: data pieces + zero pieces covering [0, B_k) exactly
  c->flat_tmpl.resize(c->info.n_buckets);
  c->flat_tensor.resize(c->info.n_buckets);
  c->flat_toff.resize(c->info.n_buckets);
  c->slot_base.resize(c->info.n_buckets);
  int slots = 0;
  for (uint32_t k = 0; k < c->info.n_buckets; ++k) {
    const zero_bucket& b = c->buckets[k];
    uint64_t pos = 0;
    auto add = [&](const void* tensor_tag, uint32_t tensor, uint64_t toff, uint64_t off, uint64_t n) {
      FlatPiece fp{};
      fp.src = tensor_tag;
      fp.dst_off = off;
      fp.count = n;
      c->flat_tmpl[k].push_back(fp);
      c->flat_tensor[k].push_back(tensor);
      c->flat_toff[k].push_back(toff);
    };
    for (uint32_t j = 0; j < b.n_pieces; ++j) {
      const zero_piece& p = c->pieces[b.first_piece + j];
      if (p.bucket_off > pos) add(nullptr, UINT32_MAX, 0, pos, p.bucket_off - pos);
      add(nullptr, p.tensor, p.tensor_off, p.bucket_off, p.count);
      pos = p.bucket_off + p.count;
    }
    if (pos < b.size) add(nullptr, UINT32_MAX, 0, pos, b.size - pos);
    c->slot_base[k] = slots;
    slots += (int)((c->flat_tmpl[k].size() + kMaxFlatPieces - 1) / kMaxFlatPieces);
  }
  c->n_slots = slots;
  c->slot_w_host.assign((size_t)std::max(slots, 1), 1.0);
  for (uint32_t k = 0; k < c->info.n_buckets; ++k) {
    const int s1 = k + 1 < c->info.n_buckets ? c->slot_base[k + 1] : slots;
    if ((c->buckets[k].flags & ZERO_TENSOR_MP_REPLICATED) && c->cfg.mp_rank != 0)
      for (int s = c->slot_base[k]; s < s1; ++s) { c->slot_w_host[s] = 0.0; c->use_slot_w = true; }
  }

  // Adam segments over this rank's local index space
  c->S_e = stage == 0 ? c->info.psi_padded : c->info.shard;
  for (uint32_t k = 0; k < c->info.n_buckets; ++k) {
    const zero_bucket& b = c->buckets[k];
    const uint64_t sl = b.size / n_d;
    AdamSeg s{};
    if (stage == 0) {
      s.local_off = b.base;
      s.count = b.size;
      s.g_off = b.base;
      s.p16_off = b.base;
    } else {
      s.local_off = b.shard_off;
      s.count = sl;
      const uint64_t mine = b.base + (uint64_t)rank * sl;
      s.g_off = (stage == 1 && !r32) ? mine : b.shard_off;
      s.p16_off = stage == 3 ? b.shard_off : mine;
    }
    c->segs_host.push_back(s);
    if ((s.local_off | s.g_off | s.p16_off | s.count) & 7) c->segs_aligned8 = false;
  }

  // arena sizes (zero_sizes doc in the header)
  const uint64_t P = c->info.psi_padded, S = c->info.shard;
  zero_sizes& z = c->sizes;
  c->opt_stride = align_up(c->S_e, 64);
  z.opt_bytes = 12ull * c->opt_stride;
  z.opt_stride_elems = c->opt_stride;
  z.p16_bytes = 2ull * (stage == 3 ? S : P);
  if (stage <= 1) z.grad_bytes = 2ull * P;
  else z.grad_bytes = coll ? (c->wide ? 4ull : 2ull) * c->pool * c->maxB : 0;
  if (stage >= 2) z.gred_bytes = (r32 ? 4ull : 2ull) * S;
  else z.gred_bytes = r32 ? 4ull * S : 0;
  z.gather_bytes = (stage == 3 && coll) ? 2ull * (c->cfg.prefetch_depth + 1) * c->max_layer : 0;
  z.scratch_bytes =
      scratch_layout(c->n_slots, c->segs_host.size(), c->buckets.size()).total;

  c->reduced.assign(c->info.n_buckets, 0);
  c->pool_pending.assign(c->pool, -1);
  c->grad_ptrs.assign(c->tensors.size(), nullptr);
  c->layer_slot.assign(c->layers.size(), -1);
  *out = c;
  return ZERO_OK;
}

zero_status zero_buffer_sizes(const zero_ctx* c, zero_sizes* out) {
  if (!c || !out) return ZERO_EINVAL;
  *out = c->sizes;
  return ZERO_OK;
}

zero_status zero_bind_buffers(zero_ctx* c, const zero_buffers* b) {
  STICKY(c);
  if (!b) return ZERO_EINVAL;
  if (c->bound) return c->fail(ZERO_ESTATE, "buffers already bound");
  const zero_sizes& z = c->sizes;
  auto need = [&](const void* p, uint64_t bytes, const char* name) -> bool {
    if (bytes == 0) return true;
    if (!p) { c->fail(ZERO_EINVAL, "arena %s (%llu bytes) is NULL", name, (unsigned long long)bytes); return false; }
    if (reinterpret_cast<uintptr_t>(p) & 255) { c->fail(ZERO_EINVAL, "arena %s is not 256-byte aligned", name); return false; }
    return true;
  };
  if (!need(b->opt, z.opt_bytes, "opt") || !need(b->p16, z.p16_bytes, "p16") || !need(b->grad, z.grad_bytes, "grad") ||
      !need(b->gred, z.gred_bytes, "gred") || !need(b->gather, z.gather_bytes, "gather") ||
      !need(b->scratch, z.scratch_bytes, "scratch"))
    return ZERO_EINVAL;
  c->bufs = *b;
  c->p32 = reinterpret_cast<float*>(b->opt);
  c->m = c->p32 + c->opt_stride;
  c->v = c->m + c->opt_stride;
  c->p16 = reinterpret_cast<uint16_t*>(b->p16);
  c->grad = reinterpret_cast<uint16_t*>(b->grad);
  c->gred = b->gred;
  c->gather = reinterpret_cast<uint16_t*>(b->gather);
  const ScratchLayout sl =
      scratch_layout(c->n_slots, c->segs_host.size(), c->buckets.size());
  char* s = reinterpret_cast<char*>(b->scratch);
  c->st = reinterpret_cast<DevState*>(s + sl.st);
  c->slots = reinterpret_cast<Slot*>(s + sl.slots);
  c->slot_w = reinterpret_cast<double*>(s + sl.slot_w);
  c->dp_partial = reinterpret_cast<RankPartial*>(s + sl.dp_partial);
  c->cta_sum = reinterpret_cast<double*>(s + sl.cta_sum);
  c->cta_flag = reinterpret_cast<uint32_t*>(s + sl.cta_flag);
  c->cta_grid = reinterpret_cast<uint32_t*>(s + sl.cta_grid);
  c->part_compute = reinterpret_cast<GridPartials*>(s + sl.part_compute);
  c->part_flat[0] = c->part_compute;
  c->part_flat[1] = reinterpret_cast<GridPartials*>(s + sl.part_flat2);
  c->part_flat[2] = reinterpret_cast<GridPartials*>(s + sl.part_flat3);
  c->part_flat[3] = reinterpret_cast<GridPartials*>(s + sl.part_flat4);
  c->part_comm = reinterpret_cast<GridPartials*>(s + sl.part_comm);
  c->my_partial = reinterpret_cast<RankPartial*>(s + sl.my_partial);
  c->gathered = reinterpret_cast<RankPartial*>(s + sl.gathered);
  c->segs = reinterpret_cast<AdamSeg*>(s + sl.segs);
  c->off_sig_flat = sl.sig_flat;
  c->off_sig_rs = sl.sig_rs;
  c->off_sig_part = sl.sig_part;
  c->off_sig_adam = sl.sig_adam;
  c->off_sig_hello = sl.sig_hello;
  c->off_hello_result = sl.hello_result;
  c->off_gathered = sl.gathered;
  c->pool_last.assign(c->pool, std::make_pair(-1, (uint64_t)0));
  c->sms = sm_count();
  if (const char* ev = getenv("ZERO_ADAM_VARIANT")) { c->adam_variant = atoi(ev); c->adam_variant_env = true; }
  if (const char* ev = getenv("ZERO_ADAM_SMALL")) c->adam_small = strtoull(ev, nullptr, 10);
  if (const char* ev = getenv("ZERO_FLAT_VECS")) c->flat_vecs = atoi(ev);
  if (const char* ev = getenv("ZERO_FLAT_CTAS")) c->flat_ctas = atoi(ev);
  if (const char* ev = getenv("ZERO_FLAT_TMA")) c->flat_tma = atoi(ev);
  if (c->flat_vecs != 2 && c->flat_vecs != 4 && c->flat_vecs != 8) c->flat_vecs = 4;
  if (c->flat_ctas < 1 || c->flat_ctas > 8) c->flat_ctas = 4;

  // streams and events
  if (c->transport == ZERO_TRANSPORT_NCCL) {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi));
    c->own_comm_stream = true;
    c->ev_pool_free.assign(c->pool, nullptr);
    for (auto& e : c->ev_pool_free) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  } else {
    c->comm_stream = c->stream;
  }
  if (const char* ev = getenv("ZERO_FLAT_CTA_PARTIALS")) c->flat_cta_partials = atoi(ev) != 0;
  if (const char* ev = getenv("ZERO_RS_CTA_PARTIALS")) c->rs_cta_partials = atoi(ev) != 0;
  c->rs_ctas = c->n_d == 8 ? 3 : 4;   // the pipelined pull at N_d = 8 holds 78 registers: 3 CTAs/SM
  if (const char* ev = getenv("ZERO_RS_CTAS")) c->rs_ctas = std::max(1, std::min(8, atoi(ev)));
  if (const char* ev = getenv("ZERO_RS_GRID")) c->rs_grid = std::max(0, std::min(kMaxGrid, atoi(ev)));
  if (const char* ev = getenv("ZERO_GATHER_GRID")) c->gather_grid = std::max(0, std::min(kMaxGrid, atoi(ev)));
  if (const char* ev = getenv("ZERO_RS_U")) c->rs_u = atoi(ev);
  if (const char* ev = getenv("ZERO_RS_PIPE")) c->rs_pipe = atoi(ev);
  if (const char* ev = getenv("ZERO_RS_MULTI")) c->rs_multi = atoi(ev) != 0;
  if (const char* ev = getenv("ZERO_SMALL_BUCKET")) c->small_bucket = strtoull(ev, nullptr, 10);
  if (const char* ev = getenv("ZERO_STEP_SMALL")) c->step_small = atoi(ev) != 0;
  if (const char* ev = getenv("ZERO_ADAM_PDL")) c->adam_pdl_ok = atoi(ev) != 0;
  if (const char* ev = getenv("ZERO_STEP_SMALL_CTAS")) c->step_small_ctas = atoi(ev);
  if (const char* ev = getenv("ZERO_FLAT_STREAMS"))
    c->n_flat_streams = std::max(1, std::min(zero_ctx::kMaxFlatStreams, atoi(ev)));
  if (const char* ev = getenv("ZERO_FLAT_PDL")) c->flat_pdl = atoi(ev) != 0 && c->transport == ZERO_TRANSPORT_LOCAL;
  if (c->flat_pdl) {
    // PDL chains the flattens on ONE stream and lets consecutive grids overlap: they must not
    // share a last-CTA combine (grid_publish's ticket and per-CTA sums), so each launch keeps
    // its own per-CTA partials
    c->n_flat_streams = 1;
    c->flat_cta_partials = true;
  }
  c->n_flat_streams_req = c->n_flat_streams;
  // simulated PEER ranks share one stream (host-ordered collectives); zero_peer_open
  // switches a cross-process PEER context to forked flatten streams + a comm stream
  if (c->transport == ZERO_TRANSPORT_PEER) c->n_flat_streams = 1;
  zero_status fs_status = create_flat_streams(c);
  if (fs_status != ZERO_OK) return fs_status;
  CK(cudaEventCreateWithFlags(&c->ev_flat, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_step, cudaEventDisableTiming));
  if (c->stage == 3) {
    CK(cudaEventCreateWithFlags(&c->ev_params, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_gjoin, cudaEventDisableTiming));
    c->gslots.resize(c->cfg.prefetch_depth + 1);
    for (auto& g : c->gslots) {
      CK(cudaEventCreateWithFlags(&g.ready, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&g.freed, cudaEventDisableTiming));
    }
  }

  // zero every arena (padding must hold 0, c-7), upload the segment table, init state
  const void* ptrs[6] = {b->opt, b->p16, b->grad, b->gred, b->gather, b->scratch};
  const uint64_t sz[6] = {z.opt_bytes, z.p16_bytes, z.grad_bytes, z.gred_bytes, z.gather_bytes, z.scratch_bytes};
  for (int i = 0; i < 6; ++i)
    if (sz[i]) CK(cudaMemsetAsync(const_cast<void*>(ptrs[i]), 0, sz[i], c->stream));
  CK(cudaMemcpyAsync(c->slot_w, c->slot_w_host.data(), sizeof(double) * c->slot_w_host.size(), cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaMemcpyAsync(c->segs, c->segs_host.data(), sizeof(AdamSeg) * c->segs_host.size(), cudaMemcpyHostToDevice,
                     c->stream));
  const float inv = (float)(1.0 / ((double)c->n_d * (double)c->cfg.loss_scale * (double)c->cfg.grad_prescale));
  CK(launch_init_state(c->st, c->cfg.loss_scale, inv, c->stream));
  c->launches++;
  // the segment table is read from host memory by the async copy: wait for it
  CK(cudaStreamSynchronize(c->stream));
  c->bound = true;
  return ZERO_OK;
}

zero_status zero_load_master(zero_ctx* c, const void* const* tensor_master) {
  STICKY(c);
  if (!c->bound) return c->fail(ZERO_ESTATE, "buffers not bound");
  if (!tensor_master) return c->fail(ZERO_EINVAL, "tensor_master is NULL");
  CK(cudaMemsetAsync(c->m, 0, 8ull * c->opt_stride, c->stream));  // m and v are contiguous
  for (uint32_t k = 0; k < c->info.n_buckets; ++k) {
    const zero_bucket& b = c->buckets[k];
    const uint64_t sl = b.size / c->n_d;
    for (uint32_t j = 0; j < b.n_pieces; ++j) {
      const zero_piece& p = c->pieces[b.first_piece + j];
      if (!tensor_master[p.tensor]) continue;  // loaded by another call (chunked init)
      LoadArgs a{};
      a.src = reinterpret_cast<const float*>(tensor_master[p.tensor]) + p.tensor_off;
      a.count = p.count;
      a.flat_off = b.base + p.bucket_off;
      if (c->stage == 0) {
        a.own_lo = b.base;
        a.own_hi = b.base + b.size;
        a.local_base = b.base;
      } else {
        a.own_lo = b.base + (uint64_t)c->rank * sl;
        a.own_hi = a.own_lo + sl;
        a.local_base = b.shard_off;
      }
      a.p32 = c->p32;
      a.p16 = c->p16;
      a.p16_mode = c->stage == 3 ? 1 : 0;
      a.p_dtype = c->pdt;
      CK(launch_load(a, c->stream));
      c->launches++;
    }
  }
  const float inv = (float)(1.0 / ((double)c->n_d * (double)c->cfg.loss_scale * (double)c->cfg.grad_prescale));
  CK(launch_init_state(c->st, c->cfg.loss_scale, inv, c->stream));
  c->launches++;
  if (c->ev_params) CK(cudaEventRecord(c->ev_params, c->stream));   // the shards are written
  return ZERO_OK;
}

}  // extern "C"

namespace {
// the global range of bucket k this rank owns and its shard offset (stage 0: all of it)
void owned_range(const zero_ctx* c, uint32_t k, uint64_t& lo, uint64_t& hi, uint64_t& local) {
  const zero_bucket& b = c->buckets[k];
  if (c->stage == 0) {
    lo = b.base;
    hi = b.base + b.size;
    local = b.base;
  } else {
    const uint64_t sl = b.size / c->n_d;
    lo = b.base + (uint64_t)c->rank * sl;
    hi = lo + sl;
    local = b.shard_off;
  }
}

zero_status shard_io(zero_ctx* c, void* const* arrs, float* shard, int to_shard) {
  for (uint32_t k = 0; k < c->info.n_buckets; ++k) {
    const zero_bucket& b = c->buckets[k];
    uint64_t lo, hi, local;
    owned_range(c, k, lo, hi, local);
    for (uint32_t j = 0; j < b.n_pieces; ++j) {
      const zero_piece& p = c->pieces[b.first_piece + j];
      if (!arrs[p.tensor]) continue;
      ShardIOArgs a{};
      a.tensor = reinterpret_cast<float*>(arrs[p.tensor]) + p.tensor_off;
      a.shard = shard;
      a.count = p.count;
      a.flat_off = b.base + p.bucket_off;
      a.own_lo = lo;
      a.own_hi = hi;
      a.local_base = local;
      a.to_shard = to_shard;
      CK(launch_shard_io(a, c->stream));
      c->launches++;
    }
  }
  return ZERO_OK;
}
}  // namespace

extern "C" {

zero_status zero_export_state(zero_ctx* c, void* const* master, void* const* m, void* const* v) {
  STICKY(c);
  if (!c->bound) return c->fail(ZERO_ESTATE, "buffers not bound");
  void* const* arrs[3] = {master, m, v};
  float* shards[3] = {c->p32, c->m, c->v};
  for (int i = 0; i < 3; ++i) {
    if (!arrs[i]) continue;
    zero_status s = shard_io(c, arrs[i], shards[i], 0);
    if (s != ZERO_OK) return s;
  }
  return ZERO_OK;
}

zero_status zero_import_state(zero_ctx* c, const void* const* master, const void* const* m, const void* const* v,
                              const zero_device_state* st) {
  STICKY(c);
  if (!c->bound) return c->fail(ZERO_ESTATE, "buffers not bound");
  if (st && !(st->loss_scale > 0.0f)) return c->fail(ZERO_EINVAL, "loss_scale must be > 0");
  if (master) {  // owned fp32 elements + the 16-bit copy derived from them (as zero_load_master)
    for (uint32_t k = 0; k < c->info.n_buckets; ++k) {
      const zero_bucket& b = c->buckets[k];
      uint64_t lo, hi, local;
      owned_range(c, k, lo, hi, local);
      for (uint32_t j = 0; j < b.n_pieces; ++j) {
        const zero_piece& p = c->pieces[b.first_piece + j];
        if (!master[p.tensor]) continue;
        LoadArgs a{};
        a.src = reinterpret_cast<const float*>(master[p.tensor]) + p.tensor_off;
        a.count = p.count;
        a.flat_off = b.base + p.bucket_off;
        a.own_lo = lo;
        a.own_hi = hi;
        a.local_base = local;
        a.p32 = c->p32;
        a.p16 = c->p16;
        a.p16_mode = c->stage == 3 ? 1 : 0;
        a.p_dtype = c->pdt;
        CK(launch_load(a, c->stream));
        c->launches++;
      }
    }
  }
  const void* const* arrs[2] = {m, v};
  float* shards[2] = {c->m, c->v};
  for (int i = 0; i < 2; ++i) {
    if (!arrs[i]) continue;
    zero_status s = shard_io(c, const_cast<void* const*>(arrs[i]), shards[i], 1);
    if (s != ZERO_OK) return s;
  }
  if (st) {
    const float inv = (float)(1.0 / ((double)c->n_d * (double)st->loss_scale * (double)c->cfg.grad_prescale));
    CK(launch_set_state(c->st, st->b1t, st->b2t, st->t, st->loss_scale, st->good_steps, inv, c->stream));
    c->launches++;
  }
  if (c->ev_params) CK(cudaEventRecord(c->ev_params, c->stream));
  return ZERO_OK;
}

zero_status zero_set_grad_ptrs(zero_ctx* c, const void* const* g) {
  STICKY(c);
  if (!g) return c->fail(ZERO_EINVAL, "null pointer array");
  c->grad_ptrs.assign(g, g + c->tensors.size());
  return ZERO_OK;
}

}  // extern "C"

namespace {

// issue the flatten of bucket k (compute stream).  epilogue at N_d == 1.
zero_status issue_flatten(zero_ctx* c, uint32_t k, const void* const* grads, cudaStream_t fs, GridPartials* part) {
  const auto& tmpl = c->flat_tmpl[k];
  void* dst = c->flat_dst_any(k);
  const int ebytes = c->gdt == DT_F32 ? 4 : 2;
  const bool epi = c->transport == ZERO_TRANSPORT_LOCAL;
  int slot = c->slot_base[k];
  for (size_t b0 = 0; b0 < tmpl.size(); b0 += kMaxFlatPieces, ++slot) {
    FlatArgs a{};
    const size_t b1 = std::min(tmpl.size(), b0 + kMaxFlatPieces);
    for (size_t j = b0; j < b1; ++j) {
      FlatPiece fp = tmpl[j];
      const uint32_t t = c->flat_tensor[k][j];
      if (t != UINT32_MAX) {
        const char* base = reinterpret_cast<const char*>(grads[t]);
        if (!base) return c->fail(ZERO_EINVAL, "gradient pointer of tensor %u is NULL", t);
        fp.src = base + c->flat_toff[k][j] * ebytes;
      } else {
        fp.src = nullptr;
      }
      a.pieces[j - b0] = fp;
    }
    a.n_pieces = (int)(b1 - b0);
    const uint64_t total = tmpl[b1 - 1].dst_off + tmpl[b1 - 1].count - tmpl[b0].dst_off;
    // TMA staging needs 16-B granules: every piece boundary and source % 8 elements
    bool tma_ok = c->flat_tma > 0 && !c->wide && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
    for (int j = 0; tma_ok && j < (int)(b1 - b0); ++j) {
      const FlatPiece& fp = a.pieces[j];
      if ((fp.dst_off | fp.count) & 7) tma_ok = false;
      if (fp.src && (reinterpret_cast<uintptr_t>(fp.src) & 15)) tma_ok = false;
    }
    const int grid = grid_for((total + 2047) / 2048, tma_ok ? flatten_tma_ctas_per_sm(c->flat_tma) : c->flat_ctas, c->sms);
    a.per_cta = align_up((total + grid - 1) / grid, 8);
    a.src_dtype = c->gdt;
    a.dst_dtype = c->pdt;
    a.epilogue = epi ? 1 : 0;
    a.dst = dst;
    a.sigma = c->cfg.grad_prescale;
    a.st = c->st;
    a.part = part;
    a.slot = c->slots + slot;
    if (epi && c->cta_sum && c->flat_cta_partials) {
      a.cta_sum = c->cta_sum + (size_t)slot * kMaxGrid;
      a.cta_flag = c->cta_flag + (size_t)slot * kMaxGrid;
      a.cta_grid = c->cta_grid + slot;
    }
    // chain behind the previous launch of this step's reduce phase on the same stream
    a.pdl = (c->flat_pdl && (c->n_reduced > 0 || b0 > 0)) ? 1 : 0;
    if (c->wide) CK(launch_flatten_wide(a, grid, fs));
    else if (tma_ok) CK(launch_flatten_tma(a, grid, fs, c->flat_tma));
    else CK(launch_flatten(a, grid, fs, c->flat_vecs));
    c->launches++;
  }
  return ZERO_OK;
}

// the stream a flatten is issued on: the caller's, or the next forked flatten stream
zero_status pick_flat_stream(zero_ctx* c, cudaStream_t* fs, GridPartials** fpart) {
  *fs = c->stream;
  *fpart = c->part_compute;
  if (c->n_flat_streams > 1) {
    const int i = (int)(c->flat_rr++ % (uint32_t)c->n_flat_streams);
    *fs = c->flat_stream[i];
    *fpart = c->part_flat[i];
    CK(cudaEventRecord(c->ev_fork, c->stream));
    CK(cudaStreamWaitEvent(*fs, c->ev_fork, 0));
    c->flat_used[i] = true;
  }
  return ZERO_OK;
}

bool batchable(const zero_ctx* c, uint32_t k) {
  return c->transport == ZERO_TRANSPORT_LOCAL && c->small_bucket && c->buckets[k].size <= c->small_bucket &&
         c->flat_tmpl[k].size() <= (size_t)kMaxFlatPieces && c->flat_cta_partials && !c->flat_pdl && !c->flat_tma &&
         !c->use_slot_w;
}

// one launch for the pending run of adjacent small buckets [pend_lo, pend_hi] (N_d = 1): their
// pieces tile [base_lo, base_hi + B_hi) contiguously; the epilogue partials go to the first
// bucket's slot and the run's other slots are cleared
// the pending run's flatten arguments (pieces in bucket order, relative to the run's first
// bucket); returns the run's element count.  per_cta is left to the caller (grid-dependent)
uint64_t pending_flat_args(zero_ctx* c, FlatArgs& a) {
  std::stable_sort(c->pend_pieces.begin(), c->pend_pieces.end(),
                   [](const std::pair<uint32_t, FlatPiece>& x, const std::pair<uint32_t, FlatPiece>& y) {
                     return x.first < y.first;
                   });
  const uint32_t lo = (uint32_t)c->pend_lo, hi = (uint32_t)c->pend_hi;
  const uint64_t base_lo = c->buckets[lo].base;
  a = FlatArgs{};
  a.n_pieces = (int)c->pend_pieces.size();
  for (int j = 0; j < a.n_pieces; ++j) {
    FlatPiece fp = c->pend_pieces[j].second;
    fp.dst_off += c->buckets[c->pend_pieces[j].first].base - base_lo;
    a.pieces[j] = fp;
  }
  const int slot = c->slot_base[lo];
  a.src_dtype = c->gdt;
  a.dst_dtype = c->pdt;
  a.epilogue = 1;
  a.dst = c->flat_dst(lo);
  a.sigma = c->cfg.grad_prescale;
  a.st = c->st;
  a.slot = c->slots + slot;
  a.cta_sum = c->cta_sum + (size_t)slot * kMaxGrid;
  a.cta_flag = c->cta_flag + (size_t)slot * kMaxGrid;
  a.cta_grid = c->cta_grid + slot;
  a.clear_slots = (uint32_t)(c->slot_base[hi] - slot);   // one slot per batchable bucket
  return c->buckets[hi].base + c->buckets[hi].size - base_lo;
}

zero_status flush_small(zero_ctx* c, bool on_caller_stream = false, bool* decided = nullptr, void* rec_dev = nullptr) {
  if (c->pend_lo < 0) return ZERO_OK;
  const uint32_t lo = (uint32_t)c->pend_lo, hi = (uint32_t)c->pend_hi;
  FlatArgs a;
  const uint64_t total = pending_flat_args(c, a);
  cudaStream_t fs = c->stream;
  GridPartials* fpart = c->part_compute;
  if (!on_caller_stream)
    if (zero_status s = pick_flat_stream(c, &fs, &fpart)) return s;
  const int grid = grid_for((total + 2047) / 2048, c->flat_ctas, c->sms);
  a.per_cta = align_up((total + grid - 1) / grid, 8);
  a.part = fpart;
  // the whole step in this launch (zero_step, a small model): its last CTA also decides
  if (decided && lo == 0 && hi + 1 == c->info.n_buckets && c->n_slots == (int)c->info.n_buckets) {
    a.decide_st = c->st;
    a.decide_out = c->my_partial;
    a.decide_part = c->part_comm;
    a.decide = decide_params(c);
    a.decide.rec_out = rec_dev;
    *decided = true;
    c->adam_pdl = on_caller_stream && c->adam_pdl_ok;   // the Adam comes next on this stream
  }
  CK(launch_flatten(a, grid, fs, c->flat_vecs));
  c->launches++;
  c->pend_lo = c->pend_hi = -1;
  c->pend_pieces.clear();
  return ZERO_OK;
}

// N_d = 1, a small model whose every bucket is in the pending run: the whole step can be one
// cooperative launch (flatten + epilogue, decision, Adam), unless a variant is forced, the
// stream is being captured, or the kernel's co-resident grid is too small
int step_small_grid(zero_ctx* c, StepSmallArgs* out, void* rec_dev);

bool fused_step_ok(zero_ctx* c) {
  if (c->transport != ZERO_TRANSPORT_LOCAL || !c->step_small || c->adam_variant_env) return false;
  if (c->pend_lo != 0 || c->pend_hi + 1 != (int)c->info.n_buckets || c->n_slots != (int)c->info.n_buckets) return false;
  if (c->S_e > c->adam_small) return false;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(c->stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return false;
  }
  return step_small_grid(c, nullptr, nullptr) > 0;
}

// the fused step's arguments and grid (0: not launchable)
int step_small_grid(zero_ctx* c, StepSmallArgs* out, void* rec_dev) {
  StepSmallArgs a{};
  const uint64_t total = pending_flat_args(c, a.f);
  a.f.decide_part = c->part_comm;            // the grid barrier's words
  AdamArgs& d = a.adam;
  d.p32 = c->p32;
  d.m = c->m;
  d.v = c->v;
  d.G = (c->stage <= 1) ? (const void*)c->grad : (const void*)c->gred;
  d.g_dtype = c->pdt;
  d.p_dtype = c->pdt;
  d.n_p16 = 1;
  d.p16[0] = c->p16;
  d.segs = c->segs;
  d.n_segs = (int)c->segs_host.size();
  d.total = c->S_e;
  d.beta1 = c->cfg.beta1;
  d.beta2 = c->cfg.beta2;
  d.eps = c->cfg.eps;
  d.omb1 = 1.0f - c->cfg.beta1;
  d.omb2 = 1.0f - c->cfg.beta2;
  d.wd = c->cfg.weight_decay > 0.0f ? 1 : 0;
  d.lrwd = (float)((double)c->cfg.lr * (double)c->cfg.weight_decay);
  d.st = c->st;
  a.dp = decide_params(c);
  a.dp.rec_out = rec_dev;
  a.st = c->st;
  a.out = c->my_partial;
  if (c->step_small_grid < 0) c->step_small_grid = step_small_max_grid(a);
  const uint64_t want = std::max<uint64_t>(std::max<uint64_t>((total + 2047) / 2048, (c->S_e + 2047) / 2048), 1);
  int cap = std::min(c->step_small_grid, kMaxGrid);
  if (c->step_small_ctas > 0) cap = std::min(cap, c->step_small_ctas);
  const int grid = (int)std::min<uint64_t>(want, (uint64_t)cap);
  if (grid <= 0) return 0;
  a.f.per_cta = align_up((total + grid - 1) / grid, 8);
  d.per_cta = align_up((c->S_e + grid - 1) / grid, 8);
  if (out) *out = a;
  return grid;
}

// LOCAL, small bucket k: join (or start) the pending run; the sources are resolved now
zero_status defer_small(zero_ctx* c, uint32_t k, const void* const* grads) {
  const auto& tmpl = c->flat_tmpl[k];
  const bool adjacent = c->pend_lo >= 0 && (k + 1 == (uint32_t)c->pend_lo || k == (uint32_t)c->pend_hi + 1);
  const uint64_t run = adjacent ? std::max(c->buckets[k].base + c->buckets[k].size,
                                           c->buckets[c->pend_hi].base + c->buckets[c->pend_hi].size) -
                                      std::min(c->buckets[k].base, c->buckets[c->pend_lo].base)
                                : 0;
  if (!adjacent || c->pend_pieces.size() + tmpl.size() > (size_t)kMaxFlatPieces || run > 4 * c->small_bucket)
    if (zero_status s = flush_small(c)) return s;
  const int ebytes = c->gdt == DT_F32 ? 4 : 2;
  for (size_t j = 0; j < tmpl.size(); ++j) {
    FlatPiece fp = tmpl[j];
    const uint32_t t = c->flat_tensor[k][j];
    if (t != UINT32_MAX) {
      const char* base = reinterpret_cast<const char*>(grads[t]);
      if (!base) return c->fail(ZERO_EINVAL, "gradient pointer of tensor %u is NULL", t);
      fp.src = base + c->flat_toff[k][j] * ebytes;
    }
    c->pend_pieces.emplace_back(k, fp);
  }
  if (c->pend_lo < 0) c->pend_lo = c->pend_hi = (int)k;
  c->pend_lo = std::min(c->pend_lo, (int)k);
  c->pend_hi = std::max(c->pend_hi, (int)k);
  return ZERO_OK;
}

// pull reduce-scatter of bucket k for rank c (PEER), sources = every member's flattened bucket
int fill_pull_rs(zero_ctx* c, ZeroGroup* g, uint32_t k, RSArgs& a) {
  const uint64_t sl = c->slice(k);
  a = RSArgs{};
  for (int j = 0; j < g->n; ++j) a.src[j] = g->ranks[j]->flat_dst(k) + (uint64_t)c->rank * sl;
  a.dst = c->rs_dst(k);
  a.count = sl;
  a.n = g->n;
  a.dtype = c->pdt;
  a.r32 = c->r32 ? 1 : 0;
  a.reduce = 1;
  a.st = c->st;
  a.part = c->part_comm;
  a.slot = c->slots + c->slot_base[k];
  return rs_setup(c, k, a, sl);
}

// simulated ranks: every rank's pull of bucket k in one launch (they share the stream and run
// concurrently, as they would on separate GPUs); per-rank launches when not eligible
zero_status issue_pull_rs_all(ZeroGroup* g, uint32_t k) {
  RSMulti m{};
  m.n = g->n;
  int grid = 0;
  for (int j = 0; j < g->n; ++j) grid = fill_pull_rs(g->ranks[j], g, k, m.r[j]);
  zero_ctx* c = g->ranks[0];
  const cudaError_t e = c->rs_multi ? launch_reduce_scatter_multi(m, grid, c->comm_stream) : cudaErrorNotSupported;
  if (e == cudaSuccess) {
    c->launches++;
  } else if (e == cudaErrorNotSupported) {
    cudaGetLastError();
    for (int j = 0; j < g->n; ++j) {
      zero_ctx* cj = g->ranks[j];
      if (launch_reduce_scatter(m.r[j], grid, cj->comm_stream) != cudaSuccess)
        return cj->fail(ZERO_ECUDA, "pull reduce-scatter launch failed");
      cj->launches++;
    }
  } else {
    return c->fail(ZERO_ECUDA, "pull reduce-scatter launch failed: %s", cudaGetErrorString(e));
  }
  for (int j = 0; j < g->n; ++j)
    g->ranks[j]->counters.reduce_scatter += g->ranks[j]->slice(k) * (uint64_t)(g->n - 1);
  return ZERO_OK;
}

zero_status finish_bucket_local(zero_ctx* c, uint32_t k) {
  c->reduced[k] = 1;
  c->n_reduced++;
  return ZERO_OK;
}

}  // namespace

extern "C" {

zero_status zero_reduce_grads(zero_ctx* c, uint32_t k, const void* const* tensor_grads) {
  STICKY(c);
  NvtxRange nvtx("zero_reduce_grads");
  if (!c->bound) return c->fail(ZERO_ESTATE, "buffers not bound");
  if (zero_status ps = poll_nccl(c)) return ps;
  if (k >= c->info.n_buckets) return c->fail(ZERO_EINVAL, "bucket %u out of range", k);
  if (c->reduced[k]) return c->fail(ZERO_ESTATE, "bucket %u already reduced this step", k);
  if (c->transport == ZERO_TRANSPORT_PEER && !c->group && !c->ipc)
    return c->fail(ZERO_ESTATE, "PEER context neither in a group nor linked by zero_peer_open");
  const void* const* grads = tensor_grads ? tensor_grads : c->grad_ptrs.data();

  // C_B pool slot reuse (stages 2/3, N_d > 1)
  const bool pooled = c->stage >= 2 && c->transport != ZERO_TRANSPORT_LOCAL;
  const uint32_t ps = pooled ? k % c->pool : 0;
  if (pooled && c->transport == ZERO_TRANSPORT_PEER && c->group) {
    const int pend = c->pool_pending[ps];
    if (pend >= 0 && c->group->flat_count[pend] < c->group->n)
      return c->fail(ZERO_ESTATE, "pool slot %u still holds bucket %d awaiting its reduce-scatter", ps, pend);
  }
  if (c->cfg.timing && !c->step_open && c->ev_used < 4096) {
    zero_ctx::StepEvents* ev;
    zero_status es = c->timing_events(&ev);
    if (es != ZERO_OK) return es;
    CK(cudaEventRecord(ev->r0, c->stream));
    c->step_open = true;
  }
  if (batchable(c, k)) {   // N_d = 1, small bucket: flattened together with its neighbours
    if (zero_status s = defer_small(c, k, grads)) return s;
    return finish_bucket_local(c, k);
  }
  if (c->transport == ZERO_TRANSPORT_LOCAL)
    if (zero_status s = flush_small(c)) return s;
  // the stream this bucket is flattened on: the caller's, or one of the forked streams
  cudaStream_t fs;
  GridPartials* fpart;
  if (zero_status s = pick_flat_stream(c, &fs, &fpart)) return s;
  if (pooled && c->transport == ZERO_TRANSPORT_NCCL) CK(cudaStreamWaitEvent(fs, c->ev_pool_free[ps], 0));
  if (pooled && c->ipc) {  // every peer finished reading this slot's previous bucket
    const auto& pl = c->pool_last[ps];
    if (pl.first >= 0) {
      WaitArgs w{c->sig(c->rank, c->off_sig_rs, (size_t)pl.first * ZERO_MAX_RANKS), c->n_d, pl.second};
      CK(launch_wait(w, fs));
      c->launches++;
    }
  }
  zero_status s = issue_flatten(c, k, grads, fs, fpart);
  if (s != ZERO_OK) return s;

  if (c->transport == ZERO_TRANSPORT_LOCAL) return finish_bucket_local(c, k);

  if (c->ipc) {  // cross-process PEER: signal "flattened", pull-reduce my slice, signal "read done"
    const uint64_t ep = c->epoch();
    const size_t kk = (size_t)k * ZERO_MAX_RANKS;
    SigArgs sa{};
    for (int j = 0; j < c->n_d; ++j) sa.dst[j] = c->sig(j, c->off_sig_flat, kk + c->rank);
    sa.n = c->n_d;
    sa.epoch = ep;
    CK(launch_signal(sa, fs));
    c->launches++;
    // the reduce-scatter starts only after the local flatten (a host-side stream
    // dependency), so its CTAs spin only on remote ranks' flatten signals
    CK(cudaEventRecord(c->ev_flat, fs));
    CK(cudaStreamWaitEvent(c->comm_stream, c->ev_flat, 0));
    const uint64_t sl = c->slice(k);
    const size_t foff = (size_t)(c->flat_dst(k) - c->grad);
    RSArgs a{};
    for (int j = 0; j < c->n_d; ++j) {
      a.src[j] = c->peer_grad[j] + foff + (uint64_t)c->rank * sl;
      a.done_sig[j] = c->sig(j, c->off_sig_rs, kk + c->rank);
    }
    a.wait_flags = c->sig(c->rank, c->off_sig_flat, kk);
    a.epoch = ep;
    a.dst = c->rs_dst(k);
    a.count = sl;
    a.n = c->n_d;
    a.dtype = c->pdt;
    a.r32 = c->r32 ? 1 : 0;
    a.reduce = 1;
    a.st = c->st;
    a.part = c->part_comm;
    a.slot = c->slots + c->slot_base[k];
    CK(launch_reduce_scatter(a, rs_setup(c, k, a, sl), c->comm_stream));
    c->launches++;
    c->counters.reduce_scatter += sl * (uint64_t)(c->n_d - 1);
    if (c->stage == 0) {  // all-reduce = RS + AG of the reduced slices
      WaitArgs w{c->sig(c->rank, c->off_sig_rs, kk), c->n_d, ep};
      CK(launch_wait(w, c->comm_stream));
      c->launches++;
      CopyArgs ca{};
      const zero_bucket& b = c->buckets[k];
      for (int i = 0; i < c->n_d; ++i) {
        ca.src[i] = c->peer_grad[i] + b.base + (uint64_t)i * sl;
        ca.dst[i] = c->grad + b.base + (uint64_t)i * sl;
      }
      for (int i = 0; i < c->n_d; ++i) ca.count[i] = sl;
      ca.n = c->n_d;
      CK(launch_copy(ca, grid_for((sl + 2047) / 2048, 2, c->sms), c->comm_stream));
      c->launches++;
      c->counters.all_gather += sl * (uint64_t)(c->n_d - 1);
    }
    if (pooled) c->pool_last[ps] = std::make_pair((int)k, ep);
    return finish_bucket_local(c, k);
  }

  if (c->transport == ZERO_TRANSPORT_PEER) {
    ZeroGroup* g = c->group;
    if (pooled) c->pool_pending[ps] = (int)k;
    c->reduced[k] = 1;  // this rank's part is done; the collective completes below
    if (++g->flat_count[k] == g->n) {
      zero_status r = issue_pull_rs_all(g, k);
      if (r != ZERO_OK) return r;
      if (c->stage == 0) {  // all-reduce = RS + AG of the reduced slices
        for (int j = 0; j < g->n; ++j) {
          zero_ctx* cj = g->ranks[j];
          CopyArgs a{};
          const uint64_t sl = cj->slice(k);
          for (int i = 0; i < g->n; ++i) {
            a.src[i] = g->ranks[i]->grad + cj->buckets[k].base + (uint64_t)i * sl;
            a.dst[i] = cj->grad + cj->buckets[k].base + (uint64_t)i * sl;
          }
          for (int i = 0; i < g->n; ++i) a.count[i] = sl;
          a.n = g->n;
          zero_ctx* cc = cj;
          if (launch_copy(a, grid_for((sl + 2047) / 2048, 2, cc->sms), cc->comm_stream) != cudaSuccess)
            return cc->fail(ZERO_ECUDA, "pull all-gather launch failed");
          cc->launches++;
          cj->counters.all_gather += sl * (uint64_t)(g->n - 1);
        }
      }
      for (int j = 0; j < g->n; ++j) g->ranks[j]->n_reduced++;
      if (++g->reduced_buckets == c->info.n_buckets) {
        for (int j = 0; j < g->n; ++j) {
          zero_ctx* cj = g->ranks[j];
          if (issue_decide_local(cj, cj->comm_stream) != cudaSuccess)
            return cj->fail(ZERO_ECUDA, "decide_local launch failed");
        }
      }
    }
    return ZERO_OK;
  }

  // NCCL: the flatten stream produced the bucket; the comm stream reduces it
  CK(cudaEventRecord(c->ev_flat, fs));
  CK(cudaStreamWaitEvent(c->comm_stream, c->ev_flat, 0));
  const zero_bucket& b = c->buckets[k];
  const uint64_t sl = c->slice(k);
  const ncclDataType_t dt = c->wide ? ncclFloat32 : nccl_dt(c->pdt);
  if (c->stage == 0) {
    NK(ncclAllReduce(c->grad + b.base, c->grad + b.base, b.size, dt, ncclSum, c->comm, c->comm_stream));
    c->counters.all_reduce += 2 * sl * (uint64_t)(c->n_d - 1);
  } else {
    // R16: 16-bit wire, NCCL rounds partial sums to 16-bit; R32: fp32 wire (2x bytes), fp32 sums
    NK(ncclReduceScatter(c->flat_dst_any(k), c->rs_dst(k), sl, dt, ncclSum, c->comm, c->comm_stream));
    c->counters.reduce_scatter += sl * (uint64_t)(c->n_d - 1);
  }
  RSArgs a{};
  a.dst = c->stage == 0 ? (void*)(c->grad + b.base + (uint64_t)c->rank * sl) : c->rs_dst(k);
  a.count = sl;
  a.n = c->n_d;
  a.dtype = c->pdt;
  a.r32 = c->r32 ? 1 : 0;
  a.reduce = 0;
  a.st = c->st;
  a.part = c->part_comm;
  a.slot = c->slots + c->slot_base[k];
  CK(launch_reduce_scatter(a, rs_setup(c, k, a, sl), c->comm_stream));
  c->launches++;
  if (pooled) CK(cudaEventRecord(c->ev_pool_free[ps], c->comm_stream));
  return finish_bucket_local(c, k);
}

}  // extern "C"

namespace {

zero_status issue_adam(zero_ctx* c, ZeroGroup* g) {
  AdamArgs a{};
  a.p32 = c->p32;
  a.m = c->m;
  a.v = c->v;
  const bool g_in_grad = c->stage == 0 || (c->stage == 1 && !c->r32);
  a.G = g_in_grad ? (const void*)c->grad : (const void*)c->gred;
  a.g_dtype = c->r32 ? DT_F32 : c->pdt;
  a.p_dtype = c->pdt;
  if (g && (c->stage == 1 || c->stage == 2)) {  // fused all-gather: store into every replica
    a.n_p16 = g->n;
    for (int j = 0; j < g->n; ++j) a.p16[j] = g->ranks[j]->p16;
  } else if (c->ipc && (c->stage == 1 || c->stage == 2)) {  // same, through the IPC peer table
    a.n_p16 = c->n_d;
    for (int j = 0; j < c->n_d; ++j) a.p16[j] = c->peer_p16[j];
  } else {
    a.n_p16 = 1;
    a.p16[0] = c->p16;
  }
  a.segs = c->segs;
  a.n_segs = (int)c->segs_host.size();
  a.total = c->S_e;
  int variant = c->adam_variant;
  // a small shard is a few tiles per SM: the TMA ring's fill latency dominates, so the
  // register-staged kernel with 4 CTAs per SM is used (unless a variant is forced)
  if (!c->adam_variant_env && c->S_e <= c->adam_small) variant = 1;
  if (adam_variant_is_tma(variant) && !c->segs_aligned8) variant = 0;  // bulk copies need 16-B granules
  a.pdl = (c->adam_pdl && variant == 1) ? 1 : 0;   // launch while the whole-step flatten finishes
  a.aligned8 = c->segs_aligned8 ? 1 : 0;
  c->adam_pdl = false;
  const int grid = grid_for((c->S_e + 2047) / 2048, adam_ctas_per_sm(variant), c->sms);
  a.per_cta = align_up((c->S_e + grid - 1) / grid, 8);
  a.beta1 = c->cfg.beta1;
  a.beta2 = c->cfg.beta2;
  a.eps = c->cfg.eps;
  a.omb1 = 1.0f - c->cfg.beta1;
  a.omb2 = 1.0f - c->cfg.beta2;
  a.wd = c->cfg.weight_decay > 0.0f ? 1 : 0;
  a.lrwd = (float)((double)c->cfg.lr * (double)c->cfg.weight_decay);
  a.st = c->st;
  CK(launch_adam(a, grid, c->comm_stream, variant));
  c->launches++;
  c->adam_launches++;
  return ZERO_OK;
}

DecideParams decide_params(const zero_ctx* c) {
  DecideParams p{};
  p.n_ranks = c->n_d;
  p.dynamic = c->cfg.dynamic_loss_scale ? 1 : 0;
  p.beta1 = c->cfg.beta1;
  p.beta2 = c->cfg.beta2;
  p.lr = c->cfg.lr;
  p.max_norm = c->cfg.max_grad_norm;
  p.min_scale = c->cfg.min_loss_scale;
  p.sigma = c->cfg.grad_prescale;
  p.window = c->cfg.scale_window;
  return p;
}

void reset_step(zero_ctx* c) {
  std::fill(c->reduced.begin(), c->reduced.end(), 0);
  c->n_reduced = 0;
  std::fill(c->pool_pending.begin(), c->pool_pending.end(), -1);
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

// zero_step, first half: join the reduce phase and form the decision inputs (the
// per-rank {sum of squares, overflow} partials, exchanged across the data-parallel group)
zero_status step_inputs(zero_ctx* c, PartialPtrs& pp, zero_ctx::StepEvents*& ev, bool* decided = nullptr,
                        void* rec_dev = nullptr) {
  if (!c->bound) return c->fail(ZERO_ESTATE, "buffers not bound");
  if (zero_status ps = poll_nccl(c)) return ps;
  if (c->step_begun) return c->fail(ZERO_ESTATE, "zero_step_begin already issued: finish with zero_step_end");
  ZeroGroup* g = c->group;
  if (g) {
    if (g->reduced_buckets != c->info.n_buckets)
      return c->fail(ZERO_ESTATE, "zero_step before every bucket was reduced by every rank (%u of %u)",
                     g->reduced_buckets, c->info.n_buckets);
    if (c->stepped_this_round) return c->fail(ZERO_ESTATE, "rank already stepped this round");
  } else if (c->n_reduced != c->info.n_buckets) {
    return c->fail(ZERO_ESTATE, "zero_step before every bucket was reduced (%u of %u)", c->n_reduced,
                   c->info.n_buckets);
  }

  // the pending run of small buckets (N_d = 1), on the caller's stream: the step follows it there;
  // when the run is the whole (small) model, the step becomes one cooperative launch instead
  if (decided && fused_step_ok(c)) {
    c->fused_pending = true;
    *decided = true;
  } else if (zero_status s = flush_small(c, true, decided, rec_dev)) {
    return s;
  }
  if (c->gather_stream) {  // no rank's Adam may rewrite a shard a gather still reads
    CK(cudaEventRecord(c->ev_gjoin, c->gather_stream));
    CK(cudaStreamWaitEvent(c->comm_stream, c->ev_gjoin, 0));
  }
  for (int i = 0; i < zero_ctx::kMaxFlatStreams; ++i) {  // join the flatten streams into the step
    if (!c->flat_used[i]) continue;
    CK(cudaEventRecord(c->ev_join[i], c->flat_stream[i]));
    CK(cudaStreamWaitEvent(c->comm_stream, c->ev_join[i], 0));
    if (c->comm_stream != c->stream) CK(cudaStreamWaitEvent(c->stream, c->ev_join[i], 0));
    c->flat_used[i] = false;
  }
  ev = nullptr;
  if (c->cfg.timing && c->step_open) {
    ev = &c->ev_pool[c->ev_used];
    CK(cudaEventRecord(ev->r1, c->comm_stream));
  }
  pp = PartialPtrs{};
  if (c->transport == ZERO_TRANSPORT_LOCAL) {
    if (!(decided && *decided))   // (else the whole-step flatten already decided)
      CK(issue_decide_local(c, c->comm_stream, decided, rec_dev));   // the flattens left per-CTA partials
    pp.p[0] = c->my_partial;
    pp.n = 1;
  } else if (c->ipc) {  // push my partial into every peer's gathered[rank], then wait for all
    CK(issue_decide_local(c, c->comm_stream));
    PushArgs pa{};
    pa.mine = c->my_partial;
    for (int j = 0; j < c->n_d; ++j) {
      pa.dst[j] = reinterpret_cast<RankPartial*>(c->peer_scratch[j] + c->off_gathered) + c->rank;
      pa.sig[j] = c->sig(j, c->off_sig_part, c->rank);
    }
    pa.n = c->n_d;
    pa.epoch = c->epoch();
    CK(launch_push_partial(pa, c->comm_stream));
    c->launches++;
    for (int j = 0; j < c->n_d; ++j) pp.p[j] = c->gathered + j;
    pp.n = c->n_d;
    pp.wait_flags = c->sig(c->rank, c->off_sig_part, 0);
    pp.epoch = c->epoch();
  } else if (c->transport == ZERO_TRANSPORT_PEER) {
    for (int j = 0; j < g->n; ++j) pp.p[j] = g->ranks[j]->my_partial;
    pp.n = g->n;
  } else {
    CK(issue_decide_local(c, c->comm_stream));
    NK(ncclAllGather(c->my_partial, c->gathered, 2, ncclFloat64, c->comm, c->comm_stream));
    for (int j = 0; j < c->n_d; ++j) pp.p[j] = c->gathered + j;
    pp.n = c->n_d;
  }
  return ZERO_OK;
}

// zero_step, second half: decision, fused Adam + recast, all-gather, bookkeeping
zero_status step_finish(zero_ctx* c, const PartialPtrs& pp, zero_ctx::StepEvents* ev, zero_step_info* host_out,
                        bool decided = false) {
  ZeroGroup* g = c->group;
  void* rec_dev = mapped_record(c, host_out);
  if (c->fused_pending) {   // flatten + decision + Adam in one cooperative launch (a small model)
    StepSmallArgs a;
    const int grid = step_small_grid(c, &a, rec_dev);
    c->fused_pending = false;
    c->pend_lo = c->pend_hi = -1;
    c->pend_pieces.clear();
    if (ev) CK(cudaEventRecord(ev->a0, c->comm_stream));
    CK(launch_step_small(a, grid, c->comm_stream));
    c->launches++;
    c->adam_launches++;
    if (ev) CK(cudaEventRecord(ev->a1, c->comm_stream));
  } else {
    if (!decided) {
      DecideParams p = decide_params(c);
      p.rec_out = rec_dev;
      CK(launch_decide_global(pp, c->st, p, c->comm_stream));
      c->launches++;
    }
    if (ev) CK(cudaEventRecord(ev->a0, c->comm_stream));
    zero_status s = issue_adam(c, g);
    if (s != ZERO_OK) return s;
    if (ev) CK(cudaEventRecord(ev->a1, c->comm_stream));
  }

  if (c->transport == ZERO_TRANSPORT_NCCL && (c->stage == 1 || c->stage == 2)) {
    // all-gather the updated 16-bit parameters per bucket, in place
    const ncclDataType_t dt = nccl_dt(c->pdt);
    NK(ncclGroupStart());
    for (uint32_t k = 0; k < c->info.n_buckets; ++k) {
      const zero_bucket& b = c->buckets[k];
      const uint64_t sl = c->slice(k);
      NK(ncclAllGather(c->p16 + b.base + (uint64_t)c->rank * sl, c->p16 + b.base, sl, dt, c->comm, c->comm_stream));
      c->counters.all_gather += sl * (uint64_t)(c->n_d - 1);
    }
    NK(ncclGroupEnd());
  } else if (c->transport == ZERO_TRANSPORT_PEER && (c->stage == 1 || c->stage == 2)) {
    for (uint32_t k = 0; k < c->info.n_buckets; ++k) c->counters.all_gather += c->slice(k) * (uint64_t)(c->n_d - 1);
  }
  if (ev && c->transport == ZERO_TRANSPORT_NCCL) CK(cudaEventRecord(ev->g1, c->comm_stream));   // end of the separate AG
  if (c->ipc) {  // the replicas (stages 1/2) / shards (stage 3) are final on every rank
    SigArgs sa{};
    for (int j = 0; j < c->n_d; ++j) sa.dst[j] = c->sig(j, c->off_sig_adam, c->rank);
    sa.n = c->n_d;
    sa.epoch = c->epoch();
    CK(launch_signal(sa, c->comm_stream));
    WaitArgs w{c->sig(c->rank, c->off_sig_adam, 0), c->n_d, c->epoch()};
    CK(launch_wait(w, c->comm_stream));
    c->launches += 2;
  }
  if (c->ev_params) CK(cudaEventRecord(c->ev_params, c->comm_stream));   // every shard is final
  if (host_out && !rec_dev)   // pageable: copy; pinned: the decision kernel already wrote it
    CK(cudaMemcpyAsync(host_out, &c->st->rec_t, sizeof(zero_step_info), cudaMemcpyDeviceToHost, c->comm_stream));
  if (ev) {
    CK(cudaEventRecord(ev->s1, c->comm_stream));
    c->ev_used++;
    c->step_open = false;
  }
  if (c->comm_stream != c->stream) {
    CK(cudaEventRecord(c->ev_step, c->comm_stream));
    CK(cudaStreamWaitEvent(c->stream, c->ev_step, 0));
  }
  c->counters.steps++;
  if (c->stage == 3) {  // the step rewrote every shard: gathered copies are stale
    for (auto& gs : c->gslots) {
      gs.layer = -1;
      gs.released = true;
    }
    std::fill(c->layer_slot.begin(), c->layer_slot.end(), -1);
    c->last_layer = -1;
    c->direction = +1;
  }
  if (g) {
    c->stepped_this_round = true;
    if (++g->stepped == g->n) {
      for (int j = 0; j < g->n; ++j) {
        reset_step(g->ranks[j]);
        g->ranks[j]->stepped_this_round = false;
      }
      std::fill(g->flat_count.begin(), g->flat_count.end(), 0);
      g->reduced_buckets = 0;
      g->stepped = 0;
    }
  } else {
    reset_step(c);
  }
  return ZERO_OK;
}

}  // namespace

extern "C" {

zero_status zero_step(zero_ctx* c, zero_step_info* host_out) {
  STICKY(c);
  NvtxRange nvtx("zero_step");
  PartialPtrs pp{};
  zero_ctx::StepEvents* ev = nullptr;
  bool decided = false;
  zero_status s = step_inputs(c, pp, ev, &decided, mapped_record(c, host_out));
  if (s != ZERO_OK) return s;
  return step_finish(c, pp, ev, host_out, decided);
}

zero_status zero_step_begin(zero_ctx* c) {
  STICKY(c);
  NvtxRange nvtx("zero_step_begin");
  PartialPtrs pp{};
  zero_ctx::StepEvents* ev = nullptr;
  zero_status s = step_inputs(c, pp, ev);
  if (s != ZERO_OK) return s;
  CK(launch_combine_partials(pp, c->dp_partial, c->comm_stream));
  c->launches++;
  if (c->comm_stream != c->stream) {  // the caller's exchange runs on its stream
    CK(cudaEventRecord(c->ev_step, c->comm_stream));
    CK(cudaStreamWaitEvent(c->stream, c->ev_step, 0));
  }
  c->pend_ev = ev ? (int)(ev - c->ev_pool.data()) : -1;
  c->step_begun = true;
  return ZERO_OK;
}

zero_status zero_step_end(zero_ctx* c, zero_step_info* host_out) {
  STICKY(c);
  NvtxRange nvtx("zero_step_end");
  if (!c->step_begun) return c->fail(ZERO_ESTATE, "zero_step_end without zero_step_begin");
  if (c->comm_stream != c->stream) {  // after the caller's exchange of the partial
    CK(cudaEventRecord(c->ev_step, c->stream));
    CK(cudaStreamWaitEvent(c->comm_stream, c->ev_step, 0));
  }
  PartialPtrs pp{};
  pp.p[0] = c->dp_partial;
  pp.n = 1;
  zero_ctx::StepEvents* ev = c->pend_ev >= 0 ? &c->ev_pool[c->pend_ev] : nullptr;
  c->step_begun = false;
  c->pend_ev = -1;
  return step_finish(c, pp, ev, host_out);
}

// ---------------------------------------------------------------------------
// cross-process PEER transport over CUDA IPC
// ---------------------------------------------------------------------------
}  // extern "C"

namespace {

struct IpcRegion {
  cudaIpcMemHandle_t handle;
  uint64_t offset;   // of the arena inside its cudaMalloc allocation
  uint64_t bytes;
};
struct IpcBlob {
  uint32_t magic, rank, n_d, stage;
  uint64_t psi_padded, scratch_bytes;
  IpcRegion region[3];  // grad, p16, scratch
};
constexpr uint32_t kIpcMagic = 0x5A45524Fu;  // "ZERO"

typedef int (*cuMemGetAddressRange_t)(unsigned long long*, size_t*, unsigned long long);
cuMemGetAddressRange_t get_range_fn() {
  static cuMemGetAddressRange_t fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
    if (h) fn = reinterpret_cast<cuMemGetAddressRange_t>(dlsym(h, "cuMemGetAddressRange_v2"));
  }
  return fn;
}

}  // namespace

extern "C" {

zero_status zero_peer_export(zero_ctx* c, void* blob, size_t* blob_bytes) {
  STICKY(c);
  if (!blob_bytes) return c->fail(ZERO_EINVAL, "blob_bytes is NULL");
  if (!blob) { *blob_bytes = sizeof(IpcBlob); return ZERO_OK; }
  if (*blob_bytes < sizeof(IpcBlob)) return c->fail(ZERO_EINVAL, "blob buffer too small (%zu)", sizeof(IpcBlob));
  if (c->transport != ZERO_TRANSPORT_PEER || c->group) return c->fail(ZERO_ESTATE, "export needs an ungrouped PEER context");
  if (!c->bound) return c->fail(ZERO_ESTATE, "buffers not bound");
  auto range = get_range_fn();
  if (!range) return c->fail(ZERO_ECUDA, "cuMemGetAddressRange unavailable");
  // the arenas' zeroing (zero_bind_buffers) must be complete before any peer can
  // write a signal into them: every rank exports before any rank opens
  CK(cudaStreamSynchronize(c->stream));
  IpcBlob b{};
  b.magic = kIpcMagic;
  b.rank = (uint32_t)c->rank;
  b.n_d = (uint32_t)c->n_d;
  b.stage = (uint32_t)c->stage;
  b.psi_padded = c->info.psi_padded;
  b.scratch_bytes = c->sizes.scratch_bytes;
  const void* ptrs[3] = {c->bufs.grad, c->bufs.p16, c->bufs.scratch};
  const uint64_t sz[3] = {c->sizes.grad_bytes, c->sizes.p16_bytes, c->sizes.scratch_bytes};
  for (int i = 0; i < 3; ++i) {
    if (!sz[i]) continue;
    unsigned long long base = 0;
    size_t bsz = 0;
    if (range(&base, &bsz, (unsigned long long)reinterpret_cast<uintptr_t>(ptrs[i])) != 0)
      return c->fail(ZERO_ECUDA, "cuMemGetAddressRange failed for arena %d", i);
    CK(cudaIpcGetMemHandle(&b.region[i].handle, reinterpret_cast<void*>(base)));
    b.region[i].offset = reinterpret_cast<uintptr_t>(ptrs[i]) - base;
    b.region[i].bytes = sz[i];
  }
  std::memcpy(blob, &b, sizeof(b));
  *blob_bytes = sizeof(b);
  return ZERO_OK;
}

zero_status zero_peer_open(zero_ctx* c, const void* const* blobs, size_t blob_bytes) {
  STICKY(c);
  if (!blobs || blob_bytes < sizeof(IpcBlob)) return c->fail(ZERO_EINVAL, "bad blobs");
  if (c->transport != ZERO_TRANSPORT_PEER || c->group || c->ipc) return c->fail(ZERO_ESTATE, "open needs an unlinked PEER context");
  if (!c->bound) return c->fail(ZERO_ESTATE, "buffers not bound");
  for (int r = 0; r < c->n_d; ++r) {
    IpcBlob b;
    std::memcpy(&b, blobs[r], sizeof(b));
    if (b.magic != kIpcMagic || (int)b.rank != r || (int)b.n_d != c->n_d || (int)b.stage != c->stage ||
        b.psi_padded != c->info.psi_padded || b.scratch_bytes != c->sizes.scratch_bytes)
      return c->fail(ZERO_EINVAL, "blob %d does not match this context (rank/layout/stage)", r);
    if (r == c->rank) {
      c->peer_grad[r] = c->grad;
      c->peer_p16[r] = c->p16;
      c->peer_scratch[r] = reinterpret_cast<char*>(c->bufs.scratch);
      continue;
    }
    void* mapped[3] = {nullptr, nullptr, nullptr};
    void* bases[3] = {nullptr, nullptr, nullptr};
    for (int i = 0; i < 3; ++i) {
      if (!b.region[i].bytes) continue;
      void* base = nullptr;
      for (int j = 0; j < i; ++j)  // arenas of one cudaMalloc segment share a handle: map it once
        if (bases[j] && !std::memcmp(&b.region[j].handle, &b.region[i].handle, sizeof(cudaIpcMemHandle_t)))
          base = bases[j];
      if (!base) {
        CK(cudaIpcOpenMemHandle(&base, b.region[i].handle, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_mapped.push_back(base);
      }
      bases[i] = base;
      mapped[i] = reinterpret_cast<char*>(base) + b.region[i].offset;
    }
    c->peer_grad[r] = reinterpret_cast<uint16_t*>(mapped[0]);
    c->peer_p16[r] = reinterpret_cast<uint16_t*>(mapped[1]);
    c->peer_scratch[r] = reinterpret_cast<char*>(mapped[2]);
  }
  // handshake over the new mappings (system-scope release/acquire through every
  // peer's scratch), bounded so that an unreachable peer is an error, not a hang
  {
    uint64_t timeout_ms = 60000;
    if (const char* ev = getenv("ZERO_PEER_TIMEOUT_MS")) timeout_ms = strtoull(ev, nullptr, 10);
    SigArgs sa{};
    for (int j = 0; j < c->n_d; ++j) sa.dst[j] = c->sig(j, c->off_sig_hello, c->rank);
    sa.n = c->n_d;
    sa.epoch = 1;
    uint32_t* dres = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(c->bufs.scratch) + c->off_hello_result);
    uint32_t hres = 1;
    CK(launch_handshake(sa, c->sig(c->rank, c->off_sig_hello, 0), timeout_ms * 1000000ull, dres, c->stream));
    CK(cudaMemcpyAsync(&hres, dres, sizeof(hres), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->launches++;
    if (hres != 0)
      return c->fail(ZERO_ECUDA, "peer handshake timed out after %llu ms (a peer did not open its mappings)",
                     (unsigned long long)timeout_ms);
  }
  c->ipc = true;
  // cross-process: the pull reduce-scatter (NVLink-bound) runs on its own stream so it
  // overlaps the next buckets' flattens (HBM-bound) on the forked flatten streams
  if (c->comm_stream == c->stream) {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi));
    c->own_comm_stream = true;
  }
  c->n_flat_streams = c->n_flat_streams_req;
  if (c->stage == 3 && !c->gather_stream) CK(cudaStreamCreateWithFlags(&c->gather_stream, cudaStreamNonBlocking));
  return create_flat_streams(c);
}

zero_status zero_sim_group(zero_ctx* const* ranks, int n) {
  if (!ranks || n < 2 || n > ZERO_MAX_RANKS) return ZERO_EINVAL;
  for (int r = 0; r < n; ++r) {
    zero_ctx* c = ranks[r];
    if (!c || c->rank != r || c->n_d != n || c->transport != ZERO_TRANSPORT_PEER || !c->bound || c->group)
      return ZERO_EINVAL;
    if (c->stage != ranks[0]->stage || c->stream != ranks[0]->stream || c->info.psi_padded != ranks[0]->info.psi_padded ||
        c->info.n_buckets != ranks[0]->info.n_buckets || c->pdt != ranks[0]->pdt || c->r32 != ranks[0]->r32)
      return c->fail(ZERO_EINVAL, "group members differ in stage/stream/layout/dtype");
  }
  ZeroGroup* g = new ZeroGroup();
  g->n = n;
  g->flat_count.assign(ranks[0]->info.n_buckets, 0);
  for (int r = 0; r < n; ++r) {
    g->ranks[r] = ranks[r];
    ranks[r]->group = g;
  }
  return ZERO_OK;
}

// ---------------------------------------------------------------------------
// stage 3: per-layer gather with prefetch
// ---------------------------------------------------------------------------
}  // extern "C"

namespace {

zero_status issue_layer_gather(zero_ctx* c, int li, int slot) {
  const LayerInfo& L = c->layers[li];
  GatherSlot& gs = c->gslots[slot];
  uint16_t* dst = c->gather + (uint64_t)slot * c->max_layer;
  if (c->transport == ZERO_TRANSPORT_NCCL) {
    CK(cudaStreamWaitEvent(c->comm_stream, gs.freed, 0));
    NK(ncclGroupStart());
    for (uint32_t k = L.k0; k < L.k1; ++k) {
      const zero_bucket& b = c->buckets[k];
      const uint64_t sl = c->slice(k);
      NK(ncclAllGather(c->p16 + b.shard_off, dst + (b.base - L.flat0), sl, nccl_dt(c->pdt), c->comm, c->comm_stream));
      c->counters.all_gather += sl * (uint64_t)(c->n_d - 1);
    }
    NK(ncclGroupEnd());
    CK(cudaEventRecord(gs.ready, c->comm_stream));
  } else {  // PEER: pull every rank's shard slice
    ZeroGroup* g = c->group;
    cudaStream_t gst = c->gather_stream ? c->gather_stream : c->stream;   // simulated ranks: the shared stream
    if (c->gather_stream) {
      CK(cudaStreamWaitEvent(gst, c->ev_params, 0));   // the shards of this epoch are final
      CK(cudaStreamWaitEvent(gst, gs.freed, 0));       // the slot's previous layer is released
    }
    for (uint32_t k = L.k0; k < L.k1; ++k) {
      const zero_bucket& b = c->buckets[k];
      const uint64_t sl = c->slice(k);
      CopyArgs a{};
      for (int j = 0; j < c->n_d; ++j) {
        a.src[j] = (g ? g->ranks[j]->p16 : c->peer_p16[j]) + b.shard_off;
        a.dst[j] = dst + (b.base - L.flat0) + (uint64_t)j * sl;
      }
      for (int j = 0; j < c->n_d; ++j) a.count[j] = sl;
      a.n = c->n_d;
      int grid = grid_for((sl + 2047) / 2048, 2, c->sms);
      if (c->gather_grid > 0) grid = std::min(grid, c->gather_grid);   // grid-stride copy: any grid is exact
      CK(launch_copy(a, grid, gst));
      c->launches++;
      c->counters.all_gather += sl * (uint64_t)(c->n_d - 1);
    }
    if (c->gather_stream) CK(cudaEventRecord(gs.ready, gst));
  }
  gs.layer = L.layer;
  gs.released = false;
  gs.lru = ++c->lru_clock;
  c->layer_slot[li] = slot;
  return ZERO_OK;
}

// a free slot: never used, or released; prefer the least recently used
int free_slot(zero_ctx* c, int keep_li) {
  int best = -1;
  for (int s = 0; s < (int)c->gslots.size(); ++s) {
    const GatherSlot& g = c->gslots[s];
    if (!g.released) continue;
    if (keep_li >= 0 && c->layer_slot[keep_li] == s) continue;
    if (best < 0 || g.lru < c->gslots[best].lru) best = s;
  }
  if (best >= 0 && c->gslots[best].layer >= 0) {
    auto it = c->layer_index.find((uint32_t)c->gslots[best].layer);
    if (it != c->layer_index.end()) c->layer_slot[it->second] = -1;
  }
  return best;
}

}  // namespace

extern "C" {

zero_status zero_gather_params(zero_ctx* c, uint32_t layer, void** views_out) {
  STICKY(c);
  NvtxRange nvtx("zero_gather_params");
  if (!c->bound) return c->fail(ZERO_ESTATE, "buffers not bound");
  if (c->stage != 3) return c->fail(ZERO_ESTATE, "zero_gather_params needs stage 3");
  auto it = c->layer_index.find(layer);
  if (it == c->layer_index.end()) return c->fail(ZERO_EINVAL, "unknown layer %u", layer);
  if (zero_status ps = poll_nccl(c)) return ps;
  const int li = it->second;
  uint16_t* base;
  if (c->transport == ZERO_TRANSPORT_LOCAL) {
    base = c->p16 + c->layers[li].flat0;  // the shard is the whole replica
  } else {
    if (c->last_layer >= 0) c->direction = (li >= c->last_layer) ? +1 : -1;
    c->last_layer = li;
    int s = c->layer_slot[li];
    if (s < 0) {
      s = free_slot(c, -1);
      if (s < 0) return c->fail(ZERO_ESTATE, "gather pool exhausted: release layers before gathering more");
      zero_status r = issue_layer_gather(c, li, s);
      if (r != ZERO_OK) return r;
    } else {
      c->gslots[s].released = false;
      c->gslots[s].lru = ++c->lru_clock;
    }
    // prefetch the next layers in the current direction into free slots
    for (uint32_t d = 1; d <= c->cfg.prefetch_depth; ++d) {
      const int nl = li + c->direction * (int)d;
      if (nl < 0 || nl >= (int)c->layers.size() || c->layer_slot[nl] >= 0) continue;
      const int fs = free_slot(c, li);
      if (fs < 0) break;
      zero_status r = issue_layer_gather(c, nl, fs);
      if (r != ZERO_OK) return r;
      c->gslots[fs].released = true;  // prefetched: reusable until someone asks for it
    }
    if (c->transport == ZERO_TRANSPORT_NCCL || c->gather_stream) CK(cudaStreamWaitEvent(c->stream, c->gslots[s].ready, 0));
    base = c->gather + (uint64_t)s * c->max_layer;
  }
  if (views_out) {
    const LayerInfo& L = c->layers[li];
    for (uint32_t t = 0; t < c->tensors.size(); ++t)
      if (c->tensors[t].layer == layer && c->tensors[t].numel > 0) views_out[t] = base + (c->tensor_flat[t] - L.flat0);
  }
  return ZERO_OK;
}

zero_status zero_release_params(zero_ctx* c, uint32_t layer) {
  STICKY(c);
  if (c->stage != 3) return c->fail(ZERO_ESTATE, "zero_release_params needs stage 3");
  auto it = c->layer_index.find(layer);
  if (it == c->layer_index.end()) return c->fail(ZERO_EINVAL, "unknown layer %u", layer);
  if (c->transport == ZERO_TRANSPORT_LOCAL) return ZERO_OK;
  const int s = c->layer_slot[it->second];
  if (s < 0) return c->fail(ZERO_ESTATE, "layer %u is not gathered", layer);
  c->gslots[s].released = true;
  if (c->transport == ZERO_TRANSPORT_NCCL || c->gather_stream) CK(cudaEventRecord(c->gslots[s].freed, c->stream));
  return ZERO_OK;
}

zero_status zero_param_view(const zero_ctx* c, uint32_t t, void** p16) {
  if (!c || !p16) return ZERO_EINVAL;
  if (t >= c->tensors.size() || c->tensor_flat[t] == UINT64_MAX) return ZERO_EINVAL;
  if (!c->bound) return ZERO_ESTATE;
  if (c->stage == 3 && c->transport != ZERO_TRANSPORT_LOCAL) return ZERO_ESTATE;
  *p16 = c->p16 + c->tensor_flat[t];
  return ZERO_OK;
}

zero_status zero_query(const zero_ctx* cc, int what, void* out, size_t n) {
  zero_ctx* c = const_cast<zero_ctx*>(cc);
  if (!c || !out) return ZERO_EINVAL;
  switch (what) {
    case ZERO_Q_LAYOUT:
      if (n < sizeof(zero_layout_info)) return ZERO_EINVAL;
      *reinterpret_cast<zero_layout_info*>(out) = c->info;
      return ZERO_OK;
    case ZERO_Q_BUCKETS:
      if (n < sizeof(zero_bucket) * c->buckets.size()) return ZERO_EINVAL;
      std::memcpy(out, c->buckets.data(), sizeof(zero_bucket) * c->buckets.size());
      return ZERO_OK;
    case ZERO_Q_PIECES:
      if (n < sizeof(zero_piece) * c->pieces.size()) return ZERO_EINVAL;
      std::memcpy(out, c->pieces.data(), sizeof(zero_piece) * c->pieces.size());
      return ZERO_OK;
    case ZERO_Q_MEMORY: {
      if (n < sizeof(zero_memory)) return ZERO_EINVAL;
      zero_memory mem{};
      const zero_sizes& z = c->sizes;
      const uint64_t S = c->info.shard;
      mem.params16 = z.p16_bytes;
      mem.optimizer = 12ull * c->S_e;                  // logical K*S_e (the arena may pad m, v to 64)
      if (c->stage <= 1) {
        mem.grads16 = z.grad_bytes;
        mem.reduced_grad_extra = z.gred_bytes;
      } else {
        mem.grads16 = 2 * S;
        mem.reduced_grad_extra = z.gred_bytes - 2 * S;
        mem.staging = z.grad_bytes;
      }
      mem.gather_pool = z.gather_bytes;
      mem.scratch = z.scratch_bytes;
      *reinterpret_cast<zero_memory*>(out) = mem;
      return ZERO_OK;
    }
    case ZERO_Q_COMM:
      if (n < sizeof(zero_comm_counters)) return ZERO_EINVAL;
      *reinterpret_cast<zero_comm_counters*>(out) = c->counters;
      return ZERO_OK;
    case ZERO_Q_STEP: {
      if (n < sizeof(zero_step_info)) return ZERO_EINVAL;
      if (!c->bound) return ZERO_ESTATE;
      STICKY(c);
      CK(cudaStreamSynchronize(c->comm_stream));
      CK(cudaStreamSynchronize(c->stream));
      CK(cudaMemcpy(out, &c->st->rec_t, sizeof(zero_step_info), cudaMemcpyDeviceToHost));
      return ZERO_OK;
    }
    case ZERO_Q_STATE: {
      if (n < sizeof(zero_device_state)) return ZERO_EINVAL;
      if (!c->bound) return ZERO_ESTATE;
      STICKY(c);
      CK(cudaStreamSynchronize(c->comm_stream));
      CK(cudaStreamSynchronize(c->stream));
      DevState d{};
      CK(cudaMemcpy(&d, c->st, sizeof(DevState), cudaMemcpyDeviceToHost));
      zero_device_state o{};
      o.b1t = d.b1t;
      o.b2t = d.b2t;
      o.t = d.t;
      o.loss_scale = d.S;
      o.good_steps = d.good;
      *reinterpret_cast<zero_device_state*>(out) = o;
      return ZERO_OK;
    }
    case ZERO_Q_TIMING: {
      if (n < sizeof(zero_timing)) return ZERO_EINVAL;
      STICKY(c);
      zero_timing tm{};
      if (c->bound && c->ev_used) {
        CK(cudaStreamSynchronize(c->comm_stream));
        CK(cudaStreamSynchronize(c->stream));
        for (size_t i = 0; i < c->ev_used; ++i) {
          float a = 0, b = 0, d = 0, g = 0;
          CK(cudaEventElapsedTime(&a, c->ev_pool[i].r0, c->ev_pool[i].r1));
          CK(cudaEventElapsedTime(&b, c->ev_pool[i].a0, c->ev_pool[i].a1));
          if (c->transport == ZERO_TRANSPORT_NCCL) CK(cudaEventElapsedTime(&g, c->ev_pool[i].a1, c->ev_pool[i].g1));
          CK(cudaEventElapsedTime(&d, c->ev_pool[i].r1, c->ev_pool[i].s1));
          tm.reduce_ms += a;
          tm.adam_ms += b;
          tm.ag_ms += g;
          tm.step_ms += d;
        }
        tm.steps = c->ev_used;
        c->ev_used = 0;
      }
      tm.kernel_launches = c->launches;
      tm.adam_launches = c->adam_launches;
      *reinterpret_cast<zero_timing*>(out) = tm;
      return ZERO_OK;
    }
    case ZERO_Q_DECISION: {
      if (n < sizeof(void*)) return ZERO_EINVAL;
      if (!c->bound) return ZERO_ESTATE;
      *reinterpret_cast<void**>(out) = c->dp_partial;
      return ZERO_OK;
    }
    default:
      return ZERO_EINVAL;
  }
}

zero_status zero_wait(zero_ctx* c, uint64_t timeout_ms) {
  STICKY(c);
  if (!c->bound) return c->fail(ZERO_ESTATE, "buffers not bound");
  cudaStream_t ss[zero_ctx::kMaxFlatStreams + 3];
  int ns = 0;
  ss[ns++] = c->stream;
  if (c->comm_stream && c->comm_stream != c->stream) ss[ns++] = c->comm_stream;
  for (int i = 0; i < zero_ctx::kMaxFlatStreams; ++i)
    if (c->flat_stream[i]) ss[ns++] = c->flat_stream[i];
  if (c->gather_stream) ss[ns++] = c->gather_stream;
  for (int i = 0; i < ns; ++i) {
    if (!c->ev_wait[i]) CK(cudaEventCreateWithFlags(&c->ev_wait[i], cudaEventDisableTiming));
    CK(cudaEventRecord(c->ev_wait[i], ss[i]));
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    bool done = true;
    for (int i = 0; i < ns; ++i) {
      const cudaError_t q = cudaEventQuery(c->ev_wait[i]);
      if (q == cudaErrorNotReady) { done = false; continue; }
      if (q != cudaSuccess) return c->fail(ZERO_ECUDA, "zero_wait: %s", cudaGetErrorString(q));
    }
    if (zero_status ps = poll_nccl(c)) return ps;
    if (done) return ZERO_OK;
    const uint64_t el =
        (uint64_t)std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    if (el >= timeout_ms) {
      if (c->transport == ZERO_TRANSPORT_NCCL) {
        char why[160];
        snprintf(why, sizeof(why), "work issued by the context did not complete within %llu ms",
                 (unsigned long long)timeout_ms);
        return abort_comm(c, why);
      }
      c->err = "zero_wait: device work did not complete within " + std::to_string(timeout_ms) + " ms";
      return ZERO_ETIMEOUT;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

zero_status zero_set_timing(zero_ctx* c, int on) {
  STICKY(c);
  if (c->step_open || c->n_reduced) return c->fail(ZERO_ESTATE, "zero_set_timing inside a step");
  c->cfg.timing = on ? 1u : 0u;
  return ZERO_OK;
}

const char* zero_last_error(const zero_ctx* c) {
  if (!c) return g_init_error.c_str();
  return c->err.c_str();
}

void zero_destroy(zero_ctx* c) {
  if (!c) return;
  if (c->bound) {
    cudaStreamSynchronize(c->stream);
    if (c->comm_stream && c->comm_stream != c->stream) cudaStreamSynchronize(c->comm_stream);
  }
  if (c->group) {  // the group dissolves with its first destroyed member
    ZeroGroup* g = c->group;
    for (int j = 0; j < g->n; ++j)
      if (g->ranks[j]) g->ranks[j]->group = nullptr;
    delete g;
  }
  for (void* p : c->ipc_mapped) cudaIpcCloseMemHandle(p);
  for (auto& e : c->ev_pool_free) if (e) cudaEventDestroy(e);
  for (auto& e : c->ev_pool) {
    cudaEventDestroy(e.r0);
    cudaEventDestroy(e.r1);
    cudaEventDestroy(e.a0);
    cudaEventDestroy(e.a1);
    cudaEventDestroy(e.g1);
    cudaEventDestroy(e.s1);
  }
  for (auto& gs : c->gslots) {
    if (gs.ready) cudaEventDestroy(gs.ready);
    if (gs.freed) cudaEventDestroy(gs.freed);
  }
  for (int i = 0; i < zero_ctx::kMaxFlatStreams; ++i) {
    if (c->flat_stream[i]) {
      cudaStreamSynchronize(c->flat_stream[i]);
      cudaStreamDestroy(c->flat_stream[i]);
    }
    if (c->ev_join[i]) cudaEventDestroy(c->ev_join[i]);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  for (auto& e : c->ev_wait) if (e) cudaEventDestroy(e);
  if (c->gather_stream) {
    cudaStreamSynchronize(c->gather_stream);
    cudaStreamDestroy(c->gather_stream);
  }
  if (c->ev_params) cudaEventDestroy(c->ev_params);
  if (c->ev_gjoin) cudaEventDestroy(c->ev_gjoin);
  if (c->ev_flat) cudaEventDestroy(c->ev_flat);
  if (c->ev_step) cudaEventDestroy(c->ev_step);
  if (c->own_comm_stream && c->comm_stream) cudaStreamDestroy(c->comm_stream);
  delete c;
}

}  // extern "C"
