// Internal types shared by the host engine (engine.cpp) and the sm_100a kernels
// (kernels.cu).  Not part of the ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace zero {

constexpr int kMaxRanks = 8;
constexpr int kMaxFlatPieces = 32;      // pieces per flatten launch (kernel-parameter table)
constexpr int kMaxGrid = 1184;          // 148 SMs x 8: upper bound of any reduction grid
constexpr int kThreads = 256;

enum DType : int { DT_F16 = 0, DT_BF16 = 1, DT_F32 = 2 };

// Per-bucket epilogue result: overflow flag and sum of (G*inv)^2 (fp64).
struct Slot {
  double sumsq;
  uint32_t flag;
  uint32_t pad;
};

// Per-rank partial combined across ranks by the decision kernel.
struct RankPartial {
  double sumsq;
  double flag;   // 0 or 1 (double so the record is one 16-byte all-gather)
};

// Scratch for the deterministic last-CTA reduction of a grid.
struct GridPartials {
  double sumsq[kMaxGrid];
  uint32_t flag[kMaxGrid];
  uint32_t ticket;
  uint32_t pad;
};

// Loss-scale / Adam scalars living on the device (reading c-4).  Only the decision
// kernel writes them; epilogues and Adam read them.
struct DevState {
  double b1t, b2t;          // running beta^t products (fp64)
  uint64_t t;               // Adam step count
  float S;                  // current loss scale
  uint32_t good;            // consecutive good steps
  float inv_cur;            // inv = fp32(1/(N*S*sigma)) for the current step's epilogues
  float inv_adam;           // inv of the step being applied (latched by the decision)
  float step_f, rsb2_f, clip_f;
  uint32_t skip;            // 1: overflow -> Adam exits
  // step record (mirrors zero_step_info, 32 bytes)
  uint64_t rec_t;
  uint32_t rec_overflow;
  float rec_scale;
  float rec_clip;
  uint32_t rec_pad;
  double rec_norm;
};

// the DevState fields the decision reads (decide_apply), loaded together
struct DevSnap {
  double b1t, b2t;
  uint64_t t;
  float S;
  uint32_t good;
  float inv_cur;
};

struct DecideParams {
  int n_ranks;
  int dynamic;
  float beta1, beta2, lr, max_norm, min_scale, sigma;
  uint32_t window;
  void* rec_out;            // device-visible pinned host copy of the step record (zero_step_info), or NULL
};

struct FlatPiece {
  const void* src;          // nullptr = zero fill (alignment gap / padding)
  uint64_t dst_off;         // element offset inside the destination bucket
  uint64_t count;
};

struct FlatArgs {
  FlatPiece pieces[kMaxFlatPieces];
  int n_pieces;
  int src_dtype, dst_dtype;
  int epilogue;             // 1: also compute the overflow flag and norm partial (N_d == 1)
  uint64_t per_cta;         // contiguous destination elements per CTA (multiple of 8)
  void* dst;
  float sigma;
  const DevState* st;
  GridPartials* part;
  Slot* slot;
  // N_d == 1: per-CTA epilogue partials of this launch's slot (no last-CTA combine in
  // the flatten; k_decide_local reduces them in a fixed order); NULL = grid_publish
  double* cta_sum;
  uint32_t* cta_flag;
  uint32_t* cta_grid;
  uint32_t clear_slots;     // batched small buckets: the next clear_slots slots' cta_grid := 0 (their
                            // elements' partials are this launch's, in cta_grid[0]'s slot)
  int pdl;                  // host: launch as a programmatic dependent of the previous flatten
  // N_d = 1, one launch holding every bucket of the step (a small model): its last CTA
  // combines the per-CTA partials (CTA order) and makes the step's decision (decide_st != NULL)
  DevState* decide_st;
  RankPartial* decide_out;
  GridPartials* decide_part;    // ticket
  DecideParams decide;
};

struct RSArgs {
  const void* src[kMaxRanks];   // rank j's bucket slice (16-bit)
  // cross-process PEER: wait until wait_flags[0..n) >= epoch before reading peers,
  // and store epoch into done_sig[0..n) (peers' "reduce-scatter done" slots) at the end
  const uint64_t* wait_flags;
  uint64_t* done_sig[kMaxRanks];
  uint64_t epoch;
  void* dst;                    // reduced slice: 16-bit (R16) or fp32 (R32)
  uint64_t count;
  int n;
  int dtype;                    // 16-bit dtype of the sources
  int r32;                      // 1: write fp32
  int reduce;                   // 0: epilogue only over dst (NCCL path: dst already reduced)
  const DevState* st;
  GridPartials* part;
  Slot* slot;
  // per-CTA epilogue partials of this bucket's slot (k_decide_local combines them in a
  // fixed order; no serial last-CTA combine at the end of every launch); NULL = grid_publish.
  // With done_sig, part->ticket still elects the last CTA, which only signals the peers.
  double* cta_sum;
  uint32_t* cta_flag;
  uint32_t* cta_grid;
  int u;                        // host: 8-element groups per thread per iteration (0 = default)
  int pipe;                     // host: software-pipelined variant (next group's loads in flight)
};

struct RSMulti {                // every simulated rank's pull reduce-scatter of one bucket
  RSArgs r[kMaxRanks];
  int n;
};

struct AdamSeg {
  uint64_t local_off, g_off, p16_off, count;
};

struct AdamArgs {
  float* p32;
  float* m;
  float* v;
  const void* G;
  void* p16[kMaxRanks];     // destinations of the recast parameters (fused all-gather)
  int n_p16;
  int p_dtype, g_dtype;
  const AdamSeg* segs;
  int n_segs;
  uint64_t total;           // elements in the shard
  uint64_t per_cta;         // contiguous elements per CTA (multiple of 8)
  float beta1, beta2, eps, omb1, omb2, lrwd;
  int wd;
  const DevState* st;
  int pdl;                  // host: launch as a programmatic dependent of the preceding kernel
  int aligned8;             // every segment's local_off, count, g_off and p16_off % 8 == 0
};

// N_d = 1, a small model: the whole step -- flatten of every bucket with the overflow/norm
// epilogue, the decision, the fused Adam -- as ONE cooperative launch (grid-wide barriers)
struct StepSmallArgs {
  FlatArgs f;                 // every bucket (one batched run); f.cta_sum/cta_flag: per-CTA partials
  AdamArgs adam;              // per_cta for the same grid
  DecideParams dp;
  DevState* st;
  RankPartial* out;
};

struct CopyArgs {             // multi-row 16-bit copy: pull all-gathers (a6/a7) and P_a's save/gather
  const void* src[kMaxRanks];
  void* dst[kMaxRanks];
  uint64_t count[kMaxRanks];  // elements of row j (grid row j copies src[j] -> dst[j])
  int n;
};

struct LoadArgs {             // master init: fp32 piece -> shard / 16-bit copy
  const float* src;
  uint64_t count;
  uint64_t flat_off;          // global flat offset of the piece's first element
  uint64_t own_lo, own_hi;    // owned global range of the bucket (stage 0: whole bucket)
  uint64_t local_base;        // shard offset of own_lo
  float* p32;
  void* p16;
  int p16_mode;               // 0: replica at global index, 1: shard at local index
  int p_dtype;
};

struct ShardIOArgs {           // checkpoint: per-tensor fp32 piece <-> owned shard elements
  float* tensor;              // the piece's first element in the per-tensor array
  float* shard;               // p32, m or v
  uint64_t count;
  uint64_t flat_off;
  uint64_t own_lo, own_hi;
  uint64_t local_base;
  int to_shard;               // 1: tensor -> shard, 0: shard -> tensor
};

// launchers (kernels.cu); return the launch error
cudaError_t launch_flatten(const FlatArgs& a, int grid, cudaStream_t s, int vecs);
cudaError_t launch_flatten_tma(const FlatArgs& a, int grid, cudaStream_t s, int variant);
// the cast/prescaled 16-bit values stored widened to fp32 (R32 over NCCL); no epilogue
cudaError_t launch_flatten_wide(const FlatArgs& a, int grid, cudaStream_t s);
int flatten_tma_ctas_per_sm(int variant);
cudaError_t launch_reduce_scatter(const RSArgs& a, int grid, cudaStream_t s);
// cudaErrorNotSupported: not eligible (the caller launches per rank instead)
cudaError_t launch_reduce_scatter_multi(const RSMulti& m, int grid, cudaStream_t s);
// cta_*: optional per-CTA flatten partials (N_d == 1), slot i at [i * kMaxGrid, + cta_grid[i])
// slot_w: optional per-slot norm weights (0 or 1; ZeRO x MP, R-MP1)
cudaError_t launch_decide_local(Slot* slots, int n_slots, RankPartial* out, cudaStream_t s,
                                const double* slot_w = nullptr, const double* cta_sum = nullptr,
                                const uint32_t* cta_flag = nullptr, const uint32_t* cta_grid = nullptr);
struct PartialPtrs {
  const RankPartial* p[kMaxRanks];
  int n;                        // partials to sum, in order
  const uint64_t* wait_flags;   // cross-process PEER: wait until wait_flags[r] >= epoch
  uint64_t epoch;
};

struct SigArgs {                // store epoch into n (peer) signal slots, release at system scope
  uint64_t* dst[kMaxRanks];
  int n;
  uint64_t epoch;
};
struct WaitArgs {               // spin until flags[0..n) >= epoch (acquire at system scope)
  const uint64_t* flags;
  int n;
  uint64_t epoch;
};
struct PushArgs {               // copy my partial into every peer's gathered[me], then signal
  const RankPartial* mine;
  RankPartial* dst[kMaxRanks];
  uint64_t* sig[kMaxRanks];
  int n;
  uint64_t epoch;
};
cudaError_t launch_signal(const SigArgs& a, cudaStream_t s);
cudaError_t launch_wait(const WaitArgs& a, cudaStream_t s);
cudaError_t launch_handshake(const SigArgs& a, const uint64_t* my_flags, uint64_t timeout_ns, uint32_t* result,
                             cudaStream_t s);
cudaError_t launch_push_partial(const PushArgs& a, cudaStream_t s);
// per-CTA epilogue partials, one CTA per slot + a last-CTA combine (n_slots <= kMaxGrid); with
// st != NULL (N_d = 1, zero_step) the last CTA also makes the decision (k_decide_global fused)
cudaError_t launch_decide_local_slots(int n_slots, RankPartial* out, cudaStream_t s, const double* slot_w,
                                      const double* cta_sum, const uint32_t* cta_flag, const uint32_t* cta_grid,
                                      GridPartials* part, DevState* st = nullptr, const DecideParams* p = nullptr);
// zero_step_begin: sum the partials of pp (waiting on its flags) into *out
cudaError_t launch_combine_partials(const PartialPtrs& pp, RankPartial* out, cudaStream_t s);
cudaError_t launch_decide_global(const PartialPtrs& partials, DevState* st, DecideParams p, cudaStream_t s);
cudaError_t launch_adam(const AdamArgs& a, int grid, cudaStream_t s, int variant);
int adam_ctas_per_sm(int variant);
// the largest co-resident grid of the fused small step (0: not available)
int step_small_max_grid(const StepSmallArgs& a);
cudaError_t launch_step_small(const StepSmallArgs& a, int grid, cudaStream_t s);
bool adam_variant_is_tma(int variant);
cudaError_t launch_copy(const CopyArgs& a, int grid, cudaStream_t s);
cudaError_t launch_load(const LoadArgs& a, cudaStream_t s);
cudaError_t launch_init_state(DevState* st, float S, float inv, cudaStream_t s);
cudaError_t launch_shard_io(const ShardIOArgs& a, cudaStream_t s);
cudaError_t launch_set_state(DevState* st, double b1t, double b2t, uint64_t t, float S, uint32_t good, float inv,
                             cudaStream_t s);
int sm_count();

}  // namespace zero
