// P_a / P_a+cpu: partitioned activation checkpoints over a model-parallel group
// (ZeRO-R, §6.1; communication §8).  The C ABI is
// declared in include/zero_b200.h; the partition rule is reading R-Pa1.
//
// The hot ops are HBM / NVLink / PCIe copies with no arithmetic:
//   save     this rank's slice of the replicated checkpoint -> the device store (the
//            engine's 128-bit copy kernel k_copy), or -> pinned host memory (P_a+cpu: a D2H on the
//            copy engine);
//   prefetch P_a+cpu: the slice -> the device staging slot (H2D, copy engine);
//   gather   every MP rank's slice -> the replicated checkpoint: PEER pulls all N_m
//            slices in one launch (grid row j reads rank j's store over the peer
//            table); NCCL runs an in-place all-gather into a staging buffer.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "zero_b200.h"
#include "zero_internal.h"

namespace {

using zero::kMaxRanks;
using zero::kThreads;

using PaCopyArgs = zero::CopyArgs;   // the engine's multi-row 16-bit copy kernel (k_copy)

int sm_count_dev() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

cudaError_t launch_pa_copy(const PaCopyArgs& a, cudaStream_t s) {
  uint64_t mx = 0;
  for (int j = 0; j < a.n; ++j) mx = std::max(mx, a.count[j]);
  if (a.n <= 0 || mx == 0) return cudaSuccess;
  static const int sms = sm_count_dev();
  // enough CTAs per source row to fill the GPU: rows x blocks ~ 4 CTAs per SM
  const uint64_t want = (mx + (uint64_t)kThreads * 32 - 1) / ((uint64_t)kThreads * 32);
  const int per_row = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)(4 * sms + a.n - 1) / a.n));
  return zero::launch_copy(a, per_row, s);
}

thread_local std::string g_pa_init_error;

}  // namespace

struct PaGroup;

struct zero_pa_ctx {
  int n_m = 1, rank = 0;
  uint32_t n_layers = 0;
  uint64_t numel = 0, padded = 0, slice = 0;
  int dtype = 0, offload = 0;
  zero_transport transport = ZERO_TRANSPORT_LOCAL;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  uint16_t* dev = nullptr;        // P_a: n_layers stores; P_a+cpu: one staging slot
  uint16_t* staging = nullptr;    // NCCL: `padded` elements for the in-place all-gather
  uint16_t* host = nullptr;       // P_a+cpu: n_layers stores (pinned)
  bool bound = false;
  std::vector<uint8_t> saved;     // per layer: saved since init
  int64_t staged_layer = -1;      // P_a+cpu: the layer held by the device staging slot
  PaGroup* group = nullptr;
  zero_pa_counters counters{};
  zero_status sticky = ZERO_OK;
  std::string err;

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
  uint64_t store_bytes() const { return (uint64_t)n_layers * slice * 2; }
  uint64_t device_bytes() const {
    uint64_t b = offload ? slice * 2 : store_bytes();
    if (transport == ZERO_TRANSPORT_NCCL) b = (b + 255) / 256 * 256 + padded * 2;
    return b;
  }
  uint64_t host_bytes() const { return offload ? store_bytes() : 0; }
  // element count of rank j's slice that lies inside the checkpoint
  uint64_t valid(int j) const {
    const uint64_t lo = (uint64_t)j * slice;
    return lo >= numel ? 0 : std::min(slice, numel - lo);
  }
  // where rank j's slice of `layer` is readable on the device at gather time
  const uint16_t* dev_slice(uint32_t layer) const { return offload ? dev : dev + (uint64_t)layer * slice; }
};

struct PaGroup {
  int n = 0;
  zero_pa_ctx* ranks[kMaxRanks] = {};
};

#define PCK(expr)                                                                             \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) return c->fail(ZERO_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)
#define PNK(expr)                                                                             \
  do {                                                                                        \
    ncclResult_t r_ = (expr);                                                                 \
    if (r_ != ncclSuccess) return c->fail(ZERO_ENCCL, "%s: %s", #expr, ncclGetErrorString(r_)); \
  } while (0)
#define PSTICKY(c)                                 \
  do {                                             \
    if (!(c)) return ZERO_EINVAL;                  \
    if ((c)->sticky != ZERO_OK) return (c)->sticky; \
  } while (0)

extern "C" {

zero_status zero_pa_init(int n_m, int rank, uint32_t n_layers, uint64_t numel, zero_dtype dtype, int offload,
                         zero_transport transport, void* nccl_comm, void* stream, zero_pa_ctx** out) {
  auto bad = [](const char* m) { g_pa_init_error = m; return ZERO_EINVAL; };
  if (!out) return bad("out is NULL");
  *out = nullptr;
  if (n_m < 1 || n_m > kMaxRanks) return bad("n_m outside 1..ZERO_MAX_RANKS");
  if (rank < 0 || rank >= n_m) return bad("rank outside 0..n_m-1");
  if (n_layers == 0 || numel == 0) return bad("n_layers and numel must be positive");
  if (dtype != ZERO_FP16 && dtype != ZERO_BF16) return bad("dtype must be FP16 or BF16");
  if (offload != 0 && offload != 1) return bad("offload must be 0 (P_a) or 1 (P_a+cpu)");
  if (transport == ZERO_TRANSPORT_PEER && n_m == 1) transport = ZERO_TRANSPORT_LOCAL;
  if (transport == ZERO_TRANSPORT_LOCAL && n_m != 1) return bad("LOCAL transport needs n_m == 1");
  if (transport == ZERO_TRANSPORT_NCCL && !nccl_comm) return bad("NCCL transport needs a communicator");
  if (transport != ZERO_TRANSPORT_LOCAL && transport != ZERO_TRANSPORT_PEER && transport != ZERO_TRANSPORT_NCCL)
    return bad("unknown transport");
  auto* c = new zero_pa_ctx();
  c->n_m = n_m;
  c->rank = rank;
  c->n_layers = n_layers;
  c->numel = numel;
  const uint64_t q = (uint64_t)n_m * 8;  // reading R-Pa1: 16-byte granules per rank
  c->padded = (numel + q - 1) / q * q;
  c->slice = c->padded / n_m;
  c->dtype = dtype;
  c->offload = offload;
  c->transport = transport;
  c->comm = reinterpret_cast<ncclComm_t>(nccl_comm);
  c->stream = reinterpret_cast<cudaStream_t>(stream);
  c->saved.assign(n_layers, 0);
  *out = c;
  return ZERO_OK;
}

zero_status zero_pa_get_info(const zero_pa_ctx* c, zero_pa_info* out) {
  if (!c || !out) return ZERO_EINVAL;
  out->numel = c->numel;
  out->padded = c->padded;
  out->slice = c->slice;
  out->device_bytes = c->device_bytes();
  out->host_bytes = c->host_bytes();
  out->n_layers = c->n_layers;
  out->n_m = (uint32_t)c->n_m;
  out->rank = (uint32_t)c->rank;
  out->offload = (uint32_t)c->offload;
  return ZERO_OK;
}

zero_status zero_pa_bind(zero_pa_ctx* c, void* device_arena, void* host_arena) {
  PSTICKY(c);
  if (c->bound) return c->fail(ZERO_ESTATE, "arenas already bound");
  if (!device_arena) return c->fail(ZERO_EINVAL, "device arena is NULL");
  if (reinterpret_cast<uintptr_t>(device_arena) & 255) return c->fail(ZERO_EINVAL, "device arena not 256-B aligned");
  if (c->offload && !host_arena) return c->fail(ZERO_EINVAL, "P_a+cpu needs a pinned host arena");
  if (c->offload) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, host_arena) != cudaSuccess || at.type != cudaMemoryTypeHost) {
      cudaGetLastError();
      return c->fail(ZERO_EINVAL, "host arena is not pinned (page-locked) host memory");
    }
  }
  c->dev = reinterpret_cast<uint16_t*>(device_arena);
  if (c->transport == ZERO_TRANSPORT_NCCL) {
    const uint64_t b = c->offload ? c->slice * 2 : c->store_bytes();
    c->staging = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(device_arena) + (b + 255) / 256 * 256);
  }
  c->host = reinterpret_cast<uint16_t*>(host_arena);
  c->bound = true;
  return ZERO_OK;
}

zero_status zero_pa_sim_group(zero_pa_ctx* const* ranks, int n) {
  if (!ranks || n < 2 || n > kMaxRanks) return ZERO_EINVAL;
  for (int r = 0; r < n; ++r) {
    zero_pa_ctx* c = ranks[r];
    if (!c || c->rank != r || c->n_m != n || c->transport != ZERO_TRANSPORT_PEER || !c->bound || c->group)
      return ZERO_EINVAL;
    const zero_pa_ctx* a = ranks[0];
    if (c->numel != a->numel || c->n_layers != a->n_layers || c->dtype != a->dtype || c->offload != a->offload ||
        c->stream != a->stream)
      return c->fail(ZERO_EINVAL, "group members differ in numel/layers/dtype/offload/stream");
  }
  auto* g = new PaGroup();
  g->n = n;
  for (int r = 0; r < n; ++r) {
    g->ranks[r] = ranks[r];
    ranks[r]->group = g;
  }
  return ZERO_OK;
}

zero_status zero_pa_save(zero_pa_ctx* c, uint32_t layer, const void* act) {
  PSTICKY(c);
  if (!c->bound) return c->fail(ZERO_ESTATE, "arenas not bound");
  if (layer >= c->n_layers) return c->fail(ZERO_EINVAL, "layer %u out of range", layer);
  if (!act) return c->fail(ZERO_EINVAL, "act is NULL");
  if (c->transport == ZERO_TRANSPORT_PEER && !c->group) return c->fail(ZERO_ESTATE, "PEER context not in a group");
  const uint64_t lo = (uint64_t)c->rank * c->slice, nv = c->valid(c->rank);
  const uint16_t* src = reinterpret_cast<const uint16_t*>(act) + lo;
  if (c->offload) {  // P_a+cpu: straight to the pinned host store on the copy engine
    uint16_t* dst = c->host + (uint64_t)layer * c->slice;
    if (nv) PCK(cudaMemcpyAsync(dst, src, nv * 2, cudaMemcpyDeviceToHost, c->stream));
    if (nv < c->slice && !c->saved[layer]) std::fill(dst + nv, dst + c->slice, (uint16_t)0);  // padding (host-owned)
    c->counters.d2h_bytes += nv * 2;
  } else {
    uint16_t* dst = c->dev + (uint64_t)layer * c->slice;
    PaCopyArgs a{};
    a.n = 1;
    a.src[0] = src;
    a.dst[0] = dst;
    a.count[0] = nv;
    PCK(launch_pa_copy(a, c->stream));
    if (nv < c->slice) PCK(cudaMemsetAsync(dst + nv, 0, (c->slice - nv) * 2, c->stream));
  }
  c->counters.saved_elems += nv;
  c->saved[layer] = 1;
  if (c->staged_layer == (int64_t)layer) c->staged_layer = -1;  // the staged copy is stale
  return ZERO_OK;
}

zero_status zero_pa_prefetch(zero_pa_ctx* c, uint32_t layer) {
  PSTICKY(c);
  if (!c->bound) return c->fail(ZERO_ESTATE, "arenas not bound");
  if (layer >= c->n_layers) return c->fail(ZERO_EINVAL, "layer %u out of range", layer);
  if (!c->saved[layer]) return c->fail(ZERO_ESTATE, "layer %u was never saved", layer);
  if (!c->offload) return ZERO_OK;
  // NCCL: land the slice at this rank's offset of the all-gather staging (in place)
  uint16_t* dst = c->transport == ZERO_TRANSPORT_NCCL ? c->staging + (uint64_t)c->rank * c->slice : c->dev;
  PCK(cudaMemcpyAsync(dst, c->host + (uint64_t)layer * c->slice, c->slice * 2, cudaMemcpyHostToDevice, c->stream));
  c->counters.h2d_bytes += c->slice * 2;
  c->staged_layer = layer;
  return ZERO_OK;
}

zero_status zero_pa_gather(zero_pa_ctx* c, uint32_t layer, void* act_out) {
  PSTICKY(c);
  if (!c->bound) return c->fail(ZERO_ESTATE, "arenas not bound");
  if (layer >= c->n_layers) return c->fail(ZERO_EINVAL, "layer %u out of range", layer);
  if (!act_out) return c->fail(ZERO_EINVAL, "act_out is NULL");
  uint16_t* out = reinterpret_cast<uint16_t*>(act_out);
  auto ready = [&](const zero_pa_ctx* r) { return r->offload ? r->staged_layer == (int64_t)layer : r->saved[layer] != 0; };
  if (c->transport == ZERO_TRANSPORT_NCCL) {
    if (!ready(c)) return c->fail(ZERO_ESTATE, "layer %u not %s on this rank", layer, c->offload ? "prefetched" : "saved");
    const ncclDataType_t dt = c->dtype == ZERO_FP16 ? ncclFloat16 : ncclBfloat16;
    uint16_t* mine = c->staging + (uint64_t)c->rank * c->slice;
    if (!c->offload) {
      PaCopyArgs m{};
      m.n = 1;
      m.src[0] = c->dev_slice(layer);
      m.dst[0] = mine;
      m.count[0] = c->slice;
      PCK(launch_pa_copy(m, c->stream));
    }
    PNK(ncclAllGather(mine, c->staging, c->slice, dt, c->comm, c->stream));
    PaCopyArgs a{};
    a.n = 1;
    a.src[0] = c->staging;
    a.dst[0] = out;
    a.count[0] = c->numel;
    PCK(launch_pa_copy(a, c->stream));
    c->counters.gathered_elems += c->numel - c->valid(c->rank);
    if (c->offload) c->staged_layer = -1;  // the staging buffer now holds the gathered copy
    return ZERO_OK;
  }
  PaCopyArgs a{};
  a.n = c->n_m;
  for (int j = 0; j < c->n_m; ++j) {
    const zero_pa_ctx* r = c->group ? c->group->ranks[j] : c;
    if (!ready(r))
      return c->fail(ZERO_ESTATE, "rank %d has not %s layer %u", j, r->offload ? "prefetched" : "saved", layer);
    a.src[j] = r->dev_slice(layer);
    a.dst[j] = out + (uint64_t)j * c->slice;
    a.count[j] = c->valid(j);
    if (j != c->rank) c->counters.gathered_elems += c->valid(j);
  }
  PCK(launch_pa_copy(a, c->stream));
  return ZERO_OK;
}

zero_status zero_pa_get_counters(const zero_pa_ctx* c, zero_pa_counters* out) {
  if (!c || !out) return ZERO_EINVAL;
  *out = c->counters;
  return ZERO_OK;
}

const char* zero_pa_last_error(const zero_pa_ctx* c) { return c ? c->err.c_str() : g_pa_init_error.c_str(); }

void zero_pa_destroy(zero_pa_ctx* c) {
  if (!c) return;
  if (c->bound) cudaStreamSynchronize(c->stream);
  if (PaGroup* g = c->group) {
    for (int r = 0; r < g->n; ++r)
      if (g->ranks[r]) g->ranks[r]->group = nullptr;
    delete g;
  }
  delete c;
}

uint64_t zero_pa_checkpoint_bytes(uint64_t layers, uint64_t batch, uint64_t seq, uint64_t hidden, int n_m,
                                  int elem_bytes) {
  if (n_m < 1 || elem_bytes < 1) return 0;
  const unsigned __int128 b = (unsigned __int128)layers * batch * seq * hidden * (unsigned)elem_bytes;
  return (uint64_t)(b / (unsigned)n_m);
}

}  // extern "C"
