// sm_100a kernels of the ZeRO-DP hot path (arXiv 1910.02054).
//
// Every kernel here is a bandwidth-bound streaming pass (no dense
// contraction on the path, so no tensor cores).  Design rules applied:
//  * 256-bit (LDG.E.256 / STG.E.256) accesses for fp32 streams and 128-bit for
//    16-bit streams, with L1::no_allocate (no reuse within a step);
//  * persistent grids sized from the SM count; contiguous per-CTA ranges;
//  * reductions (overflow flag, sum of squares for the global grad norm)
//    are warp-shuffle + shared-memory trees in fp64 with a last-CTA combine in a
//    fixed order, so results are deterministic run to run;
//  * fp32 arithmetic uses the __f*_rn intrinsics in the op order of reading c-3
//    (never contracted to FMA), conversions are cvt.rn (reading c-5).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <atomic>
#include <cstdint>

#include "zero_internal.h"

namespace zero {

// ---------------------------------------------------------------------------
// 16-bit formats
// ---------------------------------------------------------------------------
template <int DT>
struct H16;
template <>
struct H16<DT_F16> {
  static __device__ __forceinline__ float widen(uint32_t b) { return __half2float(__ushort_as_half((unsigned short)b)); }
  static __device__ __forceinline__ uint32_t narrow(float x) { return __half_as_ushort(__float2half_rn(x)); }
  static __device__ __forceinline__ uint32_t nonfinite(uint32_t b) { return (b & 0x7C00u) == 0x7C00u; }
};
template <>
struct H16<DT_BF16> {
  static __device__ __forceinline__ float widen(uint32_t b) { return __uint_as_float(b << 16); }
  static __device__ __forceinline__ uint32_t narrow(float x) { return __bfloat16_as_ushort(__float2bfloat16_rn(x)); }
  static __device__ __forceinline__ uint32_t nonfinite(uint32_t b) { return (b & 0x7F80u) == 0x7F80u; }
};

// ---------------------------------------------------------------------------
// streaming vector accesses
// ---------------------------------------------------------------------------
struct U8 { uint32_t x[8]; };
struct U4 { uint32_t x[4]; };

__device__ __forceinline__ U8 ld256(const void* p) {
  U8 r;
  asm volatile("ld.global.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.x[0]), "=r"(r.x[1]), "=r"(r.x[2]), "=r"(r.x[3]), "=r"(r.x[4]), "=r"(r.x[5]),
                 "=r"(r.x[6]), "=r"(r.x[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st256(void* p, const U8& r) {
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r.x[0]),
               "r"(r.x[1]), "r"(r.x[2]), "r"(r.x[3]), "r"(r.x[4]), "r"(r.x[5]), "r"(r.x[6]), "r"(r.x[7])
               : "memory");
}
__device__ __forceinline__ U4 ld128(const void* p) {
  U4 r;
  asm volatile("ld.global.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x[0]), "=r"(r.x[1]), "=r"(r.x[2]), "=r"(r.x[3])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st128(void* p, const U4& r) {
  asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(r.x[0]), "r"(r.x[1]),
               "r"(r.x[2]), "r"(r.x[3])
               : "memory");
}
__host__ __device__ __forceinline__ bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

// cross-process signalling (system scope)
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// A peer that never signals (a crashed rank, a protocol bug) must not wedge the GPU:
// after kSpinTimeoutNs of waiting the kernel traps, which surfaces as a sticky CUDA
// error in this process (ZERO_ECUDA) and leaves the device usable.
constexpr uint64_t kSpinTimeoutNs = 300ull * 1000000000ull;
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void wait_all(const uint64_t* flags, int n, uint64_t epoch) {
  const uint64_t t0 = globaltimer_ns();
  for (int j = 0; j < n; ++j)
    while (ld_acquire_sys(flags + j) < epoch) {
      __nanosleep(100);
      if (globaltimer_ns() - t0 > kSpinTimeoutNs) __trap();
    }
}

// TMA (cp.async.bulk) + mbarrier helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void lds128(const void* p, uint32_t (&r)[4]) {
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(smem_u32(p)));
}

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void sts128(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(p)), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void lds64(const void* p, uint32_t& a, uint32_t& b) {
  asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void sts64(void* p, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.b32 [%0], {%1,%2};" ::"r"(smem_u32(p)), "r"(a), "r"(b) : "memory");
}

// opt a kernel in to > 48 KB of dynamic shared memory, once per device
template <typename Kernel>
cudaError_t allow_dynamic_smem(Kernel k, size_t smem, std::atomic<uint64_t>& done) {
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  if (cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) return e;
  done.fetch_or(bit, std::memory_order_release);
  return cudaSuccess;
}

// 8 16-bit values packed in a U4
__device__ __forceinline__ uint32_t h_get(const U4& v, int j) { return (v.x[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu; }
__device__ __forceinline__ void h_set(U4& v, int j, uint32_t b) {
  if (j & 1) v.x[j >> 1] = (v.x[j >> 1] & 0x0000FFFFu) | (b << 16);
  else v.x[j >> 1] = (v.x[j >> 1] & 0xFFFF0000u) | b;
}

// acc += (double)u * (double)u with the fp32 -> fp64 widening done by integer ops for
// normal u (exact: rebias the exponent, shift the significand), keeping the
// conversion pipe (XU) free for the casts; zero, subnormal, inf and nan take cvt.
__device__ __noinline__ double f32_to_f64_slow(float u) { return (double)u; }  // a real branch, not a predicated cvt
__device__ __forceinline__ void sq_acc(double& acc, float u) {
  const uint32_t b = __float_as_uint(u) & 0x7FFFFFFFu;
  const uint32_t e = b >> 23;
  double d;
  if (e - 1u < 254u) d = __longlong_as_double(((uint64_t)b + (896ull << 23)) << 29);
  else if (b == 0) d = 0.0;
  else d = f32_to_f64_slow(u);
  acc += d * d;
}

// ---------------------------------------------------------------------------
// deterministic fp64 sum + OR flag over a grid (last-CTA combine)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// returns the block total in thread 0 (fixed order: butterfly, then warps ascending)
__device__ __forceinline__ void block_reduce(double& s, uint32_t& f) {
  __shared__ double ws[32];
  __shared__ uint32_t wf[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  s = warp_sum(s);
  f = __reduce_or_sync(0xffffffffu, f);
  __syncthreads();  // ws may be reused by a previous call
  if (lane == 0) { ws[warp] = s; wf[warp] = f; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    uint32_t b = 0;
    for (int i = 0; i < nw; ++i) { a += ws[i]; b |= wf[i]; }
    s = a;
    f = b;
  }
}

__device__ void grid_publish(double s, uint32_t f, GridPartials* part, Slot* slot, uint64_t* const* done_sig = nullptr,
                             int n_done = 0, uint64_t epoch = 0) {
  __shared__ bool is_last;
  block_reduce(s, f);
  if (threadIdx.x == 0) {
    part->sumsq[blockIdx.x] = s;
    part->flag[blockIdx.x] = f;
    __threadfence();
    const unsigned t = atomicAdd(&part->ticket, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double a = 0.0;
  uint32_t b = 0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
    a += __ldcg(&part->sumsq[i]);
    b |= __ldcg(&part->flag[i]);
  }
  block_reduce(a, b);
  if (threadIdx.x == 0) {
    slot->sumsq = a;
    slot->flag = b;
    part->ticket = 0;
    if (n_done) {  // every CTA has consumed its peer data: tell the peers
      __threadfence_system();
      for (int j = 0; j < n_done; ++j) st_release_sys(done_sig[j], epoch);
    }
  }
}

// the state fields the decision reads, loaded in one batch (independent loads, no branch
// between them): a caller on a latency-bound path issues them early (flat_decide)
__device__ __forceinline__ DevSnap snap_state(const DevState* st) {
  DevSnap s;
  s.b1t = __ldcg(&st->b1t);
  s.b2t = __ldcg(&st->b2t);
  s.t = __ldcg(&st->t);
  s.S = __ldcg(&st->S);
  s.good = __ldcg(&st->good);
  s.inv_cur = __ldcg(&st->inv_cur);
  return s;
}

__device__ void decide_apply(double sum, double flags, const DevSnap& s0, DevState* st, const DecideParams& p);
__device__ void decide_apply(double sum, double flags, DevState* st, const DecideParams& p);

// the last CTA of a whole-step flatten (N_d = 1, every bucket in one launch): sum the per-CTA
// partials in CTA order and make the decision -- k_decide_local_slots + k_decide_global fused
__device__ __noinline__ void flat_decide(const FlatArgs& a) {
  __shared__ bool is_last;
  __syncthreads();
  DevSnap snap;
  if (threadIdx.x == 0) {
    // the state is written only by this launch's last CTA, after every CTA's ticket: the
    // snapshot's loads overlap the fence and the ticket instead of following the reduction
    snap = snap_state(a.decide_st);
    __threadfence();
    is_last = atomicAdd(&a.decide_part->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double s = 0.0;
  uint32_t f = 0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
    s += __ldcg(&a.cta_sum[i]);
    f |= __ldcg(&a.cta_flag[i]);
  }
  block_reduce(s, f);
  if (threadIdx.x == 0) {
    a.decide_part->ticket = 0;
    a.decide_out->sumsq = s;
    a.decide_out->flag = f ? 1.0 : 0.0;
    decide_apply(s, f ? 1.0 : 0.0, snap, a.decide_st, a.decide);
  }
}

// the flatten's N_d = 1 epilogue: per-CTA partials (k_decide_local combines them in a
// fixed order), or the last-CTA grid combine into the slot
__device__ __forceinline__ void flat_publish(const FlatArgs& a, double s, uint32_t f) {
  if (a.cta_sum) {
    block_reduce(s, f);
    if (threadIdx.x == 0) {
      a.cta_sum[blockIdx.x] = s;
      a.cta_flag[blockIdx.x] = f;
      if (blockIdx.x == 0) *a.cta_grid = gridDim.x;
    }
    if (blockIdx.x == 0)
      for (uint32_t i = threadIdx.x; i < a.clear_slots; i += blockDim.x) a.cta_grid[1 + i] = 0u;
    if (a.decide_st) flat_decide(a);
  } else {
    grid_publish(s, f, a.part, a.slot);
  }
}

// ---------------------------------------------------------------------------
// K2: flatten / cast / prescale one gradient bucket (a1), + epilogue at N_d = 1
// ---------------------------------------------------------------------------
// chunk = 256 threads x V vectors x 8 elements; V is a template parameter

template <int SDT>
struct SrcLoad;
template <>
struct SrcLoad<DT_F16> {
  static constexpr int kBytes = 2;
  static __device__ __forceinline__ void vec(const void* p, float (&x)[8]) {
    U4 v = ld128(p);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = H16<DT_F16>::widen(h_get(v, j));
  }
  static __device__ __forceinline__ float one(const void* p, uint64_t i) {
    return H16<DT_F16>::widen(reinterpret_cast<const uint16_t*>(p)[i]);
  }
};
template <>
struct SrcLoad<DT_BF16> {
  static constexpr int kBytes = 2;
  static __device__ __forceinline__ void vec(const void* p, float (&x)[8]) {
    U4 v = ld128(p);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = H16<DT_BF16>::widen(h_get(v, j));
  }
  static __device__ __forceinline__ float one(const void* p, uint64_t i) {
    return H16<DT_BF16>::widen(reinterpret_cast<const uint16_t*>(p)[i]);
  }
};
template <>
struct SrcLoad<DT_F32> {
  static constexpr int kBytes = 4;
  static __device__ __forceinline__ void vec(const void* p, float (&x)[8]) {
    U8 v = ld256(p);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __uint_as_float(v.x[j]);
  }
  static __device__ __forceinline__ float one(const void* p, uint64_t i) { return reinterpret_cast<const float*>(p)[i]; }
};

// g' = RTNE16(widen(g) * sigma): a plain bit copy when sigma == 1 and the dtypes match.
// The pieces tile the destination range [pieces[0].dst_off, last end) contiguously
// (data pieces and zero pieces for alignment gaps / padding).  CTA b handles the
// contiguous slice [b*per_cta, (b+1)*per_cta) of that range, walking the pieces it
// overlaps; each thread keeps V 128-bit loads in flight.
// the N_d = 1 epilogue of one flattened 16-bit value b (reading c-4 / P:282):
//  kEpi 0: none; 1: u = fp32(b * inv), sum += u^2 (fp64), flag |= !finite(b);
//  2: inv is a power of two <= 1 (the usual case: 1/(S*sigma)), so u^2 = b^2 * inv^2 exactly
//     and the kernel scales the sum once; b^2 is formed from b's bits (normal numbers)
//     with integer ops, and the flag is read off the sum (finite iff every b is).
template <int DDT, int kEpi>
__device__ __forceinline__ void epi_elem(uint32_t b, float inv, double& sumsq, uint32_t& flag) {
  using D = H16<DDT>;
  if (kEpi == 1) {
    flag |= D::nonfinite(b);
    sq_acc(sumsq, __fmul_rn(D::widen(b), inv));
  } else if (kEpi == 2) {
    const uint32_t x = b & 0x7FFFu;
    constexpr uint32_t kMinNormal = DDT == DT_BF16 ? 0x0080u : 0x0400u;
    constexpr uint32_t kInf = DDT == DT_BF16 ? 0x7F80u : 0x7C00u;
    constexpr double kMinNormalValue = DDT == DT_BF16 ? 0x1p-126 : 0x1p-14;
    // rebias the exponent into fp64 (bias 1023): exact for normal numbers
    const uint32_t hi = DDT == DT_BF16 ? (x << 13) + (896u << 20) : (x << 10) + (1008u << 20);
    const double r = __hiloint2double((int)hi, 0);
    if (DDT == DT_BF16) {   // bf16 subnormals (< 2^-126) do not occur in practice: branch, not predicate
      if (x - kMinNormal < kInf - kMinNormal) sumsq = fma(r, r, sumsq);
      else if (x != 0) {
        const double d = f32_to_f64_slow(D::widen(b));           // subnormal, inf, nan
        sumsq = fma(d, d, sumsq);
      }
    } else {                // fp16 subnormals are common (|g| < 2^-14): handled inline, exactly
      double d;
      if (x - kMinNormal < kInf - kMinNormal) d = r;
      else if (x < kMinNormal) d = fma(2.0, r, -kMinNormalValue);   // zero / subnormal: 2r - min = m * 2^-24, exact
      else d = f32_to_f64_slow(D::widen(b));                         // inf / nan
      sumsq = fma(d, d, sumsq);
    }
  }
}

__device__ __forceinline__ bool pow2_at_most_one(float inv) {
  const uint32_t u = __float_as_uint(inv);
  return (u & 0x807FFFFFu) == 0u && u != 0u && inv <= 1.0f;   // +2^k, k <= 0, normal
}

template <int SDT, int DDT, bool kCopy, int V, int kEpi>
__device__ __forceinline__ void flatten_body(const FlatArgs& a, float inv, double& sumsq, uint32_t& flag) {
  using S = SrcLoad<SDT>;
  using D = H16<DDT>;
  const float sigma = a.sigma;
  uint16_t* dst_base = reinterpret_cast<uint16_t*>(a.dst);
  const uint64_t r0 = a.pieces[0].dst_off;
  const uint64_t r1 = a.pieces[a.n_pieces - 1].dst_off + a.pieces[a.n_pieces - 1].count;
  const uint64_t lo = r0 + (uint64_t)blockIdx.x * a.per_cta;
  const uint64_t hi = lo + a.per_cta < r1 ? lo + a.per_cta : r1;
  int p = 0;
  while (p + 1 < a.n_pieces && a.pieces[p + 1].dst_off <= lo) ++p;
  for (uint64_t cur = lo; cur < hi && p < a.n_pieces; ++p) {
    const FlatPiece pc = a.pieces[p];
    const uint64_t pend = pc.dst_off + pc.count < hi ? pc.dst_off + pc.count : hi;
    if (pend <= cur) continue;
    uint16_t* dst = dst_base + cur;                       // element 0 of this run
    const uint32_t n = (uint32_t)(pend - cur);
    if (pc.src == nullptr) {  // alignment gap or bucket padding: zeros (reading c-7)
      if (aligned(dst, 16)) {
        for (uint32_t i = threadIdx.x * 8; i < n; i += kThreads * 8) {
          if (i + 8 <= n) st128(dst + i, U4{{0u, 0u, 0u, 0u}});
          else for (uint32_t j = i; j < n; ++j) dst[j] = 0;
        }
      } else {
        for (uint32_t i = threadIdx.x; i < n; i += kThreads) dst[i] = 0;
      }
      cur = pend;
      continue;
    }
    const char* src = reinterpret_cast<const char*>(pc.src) + (cur - pc.dst_off) * S::kBytes;
    const bool vec = aligned(src, 8 * S::kBytes) && aligned(dst, 16);
    auto emit_one = [&](uint32_t j) {
      const float xv = S::one(src, j);
      const uint32_t b = kCopy ? D::narrow(xv) : D::narrow(__fmul_rn(xv, sigma));
      dst[j] = (uint16_t)b;
      epi_elem<DDT, kEpi>(b, inv, sumsq, flag);
    };
    auto emit8 = [&](uint32_t i, const float* x) {
      U4 o;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t b = kCopy ? D::narrow(x[j]) : D::narrow(__fmul_rn(x[j], sigma));
        h_set(o, j, b);
        epi_elem<DDT, kEpi>(b, inv, sumsq, flag);
      }
      st128(dst + i, o);
    };
    if (vec && kCopy && S::kBytes == 2) {  // same dtype, sigma = 1: move the bits
      const uint32_t nv = n & ~7u;
#pragma unroll 1
      for (uint32_t i0 = threadIdx.x * 8; i0 < nv; i0 += kThreads * 8 * V) {
        U4 r[V];
#pragma unroll
        for (int u = 0; u < V; ++u) {
          const uint32_t i = i0 + u * kThreads * 8;
          if (u == 0 || i < nv) r[u] = ld128(src + (uint64_t)i * 2);
        }
#pragma unroll
        for (int u = 0; u < V; ++u) {
          const uint32_t i = i0 + u * kThreads * 8;
          if (u == 0 || i < nv) {
            st128(dst + i, r[u]);
            if (kEpi) {
#pragma unroll
              for (int j = 0; j < 8; ++j) epi_elem<DDT, kEpi>(h_get(r[u], j), inv, sumsq, flag);
            }
          }
        }
      }
      for (uint32_t j = nv + threadIdx.x; j < n; j += kThreads) emit_one(j);
    } else if (vec) {
      const uint32_t nv = n & ~7u;
#pragma unroll 1
      for (uint32_t i0 = threadIdx.x * 8; i0 < nv; i0 += kThreads * 8 * V) {
        float x[V][8];
#pragma unroll
        for (int u = 0; u < V; ++u) {
          const uint32_t i = i0 + u * kThreads * 8;
          if (u == 0 || i < nv) S::vec(src + (uint64_t)i * S::kBytes, x[u]);
        }
#pragma unroll
        for (int u = 0; u < V; ++u) {
          const uint32_t i = i0 + u * kThreads * 8;
          if (u == 0 || i < nv) emit8(i, x[u]);
        }
      }
      for (uint32_t j = nv + threadIdx.x; j < n; j += kThreads) emit_one(j);
    } else {
      for (uint32_t j = threadIdx.x; j < n; j += kThreads) emit_one(j);
    }
    cur = pend;
  }
}

template <int SDT, int DDT, bool kCopy, int V>
__global__ void __launch_bounds__(kThreads, 6) k_flatten(const __grid_constant__ FlatArgs a) {  // <= 40 regs: +1 % (A/B)
  // PDL: the next bucket's flatten (independent data) may start as soon as every CTA
  // of this one is resident; a no-op without a programmatic dependent
  asm volatile("griddepcontrol.launch_dependents;");
  double sumsq = 0.0;
  uint32_t flag = 0;
  if (!a.epilogue) {
    flatten_body<SDT, DDT, kCopy, V, 0>(a, 0.0f, sumsq, flag);
  } else {
    const float inv = a.st->inv_cur;
    if (pow2_at_most_one(inv)) {
      flatten_body<SDT, DDT, kCopy, V, 2>(a, inv, sumsq, flag);
      flag = isfinite(sumsq) ? 0u : 1u;          // b^2 of a finite 16-bit value is finite in fp64
      sumsq *= (double)inv * (double)inv;        // exact: a power of two, no under/overflow
    } else {
      flatten_body<SDT, DDT, kCopy, V, 1>(a, inv, sumsq, flag);
    }
    flat_publish(a, sumsq, flag);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: complete only after the previous flatten
}

template <typename Kernel>
cudaError_t launch_pdl(Kernel kern, int grid, cudaStream_t s, const FlatArgs& a) {
  if (!a.pdl) {
    kern<<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int V>
cudaError_t launch_flatten_v(const FlatArgs& a, int grid, cudaStream_t s) {
  const bool copy = (a.sigma == 1.0f) && (a.src_dtype == a.dst_dtype);
#define ZL(SD, DD, CP) launch_pdl(k_flatten<SD, DD, CP, V>, grid, s, a)
  if (a.dst_dtype == DT_F16) {
    if (a.src_dtype == DT_F16) { if (copy) ZL(DT_F16, DT_F16, true); else ZL(DT_F16, DT_F16, false); }
    else if (a.src_dtype == DT_F32) ZL(DT_F32, DT_F16, false);
    else return cudaErrorInvalidValue;
  } else if (a.dst_dtype == DT_BF16) {
    if (a.src_dtype == DT_BF16) { if (copy) ZL(DT_BF16, DT_BF16, true); else ZL(DT_BF16, DT_BF16, false); }
    else if (a.src_dtype == DT_F32) ZL(DT_F32, DT_BF16, false);
    else return cudaErrorInvalidValue;
  } else {
    return cudaErrorInvalidValue;
  }
#undef ZL
  return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// K2 (fp32 bucket, R32 over NCCL): the same cast/prescale -- g' = RTNE16(widen(g) *
// sigma), the 16-bit value the oracle sums (c-2) -- stored widened to fp32, so that
// ncclReduceScatter sums fp32 values and no partial sum is rounded to 16-bit on the
// wire.  No epilogue: the flag and norm are taken after the reduction.
// ---------------------------------------------------------------------------
template <int SDT, int DDT>
__global__ void __launch_bounds__(kThreads) k_flatten_wide(const __grid_constant__ FlatArgs a) {
  using S = SrcLoad<SDT>;
  using D = H16<DDT>;
  const bool copy = a.sigma == 1.0f && SDT == DDT;
  float* dst_base = reinterpret_cast<float*>(a.dst);
  const uint64_t r0 = a.pieces[0].dst_off;
  const uint64_t r1 = a.pieces[a.n_pieces - 1].dst_off + a.pieces[a.n_pieces - 1].count;
  const uint64_t lo = r0 + (uint64_t)blockIdx.x * a.per_cta;
  const uint64_t hi = lo + a.per_cta < r1 ? lo + a.per_cta : r1;
  int p = 0;
  while (p + 1 < a.n_pieces && a.pieces[p + 1].dst_off <= lo) ++p;
  for (uint64_t cur = lo; cur < hi && p < a.n_pieces; ++p) {
    const FlatPiece pc = a.pieces[p];
    const uint64_t pend = pc.dst_off + pc.count < hi ? pc.dst_off + pc.count : hi;
    if (pend <= cur) continue;
    float* dst = dst_base + cur;
    const uint32_t n = (uint32_t)(pend - cur);
    if (pc.src == nullptr) {  // alignment gap or padding: zeros (reading c-7)
      for (uint32_t i = threadIdx.x; i < n; i += kThreads) dst[i] = 0.0f;
      cur = pend;
      continue;
    }
    const char* src = reinterpret_cast<const char*>(pc.src) + (cur - pc.dst_off) * S::kBytes;
    auto cast1 = [&](float x) { return D::widen(copy ? D::narrow(x) : D::narrow(__fmul_rn(x, a.sigma))); };
    if (aligned(src, 8 * S::kBytes) && aligned(dst, 32)) {
      const uint32_t nv = n & ~7u;
      for (uint32_t i = threadIdx.x * 8; i < nv; i += kThreads * 8) {
        float x[8];
        S::vec(src + (uint64_t)i * S::kBytes, x);
        U8 o;
#pragma unroll
        for (int j = 0; j < 8; ++j) o.x[j] = __float_as_uint(cast1(x[j]));
        st256(dst + i, o);
      }
      for (uint32_t j = nv + threadIdx.x; j < n; j += kThreads) dst[j] = cast1(S::one(src, j));
    } else {
      for (uint32_t j = threadIdx.x; j < n; j += kThreads) dst[j] = cast1(S::one(src, j));
    }
    cur = pend;
  }
}

cudaError_t launch_flatten_wide(const FlatArgs& a, int grid, cudaStream_t s) {
  if (a.dst_dtype == DT_F16) {
    if (a.src_dtype == DT_F16) k_flatten_wide<DT_F16, DT_F16><<<grid, kThreads, 0, s>>>(a);
    else if (a.src_dtype == DT_F32) k_flatten_wide<DT_F32, DT_F16><<<grid, kThreads, 0, s>>>(a);
    else return cudaErrorInvalidValue;
  } else if (a.dst_dtype == DT_BF16) {
    if (a.src_dtype == DT_BF16) k_flatten_wide<DT_BF16, DT_BF16><<<grid, kThreads, 0, s>>>(a);
    else if (a.src_dtype == DT_F32) k_flatten_wide<DT_F32, DT_BF16><<<grid, kThreads, 0, s>>>(a);
    else return cudaErrorInvalidValue;
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_flatten(const FlatArgs& a, int grid, cudaStream_t s, int vecs) {
  switch (vecs) {
    case 4: return launch_flatten_v<4>(a, grid, s);
    case 8: return launch_flatten_v<8>(a, grid, s);
    default: return launch_flatten_v<2>(a, grid, s);
  }
}

// ---------------------------------------------------------------------------
// K2 (TMA variant): the source pieces are streamed into shared memory by 1-D bulk
// copies (a STAGES-deep mbarrier ring fed by one producer warp); T/8 consumer
// threads cast/scale 8 elements each, compute the epilogue (N_d = 1) and store
// 128-bit.  Needs every piece offset/count % 8 == 0 and 16-B aligned sources.
// ---------------------------------------------------------------------------
struct FlatCursor {
  uint64_t cur, hi;
  int p;
  __device__ __forceinline__ bool next(const FlatArgs& a, uint32_t T, uint64_t& start, uint32_t& n, int& piece) {
    while (cur < hi && p < a.n_pieces) {
      const FlatPiece& pc = a.pieces[p];
      const uint64_t pend = pc.dst_off + pc.count < hi ? pc.dst_off + pc.count : hi;
      if (cur >= pend) { ++p; continue; }
      start = cur;
      const uint64_t left = pend - cur;
      n = left < T ? (uint32_t)left : T;
      piece = p;
      cur += n;
      return true;
    }
    return false;
  }
};

template <int SDT, int DDT, bool kCopy, int T, int STAGES>
__global__ void __launch_bounds__(T / 8 + 32, 1) k_flatten_tma(const __grid_constant__ FlatArgs a) {
  using S = SrcLoad<SDT>;
  using D = H16<DDT>;
  constexpr int kCons = T / 8;
  constexpr uint32_t kStageBytes = (uint32_t)T * S::kBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  const uint64_t r0 = a.pieces[0].dst_off;
  const uint64_t r1 = a.pieces[a.n_pieces - 1].dst_off + a.pieces[a.n_pieces - 1].count;
  const uint64_t lo = r0 + (uint64_t)blockIdx.x * a.per_cta;
  const uint64_t hi = lo + a.per_cta < r1 ? lo + a.per_cta : r1;
  int p0 = 0;
  while (p0 + 1 < a.n_pieces && a.pieces[p0 + 1].dst_off <= lo) ++p0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kCons / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double sumsq = 0.0;
  uint32_t flag = 0;
  if (warp == kCons / 32) {  // ---- producer
    if (lane == 0 && lo < hi) {
      const uint64_t pol = policy_evict_first();
      FlatCursor fc{lo, hi, p0};
      uint64_t start;
      uint32_t n;
      int piece;
      for (uint32_t it = 0; fc.next(a, T, start, n, piece); ++it) {
        const int st = it % STAGES;
        if (it >= (uint32_t)STAGES) mbar_wait(&empty[st], ((it / STAGES) - 1) & 1);
        const FlatPiece& pc = a.pieces[piece];
        if (pc.src == nullptr) {
          mbar_arrive(&full[st]);  // zero piece: nothing to load
        } else {
          mbar_expect_tx(&full[st], n * (uint32_t)S::kBytes);
          bulk_g2s(smem + st * kStageBytes,
                   reinterpret_cast<const char*>(pc.src) + (start - pc.dst_off) * S::kBytes, n * (uint32_t)S::kBytes,
                   &full[st], pol);
        }
      }
    }
  } else {  // ---- consumers
    const float sigma = a.sigma;
    const float inv = a.epilogue ? a.st->inv_cur : 0.0f;
    uint16_t* dst_base = reinterpret_cast<uint16_t*>(a.dst);
    FlatCursor fc{lo, hi, p0};
    uint64_t start;
    uint32_t n;
    int piece;
    for (uint32_t it = 0; fc.next(a, T, start, n, piece); ++it) {
      const int st = it % STAGES;
      mbar_wait(&full[st], (it / STAGES) & 1);
      const uint32_t e = threadIdx.x * 8;
      if (e < n) {
        U4 o;
        if (a.pieces[piece].src == nullptr) {
          o = U4{{0u, 0u, 0u, 0u}};
        } else {
          const unsigned char* sb = smem + st * kStageBytes + e * S::kBytes;
          float x[8];
          if (S::kBytes == 4) {
            uint32_t r[4];
            lds128(sb, r);
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = __uint_as_float(r[j]);
            lds128(sb + 16, r);
#pragma unroll
            for (int j = 0; j < 4; ++j) x[4 + j] = __uint_as_float(r[j]);
          } else {
            uint32_t r[4];
            lds128(sb, r);
            U4 g{{r[0], r[1], r[2], r[3]}};
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = H16<SDT == DT_F32 ? DT_F16 : SDT>::widen(h_get(g, j));
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t b = kCopy ? D::narrow(x[j]) : D::narrow(__fmul_rn(x[j], sigma));
            h_set(o, j, b);
            if (a.epilogue) {
              flag |= D::nonfinite(b);
              const float u = __fmul_rn(D::widen(b), inv);
              sq_acc(sumsq, u);
            }
          }
        }
        st128(dst_base + start + e, o);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
  if (a.epilogue) {
    __syncthreads();
    flat_publish(a, sumsq, flag);
  }
}

template <int SD, int DD, bool CP, int T, int STAGES>
cudaError_t launch_flatten_tma_t(const FlatArgs& a, int grid, cudaStream_t s) {
  const size_t smem = (size_t)STAGES * T * SrcLoad<SD>::kBytes + 2 * STAGES * sizeof(uint64_t);
  static std::atomic<uint64_t> configured{0};  // one bit per device
  if (cudaError_t e = allow_dynamic_smem(k_flatten_tma<SD, DD, CP, T, STAGES>, smem, configured)) return e;
  k_flatten_tma<SD, DD, CP, T, STAGES><<<grid, T / 8 + 32, smem, s>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K2 (TMA in + TMA out): the producer thread streams each chunk of the bucket's
// sources into shared memory with bulk loads and drains the finished chunk to the
// bucket with a bulk store before refilling the stage.  For a same-dtype copy at
// sigma = 1 the stage is stored as loaded and the consumers only read it (the N_d = 1
// epilogue); otherwise they write the cast/scaled 16-bit chunk into an output slot.
// Zero pieces (alignment gaps, padding) are zero-filled in shared memory.
// Needs every piece offset/count % 8 == 0, 16-B aligned sources and destination.
// ---------------------------------------------------------------------------
template <int SDT, int DDT, bool kCopy, int T, int STAGES>
__global__ void __launch_bounds__(T / 8 + 32) k_flatten_tma_st(const __grid_constant__ FlatArgs a) {
  using S = SrcLoad<SDT>;
  using D = H16<DDT>;
  constexpr int kCons = T / 8;
  constexpr uint32_t kInBytes = (uint32_t)T * S::kBytes;
  constexpr uint32_t kStageBytes = kInBytes + (kCopy ? 0u : (uint32_t)T * 2u);
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* done = full + STAGES;
  const uint64_t r0 = a.pieces[0].dst_off;
  const uint64_t r1 = a.pieces[a.n_pieces - 1].dst_off + a.pieces[a.n_pieces - 1].count;
  const uint64_t lo = r0 + (uint64_t)blockIdx.x * a.per_cta;
  const uint64_t hi = lo + a.per_cta < r1 ? lo + a.per_cta : r1;
  int p0 = 0;
  while (p0 + 1 < a.n_pieces && a.pieces[p0 + 1].dst_off <= lo) ++p0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&done[i], kCons / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double sumsq = 0.0;
  uint32_t flag = 0;
  uint16_t* dst_base = reinterpret_cast<uint16_t*>(a.dst);
  if (warp == kCons / 32) {  // ---- producer: loads ahead, stores behind
    if (lane == 0 && lo < hi) {
      const uint64_t pol = policy_evict_first();
      uint64_t pend_start[STAGES];
      uint32_t pend_n[STAGES];
      auto drain = [&](uint32_t j) {
        const int st = j % STAGES;
        mbar_wait(&done[st], (j / STAGES) & 1);
        bulk_s2g(dst_base + pend_start[st], smem + st * kStageBytes + (kCopy ? 0u : kInBytes), pend_n[st] * 2u, pol);
        bulk_commit();
      };
      FlatCursor fc{lo, hi, p0};
      uint64_t start;
      uint32_t n;
      int piece;
      uint32_t it = 0;
      for (; fc.next(a, T, start, n, piece); ++it) {
        const int st = it % STAGES;
        if (it >= (uint32_t)STAGES) {
          drain(it - STAGES);
          bulk_wait_read0();
        }
        pend_start[st] = start;
        pend_n[st] = n;
        const FlatPiece& pc = a.pieces[piece];
        if (pc.src == nullptr) {
          mbar_arrive(&full[st]);  // zero piece: the consumers fill the stage
        } else {
          mbar_expect_tx(&full[st], n * (uint32_t)S::kBytes);
          bulk_g2s(smem + st * kStageBytes,
                   reinterpret_cast<const char*>(pc.src) + (start - pc.dst_off) * S::kBytes, n * (uint32_t)S::kBytes,
                   &full[st], pol);
        }
      }
      for (uint32_t j = it > (uint32_t)STAGES ? it - STAGES : 0; j < it; ++j) drain(j);
      bulk_wait_all0();
    }
  } else {  // ---- consumers
    const float sigma = a.sigma;
    const float inv = a.epilogue ? a.st->inv_cur : 0.0f;
    FlatCursor fc{lo, hi, p0};
    uint64_t start;
    uint32_t n;
    int piece;
    for (uint32_t it = 0; fc.next(a, T, start, n, piece); ++it) {
      const int st = it % STAGES;
      mbar_wait(&full[st], (it / STAGES) & 1);
      unsigned char* sb = smem + st * kStageBytes;
      unsigned char* ob = sb + (kCopy ? 0u : kInBytes);
      const uint32_t e = threadIdx.x * 8;
      if (e < n) {
        if (a.pieces[piece].src == nullptr) {
          sts128(ob + e * 2, 0u, 0u, 0u, 0u);
        } else if (kCopy) {
          if (a.epilogue) {
            uint32_t r[4];
            lds128(sb + e * 2, r);
            U4 g{{r[0], r[1], r[2], r[3]}};
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint32_t b = h_get(g, j);
              flag |= D::nonfinite(b);
              sq_acc(sumsq, __fmul_rn(D::widen(b), inv));
            }
          }
        } else {
          float x[8];
          if (S::kBytes == 4) {
            uint32_t r[4];
            lds128(sb + e * 4, r);
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = __uint_as_float(r[j]);
            lds128(sb + e * 4 + 16, r);
#pragma unroll
            for (int j = 0; j < 4; ++j) x[4 + j] = __uint_as_float(r[j]);
          } else {
            uint32_t r[4];
            lds128(sb + e * 2, r);
            U4 g{{r[0], r[1], r[2], r[3]}};
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = H16<SDT == DT_F32 ? DT_F16 : SDT>::widen(h_get(g, j));
          }
          U4 o;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t b = D::narrow(__fmul_rn(x[j], sigma));
            h_set(o, j, b);
            if (a.epilogue) {
              flag |= D::nonfinite(b);
              sq_acc(sumsq, __fmul_rn(D::widen(b), inv));
            }
          }
          sts128(ob + e * 2, o.x[0], o.x[1], o.x[2], o.x[3]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&done[st]);
    }
  }
  if (a.epilogue) {
    __syncthreads();
    flat_publish(a, sumsq, flag);
  }
}

template <int SD, int DD, bool CP, int T, int STAGES>
cudaError_t launch_flatten_tma_st_t(const FlatArgs& a, int grid, cudaStream_t s) {
  const size_t smem = (size_t)STAGES * T * (SrcLoad<SD>::kBytes + (CP ? 0 : 2)) + 2 * STAGES * sizeof(uint64_t);
  static std::atomic<uint64_t> configured{0};  // one bit per device
  if (cudaError_t e = allow_dynamic_smem(k_flatten_tma_st<SD, DD, CP, T, STAGES>, smem, configured)) return e;
  k_flatten_tma_st<SD, DD, CP, T, STAGES><<<grid, T / 8 + 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <int T, int STAGES>
cudaError_t launch_flatten_tma_st_ts(const FlatArgs& a, int grid, cudaStream_t s) {
  const bool copy = (a.sigma == 1.0f) && (a.src_dtype == a.dst_dtype);
#define ZT(SD, DD, CP) return launch_flatten_tma_st_t<SD, DD, CP, T, STAGES>(a, grid, s)
  if (a.dst_dtype == DT_F16) {
    if (a.src_dtype == DT_F16) { if (copy) ZT(DT_F16, DT_F16, true); else ZT(DT_F16, DT_F16, false); }
    if (a.src_dtype == DT_F32) ZT(DT_F32, DT_F16, false);
  } else if (a.dst_dtype == DT_BF16) {
    if (a.src_dtype == DT_BF16) { if (copy) ZT(DT_BF16, DT_BF16, true); else ZT(DT_BF16, DT_BF16, false); }
    if (a.src_dtype == DT_F32) ZT(DT_F32, DT_BF16, false);
  }
#undef ZT
  return cudaErrorInvalidValue;
}

// TMA flatten (T 4096, 4 stages): measured 3.5 TB/s vs 4.2 TB/s for the register-staged
// k_flatten on one stream (round-1 sweep), so it is off by default (ZERO_FLAT_TMA=1).
// TMA in + TMA out (ZERO_FLAT_TMA=2): the reduce phase of the 1.5B step takes 1.38 ms vs
// 1.09 ms for k_flatten on three streams (4096x2 on 2 CTAs/SM 1.46 ms, 2048x4 on 2 CTAs/SM
// 1.44 ms), so it is off as well.
template <int T, int STAGES>
cudaError_t launch_flatten_tma_ts(const FlatArgs& a, int grid, cudaStream_t s) {
  const bool copy = (a.sigma == 1.0f) && (a.src_dtype == a.dst_dtype);
#define ZT(SD, DD, CP) return launch_flatten_tma_t<SD, DD, CP, T, STAGES>(a, grid, s)
  if (a.dst_dtype == DT_F16) {
    if (a.src_dtype == DT_F16) { if (copy) ZT(DT_F16, DT_F16, true); else ZT(DT_F16, DT_F16, false); }
    if (a.src_dtype == DT_F32) ZT(DT_F32, DT_F16, false);
  } else if (a.dst_dtype == DT_BF16) {
    if (a.src_dtype == DT_BF16) { if (copy) ZT(DT_BF16, DT_BF16, true); else ZT(DT_BF16, DT_BF16, false); }
    if (a.src_dtype == DT_F32) ZT(DT_F32, DT_BF16, false);
  }
#undef ZT
  return cudaErrorInvalidValue;
}

cudaError_t launch_flatten_tma(const FlatArgs& a, int grid, cudaStream_t s, int variant) {
  switch (variant) {
    case 2: return launch_flatten_tma_st_ts<4096, 4>(a, grid, s);
    default: return launch_flatten_tma_ts<4096, 4>(a, grid, s);
  }
}
int flatten_tma_ctas_per_sm(int) { return 1; }

// ---------------------------------------------------------------------------
// a2+a3: pull reduce-scatter of one bucket slice over a peer table (fp32 sum in
// ascending rank, one rounding for R16), fused with the overflow flag and the
// norm partial.  reduce == 0: epilogue only (slice already reduced by NCCL).
// ---------------------------------------------------------------------------
// NR: number of ranks known at compile time (2, 4, 8; 0 = a.n at run time).  U: 8-element
// groups per thread per iteration, so that U*NR 128-bit loads are in flight before the
// sums (NVLink latency is ~2 us: the pull needs many bytes in flight per SM).
// epilogue of one reduced value (as epi_elem): kEpi 1 = u = fp32(G * inv), flag per element;
// kEpi 2 = inv a power of two <= 1: sum G^2 (R32) or b^2 from the bits (R16), scaled and
// flagged once at the end of the kernel
template <int DT, bool kR32, int kEpi>
__device__ __forceinline__ void rs_epi(float G32, uint32_t b16, float inv, double& sumsq, uint32_t& flag) {
  using D = H16<DT>;
  if (kR32) {
    if (kEpi == 1) {
      flag |= (uint32_t)!isfinite(G32);
      sq_acc(sumsq, __fmul_rn(G32, inv));
    } else {
      sq_acc(sumsq, G32);
    }
  } else {
    if (kEpi == 1) {
      flag |= D::nonfinite(b16);
      sq_acc(sumsq, __fmul_rn(D::widen(b16), inv));
    } else {
      epi_elem<DT, 2>(b16, inv, sumsq, flag);
    }
  }
}

template <int DT, bool kR32, int kEpi>
__device__ __forceinline__ void rs_emit8(const RSArgs& a, uint64_t i, const float (&acc)[8], bool store, float inv,
                                         double& sumsq, uint32_t& flag) {
  using D = H16<DT>;
  if (kR32) {
    U8 o;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      o.x[j] = __float_as_uint(acc[j]);
      rs_epi<DT, true, kEpi>(acc[j], 0u, inv, sumsq, flag);
    }
    if (store) st256(reinterpret_cast<float*>(a.dst) + i, o);
  } else {
    U4 o;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t b = D::narrow(acc[j]);
      h_set(o, j, b);
      rs_epi<DT, false, kEpi>(0.0f, b, inv, sumsq, flag);
    }
    if (store) st128(reinterpret_cast<uint16_t*>(a.dst) + i, o);
  }
}

template <int DT, bool kR32, bool kReduce, bool kVec, int NR, int U, int kEpi>
__device__ __forceinline__ void rs_body(const RSArgs& a, float inv, double& sumsq, uint32_t& flag) {
  using D = H16<DT>;
  constexpr int R = NR > 0 ? NR : kMaxRanks;
  const int n = NR > 0 ? NR : a.n;
  const uint64_t step = (uint64_t)kThreads * (kVec ? 8 : 1);
  const uint64_t stride = (uint64_t)gridDim.x * step * (kVec ? U : 1);
  for (uint64_t i0 = ((uint64_t)blockIdx.x * kThreads * (kVec ? U : 1) + threadIdx.x) * (kVec ? 8 : 1); i0 < a.count;
       i0 += stride) {
    if (kVec && i0 + 8 <= a.count) {
      if (kReduce) {
        U4 v[U][R];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t i = i0 + (uint64_t)u * step;
          if (u == 0 || i + 8 <= a.count) {
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (NR > 0 || r < n) v[u][r] = ld128(reinterpret_cast<const uint16_t*>(a.src[r]) + i);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t i = i0 + (uint64_t)u * step;
          if (u == 0 || i + 8 <= a.count) {
            float acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = D::widen(h_get(v[u][0], j));
#pragma unroll
            for (int r = 1; r < R; ++r)
              if (NR > 0 || r < n) {
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], D::widen(h_get(v[u][r], j)));
              }
            rs_emit8<DT, kR32, kEpi>(a, i, acc, true, inv, sumsq, flag);
          } else if (i < a.count) {
            for (uint64_t k = i; k < a.count; ++k) {   // ragged tail of the second group
              float acc = D::widen(reinterpret_cast<const uint16_t*>(a.src[0])[k]);
              for (int r = 1; r < n; ++r) acc = __fadd_rn(acc, D::widen(reinterpret_cast<const uint16_t*>(a.src[r])[k]));
              if (kR32) {
                reinterpret_cast<float*>(a.dst)[k] = acc;
                rs_epi<DT, true, kEpi>(acc, 0u, inv, sumsq, flag);
              } else {
                const uint32_t b = D::narrow(acc);
                reinterpret_cast<uint16_t*>(a.dst)[k] = (uint16_t)b;
                rs_epi<DT, false, kEpi>(0.0f, b, inv, sumsq, flag);
              }
            }
          }
        }
      } else {  // epilogue only over the (NCCL-)reduced slice
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t i = i0 + (uint64_t)u * step;
          if (!(u == 0 || i + 8 <= a.count)) {
            for (uint64_t k = i; k < a.count; ++k) {
              if (kR32) rs_epi<DT, true, kEpi>(reinterpret_cast<const float*>(a.dst)[k], 0u, inv, sumsq, flag);
              else rs_epi<DT, false, kEpi>(0.0f, reinterpret_cast<const uint16_t*>(a.dst)[k], inv, sumsq, flag);
            }
            continue;
          }
          float acc[8];
          if (kR32) {
            U8 w = ld256(reinterpret_cast<const float*>(a.dst) + i);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = __uint_as_float(w.x[j]);
          } else {
            U4 w = ld128(reinterpret_cast<const uint16_t*>(a.dst) + i);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = D::widen(h_get(w, j));
          }
          rs_emit8<DT, kR32, kEpi>(a, i, acc, false, inv, sumsq, flag);
        }
      }
    } else {
      const uint64_t e = kVec ? (a.count < i0 + 8 ? a.count : i0 + 8) : i0 + 1;
      for (uint64_t k = i0; k < e; ++k) {
        float acc;
        if (kReduce) {
          acc = D::widen(reinterpret_cast<const uint16_t*>(a.src[0])[k]);
          for (int r = 1; r < n; ++r) acc = __fadd_rn(acc, D::widen(reinterpret_cast<const uint16_t*>(a.src[r])[k]));
        } else if (kR32) {
          acc = reinterpret_cast<const float*>(a.dst)[k];
        } else {
          acc = D::widen(reinterpret_cast<const uint16_t*>(a.dst)[k]);
        }
        if (kR32) {
          if (kReduce) reinterpret_cast<float*>(a.dst)[k] = acc;
          rs_epi<DT, true, kEpi>(acc, 0u, inv, sumsq, flag);
        } else {
          const uint32_t b = D::narrow(acc);
          if (kReduce) reinterpret_cast<uint16_t*>(a.dst)[k] = (uint16_t)b;
          rs_epi<DT, false, kEpi>(0.0f, b, inv, sumsq, flag);
        }
      }
    }
  }
}

// groups of W 16-bit elements per rank per thread (W = 8: 128-bit loads, W = 16: 256-bit);
// PIPE: the NR loads of a thread's next group are issued before the current group is summed
// and stored, so every thread keeps two groups in flight and a partial last round costs
// only its own bytes
template <int W>
struct RSVec;
template <>
struct RSVec<8> {
  using T = U4;
  static __device__ __forceinline__ T ld(const uint16_t* p) { return ld128(p); }
  static __device__ __forceinline__ uint32_t get(const T& v, int j) { return h_get(v, j); }
};
template <>
struct RSVec<16> {
  using T = U8;
  static __device__ __forceinline__ T ld(const uint16_t* p) { return ld256(p); }
  static __device__ __forceinline__ uint32_t get(const T& v, int j) { return (v.x[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu; }
};

template <int DT, bool kR32, int kEpi, int W>
__device__ __forceinline__ void rs_emit_w(const RSArgs& a, uint64_t i, const float (&acc)[W], float inv, double& sumsq,
                                          uint32_t& flag) {
  if constexpr (W == 8) {
    rs_emit8<DT, kR32, kEpi>(a, i, acc, true, inv, sumsq, flag);
  } else {
    float lo[8], hi[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { lo[j] = acc[j]; hi[j] = acc[8 + j]; }
    if (kR32) {
      rs_emit8<DT, kR32, kEpi>(a, i, lo, true, inv, sumsq, flag);
      rs_emit8<DT, kR32, kEpi>(a, i + 8, hi, true, inv, sumsq, flag);
    } else {   // one 256-bit store of 16 rounded values
      using D = H16<DT>;
      U8 o;
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        const uint32_t b0 = D::narrow(acc[j]), b1 = D::narrow(acc[j + 1]);
        o.x[j >> 1] = b0 | (b1 << 16);
        rs_epi<DT, false, kEpi>(0.0f, b0, inv, sumsq, flag);
        rs_epi<DT, false, kEpi>(0.0f, b1, inv, sumsq, flag);
      }
      st256(reinterpret_cast<uint16_t*>(a.dst) + i, o);
    }
  }
}

template <int DT, bool kR32, int NR, int kEpi, int W, bool PIPE>
__device__ __forceinline__ void rs_body_g(const RSArgs& a, float inv, double& sumsq, uint32_t& flag) {
  using D = H16<DT>;
  using V = RSVec<W>;
  const uint64_t nvec = a.count / W;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  const uint64_t first = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  typename V::T cur[NR], nxt[NR];
  if (PIPE && first < nvec) {
#pragma unroll
    for (int r = 0; r < NR; ++r) cur[r] = V::ld(reinterpret_cast<const uint16_t*>(a.src[r]) + first * W);
  }
#pragma unroll 1
  for (uint64_t g = first; g < nvec; g += stride) {
    if (PIPE) {
      const uint64_t gn = g + stride;
      if (gn < nvec) {
#pragma unroll
        for (int r = 0; r < NR; ++r) nxt[r] = V::ld(reinterpret_cast<const uint16_t*>(a.src[r]) + gn * W);
      }
    } else {
#pragma unroll
      for (int r = 0; r < NR; ++r) cur[r] = V::ld(reinterpret_cast<const uint16_t*>(a.src[r]) + g * W);
    }
    float acc[W];
#pragma unroll
    for (int j = 0; j < W; ++j) acc[j] = D::widen(V::get(cur[0], j));
#pragma unroll
    for (int r = 1; r < NR; ++r) {
#pragma unroll
      for (int j = 0; j < W; ++j) acc[j] = __fadd_rn(acc[j], D::widen(V::get(cur[r], j)));
    }
    rs_emit_w<DT, kR32, kEpi, W>(a, g * W, acc, inv, sumsq, flag);
    if (PIPE) {
#pragma unroll
      for (int r = 0; r < NR; ++r) cur[r] = nxt[r];
    }
  }
  for (uint64_t k = nvec * W + first; k < a.count; k += stride) {   // ragged tail (< W elements)
    float acc = D::widen(reinterpret_cast<const uint16_t*>(a.src[0])[k]);
    for (int r = 1; r < NR; ++r) acc = __fadd_rn(acc, D::widen(reinterpret_cast<const uint16_t*>(a.src[r])[k]));
    if (kR32) {
      reinterpret_cast<float*>(a.dst)[k] = acc;
      rs_epi<DT, true, kEpi>(acc, 0u, inv, sumsq, flag);
    } else {
      const uint32_t b = D::narrow(acc);
      reinterpret_cast<uint16_t*>(a.dst)[k] = (uint16_t)b;
      rs_epi<DT, false, kEpi>(0.0f, b, inv, sumsq, flag);
    }
  }
}

template <int DT, bool kR32, bool kReduce, bool kVec, int NR, int U>
__device__ __forceinline__ void rs_main(const RSArgs& a) {
  if (a.wait_flags) {  // every rank has flattened this bucket (cross-process PEER)
    if (threadIdx.x == 0) wait_all(a.wait_flags, a.n, a.epoch);
    __syncthreads();
  }
  const float inv = a.st->inv_cur;
  double sumsq = 0.0;
  uint32_t flag = 0;
  // U selects the body: 1/2/4 = groups of 8 per thread per iteration; 0 = pipelined 128-bit;
  // 16 = 256-bit loads; 17 = pipelined 256-bit
  constexpr bool kG = U == 0 || U >= 16;
  constexpr int kW = U >= 16 ? 16 : 8;
  constexpr bool kP = U == 0 || U == 17;
  if (pow2_at_most_one(inv)) {   // inv = 1/(N S sigma) a power of two (N a power of two)
    if constexpr (kG) rs_body_g<DT, kR32, NR, 2, kW, kP>(a, inv, sumsq, flag);
    else rs_body<DT, kR32, kReduce, kVec, NR, U, 2>(a, inv, sumsq, flag);
    flag = isfinite(sumsq) ? 0u : 1u;     // G^2 / b^2 of finite values are finite in fp64
    sumsq *= (double)inv * (double)inv;   // exact
  } else {
    if constexpr (kG) rs_body_g<DT, kR32, NR, 1, kW, kP>(a, inv, sumsq, flag);
    else rs_body<DT, kR32, kReduce, kVec, NR, U, 1>(a, inv, sumsq, flag);
  }
  if (!a.cta_sum) {
    grid_publish(sumsq, flag, a.part, a.slot, a.done_sig, a.wait_flags ? a.n : 0, a.epoch);
    return;
  }
  // per-CTA partial (combined in a fixed order by the decision kernel)
  __shared__ bool is_last;
  block_reduce(sumsq, flag);
  if (threadIdx.x == 0) {
    a.cta_sum[blockIdx.x] = sumsq;
    a.cta_flag[blockIdx.x] = flag;
    if (blockIdx.x == 0) *a.cta_grid = gridDim.x;
  }
  if (!a.wait_flags) return;
  // cross-process: the last CTA to finish reading the peers' buckets tells them so
  if (threadIdx.x == 0) is_last = atomicAdd(&a.part->ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (is_last && threadIdx.x == 0) {
    a.part->ticket = 0;
    __threadfence_system();
    for (int j = 0; j < a.n; ++j) st_release_sys(a.done_sig[j], a.epoch);
  }
}

template <int DT, bool kR32, bool kReduce, bool kVec, int NR, int U>
__global__ void __launch_bounds__(kThreads) k_reduce_scatter(const __grid_constant__ RSArgs a) {
  rs_main<DT, kR32, kReduce, kVec, NR, U>(a);
}

// simulated ranks (one process, one GPU): the pull reduce-scatters of every rank for one
// bucket in one launch, grid row y = rank y -- they run concurrently, as on an NVL8 box
template <int DT, bool kR32, int NR>
__global__ void __launch_bounds__(kThreads) k_reduce_scatter_multi(const __grid_constant__ RSMulti m) {
  rs_main<DT, kR32, true, true, NR, 0>(m.r[blockIdx.y]);
}

cudaError_t launch_reduce_scatter_multi(const RSMulti& m, int grid, cudaStream_t s) {
  const RSArgs& a0 = m.r[0];
  for (int i = 0; i < m.n; ++i) {
    const RSArgs& a = m.r[i];
    if (!a.reduce || a.pipe != 1 || a.wait_flags || a.n != a0.n || a.dtype != a0.dtype || a.r32 != a0.r32 ||
        !aligned(a.dst, a.r32 ? 32 : 16))
      return cudaErrorNotSupported;
    for (int r = 0; r < a.n; ++r)
      if (!aligned(a.src[r], 16)) return cudaErrorNotSupported;
  }
  const dim3 g(grid, m.n);
#define ZM(DT, R32)                                                                          \
  switch (a0.n) {                                                                            \
    case 2: k_reduce_scatter_multi<DT, R32, 2><<<g, kThreads, 0, s>>>(m); break;           \
    case 4: k_reduce_scatter_multi<DT, R32, 4><<<g, kThreads, 0, s>>>(m); break;           \
    case 8: k_reduce_scatter_multi<DT, R32, 8><<<g, kThreads, 0, s>>>(m); break;           \
    default: return cudaErrorNotSupported;                                                   \
  }
  if (a0.dtype == DT_F16) { if (a0.r32) { ZM(DT_F16, true) } else { ZM(DT_F16, false) } }
  else if (a0.dtype == DT_BF16) { if (a0.r32) { ZM(DT_BF16, true) } else { ZM(DT_BF16, false) } }
  else return cudaErrorNotSupported;
#undef ZM
  return cudaGetLastError();
}

template <int DT, bool R32, bool RED, int NR>
cudaError_t launch_rs_u(const RSArgs& a, int grid, cudaStream_t s, int u) {
  if (a.pipe) {   // 1: pipelined 128-bit; 2: 256-bit loads; 3: pipelined 256-bit
    switch (a.pipe) {
      case 2: k_reduce_scatter<DT, R32, RED, true, NR, 16><<<grid, kThreads, 0, s>>>(a); break;
      case 3: k_reduce_scatter<DT, R32, RED, true, NR, 17><<<grid, kThreads, 0, s>>>(a); break;
      default: k_reduce_scatter<DT, R32, RED, true, NR, 0><<<grid, kThreads, 0, s>>>(a); break;
    }
    return cudaGetLastError();
  }
  switch (u) {
    case 1: k_reduce_scatter<DT, R32, RED, true, NR, 1><<<grid, kThreads, 0, s>>>(a); break;
    case 4: k_reduce_scatter<DT, R32, RED, true, NR, 4><<<grid, kThreads, 0, s>>>(a); break;
    default: k_reduce_scatter<DT, R32, RED, true, NR, 2><<<grid, kThreads, 0, s>>>(a); break;
  }
  return cudaGetLastError();
}

template <int DT, bool R32, bool RED, bool V>
cudaError_t launch_rs_n(const RSArgs& a, int grid, cudaStream_t s) {
  if constexpr (!V) {
    k_reduce_scatter<DT, R32, RED, false, 0, 1><<<grid, kThreads, 0, s>>>(a);
  } else if constexpr (!RED) {
    k_reduce_scatter<DT, R32, RED, true, 0, 2><<<grid, kThreads, 0, s>>>(a);
  } else {
    switch (a.n) {
      case 2: return launch_rs_u<DT, R32, RED, 2>(a, grid, s, a.u ? a.u : 4);
      case 4: return launch_rs_u<DT, R32, RED, 4>(a, grid, s, a.u ? a.u : 2);
      case 8: return launch_rs_u<DT, R32, RED, 8>(a, grid, s, a.u ? a.u : 1);
      default: k_reduce_scatter<DT, R32, RED, true, 0, 1><<<grid, kThreads, 0, s>>>(a); break;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_reduce_scatter(const RSArgs& a_in, int grid, cudaStream_t s) {
  RSArgs a = a_in;
  bool vec = aligned(a.dst, a.r32 ? 32 : 16);
  if (a.reduce)
    for (int r = 0; r < a.n; ++r) vec = vec && aligned(a.src[r], 16);
  if (a.pipe >= 2) {   // 256-bit accesses need 32-B aligned sources and destination
    bool v32 = aligned(a.dst, 32);
    for (int r = 0; r < a.n; ++r) v32 = v32 && aligned(a.src[r], 32);
    if (!v32) a.pipe = 1;
  }
#define ZRV(DT, R32, RED) return vec ? launch_rs_n<DT, R32, RED, true>(a, grid, s) : launch_rs_n<DT, R32, RED, false>(a, grid, s)
#define ZRR(DT, R32) do { if (a.reduce) ZRV(DT, R32, true); else ZRV(DT, R32, false); } while (0)
  if (a.dtype == DT_F16) { if (a.r32) ZRR(DT_F16, true); else ZRR(DT_F16, false); }
  else if (a.dtype == DT_BF16) { if (a.r32) ZRR(DT_BF16, true); else ZRR(DT_BF16, false); }
#undef ZRR
#undef ZRV
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// a4: global decision (reading c-4).  decide_local folds this rank's per-bucket
// slots (ascending bucket, fixed tree) into one RankPartial; decide_global folds
// the ranks' partials in ascending rank and advances the loss-scale machine.
// ---------------------------------------------------------------------------
__device__ void decide_apply(double sum, double flags, DevState* st, const DecideParams& p);

__global__ void __launch_bounds__(1024) k_decide_local(Slot* slots, int n, RankPartial* out, const double* slot_w,
                                                           const double* cta_sum, const uint32_t* cta_flag,
                                                           const uint32_t* cta_grid) {
  if (cta_sum) {  // N_d = 1: combine each slot's per-CTA flatten partials (warp per slot, fixed order)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = warp; i < n; i += nw) {
      const uint32_t g = cta_grid[i];
      const double* cs = cta_sum + (size_t)i * kMaxGrid;
      const uint32_t* cf = cta_flag + (size_t)i * kMaxGrid;
      double s = 0.0;
      uint32_t f = 0;
#pragma unroll 4
      for (uint32_t c = lane; c < g; c += 32) {   // loads pipelined, sums in CTA order
        s += cs[c];
        f |= cf[c];
      }
      s = warp_sum(s);
      f = __reduce_or_sync(0xffffffffu, f);
      if (lane == 0) {
        slots[i].sumsq = s;
        slots[i].flag = f;
      }
    }
    __syncthreads();
  }
  double s = 0.0;
  uint32_t f = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    s += slot_w ? slot_w[i] * slots[i].sumsq : slots[i].sumsq;  // weights 0/1: exact
    f |= slots[i].flag;
  }
  block_reduce(s, f);
  if (threadIdx.x == 0) {
    out->sumsq = s;
    out->flag = f ? 1.0 : 0.0;
  }
}

// N_d = 1 with per-CTA flatten partials: one CTA per bucket slot reduces that slot's
// partials (block tree), then the last CTA to finish combines the slots in slot order
__global__ void __launch_bounds__(kThreads) k_decide_local_slots(const double* slot_w, const double* cta_sum,
                                                                 const uint32_t* cta_flag, const uint32_t* cta_grid,
                                                                 GridPartials* part, RankPartial* out,
                                                                 DevState* st, const DecideParams p) {
  __shared__ bool is_last;
  const int i = blockIdx.x;
  const uint32_t g = cta_grid[i];
  const double* cs = cta_sum + (size_t)i * kMaxGrid;
  const uint32_t* cf = cta_flag + (size_t)i * kMaxGrid;
  double s = 0.0;
  uint32_t f = 0;
  for (uint32_t c = threadIdx.x; c < g; c += blockDim.x) {
    s += cs[c];
    f |= cf[c];
  }
  block_reduce(s, f);
  if (threadIdx.x == 0) {
    part->sumsq[i] = slot_w ? slot_w[i] * s : s;   // weights 0/1 (ZeRO x MP): exact
    part->flag[i] = f;
    __threadfence();
    is_last = atomicAdd(&part->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double a = 0.0;
  uint32_t b = 0;
  for (unsigned j = threadIdx.x; j < gridDim.x; j += blockDim.x) {
    a += __ldcg(&part->sumsq[j]);
    b |= __ldcg(&part->flag[j]);
  }
  block_reduce(a, b);
  if (threadIdx.x == 0) {
    out->sumsq = a;
    out->flag = b ? 1.0 : 0.0;
    part->ticket = 0;
    if (st) decide_apply(a, b ? 1.0 : 0.0, st, p);   // N_d = 1: the rank's partial is the global one
  }
}

cudaError_t launch_decide_local_slots(int n_slots, RankPartial* out, cudaStream_t s, const double* slot_w,
                                      const double* cta_sum, const uint32_t* cta_flag, const uint32_t* cta_grid,
                                      GridPartials* part, DevState* st, const DecideParams* p) {
  k_decide_local_slots<<<n_slots, kThreads, 0, s>>>(slot_w, cta_sum, cta_flag, cta_grid, part, out, st,
                                                    p ? *p : DecideParams{});
  return cudaGetLastError();
}

cudaError_t launch_decide_local(Slot* slots, int n_slots, RankPartial* out, cudaStream_t s, const double* slot_w,
                                const double* cta_sum, const uint32_t* cta_flag, const uint32_t* cta_grid) {
  // 32 warps: one per bucket slot at a time for the N_d = 1 per-CTA partials
  k_decide_local<<<1, cta_sum ? 1024 : kThreads, 0, s>>>(slots, n_slots, out, slot_w, cta_sum, cta_flag, cta_grid);
  return cudaGetLastError();
}

// sum of the data-parallel partials in rank order (the same order as k_decide_global)
__global__ void k_combine_partials(const __grid_constant__ PartialPtrs pp, RankPartial* out) {
  if (threadIdx.x != 0) return;
  if (pp.wait_flags) wait_all(pp.wait_flags, pp.n, pp.epoch);
  double sum = 0.0, flags = 0.0;
  for (int r = 0; r < pp.n; ++r) {
    sum += pp.p[r]->sumsq;
    flags += pp.p[r]->flag;
  }
  out->sumsq = sum;
  out->flag = flags;
}
cudaError_t launch_combine_partials(const PartialPtrs& pp, RankPartial* out, cudaStream_t s) {
  k_combine_partials<<<1, 32, 0, s>>>(pp, out);
  return cudaGetLastError();
}

// the decision itself (reading c-4), one thread: overflow -> skip + back off the loss
// scale; else the clip coefficient, t, the bias-correction scalars and the scale growth
__device__ void decide_apply(double sum, double flags, const DevSnap& s0, DevState* st, const DecideParams& p) {
  const bool overflow = flags != 0.0;
  const float S_used = s0.S;
  const double norm = sqrt(sum);
  float clip = 1.0f;
  float S = s0.S;
  uint32_t good = s0.good;
  uint64_t t = s0.t;
  if (overflow) {
    st->skip = 1u;
    if (p.dynamic) {
      S = fmaxf(S * 0.5f, p.min_scale);
      good = 0;
    }
  } else {
    if (p.max_norm > 0.0f && norm > (double)p.max_norm) clip = (float)((double)p.max_norm / (norm + 1e-6));
    t += 1;
    const double b1t = s0.b1t * (double)p.beta1;
    const double b2t = s0.b2t * (double)p.beta2;
    st->t = t;
    st->b1t = b1t;
    st->b2t = b2t;
    st->step_f = (float)((double)p.lr / (1.0 - b1t));
    st->rsb2_f = (float)(1.0 / sqrt(1.0 - b2t));
    st->clip_f = clip;
    st->inv_adam = s0.inv_cur;
    st->skip = 0u;
    if (p.dynamic) {
      good += 1;
      if (good == p.window) {
        S = S * 2.0f;
        good = 0;
      }
    }
  }
  if (p.dynamic) {
    st->S = S;
    st->good = good;
  }
  st->inv_cur = (float)(1.0 / ((double)p.n_ranks * (double)S * (double)p.sigma));
  st->rec_t = t;
  st->rec_overflow = overflow ? 1u : 0u;
  st->rec_scale = S_used;
  st->rec_clip = clip;
  st->rec_pad = 0;
  st->rec_norm = norm;
  if (p.rec_out) {   // the caller's pinned record, written over PCIe (no D2H copy in the step)
    uint64_t* r = reinterpret_cast<uint64_t*>(p.rec_out);
    r[0] = t;
    r[1] = (uint64_t)(overflow ? 1u : 0u) | ((uint64_t)__float_as_uint(S_used) << 32);
    r[2] = (uint64_t)__float_as_uint(clip);
    r[3] = (uint64_t)__double_as_longlong(norm);
    // no system fence: the caller reads the record after synchronizing the stream, and a
    // kernel's writes are visible to the host once it has completed
  }
}

__device__ void decide_apply(double sum, double flags, DevState* st, const DecideParams& p) {
  decide_apply(sum, flags, snap_state(st), st, p);
}

__global__ void k_decide_global(const __grid_constant__ PartialPtrs pp, DevState* st, const DecideParams p) {
  if (threadIdx.x != 0) return;
  if (pp.wait_flags) wait_all(pp.wait_flags, pp.n, pp.epoch);
  double sum = 0.0, flags = 0.0;
  for (int r = 0; r < pp.n; ++r) {
    sum += pp.p[r]->sumsq;
    flags += pp.p[r]->flag;
  }
  decide_apply(sum, flags, st, p);
}

cudaError_t launch_decide_global(const PartialPtrs& partials, DevState* st, DecideParams p, cudaStream_t s) {
  k_decide_global<<<1, 32, 0, s>>>(partials, st, p);
  return cudaGetLastError();
}

__global__ void k_init_state(DevState* st, float S, float inv) {
  st->b1t = 1.0;
  st->b2t = 1.0;
  st->t = 0;
  st->S = S;
  st->good = 0;
  st->inv_cur = inv;
  st->inv_adam = inv;
  st->step_f = 0.0f;
  st->rsb2_f = 1.0f;
  st->clip_f = 1.0f;
  st->skip = 1u;
  st->rec_t = 0;
  st->rec_overflow = 0;
  st->rec_scale = S;
  st->rec_clip = 1.0f;
  st->rec_pad = 0;
  st->rec_norm = 0.0;
}

cudaError_t launch_init_state(DevState* st, float S, float inv, cudaStream_t s) {
  k_init_state<<<1, 1, 0, s>>>(st, S, inv);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// a5: fused partitioned Adam + 16-bit recast, stored straight into the
// all-gather buffer(s) ("only update 1/N_d of the parameters").
// 28 B/element (R16): read p32, m, v (12 B) + G (2 B); write p32, m, v + p16.
// ---------------------------------------------------------------------------
struct AdamScalars {
  float inv, step, rsb2, clip, beta1, beta2, eps, omb1, omb2, lrwd;
  int wd;
};

__device__ __forceinline__ void adam_elem(float& p, float& m, float& v, float G, const AdamScalars& c) {
  float g = __fmul_rn(G, c.inv);
  if (c.clip != 1.0f) g = __fmul_rn(g, c.clip);
  if (c.wd) p = __fsub_rn(p, __fmul_rn(c.lrwd, p));
  m = __fadd_rn(__fmul_rn(c.beta1, m), __fmul_rn(c.omb1, g));
  v = __fadd_rn(__fmul_rn(c.beta2, v), __fmul_rn(__fmul_rn(c.omb2, g), g));
  const float d = __fadd_rn(__fmul_rn(__fsqrt_rn(v), c.rsb2), c.eps);
  p = __fsub_rn(p, __fmul_rn(c.step, __fdiv_rn(m, d)));
}

template <int PDT, int GDT>
struct AdamIO {
  using P = H16<PDT>;
  static __device__ __forceinline__ void load_g(const void* G, uint64_t idx, float (&g)[8]) {
    if (GDT == DT_F32) {
      U8 w = ld256(reinterpret_cast<const float*>(G) + idx);
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = __uint_as_float(w.x[j]);
    } else {
      U4 w = ld128(reinterpret_cast<const uint16_t*>(G) + idx);
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = H16<GDT == DT_F32 ? DT_F16 : GDT>::widen(h_get(w, j));
    }
  }
  static __device__ __forceinline__ float load_g1(const void* G, uint64_t idx) {
    if (GDT == DT_F32) return reinterpret_cast<const float*>(G)[idx];
    return H16<GDT == DT_F32 ? DT_F16 : GDT>::widen(reinterpret_cast<const uint16_t*>(G)[idx]);
  }
};

// MINB: CTAs per SM the register budget is sized for; U: 8-element groups per
// thread per iteration (all loads of an iteration are issued before any math).
template <int PDT, int GDT, int U>
__device__ __forceinline__ void adam_body(const AdamArgs& a, const AdamScalars& c, uint64_t lo, uint64_t hi);

__device__ __forceinline__ void adam_scalars(const AdamArgs& a, AdamScalars& c) {
  c.beta1 = a.beta1;
  c.beta2 = a.beta2;
  c.eps = a.eps;
  c.omb1 = a.omb1;
  c.omb2 = a.omb2;
  c.lrwd = a.lrwd;
  c.wd = a.wd;
}

// index of the segment holding shard element i (segments sorted by local_off, tiling [0, total))
__device__ __forceinline__ int find_seg(const AdamArgs& a, uint64_t i) {
  int s0 = 0, s1 = a.n_segs - 1;
  while (s0 < s1) {
    const int mid = (s0 + s1 + 1) >> 1;
    if (a.segs[mid].local_off <= i) s0 = mid; else s1 = mid - 1;
  }
  return s0;
}

template <int PDT, int GDT, int MINB, int U>
__global__ void __launch_bounds__(kThreads, MINB) k_adam(const __grid_constant__ AdamArgs a) {
  // PDL (a.pdl): launched while the whole-step flatten that made the decision finishes; wait
  // for it to complete (its writes visible) before reading the decision (a no-op otherwise)
  const uint64_t lo = (uint64_t)blockIdx.x * a.per_cta;
  if (lo >= a.total) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  const uint64_t hi = lo + a.per_cta < a.total ? lo + a.per_cta : a.total;
  AdamScalars c;
  adam_scalars(a, c);
  // PDL with 8-aligned segments: the first 8-element group of every thread -- its p32/m/v
  // (written by no kernel since the previous step's Adam) and its segment -- is fetched
  // before the wait, so those loads overlap the flatten's tail; only G and the decision
  // are read after it
  const uint64_t i0 = lo + threadIdx.x * 8;
  const bool pre = a.pdl && a.aligned8 && hi - lo >= (uint64_t)kThreads * 8;
  U8 p, m, v;
  int64_t gd = 0, pd = 0;
  if (pre) {
    p = ld256(a.p32 + i0);
    m = ld256(a.m + i0);
    v = ld256(a.v + i0);
    const AdamSeg sg = a.segs[find_seg(a, i0)];
    gd = (int64_t)sg.g_off - (int64_t)sg.local_off;
    pd = (int64_t)sg.p16_off - (int64_t)sg.local_off;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the decision's outputs, all loaded before the skip branch
  const uint32_t skip = a.st->skip;
  c.inv = a.st->inv_adam;
  c.step = a.st->step_f;
  c.rsb2 = a.st->rsb2_f;
  c.clip = a.st->clip_f;
  if (skip) return;  // overflow: the whole step is skipped (reading c-4)
  if (pre) {
    using P = H16<PDT>;
    float G[8];
    AdamIO<PDT, GDT>::load_g(a.G, i0 + gd, G);
    U4 o;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float pj = __uint_as_float(p.x[j]), mj = __uint_as_float(m.x[j]), vj = __uint_as_float(v.x[j]);
      adam_elem(pj, mj, vj, G[j], c);
      p.x[j] = __float_as_uint(pj);
      m.x[j] = __float_as_uint(mj);
      v.x[j] = __float_as_uint(vj);
      h_set(o, j, P::narrow(pj));
    }
    st256(a.p32 + i0, p);
    st256(a.m + i0, m);
    st256(a.v + i0, v);
    for (int d = 0; d < a.n_p16; ++d) st128(reinterpret_cast<uint16_t*>(a.p16[d]) + (i0 + pd), o);
    adam_body<PDT, GDT, U>(a, c, lo + (uint64_t)kThreads * 8, hi);   // the rest of the range, if any
  } else {
    adam_body<PDT, GDT, U>(a, c, lo, hi);
  }
}

// the register-staged Adam over this CTA's contiguous range of the shard (k_adam and the
// fused small-model step)
template <int PDT, int GDT, int U>
__device__ __forceinline__ void adam_body(const AdamArgs& a, const AdamScalars& c, uint64_t lo, uint64_t hi) {
  using P = H16<PDT>;
  using IO = AdamIO<PDT, GDT>;
  if (lo >= hi) return;
  const int s0 = find_seg(a, lo);   // first segment containing lo
  uint64_t cur = lo;
  for (int s = s0; cur < hi && s < a.n_segs; ++s) {
    const AdamSeg sg = a.segs[s];
    const uint64_t send = sg.local_off + sg.count < hi ? sg.local_off + sg.count : hi;
    if (send <= cur) continue;
    const int64_t gd = (int64_t)sg.g_off - (int64_t)sg.local_off;
    const int64_t pd = (int64_t)sg.p16_off - (int64_t)sg.local_off;
    uint64_t vend = cur;
    if (((cur | (uint64_t)gd | (uint64_t)pd) & 7) == 0) {
      vend = cur + ((send - cur) & ~(uint64_t)7);
#pragma unroll 1
      for (uint64_t i0 = cur + threadIdx.x * 8; i0 < vend; i0 += (uint64_t)kThreads * 8 * U) {
        U8 p[U], m[U], v[U];
        float G[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t i = i0 + (uint64_t)u * kThreads * 8;
          if (u == 0 || i < vend) {
            p[u] = ld256(a.p32 + i);
            m[u] = ld256(a.m + i);
            v[u] = ld256(a.v + i);
            IO::load_g(a.G, i + gd, G[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t i = i0 + (uint64_t)u * kThreads * 8;
          if (u == 0 || i < vend) {
            U4 o;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float pj = __uint_as_float(p[u].x[j]), mj = __uint_as_float(m[u].x[j]), vj = __uint_as_float(v[u].x[j]);
              adam_elem(pj, mj, vj, G[u][j], c);
              p[u].x[j] = __float_as_uint(pj);
              m[u].x[j] = __float_as_uint(mj);
              v[u].x[j] = __float_as_uint(vj);
              h_set(o, j, P::narrow(pj));
            }
            st256(a.p32 + i, p[u]);
            st256(a.m + i, m[u]);
            st256(a.v + i, v[u]);
            for (int d = 0; d < a.n_p16; ++d) st128(reinterpret_cast<uint16_t*>(a.p16[d]) + (i + pd), o);
          }
        }
      }
    }
    for (uint64_t i = vend + threadIdx.x; i < send; i += kThreads) {  // unaligned remainder
      float p = a.p32[i], m = a.m[i], v = a.v[i];
      const float G = IO::load_g1(a.G, i + gd);
      adam_elem(p, m, v, G, c);
      a.p32[i] = p;
      a.m[i] = m;
      a.v[i] = v;
      const uint16_t b = (uint16_t)P::narrow(p);
      for (int d = 0; d < a.n_p16; ++d) reinterpret_cast<uint16_t*>(a.p16[d])[i + pd] = b;
    }
    cur = send;
  }
}

// ---------------------------------------------------------------------------
// a5 (TMA variant): the same fused Adam, with the four input streams staged into
// shared memory by 1-D bulk copies (cp.async.bulk, the TMA engine) in a
// STAGES-deep mbarrier ring.  One producer warp keeps up to STAGES tiles of
// T elements in flight per CTA (decoupled from the math), eight consumer warps
// compute from shared memory and store p32/m/v/p16 with 256/128-bit STG.
// Requires every segment offset and count to be a multiple of 8 (host checks).
// ---------------------------------------------------------------------------
// tile iterator over the CTA's contiguous range, split at segment boundaries
struct TileCursor {
  uint64_t cur, hi;
  int s;
  __device__ __forceinline__ bool next(const AdamArgs& a, uint32_t T, uint64_t& start, uint32_t& n, int64_t& gd,
                                       int64_t& pd) {
    while (cur < hi && s < a.n_segs) {
      const AdamSeg sg = a.segs[s];
      const uint64_t send = sg.local_off + sg.count < hi ? sg.local_off + sg.count : hi;
      if (cur >= send) { ++s; continue; }
      start = cur;
      const uint64_t left = send - cur;
      n = left < T ? (uint32_t)left : T;
      gd = (int64_t)sg.g_off - (int64_t)sg.local_off;
      pd = (int64_t)sg.p16_off - (int64_t)sg.local_off;
      cur += n;
      return true;
    }
    return false;
  }
};

template <int PDT, int GDT, int T, int STAGES>
__global__ void __launch_bounds__(T / 8 + 32, 1) k_adam_tma(const __grid_constant__ AdamArgs a) {
  constexpr int kCons = T / 8;  // consumer threads: 8 elements of every tile each
  using P = H16<PDT>;
  constexpr int GB = (GDT == DT_F32) ? 4 : 2;
  constexpr uint32_t kStageBytes = (uint32_t)T * (12 + GB);
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  if (a.st->skip) return;  // overflow: skip the step (reading c-4)
  const uint64_t lo = (uint64_t)blockIdx.x * a.per_cta;
  if (lo >= a.total) return;
  const uint64_t hi = lo + a.per_cta < a.total ? lo + a.per_cta : a.total;
  int s0 = 0, s1 = a.n_segs - 1;
  while (s0 < s1) {
    const int mid = (s0 + s1 + 1) >> 1;
    if (a.segs[mid].local_off <= lo) s0 = mid; else s1 = mid - 1;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kCons / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kCons / 32) {  // ---- producer warp
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      TileCursor tc{lo, hi, s0};
      uint64_t start;
      uint32_t n;
      int64_t gd, pd;
      for (uint32_t it = 0; tc.next(a, T, start, n, gd, pd); ++it) {
        const int st = it % STAGES;
        if (it >= (uint32_t)STAGES) mbar_wait(&empty[st], ((it / STAGES) - 1) & 1);
        unsigned char* base = smem + st * kStageBytes;
        mbar_expect_tx(&full[st], n * (12u + GB));
        bulk_g2s(base, a.p32 + start, n * 4u, &full[st], pol);
        bulk_g2s(base + T * 4, a.m + start, n * 4u, &full[st], pol);
        bulk_g2s(base + T * 8, a.v + start, n * 4u, &full[st], pol);
        bulk_g2s(base + T * 12, reinterpret_cast<const unsigned char*>(a.G) + (start + gd) * GB, n * (uint32_t)GB,
                 &full[st], pol);
      }
    }
    return;
  }

  // ---- consumer warps
  AdamScalars c;
  c.inv = a.st->inv_adam;
  c.step = a.st->step_f;
  c.rsb2 = a.st->rsb2_f;
  c.clip = a.st->clip_f;
  c.beta1 = a.beta1;
  c.beta2 = a.beta2;
  c.eps = a.eps;
  c.omb1 = a.omb1;
  c.omb2 = a.omb2;
  c.lrwd = a.lrwd;
  c.wd = a.wd;
  TileCursor tc{lo, hi, s0};
  uint64_t start;
  uint32_t n;
  int64_t gd, pd;
  for (uint32_t it = 0; tc.next(a, T, start, n, gd, pd); ++it) {
    const int st = it % STAGES;
    mbar_wait(&full[st], (it / STAGES) & 1);
    const unsigned char* base = smem + st * kStageBytes;
    {
      const uint32_t e = threadIdx.x * 8;
      if (e < n) {
        U8 p, m, v;
        float G[8];
        {
          uint32_t r[4];
          lds128(base + e * 4, r);
          p.x[0] = r[0]; p.x[1] = r[1]; p.x[2] = r[2]; p.x[3] = r[3];
          lds128(base + e * 4 + 16, r);
          p.x[4] = r[0]; p.x[5] = r[1]; p.x[6] = r[2]; p.x[7] = r[3];
          lds128(base + T * 4 + e * 4, r);
          m.x[0] = r[0]; m.x[1] = r[1]; m.x[2] = r[2]; m.x[3] = r[3];
          lds128(base + T * 4 + e * 4 + 16, r);
          m.x[4] = r[0]; m.x[5] = r[1]; m.x[6] = r[2]; m.x[7] = r[3];
          lds128(base + T * 8 + e * 4, r);
          v.x[0] = r[0]; v.x[1] = r[1]; v.x[2] = r[2]; v.x[3] = r[3];
          lds128(base + T * 8 + e * 4 + 16, r);
          v.x[4] = r[0]; v.x[5] = r[1]; v.x[6] = r[2]; v.x[7] = r[3];
          if (GB == 4) {
            lds128(base + T * 12 + e * 4, r);
#pragma unroll
            for (int j = 0; j < 4; ++j) G[j] = __uint_as_float(r[j]);
            lds128(base + T * 12 + e * 4 + 16, r);
#pragma unroll
            for (int j = 0; j < 4; ++j) G[4 + j] = __uint_as_float(r[j]);
          } else {
            lds128(base + T * 12 + e * 2, r);
            U4 g{{r[0], r[1], r[2], r[3]}};
#pragma unroll
            for (int j = 0; j < 8; ++j) G[j] = H16<GDT == DT_F32 ? DT_F16 : GDT>::widen(h_get(g, j));
          }
        }
        U4 o;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float pj = __uint_as_float(p.x[j]), mj = __uint_as_float(m.x[j]), vj = __uint_as_float(v.x[j]);
          adam_elem(pj, mj, vj, G[j], c);
          p.x[j] = __float_as_uint(pj);
          m.x[j] = __float_as_uint(mj);
          v.x[j] = __float_as_uint(vj);
          h_set(o, j, P::narrow(pj));
        }
        const uint64_t i = start + e;
        st256(a.p32 + i, p);
        st256(a.m + i, m);
        st256(a.v + i, v);
        for (int d = 0; d < a.n_p16; ++d) st128(reinterpret_cast<uint16_t*>(a.p16[d]) + (i + pd), o);
      }
    }
    // order this warp's generic-proxy reads of the stage before the next async-proxy
    // (bulk copy) write into it, then release the stage to the producer
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
}

template <int PD, int GD, int T, int STAGES>
cudaError_t launch_adam_tma_t(const AdamArgs& a, int grid, cudaStream_t s) {
  constexpr int GB = (GD == DT_F32) ? 4 : 2;
  const size_t smem = (size_t)STAGES * T * (12 + GB) + 2 * STAGES * sizeof(uint64_t);
  static std::atomic<uint64_t> configured{0};  // one bit per device
  if (cudaError_t e = allow_dynamic_smem(k_adam_tma<PD, GD, T, STAGES>, smem, configured)) return e;
  k_adam_tma<PD, GD, T, STAGES><<<grid, T / 8 + 32, smem, s>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// a5 (TMA in + TMA out): as k_adam_tma, but the consumers write the updated
// p32/m/v back into the stage and the recast p16 into a per-stage slot, and the
// producer thread drains the stage to global memory with 1-D bulk stores
// (cp.async.bulk.global.shared::cta, SASS UBLKCP.G.S) before refilling it.
// Consumer thread t handles elements [4t, 4t+4) and [4t + T/2, 4t + T/2 + 4) of
// the tile: every shared-memory access of a warp is contiguous (no bank conflicts).
// ---------------------------------------------------------------------------
template <int PDT, int GDT, int T, int STAGES>
__global__ void __launch_bounds__(T / 8 + 32, 1) k_adam_tma_st(const __grid_constant__ AdamArgs a) {
  constexpr int kCons = T / 8;
  using P = H16<PDT>;
  constexpr int GB = (GDT == DT_F32) ? 4 : 2;
  constexpr uint32_t kStageBytes = (uint32_t)T * (14 + GB);  // p32, m, v, G, p16
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* done = full + STAGES;
  if (a.st->skip) return;  // overflow: skip the step (reading c-4)
  const uint64_t lo = (uint64_t)blockIdx.x * a.per_cta;
  if (lo >= a.total) return;
  const uint64_t hi = lo + a.per_cta < a.total ? lo + a.per_cta : a.total;
  int s0 = 0, s1 = a.n_segs - 1;
  while (s0 < s1) {
    const int mid = (s0 + s1 + 1) >> 1;
    if (a.segs[mid].local_off <= lo) s0 = mid; else s1 = mid - 1;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&done[i], kCons / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kCons / 32) {  // ---- producer: loads ahead, stores behind
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      struct Pend { uint64_t start; uint32_t n; int64_t pd; };
      Pend pend[STAGES];
      auto drain = [&](uint32_t j) {  // tile j's results: stage -> global
        const int st = j % STAGES;
        mbar_wait(&done[st], (j / STAGES) & 1);
        unsigned char* base = smem + st * kStageBytes;
        const Pend& q = pend[st];
        bulk_s2g(a.p32 + q.start, base, q.n * 4u, pol);
        bulk_s2g(a.m + q.start, base + T * 4, q.n * 4u, pol);
        bulk_s2g(a.v + q.start, base + T * 8, q.n * 4u, pol);
        for (int d = 0; d < a.n_p16; ++d)
          bulk_s2g(reinterpret_cast<uint16_t*>(a.p16[d]) + (q.start + q.pd), base + T * (12 + GB), q.n * 2u, pol);
        bulk_commit();
      };
      TileCursor tc{lo, hi, s0};
      uint64_t start;
      uint32_t n;
      int64_t gd, pd;
      uint32_t it = 0;
      for (; tc.next(a, T, start, n, gd, pd); ++it) {
        const int st = it % STAGES;
        if (it >= (uint32_t)STAGES) {
          drain(it - STAGES);
          bulk_wait_read0();  // the stage has been read out: it may be refilled
        }
        pend[st] = Pend{start, n, pd};
        unsigned char* base = smem + st * kStageBytes;
        mbar_expect_tx(&full[st], n * (12u + GB));
        bulk_g2s(base, a.p32 + start, n * 4u, &full[st], pol);
        bulk_g2s(base + T * 4, a.m + start, n * 4u, &full[st], pol);
        bulk_g2s(base + T * 8, a.v + start, n * 4u, &full[st], pol);
        bulk_g2s(base + T * 12, reinterpret_cast<const unsigned char*>(a.G) + (start + gd) * GB, n * (uint32_t)GB,
                 &full[st], pol);
      }
      for (uint32_t j = it > (uint32_t)STAGES ? it - STAGES : 0; j < it; ++j) drain(j);
      bulk_wait_all0();
    }
    return;
  }

  // ---- consumer warps
  AdamScalars c;
  c.inv = a.st->inv_adam;
  c.step = a.st->step_f;
  c.rsb2 = a.st->rsb2_f;
  c.clip = a.st->clip_f;
  c.beta1 = a.beta1;
  c.beta2 = a.beta2;
  c.eps = a.eps;
  c.omb1 = a.omb1;
  c.omb2 = a.omb2;
  c.lrwd = a.lrwd;
  c.wd = a.wd;
  TileCursor tc{lo, hi, s0};
  uint64_t start;
  uint32_t n;
  int64_t gd, pd;
  for (uint32_t it = 0; tc.next(a, T, start, n, gd, pd); ++it) {
    const int st = it % STAGES;
    mbar_wait(&full[st], (it / STAGES) & 1);
    unsigned char* base = smem + st * kStageBytes;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t e = threadIdx.x * 4 + h * (T / 2);
      if (e < n) {  // n % 8 == 0 and e % 4 == 0: all 4 elements are in the tile
        uint32_t p[4], m[4], v[4];
        float G[4];
        lds128(base + e * 4, p);
        lds128(base + T * 4 + e * 4, m);
        lds128(base + T * 8 + e * 4, v);
        if (GB == 4) {
          uint32_t r[4];
          lds128(base + T * 12 + e * 4, r);
#pragma unroll
          for (int j = 0; j < 4; ++j) G[j] = __uint_as_float(r[j]);
        } else {
          uint32_t r0, r1;
          lds64(base + T * 12 + e * 2, r0, r1);
          constexpr int GD16 = GDT == DT_F32 ? DT_F16 : GDT;
          G[0] = H16<GD16>::widen(r0 & 0xFFFFu);
          G[1] = H16<GD16>::widen(r0 >> 16);
          G[2] = H16<GD16>::widen(r1 & 0xFFFFu);
          G[3] = H16<GD16>::widen(r1 >> 16);
        }
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float pj = __uint_as_float(p[j]), mj = __uint_as_float(m[j]), vj = __uint_as_float(v[j]);
          adam_elem(pj, mj, vj, G[j], c);
          p[j] = __float_as_uint(pj);
          m[j] = __float_as_uint(mj);
          v[j] = __float_as_uint(vj);
          o[j] = P::narrow(pj);
        }
        sts128(base + e * 4, p[0], p[1], p[2], p[3]);
        sts128(base + T * 4 + e * 4, m[0], m[1], m[2], m[3]);
        sts128(base + T * 8 + e * 4, v[0], v[1], v[2], v[3]);
        sts64(base + T * (12 + GB) + e * 2, o[0] | (o[1] << 16), o[2] | (o[3] << 16));
      }
    }
    // make this warp's generic-proxy writes of the stage visible to the bulk stores
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&done[st]);
  }
}

template <int PD, int GD, int T, int STAGES>
cudaError_t launch_adam_tma_st_t(const AdamArgs& a, int grid, cudaStream_t s) {
  constexpr int GB = (GD == DT_F32) ? 4 : 2;
  const size_t smem = (size_t)STAGES * T * (14 + GB) + 2 * STAGES * sizeof(uint64_t);
  static std::atomic<uint64_t> configured{0};  // one bit per device
  if (cudaError_t e = allow_dynamic_smem(k_adam_tma_st<PD, GD, T, STAGES>, smem, configured)) return e;
  k_adam_tma_st<PD, GD, T, STAGES><<<grid, T / 8 + 32, smem, s>>>(a);
  return cudaGetLastError();
}

// Variants kept from the round-1 sweeps (GPT-2 1.5B step on 1x B200, % of the measured
// copy peak of the box; profiles/r01_summary.md):
//   0 = register-staged, 2 CTAs/SM (85.5 %)     1 = register-staged, 4 CTAs/SM, <= 64 regs (90.1 %)
//  11 = TMA loads, STG stores, T 4096 x 2 stages, 1 CTA/SM: 512 consumers + 1 producer warp (96.1 %)
//  21 = TMA loads and TMA stores (k_adam_tma_st), T 4096 x 2 stages, 1 CTA/SM (99.3 %, default)
// (also measured and dropped -- TMA loads + STG: 2048x4 92.6 %, 2048x2 on 2 CTAs/SM 93.5 %,
//  1024x{4,6} 61-89 %, 2048x{3,6} 86-91 %, 4096x3 92 %, 6144x2 93 %, 3072x2 92 %, 4096x1 70 %;
//  TMA loads + TMA stores: 4096x3 94.9 %, 2048x4 95.2 %, 2048x3 98.3 %, 6144x2 95.5 %,
//  3072x2 94.9 %, 3072x3 95.5 %, and with several CTAs per SM 2048x2 x 2 94.0 %,
//  2048x3 x 2 92.4 %, 1024x4 x 3 89.9 %; register unroll-2 / 3 CTAs 81 %, 1 CTA unroll-4 87 %)
int adam_ctas_per_sm(int variant) {
  switch (variant) {
    case 1: return 4;
    case 11: case 21: return 1;
    default: return 2;
  }
}
bool adam_variant_is_tma(int variant) { return variant == 11 || variant == 21; }

template <int PD, int GD>
cudaError_t launch_adam_t(const AdamArgs& a, int grid, cudaStream_t s, int variant) {
  switch (variant) {
    case 11: return launch_adam_tma_t<PD, GD, 4096, 2>(a, grid, s);
    case 21: return launch_adam_tma_st_t<PD, GD, 4096, 2>(a, grid, s);
    case 1:
      if (a.pdl) {   // a programmatic dependent of the flatten before it on this stream
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kThreads);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, k_adam<PD, GD, 4, 1>, a);
      }
      k_adam<PD, GD, 4, 1><<<grid, kThreads, 0, s>>>(a);
      break;
    default: k_adam<PD, GD, 2, 1><<<grid, kThreads, 0, s>>>(a); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_adam(const AdamArgs& a, int grid, cudaStream_t s, int variant) {
  if (a.p_dtype == DT_F16) {
    if (a.g_dtype == DT_F16) return launch_adam_t<DT_F16, DT_F16>(a, grid, s, variant);
    if (a.g_dtype == DT_F32) return launch_adam_t<DT_F16, DT_F32>(a, grid, s, variant);
  } else if (a.p_dtype == DT_BF16) {
    if (a.g_dtype == DT_BF16) return launch_adam_t<DT_BF16, DT_BF16>(a, grid, s, variant);
    if (a.g_dtype == DT_F32) return launch_adam_t<DT_BF16, DT_F32>(a, grid, s, variant);
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// N_d = 1, a small model (the whole step is a few microseconds of bandwidth): flatten +
// epilogue, decision, fused Adam in ONE cooperative launch.  Phase A is k_flatten's body
// over every bucket (per-CTA {sum, flag} partials); after a grid barrier CTA 0 combines the
// partials in CTA order and makes the decision (decide_apply, as k_decide_*); after a
// second barrier every CTA runs the register Adam body over its range, reading the scalars
// the decision wrote (L1-bypassing loads: the line was cached before the barrier).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void grid_barrier(unsigned int* count, unsigned int* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int g = *(volatile unsigned int*)gen;
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*(volatile unsigned int*)gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

template <int SDT, int DDT, bool kCopy>
__global__ void __launch_bounds__(kThreads, 4) k_step_small(const __grid_constant__ StepSmallArgs a) {
  // barrier words: the DevState's record padding is not used; a GridPartials ticket pair is
  GridPartials* bar = a.f.decide_part;
  double sumsq = 0.0;
  uint32_t flag = 0;
  const float inv = a.f.st->inv_cur;
  if (pow2_at_most_one(inv)) {
    flatten_body<SDT, DDT, kCopy, 2, 2>(a.f, inv, sumsq, flag);
    flag = isfinite(sumsq) ? 0u : 1u;
    sumsq *= (double)inv * (double)inv;
  } else {
    flatten_body<SDT, DDT, kCopy, 2, 1>(a.f, inv, sumsq, flag);
  }
  block_reduce(sumsq, flag);
  if (threadIdx.x == 0) {
    a.f.cta_sum[blockIdx.x] = sumsq;
    a.f.cta_flag[blockIdx.x] = flag;
  }
  grid_barrier(&bar->ticket, &bar->pad);
  if (blockIdx.x == 0) {   // the decision, from the partials in CTA order
    double s = 0.0;
    uint32_t f = 0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
      s += __ldcg(&a.f.cta_sum[i]);
      f |= __ldcg(&a.f.cta_flag[i]);
    }
    block_reduce(s, f);
    if (threadIdx.x == 0) {
      a.out->sumsq = s;
      a.out->flag = f ? 1.0 : 0.0;
      decide_apply(s, f ? 1.0 : 0.0, a.st, a.dp);
      __threadfence();
    }
  }
  grid_barrier(&bar->ticket, &bar->pad);
  if (__ldcg(&a.st->skip)) return;   // overflow: the step is skipped (reading c-4)
  AdamScalars c;
  c.inv = __ldcg(&a.st->inv_adam);
  c.step = __ldcg(&a.st->step_f);
  c.rsb2 = __ldcg(&a.st->rsb2_f);
  c.clip = __ldcg(&a.st->clip_f);
  adam_scalars(a.adam, c);
  const uint64_t lo = (uint64_t)blockIdx.x * a.adam.per_cta;
  if (lo >= a.adam.total) return;
  adam_body<DDT, DDT, 1>(a.adam, c, lo, lo + a.adam.per_cta < a.adam.total ? lo + a.adam.per_cta : a.adam.total);
}

template <int SD, int DD, bool CP>
static cudaError_t step_small_t(const StepSmallArgs& a, int grid, cudaStream_t s, int* max_grid) {
  if (max_grid) {
    int per_sm = 0;
    if (cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step_small<SD, DD, CP>, kThreads, 0))
      return e;
    *max_grid = per_sm * sm_count();
    return cudaSuccess;
  }
  void* args[] = {const_cast<StepSmallArgs*>(&a)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_step_small<SD, DD, CP>), dim3(grid), dim3(kThreads),
                                     args, 0, s);
}

static cudaError_t step_small_dispatch(const StepSmallArgs& a, int grid, cudaStream_t s, int* max_grid) {
  const bool copy = a.f.sigma == 1.0f && a.f.src_dtype == a.f.dst_dtype;
  if (a.adam.g_dtype != a.f.dst_dtype || a.adam.p_dtype != a.f.dst_dtype) return cudaErrorNotSupported;
  if (a.f.dst_dtype == DT_F16) {
    if (a.f.src_dtype == DT_F16) return copy ? step_small_t<DT_F16, DT_F16, true>(a, grid, s, max_grid)
                                             : step_small_t<DT_F16, DT_F16, false>(a, grid, s, max_grid);
    if (a.f.src_dtype == DT_F32) return step_small_t<DT_F32, DT_F16, false>(a, grid, s, max_grid);
  } else if (a.f.dst_dtype == DT_BF16) {
    if (a.f.src_dtype == DT_BF16) return copy ? step_small_t<DT_BF16, DT_BF16, true>(a, grid, s, max_grid)
                                              : step_small_t<DT_BF16, DT_BF16, false>(a, grid, s, max_grid);
    if (a.f.src_dtype == DT_F32) return step_small_t<DT_F32, DT_BF16, false>(a, grid, s, max_grid);
  }
  return cudaErrorNotSupported;
}

int step_small_max_grid(const StepSmallArgs& a) {
  int g = 0;
  if (step_small_dispatch(a, 0, nullptr, &g) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return g;
}

cudaError_t launch_step_small(const StepSmallArgs& a, int grid, cudaStream_t s) {
  return step_small_dispatch(a, grid, s, nullptr);
}

// ---------------------------------------------------------------------------
// a6/a7 over a peer table (and P_a's save / gather): dst[j][0..count[j]) = src[j][0..count[j])
// for every row j < n (16-bit, bitwise)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_copy(const __grid_constant__ CopyArgs a) {
  const int j = blockIdx.y;
  const uint16_t* src = reinterpret_cast<const uint16_t*>(a.src[j]);
  uint16_t* dst = reinterpret_cast<uint16_t*>(a.dst[j]);
  const uint64_t count = a.count[j];
  if (src == dst) return;
  const uint64_t tid = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  const uint64_t nthr = (uint64_t)gridDim.x * kThreads;
  if (aligned(src, 16) && aligned(dst, 16)) {
    const uint64_t nv = count / 8;
    uint64_t i = tid;
    for (; i + 3 * nthr < nv; i += 4 * nthr) {   // 4 x 128-bit loads in flight (NVLink latency ~2 us)
      const U4 r0 = ld128(src + i * 8), r1 = ld128(src + (i + nthr) * 8);
      const U4 r2 = ld128(src + (i + 2 * nthr) * 8), r3 = ld128(src + (i + 3 * nthr) * 8);
      st128(dst + i * 8, r0);
      st128(dst + (i + nthr) * 8, r1);
      st128(dst + (i + 2 * nthr) * 8, r2);
      st128(dst + (i + 3 * nthr) * 8, r3);
    }
    for (; i < nv; i += nthr) st128(dst + i * 8, ld128(src + i * 8));
    for (uint64_t e = nv * 8 + tid; e < count; e += nthr) dst[e] = src[e];
  } else {
    for (uint64_t i = tid; i < count; i += nthr) dst[i] = src[i];
  }
}

cudaError_t launch_copy(const CopyArgs& a, int grid, cudaStream_t s) {
  uint64_t mx = 0;
  for (int j = 0; j < a.n; ++j) mx = a.count[j] > mx ? a.count[j] : mx;
  if (a.n <= 0 || mx == 0) return cudaSuccess;
  dim3 g(grid, a.n);
  k_copy<<<g, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// zero_load_master: fp32 master piece -> owned fp32 shard + 16-bit copy
// ---------------------------------------------------------------------------
template <int PDT>
__global__ void __launch_bounds__(kThreads) k_load(const __grid_constant__ LoadArgs a) {
  using P = H16<PDT>;
  uint16_t* p16 = reinterpret_cast<uint16_t*>(a.p16);
  for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < a.count; i += (uint64_t)gridDim.x * kThreads) {
    const float x = a.src[i];
    const uint64_t g = a.flat_off + i;
    const uint16_t b = (uint16_t)P::narrow(x);
    if (a.p16_mode == 0) p16[g] = b;
    if (g >= a.own_lo && g < a.own_hi) {
      const uint64_t l = a.local_base + (g - a.own_lo);
      a.p32[l] = x;
      if (a.p16_mode == 1) p16[l] = b;
    }
  }
}

cudaError_t launch_load(const LoadArgs& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  uint64_t blocks = (a.count + kThreads - 1) / kThreads;
  const int grid = (int)(blocks < 4096 ? blocks : 4096);
  if (a.p_dtype == DT_F16) k_load<DT_F16><<<grid, kThreads, 0, s>>>(a);
  else k_load<DT_BF16><<<grid, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// cross-process PEER signalling
// ---------------------------------------------------------------------------
__global__ void k_signal(const __grid_constant__ SigArgs a) {
  if (threadIdx.x == 0) __threadfence_system();
  __syncwarp();
  if ((int)threadIdx.x < a.n) st_release_sys(a.dst[threadIdx.x], a.epoch);
}
__global__ void k_wait(const __grid_constant__ WaitArgs a) {
  if (threadIdx.x == 0) wait_all(a.flags, a.n, a.epoch);
}
// zero_peer_open's handshake: tell every peer "rank me is linked", then wait (bounded,
// without trapping) until every peer has said the same; *result = 0 ok, 1 timed out.
__global__ void k_handshake(const __grid_constant__ SigArgs a, const uint64_t* my_flags, uint64_t timeout_ns,
                            uint32_t* result) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int j = 0; j < a.n; ++j) st_release_sys(a.dst[j], a.epoch);
  const uint64_t t0 = globaltimer_ns();
  uint32_t r = 0;
  for (int j = 0; j < a.n && !r; ++j)
    while (ld_acquire_sys(my_flags + j) < a.epoch) {
      __nanosleep(1000);
      if (globaltimer_ns() - t0 > timeout_ns) { r = 1; break; }
    }
  *result = r;
}
cudaError_t launch_handshake(const SigArgs& a, const uint64_t* my_flags, uint64_t timeout_ns, uint32_t* result,
                             cudaStream_t s) {
  k_handshake<<<1, 32, 0, s>>>(a, my_flags, timeout_ns, result);
  return cudaGetLastError();
}
__global__ void k_push_partial(const __grid_constant__ PushArgs a) {
  const int j = threadIdx.x;
  if (j < a.n) {
    *a.dst[j] = *a.mine;
    st_release_sys(a.sig[j], a.epoch);
  }
}
cudaError_t launch_signal(const SigArgs& a, cudaStream_t s) {
  k_signal<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_wait(const WaitArgs& a, cudaStream_t s) {
  k_wait<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_push_partial(const PushArgs& a, cudaStream_t s) {
  k_push_partial<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// checkpoint / resharding support
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_shard_io(const __grid_constant__ ShardIOArgs a) {
  for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < a.count; i += (uint64_t)gridDim.x * kThreads) {
    const uint64_t g = a.flat_off + i;
    if (g < a.own_lo || g >= a.own_hi) continue;
    const uint64_t l = a.local_base + (g - a.own_lo);
    if (a.to_shard) a.shard[l] = a.tensor[i];
    else a.tensor[i] = a.shard[l];
  }
}
cudaError_t launch_shard_io(const ShardIOArgs& a, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  const uint64_t blocks = (a.count + kThreads - 1) / kThreads;
  k_shard_io<<<(int)(blocks < 4096 ? blocks : 4096), kThreads, 0, s>>>(a);
  return cudaGetLastError();
}
__global__ void k_set_state(DevState* st, double b1t, double b2t, uint64_t t, float S, uint32_t good, float inv) {
  st->b1t = b1t;
  st->b2t = b2t;
  st->t = t;
  st->S = S;
  st->good = good;
  st->inv_cur = inv;
  st->inv_adam = inv;
  st->skip = 1u;
  st->rec_t = t;
  st->rec_overflow = 0;
  st->rec_scale = S;
  st->rec_clip = 1.0f;
  st->rec_norm = 0.0;
}
cudaError_t launch_set_state(DevState* st, double b1t, double b2t, uint64_t t, float S, uint32_t good, float inv,
                             cudaStream_t s) {
  k_set_state<<<1, 1, 0, s>>>(st, b1t, b2t, t, S, good, inv);
  return cudaGetLastError();
}

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

}  // namespace zero
