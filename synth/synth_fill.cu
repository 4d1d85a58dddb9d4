// GPU side of the shared seeded input generator (see synth/__init__.py for the
// recipe).  Re-implements the same counter-based splitmix64 stream so that the
// GPU tests and bench.py derive inputs on the device identical to the host ones;
// holds none of the method's arithmetic (the 16-bit cast of a generated input is
// input generation, RTNE like torch's CPU cast).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// out[i] = cast(x_{start+i} * scale), x in [-1, 1) on the 2^-23 grid;
// out_dtype 0 fp16, 1 bf16, 2 fp32; const_value: if use_const, out = cast(const_value)
__global__ void k_fill(void* out, uint64_t key, uint64_t start, uint64_t n, float scale, int out_dtype,
                       int use_const, float const_value) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    float y;
    if (use_const) {
      y = const_value;
    } else {
      const uint64_t h = splitmix64(key + start + i);
      const float x = (float)((int64_t)(h >> 40) - (1ll << 23)) * 0x1p-23f;
      y = x * scale;
    }
    if (out_dtype == 0) reinterpret_cast<__half*>(out)[i] = __float2half_rn(y);
    else if (out_dtype == 1) reinterpret_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(y);
    else reinterpret_cast<float*>(out)[i] = y;
  }
}

extern "C" int synth_fill(void* out, uint64_t key, uint64_t start, uint64_t n, float scale, int out_dtype,
                          int use_const, float const_value, void* stream) {
  if (n == 0) return 0;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_fill<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(out, key, start, n, scale, out_dtype,
                                                                              use_const, const_value);
  return (int)cudaGetLastError();
}
