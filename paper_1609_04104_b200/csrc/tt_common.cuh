// Shared device helpers for the tensortrack B200 kernels (sm_100a).
//
// Complex values are float2 (complex64) in HBM/smem and double2 (complex128)
// for the R x R Gram / solve arithmetic. Conventions follow the reference
// (`pkg/src/tensortrack/observation.py:4-11`): unconjugated measurement
// pairing, plain transpose in synthesis, ortho unshifted DFTs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tensortrack_b200.h"

#define TT_DEV __device__ __forceinline__

// ---------------------------------------------------------------- launch attributes
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, size increase). Function
// attributes are per device, so each call site keeps one cached size per device in `cache`.
#define TT_MAXDEV 64
inline cudaError_t tt_smem_attr(const void* fn, size_t bytes, size_t* cache) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < TT_MAXDEV && cache[dev] >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && dev < TT_MAXDEV) cache[dev] = bytes;
  return e;
}

// ---------------------------------------------------------------- programmatic dependent launch
// The entry-sampling frame is a chain of ~14 small kernels. Launched with programmatic stream
// serialisation, each kernel's CTAs are scheduled while its predecessor drains (the predecessor
// triggers at its start); the kernel then waits (griddepcontrol.wait: predecessor complete, memory
// visible) before its first global access. Without the attribute both instructions are no-ops.
TT_DEV void pdl_wait_and_trigger() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline cudaError_t tt_launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...);
}

// ---------------------------------------------------------------- complex
TT_DEV float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
TT_DEV float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
TT_DEV float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
TT_DEV float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
TT_DEV float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
// acc += a * conj(b)
TT_DEV float2 cfma_conj(float2 a, float2 b, float2 acc) {
  acc.x = fmaf(a.x, b.x, fmaf(a.y, b.y, acc.x));
  acc.y = fmaf(a.y, b.x, fmaf(-a.x, b.y, acc.y));
  return acc;
}
// acc += a * b
TT_DEV float2 cfma(float2 a, float2 b, float2 acc) {
  acc.x = fmaf(a.x, b.x, fmaf(-a.y, b.y, acc.x));
  acc.y = fmaf(a.x, b.y, fmaf(a.y, b.x, acc.y));
  return acc;
}
TT_DEV float cabs2(float2 a) { return a.x * a.x + a.y * a.y; }

TT_DEV double2 zadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
TT_DEV double2 zsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
TT_DEV double2 zmul(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
TT_DEV double2 zconj(double2 a) { return make_double2(a.x, -a.y); }
TT_DEV double2 zscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// acc += conj(a) * b   (fp32 inputs, exact fp64 products)
TT_DEV double2 zfma_cj(float2 a, float2 b, double2 acc) {
  const double ax = a.x, ay = a.y, bx = b.x, by = b.y;
  acc.x = fma(ax, bx, fma(ay, by, acc.x));
  acc.y = fma(ax, by, fma(-ay, bx, acc.y));
  return acc;
}
TT_DEV double2 zfma_cj(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));
  return acc;
}
TT_DEV double2 zfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
  return acc;
}
TT_DEV float2 to_f2(double2 a) { return make_float2((float)a.x, (float)a.y); }
TT_DEV double2 to_d2(float2 a) { return make_double2((double)a.x, (double)a.y); }

// ---------------------------------------------------------------- warp/block reductions
// Exact a / b for 0 <= a < 2^22, b >= 1 (index arithmetic): fp32 reciprocal estimate + one
// correction step, ~7 instructions instead of the ~20 of a generic integer divide.
TT_DEV int idiv(int a, int b) {
  int q = __float2int_rz(__fmul_rz((float)a, __frcp_rz((float)b)));
  const int r = a - q * b;
  q += (r >= b) - (r < 0);
  return q;
}

TT_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
TT_DEV float warp_sumf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
TT_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block sum (fixed tree); `red` needs blockDim.x/32 doubles.
// All threads receive the result. Contains two __syncthreads.
TT_DEV double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += red[w];
  return s;
}

// ---------------------------------------------------------------- Philox4x64-10
// numpy.random.Philox restated (numpy/random/src/philox/philox.h): Random123
// constants, counter pre-incremented before every 4-word block, so stream
// word n comes from counter (n/4 + 1), lane n%4. Pinned bit-exact against
// numpy in tests/test_oracle.py (oracle) and tests/test_gpu_sampling.py.
struct Philox4x64 {
  uint64_t v[4];
};
TT_DEV Philox4x64 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  uint64_t x0 = c0, x1 = c1, x2 = 0, x3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    const uint64_t hi0 = __umul64hi(M0, x0), lo0 = M0 * x0;
    const uint64_t hi1 = __umul64hi(M1, x2), lo1 = M1 * x2;
    const uint64_t n0 = hi1 ^ x1 ^ k0, n2 = hi0 ^ x3 ^ k1;
    x0 = n0;
    x1 = lo1;
    x2 = n2;
    x3 = lo0;
  }
  Philox4x64 o;
  o.v[0] = x0;
  o.v[1] = x1;
  o.v[2] = x2;
  o.v[3] = x3;
  return o;
}
// Generator.random() value at stream position n.
TT_DEV double philox_uniform(uint64_t k0, uint64_t k1, uint64_t n) {
  const uint64_t blk = (n >> 2) + 1ull;  // 256-bit counter; n < 2^64 never carries past word 1
  const uint64_t c1 = (blk == 0ull) ? 1ull : 0ull;
  Philox4x64 b = philox4x64_10(blk, c1, k0, k1);
  const uint64_t w = b.v[n & 3ull];
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}
// Uniform of draw m: word pos + m of the Philox stream (key0, key1), or utab[m] when the caller
// supplied the uniforms (a host Generator over another bit generator drew them: Generator.random()
// values, which is what choice / the sequential draws consume one per draw)
TT_DEV double draw_uniform(const double* utab, uint64_t k0, uint64_t k1, uint64_t pos, uint64_t m) {
  return utab ? utab[m] : philox_uniform(k0, k1, pos + m);
}

// ---------------------------------------------------------------- misc
TT_DEV int iceil_div(int a, int b) { return (a + b - 1) / b; }
TT_DEV int part_begin(int n, int parts, int p) { return (int)(((long long)n * p) / parts); }

#define TT_CUDA_TRY(expr)                                  \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return tt_fail_cuda(_e, #expr); \
  } while (0)

int tt_fail_cuda(cudaError_t e, const char* what);
int tt_fail(int code, const char* fmt, ...);
