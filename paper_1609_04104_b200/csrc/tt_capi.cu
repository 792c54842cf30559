// C ABI glue: error reporting, version, and the small value ops
// (rebalance, generic solve_gamma). Kernel entry points live with their
// kernels (tt_rows.cu, tt_entries.cu, tt_fft.cu, tt_sample.cu, tt_recon.cu).

#include <stdarg.h>
#include <stdio.h>

#include "tt_block.cuh"

static thread_local char g_err[512] = "";

int tt_fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int tt_fail_cuda(cudaError_t e, const char* what) {
  snprintf(g_err, sizeof(g_err), "CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
  return TT_ECUDA;
}

extern "C" const char* tt_version(void) { return "tensortrack_b200 0.1.0 (sm_100a)"; }
extern "C" const char* tt_last_error(void) { return g_err; }

// ---------------------------------------------------------------- rebalance (core.py:138-166)
__global__ void __launch_bounds__(256) rebalance_kernel(int nx, int ny, int R, float2* a, float2* b, int32_t* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* na = (double*)smem;
  double* nb = na + R;
  const int s = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  float2* as = a + (size_t)s * nx * R;
  float2* bs = b + (size_t)s * ny * R;
  for (int r = warp; r < 2 * R; r += nw) {
    const bool isa = r < R;
    const int rr = isa ? r : r - R;
    const int n = isa ? nx : ny;
    const float2* f = isa ? as : bs;
    double acc = 0.0;
    for (int i = lane; i < n; i += 32) {
      const float2 v = f[(size_t)i * R + rr];
      acc += (double)v.x * v.x + (double)v.y * v.y;
    }
    acc = warp_sum(acc);
    if (lane == 0) (isa ? na : nb)[rr] = sqrt(acc);
  }
  __syncthreads();
  for (int o = tid; o < (nx + ny) * R; o += blockDim.x) {
    const bool isa = o < nx * R;
    const int k = isa ? o : o - nx * R;
    const int r = k % R;
    const double x = na[r], y = nb[r];
    double sc = 1.0;
    if (x == 0.0 && y == 0.0) sc = 1.0;                       // dead component stays zero
    else if (x == 0.0 || y == 0.0) {                          // mixed: no norm-preserving rescaling
      if (status && o == 0) atomicOr(&status[s], TT_ST_ZEROCOL);
      sc = 1.0;
    } else {
      const double g = sqrt(x * y);
      sc = isa ? g / x : g / y;
    }
    float2* f = isa ? as : bs;
    f[k] = cscale(f[k], (float)sc);
  }
}

extern "C" int tt_rebalance(void* stream, int nslices, int nx, int ny, int rank, float* a, float* b, int32_t* status) {
  if (nslices < 1 || nx < 1 || ny < 1 || rank < 1 || !a || !b) return tt_fail(TT_EINVAL, "tt_rebalance: bad args");
  rebalance_kernel<<<nslices, 256, sizeof(double) * 2 * rank, (cudaStream_t)stream>>>(nx, ny, rank, (float2*)a,
                                                                                       (float2*)b, status);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

// ---------------------------------------------------------------- generic solve_gamma (tracker.py:139-156)
// (Phi^H Phi + lam I) gamma = Phi^H y for a dense complex128 Phi: one CTA,
// fp64 Gram accumulation in a fixed order, LDL^H solve.
__global__ void __launch_bounds__(256) solve_gamma_kernel(int L, int R, const double2* __restrict__ phi,
                                                          const double2* __restrict__ y, double lam,
                                                          double2* __restrict__ gamma) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int Rp = R * (R + 1) / 2;
  double2* G = (double2*)smem;
  double2* hv = G + Rp;
  double2* gam = hv + R;
  const int tid = threadIdx.x;
  for (int e = tid; e < Rp + R; e += blockDim.x) {
    if (e < Rp) {
      int r, q;
      tri_decode(e, r, q);
      double2 g = make_double2(0.0, 0.0);
      for (int l = 0; l < L; ++l) g = zfma_cj(phi[(size_t)l * R + r], phi[(size_t)l * R + q], g);
      if (r == q) g.x += lam;
      G[e] = g;
    } else {
      const int r = e - Rp;
      double2 h = make_double2(0.0, 0.0);
      for (int l = 0; l < L; ++l) h = zfma_cj(phi[(size_t)l * R + r], y[l], h);
      hv[r] = h;
    }
  }
  block_ldl_solve(G, hv, gam, R);
  for (int r = tid; r < R; r += blockDim.x) gamma[r] = L > 0 ? gam[r] : make_double2(0.0, 0.0);
}

extern "C" size_t tt_solve_scratch_bytes(int L, int R) {
  (void)L;
  (void)R;
  return 0;
}

extern "C" int tt_solve_gamma(void* stream, int L, int R, const double* phi, const double* y, double lam,
                              double* gamma_out, void* scratch) {
  (void)scratch;
  if (L < 0 || R < 1 || !gamma_out || (L > 0 && (!phi || !y))) return tt_fail(TT_EINVAL, "tt_solve_gamma: bad args");
  if (R > 64) return tt_fail(TT_EUNSUPPORTED, "tt_solve_gamma: R > 64");
  if (lam < 0) return tt_fail(TT_EINVAL, "lambda must be nonnegative");
  const size_t sm = sizeof(double2) * ((size_t)R * (R + 1) / 2 + 2 * (size_t)R);
  TT_CUDA_TRY(cudaFuncSetAttribute(solve_gamma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  solve_gamma_kernel<<<1, 256, sm, (cudaStream_t)stream>>>(L, R, (const double2*)phi, (const double2*)y, lam,
                                                           (double2*)gamma_out);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

// ---------------------------------------------------------------- norm_cap flags (tracker.py:406-408)
// Squared Frobenius norms of `batch` complex64 matrices of `n` elements each (fp64, fixed order: one CTA
// per matrix, block-strided partials then a fixed tree): the post-update factor norms of a factor history.
__global__ void __launch_bounds__(256) factor_norms2_kernel(size_t n, const float2* __restrict__ x, double* out) {
  __shared__ double red[8];
  const float2* p = x + (size_t)blockIdx.x * n;
  double acc = 0.0;
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) acc += (double)p[i].x * p[i].x + (double)p[i].y * p[i].y;
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

extern "C" int tt_factor_norms2(void* stream, int batch, size_t n, const float* x, double* out) {
  if (batch < 0 || (batch > 0 && (!x || !out))) return tt_fail(TT_EINVAL, "tt_factor_norms2: bad args");
  if (batch == 0) return TT_OK;
  factor_norms2_kernel<<<batch, 256, 0, (cudaStream_t)stream>>>(n, (const float2*)x, out);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}
