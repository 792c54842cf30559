// Batched ortho 1-D DFT down the columns of row-major (n x ncols) complex64
// matrices (sm_100a, shared memory).
//
// Replaces np.fft.fft / ifft (axis=0, norm="ortho") of the factor columns in
// build_phi (observation.py:225-226) and, through the separable identity
// ifft2(Xi) conj(B) = ifft_x(Xi conj(F_y B)), the 2-D inverse transform of
// _scatter_theta (tracker.py:186-188): no 2-D FFT is ever formed.
//
// Power-of-two n: one CTA transforms CB columns of one matrix entirely in
// shared memory with radix-2 Stockham autosort passes (ping-pong buffers,
// twiddles from an fp64 sincospi table). Other n: a direct DFT with the same
// sign/normalisation convention.

#include <math.h>

#include "tt_common.cuh"

#define FFT_NT 256

__global__ void __launch_bounds__(FFT_NT) fft_pow2_kernel(float2* __restrict__ data, int n, int logn, int ncols,
                                                          int CB, int inverse) {
  extern __shared__ __align__(16) unsigned char smem[];
  float2* buf0 = (float2*)smem;               // [CB][n]
  float2* buf1 = buf0 + (size_t)CB * n;       // [CB][n]
  float2* tw = buf1 + (size_t)CB * n;         // [n/2]
  const int tid = threadIdx.x, NT = blockDim.x;
  const int col0 = blockIdx.x * CB;
  const int cb = min(CB, ncols - col0);
  float2* mat = data + (size_t)blockIdx.y * n * ncols;
  const double sgn = inverse ? 2.0 : -2.0;
  for (int m = tid; m < n / 2; m += NT) {
    double sv, cv;
    sincospi(sgn * (double)m / (double)n, &sv, &cv);
    tw[m] = make_float2((float)cv, (float)sv);
  }
  for (int o = tid; o < n * cb; o += NT) {
    const int i = o / cb, cc = o - i * cb;
    buf0[cc * n + i] = mat[(size_t)i * ncols + col0 + cc];
  }
  __syncthreads();
  float2* in = buf0;
  float2* out = buf1;
  const int half = n >> 1;
  for (int s = 0, Ns = 1; s < logn; ++s, Ns <<= 1) {
    for (int o = tid; o < half * cb; o += NT) {
      const int cc = o / half, j = o - cc * half;
      const float2* x = in + cc * n;
      float2* y = out + cc * n;
      const int k = j & (Ns - 1);
      const float2 w = tw[k * (half / Ns)];
      const float2 v0 = x[j];
      const float2 v1 = cmul(x[j + half], w);
      const int d = ((j - k) << 1) + k;
      y[d] = cadd(v0, v1);
      y[d + Ns] = csub(v0, v1);
    }
    __syncthreads();
    float2* t = in;
    in = out;
    out = t;
  }
  const float scale = (float)(1.0 / sqrt((double)n));
  for (int o = tid; o < n * cb; o += NT) {
    const int i = o / cb, cc = o - i * cb;
    mat[(size_t)i * ncols + col0 + cc] = cscale(in[cc * n + i], scale);
  }
}

// Direct DFT for any n: each CTA handles CB columns of one matrix.
__global__ void __launch_bounds__(FFT_NT) dft_direct_kernel(float2* __restrict__ data, int n, int ncols, int CB,
                                                            int inverse) {
  extern __shared__ __align__(16) unsigned char smem[];
  float2* xin = (float2*)smem;            // [CB][n]
  float2* tw = xin + (size_t)CB * n;      // [n]
  const int tid = threadIdx.x, NT = blockDim.x;
  const int col0 = blockIdx.x * CB;
  const int cb = min(CB, ncols - col0);
  float2* mat = data + (size_t)blockIdx.y * n * ncols;
  const double sgn = inverse ? 2.0 : -2.0;
  for (int m = tid; m < n; m += NT) {
    double sv, cv;
    sincospi(sgn * (double)m / (double)n, &sv, &cv);
    tw[m] = make_float2((float)cv, (float)sv);
  }
  for (int o = tid; o < n * cb; o += NT) {
    const int i = o / cb, cc = o - i * cb;
    xin[cc * n + i] = mat[(size_t)i * ncols + col0 + cc];
  }
  __syncthreads();
  const double scale = 1.0 / sqrt((double)n);
  for (int o = tid; o < n * cb; o += NT) {
    const int kk = o / cb, cc = o - kk * cb;
    double2 acc = make_double2(0.0, 0.0);
    int idx = 0;
    for (int i = 0; i < n; ++i) {
      const float2 x = xin[cc * n + i], w = tw[idx];
      acc.x += (double)x.x * w.x - (double)x.y * w.y;
      acc.y += (double)x.x * w.y + (double)x.y * w.x;
      idx += kk;
      if (idx >= n) idx -= n;
    }
    mat[(size_t)kk * ncols + col0 + cc] = make_float2((float)(acc.x * scale), (float)(acc.y * scale));
  }
}

extern "C" int tt_fft_cols(void* stream, float* data, int n, int ncols, int batch, int inverse) {
  if (n < 1 || ncols < 1 || batch < 0 || !data) return tt_fail(TT_EINVAL, "tt_fft_cols: bad arguments");
  if (batch == 0) return TT_OK;
  if (batch > 65535) return tt_fail(TT_EINVAL, "tt_fft_cols: batch > 65535");
  cudaStream_t st = (cudaStream_t)stream;
  const bool pow2 = (n & (n - 1)) == 0;
  if (pow2 && n >= 2 && n <= 4096) {
    int logn = 0;
    while ((1 << logn) < n) ++logn;
    int CB = 16;
    while (CB > 1 && (size_t)(2 * CB * n + n / 2) * sizeof(float2) > 200 * 1024) CB >>= 1;
    if (CB > ncols) CB = ncols;
    const size_t sm = (size_t)(2 * CB * n + n / 2) * sizeof(float2);
    static size_t cfg[TT_MAXDEV] = {0};
    TT_CUDA_TRY(tt_smem_attr((const void*)fft_pow2_kernel, sm, cfg));
    dim3 grid((ncols + CB - 1) / CB, batch);
    fft_pow2_kernel<<<grid, FFT_NT, sm, st>>>((float2*)data, n, logn, ncols, CB, inverse);
  } else if (n == 1) {
    return TT_OK;  // a length-1 ortho DFT is the identity
  } else {
    if (n > 8192) return tt_fail(TT_EUNSUPPORTED, "tt_fft_cols: non-power-of-two n=%d too large", n);
    int CB = 8;
    while (CB > 1 && (size_t)(CB * n + n) * sizeof(float2) > 200 * 1024) CB >>= 1;
    if (CB > ncols) CB = ncols;
    const size_t sm = (size_t)(CB * n + n) * sizeof(float2);
    static size_t cfg2[TT_MAXDEV] = {0};
    TT_CUDA_TRY(tt_smem_attr((const void*)dft_direct_kernel, sm, cfg2));
    dim3 grid((ncols + CB - 1) / CB, batch);
    dft_direct_kernel<<<grid, FFT_NT, sm, st>>>((float2*)data, n, ncols, CB, inverse);
  }
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}
