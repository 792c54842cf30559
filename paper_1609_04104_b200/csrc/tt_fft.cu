// Batched ortho 1-D DFT down the columns of row-major (n x ncols) complex64
// matrices (sm_100a, shared memory).
//
// Replaces np.fft.fft / ifft (axis=0, norm="ortho") of the factor columns in
// build_phi (observation.py:225-226) and, through the separable identity
// ifft2(Xi) conj(B) = ifft_x(Xi conj(F_y B)), the 2-D inverse transform of
// _scatter_theta (tracker.py:186-188): no 2-D FFT is ever formed.
//
// Power-of-two n: one CTA transforms CB columns of one matrix entirely in
// shared memory with Stockham autosort passes (ping-pong buffers,
// twiddles from an fp64 sincospi table; radix-4 passes plus one radix-2 pass for odd
// log2 n). Other n: a direct DFT with the same
// sign/normalisation convention.

#include <math.h>

#include "tt_common.cuh"

#define FFT_NT 256

// Column-interleaved Stockham: the CTA's CB columns stay in their row-major order in shared memory
// ([n][CB], column fastest), so the global loads/stores are straight copies of contiguous row
// segments and every butterfly pass reads and writes consecutive columns across a warp (no bank
// conflicts). All of a thread's global loads are issued before the first shared-memory store.
#define FFT_LU 8
__global__ void __launch_bounds__(FFT_NT) fft_pow2_kernel(float2* __restrict__ data, int n, int logn, int ncols,
                                                          int CB, int inverse) {
  extern __shared__ __align__(16) unsigned char smem[];
  float2* buf0 = (float2*)smem;               // [n][CB]
  float2* buf1 = buf0 + (size_t)CB * n;       // [n][CB]
  float2* tw = buf1 + (size_t)CB * n;         // [n]
  const int tid = threadIdx.x, NT = blockDim.x;
  const int col0 = blockIdx.x * CB;
  const int cb = min(CB, ncols - col0);
  float2* mat = data + (size_t)blockIdx.y * n * ncols + col0;
  const double sgn = inverse ? 2.0 : -2.0;
  const int total = n * cb;
  for (int base = 0; base < total; base += NT * FFT_LU) {
    float2 v[FFT_LU];
#pragma unroll
    for (int u = 0; u < FFT_LU; ++u) {
      const int o = base + u * NT + tid;
      if (o < total) {
        const int i = idiv(o, cb), cc = o - i * cb;
        v[u] = mat[(size_t)i * ncols + cc];
      }
    }
#pragma unroll
    for (int u = 0; u < FFT_LU; ++u) {
      const int o = base + u * NT + tid;
      if (o < total) {
        const int i = idiv(o, cb);
        buf0[i * CB + (o - i * cb)] = v[u];
      }
    }
  }
  for (int m = tid; m < n; m += NT) {  // tw[m] = exp(+-2 pi i m / n); overlaps the loads in flight
    double sv, cv;
    sincospi(sgn * (double)m / (double)n, &sv, &cv);
    tw[m] = make_float2((float)cv, (float)sv);
  }
  __syncthreads();
  float2* in = buf0;
  float2* out = buf1;
  int Ns = 1, s = 0;
  if (logn & 1) {  // one radix-2 Stockham pass first when log2(n) is odd
    const int half = n >> 1, nb = half * cb;
    for (int o = tid; o < nb; o += NT) {
      const int j = idiv(o, cb), cc = o - j * cb;
      const float2 v0 = in[j * CB + cc];
      const float2 v1 = in[(j + half) * CB + cc];
      out[(2 * j) * CB + cc] = cadd(v0, v1);
      out[(2 * j + 1) * CB + cc] = csub(v0, v1);
    }
    __syncthreads();
    float2* t = in;
    in = out;
    out = t;
    Ns = 2;
    s = 1;
  }
  // radix-4 Stockham passes: a_q = x[j + q n/4] w^(q k), k = j mod Ns, w = exp(+-2 pi i / (4 Ns));
  // y[4(j - k) + k + m Ns] = sum_q a_q exp(+-2 pi i q m / 4)
  const int quarter = n >> 2, nb4 = quarter * cb;
  for (; s < logn; s += 2, Ns <<= 2) {
    const int tws = n / (4 * Ns);
    for (int o = tid; o < nb4; o += NT) {
      const int j = idiv(o, cb), cc = o - j * cb;
      const int k = j & (Ns - 1);
      const float2 x0 = in[j * CB + cc];
      const float2 x1 = cmul(in[(j + quarter) * CB + cc], tw[k * tws]);
      const float2 x2 = cmul(in[(j + 2 * quarter) * CB + cc], tw[2 * k * tws]);
      const float2 x3 = cmul(in[(j + 3 * quarter) * CB + cc], tw[3 * k * tws]);
      const float2 s02 = cadd(x0, x2), d02 = csub(x0, x2), s13 = cadd(x1, x3), d13 = csub(x1, x3);
      // w4 d13 with w4 = -i (forward) or +i (inverse)
      const float2 r13 = inverse ? make_float2(-d13.y, d13.x) : make_float2(d13.y, -d13.x);
      const int d = ((j - k) << 2) + k;
      out[d * CB + cc] = cadd(s02, s13);
      out[(d + Ns) * CB + cc] = cadd(d02, r13);
      out[(d + 2 * Ns) * CB + cc] = csub(s02, s13);
      out[(d + 3 * Ns) * CB + cc] = csub(d02, r13);
    }
    __syncthreads();
    float2* t = in;
    in = out;
    out = t;
  }
  const float scale = (float)(1.0 / sqrt((double)n));
  for (int o = tid; o < total; o += NT) {
    const int i = idiv(o, cb), cc = o - i * cb;
    mat[(size_t)i * ncols + cc] = cscale(in[i * CB + cc], scale);
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
    // whole rows of up to 32 columns per CTA, at most ~96 KB so that two CTAs share an SM
    int CB = ncols < 32 ? ncols : 32;
    while (CB > 1 && (size_t)(2 * CB * n + n) * sizeof(float2) > 96 * 1024) CB = (CB + 1) / 2;
    const size_t sm = (size_t)(2 * CB * n + n) * sizeof(float2);
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
