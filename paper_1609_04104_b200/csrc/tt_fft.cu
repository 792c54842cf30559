// Batched ortho 1-D DFT down the columns of row-major (n x ncols) complex64
// matrices (sm_100a, shared memory).
//
// Replaces np.fft.fft / ifft (axis=0, norm="ortho") of the factor columns in
// build_phi (observation.py:225-226) and, through the separable identity
// ifft2(Xi) conj(B) = ifft_x(Xi conj(F_y B)), the 2-D inverse transform of
// _scatter_theta (tracker.py:186-188): no 2-D FFT is ever formed.
//
// n = 16 ... 1024 (powers of two): a two-level transform n = N1 * N2 with every
// thread's N1 (then N2) points in registers and one exchange through shared
// memory (fft_reg2_kernel down the columns, fft_reg2_rows_kernel along the
// rows; HBM-bound). Other powers of two (and
// TT_FFT_STOCKHAM=1): one CTA transforms CB columns of one matrix entirely in
// shared memory with Stockham autosort passes (ping-pong buffers, radix-4
// passes plus one radix-2 pass for odd log2 n). Other n: a direct DFT with the
// same sign/normalisation convention. Twiddles are rounded from fp64 sincospi,
// cached per (device, n, direction) (TT_FFT_NO_TABLE=1: computed in the kernel).

#include <math.h>
#include <stdlib.h>

#include <mutex>

#include "tt_common.cuh"

#define FFT_NT 256

// Column-interleaved Stockham: the CTA's CB columns stay in their row-major order in shared memory
// ([n][CB], column fastest), so the global loads/stores are straight copies of contiguous row
// segments and every butterfly pass reads and writes consecutive columns across a warp (no bank
// conflicts). All of a thread's global loads are issued before the first shared-memory store.
#define FFT_LU 8
__global__ void __launch_bounds__(FFT_NT) fft_pow2_kernel(float2* __restrict__ data, int n, int logn, int ncols,
                                                          int CB, int inverse, const float2* __restrict__ twg) {
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
  if (twg) {  // the cached table of this (n, direction): the same values, one 8-byte load per entry
    for (int m = tid; m < n; m += NT) tw[m] = twg[m];
  } else {
    for (int m = tid; m < n; m += NT) {  // tw[m] = exp(+-2 pi i m / n); overlaps the loads in flight
      double sv, cv;
      sincospi(sgn * (double)m / (double)n, &sv, &cv);
      tw[m] = make_float2((float)cv, (float)sv);
    }
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

// ---------------------------------------------------------------- two-level register FFT
// n = N1 * N2 with N1, N2 in {8, 16, 32}: every thread transforms N1 (then N2) points in registers, so the
// CTA's columns cross shared memory once (one barrier) instead of once per radix-4 pass, and the global
// loads / stores go straight from / to registers as full row segments of CB columns:
//   Y[j][k1] = sum_q x[j + N2 q] w_N1^(q k1)                (stage 1: N1 points over q, per j)
//   X[k1 + N1 k2] = sum_j (w_n^(j k1) Y[j][k1]) w_N2^(j k2)  (stage 2: N2 points over j, per k1)
__constant__ float2 c_w32[32];  // exp(-2 pi i k / 32), rounded from fp64

template <int N>
struct RegFFT {
  // in-place natural-order DFT of x[0..N) (decimation in time, radix 2), forward sign; INV conjugates
  template <bool INV>
  static TT_DEV void run(float2 (&x)[N]) {
    float2 e[N / 2], o[N / 2];
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      e[i] = x[2 * i];
      o[i] = x[2 * i + 1];
    }
    RegFFT<N / 2>::template run<INV>(e);
    RegFFT<N / 2>::template run<INV>(o);
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
      float2 t;
      if (k == 0) {
        t = o[k];
      } else if (4 * k == N) {  // w = -i (forward), +i (inverse)
        t = INV ? make_float2(-o[k].y, o[k].x) : make_float2(o[k].y, -o[k].x);
      } else {
        float2 w = c_w32[k * (32 / N)];
        if (INV) w.y = -w.y;
        t = cmul(o[k], w);
      }
      x[k] = cadd(e[k], t);
      x[k + N / 2] = csub(e[k], t);
    }
  }
};
template <>
struct RegFFT<1> {
  template <bool INV>
  static TT_DEV void run(float2 (&)[1]) {}
};

template <int N1, int N2, int CB, bool INV>
__global__ void __launch_bounds__(FFT_NT) fft_reg2_kernel(float2* __restrict__ data, int ncols,
                                                          const float2* __restrict__ twg) {
  constexpr int n = N1 * N2;
  constexpr int KS = N2 * CB + CB;  // k1 stride: a warp's k1 groups land on distinct banks
  extern __shared__ __align__(16) unsigned char smem[];
  float2* ybuf = (float2*)smem;         // [N1][KS]
  float2* tw = ybuf + (size_t)N1 * KS;  // [n]
  const int tid = threadIdx.x;
  const int col0 = blockIdx.x * CB;
  const int cb = min(CB, ncols - col0);
  float2* mat = data + (size_t)blockIdx.y * n * ncols + col0;
  for (int m = tid; m < n; m += FFT_NT) tw[m] = twg[m];
  // stage 1, item (j, c): N1 points over q from global memory, twiddled into the exchange buffer
  auto load1 = [&](int it, float2 (&x)[N1]) {
    const int j = it / CB, c = it % CB;
    if (it < N2 * CB && c < cb) {
#pragma unroll
      for (int q = 0; q < N1; ++q) x[q] = mat[(size_t)(j + N2 * q) * ncols + c];
      RegFFT<N1>::template run<INV>(x);
    }
  };
  auto store1 = [&](int it, const float2 (&x)[N1]) {
    const int j = it / CB, c = it % CB;
    if (it < N2 * CB && c < cb) {
#pragma unroll
      for (int k1 = 0; k1 < N1; ++k1) ybuf[k1 * KS + j * CB + c] = k1 == 0 ? x[0] : cmul(x[k1], tw[j * k1]);
    }
  };
  {
    float2 x[N1];
    load1(tid, x);
    __syncthreads();  // the twiddle table; the first trip's loads and butterflies are ahead of it
    store1(tid, x);
    for (int it = tid + FFT_NT; it < N2 * CB; it += FFT_NT) {
      load1(it, x);
      store1(it, x);
    }
  }
  __syncthreads();
  const float scale = (float)(1.0 / sqrt((double)n));
  // stage 2, item (k1, c): N2 points over j, rows k1 + N1 k2 back to global memory
  for (int it = tid; it < N1 * CB; it += FFT_NT) {
    const int k1 = it / CB, c = it % CB;
    if (c >= cb) continue;
    float2 y[N2];
#pragma unroll
    for (int j = 0; j < N2; ++j) y[j] = ybuf[k1 * KS + j * CB + c];
    RegFFT<N2>::template run<INV>(y);
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) mat[(size_t)(k1 + N1 * k2) * ncols + c] = cscale(y[k2], scale);
  }
}

template <int N1, int N2, int CB>
static cudaError_t fft_reg2_launch(cudaStream_t st, float2* data, int ncols, int batch, int inverse,
                                   const float2* twg) {
  constexpr size_t sm = ((size_t)N1 * (N2 * CB + CB) + (size_t)N1 * N2) * sizeof(float2);
  static size_t cfg[2][TT_MAXDEV] = {{0}};
  dim3 grid((ncols + CB - 1) / CB, batch);
  if (inverse) {
    cudaError_t e = tt_smem_attr((const void*)fft_reg2_kernel<N1, N2, CB, true>, sm, cfg[1]);
    if (e != cudaSuccess) return e;
    fft_reg2_kernel<N1, N2, CB, true><<<grid, FFT_NT, sm, st>>>(data, ncols, twg);
  } else {
    cudaError_t e = tt_smem_attr((const void*)fft_reg2_kernel<N1, N2, CB, false>, sm, cfg[0]);
    if (e != cudaSuccess) return e;
    fft_reg2_kernel<N1, N2, CB, false><<<grid, FFT_NT, sm, st>>>(data, ncols, twg);
  }
  return cudaGetLastError();
}

// The same two-level transform along the LAST axis (rows of length n, in place): a CTA takes RB whole
// rows; lanes run over j (stage 1 loads x[r][j + N2 q]) and over k1 (stage 2 stores X[r][k1 + N1 k2]), so
// global accesses are contiguous runs of N2 / N1 elements. The exchange buffer is [r][j][k1] with an odd
// j stride (N1 + 1): stage 1 writes it down the j of a half-warp, stage 2 reads it along k1, both
// conflict-free for 8-byte elements. With tt_fft_cols this gives the 2-D transform without transposes.
template <int N1, int N2, int RB, bool INV>
__global__ void __launch_bounds__(FFT_NT) fft_reg2_rows_kernel(float2* __restrict__ data, long long nrows,
                                                               const float2* __restrict__ twg) {
  constexpr int n = N1 * N2;
  constexpr int JS = N1 + 1;
  constexpr int RS = N2 * JS + ((N1 == 8 && (N2 * JS) % 16 == 0) ? 8 : 0);
  extern __shared__ __align__(16) unsigned char smem[];
  float2* ybuf = (float2*)smem;         // [RB][RS]
  float2* tw = ybuf + (size_t)RB * RS;  // [n]
  const int tid = threadIdx.x;
  const long long row0 = (long long)blockIdx.x * RB;
  const int rb = (int)min((long long)RB, nrows - row0);
  float2* mat = data + (size_t)row0 * n;
  for (int m = tid; m < n; m += FFT_NT) tw[m] = twg[m];
  auto load1 = [&](int it, float2 (&x)[N1]) {
    const int r = it / N2, j = it % N2;
    if (it < RB * N2 && r < rb) {
#pragma unroll
      for (int q = 0; q < N1; ++q) x[q] = mat[(size_t)r * n + j + N2 * q];
      RegFFT<N1>::template run<INV>(x);
    }
  };
  auto store1 = [&](int it, const float2 (&x)[N1]) {
    const int r = it / N2, j = it % N2;
    if (it < RB * N2 && r < rb) {
#pragma unroll
      for (int k1 = 0; k1 < N1; ++k1) ybuf[r * RS + j * JS + k1] = k1 == 0 ? x[0] : cmul(x[k1], tw[j * k1]);
    }
  };
  {
    float2 x[N1];
    load1(tid, x);
    __syncthreads();  // the twiddle table
    store1(tid, x);
    for (int it = tid + FFT_NT; it < RB * N2; it += FFT_NT) {
      load1(it, x);
      store1(it, x);
    }
  }
  __syncthreads();
  const float scale = (float)(1.0 / sqrt((double)n));
  for (int it = tid; it < RB * N1; it += FFT_NT) {
    const int r = it / N1, k1 = it % N1;
    if (r >= rb) continue;
    float2 y[N2];
#pragma unroll
    for (int j = 0; j < N2; ++j) y[j] = ybuf[r * RS + j * JS + k1];
    RegFFT<N2>::template run<INV>(y);
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) mat[(size_t)r * n + k1 + N1 * k2] = cscale(y[k2], scale);
  }
}

template <int N1, int N2, int RB>
static cudaError_t fft_reg2_rows_launch(cudaStream_t st, float2* data, long long nrows, int inverse,
                                        const float2* twg) {
  constexpr int JS = N1 + 1;
  constexpr int RS = N2 * JS + ((N1 == 8 && (N2 * JS) % 16 == 0) ? 8 : 0);
  constexpr size_t sm = ((size_t)RB * RS + (size_t)N1 * N2) * sizeof(float2);
  static size_t cfg[2][TT_MAXDEV] = {{0}};
  const long long nblk = (nrows + RB - 1) / RB;
  if (nblk > 2147483647LL) return cudaErrorInvalidValue;
  dim3 grid((unsigned)nblk, 1);
  if (inverse) {
    cudaError_t e = tt_smem_attr((const void*)fft_reg2_rows_kernel<N1, N2, RB, true>, sm, cfg[1]);
    if (e != cudaSuccess) return e;
    fft_reg2_rows_kernel<N1, N2, RB, true><<<grid, FFT_NT, sm, st>>>(data, nrows, twg);
  } else {
    cudaError_t e = tt_smem_attr((const void*)fft_reg2_rows_kernel<N1, N2, RB, false>, sm, cfg[0]);
    if (e != cudaSuccess) return e;
    fft_reg2_rows_kernel<N1, N2, RB, false><<<grid, FFT_NT, sm, st>>>(data, nrows, twg);
  }
  return cudaGetLastError();
}

// exp(-2 pi i k / 32) into constant memory, once per device
static bool fft_w32_ready() {
  static bool done[TT_MAXDEV] = {false};
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= TT_MAXDEV) return false;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return true;
  float2 h[32];
  for (int k = 0; k < 32; ++k) {
    const double a = -2.0 * 3.14159265358979323846 * (double)k / 32.0;
    h[k] = make_float2((float)cos(a), (float)sin(a));
  }
  h[0] = make_float2(1.f, 0.f);
  h[8] = make_float2(0.f, -1.f);
  h[16] = make_float2(-1.f, 0.f);
  h[24] = make_float2(0.f, 1.f);
  if (cudaMemcpyToSymbol(c_w32, h, sizeof(h)) != cudaSuccess) {  // synchronous; fails inside a stream capture
    (void)cudaGetLastError();
    return false;
  }
  done[dev] = true;
  return true;
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

// exp(+-2 pi i m / n), m < n, rounded from fp64 (the values the kernel computes itself without a table)
__global__ void fft_twiddle_kernel(float2* __restrict__ tw, int n, int inverse) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  double sv, cv;
  sincospi((inverse ? 2.0 : -2.0) * (double)m / (double)n, &sv, &cv);
  tw[m] = make_float2((float)cv, (float)sv);
}

// Twiddle table of (device, log2 n, direction), built once: the per-CTA fp64 sincospi of n values cost
// more than the CTA's butterflies (each CTA transforms only CB <= 32 columns). Returns nullptr while the
// stream is being captured into a graph and the table does not exist yet (the kernel then computes its own).
static const float2* fft_twiddles(cudaStream_t st, int n, int logn, int inverse) {
  static float2* tab[TT_MAXDEV][13][2] = {};
  static std::mutex mu;
  if (getenv("TT_FFT_NO_TABLE")) return nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= TT_MAXDEV || logn > 12) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  float2*& t = tab[dev][logn][inverse ? 1 : 0];
  if (t) return t;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    (void)cudaGetLastError();
    return nullptr;
  }
  float2* p = nullptr;
  if (cudaMalloc(&p, (size_t)n * sizeof(float2)) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  fft_twiddle_kernel<<<(n + 255) / 256, 256, 0, st>>>(p, n, inverse);
  if (cudaStreamSynchronize(st) != cudaSuccess) {  // complete before any other stream reads it
    (void)cudaGetLastError();
    cudaFree(p);
    return nullptr;
  }
  t = p;
  return t;
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
    const float2* twg = fft_twiddles(st, n, logn, inverse);
    if (twg && n >= 16 && n <= 1024 && !getenv("TT_FFT_STOCKHAM") && fft_w32_ready()) {
      cudaError_t e = cudaSuccess;
      switch (n) {
        case 16: e = fft_reg2_launch<4, 4, 16>(st, (float2*)data, ncols, batch, inverse, twg); break;
        case 32: e = fft_reg2_launch<4, 8, 16>(st, (float2*)data, ncols, batch, inverse, twg); break;
        case 64: e = fft_reg2_launch<8, 8, 16>(st, (float2*)data, ncols, batch, inverse, twg); break;
        case 128: e = fft_reg2_launch<8, 16, 16>(st, (float2*)data, ncols, batch, inverse, twg); break;
        case 256: e = fft_reg2_launch<16, 16, 16>(st, (float2*)data, ncols, batch, inverse, twg); break;
        case 512: e = fft_reg2_launch<16, 32, 16>(st, (float2*)data, ncols, batch, inverse, twg); break;
        default: e = fft_reg2_launch<32, 32, 8>(st, (float2*)data, ncols, batch, inverse, twg); break;
      }
      TT_CUDA_TRY(e);
      return TT_OK;
    }
    // whole rows of up to 32 columns per CTA, at most ~96 KB so that two CTAs share an SM
    int CB = ncols < 32 ? ncols : 32;
    while (CB > 1 && (size_t)(2 * CB * n + n) * sizeof(float2) > 96 * 1024) CB = (CB + 1) / 2;
    const size_t sm = (size_t)(2 * CB * n + n) * sizeof(float2);
    static size_t cfg[TT_MAXDEV] = {0};
    TT_CUDA_TRY(tt_smem_attr((const void*)fft_pow2_kernel, sm, cfg));
    dim3 grid((ncols + CB - 1) / CB, batch);
    fft_pow2_kernel<<<grid, FFT_NT, sm, st>>>((float2*)data, n, logn, ncols, CB, inverse, twg);
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

// In-place ortho DFT along the last axis of nrows contiguous rows of n complex64 (n = 64, 128, 256, 512 or
// 1024; other lengths: TT_EUNSUPPORTED, the host then transposes and uses tt_fft_cols).
extern "C" int tt_fft_rows(void* stream, float* data, long long nrows, int n, int inverse) {
  if (n < 1 || nrows < 0 || !data) return tt_fail(TT_EINVAL, "tt_fft_rows: bad arguments");
  if (nrows == 0) return TT_OK;
  if (n != 16 && n != 32 && n != 64 && n != 128 && n != 256 && n != 512 && n != 1024)
    return tt_fail(TT_EUNSUPPORTED, "tt_fft_rows: n=%d (supported: powers of two from 16 to 1024)", n);
  cudaStream_t st = (cudaStream_t)stream;
  int logn = 0;
  while ((1 << logn) < n) ++logn;
  const float2* twg = fft_twiddles(st, n, logn, inverse);
  if (!twg || !fft_w32_ready())
    return tt_fail(TT_EUNSUPPORTED, "tt_fft_rows: twiddle tables unavailable (first call inside a stream capture?)");
  cudaError_t e = cudaSuccess;
  switch (n) {
    case 16: e = fft_reg2_rows_launch<4, 4, 64>(st, (float2*)data, nrows, inverse, twg); break;
    case 32: e = fft_reg2_rows_launch<4, 8, 32>(st, (float2*)data, nrows, inverse, twg); break;
    case 64: e = fft_reg2_rows_launch<8, 8, 32>(st, (float2*)data, nrows, inverse, twg); break;
    case 128: e = fft_reg2_rows_launch<8, 16, 16>(st, (float2*)data, nrows, inverse, twg); break;
    case 256: e = fft_reg2_rows_launch<16, 16, 16>(st, (float2*)data, nrows, inverse, twg); break;
    case 512: e = fft_reg2_rows_launch<16, 32, 16>(st, (float2*)data, nrows, inverse, twg); break;
    default: e = fft_reg2_rows_launch<32, 32, 8>(st, (float2*)data, nrows, inverse, twg); break;
  }
  TT_CUDA_TRY(e);
  return TT_OK;
}
