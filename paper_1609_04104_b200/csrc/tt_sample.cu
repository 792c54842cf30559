// Informative randomized sampling (sampler.py, observation.py:274-323).
//
//  * tt_row_scores   — row_scores (sampler.py:115-128) with
//                      _normalized_row_energies (:77-85) and _blend (:88-92)
//  * tt_entry_scores — entry_scores (sampler.py:95-112)
//  * tt_draw_with_replacement — draw_samples(replacement=True) (:146-162):
//                      Generator(Philox).choice + np.union1d(forced, drawn)
//  * tt_draw_without_replacement — weighted_draw_without_replacement
//                      (observation.py:279-297), the engine of
//                      variable_density_rows (:300-323)
// All probability arithmetic is fp64. One CTA per slice (n <= 65536).

#include <stdlib.h>

#include <cooperative_groups.h>

#include "tt_block.cuh"

namespace cg = cooperative_groups;

#define SMP_NT 256

// row energies e_i = sum_r |a_ir|^2 / ||a_r||^2 into en[0..n); returns false on a zero column
TT_DEV bool row_energies(const float2* a, int n, int R, double* colsq, double* en, double* red, int* sh_zero) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = NT >> 5;
  if (tid == 0) *sh_zero = 0;
  for (int r = warp; r < R; r += nw) {
    double acc = 0.0;
    for (int i = lane; i < n; i += 32) {
      const float2 v = a[(size_t)i * R + r];
      acc += (double)v.x * v.x + (double)v.y * v.y;
    }
    acc = warp_sum(acc);
    if (lane == 0) colsq[r] = acc;
  }
  __syncthreads();
  if (tid < R) {  // reciprocal squared column norms, once per column
    if (colsq[tid] == 0.0) *sh_zero = 1;
    colsq[tid] = colsq[tid] > 0.0 ? 1.0 / colsq[tid] : 0.0;
  }
  __syncthreads();
  for (int i = tid; i < n; i += NT) {
    double e = 0.0;
    for (int r = 0; r < R; ++r) {
      const float2 v = a[(size_t)i * R + r];
      e += ((double)v.x * v.x + (double)v.y * v.y) * colsq[r];
    }
    en[i] = e;
  }
  __syncthreads();
  return *sh_zero == 0;
}

TT_DEV double chunk_sum(const double* v, int n, double* red) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int chunk = (n + NT - 1) / NT;
  const int c0 = min(n, tid * chunk), c1 = min(n, c0 + chunk);
  double loc = 0.0;
  for (int i = c0; i < c1; ++i) loc += v[i];
  return block_sum(loc, red);
}

__global__ void __launch_bounds__(SMP_NT) row_scores_kernel(int nx, int ny, int R, const float2* __restrict__ a,
                                                            double beta, double* __restrict__ probs,
                                                            int32_t* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* colsq = (double*)smem;
  double* red = colsq + R;
  double* p = red + 64;
  __shared__ int sh_zero;
  const int s = blockIdx.x;
  const float2* as = a + (size_t)s * nx * R;
  double* out = probs + (size_t)s * nx;
  const bool ok = row_energies(as, nx, R, colsq, p, red, &sh_zero);
  if (!ok && threadIdx.x == 0 && status) atomicOr(&status[s], TT_ST_ZEROCOL);
  for (int i = threadIdx.x; i < nx; i += blockDim.x)
    p[i] = ((double)ny * p[i] + (double)R) / ((double)R * (double)(nx + ny));
  __syncthreads();
  const double s1 = chunk_sum(p, nx, red);
  for (int i = threadIdx.x; i < nx; i += blockDim.x) p[i] = (1.0 - beta) * (p[i] / s1) + beta / (double)nx;
  __syncthreads();
  const double s2 = chunk_sum(p, nx, red);
  for (int i = threadIdx.x; i < nx; i += blockDim.x) out[i] = p[i] / s2;
}

// entry scores: en_a (nx), en_b (ny) then the nx x ny map, normalised twice. A two-CTA cluster:
// CTA 0 scores the rows of a, CTA 1 those of b; CTA 0 combines the two sums through DSMEM.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(SMP_NT)
    entry_energy_kernel(int nx, int ny, int R, const float2* __restrict__ a, const float2* __restrict__ b,
                        double* __restrict__ ws, int32_t* status) {
  pdl_wait_and_trigger();
  extern __shared__ __align__(16) unsigned char smem[];
  double* colsq = (double*)smem;
  double* red = colsq + R;
  __shared__ int sh_zero;
  __shared__ double sh_sum;
  cg::cluster_group cl = cg::this_cluster();
  const int k = (int)cl.block_rank();
  const int n = k ? ny : nx;
  const bool ok = row_energies(k ? b : a, n, R, colsq, ws + (k ? nx : 0), red, &sh_zero);
  if (!ok && threadIdx.x == 0 && status) atomicOr(status, TT_ST_ZEROCOL);
  // total of raw scores: sum_ij (ea_i + eb_j) / (R (nx+ny)) = (ny sum ea + nx sum eb) / (R (nx+ny))
  const double sk = chunk_sum(ws + (k ? nx : 0), n, red);
  if (threadIdx.x == 0) sh_sum = sk;
  cl.sync();
  if (k == 0 && threadIdx.x == 0) {
    const double sb = *cl.map_shared_rank(&sh_sum, 1);
    const double den = (double)R * (double)(nx + ny);
    ws[nx + ny] = ((double)ny * sh_sum + (double)nx * sb) / den;
  }
  cl.sync();
}

// blended probabilities (sampler.py:88-92) and their per-block partial sums (fixed order)
__global__ void __launch_bounds__(SMP_NT) entry_map_kernel(int nx, int ny, int R, const double* __restrict__ ws,
                                                           double beta, double* __restrict__ probs,
                                                           double* __restrict__ part) {
  pdl_wait_and_trigger();
  __shared__ double red[64];
  const size_t n = (size_t)nx * ny;
  const double den = (double)R * (double)(nx + ny);
  const double tot = ws[nx + ny];
  double loc = 0.0;
  for (size_t o = blockIdx.x * (size_t)blockDim.x + threadIdx.x; o < n; o += (size_t)gridDim.x * blockDim.x) {
    const size_t i = o / ny, j = o - i * ny;
    const double raw = (ws[i] + ws[nx + j]) / den;
    const double v = (1.0 - beta) * (raw / tot) + beta / (double)n;
    probs[o] = v;
    loc += v;
  }
  const double s = block_sum(loc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
// final renormalisation: every block sums the partials in the same order, then divides its share
__global__ void __launch_bounds__(SMP_NT) entry_norm_kernel(size_t n, int nparts, const double* __restrict__ part,
                                                            double* __restrict__ probs) {
  pdl_wait_and_trigger();
  __shared__ double red[64];
  __shared__ double tot;
  double loc = 0.0;
  for (int b = threadIdx.x; b < nparts; b += blockDim.x) loc += part[b];
  const double s = block_sum(loc, red);
  if (threadIdx.x == 0) tot = s;
  __syncthreads();
  for (size_t o = blockIdx.x * (size_t)blockDim.x + threadIdx.x; o < n; o += (size_t)gridDim.x * blockDim.x)
    probs[o] = probs[o] / tot;
}
__global__ void __launch_bounds__(SMP_NT) normalize_kernel(size_t n, double* __restrict__ probs) {
  __shared__ double red[64];
  __shared__ double tot;
  double loc = 0.0;
  const size_t chunk = (n + blockDim.x - 1) / blockDim.x;
  const size_t c0 = min(n, threadIdx.x * chunk), c1 = min(n, c0 + chunk);
  for (size_t i = c0; i < c1; ++i) loc += probs[i];
  const double s = block_sum(loc, red);
  if (threadIdx.x == 0) tot = s;
  __syncthreads();
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) probs[i] = probs[i] / tot;
}

__global__ void __launch_bounds__(SMP_NT) draw_wr_kernel(int n, const double* __restrict__ probs, int ndraw,
                                                         const int32_t* forced, int nforced, uint64_t k0,
                                                         uint64_t k1, uint64_t* pos, int32_t* omega,
                                                         int32_t* count, int k, const double* utab) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* p = (double*)smem;
  double* cdf = p + n;
  double* red = cdf + n;
  int* flags = (int*)(red + 64);
  int* rows = flags + n;
  __shared__ int sh_flag;
  const int s = blockIdx.x;
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = probs[(size_t)s * n + i];
  __syncthreads();
  const uint64_t p0 = pos ? pos[s] : 0ull;
  int S;
  draw_with_replacement_block(p, cdf, flags, rows, S, n, ndraw, forced, nforced, k0, k1 + (uint64_t)s, p0, red,
                              &sh_flag, utab ? utab + (size_t)s * ndraw : nullptr);
  for (int i = threadIdx.x; i < k; i += blockDim.x) omega[(size_t)s * k + i] = i < S ? rows[i] : -1;
  if (threadIdx.x == 0) {
    count[s] = S;
    if (pos) pos[s] = p0 + (uint64_t)ndraw;
  }
}

// sequential renormalised draws without replacement (draw order) of k items from the weights in w
// (shared memory, modified), uniforms m = 0..k-1 from the table or the Philox stream at pos p0 + m;
// out[m] (global) receives draw m
TT_DEV void wor_draw_block(double* w, double* cdf, double* red, int n, int k, const double* utab, uint64_t k0,
                           uint64_t k1, uint64_t p0, int32_t* out) {
  __shared__ int sh_amb, sh_idx;
  const int tid = threadIdx.x;
  for (int m = 0; m < k; ++m) {
    const double u01 = draw_uniform(utab, k0, k1, p0, (uint64_t)m);
    for (int exact = 0; exact < 2; ++exact) {
      block_cumsum(w, cdf, n, exact != 0, red);
      const double total = cdf[n - 1];
      const double u = u01 * total;  // observation.py:292
      if (tid == 0) {
        int idx = upper_bound_d(cdf, n, u);
        const double lo = idx > 0 ? cdf[idx - 1] : -1.0;
        const double hi = idx < n ? cdf[idx] : 2.0 * total + 1.0;
        const double tol = 1e-12 * (total > 0 ? total : 1.0);
        sh_amb = (!exact && (u - lo <= tol || hi - u <= tol)) ? 1 : 0;
        sh_idx = idx < n - 1 ? idx : n - 1;
      }
      __syncthreads();
      const int amb = sh_amb;
      __syncthreads();
      if (!amb) break;
    }
    if (tid == 0) {
      out[m] = sh_idx;
      w[sh_idx] = 0.0;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(SMP_NT) draw_wor_kernel(int n, const double* __restrict__ weights, int k,
                                                          uint64_t k0, uint64_t k1, uint64_t* pos,
                                                          int32_t* out, int32_t* status, const double* utab) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* w = (double*)smem;
  double* cdf = w + n;
  double* red = cdf + n;
  const int tid = threadIdx.x, NT = blockDim.x;
  for (int i = tid; i < n; i += NT) w[i] = weights[i];
  __syncthreads();
  int nz = 0;
  for (int i = tid; i < n; i += NT) nz += w[i] != 0.0;
  double nzd = block_sum((double)nz, red);
  if (nzd < (double)k) {
    if (tid == 0 && status) atomicOr(status, TT_ST_OVERFLOW);
    return;
  }
  const uint64_t p0 = pos ? pos[0] : 0ull;
  wor_draw_block(w, cdf, red, n, k, utab, k0, k1, p0, out);
  if (tid == 0 && pos) pos[0] = p0 + (uint64_t)k;
}

// variable_density_rows (observation.py:300-323) for a block of frames of every slice at once: block
// (f, s) draws frame f of slice s from the Philox stream (key0, key1 + s) at position
// pos0[s] + f (n_rows - 1): the DC row, then n_rows - 1 sequential draws without replacement with the
// host's weights d**alpha / 2, in draw order -> out[f][s][n_rows]
__global__ void __launch_bounds__(SMP_NT) vd_rows_batch_kernel(int nslices, int n, const double* __restrict__ weights,
                                                               int n_rows, uint64_t k0, uint64_t k1,
                                                               const uint64_t* __restrict__ pos0, int32_t* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* w = (double*)smem;
  double* cdf = w + n;
  double* red = cdf + n;
  const int f = blockIdx.x / nslices, s = blockIdx.x % nslices;
  for (int i = threadIdx.x; i < n; i += blockDim.x) w[i] = weights[i];
  __syncthreads();
  int32_t* o = out + ((size_t)f * nslices + s) * n_rows;
  if (threadIdx.x == 0) o[0] = 0;
  const uint64_t p0 = (pos0 ? pos0[s] : 0ull) + (uint64_t)f * (uint64_t)(n_rows - 1);
  wor_draw_block(w, cdf, red, n, n_rows - 1, nullptr, k0, k1 + (uint64_t)s, p0, o + 1);
}

extern "C" int tt_vd_rows_batch(void* stream, int frames, int nslices, int n, const double* weights, int n_rows,
                                uint64_t key0, uint64_t key1, const uint64_t* pos0, int32_t* out) {
  if (frames < 0 || nslices < 1 || n < 1 || n_rows < 1 || n_rows > n || !weights || !out)
    return tt_fail(TT_EINVAL, "tt_vd_rows_batch: bad args");
  if (frames == 0) return TT_OK;
  const size_t sm = sizeof(double) * (2 * (size_t)n + 64);
  if (sm > 220 * 1024) return tt_fail(TT_EUNSUPPORTED, "draw domain too large for one CTA (n=%d)", n);
  TT_CUDA_TRY(cudaFuncSetAttribute(vd_rows_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  vd_rows_batch_kernel<<<(unsigned)frames * (unsigned)nslices, SMP_NT, sm, (cudaStream_t)stream>>>(
      nslices, n, weights, n_rows, key0, key1, pos0, out);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

extern "C" int tt_row_scores(void* stream, int nslices, int nx, int ny, int rank, const float* a, double beta,
                             double* probs_out, int32_t* status) {
  if (nslices < 1 || nx < 1 || ny < 1 || rank < 1 || !a || !probs_out)
    return tt_fail(TT_EINVAL, "tt_row_scores: bad arguments");
  if (!(beta >= 0.0 && beta < 1.0)) return tt_fail(TT_EINVAL, "uniform blend weight must be in [0, 1)");
  const size_t sm = sizeof(double) * ((size_t)rank + 64 + nx);
  if (sm > 200 * 1024) return tt_fail(TT_EUNSUPPORTED, "tt_row_scores: nx too large");
  TT_CUDA_TRY(cudaFuncSetAttribute(row_scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  row_scores_kernel<<<nslices, SMP_NT, sm, (cudaStream_t)stream>>>(nx, ny, rank, (const float2*)a, beta,
                                                                     probs_out, status);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

static int entry_scores_run(cudaStream_t st, int nx, int ny, int rank, const float* a, const float* b, double beta,
                            double* probs_out, int32_t* status, double* ws);

extern "C" size_t tt_entry_scores_ws_bytes(int nx, int ny) {
  return sizeof(double) * ((size_t)(nx > 0 ? nx : 0) + (ny > 0 ? ny : 0) + 1 + 4096);
}

// entry_scores with a caller-owned workspace (tt_entry_scores_ws_bytes): no allocation per call
extern "C" int tt_entry_scores_ws(void* stream, int nx, int ny, int rank, const float* a, const float* b, double beta,
                                  double* probs_out, int32_t* status, void* ws) {
  if (nx < 1 || ny < 1 || rank < 1 || !a || !b || !probs_out || !ws)
    return tt_fail(TT_EINVAL, "tt_entry_scores_ws: bad args");
  if (!(beta >= 0.0 && beta < 1.0)) return tt_fail(TT_EINVAL, "uniform blend weight must be in [0, 1)");
  return entry_scores_run((cudaStream_t)stream, nx, ny, rank, a, b, beta, probs_out, status, (double*)ws);
}

extern "C" int tt_entry_scores(void* stream, int nx, int ny, int rank, const float* a, const float* b, double beta,
                               double* probs_out, int32_t* status) {
  if (nx < 1 || ny < 1 || rank < 1 || !a || !b || !probs_out) return tt_fail(TT_EINVAL, "tt_entry_scores: bad args");
  if (!(beta >= 0.0 && beta < 1.0)) return tt_fail(TT_EINVAL, "uniform blend weight must be in [0, 1)");
  double* ws = nullptr;
  TT_CUDA_TRY(cudaMallocAsync((void**)&ws, tt_entry_scores_ws_bytes(nx, ny), (cudaStream_t)stream));
  const int rc = entry_scores_run((cudaStream_t)stream, nx, ny, rank, a, b, beta, probs_out, status, ws);
  TT_CUDA_TRY(cudaFreeAsync(ws, (cudaStream_t)stream));
  return rc;
}

static int entry_scores_run(cudaStream_t st, int nx, int ny, int rank, const float* a, const float* b, double beta,
                            double* probs_out, int32_t* status, double* ws) {
  void* stream = (void*)st;
  const size_t sm = sizeof(double) * ((size_t)rank + 64);
  TT_CUDA_TRY(tt_launch_pdl(entry_energy_kernel, dim3(2), dim3(SMP_NT), sm, (cudaStream_t)stream,
      nx, ny, rank, (const float2*)a, (const float2*)b, ws, status));
  const size_t n = (size_t)nx * ny;
  int blocks = (int)((n + SMP_NT - 1) / SMP_NT);
  if (blocks > 4096) blocks = 4096;
  TT_CUDA_TRY(tt_launch_pdl(entry_map_kernel, dim3(blocks), dim3(SMP_NT), 0, (cudaStream_t)stream,
      nx, ny, rank, ws, beta, probs_out, ws + nx + ny + 1));
  TT_CUDA_TRY(tt_launch_pdl(entry_norm_kernel, dim3(blocks), dim3(SMP_NT), 0, (cudaStream_t)stream,
      n, blocks, ws + nx + ny + 1, probs_out));
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

static int draw_wr_run(void* stream, int nslices, int n, const double* probs, int k, const int32_t* forced,
                       int nforced, uint64_t key0, uint64_t key1, uint64_t* pos, int32_t* omega_out,
                       int32_t* count_out, const double* utab) {
  if (nslices < 1 || n < 1 || k < 1 || !probs || !omega_out || !count_out)
    return tt_fail(TT_EINVAL, "trial count must be at least 1");
  if (nforced < 0 || nforced > k) return tt_fail(TT_EINVAL, "more forced indices than trials");
  if (nforced > 0 && !forced) return tt_fail(TT_EINVAL, "null forced list");
  const size_t sm = sizeof(double) * (2 * (size_t)n + 64) + sizeof(int) * 2 * (size_t)n;
  if (sm > 220 * 1024) return tt_fail(TT_EUNSUPPORTED, "draw domain too large for one CTA (n=%d)", n);
  TT_CUDA_TRY(cudaFuncSetAttribute(draw_wr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  draw_wr_kernel<<<nslices, SMP_NT, sm, (cudaStream_t)stream>>>(n, probs, k - nforced, forced, nforced, key0, key1,
                                                                  pos, omega_out, count_out, k, utab);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

extern "C" int tt_draw_with_replacement(void* stream, int nslices, int n, const double* probs, int k,
                                        const int32_t* forced, int nforced, uint64_t key0, uint64_t key1,
                                        uint64_t* pos, int32_t* omega_out, int32_t* count_out) {
  return draw_wr_run(stream, nslices, n, probs, k, forced, nforced, key0, key1, pos, omega_out, count_out, nullptr);
}

extern "C" int tt_draw_with_replacement_u(void* stream, int nslices, int n, const double* probs, int k,
                                          const int32_t* forced, int nforced, const double* uniforms,
                                          int32_t* omega_out, int32_t* count_out) {
  if (!uniforms && k > nforced) return tt_fail(TT_EINVAL, "tt_draw_with_replacement_u: null uniforms");
  return draw_wr_run(stream, nslices, n, probs, k, forced, nforced, 0, 0, nullptr, omega_out, count_out, uniforms);
}

static int draw_wor_run(void* stream, int n, const double* weights, int k, uint64_t key0, uint64_t key1,
                        uint64_t* pos, int32_t* out, int32_t* status, const double* utab) {
  if (n < 1 || k < 0 || !weights || (!out && k > 0)) return tt_fail(TT_EINVAL, "tt_draw_without_replacement: bad args");
  if (k > n) return tt_fail(TT_EINVAL, "cannot draw more items than have positive weight");
  if (k == 0) return TT_OK;
  const size_t sm = sizeof(double) * (2 * (size_t)n + 64);
  if (sm > 220 * 1024) return tt_fail(TT_EUNSUPPORTED, "draw domain too large for one CTA (n=%d)", n);
  TT_CUDA_TRY(cudaFuncSetAttribute(draw_wor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  draw_wor_kernel<<<1, SMP_NT, sm, (cudaStream_t)stream>>>(n, weights, k, key0, key1, pos, out, status, utab);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

extern "C" int tt_draw_without_replacement(void* stream, int n, const double* weights, int k, uint64_t key0,
                                           uint64_t key1, uint64_t* pos, int32_t* out, int32_t* status) {
  return draw_wor_run(stream, n, weights, k, key0, key1, pos, out, status, nullptr);
}

extern "C" int tt_draw_without_replacement_u(void* stream, int n, const double* weights, int k,
                                             const double* uniforms, int32_t* out, int32_t* status) {
  if (!uniforms && k > 0) return tt_fail(TT_EINVAL, "tt_draw_without_replacement_u: null uniforms");
  return draw_wor_run(stream, n, weights, k, 0, 0, nullptr, out, status, uniforms);
}

// ---------------------------------------------------------------- draws over large domains (global memory)
// draw_samples(replacement=True) when the domain does not fit one CTA's shared
// memory (entry sampling over nx*ny, sampler.py:95-112 + :146-162). Same
// numpy semantics as draw_wr_kernel: cdf = cumsum(p) / cdf[-1],
// idx = searchsorted(cdf, u, 'right'), union with the forced indices. The
// cumsum is a two-level parallel scan; a uniform closer to a bucket edge than
// the scan's rounding bound triggers numpy's sequential cumsum and a redo, so
// the result equals numpy's for the same probabilities. Every step is a
// kernel with device-side control (graph-capturable).
#define BIG_IPT 8  // entries per thread in the block scan
struct BigDrawScratch {
  size_t cdf, part, off, flags, ctl, cpart, coff, cq, total;
};
// log2 of the coarse CDF stride: at most 4096 coarse points (32 KB of shared memory in the draw)
static inline int big_lstride(int n) {
  int ls = 4;
  while (((n + (1 << ls) - 1) >> ls) > 4096) ++ls;
  return ls;
}
static BigDrawScratch big_layout(int n) {
  BigDrawScratch s;
  const int nb = (n + SMP_NT * BIG_IPT - 1) / (SMP_NT * BIG_IPT);
  size_t o = 0;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  s.cdf = o;   o = al(o + sizeof(double) * ((size_t)n + 1));
  s.part = o;  o = al(o + sizeof(double) * (size_t)nb);
  s.off = o;   o = al(o + sizeof(double) * ((size_t)nb + 1));
  s.flags = o; o = al(o + sizeof(int) * (size_t)n);
  s.ctl = o;   o = al(o + sizeof(int) * 4);  // [0] ambiguity flag
  s.cpart = o; o = al(o + sizeof(int) * (size_t)nb);
  s.coff = o;  o = al(o + sizeof(int) * ((size_t)nb + 1));
  s.cq = o;    o = al(o + sizeof(double) * (size_t)((n + (1 << big_lstride(n)) - 1) >> big_lstride(n)));
  s.total = o;
  return s;
}

// level 1: block-local inclusive scan (thread-sequential chunks, fixed order) and block totals
__global__ void __launch_bounds__(SMP_NT) big_scan_kernel(int n, const double* __restrict__ p, double* __restrict__ cdf,
                                                          double* __restrict__ part, int* __restrict__ ctl,
                                                          double* __restrict__ cq, int lstride) {
  pdl_wait_and_trigger();
  __shared__ double red[64];
  const int tid = threadIdx.x;
  const int base = blockIdx.x * SMP_NT * BIG_IPT + tid * BIG_IPT;
  double v[BIG_IPT];
  double loc = 0.0;
#pragma unroll
  for (int q = 0; q < BIG_IPT; ++q) {
    v[q] = base + q < n ? p[base + q] : 0.0;
    loc += v[q];
  }
  double tot;
  double run = block_excl_scan_dbl(loc, red, tot);
  const int msk = (1 << lstride) - 1;
#pragma unroll
  for (int q = 0; q < BIG_IPT; ++q) {
    run += v[q];
    const int i = base + q;
    if (i < n) {
      cdf[i] = run;
      if ((i & msk) == msk || i == n - 1) cq[i >> lstride] = run;  // coarse point: last of its chunk
    }
  }
  if (tid == 0) part[blockIdx.x] = tot;
  if (blockIdx.x == 0 && tid == 0) ctl[0] = 0;  // the draw raises it for an ambiguous uniform
}

// level 2: exclusive offsets of the block totals (block-wide, fixed order) into `off` (shared memory
// of the draw kernel); off[nb] = grand total
TT_DEV void big_offsets(int nb, const double* __restrict__ part, double* off, double* red) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int chunk = (nb + NT - 1) / NT;
  const int c0 = min(nb, tid * chunk), c1 = min(nb, c0 + chunk);
  double loc = 0.0;
  for (int b = c0; b < c1; ++b) loc += part[b];
  double tot;
  double run = block_excl_scan_dbl(loc, red, tot);
  for (int b = c0; b < c1; ++b) {
    off[b] = run;
    run += part[b];
  }
  if (tid == 0) off[nb] = tot;
  __syncthreads();
}

TT_DEV double big_cdf(const double* cdf, const double* off, int i) {
  return cdf[i] + off[i / (SMP_NT * BIG_IPT)];
}

// Rounding bound for the ambiguity test, in normalised CDF units. numpy's value at index i is
// c_i = fl(N_i / N_{n-1}) with N the sequential cumsum; to first order in u = 2^-53 and with x_i the
// exact normalised prefix, |c_i - x_i| <= u x_i (i (1 - x_i) + n - i + 1) (N_i carries i roundings;
// N_{n-1} continues the same chain, so only the n-1-i later roundings and the first-i roundings
// weighted by 1 - x_i survive the ratio). Our two-level scan passes every term through at most
// `depth` additions, so our normalised prefix is within 2 depth u of x_i (absolute, since every
// partial sum is <= the total). 5% margin for second-order terms and x_i estimated by our value.
TT_DEV double big_bound(int i, int n, double x, double depth_term) {
  const double u = 1.1102230246251565e-16;
  x = fmin(fmax(x, 0.0), 1.0);
  return 1.05 * u * (x * ((double)i * (1.0 - x) + (double)(n - i) + 1.0) + depth_term);
}

// draws: one uniform per thread, binary search on the (unnormalised) global CDF against u * total;
// a draw whose uniform lies within the rounding bound of either bucket edge raises ctl[0]
__global__ void big_draw_kernel(int n, int ndraw, const double* __restrict__ cdf, const double* __restrict__ cq,
                                const double* __restrict__ part,
                                int nb, const int* __restrict__ forced, int nforced, uint64_t k0, uint64_t k1,
                                const uint64_t* __restrict__ pos, int* __restrict__ flags, int* __restrict__ ctl,
                                double depth_term, double gscale, int lstride, const double* __restrict__ utab) {
  pdl_wait_and_trigger();
  // coarse copy of the CDF in shared memory: the last value of every 2^lstride-entry chunk; a draw
  // searches the chunks there and only lstride levels in global memory
  extern __shared__ double coarse[];
  const int sw = 1 << lstride, nc = (n + sw - 1) >> lstride;
  double* off = coarse + nc;   // [nb + 1] block offsets
  double* red = off + nb + 1;  // [64]
  {  // coarse points written by the scan (block-local prefixes), all loads in flight
    constexpr int U = 16;
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = threadIdx.x + u * blockDim.x;
      v[u] = k < nc ? cq[k] : 0.0;
    }
    big_offsets(nb, part, off, red);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = threadIdx.x + u * blockDim.x;
      if (k < nc) coarse[k] = v[u] + off[min(((k + 1) << lstride) - 1, n - 1) / (SMP_NT * BIG_IPT)];
    }
    for (int k = threadIdx.x + U * blockDim.x; k < nc; k += blockDim.x)
      coarse[k] = cq[k] + off[min(((k + 1) << lstride) - 1, n - 1) / (SMP_NT * BIG_IPT)];
  }
  __syncthreads();
  const double total = off[nb];
  const uint64_t p0 = pos[0];
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < ndraw + nforced; m += gridDim.x * blockDim.x) {
    if (m >= ndraw) {
      const int f = forced[m - ndraw];
      if (f >= 0 && f < n) flags[f] = 1;
      continue;
    }
    const double u = draw_uniform(utab, k0, k1, p0, (uint64_t)m);
    const double ut = u * total;
    int lo = 0, hi = nc;  // first chunk whose last value exceeds ut
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (coarse[mid] <= ut) lo = mid + 1;
      else hi = mid;
    }
    int q;  // last index with cdf <= u (normalised)
    if (lo == nc) {
      q = n - 1;
    } else {
      const int base = lo << lstride, end = min(base + sw, n);
      q = base - 1;
      for (int step = sw >> 1; step > 0; step >>= 1) {
        const int cand = q + step;
        if (cand < end && big_cdf(cdf, off, cand) <= ut) q = cand;
      }
      if (q + 1 < end && big_cdf(cdf, off, q + 1) <= ut) q = q + 1;  // chunk of one past the halvings
    }
    const int idx = min(q + 1, n - 1);
    bool amb = false;
    if (idx > 0) {  // numpy must also see c_{idx-1} <= u
      const double lo = big_cdf(cdf, off, idx - 1) / total;
      amb |= u - lo <= gscale * big_bound(idx - 1, n, lo, depth_term);
    }
    if (idx < n - 1) {  // ... and c_idx > u (c_{n-1} == 1 exactly)
      const double hi = big_cdf(cdf, off, idx) / total;
      amb |= hi - u <= gscale * big_bound(idx, n, hi, depth_term);
    }
    if (amb) ctl[0] = 1;
    flags[idx] = 1;
  }
}

// exact fallback (runs only when a draw was ambiguous), part 1: numpy's sequential cumsum. The chain
// of dependent fp64 adds is inherently serial (8 cycles each); thread 0 runs it out of shared memory
// and stores its results straight to global memory while warps 1.. stage the next chunk into the
// other buffer, so the chain never waits on a load. cdf[n] = cdf[-1] for the normalisation pass.
__global__ void __launch_bounds__(SMP_NT) big_exact_kernel(int n, const double* __restrict__ p,
                                                           double* __restrict__ cdf, int* __restrict__ flags,
                                                           const int* __restrict__ ctl) {
  pdl_wait_and_trigger();
  if (ctl[0] == 0) return;
  constexpr int CH = 2048;
  __shared__ __align__(16) double buf[2][CH];
  const int tid = threadIdx.x;
  const int nch = (n + CH - 1) / CH;
  auto stage = [&](int c) {  // warps 1.. load chunk c
    const int base = c * CH, cnt = min(CH, n - base);
    for (int i = tid - 32; i < cnt; i += SMP_NT - 32) buf[c & 1][i] = p[base + i];
  };
  if (tid >= 32) stage(0);
  __syncthreads();
  double c = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    if (tid >= 32) {
      if (ch + 1 < nch) stage(ch + 1);
    } else if (tid == 0) {
      const double* b = buf[ch & 1];
      double* out = cdf + (size_t)ch * CH;
      const int cnt = min(CH, n - ch * CH);
      int i = 0;
      constexpr int U = 16;
      double v[U], w[U];  // register double buffer: the next U operands load under the current adds
      auto ld = [&](double* r, int at) {
#pragma unroll
        for (int q = 0; q < U; q += 2) {
          const double2 t = *reinterpret_cast<const double2*>(b + min(at + q, CH - 2));
          r[q] = t.x;
          r[q + 1] = t.y;
        }
      };
      ld(v, 0);
      for (; i + U <= cnt; i += U) {
        ld(w, i + U);
#pragma unroll
        for (int q = 0; q < U; ++q) {
          c += v[q];  // numpy's order
          v[q] = c;
        }
#pragma unroll
        for (int q = 0; q < U; q += 2) *reinterpret_cast<double2*>(out + i + q) = make_double2(v[q], v[q + 1]);
#pragma unroll
        for (int q = 0; q < U; ++q) v[q] = w[q];
      }
      for (; i < cnt; ++i) {
        c += b[i];
        out[i] = c;
      }
    }
    __syncthreads();
  }
  if (tid == 0) cdf[n] = c;
  for (int i = tid; i < n; i += SMP_NT) flags[i] = 0;  // the redo re-marks every draw
}

// exact fallback, part 2 (grid): every draw redone against numpy's CDF, cdf[i] / cdf[-1] evaluated at
// each probe (the same rounding as numpy's cdf /= cdf[-1]), forced entries re-marked
__global__ void big_exact_redo_kernel(int n, int ndraw, const double* __restrict__ cdf,
                                      const int* __restrict__ forced, int nforced, uint64_t k0, uint64_t k1,
                                      const uint64_t* __restrict__ pos, int* __restrict__ flags,
                                      const int* __restrict__ ctl, const double* __restrict__ utab) {
  pdl_wait_and_trigger();
  if (ctl[0] == 0) return;
  const double last = cdf[n];
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < ndraw + nforced; m += gridDim.x * blockDim.x) {
    if (m >= ndraw) {
      const int f = forced[m - ndraw];
      if (f >= 0 && f < n) flags[f] = 1;
      continue;
    }
    const double u = draw_uniform(utab, k0, k1, pos[0], (uint64_t)m);
    int lo = 0, hi = n;  // searchsorted(cdf / cdf[-1], u, 'right')
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cdf[mid] / last <= u) lo = mid + 1;
      else hi = mid;
    }
    flags[lo < n ? lo : n - 1] = 1;
  }
}

// flags -> sorted unique indices + count, in three block-parallel passes (per-block counts, one-block
// scan of the counts, writes); the writes clear the flags; the stream position advances by the draws
__global__ void __launch_bounds__(SMP_NT) big_count_kernel(int n, const int* __restrict__ flags,
                                                           int* __restrict__ cpart) {
  pdl_wait_and_trigger();
  __shared__ int red[64];
  const int base = blockIdx.x * SMP_NT * BIG_IPT + threadIdx.x * BIG_IPT;
  int c = 0;
#pragma unroll
  for (int q = 0; q < BIG_IPT; ++q) c += (base + q < n && flags[base + q]) ? 1 : 0;
  int tot;
  block_excl_scan_int(c, red, tot);
  if (threadIdx.x == 0) cpart[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(SMP_NT) big_write_kernel(int n, int nb, int ndraw, int cap, int* __restrict__ flags,
                                                           const int* __restrict__ cpart, uint64_t* __restrict__ pos,
                                                           int* __restrict__ omega, int* __restrict__ count) {
  pdl_wait_and_trigger();
  __shared__ int red[64];
  __shared__ int sh_pre, sh_all;
  {  // this block's offset (counts of the blocks before it) and the total: integer sums
    int pre = 0, all = 0;
    for (int q = threadIdx.x; q < nb; q += blockDim.x) {
      const int v = cpart[q];
      all += v;
      pre += q < (int)blockIdx.x ? v : 0;
    }
    int tp, ta;
    block_excl_scan_int(pre, red, tp);
    block_excl_scan_int(all, red, ta);
    if (threadIdx.x == 0) {
      sh_pre = tp;
      sh_all = ta;
    }
    __syncthreads();
  }
  const int base = blockIdx.x * SMP_NT * BIG_IPT + threadIdx.x * BIG_IPT;
  int f[BIG_IPT];
  int c = 0;
#pragma unroll
  for (int q = 0; q < BIG_IPT; ++q) {
    f[q] = (base + q < n) ? flags[base + q] : 0;
    c += f[q] ? 1 : 0;
  }
  int tot;
  int o = sh_pre + block_excl_scan_int(c, red, tot);
#pragma unroll
  for (int q = 0; q < BIG_IPT; ++q)
    if (f[q]) {
      if (o < cap) omega[o] = base + q;
      ++o;
      flags[base + q] = 0;
    }
  const int all = sh_all;
  if (blockIdx.x == 0) {
    for (int i = all + threadIdx.x; i < cap; i += blockDim.x) omega[i] = -1;  // deterministic padding
    if (threadIdx.x == 0) {
      *count = min(all, cap);
      pos[0] += (uint64_t)ndraw;
    }
  }
}

extern "C" size_t tt_draw_scratch_bytes(int n) { return n > 0 ? big_layout(n).total : 0; }

static int draw_large_run(void* stream, int n, const double* probs, int k, const int32_t* forced, int nforced,
                          uint64_t key0, uint64_t key1, uint64_t* pos, int32_t* omega_out, int32_t* count_out,
                          void* scratch, const double* utab) {
  if (n < 1 || k < 1 || !probs || !omega_out || !count_out || !pos || !scratch)
    return tt_fail(TT_EINVAL, "tt_draw_with_replacement_large: bad args");
  if (nforced < 0 || nforced > k) return tt_fail(TT_EINVAL, "more forced indices than trials");
  if (nforced > 0 && !forced) return tt_fail(TT_EINVAL, "null forced list");
  cudaStream_t st = (cudaStream_t)stream;
  const BigDrawScratch S = big_layout(n);
  unsigned char* sb = (unsigned char*)scratch;
  double* cdf = (double*)(sb + S.cdf);
  double* part = (double*)(sb + S.part);
  double* off = (double*)(sb + S.off);
  int* flags = (int*)(sb + S.flags);
  int* ctl = (int*)(sb + S.ctl);
  const int nb = (n + SMP_NT * BIG_IPT - 1) / (SMP_NT * BIG_IPT);
  const int ndraw = k - nforced;
  // addition depth of the two-level scan: thread chunk, warp shuffle scan, warp totals, x - v, block
  // offsets (per-thread chunk + the same block scan), final cdf + off; generous
  const double depth = 2.0 * BIG_IPT + 2.0 * (5 + SMP_NT / 32 + 2) + (double)((nb + SMP_NT - 1) / SMP_NT) + 8.0;
  const double depth_term = 2.0 * depth + 8.0;
  double gscale = 1.0;
  if (const char* e = getenv("TT_DRAW_FORCE_EXACT"))  // test hook: every draw takes the exact path
    if (e[0] == '1') gscale = 1e300;
  const int ls = big_lstride(n);
  double* cq = (double*)(sb + S.cq);
  TT_CUDA_TRY(tt_launch_pdl(big_scan_kernel, dim3(nb), dim3(SMP_NT), 0, st, n, probs, cdf, part, ctl, cq, ls));
  {
    int blocks = (ndraw + nforced + 255) / 256;
    if (blocks < 1) blocks = 1;
    if (blocks > 1184) blocks = 1184;
    const size_t csm = sizeof(double) * ((size_t)((n + (1 << ls) - 1) >> ls) + nb + 1 + 64);
    if (csm > 48 * 1024) {
      static size_t set_draw[TT_MAXDEV] = {0};
      TT_CUDA_TRY(tt_smem_attr((const void*)big_draw_kernel, csm, set_draw));
    }
    TT_CUDA_TRY(tt_launch_pdl(big_draw_kernel, dim3(blocks), dim3(256), csm, st,
        n, ndraw, cdf, cq, part, nb, forced, nforced, key0, key1, pos, flags, ctl, depth_term, gscale, ls, utab));
  }
  {  // exact fallback (each part exits at once unless a draw was ambiguous)
    TT_CUDA_TRY(tt_launch_pdl(big_exact_kernel, dim3(1), dim3(SMP_NT), 0, st, n, probs, cdf, flags, ctl));
    int rbk = (ndraw + nforced + 255) / 256;
    if (rbk < 1) rbk = 1;
    if (rbk > 1184) rbk = 1184;
    TT_CUDA_TRY(tt_launch_pdl(big_exact_redo_kernel, dim3(rbk), dim3(256), 0, st,
        n, ndraw, cdf, forced, nforced, key0, key1, pos, flags, ctl, utab));
  }
  int* cpart = (int*)(sb + S.cpart);
  int* coff = (int*)(sb + S.coff);
  TT_CUDA_TRY(tt_launch_pdl(big_count_kernel, dim3(nb), dim3(SMP_NT), 0, st, n, flags, cpart));
  TT_CUDA_TRY(tt_launch_pdl(big_write_kernel, dim3(nb), dim3(SMP_NT), 0, st,
      n, nb, ndraw, k, flags, cpart, pos, omega_out, count_out));
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

extern "C" int tt_draw_with_replacement_large(void* stream, int n, const double* probs, int k, const int32_t* forced,
                                              int nforced, uint64_t key0, uint64_t key1, uint64_t* pos,
                                              int32_t* omega_out, int32_t* count_out, void* scratch) {
  return draw_large_run(stream, n, probs, k, forced, nforced, key0, key1, pos, omega_out, count_out, scratch, nullptr);
}

extern "C" int tt_draw_with_replacement_large_u(void* stream, int n, const double* probs, int k,
                                                const int32_t* forced, int nforced, const double* uniforms,
                                                uint64_t* pos, int32_t* omega_out, int32_t* count_out,
                                                void* scratch) {
  if (!uniforms && k > nforced) return tt_fail(TT_EINVAL, "tt_draw_with_replacement_large_u: null uniforms");
  return draw_large_run(stream, n, probs, k, forced, nforced, 0, 0, pos, omega_out, count_out, scratch, uniforms);
}
