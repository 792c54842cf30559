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

#include "tt_block.cuh"

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
  if (tid < R && colsq[tid] == 0.0) *sh_zero = 1;
  for (int i = tid; i < n; i += NT) {
    double e = 0.0;
    for (int r = 0; r < R; ++r) {
      const float2 v = a[(size_t)i * R + r];
      if (colsq[r] > 0.0) e += ((double)v.x * v.x + (double)v.y * v.y) / colsq[r];
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

// entry scores: en_a (nx), en_b (ny) then the nx x ny map, normalised twice
__global__ void __launch_bounds__(SMP_NT) entry_energy_kernel(int nx, int ny, int R, const float2* __restrict__ a,
                                                              const float2* __restrict__ b, double* __restrict__ ws,
                                                              int32_t* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* colsq = (double*)smem;
  double* red = colsq + R;
  __shared__ int sh_zero;
  const bool oka = row_energies(a, nx, R, colsq, ws, red, &sh_zero);
  __syncthreads();
  const bool okb = row_energies(b, ny, R, colsq, ws + nx, red, &sh_zero);
  if ((!oka || !okb) && threadIdx.x == 0 && status) atomicOr(status, TT_ST_ZEROCOL);
  // total of raw scores: sum_ij (ea_i + eb_j) / (R (nx+ny)) = (ny sum ea + nx sum eb) / (R (nx+ny))
  const double sa = chunk_sum(ws, nx, red);
  const double sb = chunk_sum(ws + nx, ny, red);
  if (threadIdx.x == 0) {
    const double den = (double)R * (double)(nx + ny);
    ws[nx + ny] = ((double)ny * sa + (double)nx * sb) / den;
  }
}

__global__ void entry_map_kernel(int nx, int ny, int R, const double* __restrict__ ws, double beta,
                                 double* __restrict__ probs) {
  const size_t n = (size_t)nx * ny;
  const double den = (double)R * (double)(nx + ny);
  const double tot = ws[nx + ny];
  for (size_t o = blockIdx.x * (size_t)blockDim.x + threadIdx.x; o < n; o += (size_t)gridDim.x * blockDim.x) {
    const size_t i = o / ny, j = o - i * ny;
    const double raw = (ws[i] + ws[nx + j]) / den;
    probs[o] = (1.0 - beta) * (raw / tot) + beta / (double)n;
  }
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
                                                         int32_t* count, int k) {
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
                              &sh_flag);
  for (int i = threadIdx.x; i < k; i += blockDim.x) omega[(size_t)s * k + i] = i < S ? rows[i] : -1;
  if (threadIdx.x == 0) {
    count[s] = S;
    if (pos) pos[s] = p0 + (uint64_t)ndraw;
  }
}

// sequential renormalised draws without replacement (draw order)
__global__ void __launch_bounds__(SMP_NT) draw_wor_kernel(int n, const double* __restrict__ weights, int k,
                                                          uint64_t k0, uint64_t k1, uint64_t* pos,
                                                          int32_t* out, int32_t* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* w = (double*)smem;
  double* cdf = w + n;
  double* red = cdf + n;
  __shared__ int sh_amb, sh_idx;
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
  for (int m = 0; m < k; ++m) {
    const double u01 = philox_uniform(k0, k1, p0 + (uint64_t)m);
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
  if (tid == 0 && pos) pos[0] = p0 + (uint64_t)k;
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

extern "C" int tt_entry_scores(void* stream, int nx, int ny, int rank, const float* a, const float* b, double beta,
                               double* probs_out, int32_t* status) {
  if (nx < 1 || ny < 1 || rank < 1 || !a || !b || !probs_out) return tt_fail(TT_EINVAL, "tt_entry_scores: bad args");
  if (!(beta >= 0.0 && beta < 1.0)) return tt_fail(TT_EINVAL, "uniform blend weight must be in [0, 1)");
  // probs_out doubles as workspace for the energies only if large enough; use a temporary
  double* ws = nullptr;
  TT_CUDA_TRY(cudaMallocAsync((void**)&ws, sizeof(double) * (nx + ny + 1), (cudaStream_t)stream));
  const size_t sm = sizeof(double) * ((size_t)rank + 64);
  entry_energy_kernel<<<1, SMP_NT, sm, (cudaStream_t)stream>>>(nx, ny, rank, (const float2*)a, (const float2*)b, ws,
                                                                status);
  const size_t n = (size_t)nx * ny;
  int blocks = (int)((n + SMP_NT - 1) / SMP_NT);
  if (blocks > 4096) blocks = 4096;
  entry_map_kernel<<<blocks, SMP_NT, 0, (cudaStream_t)stream>>>(nx, ny, rank, ws, beta, probs_out);
  normalize_kernel<<<1, SMP_NT, 0, (cudaStream_t)stream>>>(n, probs_out);
  TT_CUDA_TRY(cudaFreeAsync(ws, (cudaStream_t)stream));
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

extern "C" int tt_draw_with_replacement(void* stream, int nslices, int n, const double* probs, int k,
                                        const int32_t* forced, int nforced, uint64_t key0, uint64_t key1,
                                        uint64_t* pos, int32_t* omega_out, int32_t* count_out) {
  if (nslices < 1 || n < 1 || k < 1 || !probs || !omega_out || !count_out)
    return tt_fail(TT_EINVAL, "trial count must be at least 1");
  if (nforced < 0 || nforced > k) return tt_fail(TT_EINVAL, "more forced indices than trials");
  if (nforced > 0 && !forced) return tt_fail(TT_EINVAL, "null forced list");
  const size_t sm = sizeof(double) * (2 * (size_t)n + 64) + sizeof(int) * 2 * (size_t)n;
  if (sm > 220 * 1024) return tt_fail(TT_EUNSUPPORTED, "draw domain too large for one CTA (n=%d)", n);
  TT_CUDA_TRY(cudaFuncSetAttribute(draw_wr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  draw_wr_kernel<<<nslices, SMP_NT, sm, (cudaStream_t)stream>>>(n, probs, k - nforced, forced, nforced, key0, key1,
                                                                  pos, omega_out, count_out, k);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

extern "C" int tt_draw_without_replacement(void* stream, int n, const double* weights, int k, uint64_t key0,
                                           uint64_t key1, uint64_t* pos, int32_t* out, int32_t* status) {
  if (n < 1 || k < 0 || !weights || (!out && k > 0)) return tt_fail(TT_EINVAL, "tt_draw_without_replacement: bad args");
  if (k > n) return tt_fail(TT_EINVAL, "cannot draw more items than have positive weight");
  if (k == 0) return TT_OK;
  const size_t sm = sizeof(double) * (2 * (size_t)n + 64);
  if (sm > 220 * 1024) return tt_fail(TT_EUNSUPPORTED, "draw domain too large for one CTA (n=%d)", n);
  TT_CUDA_TRY(cudaFuncSetAttribute(draw_wor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  draw_wor_kernel<<<1, SMP_NT, sm, (cudaStream_t)stream>>>(n, weights, k, key0, key1, pos, out, status);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}
