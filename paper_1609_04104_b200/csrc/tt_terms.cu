// Standalone pieces of the index-list step for the reference API functions
// that callers use on their own:
//   tt_residual    e = y - Phi gamma                      (tracker.py:388, instantaneous_cost :163-173)
//   tt_data_terms  D_A = conj(gamma) . Xi conj(Bh), D_B = conj(gamma) . Xi^T conj(Ah)
//                  (_gradient_data_terms, tracker.py:208-228) and the closed-form curvature
//                  c_r = max(max_i sum_{j:(i,j)} |Bh_jr|^2, max_j sum_i |Ah_ir|^2) of hessian_bound
//                  (tracker.py:337-364)
// on measurement-domain factors (Ah, Bh) = (F_x A, F_y B) for Fourier masks.

#include "tt_block.cuh"

__global__ void terms_resid_kernel(int nmeas, int R, const float2* __restrict__ ah, const float2* __restrict__ bh,
                                   const int* __restrict__ idx, const float2* __restrict__ y,
                                   const float2* __restrict__ gamma, float2* __restrict__ e) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nmeas; l += gridDim.x * blockDim.x) {
    const int i = idx[2 * l], j = idx[2 * l + 1];
    double2 s = make_double2(0.0, 0.0);
    for (int r = 0; r < R; ++r) s = zfma(zmul(to_d2(ah[(size_t)i * R + r]), to_d2(bh[(size_t)j * R + r])), to_d2(gamma[r]), s);
    e[l] = make_float2((float)((double)y[l].x - s.x), (float)((double)y[l].y - s.y));
  }
}

__global__ void terms_scatter_kernel(int nmeas, int ny, const int* __restrict__ idx, const float2* __restrict__ e,
                                     float2* __restrict__ xi, float* __restrict__ mk) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nmeas; l += gridDim.x * blockDim.x) {
    const size_t o = (size_t)idx[2 * l] * ny + idx[2 * l + 1];
    xi[o] = e[l];
    mk[o] = 1.f;
  }
}

// role 0: rows i -> D_A, c0 ; role 1: rows j -> D_B, c1   (one thread per (row, r))
__global__ void terms_backproj_kernel(int nx, int ny, int R, const float2* __restrict__ ah, const float2* __restrict__ bh,
                                      const float2* __restrict__ xi, const float* __restrict__ mk,
                                      const float2* __restrict__ gamma, float2* __restrict__ dA,
                                      float2* __restrict__ dB, float* __restrict__ c0, float* __restrict__ c1) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (blockIdx.y == 0) {
    if (o >= nx * R) return;
    const int i = o / R, r = o - i * R;
    float2 acc = make_float2(0.f, 0.f);
    float cs = 0.f;
    for (int j = 0; j < ny; ++j) {
      const float2 b = bh[(size_t)j * R + r];
      acc = cfma_conj(xi[(size_t)i * ny + j], b, acc);
      cs = fmaf(mk[(size_t)i * ny + j], cabs2(b), cs);
    }
    dA[o] = cmul(cconj(gamma[r]), acc);
    c0[o] = cs;
  } else {
    if (o >= ny * R) return;
    const int j = o / R, r = o - j * R;
    float2 acc = make_float2(0.f, 0.f);
    float cs = 0.f;
    for (int i = 0; i < nx; ++i) {
      const float2 a = ah[(size_t)i * R + r];
      acc = cfma_conj(xi[(size_t)i * ny + j], a, acc);
      cs = fmaf(mk[(size_t)i * ny + j], cabs2(a), cs);
    }
    dB[o] = cmul(cconj(gamma[r]), acc);
    c1[o] = cs;
  }
}

__global__ void terms_cmax_kernel(int nx, int ny, int R, const float* __restrict__ c0, const float* __restrict__ c1,
                                  double* __restrict__ cmax) {
  const int r = blockIdx.x;
  double m = 0.0;
  for (int i = threadIdx.x; i < nx; i += blockDim.x) m = fmax(m, (double)c0[(size_t)i * R + r]);
  for (int j = threadIdx.x; j < ny; j += blockDim.x) m = fmax(m, (double)c1[(size_t)j * R + r]);
  m = warp_max(m);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    cmax[r] = t;
  }
}

extern "C" size_t tt_terms_scratch_bytes(int nx, int ny, int rank) {
  const size_t a = ((size_t)nx * ny * 8 + 255) & ~(size_t)255;
  const size_t b = ((size_t)nx * ny * 4 + 255) & ~(size_t)255;
  const size_t c = ((size_t)(nx + ny) * rank * 4 + 255) & ~(size_t)255;
  return a + b + c;
}

extern "C" int tt_residual(void* stream, int nx, int ny, int rank, int nmeas, const float* ah, const float* bh,
                           const int32_t* idx, const float* y, const float* gamma, float* e_out) {
  (void)nx;
  (void)ny;
  if (rank < 1 || nmeas < 0) return tt_fail(TT_EINVAL, "tt_residual: bad shape");
  if (nmeas == 0) return TT_OK;
  if (!ah || !bh || !idx || !y || !gamma || !e_out) return tt_fail(TT_EINVAL, "tt_residual: null buffer");
  int blocks = (nmeas + 255) / 256;
  if (blocks > 2048) blocks = 2048;
  terms_resid_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(nmeas, rank, (const float2*)ah, (const float2*)bh, idx,
                                                                (const float2*)y, (const float2*)gamma, (float2*)e_out);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

extern "C" int tt_data_terms(void* stream, int nx, int ny, int rank, int nmeas, const float* ah, const float* bh,
                             const int32_t* idx, const float* e, const float* gamma, float* dA, float* dB,
                             double* cmax, void* scratch) {
  if (nx < 1 || ny < 1 || rank < 1 || nmeas < 0) return tt_fail(TT_EINVAL, "tt_data_terms: bad shape");
  if (!ah || !bh || !gamma || !dA || !dB || !cmax || !scratch || (nmeas > 0 && (!idx || !e)))
    return tt_fail(TT_EINVAL, "tt_data_terms: null buffer");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned char* sb = (unsigned char*)scratch;
  const size_t a = ((size_t)nx * ny * 8 + 255) & ~(size_t)255;
  const size_t b = ((size_t)nx * ny * 4 + 255) & ~(size_t)255;
  float2* xi = (float2*)sb;
  float* mk = (float*)(sb + a);
  float* c0 = (float*)(sb + a + b);
  float* c1 = c0 + (size_t)nx * rank;
  TT_CUDA_TRY(cudaMemsetAsync(xi, 0, sizeof(float2) * (size_t)nx * ny, st));
  TT_CUDA_TRY(cudaMemsetAsync(mk, 0, sizeof(float) * (size_t)nx * ny, st));
  if (nmeas > 0) {
    int blocks = (nmeas + 255) / 256;
    if (blocks > 2048) blocks = 2048;
    terms_scatter_kernel<<<blocks, 256, 0, st>>>(nmeas, ny, idx, (const float2*)e, xi, mk);
  }
  const int m = (nx > ny ? nx : ny) * rank;
  terms_backproj_kernel<<<dim3((m + 127) / 128, 2), 128, 0, st>>>(nx, ny, rank, (const float2*)ah, (const float2*)bh,
                                                                  xi, mk, (const float2*)gamma, (float2*)dA,
                                                                  (float2*)dB, c0, c1);
  terms_cmax_kernel<<<rank, 256, 0, st>>>(nx, ny, rank, c0, c1, cmax);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}
