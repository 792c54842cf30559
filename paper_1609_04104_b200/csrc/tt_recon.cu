// Frame reconstruction X_f = A_f diag(gamma_f) B_f^T, batched over frames.
//
// Reference: core.synthesize_slice (core.py:91-104, einsum over the rank) and
// mri.reconstruct_frame (mri.py:107-121, (A1 * gamma) @ A2.T, plain
// transpose). In run_adaptive it is called once per frame with the
// post-update factors and that frame's gamma (experiment.py:525).
//
// Each CTA produces a 64 x 64 output tile: the gamma-scaled A tile and the B
// tile are staged transposed ([r][64]) in shared memory and every thread
// accumulates a 4 x 4 register block over r (complex fp32 FMAs), then writes
// rows of 16 consecutive complex64 values (128 B segments).

#include "tt_common.cuh"

#define RC_T 64
#define RC_NT 256
#define RC_RMAX 64
#define RC_TP (RC_T + 1)  // padded row of the staged [r][64] tiles: conflict-free transposing stores

__global__ void __launch_bounds__(RC_NT) recon_kernel(int nx, int ny, int R, const float2* __restrict__ A,
                                                      const float2* __restrict__ B, const float2* __restrict__ gamma,
                                                      float2* __restrict__ X) {
  extern __shared__ __align__(16) float2 rsm[];
  float2* as = rsm;               // [R][RC_TP]
  float2* bs = rsm + R * RC_TP;   // [R][RC_TP]
  const int tid = threadIdx.x;
  const int f = blockIdx.z;
  const int i0 = blockIdx.y * RC_T, j0 = blockIdx.x * RC_T;
  const float2* Af = A + (size_t)f * nx * R;
  const float2* Bf = B + (size_t)f * ny * R;
  const float2* gf = gamma + (size_t)f * R;
  // staging: all of a thread's global loads in flight before the first shared-memory store
  // (the A / B tiles are contiguous rows of R values; up to 4 (A, B) pairs per thread per batch)
  for (int base = 0; base < RC_T * R; base += 4 * RC_NT) {
    float2 va[4], vb[4], vg[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int o = base + u * RC_NT + tid;
      va[u] = vb[u] = vg[u] = make_float2(0.f, 0.f);
      if (o < RC_T * R) {
        const int ii = idiv(o, R), r = o - ii * R;
        const int i = i0 + ii, j = j0 + ii;
        vg[u] = gf[r];
        if (i < nx) va[u] = Af[(size_t)i * R + r];
        if (j < ny) vb[u] = Bf[(size_t)j * R + r];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int o = base + u * RC_NT + tid;
      if (o < RC_T * R) {
        const int ii = idiv(o, R), r = o - ii * R;
        as[r * RC_TP + ii] = cmul(va[u], vg[u]);
        bs[r * RC_TP + ii] = vb[u];
      }
    }
  }
  __syncthreads();
  const int tj = tid & 15, ti = tid >> 4;  // 16 x 16 threads, 4 x 4 outputs each
  float2 acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = make_float2(0.f, 0.f);
  for (int r = 0; r < R; ++r) {
    float2 av[4], bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) av[u] = as[r * RC_TP + ti + 16 * u];
#pragma unroll
    for (int v = 0; v < 4; ++v) bv[v] = bs[r * RC_TP + tj + 16 * v];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = cfma(av[u], bv[v], acc[u][v]);
  }
  float2* Xf = X + (size_t)f * nx * ny;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = i0 + ti + 16 * u;
    if (i >= nx) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int j = j0 + tj + 16 * v;
      if (j < ny) Xf[(size_t)i * ny + j] = acc[u][v];
    }
  }
}

extern "C" int tt_reconstruct(void* stream, int frames, int nx, int ny, int rank, const float* a, const float* b,
                              const float* gamma, float* x_out) {
  if (frames < 0 || nx < 1 || ny < 1 || rank < 1 || !a || !b || !gamma || !x_out)
    return tt_fail(TT_EINVAL, "tt_reconstruct: bad arguments");
  if (rank > RC_RMAX) return tt_fail(TT_EUNSUPPORTED, "tt_reconstruct: rank > %d", RC_RMAX);
  if (frames == 0) return TT_OK;
  if (frames > 65535) return tt_fail(TT_EINVAL, "tt_reconstruct: frames > 65535 per call");
  const size_t sm = sizeof(float2) * 2 * RC_TP * (size_t)rank;
  static size_t cfg[TT_MAXDEV] = {0};
  TT_CUDA_TRY(tt_smem_attr((const void*)recon_kernel, sm, cfg));
  dim3 grid((ny + RC_T - 1) / RC_T, (nx + RC_T - 1) / RC_T, frames);
  recon_kernel<<<grid, RC_NT, sm, (cudaStream_t)stream>>>(nx, ny, rank, (const float2*)a, (const float2*)b,
                                                          (const float2*)gamma, (float2*)x_out);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}
