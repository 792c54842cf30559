// Frame reconstruction X_f = A_f diag(gamma_f) B_f^T, batched over frames.
//
// Reference: core.synthesize_slice (core.py:91-104, einsum over the rank) and
// mri.reconstruct_frame (mri.py:107-121, (A1 * gamma) @ A2.T, plain
// transpose). In run_adaptive it is called once per frame with the
// post-update factors and that frame's gamma (experiment.py:525).
//
// R <= 32 runs on the tensor cores (tt_recon_tc.cu); this CUDA-core form covers R up to 64.
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

int tt_recon_tc(cudaStream_t st, int frames, int nx, int ny, int rank, const float2* a, const float2* b,
                const float2* g, float2* x, int vec);  // tt_recon_tc.cu

extern "C" int tt_reconstruct(void* stream, int frames, int nx, int ny, int rank, const float* a, const float* b,
                              const float* gamma, float* x_out) {
  if (frames < 0 || nx < 1 || ny < 1 || rank < 1 || !a || !b || !gamma || !x_out)
    return tt_fail(TT_EINVAL, "tt_reconstruct: bad arguments");
  if (rank > RC_RMAX) return tt_fail(TT_EUNSUPPORTED, "tt_reconstruct: rank > %d", RC_RMAX);
  if (frames == 0) return TT_OK;
  if (frames > 65535) return tt_fail(TT_EINVAL, "tt_reconstruct: frames > 65535 per call");
  // R <= 32: the tensor-core form (3xTF32 on tcgen05, tt_recon_tc.cu); TT_RECON_FFMA=1 selects the
  // CUDA-core form below at any rank (tests compare the two)
  const char* env = getenv("TT_RECON_FFMA");
  if (rank <= 32 && !(env && env[0] == '1'))
    return tt_recon_tc((cudaStream_t)stream, frames, nx, ny, rank, (const float2*)a, (const float2*)b,
                       (const float2*)gamma, (float2*)x_out, (ny % 2 == 0 && ((size_t)x_out & 15) == 0) ? 1 : 0);
  const size_t sm = sizeof(float2) * 2 * RC_TP * (size_t)rank;
  static size_t cfg[TT_MAXDEV] = {0};
  TT_CUDA_TRY(tt_smem_attr((const void*)recon_kernel, sm, cfg));
  dim3 grid((ny + RC_T - 1) / RC_T, (nx + RC_T - 1) / RC_T, frames);
  recon_kernel<<<grid, RC_NT, sm, (cudaStream_t)stream>>>(nx, ny, rank, (const float2*)a, (const float2*)b,
                                                          (const float2*)gamma, (float2*)x_out);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

// NMSE per frame (metrics.nmse, metrics.py:53-62): ||X_f - Xhat_f||^2 / ||X_f||^2 over complex64 frames,
// fp64 sums. Deterministic: fixed per-block partials ([frames][NB]), then one warp per frame sums them in
// a fixed order. Off the timed path (the bench's and run_online's quality check).
#define NM_NT 256
#define NM_NB 32
__global__ void __launch_bounds__(NM_NT) nmse_part_kernel(size_t n, const float2* __restrict__ truth,
                                                          const float2* __restrict__ est, double2* __restrict__ part) {
  const int f = blockIdx.y;
  const float2* t = truth + (size_t)f * n;
  const float2* e = est + (size_t)f * n;
  double num = 0.0, den = 0.0;
  for (size_t i = (size_t)blockIdx.x * NM_NT + threadIdx.x; i < n; i += (size_t)NM_NB * NM_NT) {
    const float2 a = t[i], b = e[i];
    const double dx = (double)a.x - b.x, dy = (double)a.y - b.y;
    num += dx * dx + dy * dy;
    den += (double)a.x * a.x + (double)a.y * a.y;
  }
  __shared__ double sn[NM_NT / 32], sd[NM_NT / 32];
  num = warp_sum(num);
  den = warp_sum(den);
  if ((threadIdx.x & 31) == 0) {
    sn[threadIdx.x >> 5] = num;
    sd[threadIdx.x >> 5] = den;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < NM_NT / 32; ++w) {
      a += sn[w];
      b += sd[w];
    }
    part[(size_t)f * NM_NB + blockIdx.x] = make_double2(a, b);
  }
}
__global__ void nmse_final_kernel(int frames, const double2* __restrict__ part, double* __restrict__ out) {
  const int f = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (f >= frames) return;
  const double2 v = part[(size_t)f * NM_NB + lane];  // NM_NB == 32: one partial per lane
  const double num = warp_sum(v.x), den = warp_sum(v.y);
  if (lane == 0) out[f] = den > 0.0 ? num / den : __longlong_as_double(0x7ff8000000000000ll);
}

extern "C" int tt_nmse(void* stream, int frames, size_t n, const float* truth, const float* est, double* work,
                       double* out) {
  if (frames < 0 || !truth || !est || !work || !out) return tt_fail(TT_EINVAL, "tt_nmse: bad arguments");
  if (frames == 0) return TT_OK;
  if (frames > 65535) return tt_fail(TT_EINVAL, "tt_nmse: frames > 65535 per call");
  cudaStream_t st = (cudaStream_t)stream;
  nmse_part_kernel<<<dim3(NM_NB, frames), NM_NT, 0, st>>>(n, (const float2*)truth, (const float2*)est, (double2*)work);
  nmse_final_kernel<<<(frames + 7) / 8, 256, 0, st>>>(frames, (const double2*)work, out);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}
extern "C" size_t tt_nmse_work_doubles(int frames) { return (size_t)(frames > 0 ? frames : 0) * NM_NB * 2; }
