// Isolated timing: Gauss-Jordan with 1x1 pivots (block_gj_solve) vs 2x2 block pivots (gj2, one
// barrier per pivot pair), same Hermitian positive definite system. nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -I include
#include <cstdio>
#include "../../paper_1609_04104_b200/csrc/tt_block.cuh"
int tt_fail_cuda(cudaError_t, const char*) { return 4; }
int tt_fail(int c, const char*, ...) { return c; }

// scratch: 2 buffers x [colA W | colB W | rowA W | rowB W] double2 (8 W)
template <int EPT>
__device__ void gj2(const double2* G, const double2* hin, double2* gam, double2* sc, int R) {
  const int tid = threadIdx.x, NT = blockDim.x, W = R + 1;
  const int ng = NT / R, grp = tid / R, i = tid - grp * R;
  const bool live = grp < ng;
  int rj[EPT];
  double2 g[EPT];
#pragma unroll
  for (int m = 0; m < EPT; ++m) {
    const int j = grp + m * ng;
    rj[m] = -1;
    g[m] = make_double2(0.0, 0.0);
    if (live && j < W) {
      rj[m] = j;
      if (j == R) g[m] = hin[i];
      else if (i >= j) g[m] = G[i * (i + 1) / 2 + j];
      else g[m] = zconj(G[j * (j + 1) / 2 + i]);
      if (j == 0) sc[i] = g[m];                 // colA
      else if (j == 1) sc[W + i] = g[m];        // colB
      if (i == 0) sc[2 * W + j] = g[m];         // rowA
      else if (i == 1) sc[3 * W + j] = g[m];    // rowB
    }
  }
  __syncthreads();
  const uint32_t base = smem_addr(sc);
  const uint32_t bstride = 64u * W;  // one buffer = 4 W double2
  for (int k = 0, b = 0; k < R; k += 2, b ^= 1) {
    const uint32_t cur = base + (b ? bstride : 0u), nxt = base + (b ? 0u : bstride);
    const bool two = k + 1 < R;
    const double2 c0 = lds_d2(cur + 16u * i), c1 = lds_d2(cur + 16u * (W + i));
    double2 r0[EPT], r1[EPT];
#pragma unroll
    for (int m = 0; m < EPT; ++m) {
      const int j = rj[m] < 0 ? 0 : rj[m];
      r0[m] = lds_d2(cur + 16u * (2 * W + j));
      r1[m] = lds_d2(cur + 16u * (3 * W + j));
    }
    const double p00 = lds_d(cur + 16u * (2 * W + k));
    double2 p01 = lds_d2(cur + 16u * (2 * W + k + 1));
    double p11 = lds_d(cur + 16u * (3 * W + k + 1));
    if (!two) { p01 = make_double2(0.0, 0.0); p11 = 1.0; }
    const double det = fma(p00, p11, -(p01.x * p01.x + p01.y * p01.y));
    const double id = det > 0.0 ? fast_rcp(det) : 0.0;
    const double q00 = p11 * id, q11 = p00 * id;
    const double2 q01 = make_double2(-p01.x * id, -p01.y * id), q10 = make_double2(-p01.x * id, p01.y * id);
    const bool piv0 = i == k, piv1 = two && i == k + 1, piv = piv0 || piv1;
    const double2 c1e = two ? c1 : make_double2(0.0, 0.0);
    // other rows: f = -[c0 c1] Pinv (accumulated onto g); pivot rows: f = Pinv row, g replaced
    double2 f0 = zadd(zscale(c0, q00), zmul(c1e, q10));
    double2 f1 = zadd(zmul(c0, q01), zscale(c1e, q11));
    f0 = piv0 ? make_double2(q00, 0.0) : (piv1 ? q10 : make_double2(-f0.x, -f0.y));
    f1 = piv0 ? q01 : (piv1 ? make_double2(q11, 0.0) : make_double2(-f1.x, -f1.y));
#pragma unroll
    for (int m = 0; m < EPT; ++m) {
      const int j = rj[m];
      const bool act = j > k + (two ? 1 : 0);
      const double2 base_g = piv ? make_double2(0.0, 0.0) : g[m];
      const double2 v = zfma(f1, r1[m], zfma(f0, r0[m], base_g));
      if (act) g[m] = v;
      const bool c2 = act && j == k + 2, c3 = act && j == k + 3;
      sts_d2_if(c2, nxt + 16u * i, v);
      sts_d2_if(c3, nxt + 16u * (W + i), v);
      sts_d2_if(act && i == k + 2, nxt + 16u * (2 * W + j), v);
      sts_d2_if(act && i == k + 3, nxt + 16u * (3 * W + j), v);
    }
    __syncthreads();
  }
#pragma unroll
  for (int m = 0; m < EPT; ++m)
    if (live && rj[m] == R) gam[i] = g[m];
  __syncthreads();
}

template <int EPT, int EPG>
__global__ void kb(int R, long long* cyc, double2* out, int reps) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int tid = threadIdx.x, Rp = R * (R + 1) / 2;
  double2* G = (double2*)sm; double2* hin = G + Rp; double2* gam = hin + R; double2* sc = gam + R;
  long long t1 = 0, t2 = 0;
  for (int it = 0; it < reps; ++it) {
    for (int v = 0; v < 2; ++v) {
      for (int e = tid; e < Rp; e += blockDim.x) { int i, j; tri_decode(e, i, j); G[e] = make_double2(i == j ? 10.0 + i : 0.1 / (1 + i + j), i == j ? 0.0 : 0.05 * ((i * 7 + j) % 5 - 2)); }
      for (int r = tid; r < R; r += blockDim.x) hin[r] = make_double2(1.0 + r, 0.5 - 0.1 * r);
      __syncthreads();
      long long t0 = clock64();
      if (v == 0) block_gj_solve<EPG>(G, hin, gam, sc, R);
      else gj2<EPT>(G, hin, gam, sc, R);
      long long dt = clock64() - t0;
      if (v == 0) t1 += dt; else t2 += dt;
      if (tid < R) out[v * 64 + tid] = gam[tid];
      __syncthreads();
    }
  }
  if (tid == 0) { cyc[0] = t1 / reps; cyc[1] = t2 / reps; }
}
template <int EPT, int EPG>
void run(int R, long long* c, double2* o) {
  size_t sm = 16 * (R * (R + 1) / 2 + 2 * R + 8 * (R + 1)) + 64;
  cudaFuncSetAttribute(kb<EPT, EPG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  kb<EPT, EPG><<<1, 256, sm>>>(R, c, o, 20);
  cudaError_t err = cudaDeviceSynchronize();
  double md = 0, mx = 0;
  for (int r = 0; r < R; ++r) {
    double dx = o[r].x - o[64 + r].x, dy = o[r].y - o[64 + r].y;
    md = fmax(md, sqrt(dx * dx + dy * dy)); mx = fmax(mx, sqrt(o[r].x * o[r].x + o[r].y * o[r].y));
  }
  printf("%s R=%d  gj %lld cyc   gj2 %lld cyc   max|diff|/max|x| %.3e\n", cudaGetErrorString(err), R, c[0], c[1], md / mx);
}
int main() {
  long long* c; double2* o; cudaMallocManaged(&c, 64); cudaMallocManaged(&o, 128 * 16);
  run<1, 1>(10, c, o);
  run<1, 1>(11, c, o);
  run<2, 2>(16, c, o);
  run<2, 2>(20, c, o);
  run<5, 5>(32, c, o);
}
