// Isolated timing and agreement: Gauss-Jordan with 1 x 1 pivots (block_gj_solve) vs 2 x 2 pivot blocks
// (block_gj2_solve), same Hermitian positive definite system (a Gram-like matrix + lambda I), 256 threads.
// Result (B200): R = 10 / 16 / 20 / 32: 2.9k / 4.7k / 5.8k / 16.5k cycles for block_gj_solve against 4.7k /
// 8.1k / 9.6k / 18.7k for the 2 x 2 form (agreement 1e-13): the 2 x 2 step's dependency chain (determinant,
// reciprocal, the inverse block, the row coefficients) costs more than the barriers it saves.
#include <cmath>
#include <cstdio>
#include "../../paper_1609_04104_b200/csrc/tt_block.cuh"

// the 2 x 2-pivot variant under test (slower than block_gj_solve at R = 10..32: not used by the kernels)
// Gauss-Jordan with 2 x 2 pivot blocks (half the barrier steps of block_gj_solve): at step p the rows
// i outside {p, p+1} take g[i][j] -= (alpha_i, beta_i) . (M[p][j], M[p+1][j]) for j > p + 1 with
// (alpha_i, beta_i) = (M[i][p], M[i][p+1]) P^-1, P the pivot block. A block whose determinant is not
// safely positive (|det| <= 1e-12 |a| |d|, or a non-positive leading pivot) is taken as a 1 x 1 step
// instead (the decision is block-uniform: every thread reads the same pivot entries); a non-positive 1 x 1
// pivot drops its component (gamma_p = 0), as block_gj_solve does. At the end the matrix is block
// diagonal and gamma_block = P_block^-1 rhs_block. Same thread layout and operand caching as
// block_gj_solve. scratch: gj2_scratch_d2(R) double2. Ends with __syncthreads.
__host__ __device__ inline int gj2_scratch_d2(int R) { return 2 * (2 * R + 2 * (R + 1)) + 3 * R + 2; }
template <int EPT>
TT_DEV void block_gj2_solve(const double2* G, const double2* hin, double2* gam, double2* scr, int R) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int W = R + 1;
  const int ng = NT / R, grp = tid / R, i = tid - grp * R;
  const bool live = grp < ng;
  // buffer layout (double2): [c0: R][c1: R][r0: W][r1: W], two buffers; then pinv [2R], rhs [R], pst (ints)
  const int BS = 2 * R + 2 * W;
  double2* pinv = scr + 2 * BS;
  double2* rhs = pinv + 2 * R;
  int* pst = (int*)(rhs + R);
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
      if (j < 2) scr[j * R + i] = g[m];              // pivot columns 0, 1
      if (i < 2) scr[2 * R + i * W + j] = g[m];      // pivot rows 0, 1
    }
  }
  __syncthreads();
  const uint32_t base = smem_addr(scr);
  const uint32_t bstride = 16u * BS;
  const uint32_t oci = 16u * (live ? i : 0);
  int p = 0;
  uint32_t cur = 0u;
  while (p < R) {
    const uint32_t nxt = bstride - cur;
    const uint32_t c0 = base + cur, c1 = c0 + 16u * R, r0 = c0 + 32u * R, r1 = r0 + 16u * W;
    // operands first (independent of the pivot inverse): the pivot block, the row's pivot-column entries,
    // the pivot-row entries of the thread's columns
    const double2 a = lds_d2(r0 + 16u * p);
    const bool has2 = p + 1 < R;
    const double2 b = has2 ? lds_d2(r0 + 16u * (p + 1)) : make_double2(0.0, 0.0);
    const double2 c = has2 ? lds_d2(r1 + 16u * p) : make_double2(0.0, 0.0);
    const double2 d = has2 ? lds_d2(r1 + 16u * (p + 1)) : make_double2(0.0, 0.0);
    const double2 x = lds_d2(c0 + oci);
    const double2 y = lds_d2(c1 + oci);
    double2 v0[EPT], v1[EPT];
#pragma unroll
    for (int m = 0; m < EPT; ++m) {
      const uint32_t o = 16u * (uint32_t)(rj[m] < 0 ? 0 : rj[m]);
      v0[m] = lds_d2(r0 + o);
      v1[m] = lds_d2(r1 + o);
    }
    const double2 det = zsub(zmul(a, d), zmul(b, c));
    const bool two = has2 && a.x > 0.0 && d.x > 0.0 && det.x > 1e-12 * a.x * d.x;
    double2 i00, i01, i10, i11;
    {
      const double ir = fast_rcp(det.x * det.x + det.y * det.y);
      const double2 idet = make_double2(det.x * ir, -det.y * ir);  // 1 / det
      i00 = zmul(d, idet);
      i01 = zmul(make_double2(-b.x, -b.y), idet);
      i10 = zmul(make_double2(-c.x, -c.y), idet);
      i11 = zmul(a, idet);
    }
    const double id1 = a.x > 0.0 ? fast_rcp(a.x) : 0.0;
    const int q = p + (two ? 2 : 1);  // the next pivot start
    const bool prow = i == p || (two && i == p + 1);
    double2 al, be;
    if (two) {
      al = zadd(zmul(x, i00), zmul(y, i10));
      be = zadd(zmul(x, i01), zmul(y, i11));
    } else {
      al = zscale(x, id1);
      be = make_double2(0.0, 0.0);
    }
    if (prow || !live) {
      al = make_double2(0.0, 0.0);
      be = al;
    }
#pragma unroll
    for (int m = 0; m < EPT; ++m) {
      const int j = rj[m];
      if (j >= q) {
        g[m] = zsub(g[m], zadd(zmul(al, v0[m]), zmul(be, v1[m])));
        // publish the next pivot columns / rows
        sts_d2_if(j < q + 2, base + nxt + 16u * ((j - q) * R + i), g[m]);
        sts_d2_if(i == q || i == q + 1, base + nxt + 16u * (2 * R + (i - q) * W + j), g[m]);
      }
    }
    if (tid == 0) {
      if (two) {
        pinv[2 * p] = i00;
        pinv[2 * p + 1] = i01;
        pinv[2 * p + 2] = i10;
        pinv[2 * p + 3] = i11;
        pst[p] = p;
        pst[p + 1] = p;
      } else {
        pinv[2 * p] = make_double2(id1, 0.0);
        pst[p] = -1 - p;  // a 1 x 1 block
      }
    }
    p = q;
    cur = nxt;
    __syncthreads();
  }
#pragma unroll
  for (int m = 0; m < EPT; ++m)
    if (live && rj[m] == R) rhs[i] = g[m];
  __syncthreads();
  if (tid < R) {
    const int st = pst[tid];
    gam[tid] = st < 0 ? zmul(pinv[2 * tid], rhs[tid])
                      : zadd(zmul(pinv[2 * tid], rhs[st]), zmul(pinv[2 * tid + 1], rhs[st + 1]));
  }
  __syncthreads();
}


template <int EPT>
__global__ void k(int R, long long* cyc, double2* out, int reps) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int tid = threadIdx.x, Rp = R * (R + 1) / 2;
  double2* G = (double2*)sm;
  double2* hin = G + Rp;
  double2* gam = hin + R;
  double2* scr = gam + R;
  long long t1 = 0, t2 = 0;
  for (int it = 0; it < reps; ++it) {
    for (int v = 0; v < 2; ++v) {
      for (int e = tid; e < Rp; e += blockDim.x) {
        int i, j;
        tri_decode(e, i, j);
        // a dense HPD matrix: sum of outer products + lambda I
        double2 acc = make_double2(i == j ? 0.05 : 0.0, 0.0);
        for (int s = 0; s < 3 * R; ++s) {
          const double2 xi = make_double2(sin(0.3 * s + i), cos(0.7 * s * (i + 1)));
          const double2 xj = make_double2(sin(0.3 * s + j), cos(0.7 * s * (j + 1)));
          acc = zfma_cj(xj, xi, acc);  // conj(x_j) x_i: row i col j of X^H X
        }
        G[e] = acc;
      }
      for (int r = tid; r < R; r += blockDim.x) hin[r] = make_double2(1.0 + r, 0.5 - 0.1 * r);
      __syncthreads();
      long long t0 = clock64();
      if (v == 0) block_gj_solve<EPT>(G, hin, gam, scr, R);
      else block_gj2_solve<EPT>(G, hin, gam, scr, R);
      long long dt = clock64() - t0;
      if (v == 0) t1 += dt; else t2 += dt;
      if (tid < R) out[v * 64 + tid] = gam[tid];
      __syncthreads();
    }
  }
  if (tid == 0) { cyc[0] = t1 / reps; cyc[1] = t2 / reps; }
}
template <int EPT>
void run(int R, long long* c, double2* o) {
  size_t sm = 16 * (R * (R + 1) / 2 + 2 * R + gj2_scratch_d2(R) + 8 * (R + 1)) + 64;
  cudaFuncSetAttribute(k<EPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<EPT><<<1, 256, sm>>>(R, c, o, 20);
  cudaError_t err = cudaDeviceSynchronize();
  double md = 0, mx = 0;
  for (int r = 0; r < R; ++r) {
    const double dx = o[r].x - o[64 + r].x, dy = o[r].y - o[64 + r].y;
    md = fmax(md, sqrt(dx * dx + dy * dy));
    mx = fmax(mx, sqrt(o[r].x * o[r].x + o[r].y * o[r].y));
  }
  printf("%s R=%2d  gj %6lld cycles   gj2x2 %6lld cycles   max|diff|/max|x| %.3e\n", cudaGetErrorString(err), R, c[0],
         c[1], md / mx);
}
int main() {
  long long* c;
  double2* o;
  cudaMallocManaged(&c, 64);
  cudaMallocManaged(&o, 128 * 16);
  run<1>(10, c, o);
  run<2>(16, c, o);
  run<2>(20, c, o);
  run<5>(32, c, o);
  return 0;
}
