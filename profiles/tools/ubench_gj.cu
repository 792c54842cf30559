// Isolated timing: Gauss-Jordan (block_gj_solve) vs 2x2-blocked LDL^H (block_ldl2_solve), same system.
#include <cstdio>
#include "../../paper_1609_04104_b200/csrc/tt_block.cuh"
int tt_fail_cuda(cudaError_t, const char*) { return 4; }
int tt_fail(int c, const char*, ...) { return c; }
template <int EPT, int EPG>
__global__ void k(int R, long long* cyc, double2* out, int reps) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int tid = threadIdx.x, Rp = R * (R + 1) / 2;
  double2* G = (double2*)sm; double2* hin = G + Rp; double2* gam = hin + R; double2* colb = gam + R;
  double* blk = (double*)(colb + 4 * (R + 1)); double2* zf = (double2*)(blk + 4 * (R / 2 + 1));
  long long tl = 0, tg = 0;
  for (int it = 0; it < reps; ++it) {
    for (int v = 0; v < 2; ++v) {
      for (int e = tid; e < Rp; e += blockDim.x) { int i, j; tri_decode(e, i, j); G[e] = make_double2(i == j ? 10.0 + i : 0.1 / (1 + i + j), i == j ? 0.0 : 0.05 * ((i * 7 + j) % 5 - 2)); }
      for (int r = tid; r < R; r += blockDim.x) hin[r] = make_double2(1.0 + r, 0.5 - 0.1 * r);
      __syncthreads();
      long long t0 = clock64();
      if (v == 0) block_ldl2_solve<EPT>(G, hin, gam, colb, blk, zf, R);
      else block_gj_solve<EPG>(G, hin, gam, colb, R);
      long long dt = clock64() - t0;
      if (v == 0) tl += dt; else tg += dt;
      if (tid < R) out[v * 64 + tid] = gam[tid];
      __syncthreads();
    }
  }
  if (tid == 0) { cyc[0] = tl / reps; cyc[1] = tg / reps; }
}
template <int EPT, int EPG>
void run(int R, long long* c, double2* o) {
  size_t sm = 16 * (R * (R + 1) / 2 + 2 * R + 4 * (R + 1) + R) + 8 * 4 * (R / 2 + 1) + 64;
  cudaFuncSetAttribute(k<EPT, EPG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<EPT, EPG><<<1, 256, sm>>>(R, c, o, 20);
  cudaError_t err = cudaDeviceSynchronize();
  double md = 0, mx = 0;
  for (int r = 0; r < R; ++r) {
    double dx = o[r].x - o[64 + r].x, dy = o[r].y - o[64 + r].y;
    md = fmax(md, sqrt(dx * dx + dy * dy)); mx = fmax(mx, sqrt(o[r].x * o[r].x + o[r].y * o[r].y));
  }
  printf("x0 ldl (%.9f,%.9f) gj (%.9f,%.9f)\n", o[0].x, o[0].y, o[64].x, o[64].y);
  printf("%s R=%d  ldl2 %lld cyc   gj %lld cyc   max|diff|/max|x| %.3e\n", cudaGetErrorString(err), R, c[0], c[1], md / mx);
}
int main() {
  long long* c; double2* o; cudaMallocManaged(&c, 64); cudaMallocManaged(&o, 128 * 16);
  run<2, 1>(10, c, o);
  run<2, 2>(16, c, o);
  run<2, 2>(20, c, o);
  run<4, 5>(32, c, o);
  run<9, 17>(64, c, o);
}
