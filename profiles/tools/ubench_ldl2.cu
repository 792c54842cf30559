// Isolated timing of the production block_ldl2_solve (tt_block.cuh) with per-step stamps.
#include <cstdio>
#include "../../paper_1609_04104_b200/csrc/tt_block.cuh"
int tt_fail_cuda(cudaError_t, const char*) { return 4; }
int tt_fail(int c, const char*, ...) { return c; }
template <int EPT>
__global__ void k(int R, long long* cyc, double2* out, int reps) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int tid = threadIdx.x, Rp = R * (R + 1) / 2;
  double2* G = (double2*)sm; double2* hin = G + Rp; double2* gam = hin + R; double2* colb = gam + R;
  double* blk = (double*)(colb + 4 * (R + 1)); double2* zf = (double2*)(blk + 4 * (R / 2 + 1));
  long long tot = 0;
  for (int it = 0; it < reps; ++it) {
    for (int e = tid; e < Rp; e += blockDim.x) { int i, j; tri_decode(e, i, j); G[e] = make_double2(i == j ? 10.0 + i : 0.1 / (1 + i + j), i == j ? 0.0 : 0.05); }
    for (int r = tid; r < R; r += blockDim.x) hin[r] = make_double2(1.0 + r, 0.5);
    __syncthreads();
    long long t0 = clock64();
    block_ldl2_solve<EPT>(G, hin, gam, colb, blk, zf, R);
    tot += clock64() - t0;
  }
  if (tid == 0) cyc[0] = tot / reps;
  if (tid < R) out[tid] = gam[tid];
}
int main() {
  long long* c; double2* o; cudaMallocManaged(&c, 64); cudaMallocManaged(&o, 64 * 16);
  for (int R : {10, 20, 32, 64}) {
    size_t sm = 16 * (R * (R + 1) / 2 + 2 * R + 4 * (R + 1) + R) + 8 * 4 * (R / 2 + 1) + 64;
    int E = R * (R + 1) / 2 + R;
    if (E <= 512) { cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); k<2><<<1, 256, sm>>>(R, c, o, 10); }
    else if (E <= 1024) { cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); k<4><<<1, 256, sm>>>(R, c, o, 10); }
    else { cudaFuncSetAttribute(k<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); k<9><<<1, 256, sm>>>(R, c, o, 10); }
    cudaError_t err = cudaDeviceSynchronize();
    printf("err %s R=%d blocked LDL: %lld cycles  gam0=(%.6f,%.6f)\n", cudaGetErrorString(err), R, c[0], o[0].x, o[0].y);
  }
}
