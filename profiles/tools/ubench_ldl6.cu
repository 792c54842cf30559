#include <cstdio>
#include "../../paper_1609_04104_b200/csrc/tt_block.cuh"
#include "ldl_reg.cuh"
int tt_fail_cuda(cudaError_t, const char*) { return 4; }
int tt_fail(int c, const char*, ...) { return c; }
template <int EPT>
__global__ void k(int R, long long* cyc, double2* out, int reps) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int tid = threadIdx.x, Rp = R * (R + 1) / 2;
  double2* Gin = (double2*)sm; double2* Gout = Gin + Rp; double2* hin = Gout + Rp; double2* hv = hin + R; double2* gam = hv + R;
  double2* colb = gam + R; double* invb = (double*)(colb + 2 * (R + 1));  // [2 + R]
  long long tot = 0;
  for (int it = 0; it < reps; ++it) {
    for (int e = tid; e < Rp; e += blockDim.x) { int i, j; tri_decode(e, i, j); Gin[e] = make_double2(i == j ? 10.0 + i : 0.1 / (1 + i + j), i == j ? 0.0 : 0.05); }
    for (int r = threadIdx.x; r < R; r += blockDim.x) hin[r] = make_double2(1.0 + r, 0.5);
    __syncthreads();
    long long t0 = clock64();
    ldl_reg_solve<EPT>(Gin, hin, Gout, hv, colb, invb, gam, R);
    long long t1 = clock64();
    tot += t1 - t0;
    if (tid == 0 && it == reps - 1) { cyc[1] = g_t_fwd - t0; cyc[2] = t1 - g_t_fwd; }
  }
  if (tid == 0) cyc[0] = tot / reps;
  if (tid < R) out[tid] = gam[tid];
}
int main() {
  long long* c; double2* o; cudaMallocManaged(&c, 64); cudaMallocManaged(&o, 64 * 16);
  for (int NTH : {256, 128}) for (int R : {20, 32}) {
    size_t sm = 16 * (R * (R + 1)) + 16 * 3 * R + 16 * 2 * (R + 1) + 8 * (R + 2) + 64;
    int E = R * (R + 1) / 2 + R;
    if (E <= 2 * NTH && NTH == 256) { cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); k<2><<<1, NTH, sm>>>(R, c, o, 10); }
    else if (E <= 5 * NTH) { cudaFuncSetAttribute(k<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); k<5><<<1, NTH, sm>>>(R, c, o, 10); }
    else { cudaFuncSetAttribute(k<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); k<9><<<1, NTH, sm>>>(R, c, o, 10); }
    printf("err %s ", cudaGetErrorString(cudaDeviceSynchronize()));
    printf("NT %d fwd %lld back %lld  R=%d reg LDL: %lld cycles/solve  gam0=(%g,%g) gamR-1=(%g,%g)\n", NTH, c[1], c[2], R, c[0], o[0].x, o[0].y, o[R-1].x, o[R-1].y);
  }
}
