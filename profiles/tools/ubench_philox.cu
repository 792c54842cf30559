#include <cstdio>
#include "../../paper_1609_04104_b200/csrc/tt_block.cuh"
int tt_fail_cuda(cudaError_t, const char*) { return 4; }
int tt_fail(int c, const char*, ...) { return c; }
__global__ void k(long long* cyc, double* out, int n) {
  __shared__ double cdf[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) cdf[i] = (i + 1) / 256.0;
  __syncthreads();
  uint64_t pos = threadIdx.x;
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double u = philox_uniform(7, 3, pos + (uint64_t)(acc > 10.0)); acc += u; pos += 32; }
  long long t1 = clock64();
  int idx = 0;
  for (int i = 0; i < n; ++i) { idx = upper_bound_d(cdf, 256, (idx & 255) / 256.0 + 0.001); }
  long long t2 = clock64();
  double w = 1.0;
  for (int i = 0; i < n; ++i) { w = warp_sum(w) * 0.03125; }
  long long t3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
  out[threadIdx.x] = acc + idx + w;
}
int main() {
  long long* c; double* o; cudaMallocManaged(&c, 64); cudaMallocManaged(&o, 8192);
  int n = 100;
  for (int nt : {32, 256}) {
    k<<<1, nt>>>(c, o, n); cudaDeviceSynchronize(); k<<<1, nt>>>(c, o, n); cudaDeviceSynchronize();
    printf("threads %d: philox %.0f  upper_bound(256) %.0f  warp_sum(double) %.0f cycles\n", nt, c[0] / (double)n, c[1] / (double)n, c[2] / (double)n);
  }
}
