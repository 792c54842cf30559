// Dependent fp64 add chain latency (one thread), the cost model of the large-domain draw's exact
// fallback (numpy's sequential cumsum). nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
__global__ void chain(const double* p, double* out, long long* cyc, int n) {
  double c = 0.0, v0 = p[0], v1 = p[1], v2 = p[2], v3 = p[3];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    c += v0; c += v1; c += v2; c += v3;
  }
  long long t1 = clock64();
  out[0] = c;
  cyc[0] = t1 - t0;
}
__global__ void chain_f(const float* p, float* out, long long* cyc, int n) {
  float c = 0.f, v0 = p[0], v1 = p[1], v2 = p[2], v3 = p[3];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    c += v0; c += v1; c += v2; c += v3;
  }
  long long t1 = clock64();
  out[0] = c;
  cyc[0] = t1 - t0;
}
int main() {
  double *p, *o; float *pf, *of; long long* cy;
  cudaMalloc(&p, 64); cudaMalloc(&o, 64); cudaMalloc(&pf, 64); cudaMalloc(&of, 64); cudaMalloc(&cy, 8);
  cudaMemset(p, 0, 64); cudaMemset(pf, 0, 64);
  const int n = 1 << 16;
  long long c;
  for (int r = 0; r < 2; ++r) {
    chain<<<1, 1>>>(p, o, cy, n); cudaMemcpy(&c, cy, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent: %.2f cycles\n", (double)c / (4.0 * n));
    chain_f<<<1, 1>>>(pf, of, cy, n); cudaMemcpy(&c, cy, 8, cudaMemcpyDeviceToHost);
    printf("FADD dependent: %.2f cycles\n", (double)c / (4.0 * n));
  }
  return 0;
}
