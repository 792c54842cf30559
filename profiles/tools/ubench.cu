#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, double a, double b) {
  __shared__ double sm[1024];
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; idx[i] = (i * 7 + 1) & 1023; }
  __syncthreads();
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);           // dependent DFMA chain
  long long t1 = clock64();
  float xf = (float)a;
  for (int i = 0; i < n; ++i) xf = fmaf(xf, (float)b, (float)a);
  long long t2 = clock64();
  int j = threadIdx.x;
  for (int i = 0; i < n; ++i) j = idx[j];                  // dependent LDS chain
  long long t3 = clock64();
  double r;
  double y = a;
  for (int i = 0; i < n; ++i) { asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y)); y = r + 1.0; }
  long long t4 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) z = 1.0 / (z + 1.0);
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
  out[threadIdx.x] = x + xf + j + y + z;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8192); cudaMallocManaged(&c, 64);
  int n = 1000;
  for (int nt : {32, 256}) {
    k<<<1, nt>>>(o, c, n, 0.5, 0.999); cudaDeviceSynchronize();
    k<<<1, nt>>>(o, c, n, 0.5, 0.999); cudaDeviceSynchronize();
    printf("threads %d: dfma %.1f  ffma %.1f  lds %.1f  rcp64 %.1f  ddiv %.1f  bar %.1f cycles/op\n", nt,
           c[0] / (double)n, c[1] / (double)n, c[2] / (double)n, c[3] / (double)n, c[4] / (double)n, c[5] / (double)n);
  }
  return 0;
}
