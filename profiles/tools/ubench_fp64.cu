// Throughput of DFMA, FFMA and F2F.F64.F32 per SM on the B200 (sm_100a): one CTA per SM, 8 warps,
// 8 independent chains per thread, clock64 around the loop. Decides the fp64-accumulating GEMMs
// of the rows kernel (exact products of fp32 operands).
#include <cstdio>
#include <cuda_runtime.h>
#define N_IT 4096
__global__ void k_dfma(double* out, long long* cyc, double s) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < N_IT; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], s, 1.0);
  __syncthreads();
  long long t1 = clock64();
  double r = 0;
  for (int i = 0; i < 8; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_ffma(float* out, long long* cyc, float s) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < N_IT; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], s, 1.0f);
  __syncthreads();
  long long t1 = clock64();
  float r = 0;
  for (int i = 0; i < 8; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// conversion + DFMA mix: per iteration 2 F2F (fp32 -> fp64) feeding 8 DFMA (a GEMM inner step)
__global__ void k_cvt(double* out, long long* cyc, const float* src) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0;
  float x = src[threadIdx.x], y = src[threadIdx.x + 32];
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < N_IT; ++it) {
    double dx = (double)x, dy = (double)y;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(dx, (i & 1) ? dy : dx, a[i]);
    x += 1.0f;
    y -= 1.0f;
  }
  __syncthreads();
  long long t1 = clock64();
  double r = 0;
  for (int i = 0; i < 8; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* od; float* of; long long* cyc; float* src;
  cudaMalloc(&od, 148 * 1024 * 8); cudaMalloc(&of, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&src, 4096); cudaMemset(src, 0, 4096);
  long long h[148];
  for (int nt : {256, 512, 1024}) {
    k_dfma<<<148, nt>>>(od, cyc, 0.999); cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("threads %4d  DFMA/clk/SM %.1f\n", nt, (double)nt * N_IT * 8 / h[0]);
    k_ffma<<<148, nt>>>(of, cyc, 0.999f); cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("threads %4d  FFMA/clk/SM %.1f\n", nt, (double)nt * N_IT * 8 / h[0]);
    k_cvt<<<148, nt>>>(od, cyc, src); cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("threads %4d  (2 F2F + 8 DFMA) DFMA/clk/SM %.1f\n", nt, (double)nt * N_IT * 8 / h[0]);
  }
  return 0;
}
