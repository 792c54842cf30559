// Throughput of the legacy warp-level tensor-core MMA on the B200 (sm_100a): mma.sync m16n8k8 TF32 (fp32
// accumulate) and m16n8k16 BF16, 8 independent accumulators per warp, 8 warps per CTA, one CTA per SM.
// Decides whether a split-TF32 reconstruction (X = A diag(gamma) B^T at fp32 accuracy) can beat the fp32
// CUDA cores (~38 TFLOP/s on the GEMM-shaped recon kernel).
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
template <int KIND>
__global__ void k(float* out, long long* cyc) {
  float acc[8][4];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  unsigned a0 = threadIdx.x, a1 = threadIdx.x * 3, a2 = threadIdx.x * 5, a3 = threadIdx.x * 7, b0 = 11, b1 = 13;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+f"(acc[i][0]), "+f"(acc[i][1]), "+f"(acc[i][2]), "+f"(acc[i][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+f"(acc[i][0]), "+f"(acc[i][1]), "+f"(acc[i][2]), "+f"(acc[i][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) s += acc[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* o;
  long long* c;
  cudaMalloc(&o, 148 * 256 * 4);
  cudaMallocManaged(&c, 148 * 8);
  for (int kind = 0; kind < 2; ++kind) {
    if (kind == 0) k<0><<<148, 256>>>(o, c); else k<1><<<148, 256>>>(o, c);
    cudaDeviceSynchronize();
    const double flop_per_mma = kind == 0 ? 2.0 * 16 * 8 * 8 : 2.0 * 16 * 8 * 16;
    const double flops = flop_per_mma * 8 * ITERS * 8;  // 8 warps x ITERS x 8 mma per SM
    const double tf = flops / c[0] * 1.965e9 * 148 / 1e12;
    printf("%s: %lld cycles, %.0f TFLOP/s (148 SMs at 1.965 GHz)\n", kind == 0 ? "mma.sync m16n8k8 tf32" : "mma.sync m16n8k16 bf16",
           c[0], tf);
  }
  return 0;
}
