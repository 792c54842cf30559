// cgemm_tile vs cgemm_v2 variants at the rows-kernel GEMM shapes
#include <cstdio>
#include "../../paper_1609_04104_b200/csrc/tt_block.cuh"
int tt_fail_cuda(cudaError_t, const char*) { return 4; }
int tt_fail(int c, const char*, ...) { return c; }
struct Shape { const char* name; int M, N, K, a_m, a_k, b_k, b_n; };
template <int V>
__global__ void k(Shape sh, long long* cyc, float* chk, int reps) {
  extern __shared__ __align__(16) unsigned char sm[];
  float2* A = (float2*)sm;
  float2* B = A + 128 * 64;
  float2* red = B + 128 * 64;
  float2* out = red + 2048;
  const int tid = threadIdx.x;
  for (int i = tid; i < 128 * 64; i += blockDim.x) A[i] = make_float2(0.001f * (i % 97), 0.002f * (i % 31));
  for (int i = tid; i < 128 * 64; i += blockDim.x) B[i] = make_float2(0.003f * (i % 13), -0.001f * (i % 7));
  for (int i = tid; i < 128 * 32; i += blockDim.x) out[i] = make_float2(0.f, 0.f);
  __syncthreads();
  long long tot = 0;
  auto o = [&](int m, int n, float2 v) { out[m * sh.N + n] = cadd(out[m * sh.N + n], v); };
  for (int it = 0; it < reps; ++it) {
    __syncthreads();
    long long t0 = clock64();
    if (V == 0) {
      const int ks = gemm_split(sh.M, sh.N, sh.K, 2, 4, 2048);
      cgemm_tile<2, 4, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, ks, red, o);
    } else if (V == 1) cgemm_v2<2, 4, 1, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, o);
    else if (V == 2) cgemm_v2<2, 4, 2, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, o);
    else if (V == 3) cgemm_v2<2, 4, 4, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, o);
    else if (V == 4) cgemm_v2<2, 4, 8, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, o);
    else if (V == 5) cgemm_v2<4, 4, 1, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, o);
    else if (V == 6) cgemm_v2<4, 4, 2, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, o);
    else if (V == 7) cgemm_v2<1, 4, 4, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, o);
    else if (V == 8) cgemm_v2<1, 4, 8, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, o);
    else if (V == 9) cgemm_v2<2, 2, 4, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, o);
    __syncthreads();
    tot += clock64() - t0;
  }
  if (tid == 0) cyc[V] = tot / reps;
  __syncthreads();
  if (tid == 0) { float s = 0; for (int i = 0; i < sh.M * sh.N; ++i) s += out[i].x + 0.5f * out[i].y; chk[V] = s / reps; }
}
template <int V> void run(Shape s, long long* c, float* ch, size_t smem) {
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<V><<<1, 256, smem>>>(s, c, ch, 20);
}
int main() {
  long long* c; float* ch; cudaMallocManaged(&c, 8 * 16); cudaMallocManaged(&ch, 4 * 16);
  Shape shapes[] = {{"C2 W 16x20x64", 16, 20, 64, 1, 16, 20, 1}, {"C2 Z 64x20x16", 64, 20, 16, 16, 1, 20, 1},
                    {"C2 Q 16x20x20", 16, 20, 20, 20, 1, 20, 1}, {"C2 P 4x20x20", 4, 20, 20, 20, 1, 20, 1},
                    {"C3 W 128x16x52", 128, 16, 52, 1, 128, 16, 1}, {"C3 Z 52x16x128", 52, 16, 128, 128, 1, 16, 1},
                    {"C3 Q 128x16x16", 128, 16, 16, 16, 1, 16, 1}, {"C3 P 26x16x16", 26, 16, 16, 16, 1, 16, 1}};
  size_t smem = 8 * (128 * 64 + 128 * 64 + 2048 + 128 * 32);
  const char* vn[] = {"tile", "2x4/1", "2x4/2", "2x4/4", "2x4/8", "4x4/1", "4x4/2", "1x4/4", "1x4/8", "2x2/4"};
  for (auto& s : shapes) {
    run<0>(s, c, ch, smem); run<1>(s, c, ch, smem); run<2>(s, c, ch, smem); run<3>(s, c, ch, smem); run<4>(s, c, ch, smem);
    run<5>(s, c, ch, smem); run<6>(s, c, ch, smem); run<7>(s, c, ch, smem); run<8>(s, c, ch, smem); run<9>(s, c, ch, smem);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%-16s %s |", s.name, cudaGetErrorString(e));
    for (int v = 0; v < 10; ++v) printf(" %s:%lld%s", vn[v], c[v], fabsf(ch[v] - ch[0]) > 1e-3f * fabsf(ch[0]) + 1e-4f ? "(!)" : "");
    printf("\n");
  }
}
