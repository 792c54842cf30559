#include <cstdio>
#include "../../paper_1609_04104_b200/csrc/tt_block.cuh"
int tt_fail_cuda(cudaError_t, const char*) { return 4; }
int tt_fail(int c, const char*, ...) { return c; }
struct Shape { const char* name; int M, N, K, a_m, a_k, b_k, b_n; };

// variant: explicit register double buffering of the operands (next k loaded before the current FMAs)
template <int TM, int TN, bool CA, bool CB, int UNR, typename Out>
TT_DEV void cgemm_pf(int M, int N, int K, const float2* A, int a_m, int a_k, const float2* B, int b_k, int b_n,
                     int KS, float2* red, Out out) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int tn = (N + TN - 1) / TN, tiles = ((M + TM - 1) / TM) * tn;
  const int items = tiles * KS;
  for (int it = tid; it < items; it += NT) {
    const int ks = idiv(it, tiles), tile = it - ks * tiles;
    const int mt = idiv(tile, tn);
    const int m0 = mt * TM, n0 = (tile - mt * tn) * TN;
    const int k0 = idiv(K * ks, KS), k1 = idiv(K * (ks + 1), KS);
    float2 acc[TM][TN];
#pragma unroll
    for (int u = 0; u < TM; ++u)
#pragma unroll
      for (int v = 0; v < TN; ++v) acc[u][v] = make_float2(0.f, 0.f);
    const float2* Ap[TM];
    const float2* Bp[TN];
#pragma unroll
    for (int u = 0; u < TM; ++u) Ap[u] = A + (size_t)min(m0 + u, M - 1) * a_m;
#pragma unroll
    for (int v = 0; v < TN; ++v) Bp[v] = B + (size_t)min(n0 + v, N - 1) * b_n;
    float2 a[TM], b[TN];
    if (k0 < k1) {
#pragma unroll
      for (int u = 0; u < TM; ++u) a[u] = Ap[u][(size_t)k0 * a_k];
#pragma unroll
      for (int v = 0; v < TN; ++v) b[v] = Bp[v][(size_t)k0 * b_k];
    }
#pragma unroll UNR
    for (int k = k0; k < k1; ++k) {
      float2 an[TM], bn[TN];
      const int kn = min(k + 1, k1 - 1);
#pragma unroll
      for (int u = 0; u < TM; ++u) an[u] = Ap[u][(size_t)kn * a_k];
#pragma unroll
      for (int v = 0; v < TN; ++v) bn[v] = Bp[v][(size_t)kn * b_k];
#pragma unroll
      for (int u = 0; u < TM; ++u) {
        if (CA) a[u].y = -a[u].y;
      }
#pragma unroll
      for (int v = 0; v < TN; ++v) {
        if (CB) b[v].y = -b[v].y;
      }
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; ++v) acc[u][v] = cfma(a[u], b[v], acc[u][v]);
#pragma unroll
      for (int u = 0; u < TM; ++u) a[u] = an[u];
#pragma unroll
      for (int v = 0; v < TN; ++v) b[v] = bn[v];
    }
#pragma unroll
    for (int u = 0; u < TM; ++u)
#pragma unroll
      for (int v = 0; v < TN; ++v) {
        const int m = m0 + u, n = n0 + v;
        if (m < M && n < N) {
          if (KS == 1) out(m, n, acc[u][v]);
          else red[((size_t)ks * M + m) * N + n] = acc[u][v];
        }
      }
  }
  if (KS > 1) {
    __syncthreads();
    for (int o = tid; o < M * N; o += NT) {
      float2 s = red[o];
#pragma unroll
      for (int ks = 1; ks < 8; ++ks)
        if (ks < KS) s = cadd(s, red[(size_t)ks * M * N + o]);
      const int om = idiv(o, N);
      out(om, o - om * N, s);
    }
  }
}

template <int V>
__global__ void k(Shape sh, long long* cyc, float* chk, int reps) {
  extern __shared__ __align__(16) unsigned char sm[];
  float2* A = (float2*)sm; float2* B = A + 128 * 64; float2* red = B + 128 * 64; float2* out = red + 4096;
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
    if (V == 0) { const int ks = gemm_split(sh.M, sh.N, sh.K, 2, 4, 2048);
      cgemm_tile<2, 4, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, ks, red, o); }
    if (V == 1) { const int ks = gemm_split(sh.M, sh.N, sh.K, 2, 4, 2048);
      cgemm_pf<2, 4, false, true, 1>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, ks, red, o); }
    if (V == 2) { const int ks = gemm_split(sh.M, sh.N, sh.K, 2, 4, 2048);
      cgemm_pf<2, 4, false, true, 2>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, ks, red, o); }
    if (V == 3) { const int ks = gemm_split(sh.M, sh.N, sh.K, 4, 4, 4096);
      cgemm_tile<4, 4, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, ks, red, o); }
    if (V == 4) { const int ks = gemm_split(sh.M, sh.N, sh.K, 4, 4, 4096);
      cgemm_pf<4, 4, false, true, 1>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, ks, red, o); }
    if (V == 5) { const int ks = gemm_split(sh.M, sh.N, sh.K, 2, 4, 4096);
      cgemm_tile<2, 4, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, ks, red, o); }
    if (V == 6) { const int ks = gemm_split(sh.M, sh.N, sh.K, 4, 2, 4096);
      cgemm_tile<4, 2, false, true>(sh.M, sh.N, sh.K, A, sh.a_m, sh.a_k, B, sh.b_k, sh.b_n, ks, red, o); }
    __syncthreads();
    tot += clock64() - t0;
  }
  if (tid == 0) { cyc[V] = tot / reps; float s = 0; for (int i = 0; i < sh.M * sh.N; ++i) s += out[i].x + 0.5f * out[i].y; chk[V] = s / reps; }
}
template <int V> void run(Shape s, long long* c, float* ch, size_t smem) {
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<V><<<1, 256, smem>>>(s, c, ch, 20);
}
int main() {
  long long* c; float* ch; cudaMallocManaged(&c, 8 * 16); cudaMallocManaged(&ch, 4 * 16);
  Shape shapes[] = {{"C2 W 16x20x64", 16, 20, 64, 1, 16, 20, 1}, {"C2 Z 64x20x16", 64, 20, 16, 16, 1, 20, 1},
                    {"C2 Q 16x20x20", 16, 20, 20, 20, 1, 20, 1}, {"C3 W 128x16x52", 128, 16, 52, 1, 128, 16, 1},
                    {"C3 Z 52x16x128", 52, 16, 128, 128, 1, 16, 1}, {"C3 Q 128x16x16", 128, 16, 16, 16, 1, 16, 1},
                    {"C4 W 64x32x128", 64, 32, 128, 1, 64, 32, 1}, {"C4 Z 128x32x64", 128, 32, 64, 64, 1, 32, 1},
                    {"C4 Q 64x32x32", 64, 32, 32, 32, 1, 32, 1}};
  size_t smem = 8 * (128 * 64 + 128 * 64 + 4096 + 128 * 32);
  const char* vn[] = {"tile2x4", "pf2x4/1", "pf2x4/2", "tile4x4", "pf4x4", "tile2x4cap4k", "tile4x2"};
  for (auto& s : shapes) {
    run<0>(s, c, ch, smem); run<1>(s, c, ch, smem); run<2>(s, c, ch, smem); run<3>(s, c, ch, smem); run<4>(s, c, ch, smem); run<5>(s, c, ch, smem); run<6>(s, c, ch, smem);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%-16s %s |", s.name, cudaGetErrorString(e));
    for (int v = 0; v < 7; ++v) printf(" %s:%lld%s", vn[v], c[v], fabsf(ch[v] - ch[0]) > 1e-3f * fabsf(ch[0]) + 1e-4f ? "(!)" : "");
    printf("\n");
  }
  return 0;
}
