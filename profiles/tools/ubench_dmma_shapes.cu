// zgemm_dmma (tt_block.cuh) and four variants in isolation at the mirrored rows kernel's call shapes
// (config 3: R = 16, S = 42, nJ = 128; config 2: R = 20, S = 48, nJ = 16): one CTA of 256 threads per SM,
// operands in shared memory with the kernel's padded strides, clock64 per call (median of 20 calls).
#include <algorithm>
#include <cstdio>
#include <vector>
#include "../../paper_1609_04104_b200/csrc/tt_block.cuh"


// P: the operand loads of step t + 1 issued before the DMMAs of step t (register double buffer), balanced M groups
TT_DEV void dmma_m8n8k4_nv(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
template <int G, typename AT, typename Out>
TT_DEV void zgemm_dmma_p(int M, int R, int K, const AT* A, int a_m, int a_k, const double2* B, int b_k, int KS,
                         Out out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int row = lane >> 2, kq = lane & 3;
  const int MB = (M + 7) >> 3, NB = (R + 3) >> 2, MG = (MB + G - 1) / G;
  const int kpairs = (K + 3) >> 2;
  const int items = MG * NB * KS;
  for (int it = warp; it < items; it += nw) {
    const int ks = idiv(it, MG * NB), rest = it - ks * MG * NB;
    const int mg = idiv(rest, NB), nb = rest - mg * NB;
    const int gb0 = idiv(MB * mg, MG), gcount = idiv(MB * (mg + 1), MG) - gb0;
    const int t0 = idiv(kpairs * ks, KS), t1 = idiv(kpairs * (ks + 1), KS);
    const int rb = nb * 4 + (row >> 1), q = row & 1;
    const bool rok = rb < R;
    const AT* ap[G];
    bool mok[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int m = ((gb0 + g) << 3) + row;
      mok[g] = g < gcount && m < M;
      ap[g] = A + (size_t)min(m, M - 1) * a_m;
    }
    double acc[G][2];
#pragma unroll
    for (int g = 0; g < G; ++g) acc[g][0] = acc[g][1] = 0.0;
    const double2* bp = B + min(rb, R - 1);
    if (t0 < t1) {
      AT an[G];
      double2 bn;
      {
        const int kc = min(4 * t0 + kq, K - 1);
        bn = bp[(size_t)kc * b_k];
#pragma unroll
        for (int g = 0; g < G; ++g) an[g] = ap[g][(size_t)kc * a_k];
      }
      for (int t = t0; t < t1; ++t) {
        AT ac[G];
#pragma unroll
        for (int g = 0; g < G; ++g) ac[g] = an[g];
        const double2 braw = bn;
        if (t + 1 < t1) {
          const int kc = min(4 * (t + 1) + kq, K - 1);
          bn = bp[(size_t)kc * b_k];
#pragma unroll
          for (int g = 0; g < G; ++g) an[g] = ap[g][(size_t)kc * a_k];
        }
        const bool kok = 4 * t + kq < K;
        const bool bv = kok && rok;
        const double bx = bv ? braw.x : 0.0, by = bv ? braw.y : 0.0;
        const double b0 = q == 0 ? bx : -by, b1 = q == 0 ? by : bx;
        double ar[G], ai[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const bool av = kok && mok[g];
          ar[g] = av ? (double)ac[g].x : 0.0;
          ai[g] = av ? (double)ac[g].y : 0.0;
        }
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (g < gcount) dmma_m8n8k4_nv(acc[g][0], acc[g][1], ar[g], b0);
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (g < gcount) dmma_m8n8k4_nv(acc[g][0], acc[g][1], ai[g], b1);
      }
    }
    const int r = nb * 4 + kq;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int m = ((gb0 + g) << 3) + row;
      if (g < gcount && m < M && r < R) out(m, r, ks, make_double2(acc[g][0], acc[g][1]));
    }
  }
}

// ---- variants under test
// U: zgemm_dmma with the k loop unrolled by UNR (the compiler pipelines the loads of the unrolled steps)
template <int G, int UNR, typename AT, typename Out>
TT_DEV void zgemm_dmma_u(int M, int R, int K, const AT* A, int a_m, int a_k, const double2* B, int b_k, int KS,
                         Out out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int row = lane >> 2, kq = lane & 3;
  const int MB = (M + 7) >> 3, NB = (R + 3) >> 2, MG = (MB + G - 1) / G;
  const int kpairs = (K + 3) >> 2;
  const int items = MG * NB * KS;
  for (int it = warp; it < items; it += nw) {
    const int ks = idiv(it, MG * NB), rest = it - ks * MG * NB;
    const int mg = idiv(rest, NB), nb = rest - mg * NB;
    const int gb0 = idiv(MB * mg, MG), gcount = idiv(MB * (mg + 1), MG) - gb0;
    const int t0 = idiv(kpairs * ks, KS), t1 = idiv(kpairs * (ks + 1), KS);
    const int rb = nb * 4 + (row >> 1), q = row & 1;
    const bool rok = rb < R;
    const AT* ap[G];
    bool mok[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int m = ((gb0 + g) << 3) + row;
      mok[g] = g < gcount && m < M;
      ap[g] = A + (size_t)min(m, M - 1) * a_m;
    }
    double acc[G][2];
#pragma unroll
    for (int g = 0; g < G; ++g) acc[g][0] = acc[g][1] = 0.0;
    const double2* bp = B + min(rb, R - 1);
#pragma unroll UNR
    for (int t = t0; t < t1; ++t) {
      const int k = 4 * t + kq;
      const bool kok = k < K;
      const int kc = min(k, K - 1);
      const double2 braw = bp[(size_t)kc * b_k];
      const bool bv = kok && rok;
      const double bx = bv ? braw.x : 0.0, by = bv ? braw.y : 0.0;
      const double b0 = q == 0 ? bx : -by, b1 = q == 0 ? by : bx;
      double ar[G], ai[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const AT a = ap[g][(size_t)kc * a_k];
        const bool av = kok && mok[g];
        ar[g] = av ? (double)a.x : 0.0;
        ai[g] = av ? (double)a.y : 0.0;
      }
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (g < gcount) dmma_m8n8k4_nv(acc[g][0], acc[g][1], ar[g], b0);
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (g < gcount) dmma_m8n8k4_nv(acc[g][0], acc[g][1], ai[g], b1);
    }
    const int r = nb * 4 + kq;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int m = ((gb0 + g) << 3) + row;
      if (g < gcount && m < M && r < R) out(m, r, ks, make_double2(acc[g][0], acc[g][1]));
    }
  }
}
// I: K interleaved (k' = 2k + p: one scalar A component and one B component per lane per DMMA), unrolled
template <int G, int UNR, typename AT, typename Out>
TT_DEV void zgemm_dmma_i(int M, int R, int K, const AT* A, int a_m, int a_k, const double2* B, int b_k, int KS,
                         Out out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int row = lane >> 2, kq = lane & 3;
  const int MB = (M + 7) >> 3, NB = (R + 3) >> 2, MG = (MB + G - 1) / G;
  const int ksteps = (2 * K + 3) >> 2;  // steps of 4 interleaved k'
  const int items = MG * NB * KS;
  typedef decltype(A->x) ET;
  for (int it = warp; it < items; it += nw) {
    const int ks = idiv(it, MG * NB), rest = it - ks * MG * NB;
    const int mg = idiv(rest, NB), nb = rest - mg * NB;
    const int gb0 = idiv(MB * mg, MG), gcount = idiv(MB * (mg + 1), MG) - gb0;
    const int t0 = idiv(ksteps * ks, KS), t1 = idiv(ksteps * (ks + 1), KS);
    const int n = nb * 8 + row, rb = n >> 1, q = n & 1;  // B fragment column n' = 2 rb + q
    const bool rok = rb < R;
    const ET* ap[G];
    bool mok[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int m = ((gb0 + g) << 3) + row;
      mok[g] = g < gcount && m < M;
      ap[g] = (const ET*)(A + (size_t)min(m, M - 1) * a_m);
    }
    double acc[G][2];
#pragma unroll
    for (int g = 0; g < G; ++g) acc[g][0] = acc[g][1] = 0.0;
    const double* bp = (const double*)(B + min(rb, R - 1));
#pragma unroll UNR
    for (int t = t0; t < t1; ++t) {
      const int kk = 4 * t + kq, k = kk >> 1, p = kk & 1;
      const bool kok = k < K;
      const int kc = min(k, K - 1);
      // B'[2k + p][2 rb + q] of conj(B): p == q -> B.x, else B.y, negated for (p, q) = (0, 1)
      const double bvv = bp[(size_t)kc * 2 * b_k + (p == q ? 0 : 1)];
      const double bf = (kok && rok) ? ((p == 0 && q == 1) ? -bvv : bvv) : 0.0;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const ET a = ap[g][(size_t)kc * 2 * a_k + p];
        const double af = (kok && mok[g]) ? (double)a : 0.0;
        if (g < gcount) dmma_m8n8k4_nv(acc[g][0], acc[g][1], af, bf);
      }
    }
    const int r = nb * 4 + kq;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int m = ((gb0 + g) << 3) + row;
      if (g < gcount && m < M && r < R) out(m, r, ks, make_double2(acc[g][0], acc[g][1]));
    }
  }
}

struct Sink {
  double2* acc;
  int R;
  TT_DEV void operator()(int m, int n, int ks, double2 v) const { acc[((ks * 64 + m) * R + n) & 4095] = v; }
};

// WHICH: 0 Z (A = Y rows, fp32), 1 W (A = Y^T, fp32), 2 GB (A = Bh^T, fp64), 3 Q (A = Bh rows, fp64)
template <int WHICH, int PIPE, int G>
__global__ void __launch_bounds__(256, 1) kb(int S, int NJ, int R, int RS, int YSR, int KS, long long* cyc, double2* sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  float2* ys = (float2*)sm;
  double2* b64 = (double2*)(ys + 64 * YSR);
  double2* out = b64 + 128 * RS;
  for (int o = threadIdx.x; o < 64 * YSR; o += 256) ys[o] = make_float2(o * 1e-3f, -o * 2e-3f);
  for (int o = threadIdx.x; o < 128 * RS; o += 256) b64[o] = make_double2(o * 1e-3, o * 3e-3);
  __syncthreads();
  Sink snk{out, R};
  for (int rep = 0; rep < 21; ++rep) {
    __syncthreads();
    long long t0 = clock64();
    if (WHICH == 0) {
if (PIPE == 0) zgemm_dmma_v1<G>(S, R, NJ, ys, YSR, 1, b64, RS, KS, snk); else if (PIPE == 1) zgemm_dmma_p<G>(S, R, NJ, ys, YSR, 1, b64, RS, KS, snk); else if (PIPE == 2) zgemm_dmma_u<G, 4>(S, R, NJ, ys, YSR, 1, b64, RS, KS, snk); else if (PIPE == 5) zgemm_dmma<G>(S, R, NJ, ys, YSR, 1, b64, RS, KS, snk); else if (PIPE == 3) zgemm_dmma_i<G, 4>(S, R, NJ, ys, YSR, 1, b64, RS, KS, snk); else zgemm_dmma_i<G, 8>(S, R, NJ, ys, YSR, 1, b64, RS, KS, snk);
    } else if (WHICH == 1) {
if (PIPE == 0) zgemm_dmma_v1<G>(NJ, R, S, ys, 1, YSR, b64, RS, KS, snk); else if (PIPE == 1) zgemm_dmma_p<G>(NJ, R, S, ys, 1, YSR, b64, RS, KS, snk); else if (PIPE == 2) zgemm_dmma_u<G, 4>(NJ, R, S, ys, 1, YSR, b64, RS, KS, snk); else if (PIPE == 5) zgemm_dmma<G>(NJ, R, S, ys, 1, YSR, b64, RS, KS, snk); else if (PIPE == 3) zgemm_dmma_i<G, 4>(NJ, R, S, ys, 1, YSR, b64, RS, KS, snk); else zgemm_dmma_i<G, 8>(NJ, R, S, ys, 1, YSR, b64, RS, KS, snk);
    } else if (WHICH == 2) {
if (PIPE == 0) zgemm_dmma_v1<G>(R, R, NJ, b64, 1, RS, b64, RS, KS, snk); else if (PIPE == 1) zgemm_dmma_p<G>(R, R, NJ, b64, 1, RS, b64, RS, KS, snk); else if (PIPE == 2) zgemm_dmma_u<G, 4>(R, R, NJ, b64, 1, RS, b64, RS, KS, snk); else if (PIPE == 5) zgemm_dmma<G>(R, R, NJ, b64, 1, RS, b64, RS, KS, snk); else if (PIPE == 3) zgemm_dmma_i<G, 4>(R, R, NJ, b64, 1, RS, b64, RS, KS, snk); else zgemm_dmma_i<G, 8>(R, R, NJ, b64, 1, RS, b64, RS, KS, snk);
    } else {
if (PIPE == 0) zgemm_dmma_v1<G>(NJ, R, R, b64, RS, 1, b64, RS, KS, snk); else if (PIPE == 1) zgemm_dmma_p<G>(NJ, R, R, b64, RS, 1, b64, RS, KS, snk); else if (PIPE == 2) zgemm_dmma_u<G, 4>(NJ, R, R, b64, RS, 1, b64, RS, KS, snk); else if (PIPE == 5) zgemm_dmma<G>(NJ, R, R, b64, RS, 1, b64, RS, KS, snk); else if (PIPE == 3) zgemm_dmma_i<G, 4>(NJ, R, R, b64, RS, 1, b64, RS, KS, snk); else zgemm_dmma_i<G, 8>(NJ, R, R, b64, RS, 1, b64, RS, KS, snk);
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && rep > 0) cyc[blockIdx.x * 20 + rep - 1] = t1 - t0;
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = out[5];
}

template <int WHICH, int PIPE, int G>
void run(const char* name, int S, int NJ, int R, int KS) {
  int RS = R;
  while (RS % 8 != 2 && RS % 8 != 6) ++RS;
  const int YSR = ((NJ + 11) & ~15) + 4;
  long long* cyc;
  double2* sink;
  cudaMalloc(&cyc, 148 * 20 * 8);
  cudaMalloc(&sink, 148 * 16);
  const size_t smem = 64 * YSR * 8 + 128 * RS * 16 + 4096 * 16;
  cudaFuncSetAttribute(kb<WHICH, PIPE, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kb<WHICH, PIPE, G><<<148, 256, smem>>>(S, NJ, R, RS, YSR, KS, cyc, sink);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  std::vector<long long> h(148 * 20);
  cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  const int M = WHICH == 0 ? S : WHICH == 1 ? NJ : WHICH == 2 ? R : NJ;
  const int K = WHICH == 0 ? NJ : WHICH == 1 ? S : WHICH == 2 ? NJ : R;
  const double dmma = (double)((M + 7) / 8) * ((R + 3) / 4) * ((K + 3) / 4) * 2;
  printf("%-26s pipe %d G %d KS %d  M %3d N %2d K %3d: %s median %6lld cycles  (%.1f cycles per DMMA per SM)\n", name,
         PIPE, G, KS, M, R, K, cudaGetErrorString(e), h[h.size() / 2], h[h.size() / 2] / dmma);
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  for (int v : {0, 5}) {
    printf("--- variant %d\n", v);
#define RUNV(W, G, name, S_, NJ_, R_, KS_) \
    if (v == 0) run<W, 0, G>(name, S_, NJ_, R_, KS_); else if (v == 1) run<W, 1, G>(name, S_, NJ_, R_, KS_); \
    else if (v == 2) run<W, 2, G>(name, S_, NJ_, R_, KS_); else if (v == 3) run<W, 3, G>(name, S_, NJ_, R_, KS_); \
    else if (v == 5) run<W, 5, G>(name, S_, NJ_, R_, KS_); else run<W, 4, G>(name, S_, NJ_, R_, KS_);
    RUNV(0, 4, "c3 Z", 42, 128, 16, 1)
    RUNV(0, 3, "c3 Z", 42, 128, 16, 1)
    RUNV(0, 6, "c3 Z", 42, 128, 16, 2)
    RUNV(0, 6, "c3 Z", 42, 128, 16, 1)
    RUNV(1, 4, "c3 W", 42, 128, 16, 1)
    RUNV(1, 2, "c3 W", 42, 128, 16, 1)
    RUNV(2, 4, "c3 GB", 42, 128, 16, 2)
    RUNV(3, 4, "c3 Q", 42, 128, 16, 1)
    RUNV(0, 4, "c2 Z", 48, 16, 20, 1)
    RUNV(1, 4, "c2 W", 48, 16, 20, 1)
    RUNV(2, 4, "c2 GB", 48, 16, 20, 1)
    RUNV(3, 4, "c2 Q", 48, 16, 20, 1)
  }
  return 0;
}
