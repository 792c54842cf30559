// The rows kernel's fp64-accumulating data GEMMs in isolation (config-3 CTA shapes: S = 42 sampled rows,
// nJ = 128 own columns, R = 16): Z = Y conj(Bh) (S x R, K = nJ, K split in parts) and
// W = Y^T conj(Ah_S) (nJ x R, K = S). One CTA of 256 threads per SM, operands in shared memory,
// clock64 per call (median of 20 calls). Compares register tiles and operand precisions.
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../../paper_1609_04104_b200/csrc/tt_block.cuh"

constexpr int S = 42, NJ = 128, R = 16, YSR = 130;

struct OutZ {
  double2* dst;
  int pstride;
  TT_DEV void operator()(int m, int n, int ks, double2 v) const { dst[(size_t)ks * pstride + m * R + n] = v; }
};
struct OutW {
  double2* acc;
  TT_DEV void operator()(int m, int n, int ks, double2 v) const { acc[m * R + n] = zadd(acc[m * R + n], v); }
};

template <int TM, int TN, int WHICH>
__global__ void __launch_bounds__(256, 1) bench(const float2* gy, const double2* gb, double2* gout, long long* cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  float2* ys = (float2*)sm;
  double2* bh = (double2*)(ys + S * YSR);
  double2* ah = bh + NJ * R;
  double2* w = ah + S * R;
  for (int o = threadIdx.x; o < S * YSR; o += 256) ys[o] = gy[o];
  for (int o = threadIdx.x; o < NJ * R; o += 256) bh[o] = gb[o];
  for (int o = threadIdx.x; o < S * R; o += 256) ah[o] = gb[o];
  for (int o = threadIdx.x; o < NJ * R; o += 256) w[o] = make_double2(0, 0);
  __syncthreads();
  const int tiles = ((S + TM - 1) / TM) * ((R + TN - 1) / TN);
  const int zks = max(1, min(256 / tiles, 8));
  for (int rep = 0; rep < 21; ++rep) {
    __syncthreads();
    long long t0 = clock64();
    if (WHICH == 0) {
      OutZ o{gout + (size_t)blockIdx.x * 8 * S * R, S * R};
      zgemm_fd<TM, TN, true, true>(S, R, NJ, ys, YSR, 1, bh, R, 1, zks, (double2*)nullptr, o);
    } else {
      OutW o{w};
      zgemm_fd<TM, TN, true, false>(NJ, R, S, ys, 1, YSR, ah, R, 1, 1, (double2*)nullptr, o);
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && rep > 0) cyc[blockIdx.x * 20 + rep - 1] = t1 - t0;
  }
  if (WHICH == 1)
    for (int o = threadIdx.x; o < NJ * R; o += 256) gout[o] = w[o];
}

template <int TM, int TN, int WHICH>
void run(const char* name, float2* gy, double2* gb, double2* go, long long* cyc) {
  size_t sm = S * YSR * 8 + NJ * R * 16 + S * R * 16 + NJ * R * 16;
  cudaFuncSetAttribute(bench<TM, TN, WHICH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  bench<TM, TN, WHICH><<<148, 256, sm>>>(gy, gb, go, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148 * 20);
  cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  const double dfma = 4.0 * S * NJ * R;
  printf("%-28s %s  median %lld cycles  (%.1f DFMA/clk/SM of 64)\n", name, cudaGetErrorString(e), h[h.size() / 2],
         dfma / h[h.size() / 2]);
}


// ---- DMMA (mma.sync m8n8k4 f64) versions: complex GEMMs as real GEMMs with interleaved (re, im) K and N
TT_DEV void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// B'[kk][n] of conj(B): kk = 2k + p (Y component), n = 2r + q (output component): p == q -> B.x, else B.y,
// negated for (p, q) = (0, 1)
TT_DEV double bfrag(const double2* B, int k, int r, int p, int q) {
  const double2 v = B[k * R + r];
  const double x = p == q ? v.x : v.y;
  return (p == 0 && q == 1) ? -x : x;
}
// W (NJ x R) = Y^T conj(Ah_S): warp w owns M-blocks 2w, 2w+1 (16 rows j) x all 4 N-blocks; K' = 2S
TT_DEV void w_dmma(const float2* ys, const double2* ah, double2* w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int kq = lane & 3, row = lane >> 2;
  const float* yf = (const float*)ys;
  for (int kk0 = 0; kk0 < 2 * S; kk0 += 4) {
    const int kk = kk0 + kq, k = kk >> 1, p = kk & 1;
    double af[2], bf[4];
#pragma unroll
    for (int mb = 0; mb < 2; ++mb) {
      const int j = (2 * warp + mb) * 8 + row;
      af[mb] = k < S ? (double)yf[2 * (k * YSR + j) + p] : 0.0;
    }
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      const int n = nb * 8 + row;
      bf[nb] = k < S ? bfrag(ah, k, n >> 1, p, n & 1) : 0.0;
    }
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb][0], acc[mb][nb][1], af[mb], bf[nb]);
  }
#pragma unroll
  for (int mb = 0; mb < 2; ++mb)
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      const int j = (2 * warp + mb) * 8 + row, r = nb * 4 + kq;
      w[j * R + r] = zadd(w[j * R + r], make_double2(acc[mb][nb][0], acc[mb][nb][1]));
    }
}
// Z (S x R) = Y conj(Bh): 6 M-blocks (rows k, padded to 48) x 4 N-blocks, K' = 2 NJ split in halves;
// warp w: K half w / 4, N-block w % 4, all 6 M-blocks
TT_DEV void z_dmma(const float2* ys, const double2* bh, double2* zp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = warp >> 2, nb = warp & 3;
  double acc[6][2];
#pragma unroll
  for (int a = 0; a < 6; ++a) acc[a][0] = acc[a][1] = 0.0;
  const int kq = lane & 3, row = lane >> 2;
  const float* yf = (const float*)ys;
  const int n = nb * 8 + row, r = n >> 1, q = n & 1;
  for (int kk0 = half * NJ; kk0 < (half + 1) * NJ; kk0 += 4) {
    const int kk = kk0 + kq, j = kk >> 1, p = kk & 1;
    const double bf = bfrag(bh, j, r, p, q);
    double af[6];
#pragma unroll
    for (int mb = 0; mb < 6; ++mb) {
      const int i = mb * 8 + row;
      af[mb] = i < S ? (double)yf[2 * (i * YSR + j) + p] : 0.0;
    }
#pragma unroll
    for (int mb = 0; mb < 6; ++mb) dmma(acc[mb][0], acc[mb][1], af[mb], bf);
  }
#pragma unroll
  for (int mb = 0; mb < 6; ++mb) {
    const int i = mb * 8 + row, rr = nb * 4 + kq;
    if (i < S) zp[(size_t)half * S * R + i * R + rr] = make_double2(acc[mb][0], acc[mb][1]);
  }
}
template <int WHICH>
__global__ void __launch_bounds__(256, 1) bench_dmma(const float2* gy, const double2* gb, double2* gout, long long* cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  float2* ys = (float2*)sm;
  double2* bh = (double2*)(ys + 48 * YSR);
  double2* ah = bh + NJ * R;
  double2* w = ah + 48 * R;
  for (int o = threadIdx.x; o < 48 * YSR; o += 256) ys[o] = o < S * YSR ? gy[o] : make_float2(0.f, 0.f);
  for (int o = threadIdx.x; o < NJ * R; o += 256) bh[o] = gb[o];
  for (int o = threadIdx.x; o < S * R; o += 256) ah[o] = gb[o];
  for (int o = threadIdx.x; o < NJ * R; o += 256) w[o] = make_double2(0, 0);
  __syncthreads();
  for (int rep = 0; rep < 21; ++rep) {
    __syncthreads();
    long long t0 = clock64();
    if (WHICH == 0) z_dmma(ys, bh, gout + (size_t)blockIdx.x * 8 * S * R);
    else w_dmma(ys, ah, w);
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && rep > 0) cyc[blockIdx.x * 20 + rep - 1] = t1 - t0;
  }
  if (WHICH == 1)
    for (int o = threadIdx.x; o < NJ * R; o += 256) gout[o] = w[o];
}
template <int WHICH>
void run_dmma(const char* name, float2* gy, double2* gb, double2* go, long long* cyc) {
  size_t sm = 48 * YSR * 8 + NJ * R * 16 + 48 * R * 16 + NJ * R * 16;
  cudaFuncSetAttribute(bench_dmma<WHICH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  bench_dmma<WHICH><<<148, 256, sm>>>(gy, gb, go, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148 * 20);
  cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  const double dfma = 4.0 * S * NJ * R;
  printf("%-28s %s  median %lld cycles  (%.1f DFMA/clk/SM of 64)\n", name, cudaGetErrorString(e), h[h.size() / 2],
         dfma / h[h.size() / 2]);
}
// reference results (same inputs) to validate the DMMA mapping against zgemm_fd
template <int WHICH>
__global__ void check_dmma(const float2* gy, const double2* gb, double2* o1, double2* o2) {
  extern __shared__ __align__(16) unsigned char sm[];
  float2* ys = (float2*)sm;
  double2* bh = (double2*)(ys + 48 * YSR);
  double2* ah = bh + NJ * R;
  double2* w = ah + 48 * R;
  for (int o = threadIdx.x; o < 48 * YSR; o += 256) ys[o] = o < S * YSR ? gy[o] : make_float2(0.f, 0.f);
  for (int o = threadIdx.x; o < NJ * R; o += 256) bh[o] = gb[o];
  for (int o = threadIdx.x; o < S * R; o += 256) ah[o] = gb[o];
  for (int o = threadIdx.x; o < NJ * R; o += 256) w[o] = make_double2(0, 0);
  __syncthreads();
  if (WHICH == 0) {
    z_dmma(ys, bh, o1);
    OutZ oz{o2, S * R};
    zgemm_fd<2, 4, true, true>(S, R, NJ, ys, YSR, 1, bh, R, 1, 2, (double2*)nullptr, oz);
  } else {
    w_dmma(ys, ah, w);
    __syncthreads();
    for (int o = threadIdx.x; o < NJ * R; o += 256) { o1[o] = w[o]; w[o] = make_double2(0, 0); }
    __syncthreads();
    OutW ow{w};
    zgemm_fd<2, 4, true, false>(NJ, R, S, ys, 1, YSR, ah, R, 1, 1, (double2*)nullptr, ow);
    __syncthreads();
    for (int o = threadIdx.x; o < NJ * R; o += 256) o2[o] = w[o];
  }
}
template <int WHICH>
void check(const char* name, float2* gy, double2* gb) {
  double2 *o1, *o2;
  const int n = WHICH == 0 ? 2 * S * R : NJ * R;
  cudaMalloc(&o1, n * 16); cudaMalloc(&o2, n * 16);
  size_t sm = 48 * YSR * 8 + NJ * R * 16 + 48 * R * 16 + NJ * R * 16;
  cudaFuncSetAttribute(check_dmma<WHICH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  check_dmma<WHICH><<<1, 256, sm>>>(gy, gb, o1, o2);
  cudaDeviceSynchronize();
  std::vector<double2> h1(n), h2(n);
  cudaMemcpy(h1.data(), o1, n * 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), o2, n * 16, cudaMemcpyDeviceToHost);
  double num = 0, den = 0;
  for (int i = 0; i < n; ++i) {
    num += (h1[i].x - h2[i].x) * (h1[i].x - h2[i].x) + (h1[i].y - h2[i].y) * (h1[i].y - h2[i].y);
    den += h2[i].x * h2[i].x + h2[i].y * h2[i].y;
  }
  printf("%s: DMMA vs zgemm_fd rel %.3e\n", name, sqrt(num / den));
}


// the rows kernel's zgemm_dmma (tt_block.cuh) at the config-3 shapes
template <int G, int WHICH>
__global__ void __launch_bounds__(256, 1) bench_zd(const float2* gy, const double2* gb, double2* gout, long long* cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  float2* ys = (float2*)sm;
  double2* bh = (double2*)(ys + 48 * YSR);
  double2* ah = bh + NJ * R;
  double2* w = ah + 48 * R;
  float2* bl = (float2*)(w + NJ * R);
  for (int o = threadIdx.x; o < 48 * YSR; o += 256) ys[o] = o < S * YSR ? gy[o] : make_float2(0.f, 0.f);
  for (int o = threadIdx.x; o < NJ * R; o += 256) { bh[o] = gb[o]; bl[o] = make_float2((float)gb[o].x, (float)gb[o].y); }
  for (int o = threadIdx.x; o < S * R; o += 256) ah[o] = gb[o];
  for (int o = threadIdx.x; o < NJ * R; o += 256) w[o] = make_double2(0, 0);
  __syncthreads();
  for (int rep = 0; rep < 21; ++rep) {
    __syncthreads();
    long long t0 = clock64();
    if (WHICH == 0) {
      OutZ o{gout + (size_t)blockIdx.x * 8 * S * R, S * R};
      const int items = ((((S + 7) >> 3) + G - 1) / G) * ((R + 3) >> 2);
      zgemm_dmma<G>(S, R, NJ, ys, YSR, 1, bh, R, max(1, 8 / items), o);
    } else if (WHICH == 1) {
      OutW o{w};
      zgemm_dmma<G>(NJ, R, S, ys, 1, YSR, ah, R, 1, o);
    } else {  // the Q correction: M = NJ, K = R, A = fp32 Bh rows, B = an R x R fp64 factor
      OutW o{w};
      zgemm_dmma<G>(NJ, R, R, bl, R, 1, ah, R, 1, o);
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && rep > 0) cyc[blockIdx.x * 20 + rep - 1] = t1 - t0;
  }
  if (WHICH == 1)
    for (int o = threadIdx.x; o < NJ * R; o += 256) gout[o] = w[o];
}
template <int G, int WHICH>
void run_zd(const char* name, float2* gy, double2* gb, double2* go, long long* cyc) {
  size_t sm = 48 * YSR * 8 + NJ * R * 16 + 48 * R * 16 + NJ * R * 16 + NJ * R * 8;
  cudaFuncSetAttribute(bench_zd<G, WHICH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  bench_zd<G, WHICH><<<148, 256, sm>>>(gy, gb, go, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148 * 20);
  cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  const double dfma = 4.0 * (WHICH == 2 ? (double)NJ * R * R : (double)S * NJ * R);
  printf("%-28s %s  median %lld cycles  (%.1f DFMA/clk/SM of 64)\n", name, cudaGetErrorString(e), h[h.size() / 2],
         dfma / h[h.size() / 2]);
}

int main() {
  float2* gy; double2* gb; double2* go; long long* cyc;
  cudaMalloc(&gy, S * YSR * 8); cudaMalloc(&gb, NJ * R * 16); cudaMalloc(&go, 148 * 8 * S * R * 16 + NJ * R * 16);
  cudaMalloc(&cyc, 148 * 20 * 8);
  std::vector<float2> hy(S * YSR); for (auto& v : hy) v = make_float2(rand() / 1e9f, rand() / 1e9f);
  std::vector<double2> hb(NJ * R); for (auto& v : hb) v = make_double2(rand() / 1e9, rand() / 1e9);
  cudaMemcpy(gy, hy.data(), hy.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(gb, hb.data(), hb.size() * 16, cudaMemcpyHostToDevice);
  run<2, 4, 0>("Z 2x4", gy, gb, go, cyc);
  run<4, 4, 0>("Z 4x4", gy, gb, go, cyc);
  run<2, 8, 0>("Z 2x8", gy, gb, go, cyc);
  run<1, 8, 0>("Z 1x8", gy, gb, go, cyc);
  run<2, 2, 0>("Z 2x2", gy, gb, go, cyc);
  run<2, 4, 1>("W 2x4", gy, gb, go, cyc);
  run<4, 4, 1>("W 4x4", gy, gb, go, cyc);
  run<2, 8, 1>("W 2x8", gy, gb, go, cyc);
  run<1, 8, 1>("W 1x8", gy, gb, go, cyc);
  run<4, 2, 1>("W 4x2", gy, gb, go, cyc);
  run_dmma<0>("Z dmma", gy, gb, go, cyc);
  run_dmma<1>("W dmma", gy, gb, go, cyc);
  run_zd<4, 0>("Z zgemm_dmma G4", gy, gb, go, cyc);
  run_zd<2, 0>("Z zgemm_dmma G2", gy, gb, go, cyc);
  run_zd<8, 0>("Z zgemm_dmma G8", gy, gb, go, cyc);
  run_zd<4, 1>("W zgemm_dmma G4", gy, gb, go, cyc);
  run_zd<2, 1>("W zgemm_dmma G2", gy, gb, go, cyc);
  run_zd<8, 1>("W zgemm_dmma G8", gy, gb, go, cyc);
  run_zd<4, 2>("Qcorr zgemm_dmma G4", gy, gb, go, cyc);
  run_zd<2, 2>("Qcorr zgemm_dmma G2", gy, gb, go, cyc);
  check<0>("Z", gy, gb);
  check<1>("W", gy, gb);
  return 0;
}
