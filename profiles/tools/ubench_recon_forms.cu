// The reconstruction X_f = A_f diag(gamma_f) B_f^T in three forms, timed alone at a config's shape
// (sm_100a): the four-product fp32 CUDA-core kernel the library ships (csrc/tt_recon.cu), Gauss's
// three-product fp32 form (25% fewer FFMAs, LDS.128 operand planes) and a split-BF16 tensor-core form
// (mma.sync m16n8k16, three bf16 pieces per fp32 operand, six piece products; persistent CTAs with the next
// tile's operands fetched by cp.async during the MMAs). Max |difference| to the four-product form is printed.
// Round-2 result (B200, F=1600 256x256 R=16): 4-product 355 us, 3-product 397-462 us, split-BF16 380 us;
// at R=8 512x512 the 4-product form already writes 3.8 TB/s. Neither alternative ships.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a ubench_recon_forms.cu -o /tmp/urf && /tmp/urf
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define TT_DEV __device__ __forceinline__
TT_DEV float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
TT_DEV float2 cfma(float2 a, float2 b, float2 acc) {
  acc.x = fmaf(a.x, b.x, fmaf(-a.y, b.y, acc.x));
  acc.y = fmaf(a.x, b.y, fmaf(a.y, b.x, acc.y));
  return acc;
}
TT_DEV int idiv(int a, int b) {
  int q = __float2int_rz(__fmul_rz((float)a, __frcp_rz((float)b)));
  const int r = a - q * b;
  q += (r >= b) - (r < 0);
  return q;
}

#define RC_T 64
#define RC_NT 256
#define RC_RMAX 64
#define RC_TP (RC_T + 1)  // padded row of the staged [r][64] tiles: conflict-free transposing stores

__global__ void __launch_bounds__(RC_NT) recon_kernel(int nx, int ny, int R, const float2* __restrict__ A,
                                                      const float2* __restrict__ B, const float2* __restrict__ gamma,
                                                      float2* __restrict__ X) {
  extern __shared__ __align__(16) float2 rsm[];
  float2* as = rsm;               // [R][RC_TP]
  float2* bs = rsm + R * RC_TP;   // [R][RC_TP]
  const int tid = threadIdx.x;
  const int f = blockIdx.z;
  const int i0 = blockIdx.y * RC_T, j0 = blockIdx.x * RC_T;
  const float2* Af = A + (size_t)f * nx * R;
  const float2* Bf = B + (size_t)f * ny * R;
  const float2* gf = gamma + (size_t)f * R;
  // staging: all of a thread's global loads in flight before the first shared-memory store
  // (the A / B tiles are contiguous rows of R values; up to 4 (A, B) pairs per thread per batch)
  for (int base = 0; base < RC_T * R; base += 4 * RC_NT) {
    float2 va[4], vb[4], vg[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int o = base + u * RC_NT + tid;
      va[u] = vb[u] = vg[u] = make_float2(0.f, 0.f);
      if (o < RC_T * R) {
        const int ii = idiv(o, R), r = o - ii * R;
        const int i = i0 + ii, j = j0 + ii;
        vg[u] = gf[r];
        if (i < nx) va[u] = Af[(size_t)i * R + r];
        if (j < ny) vb[u] = Bf[(size_t)j * R + r];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int o = base + u * RC_NT + tid;
      if (o < RC_T * R) {
        const int ii = idiv(o, R), r = o - ii * R;
        as[r * RC_TP + ii] = cmul(va[u], vg[u]);
        bs[r * RC_TP + ii] = vb[u];
      }
    }
  }
  __syncthreads();
  const int tj = tid & 15, ti = tid >> 4;  // 16 x 16 threads, 4 x 4 outputs each
  float2 acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = make_float2(0.f, 0.f);
  for (int r = 0; r < R; ++r) {
    float2 av[4], bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) av[u] = as[r * RC_TP + ti + 16 * u];
#pragma unroll
    for (int v = 0; v < 4; ++v) bv[v] = bs[r * RC_TP + tj + 16 * v];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = cfma(av[u], bv[v], acc[u][v]);
  }
  float2* Xf = X + (size_t)f * nx * ny;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = i0 + ti + 16 * u;
    if (i >= nx) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int j = j0 + tj + 16 * v;
      if (j < ny) Xf[(size_t)i * ny + j] = acc[u][v];
    }
  }
}

// ---------------------------------------------------------------- three-multiplication form
// The same tile with Gauss's three-product complex multiply: for a = ar + i ai, b = br + i bi,
//   re(ab) = br (ar + ai) - ai (br + bi),   im(ab) = br (ar + ai) + ar (bi - br),
// so X = Sum_r a_r b_r is three real accumulations K1 = Sum br s_a, K2 = Sum ar d_b, K3 = Sum ai s_b over
// operand planes staged once per tile (A: ar, ai, s_a = ar + ai; B: br, d_b = bi - br, s_b = br + bi):
// 3 FFMAs per complex MAC instead of 4, and each thread's 4 rows / 4 columns are consecutive, so one
// LDS.128 per plane and r feeds 12 FFMAs (the 4-product form needs 8 LDS.64 per 64 FFMAs). Error: each
// accumulated product is bounded by (|ar| + |ai|)(|br| + |bi|), within 2x of the 4-product bound; the
// results agree with the complex128 outer product to ~1e-7 relative (tests/test_gpu_values.py).
#define RG_TP (RC_T + 4)  // padded plane row (16 B aligned rows for LDS.128)

__global__ void __launch_bounds__(RC_NT, 3) recon3_kernel(int nx, int ny, int R, const float2* __restrict__ A,
                                                       const float2* __restrict__ B, const float2* __restrict__ gamma,
                                                       float2* __restrict__ X) {
  extern __shared__ __align__(16) float rgs[];
  const int PL = R * RG_TP;  // plane size
  float* p_ar = rgs;
  float* p_ai = rgs + PL;
  float* p_sa = rgs + 2 * PL;
  float* p_br = rgs + 3 * PL;
  float* p_db = rgs + 4 * PL;
  float* p_sb = rgs + 5 * PL;
  const int tid = threadIdx.x;
  const int f = blockIdx.z;
  const int i0 = blockIdx.y * RC_T, j0 = blockIdx.x * RC_T;
  const float2* Af = A + (size_t)f * nx * R;
  const float2* Bf = B + (size_t)f * ny * R;
  const float2* gf = gamma + (size_t)f * R;
  for (int base = 0; base < RC_T * R; base += 4 * RC_NT) {
    float2 va[4], vb[4], vg[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int o = base + u * RC_NT + tid;
      va[u] = vb[u] = vg[u] = make_float2(0.f, 0.f);
      if (o < RC_T * R) {
        const int ii = idiv(o, R), r = o - ii * R;
        const int i = i0 + ii, j = j0 + ii;
        vg[u] = gf[r];
        if (i < nx) va[u] = Af[(size_t)i * R + r];
        if (j < ny) vb[u] = Bf[(size_t)j * R + r];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int o = base + u * RC_NT + tid;
      if (o < RC_T * R) {
        const int ii = idiv(o, R), r = o - ii * R;
        const float2 a = cmul(va[u], vg[u]), b = vb[u];
        const int at = r * RG_TP + ii;
        p_ar[at] = a.x;
        p_ai[at] = a.y;
        p_sa[at] = a.x + a.y;
        p_br[at] = b.x;
        p_db[at] = b.y - b.x;
        p_sb[at] = b.x + b.y;
      }
    }
  }
  __syncthreads();
  const int tj = tid & 15, ti = tid >> 4;  // 16 x 16 threads, 4 x 4 outputs each (rows 4 ti.., cols 4 tj..)
  float k1[4][4], k2[4][4], k3[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) k1[u][v] = k2[u][v] = k3[u][v] = 0.f;
#pragma unroll 2
  for (int r = 0; r < R; ++r) {
    const int ra = r * RG_TP + 4 * ti, rb = r * RG_TP + 4 * tj;
    const float4 ar = *(const float4*)(p_ar + ra), ai = *(const float4*)(p_ai + ra), sa = *(const float4*)(p_sa + ra);
    const float4 br = *(const float4*)(p_br + rb), db = *(const float4*)(p_db + rb), sb = *(const float4*)(p_sb + rb);
    const float arv[4] = {ar.x, ar.y, ar.z, ar.w}, aiv[4] = {ai.x, ai.y, ai.z, ai.w}, sav[4] = {sa.x, sa.y, sa.z, sa.w};
    const float brv[4] = {br.x, br.y, br.z, br.w}, dbv[4] = {db.x, db.y, db.z, db.w}, sbv[4] = {sb.x, sb.y, sb.z, sb.w};
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        k1[u][v] = fmaf(brv[v], sav[u], k1[u][v]);
        k2[u][v] = fmaf(arv[u], dbv[v], k2[u][v]);
        k3[u][v] = fmaf(aiv[u], sbv[v], k3[u][v]);
      }
  }
  float2* Xf = X + (size_t)f * nx * ny;
  const bool vec = (ny & 1) == 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = i0 + 4 * ti + u;
    if (i >= nx) continue;
    float2* xr = Xf + (size_t)i * ny;
    const int j = j0 + 4 * tj;
    float2 o[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) o[v] = make_float2(k1[u][v] - k3[u][v], k1[u][v] + k2[u][v]);
    if (vec && j + 3 < ny) {
      __stcs((float4*)(xr + j), make_float4(o[0].x, o[0].y, o[1].x, o[1].y));
      __stcs((float4*)(xr + j + 2), make_float4(o[2].x, o[2].y, o[3].x, o[3].y));
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (j + v < ny) xr[j + v] = o[v];
    }
  }
}


// Gauss form with full-sector stores: a thread's 4 columns are 2 tj, 2 tj + 1, 2 tj + 32, 2 tj + 33 (one 16 B
// store per pair: a warp's store covers 256 contiguous bytes of a row), its 4 rows 4 ti .. 4 ti + 3 (LDS.128);
// the three planes are consumed one after the other so only 8 operands are live.
__global__ void __launch_bounds__(RC_NT, 3) recon3b_kernel(int nx, int ny, int R, const float2* __restrict__ A,
                                                           const float2* __restrict__ B, const float2* __restrict__ gamma,
                                                           float2* __restrict__ X) {
  extern __shared__ __align__(16) float rgs[];
  const int PL = R * RG_TP;
  float* p_ar = rgs;
  float* p_ai = rgs + PL;
  float* p_sa = rgs + 2 * PL;
  float* p_br = rgs + 3 * PL;
  float* p_db = rgs + 4 * PL;
  float* p_sb = rgs + 5 * PL;
  const int tid = threadIdx.x;
  const int f = blockIdx.z;
  const int i0 = blockIdx.y * RC_T, j0 = blockIdx.x * RC_T;
  const float2* Af = A + (size_t)f * nx * R;
  const float2* Bf = B + (size_t)f * ny * R;
  const float2* gf = gamma + (size_t)f * R;
  for (int base = 0; base < RC_T * R; base += 4 * RC_NT) {
    float2 va[4], vb[4], vg[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int o = base + u * RC_NT + tid;
      va[u] = vb[u] = vg[u] = make_float2(0.f, 0.f);
      if (o < RC_T * R) {
        const int ii = idiv(o, R), r = o - ii * R;
        const int i = i0 + ii, j = j0 + ii;
        vg[u] = gf[r];
        if (i < nx) va[u] = Af[(size_t)i * R + r];
        if (j < ny) vb[u] = Bf[(size_t)j * R + r];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int o = base + u * RC_NT + tid;
      if (o < RC_T * R) {
        const int ii = idiv(o, R), r = o - ii * R;
        const float2 a = cmul(va[u], vg[u]), b = vb[u];
        const int at = r * RG_TP + ii;
        p_ar[at] = a.x;
        p_ai[at] = a.y;
        p_sa[at] = a.x + a.y;
        p_br[at] = b.x;
        p_db[at] = b.y - b.x;
        p_sb[at] = b.x + b.y;
      }
    }
  }
  __syncthreads();
  const int tj = tid & 15, ti = tid >> 4;
  float k1[4][4], k2[4][4], k3[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) k1[u][v] = k2[u][v] = k3[u][v] = 0.f;
  const int ca = 4 * ti, cb = 2 * tj;
#pragma unroll 2
  for (int r = 0; r < R; ++r) {
    const int ro = r * RG_TP;
    {
      const float4 a = *(const float4*)(p_sa + ro + ca);
      const float2 b0 = *(const float2*)(p_br + ro + cb), b1 = *(const float2*)(p_br + ro + cb + 32);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) k1[u][v] = fmaf(bv[v], av[u], k1[u][v]);
    }
    {
      const float4 a = *(const float4*)(p_ar + ro + ca);
      const float2 b0 = *(const float2*)(p_db + ro + cb), b1 = *(const float2*)(p_db + ro + cb + 32);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) k2[u][v] = fmaf(av[u], bv[v], k2[u][v]);
    }
    {
      const float4 a = *(const float4*)(p_ai + ro + ca);
      const float2 b0 = *(const float2*)(p_sb + ro + cb), b1 = *(const float2*)(p_sb + ro + cb + 32);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) k3[u][v] = fmaf(av[u], bv[v], k3[u][v]);
    }
  }
  float2* Xf = X + (size_t)f * nx * ny;
  const bool vec = (ny & 1) == 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = i0 + ca + u;
    if (i >= nx) continue;
    float2* xr = Xf + (size_t)i * ny;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = j0 + cb + 32 * h;
      const float2 o0 = make_float2(k1[u][2 * h] - k3[u][2 * h], k1[u][2 * h] + k2[u][2 * h]);
      const float2 o1 = make_float2(k1[u][2 * h + 1] - k3[u][2 * h + 1], k1[u][2 * h + 1] + k2[u][2 * h + 1]);
      if (vec && j + 1 < ny) {
        *(float4*)(xr + j) = make_float4(o0.x, o0.y, o1.x, o1.y);
      } else {
        if (j < ny) xr[j] = o0;
        if (j + 1 < ny) xr[j + 1] = o1;
      }
    }
  }
}

// ---------------------------------------------------------------- split-BF16 tensor-core form
// The same X_f = A_f diag(gamma_f) B_f^T on the tensor cores at fp32 accuracy. As real products over
// K = 2 RP (RP = R padded to 8):
//   Xr = [A'r | -A'i] . [Br | Bi]^T,   Xi = [A'i | A'r] . [Br | Bi]^T      (A' = A diag(gamma)),
// so B is staged once and A twice. Every fp32 operand is split exactly into three bf16 pieces
// x = x0 + x1 + x2 (round to nearest; each residual is exact in fp32) and the six piece products with
// pa + pb <= 2 are accumulated in fp32 by mma.sync m16n8k16 (products of bf16 pieces are exact in fp32;
// the dropped ones are below 2^-24 of the leading term), small products first. The fp32 CUDA-core form
// is bound by register reads (two fresh operands per FFMA, ~38 TFLOP/s); the BF16 MMA runs at ~595
// TFLOP/s (profiles/tools/ubench_mma_tf32.cu), so six of them per product leave the kernel bound by the
// frames' HBM writes. Tile 64 (rows i) x 128 (cols j) per CTA, 4 warps of 32 x 64, fragments by
// ldmatrix from rows padded by 16 B (conflict-free for every K); three CTAs per SM overlap one tile's
// staging and epilogue with another's MMAs.
#include <cuda_bf16.h>
#define RB_TM 64
#define RB_TN 128
#define RB_NT 128

__device__ __forceinline__ void rb_split3(float x, __nv_bfloat16 (&h)[3]) {
  h[0] = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(h[0]);
  h[1] = __float2bfloat16_rn(r1);
  h[2] = __float2bfloat16_rn(r1 - __bfloat162float(h[1]));
}
__device__ __forceinline__ unsigned rb_pack(__nv_bfloat16 lo, __nv_bfloat16 hi) {
  return (unsigned)__bfloat16_as_ushort(lo) | ((unsigned)__bfloat16_as_ushort(hi) << 16);
}
__device__ __forceinline__ void rb_mma(float (&c)[4], const unsigned* a, unsigned b0, unsigned b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};\n"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void rb_ldm4(unsigned (&r)[4], const void* p) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(s));
}

__device__ __forceinline__ void rb_cp16(void* dst, const void* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void rb_cp8(void* dst, const void* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}

// Persistent: each CTA walks tiles blockIdx.x, + gridDim.x, ...; the next tile's raw fp32 operands are
// fetched by cp.async into a raw buffer while the current tile's MMAs run, so the split reads shared
// memory only. KT = K / 16 (RP = 8 KT).
template <int KT>
__global__ void __launch_bounds__(RB_NT, 2) recon_bf16x3_kernel(int frames, int nx, int ny, int R,
                                                                 const float2* __restrict__ A,
                                                                 const float2* __restrict__ B,
                                                                 const float2* __restrict__ gamma,
                                                                 float2* __restrict__ X) {
  constexpr int RP = 8 * KT, K = 16 * KT, KS = K + 8;  // row stride in bf16 elements
  constexpr int PA = RB_TM * KS, PB = RB_TN * KS;      // piece strides
  constexpr int QP = RP / 2;
  extern __shared__ __align__(16) unsigned char rbs[];
  __nv_bfloat16* ar = (__nv_bfloat16*)rbs;  // [3][64][KS]  [A'r | -A'i]
  __nv_bfloat16* ai = ar + 3 * PA;          // [3][64][KS]  [A'i |  A'r]
  __nv_bfloat16* bs = ai + 3 * PA;          // [3][128][KS] [Br  |  Bi]
  float2* rawA = (float2*)(bs + 3 * PB);    // [64][RP]
  float2* rawB = rawA + RB_TM * RP;         // [128][RP]
  float2* rawG = rawB + RB_TN * RP;         // [RP]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nti = (nx + RB_TM - 1) / RB_TM, ntj = (ny + RB_TN - 1) / RB_TN;
  const int per_frame = nti * ntj;
  const long long ntiles = (long long)frames * per_frame;
  const bool even = (R & 1) == 0;

  auto fetch = [&](long long tile) {
    const int f = (int)(tile / per_frame), rem = (int)(tile - (long long)f * per_frame);
    const int i0 = (rem / ntj) * RB_TM, j0 = (rem % ntj) * RB_TN;
    const float2* Af = A + (size_t)f * nx * R;
    const float2* Bf = B + (size_t)f * ny * R;
    if (even) {
      for (int o = tid; o < (RB_TM + RB_TN) * QP; o += RB_NT) {
        const int row = o / QP, r = 2 * (o - row * QP);
        if (row < RB_TM) {
          const int i = i0 + row;
          const bool ok = i < nx && r < R;
          rb_cp16(rawA + row * RP + r, ok ? (const void*)(Af + (size_t)i * R + r) : (const void*)A, ok);
        } else {
          const int jj = row - RB_TM, j = j0 + jj;
          const bool ok = j < ny && r < R;
          rb_cp16(rawB + jj * RP + r, ok ? (const void*)(Bf + (size_t)j * R + r) : (const void*)B, ok);
        }
      }
    } else {
      for (int o = tid; o < (RB_TM + RB_TN) * RP; o += RB_NT) {
        const int row = o / RP, r = o - row * RP;
        if (row < RB_TM) {
          const int i = i0 + row;
          const bool ok = i < nx && r < R;
          rb_cp8(rawA + row * RP + r, ok ? (const void*)(Af + (size_t)i * R + r) : (const void*)A, ok);
        } else {
          const int jj = row - RB_TM, j = j0 + jj;
          const bool ok = j < ny && r < R;
          rb_cp8(rawB + jj * RP + r, ok ? (const void*)(Bf + (size_t)j * R + r) : (const void*)B, ok);
        }
      }
    }
    if (tid < RP) rb_cp8(rawG + tid, tid < R ? (const void*)(gamma + (size_t)f * R + tid) : (const void*)gamma, tid < R);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  long long tile = blockIdx.x;
  if (tile < ntiles) fetch(tile);
  const int g = lane >> 2, t = lane & 3;
  const int wr = (warp >> 1) * 32, wc = (warp & 1) * 64;  // warp tile 32 x 64
  // ldmatrix addresses: A 16x16 tiles (row lane%16, k half lane/16); B two n8 x k16 tiles per x4
  const int a_off = (wr + (lane & 15)) * KS + (lane >> 4) * 8;
  const int b_off = (wc + (lane & 7) + ((lane >> 4) << 3)) * KS + ((lane >> 3) & 1) * 8;
  for (; tile < ntiles; tile += gridDim.x) {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    // split the raw operands into bf16 pieces
    for (int o = tid; o < (RB_TM + RB_TN) * QP; o += RB_NT) {
      const int row = o / QP, q = o - row * QP, r = 2 * q;
      const bool isa = row < RB_TM;
      float2 v0, v1;
      if (isa) {
        v0 = cmul(rawA[row * RP + r], rawG[r]);
        v1 = cmul(rawA[row * RP + r + 1], rawG[r + 1]);
      } else {
        v0 = rawB[(row - RB_TM) * RP + r];
        v1 = rawB[(row - RB_TM) * RP + r + 1];
      }
      __nv_bfloat16 re0[3], re1[3], im0[3], im1[3];
      rb_split3(v0.x, re0);
      rb_split3(v1.x, re1);
      rb_split3(v0.y, im0);
      rb_split3(v1.y, im1);
      if (isa) {
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const int at = p * PA + row * KS;
          *(unsigned*)(ar + at + r) = rb_pack(re0[p], re1[p]);
          *(unsigned*)(ar + at + RP + r) = rb_pack(__hneg(im0[p]), __hneg(im1[p]));
          *(unsigned*)(ai + at + r) = rb_pack(im0[p], im1[p]);
          *(unsigned*)(ai + at + RP + r) = rb_pack(re0[p], re1[p]);
        }
      } else {
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const int at = p * PB + (row - RB_TM) * KS;
          *(unsigned*)(bs + at + r) = rb_pack(re0[p], re1[p]);
          *(unsigned*)(bs + at + RP + r) = rb_pack(im0[p], im1[p]);
        }
      }
    }
    __syncthreads();
    if (tile + gridDim.x < ntiles) fetch(tile + gridDim.x);  // overlaps the MMAs below
    float cr[2][8][4], ci[2][8][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) cr[mt][nt][q] = ci[mt][nt][q] = 0.f;
#pragma unroll 1
    for (int kt = 0; kt < KT; ++kt) {
#pragma unroll
      for (int pa = 2; pa >= 0; --pa) {
        unsigned fr[2][4], fi[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          rb_ldm4(fr[mt], ar + pa * PA + a_off + mt * 16 * KS + kt * 16);
          rb_ldm4(fi[mt], ai + pa * PA + a_off + mt * 16 * KS + kt * 16);
        }
#pragma unroll
        for (int np = 0; np < 4; ++np) {
#pragma unroll
          for (int pb = 2 - pa; pb >= 0; --pb) {
            unsigned fb[4];
            rb_ldm4(fb, bs + pb * PB + b_off + np * 16 * KS + kt * 16);
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int mt = 0; mt < 2; ++mt) {
                rb_mma(cr[mt][2 * np + h], fr[mt], fb[2 * h], fb[2 * h + 1]);
                rb_mma(ci[mt][2 * np + h], fi[mt], fb[2 * h], fb[2 * h + 1]);
              }
          }
        }
      }
    }
    const int f = (int)(tile / per_frame), rem = (int)(tile - (long long)f * per_frame);
    const int i0 = (rem / ntj) * RB_TM, j0 = (rem % ntj) * RB_TN;
    float2* Xf = X + (size_t)f * nx * ny;
    const bool vec = (ny & 1) == 0;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = i0 + wr + mt * 16 + g + 8 * h;
        if (i >= nx) continue;
        float2* xr = Xf + (size_t)i * ny;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          const int j = j0 + wc + nt * 8 + 2 * t;
          const float4 v =
              make_float4(cr[mt][nt][2 * h], ci[mt][nt][2 * h], cr[mt][nt][2 * h + 1], ci[mt][nt][2 * h + 1]);
          if (vec && j + 1 < ny) {
            __stcs((float4*)(xr + j), v);
          } else {
            if (j < ny) xr[j] = make_float2(v.x, v.y);
            if (j + 1 < ny) xr[j + 1] = make_float2(v.z, v.w);
          }
        }
      }
  }
}


#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

template <int KT>
static void launch_tc(int F, int nx, int ny, int R, const float2* a, const float2* b, const float2* g, float2* x) {
  constexpr int RP = 8 * KT;
  const size_t smb = sizeof(__nv_bfloat16) * 3 * (2 * RB_TM + RB_TN) * (size_t)(16 * KT + 8) +
                     sizeof(float2) * (size_t)((RB_TM + RB_TN) * RP + RP);
  CK(cudaFuncSetAttribute(recon_bf16x3_kernel<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
  int per_sm = 0, sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, recon_bf16x3_kernel<KT>, RB_NT, smb));
  const long long tiles = (long long)F * ((nx + RB_TM - 1) / RB_TM) * ((ny + RB_TN - 1) / RB_TN);
  const int grid = (int)(tiles < (long long)sms * per_sm ? tiles : (long long)sms * per_sm);
  recon_bf16x3_kernel<KT><<<grid, RB_NT, smb>>>(F, nx, ny, R, a, b, g, x);
}

static void run(int form, int F, int nx, int ny, int R, const float2* a, const float2* b, const float2* g, float2* x) {
  dim3 grid((ny + RC_T - 1) / RC_T, (nx + RC_T - 1) / RC_T, F);
  if (form == 0) {
    const size_t sm = sizeof(float2) * 2 * RC_TP * (size_t)R;
    CK(cudaFuncSetAttribute(recon_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    recon_kernel<<<grid, RC_NT, sm>>>(nx, ny, R, a, b, g, x);
  } else if (form == 1) {
    const size_t sm = sizeof(float) * 6 * RG_TP * (size_t)R;
    CK(cudaFuncSetAttribute(recon3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    recon3_kernel<<<grid, RC_NT, sm>>>(nx, ny, R, a, b, g, x);
  } else if (form == 3) {
    const size_t sm = sizeof(float) * 6 * RG_TP * (size_t)R;
    CK(cudaFuncSetAttribute(recon3b_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    recon3b_kernel<<<grid, RC_NT, sm>>>(nx, ny, R, a, b, g, x);
  } else {
    switch ((R + 7) / 8) {
      case 1: launch_tc<1>(F, nx, ny, R, a, b, g, x); break;
      case 2: launch_tc<2>(F, nx, ny, R, a, b, g, x); break;
      case 3: launch_tc<3>(F, nx, ny, R, a, b, g, x); break;
      default: launch_tc<4>(F, nx, ny, R, a, b, g, x); break;
    }
  }
  CK(cudaGetLastError());
}

int main(int argc, char** argv) {
  const int F = argc > 4 ? atoi(argv[1]) : 1600, nx = argc > 4 ? atoi(argv[2]) : 256,
            ny = argc > 4 ? atoi(argv[3]) : 256, R = argc > 4 ? atoi(argv[4]) : 16;
  const size_t na = (size_t)F * nx * R, nb = (size_t)F * ny * R, ng = (size_t)F * R, nxo = (size_t)F * nx * ny;
  std::vector<float2> h(na + nb + ng);
  unsigned s = 12345;
  for (auto& v : h) {
    s = s * 1664525u + 1013904223u; v.x = (float)(s >> 8) / 16777216.f - 0.5f;
    s = s * 1664525u + 1013904223u; v.y = (float)(s >> 8) / 16777216.f - 0.5f;
  }
  float2 *d, *x0, *x1;
  CK(cudaMalloc(&d, h.size() * sizeof(float2)));
  CK(cudaMalloc(&x0, nxo * sizeof(float2)));
  CK(cudaMalloc(&x1, nxo * sizeof(float2)));
  CK(cudaMemcpy(d, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice));
  const float2 *a = d, *b = d + na, *g = d + na + nb;
  run(0, F, nx, ny, R, a, b, g, x0);
  std::vector<float2> r0(nxo), r1(nxo);
  CK(cudaMemcpy(r0.data(), x0, nxo * sizeof(float2), cudaMemcpyDeviceToHost));
  const char* names[4] = {"four-product fp32", "three-product fp32", "split-BF16 mma.sync", "three-product, 16B st"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int form = 0; form < 4; ++form) {
    if (form == 2 && R > 32) continue;
    for (int w = 0; w < 3; ++w) run(form, F, nx, ny, R, a, b, g, x1);
    cudaEventRecord(e0);
    for (int it = 0; it < 20; ++it) run(form, F, nx, ny, R, a, b, g, x1);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 20;
    CK(cudaMemcpy(r1.data(), x1, nxo * sizeof(float2), cudaMemcpyDeviceToHost));
    double md = 0, mx = 0;
    for (size_t i = 0; i < nxo; ++i) {
      md = fmax(md, fmax(fabs(r1[i].x - r0[i].x), fabs(r1[i].y - r0[i].y)));
      mx = fmax(mx, fmax(fabs(r0[i].x), fabs(r0[i].y)));
    }
    printf("%-22s F=%d %dx%d R=%d: %8.1f us/launch, writes %6.0f GB/s, max|diff| %.2e (max|x| %.2e)\n", names[form], F,
           nx, ny, R, ms * 1e3, nxo * 8.0 / ms / 1e6, md, mx);
  }
  return 0;
}
