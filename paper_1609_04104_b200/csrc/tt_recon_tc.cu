// Frame reconstruction X_f = A_f diag(gamma_f) B_f^T on the 5th-generation tensor cores (tcgen05, TMEM).
//
// Same product as recon_kernel (tt_recon.cu; reference core.synthesize_slice core.py:91-104 and
// mri.reconstruct_frame mri.py:107-121), for R <= 32. The complex product is one real GEMM whose output
// columns are the interleaved (re, im) pairs of a complex64 row, so the accumulator rows leave TMEM as
// contiguous complex64 output:
//   X[i][2j + 0] = sum_k A2[i][k] B2[2j + 0][k],   A2 = [A'r | A'i],  B2[2j + 0] = [Br | -Bi]
//   X[i][2j + 1] = sum_k A2[i][k] B2[2j + 1][k],                      B2[2j + 1] = [Bi |  Br]
// with A' = A diag(gamma), K = 2 RP (RP = R padded to 4, zeros beyond R). fp32 accuracy from TF32 inputs
// (3xTF32): every operand is split x = hi + lo with hi, lo rounded to TF32 (cvt.rna), and the tile
// accumulates lo*hi + hi*lo + hi*hi in fp32 (the dropped lo*lo term and lo's own rounding are ~2^-22 of
// |x|; the four-product CUDA-core form stays in tt_recon.cu for R > 32 and as the check).
//
// One persistent CTA per SM (512 TMEM columns: two 128 x 256 fp32 accumulators). Warps 0-3 stage a tile's
// operands (fp32 loads, gamma scaling, the TF32 split) into shared memory in the no-swizzle K-major core-
// matrix layout, thread 0 then issues the tile's 3 Kp/8 tcgen05.mma (M 128, N 256, K 8) into accumulator
// n % 2 and commits them to an mbarrier; warps 4-7 drain the other accumulator with tcgen05.ld (one output
// row per thread, 128 contiguous bytes per 32 columns) while the next tile is staged and multiplied. The
// kernel is bound by the HBM writes of the frames.
#include <stdlib.h>

#include "tt_block.cuh"
#include "tt_common.cuh"

#define RT_M 128   // accumulator rows = TMEM lanes = output rows per tile
#define RT_NC 128  // complex output columns per tile (256 real accumulator columns)
#define RT_NT 256  // warps 0-3: operand staging (thread 0 issues the MMAs); warps 4-7: TMEM drain

namespace {

// UMMA shared-memory descriptor, K-major, no swizzle (cute/arch/mma_sm100_desc.hpp SmemDescriptor: start
// address >> 4 at [0,14), leading byte offset >> 4 at [16,30) = the K-adjacent core matrix stride, stride
// byte offset >> 4 at [32,46) = the 8-row group stride, version 1 at [46,48), layout type 0 at [61,64)).
TT_DEV unsigned long long umma_desc(unsigned saddr, unsigned lbo, unsigned sbo) {
  return (unsigned long long)((saddr & 0x3FFFF) >> 4) | ((unsigned long long)(lbo >> 4) << 16) |
         ((unsigned long long)(sbo >> 4) << 32) | (1ull << 46);
}
// instruction descriptor, kind::tf32 (InstrDescriptor): D f32 [4,6) = 1, A tf32 [7,10) = 2, B tf32 [10,13) = 2,
// both K-major, N >> 3 at [17,23), M >> 4 at [24,29)
constexpr unsigned RT_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((2u * RT_NC >> 3) << 17) | ((RT_M >> 4) << 24);

TT_DEV void umma_tf32(unsigned tmem_d, unsigned long long da, unsigned long long db, unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(RT_IDESC), "r"(accumulate)
      : "memory");
}
TT_DEV void umma_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
TT_DEV void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
TT_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
TT_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
TT_DEV float tf32_rna(float x) {
  unsigned u;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(u) : "f"(x));
  return __uint_as_float(u);
}
TT_DEV void split4(float4 v, float4& hi, float4& lo) {
  hi = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
  lo = make_float4(tf32_rna(v.x - hi.x), tf32_rna(v.y - hi.y), tf32_rna(v.z - hi.z), tf32_rna(v.w - hi.w));
}
// 32 consecutive TMEM columns of this thread's lane
#define RT_LD32(taddr, v)                                                                                        \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"  \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                      \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), \
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),       \
                 "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),     \
                 "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),     \
                 "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                                                          \
               : "r"(taddr))

}  // namespace

// KC = 16-byte K chunks per operand row (Kp = 4 KC real, RP = 2 KC complex per half)
template <int KC>
__global__ void __launch_bounds__(RT_NT, 1) recon_tc_kernel(int frames, int nx, int ny, int R,
                                                            const float2* __restrict__ A, const float2* __restrict__ B,
                                                            const float2* __restrict__ gamma, float2* __restrict__ X,
                                                            int vec) {
  constexpr int Kp = 4 * KC, HC = KC / 2;  // HC: chunks per half (re | im), 4 complex per chunk
  constexpr unsigned SBO = KC * 128;        // bytes per 8-row group (all its K chunks, 128 B each)
  constexpr unsigned A_BYTES = RT_M * Kp * 4, B_BYTES = 2 * RT_NC * Kp * 4;
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* a_hi = sm;
  unsigned char* a_lo = sm + A_BYTES;
  unsigned char* b_hi = sm + 2 * A_BYTES;
  unsigned char* b_lo = b_hi + B_BYTES;
  unsigned long long* mma_done = (unsigned long long*)(b_lo + B_BYTES);  // [2], one arrival (the commit)
  unsigned long long* acc_free = mma_done + 2;                             // [2], 128 arrivals (the drain)
  unsigned* tmem_slot = (unsigned*)(acc_free + 2);
  float2* gs = (float2*)(acc_free + 4);          // the tile's gamma (2 KC values)
  float* tbuf = (float*)(gs + 2 * KC);            // drain transpose: 4 warps x 32 rows x 36 floats
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    mbar_init(&mma_done[0], 1);
    mbar_init(&mma_done[1], 1);
    mbar_init(&acc_free[0], 128);
    mbar_init(&acc_free[1], 128);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = *tmem_slot;

  const int tiles_i = (nx + RT_M - 1) / RT_M, tiles_j = (ny + RT_NC - 1) / RT_NC;
  const int per_frame = tiles_i * tiles_j;
  const long long ntiles = (long long)frames * per_frame;
  auto tile_origin = [&](long long t, int& f, int& i0, int& j0) {
    f = (int)(t / per_frame);
    const int rem = (int)(t - (long long)f * per_frame);
    i0 = (rem / tiles_j) * RT_M;
    j0 = (rem % tiles_j) * RT_NC;
  };
  // byte offset of (row, 16-byte K chunk) in the core-matrix layout
  auto cm = [&](int row, int chunk) -> unsigned {
    return (unsigned)(row >> 3) * SBO + (unsigned)chunk * 128u + (unsigned)(row & 7) * 16u;
  };

  if (warp < 4) {
    // ---------------- staging + MMA issue. The next tile's raw operands are loaded into registers right
    // after a tile's MMAs are issued (they land while the tensor cores run); the split waits only for the
    // MMAs that still read shared memory.
    float2 ra[HC][4], rb[HC][4], rg = make_float2(0.f, 0.f);
    auto fetch = [&](long long t) {
      int f, i0, j0;
      tile_origin(t, f, i0, j0);
      const float2* Af = A + (size_t)f * nx * R;
      const float2* Bf = B + (size_t)f * ny * R;
#pragma unroll
      for (int u = 0; u < HC; ++u) {
        const int it = tid + 128 * u;  // RT_M * HC items, HC per thread
        const int row = it / HC, c = it - row * HC, i = i0 + row, j = j0 + row;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = 4 * c + e;
          ra[u][e] = (i < nx && r < R) ? __ldg(Af + (size_t)i * R + r) : make_float2(0.f, 0.f);
          rb[u][e] = (j < ny && r < R) ? __ldg(Bf + (size_t)j * R + r) : make_float2(0.f, 0.f);
        }
      }
      if (tid < R) rg = __ldg(gamma + (size_t)f * R + tid);
    };
    int n = 0;
    if ((long long)blockIdx.x < ntiles) fetch(blockIdx.x);
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++n) {
      if (n >= 1) mbar_wait(&mma_done[(n - 1) & 1], ((n - 1) >> 1) & 1);  // the previous tile's MMAs read smem
      if (tid < 2 * KC) gs[tid] = rg;  // RP = 2 KC gamma values (zeros past R)
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
#pragma unroll
      for (int u = 0; u < HC; ++u) {
        const int it = tid + 128 * u;
        const int row = it / HC, c = it - row * HC;
        float4 hi, lo;
        {  // A' = A diag(gamma): row `row`, re chunk c and im chunk HC + c
          float2 v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) v[e] = cmul(ra[u][e], gs[4 * c + e]);
          split4(make_float4(v[0].x, v[1].x, v[2].x, v[3].x), hi, lo);
          *(float4*)(a_hi + cm(row, c)) = hi;
          *(float4*)(a_lo + cm(row, c)) = lo;
          split4(make_float4(v[0].y, v[1].y, v[2].y, v[3].y), hi, lo);
          *(float4*)(a_hi + cm(row, HC + c)) = hi;
          *(float4*)(a_lo + cm(row, HC + c)) = lo;
        }
        {  // B rows 2 jj = [Br | -Bi], 2 jj + 1 = [Bi | Br]
          const int jj = row;
          const float4 vr = make_float4(rb[u][0].x, rb[u][1].x, rb[u][2].x, rb[u][3].x);
          const float4 vi = make_float4(rb[u][0].y, rb[u][1].y, rb[u][2].y, rb[u][3].y);
          split4(vr, hi, lo);
          *(float4*)(b_hi + cm(2 * jj, c)) = hi;
          *(float4*)(b_lo + cm(2 * jj, c)) = lo;
          *(float4*)(b_hi + cm(2 * jj + 1, HC + c)) = hi;
          *(float4*)(b_lo + cm(2 * jj + 1, HC + c)) = lo;
          split4(vi, hi, lo);
          *(float4*)(b_hi + cm(2 * jj + 1, c)) = hi;
          *(float4*)(b_lo + cm(2 * jj + 1, c)) = lo;
          hi = make_float4(-hi.x, -hi.y, -hi.z, -hi.w);  // the split of -x is -(split of x)
          lo = make_float4(-lo.x, -lo.y, -lo.z, -lo.w);
          *(float4*)(b_hi + cm(2 * jj, HC + c)) = hi;
          *(float4*)(b_lo + cm(2 * jj, HC + c)) = lo;
        }
      }
      fence_proxy_async_smem();  // the operand stores, before the tensor cores read them
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (tid == 0) {
        const int b = n & 1;
        if (n >= 2) mbar_wait(&acc_free[b], ((n - 2) >> 1) & 1);  // the drain of tile n - 2 is done
        tc_fence_after();
        const unsigned d = tmem + (unsigned)b * (2 * RT_NC);
        const unsigned sa_hi = smem_u32(a_hi), sa_lo = smem_u32(a_lo), sb_hi = smem_u32(b_hi), sb_lo = smem_u32(b_lo);
#pragma unroll
        for (int kk = 0; kk < Kp / 8; ++kk) {
          const unsigned ko = (unsigned)kk * 256u;  // two 16-byte chunks per K = 8 step
          umma_tf32(d, umma_desc(sa_lo + ko, 128, SBO), umma_desc(sb_hi + ko, 128, SBO), kk > 0);
          umma_tf32(d, umma_desc(sa_hi + ko, 128, SBO), umma_desc(sb_lo + ko, 128, SBO), 1);
          umma_tf32(d, umma_desc(sa_hi + ko, 128, SBO), umma_desc(sb_hi + ko, 128, SBO), 1);
        }
        umma_commit(&mma_done[b]);
      }
      __syncwarp();
      if (t + gridDim.x < ntiles) fetch(t + gridDim.x);
    }
  } else {
    // ---------------- TMEM drain: a warp owns the 32 accumulator lanes (rows) of its quarter (warp % 4);
    // each 32-column chunk goes through a padded shared-memory transpose so every store instruction writes
    // four full 128-byte row segments
    const int q = warp & 3;
    float* tb = tbuf + q * (32 * 36);
    int n = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++n) {
      int f, i0, j0;
      tile_origin(t, f, i0, j0);
      const int b = n & 1;
      mbar_wait(&mma_done[b], (n >> 1) & 1);
      tc_fence_after();
      const unsigned taddr = tmem + ((unsigned)(32 * q) << 16) + (unsigned)b * (2 * RT_NC);
      float2* Xf = X + (size_t)f * nx * ny;
#pragma unroll 1
      for (int c = 0; c < 2 * RT_NC / 32; c += 2) {
        unsigned v[2][32];
        RT_LD32(taddr + 32 * c, v[0]);
        RT_LD32(taddr + 32 * (c + 1), v[1]);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            *(float4*)(tb + lane * 36 + 4 * e) = make_float4(__uint_as_float(v[h][4 * e]), __uint_as_float(v[h][4 * e + 1]),
                                                              __uint_as_float(v[h][4 * e + 2]), __uint_as_float(v[h][4 * e + 3]));
          __syncwarp();
          const int jc = j0 + 16 * (c + h) + 2 * (lane & 7);  // this lane's two complex columns
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int rr = 4 * k + (lane >> 3), i = i0 + 32 * q + rr;
            const float4 w = *(const float4*)(tb + rr * 36 + 4 * (lane & 7));
            if (i < nx) {
              float2* xr = Xf + (size_t)i * ny;
              if (vec && jc + 1 < ny) {
                *(float4*)(xr + jc) = w;
              } else {
                if (jc < ny) xr[jc] = make_float2(w.x, w.y);
                if (jc + 1 < ny) xr[jc + 1] = make_float2(w.z, w.w);
              }
            }
          }
          __syncwarp();
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_free[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

template <int KC>
static int recon_tc_launch(cudaStream_t st, int frames, int nx, int ny, int R, const float2* a, const float2* b,
                           const float2* g, float2* x, int vec) {
  const size_t smb = (size_t)(RT_M + 2 * RT_NC) * 4 * KC * 4 * 2 + 64 + 8 * 2 * KC + 4 * 32 * 36 * 4;
  static size_t cfg[TT_MAXDEV] = {0};
  static int sms[TT_MAXDEV] = {0};
  int dev = 0;
  TT_CUDA_TRY(cudaGetDevice(&dev));
  const int d = dev < TT_MAXDEV ? dev : 0;
  TT_CUDA_TRY(tt_smem_attr((const void*)recon_tc_kernel<KC>, smb, cfg));
  if (sms[d] == 0) TT_CUDA_TRY(cudaDeviceGetAttribute(&sms[d], cudaDevAttrMultiProcessorCount, dev));
  const long long tiles = (long long)frames * ((nx + RT_M - 1) / RT_M) * ((ny + RT_NC - 1) / RT_NC);
  if (tiles == 0) return TT_OK;
  const int grid = (int)(tiles < sms[d] ? tiles : sms[d]);
  recon_tc_kernel<KC><<<grid, RT_NT, smb, st>>>(frames, nx, ny, R, a, b, g, x, vec);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

// called by tt_reconstruct (tt_recon.cu) for rank <= 32; returns TT_EUNSUPPORTED above
int tt_recon_tc(cudaStream_t st, int frames, int nx, int ny, int rank, const float2* a, const float2* b,
                const float2* g, float2* x, int vec) {
  switch ((rank + 7) / 8) {
    case 1: return recon_tc_launch<4>(st, frames, nx, ny, rank, a, b, g, x, vec);
    case 2: return recon_tc_launch<8>(st, frames, nx, ny, rank, a, b, g, x, vec);
    case 3: return recon_tc_launch<12>(st, frames, nx, ny, rank, a, b, g, x, vec);
    case 4: return recon_tc_launch<16>(st, frames, nx, ny, rank, a, b, g, x, vec);
    default: return TT_EUNSUPPORTED;
  }
}
