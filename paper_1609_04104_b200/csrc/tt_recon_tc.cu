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
// One persistent CTA per SM (512 TMEM columns: two 128 x 256 fp32 accumulators); tiles are handed out by a
// global counter (the first tile of a CTA is its block index), so CTAs that become resident late - the
// reconstruction of a block of frames overlaps the tracking of the next one, which holds most SMs - take
// only what is left, and the CTAs on the free SMs keep working meanwhile. Warps 0-3 stage a tile's
// operands (fp32 loads, gamma scaling, the TF32 split) into shared memory in the no-swizzle K-major core-
// matrix layout, thread 0 then issues the tile's 3 Kp/8 tcgen05.mma (M 128, N 256, K 8) into accumulator
// n % 2 and commits them to an mbarrier; warps 4-7 drain the other accumulator with tcgen05.ld (one output
// row per thread, 128 contiguous bytes per 32 columns) while the next tile is staged and multiplied. The
// kernel is bound by the HBM writes of the frames.
#include <cuda.h>
#include <stdlib.h>
#include <string.h>

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
                                                            int vec, unsigned* __restrict__ tile_ctr,
                                                            const __grid_constant__ CUtensorMap xmap) {
  constexpr int Kp = 4 * KC, HC = KC / 2;  // HC: chunks per half (re | im), 4 complex per chunk
  constexpr unsigned SBO = KC * 128;        // bytes per 8-row group (all its K chunks, 128 B each)
  constexpr unsigned A_BYTES = RT_M * Kp * 4, B_BYTES = 2 * RT_NC * Kp * 4;
  constexpr int NOB = KC <= 12 ? 4 : 2;  // output boxes in flight per drain warp
  constexpr unsigned OB_BYTES = 4 * NOB * 4096 > 4 * 32 * 36 * 4 ? 4 * NOB * 4096 : 4 * 32 * 36 * 4;
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* a_hi = sm;
  unsigned char* a_lo = sm + A_BYTES;
  unsigned char* b_hi = sm + 2 * A_BYTES;
  unsigned char* b_lo = b_hi + B_BYTES;
  // drain staging: with a tensor map (vec) NOB 4 KB boxes per drain warp, 1024-byte aligned (128-byte swizzle);
  // without one, one padded transpose buffer per warp in the same space
  unsigned char* obuf = b_lo + B_BYTES;
  float* tbuf = (float*)obuf;  // 4 warps x 32 rows x 36 floats
  unsigned long long* mma_done = (unsigned long long*)(obuf + OB_BYTES);  // [2], one arrival (the commit)
  unsigned long long* acc_free = mma_done + 2;                             // [2], 128 arrivals (the drain)
  unsigned* tmem_slot = (unsigned*)(acc_free + 2);
  unsigned long long* tq_full = acc_free + 4;      // [4], one arrival: tile-queue entry n is in tq[n % 4]
  volatile int* tq = (volatile int*)(tq_full + 4);  // [4] tile of entry n (-1: no more tiles)
  volatile int* bc = tq + 4;                       // [2] the staging warps' next tile (written by thread 0)
  float2* gs = (float2*)(bc + 4);                  // the tile's gamma (2 KC values)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    mbar_init(&mma_done[0], 1);
    mbar_init(&mma_done[1], 1);
    mbar_init(&acc_free[0], 128);
    mbar_init(&acc_free[1], 128);
    for (int i = 0; i < 4; ++i) mbar_init(&tq_full[i], 1);
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
  const int ntiles = frames * per_frame;  // < 2^31 (checked at the launch)
  auto tile_origin = [&](int t, int& f, int& i0, int& j0) {
    f = t / per_frame;
    const int rem = t - f * per_frame;
    i0 = (rem / tiles_j) * RT_M;
    j0 = (rem % tiles_j) * RT_NC;
  };
  // byte offset of (row, 16-byte K chunk) in the core-matrix layout
  auto cm = [&](int row, int chunk) -> unsigned {
    return (unsigned)(row >> 3) * SBO + (unsigned)chunk * 128u + (unsigned)(row & 7) * 16u;
  };

  if (warp < 4) {
    // ---------------- staging + MMA issue. Thread = one operand row (A row tid, B row tid of the tile), its
    // HC chunks of 4 complex in turn: a quarter warp's 16-byte stores of one chunk fill one 128-byte core-
    // matrix row group (no bank conflicts). The next tile's raw operands are loaded into registers right
    // after a tile's MMAs are issued (they land while the tensor cores run); the split waits only for the
    // MMAs that still read shared memory.
    float2 ra[HC][4], rb[HC][4], rg = make_float2(0.f, 0.f);
    const bool ldvec = (R % 4 == 0) && (((size_t)A | (size_t)B) & 15) == 0;
    auto fetch = [&](int t) {
      int f, i0, j0;
      tile_origin(t, f, i0, j0);
      const int i = i0 + tid, j = j0 + tid;
      const float2* Ar = A + ((size_t)f * nx + (i < nx ? i : 0)) * R;
      const float2* Br = B + ((size_t)f * ny + (j < ny ? j : 0)) * R;
#pragma unroll
      for (int u = 0; u < HC; ++u) {
        if (ldvec) {
          float4 p0 = make_float4(0.f, 0.f, 0.f, 0.f), p1 = p0, q0 = p0, q1 = p0;
          if (4 * u < R) {
            if (i < nx) {
              p0 = __ldg((const float4*)(Ar + 4 * u));
              p1 = __ldg((const float4*)(Ar + 4 * u) + 1);
            }
            if (j < ny) {
              q0 = __ldg((const float4*)(Br + 4 * u));
              q1 = __ldg((const float4*)(Br + 4 * u) + 1);
            }
          }
          ra[u][0] = make_float2(p0.x, p0.y), ra[u][1] = make_float2(p0.z, p0.w);
          ra[u][2] = make_float2(p1.x, p1.y), ra[u][3] = make_float2(p1.z, p1.w);
          rb[u][0] = make_float2(q0.x, q0.y), rb[u][1] = make_float2(q0.z, q0.w);
          rb[u][2] = make_float2(q1.x, q1.y), rb[u][3] = make_float2(q1.z, q1.w);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = 4 * u + e;
            ra[u][e] = (i < nx && r < R) ? __ldg(Ar + r) : make_float2(0.f, 0.f);
            rb[u][e] = (j < ny && r < R) ? __ldg(Br + r) : make_float2(0.f, 0.f);
          }
        }
      }
      if (tid < R) rg = __ldg(gamma + (size_t)f * R + tid);
    };
    // B2 rows 2 jj = [Br | -Bi] and 2 jj + 1 = [Bi | Br]: a value goes to an even row (16-byte slots 0, 2, 4, 6
    // of a row group) and to an odd one (slots 1, 3, 5, 7). In each store instruction the lanes with jj % 8 < 4
    // write the even row and the others the odd one, so a quarter warp covers all eight slots.
    const int jj = tid;
    const bool ev = (jj & 4) == 0;
    int n = 0;
    // thread 0 draws the tiles two ahead (tile n + 1 is fetched during tile n's MMAs): grid <= ntiles
    int tnext = 0;
    if (tid == 0) tnext = (int)gridDim.x + (int)atomicAdd(tile_ctr, 1u);
    fetch(blockIdx.x);
    for (int t = blockIdx.x; t < ntiles; ++n) {
      if (n >= 1) mbar_wait(&mma_done[(n - 1) & 1], ((n - 1) >> 1) & 1);  // the previous tile's MMAs read smem
      if (tid < 2 * KC) gs[tid] = rg;  // RP = 2 KC gamma values (zeros past R)
      if (tid == 0) {
        bc[n & 1] = tnext;
        tq[n & 3] = t;  // the drain warps are at most two tiles behind: slot (n - 4) % 4 is free
        mbar_arrive(&tq_full[n & 3]);
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      const int tn = bc[n & 1];
#pragma unroll
      for (int c = 0; c < HC; ++c) {
        float4 hi, lo;
        {  // A' = A diag(gamma): row tid, re chunk c and im chunk HC + c
          float2 v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) v[e] = cmul(ra[c][e], gs[4 * c + e]);
          split4(make_float4(v[0].x, v[1].x, v[2].x, v[3].x), hi, lo);
          *(float4*)(a_hi + cm(tid, c)) = hi;
          *(float4*)(a_lo + cm(tid, c)) = lo;
          split4(make_float4(v[0].y, v[1].y, v[2].y, v[3].y), hi, lo);
          *(float4*)(a_hi + cm(tid, HC + c)) = hi;
          *(float4*)(a_lo + cm(tid, HC + c)) = lo;
        }
        {
          const float4 vr = make_float4(rb[c][0].x, rb[c][1].x, rb[c][2].x, rb[c][3].x);
          const float4 vi = make_float4(rb[c][0].y, rb[c][1].y, rb[c][2].y, rb[c][3].y);
          const unsigned e_re = cm(2 * jj, c), o_re = cm(2 * jj + 1, HC + c);  // Br: even row re half, odd row im half
          const unsigned o_im = cm(2 * jj + 1, c), e_im = cm(2 * jj, HC + c);  // Bi: odd row re half, -Bi: even row im half
          split4(vr, hi, lo);
          *(float4*)(b_hi + (ev ? e_re : o_re)) = hi;
          *(float4*)(b_lo + (ev ? e_re : o_re)) = lo;
          *(float4*)(b_hi + (ev ? o_re : e_re)) = hi;
          *(float4*)(b_lo + (ev ? o_re : e_re)) = lo;
          split4(vi, hi, lo);
          // the split of -x is -(split of x)
          const float4 nhi = make_float4(-hi.x, -hi.y, -hi.z, -hi.w), nlo = make_float4(-lo.x, -lo.y, -lo.z, -lo.w);
          *(float4*)(b_hi + (ev ? e_im : o_im)) = ev ? nhi : hi;
          *(float4*)(b_lo + (ev ? e_im : o_im)) = ev ? nlo : lo;
          *(float4*)(b_hi + (ev ? o_im : e_im)) = ev ? hi : nhi;
          *(float4*)(b_lo + (ev ? o_im : e_im)) = ev ? lo : nlo;
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
        tnext = tn < ntiles ? (int)gridDim.x + (int)atomicAdd(tile_ctr, 1u) : ntiles;
      }
      __syncwarp();
      if (tn < ntiles) fetch(tn);
      t = tn;
    }
    if (tid == 0) {
      tq[n & 3] = -1;
      mbar_arrive(&tq_full[n & 3]);
    }
  } else {
    // ---------------- TMEM drain: a warp owns the 32 accumulator lanes (rows) of its quarter (warp % 4).
    // A 32-column chunk (one output row segment of 128 bytes per lane) is written to a 4 KB shared-memory box
    // in the 128-byte swizzle (16-byte slot e of row r at slot e ^ (r % 8): conflict-free) and leaves as ONE
    // bulk tensor store (TMA; rows and columns past the frame are clipped by the tensor map), NOB boxes in
    // flight per warp; the next two chunks leave TMEM while the current ones are stored. Without a tensor map
    // (odd ny or an unaligned output) the chunks go through a padded transpose and plain stores.
    const int q = warp & 3;
    float* tb = tbuf + q * (32 * 36);
    unsigned char* ob = obuf + q * (NOB * 4096);
    unsigned box = 0;  // boxes issued by this warp
    // the frames are written once and read by nobody on the device soon: evict-first in L2, so the stream of
    // output lines does not displace the tracking clusters' exchange buffers and factor history
    unsigned long long l2_first;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(l2_first));
    for (int n = 0;; ++n) {
      mbar_wait(&tq_full[n & 3], (n >> 2) & 1);
      const int t = tq[n & 3];
      if (t < 0) break;
      int f, i0, j0;
      tile_origin(t, f, i0, j0);
      const int b = n & 1;
      mbar_wait(&mma_done[b], (n >> 1) & 1);
      tc_fence_after();
      const unsigned taddr = tmem + ((unsigned)(32 * q) << 16) + (unsigned)b * (2 * RT_NC);
      float2* Xf = X + (size_t)f * nx * ny;
      unsigned v[2][2][32];  // [ping-pong][chunk of the pair][column]
      RT_LD32(taddr, v[0][0]);
      RT_LD32(taddr + 32, v[0][1]);
#pragma unroll
      for (int c = 0; c < 2 * RT_NC / 32; c += 2) {
        const int pp = (c >> 1) & 1;
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (c + 2 < 2 * RT_NC / 32) {
          RT_LD32(taddr + 32 * (c + 2), v[pp ^ 1][0]);
          RT_LD32(taddr + 32 * (c + 3), v[pp ^ 1][1]);
        }
        if (vec) {
          // the pair's two boxes: the bulk stores that last read them are done reading (lane 0 owns the
          // warp's bulk groups, one group per pair)
          unsigned char* o = ob + (box % NOB) * 4096;  // NOB is even: the pair is contiguous
          box += 2;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(NOB / 2 - 1) : "memory");
          __syncwarp();
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int e = 0; e < 8; ++e)
              *(float4*)(o + h * 4096 + lane * 128 + ((e ^ (lane & 7)) << 4)) =
                  make_float4(__uint_as_float(v[pp][h][4 * e]), __uint_as_float(v[pp][h][4 * e + 1]),
                              __uint_as_float(v[pp][h][4 * e + 2]), __uint_as_float(v[pp][h][4 * e + 3]));
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (j0 + 16 * (c + h) < ny)
                asm volatile(
                    "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;\n" ::
                        "l"(&xmap),
                    "r"(2 * (j0 + 16 * (c + h))), "r"(i0 + 32 * q), "r"(f), "r"(smem_u32(o + h * 4096)), "l"(l2_first)
                    : "memory");
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
          }
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              *(float4*)(tb + lane * 36 + 4 * e) =
                  make_float4(__uint_as_float(v[pp][h][4 * e]), __uint_as_float(v[pp][h][4 * e + 1]),
                              __uint_as_float(v[pp][h][4 * e + 2]), __uint_as_float(v[pp][h][4 * e + 3]));
            __syncwarp();
            const int jc = j0 + 16 * (c + h) + 2 * (lane & 7);  // this lane's two complex columns
#pragma unroll 1
            for (int k = 0; k < 8; ++k) {
              const int rr = 4 * k + (lane >> 3), i = i0 + 32 * q + rr;
              const float4 w = *(const float4*)(tb + rr * 36 + 4 * (lane & 7));
              if (i < nx) {
                float2* xr = Xf + (size_t)i * ny;
                if (jc < ny) xr[jc] = make_float2(w.x, w.y);
                if (jc + 1 < ny) xr[jc + 1] = make_float2(w.z, w.w);
              }
            }
            __syncwarp();
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_free[b]);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");  // the warp's stores are complete
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (the library links cudart only)
typedef CUresult (*tensormap_encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                        const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                        CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static tensormap_encode_fn tensormap_encoder() {
  static tensormap_encode_fn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (tensormap_encode_fn)p;
  }
  return fn;
}

// The tile counter of one launch: a slot of a per-device ring, zeroed on the launch's stream ahead of the
// kernel (a memset node under graph capture). RT_CTRS launches can be in flight per device.
#define RT_CTRS 1024
static cudaError_t recon_tile_counter(int d, cudaStream_t st, unsigned** out) {
  static unsigned* ring[TT_MAXDEV] = {nullptr};
  static unsigned next[TT_MAXDEV] = {0};
  if (!ring[d]) {
    cudaError_t e = cudaMalloc((void**)&ring[d], RT_CTRS * sizeof(unsigned));
    if (e != cudaSuccess) return e;
  }
  unsigned* c = ring[d] + (__sync_fetch_and_add(&next[d], 1u) % RT_CTRS);
  *out = c;
  return cudaMemsetAsync(c, 0, sizeof(unsigned), st);
}

template <int KC>
static int recon_tc_launch(cudaStream_t st, int frames, int nx, int ny, int R, const float2* a, const float2* b,
                           const float2* g, float2* x, int vec) {
  const size_t ob = (KC <= 12 ? 4 : 2) * 4 * 4096;
  const size_t smb = (size_t)(RT_M + 2 * RT_NC) * 4 * KC * 4 * 2 + (ob > 4 * 32 * 36 * 4 ? ob : 4 * 32 * 36 * 4) + 128 +
                     8 * 2 * KC;
  static size_t cfg[TT_MAXDEV] = {0};
  static int sms[TT_MAXDEV] = {0};
  int dev = 0;
  TT_CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= TT_MAXDEV) return tt_fail(TT_EUNSUPPORTED, "tt_reconstruct: device index %d", dev);
  const int d = dev;
  TT_CUDA_TRY(tt_smem_attr((const void*)recon_tc_kernel<KC>, smb, cfg));
  if (sms[d] == 0) TT_CUDA_TRY(cudaDeviceGetAttribute(&sms[d], cudaDevAttrMultiProcessorCount, dev));
  const long long tiles = (long long)frames * ((nx + RT_M - 1) / RT_M) * ((ny + RT_NC - 1) / RT_NC);
  if (tiles == 0) return TT_OK;
  if (tiles > 0x7fffffffLL - 4096) return tt_fail(TT_EUNSUPPORTED, "tt_reconstruct: more than 2^31 output tiles");
  int grid = (int)(tiles < sms[d] ? tiles : sms[d]);
  if (const char* e = getenv("TT_RECON_MAXCTAS")) {  // experiment hook: fewer persistent CTAs
    const int m = atoi(e);
    if (m > 0 && m < grid) grid = m;
  }
  unsigned* ctr = nullptr;
  TT_CUDA_TRY(recon_tile_counter(d, st, &ctr));
  // the output as a 3-D fp32 tensor (2 ny, nx, frames) for the drain's bulk tensor stores: 32 x 32 boxes,
  // 128-byte swizzle. Needs 16-byte row strides (even ny) and base; otherwise the plain-store drain runs.
  CUtensorMap xmap;
  memset(&xmap, 0, sizeof(xmap));
  if (vec) {
    tensormap_encode_fn enc = tensormap_encoder();
    if (!enc) return tt_fail(TT_EUNSUPPORTED, "tt_reconstruct: cuTensorMapEncodeTiled is not available from this driver");
    const cuuint64_t gdim[3] = {(cuuint64_t)2 * ny, (cuuint64_t)nx, (cuuint64_t)frames};
    const cuuint64_t gstr[2] = {(cuuint64_t)ny * 8, (cuuint64_t)nx * ny * 8};
    const cuuint32_t box[3] = {32, 32, 1}, estr[3] = {1, 1, 1};
    const CUresult r = enc(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)x, gdim, gstr, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return tt_fail(TT_ECUDA, "tt_reconstruct: cuTensorMapEncodeTiled failed (%d)", (int)r);
  }
  recon_tc_kernel<KC><<<grid, RT_NT, smb, st>>>(frames, nx, ny, R, a, b, g, x, vec, ctr, xmap);
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
