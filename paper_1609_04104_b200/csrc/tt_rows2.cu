// Mirrored-state persistent online step for Cartesian row masks (sm_100a): the small-image form of the
// rows kernel (tt_rows.cu) with two cluster barriers per frame instead of four and no L2 exchanges.
//
// Reference path (tensortrack, /root/reference/pkg/src/tensortrack), as tt_rows.cu:
//   tracker.track_step (FourierMask rows)       tracker.py:367-411
//   sampler.row_scores + draw_samples           sampler.py:77-170
//   experiment.run_adaptive per-frame body      experiment.py:482-530
//
// Same k-space formulation as tt_rows.cu: state Ah = F_x A, Bh = F_y B; for sampled rows S and
// data Y (S x Ny): GA = Ah_S^H Ah_S, GB = Bh^H Bh, W = Y^T conj(Ah_S), Z = Y conj(Bh), gamma = (GA.*GB + lam
// I)^-1 h, P_S = Z - Ah_S diag(gamma) GB^T, Q = W - Bh diag(gamma) GA^T, k-space updates.
//
// Layout (one thread-block cluster of CL CTAs per slice): every CTA holds a MIRROR of the whole Ah (nx x R
// fp32, identical bits in every CTA) and its own rows J_c of Bh (= the Y columns J_c). Per frame:
//   (1) GB: CTA c sums its block of packed entries over the CTAs' partials (received last frame) and
//       broadcasts them into every CTA (DSMEM stores);
//   (2) column norms, (3) row scores of all rows and the draw, (5) Ah_S and GA: redundant in every CTA
//       from the mirror (no exchange: the informative draw needs no barrier at all);
//   (4)/(6) Y rows of own columns by bulk copy (TMA), W = Y_J^T conj(Ah_S), the Z partial over own columns
//       scattered by sampled-row block to the block's owner, h and ||Y||^2 partials broadcast;
//   B1 (cluster barrier: release/acquire orders the DSMEM stores)
//   (8) fp64 Gram + ridge solve (redundant), cost, step;
//   (9) CTA c updates its block of sampled rows (P) and stores the new rows into every CTA's mirror;
//       (10) non-sampled rows scale by the step's cfac locally; (11) own Bh rows (Q);
//       (12) GB partials of the updated own Bh rows scattered to the entry owners;
//   B2; (15) factor history.
// Every cross-CTA value lands in the consumer's shared memory before the barrier that orders it; the
// only global traffic is the truth rows (Y), the resident state at launch start/end and the outputs.
// Used when the mirror fits shared memory (tt_rows_mirror_fits; config 2 and 3 shapes), otherwise
// tt_rows.cu's kernel runs. The arithmetic of every product and sum follows tt_rows.cu's order, except the
// column norms (summed over all rows in one pass here), so the two agree to rounding.

#include <cooperative_groups.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "tt_block.cuh"
#include "tt_mirror.cuh"

namespace cg = cooperative_groups;

#define MR_NT 256
constexpr int MR_ZG = 4;  // 8-row M blocks per DMMA work item


static inline size_t mr_al16(size_t x) { return (x + 15) & ~(size_t)15; }
// K parts of the GB partial GEMM (one DMMA item per warp: ceil(R / 4) column blocks per part)
__host__ __device__ inline int mr_gb_parts(int R) {
  const int nb = (R + 3) / 4;
  return nb >= 8 ? 1 : 8 / nb;
}

static bool mirror_make_plan(int nx, int ny, int R, int Smax, int CL, MirrorPlan* p) {
  const size_t maxsmem = 227 * 1024 - 512;  // the opt-in limit less the kernel's static __shared__ words
  if (R < 1 || R > 32 || CL < 1 || CL > 16 || nx > 4 * MR_NT) return false;
  p->CL = CL;
  p->nJm = (ny + CL - 1) / CL;
  p->Rp = R * (R + 1) / 2;
  p->sblk = (Smax + CL - 1) / CL;
  p->eblk = (p->Rp + CL - 1) / CL;
  // Y tile row stride = 4 (mod 16) complex: 16 B aligned rows for the bulk copies, DMMA fragments conflict-free
  p->ysr = ((p->nJm + 11) & ~15) + 4;
  // padded row strides of the DMMA operands (complex elements): fp64 rows 2 (mod 8) apart put the 4 k-rows of
  // a B fragment (and of a transposed A fragment) on disjoint banks; fp32 row-major A rows 4 (mod 16) apart
  p->rs64 = R;
  while (p->rs64 % 8 != 2 && p->rs64 % 8 != 6) ++p->rs64;
  p->rs32 = R;
  while (p->rs32 % 16 != 4 && p->rs32 % 16 != 12) ++p->rs32;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = mr_al16(o + bytes);
    return (int)at;
  };
  p->o_ahf = take(8 * (size_t)nx * R);
  p->o_bh64 = take(16 * (size_t)p->nJm * p->rs64);
  // U: the Y tile | the draw's probabilities + CDF | column-norm partials | h partials | GB partial tiles
  size_t u = 8 * (size_t)Smax * p->ysr;
  if (16 * (size_t)nx > u) u = 16 * (size_t)nx;
  if (16 * (size_t)MR_NT > u) u = 16 * (size_t)MR_NT;
  const size_t gbp = 16 * (size_t)R * R * mr_gb_parts(R);  // the GB partial GEMM's K parts
  if (gbp > u) u = gbp;
  p->o_u = take(u);
  p->o_ahs = take(16 * (size_t)Smax * p->rs64);
  p->o_wacc = take(16 * (size_t)p->nJm * R);
  p->o_zrecv = take(16 * (size_t)CL * p->sblk * R);
  p->o_hrecv = take(16 * (size_t)CL * R);
  p->o_ynrecv = take(8 * (size_t)CL);
  p->o_gbrecv = take(16 * (size_t)CL * p->eblk);
  p->o_gbfull = take(16 * (size_t)p->Rp);
  p->o_G = take(16 * (size_t)p->Rp);
  p->o_gaf = take(16 * (size_t)R * p->rs64);
  p->o_gbf = take(16 * (size_t)R * p->rs64);
  p->o_vec = take(16 * 3 * (size_t)R + 8 * 4 * (size_t)R + 8 * (size_t)R + 8 * 16);
  p->o_tab = take(2 * (size_t)p->Rp);
  p->o_colb = take(64 * (size_t)(R + 1));
  p->o_flags = take(4 * (size_t)nx);
  p->o_rows = take(4 * (size_t)Smax);
  p->o_forced = take(4 * (size_t)Smax);
  p->o_usm = take(8 * (size_t)Smax);
  p->o_red = take(8 * 64);
  p->o_zown = take(4 * (size_t)Smax);
  p->o_eown = take(4 * (size_t)p->Rp);
  p->smem = (int)o;
  return o <= maxsmem;
}

// ---------------------------------------------------------------- cold paths (out of line)
// Static row table validation: range and duplicates (observation.py:41-55), as tt_rows.cu.
static __device__ __noinline__ int mr_load_static_rows(const tt_rows_args& a, int f, int s, int* rows, int* flags,
                                                       int* sh_err) {
  const int tid = threadIdx.x, NT = blockDim.x, nx = a.nx, Smax = a.max_rows;
  const int* tab_rows = a.rows_tab + ((size_t)f * a.nslices + s) * Smax;
  const int cnt = a.rows_cnt[(size_t)f * a.nslices + s];
  for (int i = tid; i < nx; i += NT) flags[i] = 0;
  __syncthreads();
  int S = 0;
  if (cnt < 0 || cnt > Smax) {
    if (tid == 0) atomicOr(sh_err, TT_ST_OVERFLOW);
  } else {
    for (int k = tid; k < cnt; k += NT) {
      const int i = tab_rows[k];
      rows[k] = i;
      if (i < 0 || i >= nx) atomicOr(sh_err, TT_ST_BADROW);
      else if (atomicAdd(&flags[i], 1) > 0) atomicOr(sh_err, TT_ST_DUPROW);
    }
    S = cnt;
  }
  __syncthreads();
  if (*sh_err & (TT_ST_BADROW | TT_ST_DUPROW | TT_ST_OVERFLOW)) S = 0;
  return S;
}

// The informative rows of one frame from the raw row scores s (in p, nx entries; sampler.py:77-92,
// :146-169), identical in every CTA: the blended CDF in closed form from one block scan, one branch-free
// binary search per draw, the union with the forced rows by a block scan (np.union1d); a uniform within
// 1e-12 of a CDF edge redoes the frame over numpy's sequential cumsum; without replacement the sequential
// renormalised draws (weighted_draw_without_replacement). p is overwritten by the probabilities; the
// rows land in rows[0..S) ascending. Same arithmetic as tt_rows.cu's draw. Returns S in every thread.
static __device__ __noinline__ int mr_draw_rows(double* p, double* cdf, int* flags, int* rows, int nx, int ndraw,
                                                const double* usm, const int* forced, int nforced, unsigned fmask,
                                                int top, double beta, bool wor, double* red) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5;
  __shared__ int s_S, s_amb, s_idx;
  const double inx = 1.0 / (double)nx;
  if (tid == 0) s_amb = 0;
  __syncthreads();
  if (!wor) {
    const int ipt = (nx + NT - 1) / NT;
    const int r0 = min(nx, tid * ipt), r1 = min(nx, r0 + ipt);
    double sv[4], cv[4];
    double loc = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      sv[j] = (j < ipt && r0 + j < r1) ? p[r0 + j] : 0.0;
      loc += sv[j];
    }
    double S1;
    double run = block_excl_scan_dbl(loc, red, S1);
    const double w1 = (1.0 - beta) * fast_rcp(S1), w0 = beta * inx;
    const double il = fast_rcp(fma(w1, S1, w0 * (double)nx));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j < ipt && r0 + j < r1) {
        run += sv[j];
        cv[j] = fma(w1, run, w0 * (double)(r0 + j + 1)) * il;
        cdf[r0 + j] = cv[j];
        p[r0 + j] = fma(sv[j], w1, w0);  // probabilities for the exact fallback
        flags[r0 + j] = 0;
      }
    }
    __syncthreads();
    for (int m = tid; m < ndraw; m += NT) {
      const double u = usm[m];
      int pos = -1;  // last index with cdf <= u
      for (int step = top; step > 0; step >>= 1) {
        const int cand = pos + step;
        if (cand < nx && cdf[cand] <= u) pos = cand;
      }
      const int idx = min(pos + 1, nx - 1);
      const double lo = idx > 0 ? cdf[idx - 1] : -1.0;
      if (u - lo <= 1e-12 || (idx < nx - 1 && cdf[idx] - u <= 1e-12)) s_amb = 1;
      flags[idx] = 1;
    }
    __syncthreads();
    if (!s_amb) {
      unsigned hit = fmask;  // forced lines (np.union1d)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < ipt && r0 + j < r1 && flags[r0 + j]) hit |= 1u << j;
      int tot;
      int o = block_excl_scan_int(__popc(hit), (int*)red, tot);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (hit & (1u << j)) rows[o++] = r0 + j;
      __syncthreads();
      return tot;
    }
  } else {
    // probabilities of the sequential draws: the raw scores normalised and blended (fixed-order sum)
    double S1;
    block_sum_range(p, nx, red, S1);
    const double w1 = (1.0 - beta) / S1, w0 = beta / (double)nx;
    for (int i = tid; i < nx; i += NT) p[i] = fma(p[i], w1, w0);
    __syncthreads();
  }
  if (wor) {
    for (int i = tid; i < nx; i += NT) flags[i] = 0;
    __syncthreads();
    for (int m = tid; m < nforced; m += NT) {
      const int fr = forced[m];
      if (fr >= 0 && fr < nx) p[fr] = 0.0;
    }
    __syncthreads();
    for (int m = 0; m < ndraw; ++m) {
      for (int exact = 0; exact < 2; ++exact) {
        block_cumsum(p, cdf, nx, exact != 0, red);
        if (tid == 0) {
          const double total = cdf[nx - 1];
          const double u = usm[m] * total;
          const int idx = upper_bound_d(cdf, nx, u);
          const double lo = idx > 0 ? cdf[idx - 1] : -1.0;
          const double hi = idx < nx ? cdf[idx] : 2.0 * total + 1.0;
          const double tol = 1e-12 * (total > 0.0 ? total : 1.0);
          s_amb = (!exact && (u - lo <= tol || hi - u <= tol)) ? 1 : 0;
          s_idx = idx < nx - 1 ? idx : nx - 1;
        }
        __syncthreads();
        const int amb = s_amb;
        __syncthreads();
        if (!amb) break;
      }
      if (tid == 0) {
        flags[s_idx] = 1;
        p[s_idx] = 0.0;
      }
      __syncthreads();
    }
  } else {
    // a uniform within 1e-12 of a CDF boundary: numpy's sequential cumsum, cdf /= cdf[-1], redo the draws
    if (tid == 0) {
      double cacc = 0.0;
      for (int i = 0; i < nx; ++i) {
        cacc += p[i];
        cdf[i] = cacc;
      }
    }
    __syncthreads();
    const double last = cdf[nx - 1];
    __syncthreads();
    for (int i = tid; i < nx; i += NT) {
      cdf[i] = cdf[i] / last;
      flags[i] = 0;
    }
    __syncthreads();
    for (int m = tid; m < ndraw; m += NT) {
      const int idx = upper_bound_d(cdf, nx, usm[m]);
      flags[idx < nx ? idx : nx - 1] = 1;
    }
    __syncthreads();
  }
  if (warp == 0) {  // forced lines, then compaction -> sorted unique rows (np.union1d)
    for (int m = lane; m < nforced; m += 32) {
      const int fr = forced[m];
      if (fr >= 0 && fr < nx) flags[fr] = 1;
    }
    __syncwarp();
    const int chunk = (nx + 31) / 32;
    const int q0 = min(nx, lane * chunk), q1 = min(nx, q0 + chunk);
    int cnt = 0;
    for (int i = q0; i < q1; ++i) cnt += flags[i];
    int x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    int o = x - cnt;
    for (int i = q0; i < q1; ++i)
      if (flags[i]) rows[o++] = i;
    if (lane == 31) s_S = x;
  }
  __syncthreads();
  return s_S;
}

// GB partial over this CTA's Bh rows on the fp64 tensor cores: C = Bh_J^T conj(Bh_J) (so C[q][r] = GB[r][q]),
// K = the own rows split in mr_gb_parts(R) parts summed in order, each packed entry delivered into its
// owner's gbrecv slot c (eown: owner << 16 | position in the owner's block).
struct MrEpiParts {
  double2* dst;
  int R;
  TT_DEV void operator()(int m, int n, int ks, double2 v) const { dst[((size_t)ks * R + m) * R + n] = v; }
};
static __device__ __noinline__ void mr_gb_scatter(const double2* bh64, int R, int RS, int nJ, int Rp, int c,
                                                  int eblk, const unsigned short* tab, const int* eown, double2* gbt,
                                                  double2* gbrecv) {
  cg::cluster_group cluster = cg::this_cluster();
  const int tid = threadIdx.x, NT = blockDim.x;
  const int KS = mr_gb_parts(R);
  zgemm_dmma<MR_ZG>(R, R, nJ, bh64, 1, RS, bh64, RS, KS, MrEpiParts{gbt, R});
  __syncthreads();
  for (int e = tid; e < Rp; e += NT) {
    const int ij = tab[e];
    const int r = ij >> 8, q = ij & 255;
    double2 acc = gbt[q * R + r];
    for (int ks = 1; ks < KS; ++ks) acc = zadd(acc, gbt[((size_t)ks * R + q) * R + r]);
    const int ow = eown[e];
    *(cluster.map_shared_rank(gbrecv, ow >> 16) + (size_t)c * eblk + (ow & 0xffff)) = acc;
  }
  __syncthreads();
}

// ---------------------------------------------------------------- GEMM epilogues
struct MrEpiW {  // W accumulation (fp64)
  double2* acc;
  int R;
  TT_DEV void operator()(int m, int n, int ks, double2 v) const {
    (void)ks;
    acc[m * R + n] = zadd(acc[m * R + n], v);
  }
};
struct MrEpiZ {  // Z partial row m -> the owner of m's sampled-row block, slot c (zown: owner << 16 | row)
  double2* zrecv;
  const int* zown;
  int R, c, sblk;
  TT_DEV void operator()(int m, int n, int ks, double2 v) const {
    (void)ks;
    const int ow = zown[m];
    *(cg::this_cluster().map_shared_rank(zrecv, ow >> 16) + ((size_t)c * sblk + (ow & 0xffff)) * R + n) = v;
  }
};
struct MrEpiGA {  // C = Ah_S^T conj(Ah_S): C[m][n] = GA[n][m] -> packed G (lower) and the full Hermitian gaf
  double2* G;
  double2* gaf;
  int RS;  // gaf row stride
  TT_DEV void operator()(int m, int n, int ks, double2 v) const {
    (void)ks;
    if (n < m) return;
    G[tri_idx(n, m)] = v;
    gaf[n * RS + m] = v;
    if (n > m) gaf[m * RS + n] = zconj(v);
  }
};
struct MrEpiP {  // sampled row m of this CTA's block: cfac Ah + mu conj(g) (Z - corr) -> every CTA's mirror
  const double2* zsum;
  const double2* aown;  // the block's Ah_S rows (fp64 copies of the fp32 state), row stride RS
  const int* rowid;     // mirror row of block row m
  const double2* gam;
  float2* ahf;
  double cfac, mu;
  int R, RS, CL;
  TT_DEV void operator()(int m, int n, int ks, double2 v) const {
    (void)ks;
    const int o = m * R + n;
    const double2 inc = zscale(zmul(zconj(gam[n]), zsub(zsum[o], v)), mu);
    const float2 nv = to_f2(zadd(zscale(aown[m * RS + n], cfac), inc));
    const size_t at = (size_t)rowid[m] * R + n;
    cg::cluster_group cl = cg::this_cluster();
    for (int q = 0; q < CL; ++q) *(cl.map_shared_rank(ahf, q) + at) = nv;
  }
};
struct MrEpiQ {  // own Bh rows: cfac Bh + mu conj(g) (W - corr), fp64 (into acc = W)
  double2* acc;
  const double2* base;  // the own Bh rows (fp64 copies of the fp32 state), row stride RS
  const double2* gam;
  double cfac, mu;
  int R, RS;
  TT_DEV void operator()(int m, int n, int ks, double2 v) const {
    (void)ks;
    const int o = m * R + n;
    acc[o] = zadd(zscale(base[m * RS + n], cfac), zscale(zmul(zconj(gam[n]), zsub(acc[o], v)), mu));
  }
};

// ---------------------------------------------------------------- the kernel
template <int SOLV>
__global__ void __launch_bounds__(MR_NT, 1) tt_rows_mirror_kernel(const __grid_constant__ tt_rows_args a,
                                                                  const __grid_constant__ MirrorPlan pl) {
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int tid = threadIdx.x, NT = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int CL = pl.CL;
  const int c = (int)cluster.block_rank();
  const int s = (int)(blockIdx.x / CL);
  const int nx = a.nx, ny = a.ny, R = a.rank, Smax = a.max_rows, Rp = pl.Rp;
  const int j0 = part_begin(ny, CL, c), nJ = part_begin(ny, CL, c + 1) - j0;
  const int i0 = part_begin(nx, CL, c), nI = part_begin(nx, CL, c + 1) - i0;  // rows this CTA writes out
  const int eb = part_begin(Rp, CL, c), ee = part_begin(Rp, CL, c + 1);
  const int RS64 = pl.rs64;  // padded row stride of the fp64 operands bh64 / ahs64 / gaf / gbf

  float2* ahf = (float2*)(smem + pl.o_ahf);
  double2* bh64 = (double2*)(smem + pl.o_bh64);
  unsigned char* U = smem + pl.o_u;
  float2* ys = (float2*)U;
  double* pbuf = (double*)U;
  double* cdf = pbuf + nx;
  double* cnp = (double*)U;
  double2* hpart = (double2*)U;
  double2* gbt = (double2*)U;
  double2* ahs64 = (double2*)(smem + pl.o_ahs);
  double2* wacc = (double2*)(smem + pl.o_wacc);
  double2* zrecv = (double2*)(smem + pl.o_zrecv);
  double2* hrecv = (double2*)(smem + pl.o_hrecv);
  double* ynrecv = (double*)(smem + pl.o_ynrecv);
  double2* gbrecv = (double2*)(smem + pl.o_gbrecv);
  double2* gbfull = (double2*)(smem + pl.o_gbfull);
  double2* G = (double2*)(smem + pl.o_G);
  double2* gaf = (double2*)(smem + pl.o_gaf);
  double2* gbf = (double2*)(smem + pl.o_gbf);
  double2* gam = (double2*)(smem + pl.o_vec);
  double2* hv = gam + R;
  double2* hsave = hv + R;
  double* nrm = (double*)(hsave + R);
  double* inrm = nrm + R;
  double* gda = inrm + R;
  double* gdb = gda + R;
  float2* gamf = (float2*)(gdb + R);
  double* scal = (double*)(gamf + R);  // 16 scalars
  unsigned short* tab = (unsigned short*)(smem + pl.o_tab);
  double2* colb = (double2*)(smem + pl.o_colb);
  int* flags = (int*)(smem + pl.o_flags);
  int* rows = (int*)(smem + pl.o_rows);
  int* forced = (int*)(smem + pl.o_forced);
  double* usm = (double*)(smem + pl.o_usm);
  double* red = (double*)(smem + pl.o_red);
  int* zown = (int*)(smem + pl.o_zown);
  int* eown = (int*)(smem + pl.o_eown);
  __shared__ int sh_err;
  __shared__ __align__(8) unsigned long long ybar;  // completion of the frame's bulk Y-row copies
  long long* pclk = (a.phase_clock != nullptr && blockIdx.x == 0) ? (long long*)a.phase_clock : nullptr;
#define STAMP(k)                                                                                   \
  do {                                                                                             \
    if (pclk != nullptr) stamp_if(tid == 0, pclk + (size_t)f * 32 + (k));                           \
  } while (0)

  // ---- resident state and constants
  {
    const float2* asrc = (const float2*)a.ah_in + (size_t)s * nx * R;
    for (int o = tid; o < nx * R; o += NT) ahf[o] = asrc[o];
    const float2* bsrc = (const float2*)a.bh_in + ((size_t)s * ny + j0) * R;
    for (int o = tid; o < nJ * R; o += NT) {
      const int jj = idiv(o, R), r = o - jj * R;
      const float2 v = bsrc[o];
      bh64[jj * RS64 + r] = to_d2(v);  // the fp32 state, held exactly in fp64
    }
    if (a.policy == TT_POLICY_INFORMATIVE)
      for (int m = tid; m < a.nforced; m += NT) forced[m] = a.forced[m];
  }
  ldl_table_init(tab, R);
  for (int e = tid; e < Rp; e += NT) {  // owner of every packed Gram entry, position in its block
    int q = 0;
    while (q + 1 < CL && part_begin(Rp, CL, q + 1) <= e) ++q;
    eown[e] = (q << 16) | (e - part_begin(Rp, CL, q));
  }
  const bool y_bulk = !a.y_host && (nJ & 1) == 0 && (j0 & 1) == 0 && (ny & 1) == 0 && ((size_t)a.ysrc & 15) == 0 &&
                      (size_t)Smax * nJ * sizeof(float2) < (1u << 20);
  unsigned yph = 0;
  if (tid == 0) {
    mbar_init(&ybar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_proxy_async_smem();
  unsigned fmask = 0u;  // forced lines among this thread's rows of the block-wide draw
  int top = 1;          // largest power of two <= nx
  while (2 * top <= nx) top *= 2;
  if (a.policy == TT_POLICY_INFORMATIVE) {
    const int ipt = (nx + NT - 1) / NT, r0 = tid * ipt;
    for (int m = 0; m < a.nforced; ++m) {
      const int d = a.forced[m] - r0;
      if (d >= 0 && d < ipt && r0 + d < nx) fmask |= 1u << d;
    }
  }
  double alpha_bar = a.alpha_bar ? a.alpha_bar[s] : 0.0;
  uint64_t ppos = (a.policy == TT_POLICY_INFORMATIVE && a.philox_pos) ? a.philox_pos[s] : 0ull;
  const double ncap2 = a.norm_cap * a.norm_cap;
  bool prev_upd = false;
  int status = 0;
  const int ndraw = a.policy == TT_POLICY_INFORMATIVE ? max(a.k_draws - a.nforced, 0) : 0;
  const uint64_t k1s = a.key1 + (uint64_t)s;
  const bool gather = a.y_mode == TT_Y_GATHER;
  if (a.policy == TT_POLICY_INFORMATIVE)  // the first frame's uniforms (later ones are drawn at B1)
    for (int m = tid; m < ndraw; m += NT) usm[m] = philox_uniform(a.key0, k1s, ppos + (uint64_t)m);
  __syncthreads();
  // GB of the initial Bh: partials scattered to the entry owners
  mr_gb_scatter(bh64, R, RS64, nJ, Rp, c, pl.eblk, tab, eown, gbt, gbrecv);
  cluster_barrier();

  for (int f = 0; f < a.frames; ++f) {
    const long long t = a.t0 + f;
    const double lt = a.lam / (double)t;
    STAMP(0);
    // ======== (1) GB: own packed entries, CTA-ordered sum, broadcast to every CTA
    for (int e = eb + tid; e < ee; e += NT) {
      double2 v = gbrecv[e - eb];
      for (int q = 1; q < CL; ++q) v = zadd(v, gbrecv[(size_t)q * pl.eblk + e - eb]);
      for (int q = 0; q < CL; ++q) *(cluster.map_shared_rank(gbfull, q) + e) = v;
    }
    // ======== (2) column norms of the whole Ah (every CTA, one order)
    const int cparts = NT / R;
    if (tid < cparts * R) {
      const int r = tid % R, part = tid / R;
      double acc = 0.0;
      for (int i = part; i < nx; i += cparts) {
        const float2 v = ahf[i * R + r];
        acc += (double)v.x * v.x + (double)v.y * v.y;
      }
      cnp[part * R + r] = acc;
    }
    if (tid == 0) sh_err = 0;
    __syncthreads();
    if (tid < R) {
      double n2 = 0.0;
      for (int part = 0; part < cparts; ++part) n2 += cnp[part * R + tid];
      nrm[tid] = n2;
      inrm[tid] = n2 > 0.0 ? fast_rcp(n2) : 0.0;
    }
    __syncthreads();
    STAMP(1);
    // ======== (3) the frame's rows
    int S;
    if (a.policy == TT_POLICY_INFORMATIVE) {
      // raw row scores of every row (sampler.py:77-85, :126): one row per thread, the rank terms taken
      // from a row-dependent start (i mod R) so the lanes of a warp spread over the shared-memory banks
      const double cs = (double)ny, cr = (double)R, cd = 1.0 / ((double)R * (double)(nx + ny));
      for (int i = tid; i < nx; i += NT) {
        double e = 0.0;
        int r = i % R;
        const float2* row = ahf + i * R;
        for (int k = 0; k < R; ++k) {
          const float2 v = row[r];
          e = fma((double)v.x * v.x + (double)v.y * v.y, inrm[r], e);
          r = r + 1 == R ? 0 : r + 1;
        }
        pbuf[i] = (cs * e + cr) * cd;
      }
      if (tid < R && nrm[tid] == 0.0) atomicOr(&sh_err, TT_ST_ZEROCOL);
      __syncthreads();
      STAMP(2);
      S = mr_draw_rows(pbuf, cdf, flags, rows, nx, ndraw, usm, forced, a.nforced, fmask, top, a.beta,
                       a.draw_wor != 0, red);
      ppos += (uint64_t)ndraw;
    } else {
      S = mr_load_static_rows(a, f, s, rows, flags, &sh_err);
    }
    status |= sh_err;
    STAMP(3);
    // ======== (4) Y rows of own columns: one bulk copy per row (warp 0, completion on ybar) or cp.async
    fence_proxy_async_smem();  // this frame's generic accesses of U before the async-proxy writes into it
    __syncthreads();
    const float2* ybase = gather ? (const float2*)a.ysrc + (size_t)f * a.y_frame_stride + (size_t)s * a.y_slice_stride + j0
                                 : (const float2*)a.ysrc + ((size_t)f * a.nslices + s) * Smax * ny + j0;
    if (S > 0 && nJ > 0) {
      if (y_bulk) {
        if (warp == 0) {
          if (lane == 0) mbar_arrive_expect_tx(&ybar, (unsigned)(S * nJ * sizeof(float2)));
          __syncwarp();
          for (int kk = lane; kk < S; kk += 32)
            bulk_g2s(&ys[(size_t)kk * pl.ysr], ybase + (size_t)(gather ? rows[kk] : kk) * ny,
                     (unsigned)(nJ * sizeof(float2)), &ybar);
        }
      } else {
        for (int o = tid; o < S * nJ; o += NT) {
          const int kk = idiv(o, nJ), jj = o - kk * nJ;
          cp_async8(&ys[kk * pl.ysr + jj], ybase + (size_t)(gather ? rows[kk] : kk) * ny + jj);
        }
      }
    }
    // ======== (5) sampled-row marks, Ah_S (fp64) and GA from the mirror, while the rows land
    for (int i = tid; i < nx; i += NT) flags[i] = -1;
    for (int o = tid; o < nJ * R; o += NT) wacc[o] = make_double2(0.0, 0.0);
    __syncthreads();
    for (int k = tid; k < S; k += NT) {
      flags[rows[k]] = k;
      // owner of sampled row k (the CTA that updates it: the largest q with floor(S q / CL) <= k) and the
      // position in the owner's block
      const int q = ((k + 1) * CL - 1) / S;
      zown[k] = (q << 16) | (k - (S * q) / CL);
    }
    for (int o = tid; o < S * R; o += NT) {
      const int k = idiv(o, R), r = o - k * R;
      ahs64[k * RS64 + r] = to_d2(ahf[rows[k] * R + r]);
    }
    __syncthreads();
    zgemm_dmma<MR_ZG>(R, R, S, ahs64, 1, RS64, ahs64, RS64, 1, MrEpiGA{G, gaf, RS64});  // GA (fp64 tensor cores)
    STAMP(4);
    // ======== (6) W = Y_J^T conj(Ah_S), the Z partial (owners' blocks), h and ||Y||^2 partials
    double ysq = 0.0;
    if (S > 0 && nJ > 0) {
      if (y_bulk) {
        mbar_wait(&ybar, yph);
        yph ^= 1u;
      } else {
        cp_async_wait_all();
      }
    }
    __syncthreads();
    STAMP(5);
    for (int o = tid; o < S * nJ; o += NT) {
      const int kk = idiv(o, nJ), jj = o - kk * nJ;
      const float2 v = ys[kk * pl.ysr + jj];
      ysq += (double)v.x * v.x + (double)v.y * v.y;
    }
    if (S > 0) {
      zgemm_dmma<MR_ZG>(nJ, R, S, ys, 1, pl.ysr, ahs64, RS64, 1, MrEpiW{wacc, R});
      zgemm_dmma<3>(S, R, nJ, ys, pl.ysr, 1, bh64, RS64, 1, MrEpiZ{zrecv, zown, R, c, pl.sblk});
    }
    __syncthreads();
    STAMP(6);
    {
      const int hparts = max(1, min(NT / R, nJ));
      if (tid < hparts * R) {
        const int r = tid % R, part = tid / R;
        double2 h = make_double2(0.0, 0.0);
        for (int jj = part; jj < nJ; jj += hparts) h = zfma_cj(bh64[jj * RS64 + r], wacc[jj * R + r], h);
        hpart[part * R + r] = h;
      }
      __syncthreads();
      if (tid < R) {
        double2 h = make_double2(0.0, 0.0);
        for (int part = 0; part < hparts; ++part) h = zadd(h, hpart[part * R + tid]);
        for (int q = 0; q < CL; ++q) *(cluster.map_shared_rank(hrecv, q) + (size_t)c * R + tid) = h;
      }
    }
    {
      const double yt = block_sum(ysq, red);
      if (tid == 0)
        for (int q = 0; q < CL; ++q) *(cluster.map_shared_rank(ynrecv, q) + c) = yt;
    }
    STAMP(7);
    cluster_arrive();  // ------------------------------------------------ B1 (split: the next frame's
    if (a.policy == TT_POLICY_INFORMATIVE && f + 1 < a.frames)  //        uniforms while it completes)
      for (int m = tid; m < ndraw; m += NT) usm[m] = philox_uniform(a.key0, k1s, ppos + (uint64_t)m);
    cluster_wait();
    STAMP(8);

    // ======== (8) fp64 Gram + ridge solve (every CTA, identical inputs), cost, step
    if (tid < R) {
      double2 h = hrecv[tid];
      for (int q = 1; q < CL; ++q) h = zadd(h, hrecv[(size_t)q * R + tid]);
      hv[tid] = h;
      hsave[tid] = h;
    }
    if (tid == R) {
      double y2 = 0.0;
      for (int q = 0; q < CL; ++q) y2 += ynrecv[q];
      scal[0] = y2;
    }
    for (int e = tid; e < Rp; e += NT) {
      const int ij = tab[e];
      const int r = ij >> 8, q = ij & 255;
      const double2 gae = G[e], gbe = gbfull[e];
      double2 gg = zmul(gae, gbe);
      if (r == q) {
        gg.x += a.lam;
        gda[r] = gae.x;
        gdb[r] = gbe.x;
      }
      G[e] = gg;
      gbf[r * RS64 + q] = gbe;
      gbf[q * RS64 + r] = zconj(gbe);
    }
    __syncthreads();
    if (warp == 0) {  // ||Bh||^2 = trace(GB); ||Ah||^2 from the column norms
      double v = 0.0, w = 0.0;
      for (int r = lane; r < R; r += 32) {
        v += gdb[r];
        w += nrm[r];
      }
      for (int o = 16; o > 0; o >>= 1) {
        v += __shfl_xor_sync(0xffffffffu, v, o);
        w += __shfl_xor_sync(0xffffffffu, w, o);
      }
      if (lane == 0) {
        scal[2] = v;
        scal[1] = w;
      }
    }
    STAMP(9);
    double mu_used = 0.0, alpha = 0.0, cost;
    const bool update = S > 0;
    if (update) {
      if (SOLV == 1) block_gj_solve<1>(G, hv, gam, colb, R);
      else if (SOLV == 2) block_gj_solve<2>(G, hv, gam, colb, R);
      else block_gj_solve<5>(G, hv, gam, colb, R);
      STAMP(10);
      if (warp == 0) {
        double gh = 0.0, gg = 0.0, tp = 0.0;
        for (int r = lane; r < R; r += 32) {
          const double2 g = gam[r], h = hsave[r];
          gh += g.x * h.x + g.y * h.y;  // Re(conj(g) h)
          const double g2 = g.x * g.x + g.y * g.y;
          gg += g2;
          tp = fmax(tp, g2 * fmax(gda[r], gdb[r]));
          gamf[r] = to_f2(g);
        }
        gh = warp_sum(gh);
        gg = warp_sum(gg);
        tp = warp_max(tp);
        if (lane == 0) {
          scal[3] = gh;
          scal[4] = gg;
          scal[5] = tp;
        }
      }
      __syncthreads();
      const double energy = scal[1] + scal[2];
      const double e2 = scal[0] - scal[3] - a.lam * scal[4];
      cost = 0.5 * e2 + 0.5 * lt * energy;
      if (a.step_mode == TT_STEP_HESSIAN) {
        alpha = fmin(fmax(lt + scal[5], a.c_floor), a.c_cap);  // tracker.py:364
        alpha_bar += alpha;
        mu_used = 1.0 / alpha_bar;
      } else {
        mu_used = a.mu;
      }
      if (!isfinite(cost) || !isfinite(scal[3])) status |= TT_ST_NONFINITE;
    } else {
      if (tid < R) {
        gam[tid] = make_double2(0.0, 0.0);
        gamf[tid] = make_float2(0.f, 0.f);
      }
      cost = 0.5 * lt * (scal[1] + scal[2]);
      __syncthreads();
    }
    if (a.norm_out && c == 0 && tid == 0 && f > 0)  // the previous frame's post-update norms
      a.norm_out[((size_t)f - 1) * a.nslices + s] = (prev_upd && (scal[1] > ncap2 || scal[2] > ncap2)) ? 1 : 0;
    prev_upd = update;
    STAMP(11);

    // ======== (9)-(12) updates: own block of sampled rows into every mirror, cfac elsewhere, own Bh rows
    if (update) {
      const double cfac = 1.0 - mu_used * lt;
      const int kb = part_begin(S, CL, c), nb = part_begin(S, CL, c + 1) - kb;
      for (int o = tid; o < R * R; o += NT) {  // gamma-scaled R x R factors (GA, GB not read again)
        const int q = idiv(o, R), r = o - q * R;
        const double2 cgm = zconj(gam[q]);
        gaf[q * RS64 + r] = zmul(cgm, gaf[q * RS64 + r]);
        gbf[q * RS64 + r] = zmul(cgm, gbf[q * RS64 + r]);
      }
      for (int o = tid; o < nb * R; o += NT) {  // Z of the block rows: CTA-ordered sum in place (slot 0)
        const int m = idiv(o, R), r = o - m * R;
        double2 z = zrecv[o];
        for (int q = 1; q < CL; ++q) z = zadd(z, zrecv[((size_t)q * pl.sblk + m) * R + r]);
        zrecv[o] = z;
      }
      __syncthreads();
      STAMP(12);
      const double2* aown = ahs64 + (size_t)kb * RS64;  // the block's Ah_S rows
      zgemm_dmma<MR_ZG>(nb, R, R, aown, RS64, 1, gbf, RS64, 1,
                        MrEpiP{zrecv, aown, rows + kb, gam, ahf, cfac, mu_used, R, RS64, CL});
      STAMP(16);
      zgemm_dmma<MR_ZG>(nJ, R, R, bh64, RS64, 1, gaf, RS64, 1, MrEpiQ{wacc, bh64, gam, cfac, mu_used, R, RS64});
      __syncthreads();
      STAMP(13);
      // rows outside the frame's sample: cfac (tracker.py:402-404); a row per thread, the row's elements from
      // a row-dependent start (lanes spread over the banks)
      for (int i = tid; i < nx; i += NT)
        if (flags[i] < 0) {
          float2* rowp = ahf + i * R;
          int r = i % R;
#pragma unroll 4
          for (int k = 0; k < R; ++k) {
            rowp[r] = to_f2(zscale(to_d2(rowp[r]), cfac));
            r = r + 1 == R ? 0 : r + 1;
          }
        }
      for (int o = tid; o < nJ * R; o += NT) {
        const int jj = idiv(o, R), r = o - jj * R;
        bh64[jj * RS64 + r] = to_d2(to_f2(wacc[o]));  // the state is fp32, held exactly in fp64
      }
      __syncthreads();
      STAMP(17);
      mr_gb_scatter(bh64, R, RS64, nJ, Rp, c, pl.eblk, tab, eown, gbt, gbrecv);  // next frame's GB
    }
    STAMP(14);
    // ======== outputs
    const size_t fs = (size_t)f * a.nslices + s;
    if (c == 0) {
      if (a.gamma_out && tid < R) ((float2*)a.gamma_out)[fs * R + tid] = gamf[tid];
      if (tid == 0) {
        if (a.cost_out) a.cost_out[fs] = cost;
        if (a.mu_out) a.mu_out[fs] = mu_used;
        if (a.alpha_out) a.alpha_out[fs] = alpha;
        if (a.cnt_out) a.cnt_out[fs] = S;
      }
      if (a.rows_out)
        for (int k = tid; k < Smax; k += NT) a.rows_out[fs * Smax + k] = k < S ? rows[k] : -1;
    }
    cluster_barrier();  // ------------------------------------------------ B2
    STAMP(15);
    if (a.ah_hist) {
      float2* dst = (float2*)a.ah_hist + (fs * nx + i0) * R;
      for (int o = tid; o < nI * R; o += NT) dst[o] = ahf[(size_t)i0 * R + o];
    }
    if (a.bh_hist) {
      float2* dst = (float2*)a.bh_hist + (fs * ny + j0) * R;
      for (int o = tid; o < nJ * R; o += NT) dst[o] = to_f2(bh64[idiv(o, R) * (RS64 - R) + o]);
    }
  }
#undef STAMP

  // ---- write back the resident state
  {
    float2* dst = (float2*)a.ah_out + ((size_t)s * nx + i0) * R;
    for (int o = tid; o < nI * R; o += NT) dst[o] = ahf[(size_t)i0 * R + o];
    float2* dsb = (float2*)a.bh_out + ((size_t)s * ny + j0) * R;
    for (int o = tid; o < nJ * R; o += NT) dsb[o] = to_f2(bh64[idiv(o, R) * (RS64 - R) + o]);
  }
  if (a.norm_out && a.frames > 0) {  // the last frame's post-update norms: trace(GB) of the final Bh
    double tr = 0.0;
    for (int e = eb + tid; e < ee; e += NT) {
      const int ij = tab[e];
      if ((ij >> 8) == (ij & 255)) {
        double v = gbrecv[e - eb].x;
        for (int q = 1; q < CL; ++q) v += gbrecv[(size_t)q * pl.eblk + e - eb].x;
        tr += v;
      }
    }
    tr = block_sum(tr, red);
    if (tid == 0) *(cluster.map_shared_rank(ynrecv, 0) + c) = tr;
    double na = 0.0;
    for (int o = tid; o < nx * R; o += NT) na += (double)ahf[o].x * ahf[o].x + (double)ahf[o].y * ahf[o].y;
    na = block_sum(na, red);
    cluster_barrier();
    if (c == 0 && tid == 0) {
      double nb2 = 0.0;
      for (int q = 0; q < CL; ++q) nb2 += ynrecv[q];
      a.norm_out[(size_t)(a.frames - 1) * a.nslices + s] = (prev_upd && (na > ncap2 || nb2 > ncap2)) ? 1 : 0;
    }
  }
  if (c == 0 && tid == 0) {
    if (a.alpha_bar) a.alpha_bar[s] = alpha_bar;
    if (a.policy == TT_POLICY_INFORMATIVE && a.philox_pos) a.philox_pos[s] = ppos;
  }
  if (status && tid == 0 && a.status) atomicOr(&a.status[s], status);
  cluster_barrier();  // no CTA leaves while a peer may still address its shared memory
}

// ---------------------------------------------------------------- host side
// Whether the mirrored kernel runs this launch (and its plan): row masks without sharding or a residual
// output, Gauss-Jordan ranks (R <= 32), the whole Ah plus the frame's Y tile within shared memory.
// Opt-in: TT_ROWS_MIRROR=1.
bool tt_rows_mirror_plan(const tt_rows_args* a, int CL, MirrorPlan* pl) {
  // opt-in (TT_ROWS_MIRROR=1): measured slower than tt_rows.cu's kernel at the config 2 / 3 shapes
  // (its redundant per-CTA Gram work and small fp64 tensor-core GEMMs outweigh the two
  // cluster barriers and L2 round trips it saves)
  const char* e = getenv("TT_ROWS_MIRROR");
  if (!e || e[0] != '1') return false;
  if (a->shard_world > 0 || a->resid_out) return false;
  if (gj_ept(a->rank, MR_NT) > 5) return false;
  return mirror_make_plan(a->nx, a->ny, a->rank, a->max_rows, CL, pl);
}

extern "C" int tt_rows_mirror_fits(int nx, int ny, int rank, int max_rows, int cluster) {
  const char* e = getenv("TT_ROWS_MIRROR");
  if (!e || e[0] != '1') return 0;
  MirrorPlan pl;
  if (gj_ept(rank, MR_NT) > 5) return 0;
  return mirror_make_plan(nx, ny, rank, max_rows, cluster, &pl) ? 1 : 0;
}

int tt_rows_mirror_launch(void* stream, const tt_rows_args* a, const MirrorPlan& pl) {
  typedef void (*Fn)(const tt_rows_args, const MirrorPlan);
  static const Fn fns[3] = {tt_rows_mirror_kernel<1>, tt_rows_mirror_kernel<2>, tt_rows_mirror_kernel<5>};
  static size_t configured[3][TT_MAXDEV] = {{0}};
  const int ept = gj_ept(a->rank, MR_NT);
  const int which = ept <= 1 ? 0 : ept <= 2 ? 1 : 2;
  const Fn fn = fns[which];
  int dev = 0;
  TT_CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= TT_MAXDEV || configured[which][dev] < (size_t)pl.smem) {
    TT_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    TT_CUDA_TRY(tt_smem_attr((const void*)fn, (size_t)pl.smem, configured[which]));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a->nslices * pl.CL), 1, 1);
  cfg.blockDim = dim3(MR_NT, 1, 1);
  cfg.dynamicSmemBytes = (size_t)pl.smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)pl.CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TT_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, *a, pl));
  return TT_OK;
}
