// Fused persistent online MM step for Cartesian row masks (sm_100a).
//
// Reference path (tensortrack, /root/reference/pkg/src/tensortrack):
//   tracker.track_step                          tracker.py:367-411
//     build_phi (FourierMask branch)            observation.py:224-228
//     solve_gamma (SVD ridge)                   tracker.py:139-156
//     residual + cost                           tracker.py:386-389
//     hessian_bound / power method              tracker.py:307-364
//     factor_gradient (_scatter_theta, ifft2)   tracker.py:176-228, 241-262
//     update                                    tracker.py:402-404
//   sampler.row_scores + draw_samples           sampler.py:77-170
//   experiment.run_adaptive per-frame body      experiment.py:482-530
//
// B200 formulation. The state is held as k-space factors
// Ah = F_x A, Bh = F_y B. Since F is unitary, the reference's image-domain
// update A <- A - mu((lam/t)A - conj(gamma) . F^-1 P) is exactly
// Ah <- (1 - mu lam/t) Ah + mu conj(gamma) . P, so no FFT sits inside the
// frame loop. For a row mask S (|S| rows, all Ny columns) with data Y (S x Ny):
//   GA = Ah_S^H Ah_S, GB = Bh^H Bh          (fp64, R x R, Hermitian)
//   Phi^H Phi = GA .* GB                    (separable Gram)
//   W = Y^T conj(Ah_S)        (Ny x R)      h = sum_j conj(Bh_j) . W_j
//   Z = Y conj(Bh)            (S x R)
//   gamma = (GA.*GB + lam I)^-1 h           (fp64 LDL^H)
//   P_S = Z - Ah_S diag(gamma) GB^T         Q = W - Bh diag(gamma) GA^T
//   ||e||^2 = ||Y||^2 - Re(gamma^H h) - lam ||gamma||^2
//   alpha = lam/t + max_r |gamma_r|^2 max(GA_rr, GB_rr)  (exact closed form of
//           the reference power iteration for row masks)
//
// Parallel layout: one thread-block cluster of CL CTAs per slice. CTA c owns
// k-space rows I_c of Ah and rows J_c of Bh (= Y columns J_c), resident in
// shared memory for all frames. Cross-CTA data goes through L2-resident
// scratch (ld/st .cg) between hardware cluster barriers (3 per frame for
// static masks, 4 for informative ones). The small R x R solve is done
// redundantly by every CTA, so nothing is broadcast.

#include <cooperative_groups.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "tt_block.cuh"
#include "tt_mirror.cuh"

namespace cg = cooperative_groups;

#define ROWS_NT 256
#define ROWS_UF 32  // frames of precomputed Philox uniforms per refill
#define ROWS_ZKS 8  // K parts of the Z GEMM per CTA (fp64 partials in L2, summed by the rows' owners)
// register tile of the small GEMMs (cgemm_tile): 4 rows x 2 columns of the output per thread beat 2 x 4
// at every rows-kernel shape, same accumulator count (profiles/tools/ubench_gemm42.cu: C4 Z 27.6k -> 21.3k cycles)
constexpr int GTM = 4, GTN = 2;
// register tile of the fp64-accumulating data GEMMs (zgemm_tile): F2F conversions per k step = TM + TN
// complex operands, DFMA = 4 TM TN
constexpr int ZTM = 2, ZTN = 4;
constexpr int ZG = 4;   // 8-row M blocks per DMMA work item (zgemm_dmma)
constexpr int ZGZ = 6;  // ... for the Z GEMM (short M = sampled rows, long K: K parts instead of M groups;
                        // profiles/tools/ubench_dmma_shapes.cu: config 3 Z 11.9k -> 9.5k cycles)

struct RowsPlan {
  int CL, KT, nIm, nJm, Rp, red_cap, tight, ysr;
  int o_ahl, o_bhl, o_bh64, o_u1, o_gaf, o_gbf, o_vec, o_tab, o_flags, o_rows, o_forced, o_usm, o_own, o_wacc, o_zs, o_red2,
      o_u2, o_red;
  int smem;
};

struct RowsScratch {
  size_t cn, gbp, gb, ga, sraw, ahs, zp, hp, yn, unif, per_slice;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline RowsScratch rows_scratch_layout(int nx, int ny, int R, int Smax, int CL) {
  RowsScratch s;
  const size_t Rp = (size_t)R * (R + 1) / 2;
  size_t o = 0;
  s.cn = o;   o = al16(o + sizeof(double) * CL * R);
  s.gbp = o;  o = al16(o + sizeof(double2) * CL * Rp);
  s.gb = o;   o = al16(o + sizeof(double2) * Rp);
  s.ga = o;   o = al16(o + sizeof(double2) * Rp);
  s.sraw = o; o = al16(o + sizeof(double) * nx);
  s.ahs = o;  o = al16(o + sizeof(float2) * (size_t)Smax * R);
  s.zp = o;   o = al16(o + sizeof(double2) * (size_t)CL * ROWS_ZKS * Smax * R);  // Z partials [CTA][K part], fp64
  s.hp = o;   o = al16(o + sizeof(double2) * CL * R);
  s.yn = o;   o = al16(o + sizeof(double) * CL);
  s.unif = o; o = al16(o + sizeof(double) * (size_t)ROWS_UF * Smax);  // Philox uniforms, ROWS_UF frames
  s.per_slice = al16(o + 256);
  (void)ny;
  return s;
}

static bool rows_make_plan_cap(int nx, int ny, int R, int Smax, int CL, int red_cap, bool tight, RowsPlan* p);
// The K-split reduction buffer of the small GEMMs is optional: when shared
// memory is tight the plan drops it and every GEMM runs with KS = 1. When even
// that does not fit (R = 64 at 1024^2) the "tight" plan also drops the fp32
// copies of GA / GB: the two update GEMMs run one after the other with their
// gamma-scaled R x R operand built in the (then free) solver workspace U1.
static bool rows_make_plan(int nx, int ny, int R, int Smax, int CL, RowsPlan* p) {
  if (const char* e = getenv("TT_ROWS_FORCE_TIGHT"))  // test hook: the tight plan at any shape (R >= 24)
    if (e[0] == '1' && R >= 24) return rows_make_plan_cap(nx, ny, R, Smax, CL, 0, true, p);
  // prefer the K-split buffer, but not at the cost of a second k tile of Y rows (the one-tile path overlaps the
  // Z partial with the cluster's Ah_S exchange)
  RowsPlan q;
  const bool with_red = rows_make_plan_cap(nx, ny, R, Smax, CL, 2048, false, &q);
  if (with_red && q.KT >= Smax) {
    *p = q;
    return true;
  }
  if (rows_make_plan_cap(nx, ny, R, Smax, CL, 0, false, p)) {
    if (with_red && q.KT > p->KT) *p = q;
    return true;
  }
  if (with_red) {
    *p = q;
    return true;
  }
  return rows_make_plan_cap(nx, ny, R, Smax, CL, 0, true, p);
}
static bool rows_make_plan_cap(int nx, int ny, int R, int Smax, int CL, int red_cap, bool tight, RowsPlan* p) {
  const int maxsmem = 227 * 1024 - 256;  // the opt-in limit less the kernel's static __shared__ words
  if (R > 64) return false;
  p->CL = CL;
  p->nIm = (nx + CL - 1) / CL;
  p->nJm = (ny + CL - 1) / CL;
  p->Rp = R * (R + 1) / 2;
  p->red_cap = red_cap;
  p->tight = tight ? 1 : 0;
  size_t o = 0;
  p->o_ahl = (int)o;    o = al16(o + sizeof(float2) * p->nIm * R);
  p->o_bhl = (int)o;    o = al16(o + sizeof(float2) * p->nJm * R);
  p->o_bh64 = (int)o;   o = al16(o + (tight ? 0 : sizeof(double2) * p->nJm * R));  // fp64 copy of the Bh rows
  p->o_u1 = (int)o;     // packed fp64 Gram / LDL workspace  |  p + cdf (draw phase)  |  tight: update operand
  {
    size_t g = sizeof(double2) * (size_t)p->Rp;
    size_t d = sizeof(double) * 2 * (size_t)nx;
    size_t m = tight ? sizeof(float2) * (size_t)R * R : 0;
    if (d > g) g = d;
    if (m > g) g = m;
    o = al16(o + g);
  }
  const size_t gfull = tight ? 0 : sizeof(double2) * R * R;
  p->o_gaf = (int)o;    o = al16(o + gfull);  // full Hermitian fp64 GA, GB (not in the tight plan)
  p->o_gbf = (int)o;    o = al16(o + gfull);
  // vec: gam, hv, hsave (double2 R); nrm, inrm, inv, gda, gdb (double R); gamf (float2 R); 16 scalars
  //      + LDL scratch: colb 4 (R+1) double2, blk 4 (R/2+1) double, zf R double2
  p->o_vec = (int)o;    o = al16(o + sizeof(double2) * R * 3 + sizeof(double) * R * 5 + sizeof(float2) * R + 128 +
                                 sizeof(double2) * 4 * (R + 1) + sizeof(double) * 4 * (R / 2 + 1) + sizeof(double2) * R);
  p->o_tab = (int)o;    o = al16(o + sizeof(unsigned short) * p->Rp);
  p->o_flags = (int)o;  o = al16(o + sizeof(int) * (nx > p->nIm ? nx : p->nIm));
  p->o_rows = (int)o;   o = al16(o + sizeof(int) * Smax);
  p->o_forced = (int)o; o = al16(o + sizeof(int) * Smax);
  p->o_usm = (int)o;    o = al16(o + sizeof(double) * Smax);  // this frame's uniforms
  p->o_own = (int)o;    o = al16(o + sizeof(int) * 2 * p->nIm);
  p->o_wacc = (int)o;   o = al16(o + sizeof(double2) * p->nJm * R);  // W (fp64 sums), then the new Bh rows
  p->o_zs = (int)o;     o = al16(o + (tight ? 0 : sizeof(double2) * (p->nIm < Smax ? p->nIm : Smax) * R));  // Z of
                                                                                 // owned sampled rows, then mu conj(g) P
                                                                                 // (tight plan: in U2, free after B4)
  p->o_red2 = (int)o;   o = al16(o + sizeof(double2) * p->red_cap);  // K-split partials (fp64 or fp32)
  p->o_u2 = (int)o;
  size_t fixed = o + sizeof(double) * 64;
  if (fixed > (size_t)maxsmem) return false;
  // U2: k-tiles (ys KT x ysr fp32, ahs KT x R fp64) | GB partial tiles + colnorm partials (phase a) |
  // gamma-scaled GEMM operands. Phase (a): GB partial tiles (4 double2 per item, <= max(2 NT, tiles) items)
  // + colnorm partials (<= NT doubles); the h partials later (<= NT double2)
  const int gb_rt = (R + 1) / 2, gb_nt = gb_rt * (gb_rt + 1) / 2;
  size_t other = 4 * sizeof(double2) * (size_t)(gb_nt > 2 * ROWS_NT ? gb_nt : 2 * ROWS_NT) + sizeof(double) * ROWS_NT + 256;
  // Y tile row stride = 4 (mod 16) complex: 16 B aligned rows (bulk copies), 8 banks apart (the Z GEMM's
  // DMMA A fragments read 4 consecutive columns of 8 rows: conflict-free)
  p->ysr = ((p->nJm + 11) & ~15) + 4;
  const size_t v2 = sizeof(float2) * (size_t)R * p->nIm;  // tight: the P increments; else the owned sampled Ah rows
  if (v2 > other) other = v2;
  size_t avail = maxsmem - fixed;
  int KT = (int)(avail / (sizeof(float2) * (size_t)p->ysr + sizeof(double2) * (size_t)R));
  if (KT > Smax) KT = Smax;
  if (KT > 128) KT = 128;
  if (KT < 1) return false;
  p->KT = KT;
  size_t tiles = (sizeof(float2) * (size_t)p->ysr + sizeof(double2) * (size_t)R) * (size_t)KT;
  size_t u2 = tiles > other ? tiles : other;
  if (fixed + u2 > (size_t)maxsmem) return false;
  o = al16(o + u2);
  p->o_red = (int)o;
  o += sizeof(double) * 64;
  p->smem = (int)o;
  return true;
}

// ---------------------------------------------------------------- GEMM epilogues
// The four small GEMMs of a frame share one cgemm_tile instantiation (one copy of its code in the
// frame loop); the epilogue is selected by a block-uniform mode.
// The data GEMMs (W, Z) accumulate in fp64 (zgemm_tile) and deliver double2; the model-part corrections
// (K = R, fp32 operands: cgemm_tile) deliver float2 and are subtracted from the fp64 W / Z in fp64, so the
// update keeps the digits the cancellation would cost in fp32.
enum { EPI_W_ACC = 0, EPI_Z_STORE = 1, EPI_Q_UPDATE = 2, EPI_P_UPDATE = 3, EPI_P_MAPPED = 4 };
struct RowsEpiGB {    // GB partial on the fp64 tensor cores: C = Bh_J^T conj(Bh_J), C[m][n] = GB[n][m]
  double2* dst;       // this CTA's packed partial slots (L2)
  TT_DEV void operator()(int m, int n, int ks, double2 v) const {
    (void)ks;
    if (n < m) return;
    double2* d = dst + tri_idx(n, m);
    __stcg(&d->x, v.x);
    __stcg(&d->y, v.y);
  }
};
struct RowsEpiD {     // W / Z: fp64 values
  int mode, R;
  double2* acc;       // W: wacc
  double2* gdst;      // Z: L2 partials of this CTA, one slot of `pstride` per K part
  int pstride;
  TT_DEV void operator()(int m, int n, int ks, double2 v) const {
    const int o = m * R + n;
    if (mode == EPI_W_ACC) {
      acc[o] = zadd(acc[o], v);
    } else {
      double2* d = gdst + (size_t)ks * pstride + o;
      __stcg(&d->x, v.x);
      __stcg(&d->y, v.y);
    }
  }
};
struct RowsEpi {      // Q / P updates: fp32 correction v, fp64 arithmetic
  int mode, R;
  double2* acc;         // Q: wacc (in: W, out: new Bh rows) | P: zs (in: Z sums, out: mu conj(g) P)
  const float2* base;   // Q: bhl
  const double2* gam;   // this frame's gamma (fp64)
  double cfac, mu;
  const int* rmap;      // P_MAPPED (tight plan): local row -> position in the owned sampled rows, or -1
  // P_MAPPED (tight plan): Z summed straight from the CTAs' fp64 partials in L2, the increment stored fp32
  const int* own_k;
  const double2* zp;
  int zstride, CL;
  float2* inc32;
  // the fp64 corrections of the DMMA path
  TT_DEV void operator()(int m, int n, int ks, double2 v) const {
    (void)ks;
    const int o = m * R + n;
    if (mode == EPI_Q_UPDATE)
      acc[o] = zadd(zscale(to_d2(base[o]), cfac), zscale(zmul(zconj(gam[n]), zsub(acc[o], v)), mu));
    else  // EPI_P_UPDATE: mu conj(g) P
      acc[o] = zscale(zmul(zconj(gam[n]), zsub(acc[o], v)), mu);
  }
  TT_DEV void operator()(int m, int n, float2 v) const {
    int o = m * R + n;
    switch (mode) {
      case EPI_Q_UPDATE:
        acc[o] = zadd(zscale(to_d2(base[o]), cfac), zscale(zmul(zconj(gam[n]), zsub(acc[o], to_d2(v))), mu));
        break;
      case EPI_P_MAPPED: {  // tight plan: the GEMM ran over every local row, keep the sampled ones
        const int q = rmap[m];
        if (q < 0) break;
        const double2 z = sum_parts2n(zp + (size_t)own_k[q] * R + n, (size_t)zstride, CL);
        inc32[q * R + n] = to_f2(zscale(zmul(zconj(gam[n]), zsub(z, to_d2(v))), mu));
        break;
      }
      default:
        acc[o] = zscale(zmul(zconj(gam[n]), zsub(acc[o], to_d2(v))), mu);  // mu conj(g) P
        break;
    }
  }
};

// Inter-cluster barrier of a cooperative launch (every CTA co-resident): a monotonic arrival counter,
// one zeroed uint32 per launch; the k-th barrier completes when it reaches k * gridDim.x.
TT_DEV void grid_sync(unsigned* ctr, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned target = (++gen) * gridDim.x;
    atomicAdd(ctr, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
    __threadfence();
  } else {
    ++gen;
  }
  __syncthreads();
}

// ---------------------------------------------------------------- cold paths (kept out of line)
// Static row table validation: range and duplicates (observation.py:41-55).
static __device__ __noinline__ int load_static_rows(const tt_rows_args& a, int f, int s, int* rows, int* flags,
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

// Residual e = Y - Ah_S diag(gamma) Bh^T on this CTA's columns (pre-update),
// in measurement order (tracker.py:388, StepReport.residual).
static __device__ __noinline__ void write_residual(const tt_rows_args& a, const RowsPlan& pl, int f, int s, int S,
                                                   int j0, int nJ, const int* rows, const float2* g_ahs,
                                                   const float2* gamf, const float2* bhl, float2* ys, float2* ahs) {
  const int tid = threadIdx.x, NT = blockDim.x, R = a.rank, ny = a.ny, Smax = a.max_rows, KT = pl.KT;
  for (int k0 = 0; k0 < S; k0 += KT) {
    const int kt = min(KT, S - k0);
    for (int o = tid; o < kt * nJ; o += NT) {
      const int kk = o / nJ, jj = o - kk * nJ;
      const float2* src = a.y_mode == TT_Y_GATHER
                              ? (const float2*)a.ysrc + (size_t)f * a.y_frame_stride + (size_t)s * a.y_slice_stride +
                                    (size_t)rows[k0 + kk] * ny + j0
                              : (const float2*)a.ysrc + (((size_t)f * a.nslices + s) * Smax + k0 + kk) * ny + j0;
      ys[kk * pl.ysr + jj] = src[jj];
    }
    for (int o = tid; o < kt * R; o += NT) {
      float2 v;
      v.x = __ldcg(&g_ahs[(size_t)k0 * R + o].x);
      v.y = __ldcg(&g_ahs[(size_t)k0 * R + o].y);
      ahs[o] = cmul(v, gamf[o % R]);
    }
    __syncthreads();
    for (int o = tid; o < kt * nJ; o += NT) {
      const int kk = o / nJ, jj = o - kk * nJ;
      float2 e = ys[kk * pl.ysr + jj];
      float2 sacc = make_float2(0.f, 0.f);
      for (int r = 0; r < R; ++r) sacc = cfma(ahs[kk * R + r], bhl[jj * R + r], sacc);
      float2* dst = (float2*)a.resid_out + (((size_t)f * a.nslices + s) * Smax + k0 + kk) * ny + j0 + jj;
      *dst = csub(e, sacc);
    }
    __syncthreads();
  }
}

// Informative rows without replacement (draw_samples(replacement=False), sampler.py:163-169): the
// probabilities w (forced rows zeroed here) drawn from by k sequential renormalised draws
// (weighted_draw_without_replacement, observation.py:279-297): per draw cumsum(w), u = u01 * total,
// searchsorted(cdf, u, 'right'), w[idx] = 0. The cumsum is a block scan; a uniform within 1e-12 total of a
// bucket edge redoes that draw over numpy's sequential cumsum, so the rows equal numpy's for identical
// probabilities. Marks flags[idx] = 1 (cleared here); the caller adds the forced rows and compacts.
static __device__ __noinline__ void rows_draw_wor(double* w, double* cdf, int* flags, int nx, int ndraw,
                                                  const double* usm, const int* forced, int nforced, double* red) {
  const int tid = threadIdx.x, NT = blockDim.x;
  __shared__ int s_idx, s_amb;
  for (int i = tid; i < nx; i += NT) flags[i] = 0;
  __syncthreads();
  for (int m = tid; m < nforced; m += NT) {
    const int fr = forced[m];
    if (fr >= 0 && fr < nx) w[fr] = 0.0;
  }
  __syncthreads();
  for (int m = 0; m < ndraw; ++m) {
    for (int exact = 0; exact < 2; ++exact) {
      block_cumsum(w, cdf, nx, exact != 0, red);
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
      w[s_idx] = 0.0;
    }
    __syncthreads();
  }
}

// Post-update ||Ah||_F^2, ||Bh||_F^2 of the resident state (own rows / columns), summed over the cluster
// in CTA order through `slot` (CL double2 in L2); the result is valid in CTA 0 after the call.
static __device__ __noinline__ double2 cluster_state_norms(const float2* ahl, int nIA, const float2* bhl, int nJB,
                                                           double2* slot, int c, int CL, double* red) {
  double pa = 0.0, pb = 0.0;
  for (int o = threadIdx.x; o < nIA; o += blockDim.x) pa += (double)ahl[o].x * ahl[o].x + (double)ahl[o].y * ahl[o].y;
  for (int o = threadIdx.x; o < nJB; o += blockDim.x) pb += (double)bhl[o].x * bhl[o].x + (double)bhl[o].y * bhl[o].y;
  pa = block_sum(pa, red);
  pb = block_sum(pb, red);
  if (threadIdx.x == 0) {
    __stcg(&slot[c].x, pa);
    __stcg(&slot[c].y, pb);
  }
  cluster_barrier();
  return sum_parts2(slot, 1, CL);
}

// GB partial over a CTA's columns for wide column blocks (out of line: narrow blocks, config 2, keep
// the frame loop's instruction footprint): 2 x 2 register tiles of the lower triangle (four products
// per four operand loads), the columns split in `parts` interleaved parts, then a fixed-order sum of
// the parts per packed entry into dst_g.
template <bool TIGHT>
static __device__ __noinline__ void gb_partials_tiled(const float2* bhl, const double2* bh64, int R, int nJ, int Rp,
                                                      int gb_nt, int gb_parts, const unsigned short* tab,
                                                      double2* gbt, double2* dst_g, int jo, int jstep) {
  const int tid = threadIdx.x, NT = blockDim.x;
  for (int it = tid; it < gb_nt * gb_parts; it += NT) {
    const int part = idiv(it, gb_nt), t = it - part * gb_nt;
    int tr, tq;
    tri_decode(t, tr, tq);
    const int r0 = 2 * tr, q0 = 2 * tq, r1 = min(r0 + 1, R - 1), q1 = min(q0 + 1, R - 1);
    double2 a00 = make_double2(0.0, 0.0), a01 = a00, a10 = a00, a11 = a00;
    if (TIGHT) {  // fp32 operands converted on the fly (same products)
      for (int jj = jo + part * jstep; jj < nJ; jj += gb_parts * jstep) {
        const float2* row = bhl + jj * R;
        const float2 br0 = row[r0], br1 = row[r1], bq0 = row[q0], bq1 = row[q1];
        a00 = zfma_cj(br0, bq0, a00);
        a01 = zfma_cj(br0, bq1, a01);
        a10 = zfma_cj(br1, bq0, a10);
        a11 = zfma_cj(br1, bq1, a11);
      }
    } else {
      for (int jj = jo + part * jstep; jj < nJ; jj += gb_parts * jstep) {
        const double2* row = bh64 + jj * R;
        const double2 br0 = row[r0], br1 = row[r1], bq0 = row[q0], bq1 = row[q1];
        a00 = zfma_cj(br0, bq0, a00);
        a01 = zfma_cj(br0, bq1, a01);
        a10 = zfma_cj(br1, bq0, a10);
        a11 = zfma_cj(br1, bq1, a11);
      }
    }
    double2* dst = gbt + 4 * (size_t)it;
    dst[0] = a00;
    dst[1] = a01;
    dst[2] = a10;
    dst[3] = a11;
  }
  __syncthreads();
  for (int e = tid; e < Rp; e += NT) {
    const int ij = tab[e];
    const int r = ij >> 8, q = ij & 255;
    const int t = tri_idx(r >> 1, q >> 1), sub = ((r & 1) << 1) | (q & 1);
    double2 acc = gbt[4 * t + sub];
    for (int part = 1; part < gb_parts; ++part) acc = zadd(acc, gbt[4 * ((size_t)part * gb_nt + t) + sub]);
    __stcg(&dst_g[e].x, acc.x);
    __stcg(&dst_g[e].y, acc.y);
  }
}

// ---------------------------------------------------------------- the kernel
// SOLV: the one solver compiled in (1 / 2 / 5: Gauss-Jordan entries per thread, 9: 2x2-blocked LDL^H);
// SHARD: whether the row-sharding phases are compiled in; TIGHT: the tight shared-memory plan
// (rows_make_plan_cap). Every inlined variant costs instruction-cache lines in the frame loop,
// so each launch gets only the code it runs.
template <int SOLV, bool SHARD, bool TIGHT = false>
__global__ void __launch_bounds__(ROWS_NT, 1) tt_rows_kernel(const __grid_constant__ tt_rows_args a,
                                                             const __grid_constant__ RowsPlan pl) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, NT = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int CL = pl.CL;
  const int c = (int)(blockIdx.x % CL);
  const int qid = (int)(blockIdx.x / CL);  // cluster index: slice, or rank of a local multi-rank launch
  const int nx = a.nx, ny = a.ny, R = a.rank, Smax = a.max_rows, Rp = pl.Rp;
  // row sharding: this rank holds k-space rows [R0, R0 + nxs) of Ah (all rows when off). With
  // shard_local every rank of the sharding is a cluster of this launch (one GPU, several clusters);
  // each reads the full Ah at its row offset, has its own scratch and payload slot, and only rank 0
  // writes the replicated outputs (Bh, gamma, cost, step state).
  const bool shard = SHARD && a.shard_world > 0;
  const bool multi = shard && a.shard_local != 0;
  const int s = multi ? 0 : qid;  // slice
  const int srank = multi ? qid : a.shard_rank;
  const bool lead = !multi || qid == 0;
  // fused: one cooperative launch runs both phases of every frame, the payload reduced in-kernel between
  // two inter-cluster barriers; payload slots double-buffered by frame parity
  const bool fused = multi && a.shard_fused != 0;
  unsigned gsync_gen = 0;
  // fused: the replicated Bh's GB partial Gram is split across the ranks (rank q takes the columns
  // jj = q (mod world) of every CTA's block) and summed with the payload
  const int gb_jo = fused ? qid : 0, gb_js = fused ? a.shard_world : 1;
  const int R0 = shard ? part_begin(nx, a.shard_world, srank) : 0;
  const int nxs = shard ? part_begin(nx, a.shard_world, srank + 1) - R0 : nx;
  const int i0 = R0 + part_begin(nxs, CL, c), nI = part_begin(nxs, CL, c + 1) - part_begin(nxs, CL, c);
  const int aoff = i0 - R0;  // first own row inside the rank's Ah buffers
  const size_t arow = multi ? (size_t)i0 : (size_t)s * nxs + aoff;  // first own row in ah_in / ah_out
  const int j0 = part_begin(ny, CL, c), nJ = part_begin(ny, CL, c + 1) - j0;
  const int KT = pl.KT;

  float2* ahl = (float2*)(smem + pl.o_ahl);
  float2* bhl = (float2*)(smem + pl.o_bhl);
  double2* G = (double2*)(smem + pl.o_u1);
  double* pbuf = (double*)(smem + pl.o_u1);
  double* cdf = pbuf + nx;
  double2* gaf = (double2*)(smem + pl.o_gaf);  // full Hermitian GA, GB (fp64, row-major)
  double2* gbf = (double2*)(smem + pl.o_gbf);
  double2* gam = (double2*)(smem + pl.o_vec);
  double2* hv = gam + R;
  double2* hsave = hv + R;
  double* nrm = (double*)(hsave + R);
  double* inrm = nrm + R;
  double* inv = inrm + R;
  double* gda = inv + R;
  double* gdb = gda + R;
  float2* gamf = (float2*)(gdb + R);
  double* scal = (double*)(gamf + R);  // 16 scalars
  double2* colb = (double2*)(scal + 16);
  double* blk = (double*)(colb + 4 * (R + 1));
  double2* zf = (double2*)(blk + 4 * (R / 2 + 1));
  unsigned short* tab = (unsigned short*)(smem + pl.o_tab);
  int* flags = (int*)(smem + pl.o_flags);
  int* rows = (int*)(smem + pl.o_rows);
  int* forced = (int*)(smem + pl.o_forced);
  double* usm = (double*)(smem + pl.o_usm);
  int* own_k = (int*)(smem + pl.o_own);  // sampled rows owned by this CTA: measurement index
  int* own_li = own_k + pl.nIm;          // and local row
  double2* wacc = (double2*)(smem + pl.o_wacc);
  double2* zs = (double2*)(smem + pl.o_zs);
  float2* zs32 = (float2*)(smem + pl.o_u2);  // tight plan: the P increments (U2 is free from B4 on)
  float2* red2 = (float2*)(smem + pl.o_red2);     // fp32 K-split partials (corrections)
  double2* red2d = (double2*)(smem + pl.o_red2);  // fp64 K-split partials (W, Z)
  float2* ys = (float2*)(smem + pl.o_u2);                   // [KT][ysr] the frame's Y rows (own columns)
  double2* ahs64 = (double2*)(ys + (size_t)KT * pl.ysr);    // [KT][R] the frame's Ah_S rows, fp64
  float2* ahs = (float2*)ahs64;                             // scratch of write_residual
  // phase (a) only: Bh in fp64 (not in the tight plan), GB partial tiles [parts][tiles][4], then the
  // colnorm partials [parts][R]
  const int gb_rt = (R + 1) >> 1, gb_nt = gb_rt * (gb_rt + 1) / 2;  // 2 x 2 tiles of the lower triangle
  // one packed entry per thread unless that leaves threads idle over a long column block (config 3)
  const bool gb_tiled = nJ * R >= 1024 && Rp <= NT;
  const int gb_parts = max(1, (NT + gb_nt / 2) / gb_nt);
  double2* bh64 = (double2*)(smem + pl.o_bh64);  // fp64 copy of the Bh rows (not in the tight plan)
  double2* gbt = (double2*)(smem + pl.o_u2);
  double* cnp = (double*)(gbt + 4 * (size_t)max(2 * NT, gb_nt));
  float2* vop = (float2*)(smem + pl.o_u2);              // update only: gamma-scaled GEMM operand
  double* red = (double*)(smem + pl.o_red);
  (void)inv;
  __shared__ int sh_S, sh_err, sh_own, sh_amb, sh_Sglob;
  __shared__ __align__(8) unsigned long long ybar;  // completion of the frame's bulk Y-row copies
  long long* pclk = (a.phase_clock != nullptr && blockIdx.x == 0) ? (long long*)a.phase_clock : nullptr;
  // branch-free (a lane-0 branch would leave warp 0 diverged and send later shuffles down the slow path)
#define STAMP(k)                                                                                   \
  do {                                                                                             \
    if (pclk != nullptr) stamp_if(tid == 0, pclk + (size_t)it * 32 + (k));                          \
  } while (0)

  // global scratch for this slice
  const RowsScratch L = rows_scratch_layout(nx, ny, R, Smax, CL);
  unsigned char* sb = (unsigned char*)a.scratch + (size_t)(multi ? qid : s) * L.per_slice;
  double* g_cn = (double*)(sb + L.cn);
  double2* g_gbp = (double2*)(sb + L.gbp);
  double2* g_gb = (double2*)(sb + L.gb);
  double2* g_ga = (double2*)(sb + L.ga);
  double* g_sraw = (double*)(sb + L.sraw);
  float2* g_ahs = (float2*)(sb + L.ahs);
  double2* g_zp = (double2*)(sb + L.zp);
  double2* g_hp = (double2*)(sb + L.hp);
  double* g_yn = (double*)(sb + L.yn);
  double* g_unif = (double*)(sb + L.unif);

  // ---- load resident state and constants once
  {
    const float2* src = (const float2*)a.ah_in + arow * R;
    for (int o = tid; o < nI * R; o += NT) ahl[o] = src[o];
    const float2* srb = (const float2*)a.bh_in + ((size_t)s * ny + j0) * R;
    for (int o = tid; o < nJ * R; o += NT) {
      bhl[o] = srb[o];
      if (!TIGHT) bh64[o] = to_d2(srb[o]);
    }
    if (a.policy == TT_POLICY_INFORMATIVE)
      for (int m = tid; m < a.nforced; m += NT) forced[m] = a.forced[m];
  }
  ldl_table_init(tab, R);
  // Y rows by bulk copy (TMA) when every row segment is 16-byte aligned and sized, else cp.async
  // (host truth: 8-byte cp.async reads of the sampled rows over the host link; the bulk copies take device
  // memory)
  const bool y_bulk = !a.y_host && (nJ & 1) == 0 && (j0 & 1) == 0 && (ny & 1) == 0 && ((size_t)a.ysrc & 15) == 0 &&
                      (size_t)KT * nJ * sizeof(float2) < (1u << 20);
  unsigned yph = 0;
  if (tid == 0) {
    mbar_init(&ybar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_proxy_async_smem();
  // forced lines among this thread's rows of the block-wide draw (bits, registers for the whole launch)
  unsigned fmask = 0u;
  int top = 1;  // largest power of two <= nx (binary search of the CDF)
  while (2 * top <= nx) top *= 2;
  const double inx = 1.0 / (double)nx;
  if (a.policy == TT_POLICY_INFORMATIVE && nx <= 4 * NT) {
    const int ipt = (nx + NT - 1) / NT, r0 = tid * ipt;
    for (int m = 0; m < a.nforced; ++m) {
      const int d = a.forced[m] - r0;
      if (d >= 0 && d < ipt && r0 + d < nx) fmask |= 1u << d;
    }
  }
  double alpha_bar = a.alpha_bar ? a.alpha_bar[s] : 0.0;
  const double ncap2 = a.norm_cap * a.norm_cap;
  bool prev_upd = false;  // norm_cap: whether the previous frame updated the state
  uint64_t ppos = (a.policy == TT_POLICY_INFORMATIVE && a.philox_pos) ? a.philox_pos[s] : 0ull;
  int status = 0;
  const int eb = part_begin(Rp, CL, c), ee = part_begin(Rp, CL, c + 1);
  const int cparts = NT / R;  // column-norm partial sums per column
  __syncthreads();

  for (int it = 0; it < (fused ? 2 * a.frames : a.frames); ++it) {
    const int f = fused ? it >> 1 : it;
    // 0 full step, 1 partials -> payload, 2 payload -> update
    const int phase = !shard ? 0 : fused ? 1 + (it & 1) : a.shard_phase;
    const size_t xgl = (size_t)Rp * (fused ? 4 : 2) + 2;  // fused slots also carry GB: [GA][2 scalars][GB]
    double2* xwp = (double2*)a.xw + (fused ? (size_t)(f & 1) * a.shard_world * ny * R : 0);
    double* xgp = a.xg + (fused ? (size_t)(f & 1) * a.shard_world * xgl : 0);
    auto xg_at = [&](size_t k) { return __ldcg(xgp + k); };  // the reduced payload (slot 0)
    const long long t = a.t0 + f;
    const double lt = a.lam / (double)t;
    STAMP(0);
    int S = 0;
    int Sglob = 0;  // measurements of the whole frame (S becomes this rank's share under row sharding)
    const int ndraw = a.policy == TT_POLICY_INFORMATIVE ? max(a.k_draws - a.nforced, 0) : 0;
    const uint64_t k1s = a.key1 + (uint64_t)s;
    if (phase != 2) {
    // ======== (a) column-norm partials of Ah (own rows), Bh staged in fp64, packed GB partials
    if (tid < cparts * R) {
      const int r = tid % R, part = tid / R;
      double acc = 0.0;
      for (int li = part; li < nI; li += cparts) {
        const float2 v = ahl[li * R + r];
        acc += (double)v.x * v.x + (double)v.y * v.y;
      }
      cnp[part * R + r] = acc;
    }
    __syncthreads();
    if (tid < R) {
      double acc = 0.0;
      for (int part = 0; part < cparts; ++part) acc += cnp[part * R + tid];
      __stcg(&g_cn[c * R + tid], acc);
    }
    STAMP(26);
    // GB partial over own columns: wide column blocks tiled (gb_partials_tiled), narrow ones one
    // packed entry per thread
    if (gb_tiled) {
      gb_partials_tiled<TIGHT>(bhl, bh64, R, nJ, Rp, gb_nt, gb_parts, tab, gbt, g_gbp + (size_t)c * Rp, gb_jo, gb_js);
    } else if (!TIGHT && Rp > NT && gb_js == 1) {
      // large ranks (config 4: R = 32, 528 packed entries over 256 threads) on the fp64 tensor cores: the full
      // R x R product over the own rows, the lower triangle kept (the same exact products, another K order)
      zgemm_dmma<ZG>(R, R, nJ, bh64, 1, R, bh64, R, 1, RowsEpiGB{g_gbp + (size_t)c * Rp});
    } else {
      for (int e = tid; e < Rp; e += NT) {
        const int ij = tab[e];
        const int r = ij >> 8, q = ij & 255;
        double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
        int jj = gb_jo;
        if (TIGHT) {
          for (; jj + gb_js < nJ; jj += 2 * gb_js) {
            acc = zfma_cj(bhl[jj * R + r], bhl[jj * R + q], acc);
            acc2 = zfma_cj(bhl[(jj + gb_js) * R + r], bhl[(jj + gb_js) * R + q], acc2);
          }
          if (jj < nJ) acc = zfma_cj(bhl[jj * R + r], bhl[jj * R + q], acc);
        } else {
          for (; jj + gb_js < nJ; jj += 2 * gb_js) {
            acc = zfma_cj(bh64[jj * R + r], bh64[jj * R + q], acc);
            acc2 = zfma_cj(bh64[(jj + gb_js) * R + r], bh64[(jj + gb_js) * R + q], acc2);
          }
          if (jj < nJ) acc = zfma_cj(bh64[jj * R + r], bh64[jj * R + q], acc);
        }
        acc = zadd(acc, acc2);
        __stcg(&g_gbp[(size_t)c * Rp + e].x, acc.x);
        __stcg(&g_gbp[(size_t)c * Rp + e].y, acc.y);
      }
    }
    if (ndraw > 0 && f % ROWS_UF == 0) {
      // Philox uniforms of the next ROWS_UF frames (stream positions are state independent), split
      // over the cluster; the barrier below publishes them. Saves a Philox block per draw per frame.
      const int nf = min(ROWS_UF, a.frames - f);
      for (int it = c * NT + tid; it < nf * ndraw; it += CL * NT)
        __stcg(&g_unif[it], philox_uniform(a.key0, k1s, ppos + (uint64_t)it));
    }
    STAMP(1);
    cluster_barrier();  // ---------------------------------------------- B1
    STAMP(2);
    for (int e = eb + tid - 32; tid >= 32 && e < ee; e += NT - 32) {
      const double2 g = sum_parts2(g_gbp + e, (size_t)Rp, CL);
      double* dst = fused ? xgp + (size_t)qid * xgl + 2 * Rp + 2 + 2 * e : (double*)&g_gb[e];  // rank's share
      __stcg(dst, g.x);
      __stcg(dst + 1, g.y);
    }
    for (int m = tid; m < ndraw; m += NT) usm[m] = __ldcg(&g_unif[(f % ROWS_UF) * ndraw + m]);  // in flight with
    for (int r = tid; r < R && tid < 32; r += 32) {                                                // the norm sums
      const double n2 = sum_parts(g_cn + r, (size_t)R, CL);
      nrm[r] = n2;
      inrm[r] = n2 > 0.0 ? fast_rcp(n2) : 0.0;
    }
    STAMP(24);
    if (tid == 0) sh_err = 0;
    __syncthreads();
    STAMP(27);

    }  // phase != 2
    if (a.policy == TT_POLICY_INFORMATIVE) {
      // row sharding: every rank draws the frame's rows from the same full raw-score vector (sraw_in,
      // built from the all-gathered row energies); otherwise each CTA scores its own rows
      const double* sraw = a.sraw_in ? a.sraw_in : g_sraw;
      if (!a.sraw_in) {
      // raw row scores for own rows (sampler.py:77-85, :126)
      const double cs = (double)ny, cr = (double)R, cd = 1.0 / ((double)R * (double)(nx + ny));
      if (nI * 2 <= NT) {
        // short row blocks (config 2): tpr lanes per row (rank terms split, fixed-order butterfly), so the
        // fp64 chain is R / tpr long
        int tpr = 32;
        while (tpr > 1 && tpr * nI > NT) tpr >>= 1;
        const int sub = lane & (tpr - 1);
        for (int base = 0; base < nI; base += NT / tpr) {  // uniform trip count (full-warp shuffles)
          const int i = base + tid / tpr;
          double e = 0.0;
          if (i < nI)
            for (int r = sub; r < R; r += tpr) {
              const float2 v = ahl[i * R + r];
              e = fma((double)v.x * v.x + (double)v.y * v.y, inrm[r], e);
            }
          for (int o = 1; o < tpr; o <<= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
          if (sub == 0 && i < nI) __stcg(&g_sraw[i0 + i], (cs * e + cr) * cd);
        }
      } else {
        // long row blocks (config 3): a row per thread, the rank terms from a row-dependent start so the
        // lanes of a warp spread over the shared-memory banks (rows are R complex apart: one bank otherwise)
        for (int i = tid; i < nI; i += NT) {
          const float2* rowp = ahl + i * R;
          double e = 0.0;
          int r = (i0 + i) % R;
          for (int k = 0; k < R; ++k) {
            const float2 v = rowp[r];
            e = fma((double)v.x * v.x + (double)v.y * v.y, inrm[r], e);
            r = r + 1 == R ? 0 : r + 1;
          }
          __stcg(&g_sraw[i0 + i], (cs * e + cr) * cd);
        }
      }
      if (tid < R && nrm[tid] == 0.0) atomicOr(&sh_err, TT_ST_ZEROCOL);
      STAMP(3);
      cluster_barrier();  // -------------------------------------------- B2
      }
      STAMP(4);
      const bool wor = a.draw_wor != 0;
      if (nx <= 4 * NT && !wor) {
        // Block-wide probabilities -> CDF -> draws -> sorted union, every warp busy (sampler.py:88-92,
        // :146-162). Thread t owns rows [r0, r1) (consecutive). One scan of the raw scores s gives
        // the blended CDF in closed form: with w1 = (1-beta)/sum(s), w0 = beta/nx,
        //   cdf_i = (w1 C_i + w0 (i+1)) / (w1 sum(s) + w0 nx),  C_i = s_0 + .. + s_i
        // (numpy's cumsum(p) / cdf[-1] up to rounding; the 1e-12 guard below covers the difference).
        const int ipt = (nx + NT - 1) / NT;
        const int r0 = min(nx, tid * ipt), r1 = min(nx, r0 + ipt);
        double sv[4], cv[4];
        double loc = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          sv[j] = (j < ipt && r0 + j < r1) ? __ldcg(&sraw[r0 + j]) : 0.0;
          loc += sv[j];
        }
        double S1;
        double run = block_excl_scan_dbl(loc, red, S1);
        const double w1 = (1.0 - a.beta) * fast_rcp(S1), w0 = a.beta * inx;
        const double il = fast_rcp(fma(w1, S1, w0 * (double)nx));
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j < ipt && r0 + j < r1) {
            run += sv[j];
            cv[j] = fma(w1, run, w0 * (double)(r0 + j + 1)) * il;
            cdf[r0 + j] = cv[j];
            pbuf[r0 + j] = fma(sv[j], w1, w0);  // probabilities for the exact fallback
            flags[r0 + j] = 0;
          }
        }
        if (tid == 0) sh_amb = 0;
        __syncthreads();
        STAMP(29);
        // draws, one per thread: idx = searchsorted(cdf, u, 'right') by a branch-free binary search
        for (int m = tid; m < ndraw; m += NT) {
          const double u = usm[m];
          int pos = -1;  // last index with cdf <= u
          for (int step = top; step > 0; step >>= 1) {
            const int cand = pos + step;
            if (cand < nx && cdf[cand] <= u) pos = cand;
          }
          const int idx = min(pos + 1, nx - 1);
          const double lo = idx > 0 ? cdf[idx - 1] : -1.0;
          if (u - lo <= 1e-12 || (idx < nx - 1 && cdf[idx] - u <= 1e-12)) sh_amb = 1;
          flags[idx] = 1;
        }
        __syncthreads();
        STAMP(30);
        unsigned hit = fmask;  // forced lines (np.union1d)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < ipt && r0 + j < r1 && flags[r0 + j]) hit |= 1u << j;
        int tot;
        int o = block_excl_scan_int(__popc(hit), (int*)red, tot);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (hit & (1u << j)) rows[o++] = r0 + j;
        if (tid == 0) sh_S = tot;
        STAMP(31);
      }
      if (nx > 4 * NT || wor || sh_amb) {
        // generic width, or a uniform within 1e-12 of a CDF boundary: numpy's sequential cumsum
        // of the probabilities, cdf /= cdf[-1], per-draw searchsorted, forced union, compaction;
        // draws without replacement: the sequential renormalised draws over the same probabilities
        if (nx > 4 * NT || wor) {
          for (int i = tid; i < nx; i += NT) pbuf[i] = __ldcg(&sraw[i]);
          __syncthreads();
          double S1;
          const double loc = block_sum_range(pbuf, nx, red, S1);
          (void)loc;
          const double w1 = (1.0 - a.beta) / S1, w0 = a.beta / (double)nx;
          for (int i = tid; i < nx; i += NT) pbuf[i] = fma(pbuf[i], w1, w0);
        }
        __syncthreads();
        if (wor) {
          rows_draw_wor(pbuf, cdf, flags, nx, ndraw, usm, forced, a.nforced, red);
        } else {
          if (tid == 0) {
            double cacc = 0.0;
            for (int i = 0; i < nx; ++i) {
              cacc += pbuf[i];
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
          for (int m = lane; m < a.nforced; m += 32) {
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
          if (lane == 31) sh_S = x;
        }
      }
      ppos += (uint64_t)max(a.k_draws - a.nforced, 0);
      if (shard) {
        // the frame's full row set -> rows_out / cnt_out (the host hands it to phase 2 as its static
        // table), then keep this rank's rows like a static table
        __syncthreads();
        const int Sall = sh_S;
        Sglob = Sall;
        if (c == 0) {
          for (int k = tid; a.rows_out && k < Smax; k += NT) a.rows_out[k] = k < Sall ? rows[k] : -1;
          if (tid == 0 && a.cnt_out) a.cnt_out[0] = Sall;
        }
        __syncthreads();
        if (warp == 0) {
          int cnt = 0;
          for (int base = 0; base < Sall; base += 32) {
            const int k = base + lane;
            const int i = k < Sall ? rows[k] : -1;
            const bool keep = i >= R0 && i < R0 + nxs;
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            __syncwarp();
            if (keep) rows[cnt + __popc(m & ((1u << lane) - 1u))] = i;
            cnt += __popc(m);
            __syncwarp();
          }
          if (lane == 0) sh_S = cnt;
        }
      }
      STAMP(20);
    } else if (fused && phase == 2) {
      // the frame's row table (this rank's share, filtered in phase 1) is still in shared memory
      Sglob = sh_Sglob;
    } else {
      if (tid == 0) sh_err = 0;
      __syncthreads();
      S = load_static_rows(a, f, s, rows, flags, &sh_err);
      Sglob = S;
      if (tid == 0) sh_Sglob = S;
      if (shard && warp == 0) {
        // keep only this rank's rows, in measurement order (the other ranks take the rest)
        int cnt = 0;
        for (int base = 0; base < S; base += 32) {
          const int k = base + lane;
          const int i = k < S ? rows[k] : -1;
          const bool keep = i >= R0 && i < R0 + nxs;
          const unsigned m = __ballot_sync(0xffffffffu, keep);
          __syncwarp();
          if (keep) rows[cnt + __popc(m & ((1u << lane) - 1u))] = i;
          cnt += __popc(m);
          __syncwarp();
        }
        if (lane == 0) sh_S = cnt;
      } else if (tid == 0) {
        sh_S = S;
      }
    }
    fence_proxy_async_smem();  // this frame's generic accesses of U2 before the bulk copies into it
    __syncthreads();
    STAMP(5);
    S = sh_S;
    if (!shard) Sglob = S;
    status |= sh_err;
    // K parts of the Z GEMM: enough items for the block, the same count in every CTA of the cluster (the
    // rows' owners sum CL * zks partial slots)
    int zks;
    {
      const int zM = min(KT, max(S, 1));
      if (TIGHT) {  // CUDA-core tiles, one per thread
        const int ztiles = ((zM + ZTM - 1) / ZTM) * ((R + ZTN - 1) / ZTN);
        zks = max(1, min(NT / ztiles, min(ROWS_ZKS, pl.nJm / 4)));
      } else {      // DMMA items (4 M blocks x 1 r block), one per warp
        const int items = ((((zM + 7) >> 3) + ZGZ - 1) / ZGZ) * ((R + 3) >> 2);
        zks = max(1, min((NT / 32) / items, min(ROWS_ZKS, (pl.nJm + 3) / 4)));
      }
    }

    const bool gather = a.y_mode == TT_Y_GATHER;
    const float2* ybase = gather ? (const float2*)a.ysrc + (size_t)f * a.y_frame_stride + (size_t)s * a.y_slice_stride + j0
                                 : (const float2*)a.ysrc + ((size_t)f * a.nslices + s) * Smax * ny + j0;
    // Y rows [k0, k0 + kt) of this CTA's columns into the k tile: one bulk copy per row issued by warp 0
    // (completion on ybar), or 8-byte cp.async by every thread
    auto issue_y = [&](int k0, int kt) {
      if (kt <= 0 || nJ <= 0) return;
      if (y_bulk) {
        // the rows dealt round robin to the warps: a warp issues its bulk copies one lane after the other
        // (~90 cycles each), so one issuing warp held the block at the next barrier for ~2k cycles per frame.
        // The one arrival carries the tile's byte count; copies of other warps may complete before it (the
        // transaction count goes negative until then, the phase still needs the arrival).
        if (tid == 0) mbar_arrive_expect_tx(&ybar, (unsigned)(kt * nJ * sizeof(float2)));
        const int nwarps = NT >> 5;
        for (int kk = warp + nwarps * lane; kk < kt; kk += NT)
          bulk_g2s(&ys[(size_t)kk * pl.ysr], ybase + (size_t)(gather ? rows[k0 + kk] : k0 + kk) * ny,
                   (unsigned)(nJ * sizeof(float2)), &ybar);
      } else {
        for (int o = tid; o < kt * nJ; o += NT) {
          const int kk = idiv(o, nJ), jj = o - kk * nJ;
          cp_async8(&ys[kk * pl.ysr + jj], ybase + (size_t)(gather ? rows[k0 + kk] : k0 + kk) * ny + jj);
        }
      }
    };
    auto wait_y = [&](int kt) {
      if (kt <= 0 || nJ <= 0) return;
      if (y_bulk) {
        mbar_wait(&ybar, yph);
        yph ^= 1u;
      } else {
        cp_async_wait_all();
      }
    };
    if (phase != 2) issue_y(0, min(KT, S));  // the first Y tile in flight before the publish below
    // ======== (b) publish own sampled rows of Ah; list them
    if (tid == 0) sh_own = 0;
    for (int li = tid; li < nI; li += NT) flags[li] = -1;
    __syncthreads();
    for (int k = tid; k < S; k += NT) {
      const int i = rows[k];
      if (i >= i0 && i < i0 + nI) flags[i - i0] = k;
    }
    for (int o = tid; phase != 2 && o < S * R; o += NT) {
      const int k = idiv(o, R), r = o - k * R;
      const int i = rows[k];
      if (i >= i0 && i < i0 + nI) {
        const float2 v = ahl[(i - i0) * R + r];
        __stcg(&g_ahs[(size_t)k * R + r].x, v.x);
        __stcg(&g_ahs[(size_t)k * R + r].y, v.y);
      }
    }
    STAMP(6);
    cluster_arrive();  // ------------------------------------------------ B3 (split)

    for (int o = tid; o < nJ * R; o += NT) wacc[o] = make_double2(0.0, 0.0);
    for (int e = eb + tid; e < ee; e += NT) G[e - eb] = make_double2(0.0, 0.0);
    __syncthreads();  // row marks visible to warp 0
    if (warp == 0) {  // compact the owned sampled rows (ascending local row)
      const int chunk = (nI + 31) / 32;
      const int q0 = min(nI, lane * chunk), q1 = min(nI, q0 + chunk);
      int cnt = 0;
      for (int li = q0; li < q1; ++li) cnt += flags[li] >= 0;
      int x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      int o = x - cnt;
      for (int li = q0; li < q1; ++li)
        if (flags[li] >= 0) {
          own_k[o] = flags[li];
          own_li[o] = li;
          flags[li] = o;  // local row -> position in the owned list
          ++o;
        }
      if (lane == 31) sh_own = x;
    }
    // ======== (c) heavy phase: W, Z partials, GA (own entries), ||Y||^2
    double ysq = 0.0;
    const bool one_tile = phase != 2 && S > 0 && S <= KT;
    if (one_tile) {
      // all sampled rows in one tile: the Z partial needs only Y and the resident Bh, so it runs inside
      // the B3 window; B3 completes, Ah_S arrives and GA / W follow. Z and W share one GEMM call site.
      wait_y(S);
      __syncthreads();
      STAMP(16);
      for (int o = tid; o < S * nJ; o += NT) {
        const int kk = idiv(o, nJ), jj = o - kk * nJ;
        const float2 v = ys[kk * pl.ysr + jj];
        ysq += (double)v.x * v.x + (double)v.y * v.y;
      }
      for (int gsel = 0; gsel < 2; ++gsel) {
        const bool z = gsel == 0;
        if (!z) {
          cluster_wait();  // ------------------------------------------------ B3 complete
          for (int o = tid; o < S * R; o += NT) {
            float2 v;
            v.x = __ldcg(&g_ahs[o].x);
            v.y = __ldcg(&g_ahs[o].y);
            ahs64[o] = to_d2(v);
          }
          __syncthreads();
          const int nq = 4 * (ee - eb);  // GA own packed entries (4-way k split, fixed-order quad sum)
          for (int base = tid & ~31; base < nq; base += NT) {  // warp-uniform trip count
            const int eq = base + lane;
            const int e = eb + (eq >> 2), part = eq & 3;
            double2 g = make_double2(0.0, 0.0);
            if (eq < nq) {
              const int ij = tab[e];
              const int r = ij >> 8, q = ij & 255;
              for (int kk = part; kk < S; kk += 4) g = zfma_cj(ahs64[kk * R + r], ahs64[kk * R + q], g);
            }
            g.x += __shfl_xor_sync(0xffffffffu, g.x, 1);
            g.y += __shfl_xor_sync(0xffffffffu, g.y, 1);
            g.x += __shfl_xor_sync(0xffffffffu, g.x, 2);
            g.y += __shfl_xor_sync(0xffffffffu, g.y, 2);
            if (part == 0 && eq < nq) G[e - eb] = zadd(G[e - eb], g);
          }
          STAMP(18);
        }
        if (z) {  // Z partial over own columns, K split into zks parts delivered to L2 as they are
          const RowsEpiD epi{EPI_Z_STORE, R, wacc, g_zp + (size_t)c * zks * Smax * R, Smax * R};
          if (TIGHT)
            zgemm_fd<ZTM, ZTN, true, true>(S, R, nJ, ys, pl.ysr, 1, bhl, R, 1, zks, red2d, epi);
          else
            zgemm_dmma<ZGZ>(S, R, nJ, ys, pl.ysr, 1, bh64, R, zks, epi);
        } else {
          const RowsEpiD epi{EPI_W_ACC, R, wacc, nullptr, 0};
          if (TIGHT)
            zgemm_fd<ZTM, ZTN, true, false>(nJ, R, S, ys, 1, pl.ysr, ahs64, R, 1,
                                            gemm_split(nJ, R, S, ZTM, ZTN, pl.red_cap), red2d, epi);
          else
            zgemm_dmma<ZG>(nJ, R, S, ys, 1, pl.ysr, ahs64, R, 1, epi);
        }
        __syncthreads();
        STAMP(z ? 17 : 19);
      }
    } else {
      cluster_wait();  // ---------------------------------------------------- B3 complete
    }
    __syncthreads();  // warp 0's owned-row list (written after its arrive) is visible to all warps
    STAMP(7);
    const int nown = sh_own;

    for (int k0 = 0; !one_tile && phase != 2 && k0 < S; k0 += KT) {  // general case: several k tiles
      const int kt = min(KT, S - k0);
      if (k0 > 0) issue_y(k0, kt);
      for (int o = tid; o < kt * R; o += NT) {
        float2 v;
        v.x = __ldcg(&g_ahs[(size_t)(k0) * R + o].x);
        v.y = __ldcg(&g_ahs[(size_t)(k0) * R + o].y);
        ahs64[o] = to_d2(v);
      }
      __syncthreads();
      // GA own packed entries first: they need only Ah_S, so they run while the Y rows are in flight
      // (4-way k split per entry, fixed-order quad reduction)
      {
        const int nq = 4 * (ee - eb);
        for (int base = tid & ~31; base < nq; base += NT) {  // warp-uniform trip count
          const int eq = base + lane;
          const int e = eb + (eq >> 2), part = eq & 3;
          double2 g = make_double2(0.0, 0.0);
          if (eq < nq) {
            const int ij = tab[e];
            const int r = ij >> 8, q = ij & 255;
            for (int kk = part; kk < kt; kk += 4) g = zfma_cj(ahs64[kk * R + r], ahs64[kk * R + q], g);
          }
          g.x += __shfl_xor_sync(0xffffffffu, g.x, 1);
          g.y += __shfl_xor_sync(0xffffffffu, g.y, 1);
          g.x += __shfl_xor_sync(0xffffffffu, g.x, 2);
          g.y += __shfl_xor_sync(0xffffffffu, g.y, 2);
          if (part == 0 && eq < nq) G[e - eb] = zadd(G[e - eb], g);
        }
      }
      wait_y(kt);
      __syncthreads();
      if (k0 == 0) STAMP(16);
      for (int o = tid; o < kt * nJ; o += NT) {
        const int kk = idiv(o, nJ), jj = o - kk * nJ;
        const float2 v = ys[kk * pl.ysr + jj];
        ysq += (double)v.x * v.x + (double)v.y * v.y;
      }
      // W[jj][r] += sum_k Y[k][jj] conj(Ah_S[k][r]), then the Z partial over own columns
      // Z[k][r] = sum_jj Y[k][jj] conj(Bh[jj][r]): one call site, so one copy of the GEMM code
      for (int gsel = 0; gsel < 2; ++gsel) {
        const bool w = gsel == 0;
        if (w) {
          const RowsEpiD epi{EPI_W_ACC, R, wacc, nullptr, 0};
          if (TIGHT)
            zgemm_fd<ZTM, ZTN, true, false>(nJ, R, kt, ys, 1, pl.ysr, ahs64, R, 1,
                                            gemm_split(nJ, R, kt, ZTM, ZTN, pl.red_cap), red2d, epi);
          else
            zgemm_dmma<ZG>(nJ, R, kt, ys, 1, pl.ysr, ahs64, R, 1, epi);
        } else {
          const RowsEpiD epi{EPI_Z_STORE, R, wacc, g_zp + ((size_t)c * zks * Smax + k0) * R, Smax * R};
          if (TIGHT)
            zgemm_fd<ZTM, ZTN, true, true>(kt, R, nJ, ys, pl.ysr, 1, bhl, R, 1, zks, red2d, epi);
          else
            zgemm_dmma<ZGZ>(kt, R, nJ, ys, pl.ysr, 1, bh64, R, zks, epi);
        }
        if (w) __syncthreads();  // the K-split buffer is reused
      }
      if (k0 == 0) STAMP(18);
      if (k0 == 0) STAMP(19);
      fence_proxy_async_smem();  // the tile's generic reads before the next tile's bulk copies
      __syncthreads();
    }
    STAMP(8);
    if (phase == 1) {
      // this rank's partials -> payload (the caller all-reduces xw and xg across ranks)
      double2* xw1 = xwp + (multi ? (size_t)qid * ny * R : 0);  // this rank's payload slot
      double* xg1 = xgp + (multi ? (size_t)qid * xgl : 0);
      for (int o = tid; o < nJ * R; o += NT) xw1[(size_t)j0 * R + o] = wacc[o];
      for (int e = eb + tid; e < ee; e += NT) {
        xg1[2 * e] = G[e - eb].x;
        xg1[2 * e + 1] = G[e - eb].y;
      }
      if (warp == 0) {  // this rank's ||Ah||^2, fixed order
        double v = 0.0;
        for (int r = lane; r < R; r += 32) v += nrm[r];
        v = warp_sum(v);
        if (lane == 0) scal[1] = v;
      }
      const double yt = block_sum(ysq, red);
      if (tid == 0) __stcg(&g_yn[c], yt);
      cluster_barrier();
      if (c == 0 && tid == 0) {
        xg1[2 * Rp] = sum_parts(g_yn, 1, CL);
        xg1[2 * Rp + 1] = scal[1];  // this rank's ||Ah||^2
      }
      if (fused) {
        // every rank's slot written -> fixed-order sum into slot 0 (tt_rows_shard_reduce's arithmetic),
        // split over all CTAs of the launch (four elements per thread in flight) -> phase 2
        grid_sync(a.grid_sync, gsync_gen);
        const size_t nw = 2 * (size_t)ny * R, ntot = nw + xgl, step = (size_t)gridDim.x * NT;
        double* xwf = (double*)xwp;
        for (size_t i0r = (size_t)blockIdx.x * NT + tid; i0r < ntot; i0r += 4 * step) {
          double v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const size_t i = i0r + u * step;
            v[u] = 0.0;
            if (i < nw) {
              double x = __ldcg(xwf + i);
              for (int r = 1; r < a.shard_world; ++r) x += __ldcg(xwf + (size_t)r * nw + i);
              v[u] = x;
            } else if (i < ntot) {
              const size_t k = i - nw;
              double x = __ldcg(xgp + k);
              for (int r = 1; r < a.shard_world; ++r) x += __ldcg(xgp + (size_t)r * xgl + k);
              v[u] = x;
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const size_t i = i0r + u * step;
            if (i < nw) __stcg(xwf + i, v[u]);
            else if (i < ntot) __stcg(xgp + (i - nw), v[u]);
          }
        }
        grid_sync(a.grid_sync, gsync_gen);
      }
      continue;  // phase 2 finishes the frame after the all-reduce
    }
    if (phase == 2)  // reduced W of this CTA's columns
      for (int o = tid; o < nJ * R; o += NT) {
        const double2* src = xwp + (size_t)j0 * R + o;
        wacc[o] = make_double2(__ldcg(&src->x), __ldcg(&src->y));
      }
    __syncthreads();
    // h partial: sum_jj conj(Bh[jj][r]) W[jj][r], all threads: (column r, part) then a fixed-order sum
    {
      // hparts x R <= NT double2 in U2 (free between the heavy phase and the updates; the plan reserves
      // >= 64 NT bytes there)
      const int hparts = max(1, min(NT / R, nJ));
      double2* hpart = (double2*)(smem + pl.o_u2);
      if (tid < hparts * R) {
        const int r = tid % R, part = tid / R;
        double2 h = make_double2(0.0, 0.0);
        for (int jj = part; jj < nJ; jj += hparts)
          h = zfma_cj(TIGHT ? to_d2(bhl[jj * R + r]) : bh64[jj * R + r], wacc[jj * R + r], h);
        hpart[part * R + r] = h;
      }
      __syncthreads();
      if (tid < R) {
        double2 h = make_double2(0.0, 0.0);
        for (int part = 0; part < hparts; ++part) h = zadd(h, hpart[part * R + tid]);
        __stcg(&g_hp[c * R + tid].x, h.x);
        __stcg(&g_hp[c * R + tid].y, h.y);
      }
    }
    for (int e = eb + tid; phase == 0 && e < ee; e += NT) {
      __stcg(&g_ga[e].x, G[e - eb].x);
      __stcg(&g_ga[e].y, G[e - eb].y);
    }
    {
      const double yt = block_sum(ysq, red);
      if (tid == 0 && phase == 0) __stcg(&g_yn[c], yt);
    }
    STAMP(9);
    cluster_barrier();  // ---------------------------------------------- B4
    STAMP(10);

    // ======== (d) redundant fp64 solve; cluster sums of Z for owned rows prefetched alongside.
    // The L2 loads of this phase are issued together: the thread's first packed Gram entry before the
    // Z sums, the h and ||Y||^2 partial sums on the top threads (which own no Z row / Gram entry).
    double2 gae0 = make_double2(0.0, 0.0), gbe0 = gae0;
    if (tid < Rp) {
      gae0 = phase == 2 ? make_double2(xg_at(2 * tid), xg_at(2 * tid + 1)) : __ldcg(&g_ga[tid]);
      gbe0 = fused ? make_double2(__ldcg(xgp + 2 * Rp + 2 + 2 * tid), __ldcg(xgp + 2 * Rp + 3 + 2 * tid))
                   : __ldcg(&g_gb[tid]);
    }
    for (int o = tid; o < nown * R; o += NT) {
      const int m = idiv(o, R), r = o - m * R;
      if (!TIGHT) zs[o] = sum_parts2n(g_zp + (size_t)own_k[m] * R + r, (size_t)Smax * R, CL * zks);
    }
    {
      const int hr = tid - (NT - R);
      if (hr >= 0) {
        const double2 h = sum_parts2(g_hp + hr, (size_t)R, CL);
        hv[hr] = h;
        hsave[hr] = h;
      }
      if (tid == NT - R - 1) {
        if (phase == 2) {
          scal[0] = xg_at(2 * Rp);      // ||Y||^2 over all ranks
          scal[1] = xg_at(2 * Rp + 1);  // ||Ah||^2 over all ranks
        } else {
          scal[0] = sum_parts(g_yn, 1, CL);
        }
      }
    }
    // the entries past the first: every load of the thread issued before the first use (R = 32: 3 entries)
    constexpr int GPF = 3;
    double2 gap[GPF], gbp[GPF];
#pragma unroll
    for (int u = 1; u < GPF; ++u) {
      const int e = tid + u * NT;
      gap[u] = gbp[u] = make_double2(0.0, 0.0);
      if (e < Rp) {
        gap[u] = phase == 2 ? make_double2(xg_at(2 * e), xg_at(2 * e + 1)) : __ldcg(&g_ga[e]);
        gbp[u] = fused ? make_double2(__ldcg(xgp + 2 * Rp + 2 + 2 * e), __ldcg(xgp + 2 * Rp + 3 + 2 * e))
                       : __ldcg(&g_gb[e]);
      }
    }
    gap[0] = gae0;
    gbp[0] = gbe0;
    for (int e = tid, u = 0; e < Rp; e += NT, ++u) {
      const int ij = tab[e];
      const int r = ij >> 8, q = ij & 255;
      double2 gae, gbe;
      if (u < GPF) {
        gae = gap[0];
        gbe = gbp[0];
#pragma unroll
        for (int w = 1; w < GPF; ++w)
          if (u == w) {
            gae = gap[w];
            gbe = gbp[w];
          }
      } else {
        gae = phase == 2 ? make_double2(xg_at(2 * e), xg_at(2 * e + 1)) : __ldcg(&g_ga[e]);
        gbe = fused ? make_double2(__ldcg(xgp + 2 * Rp + 2 + 2 * e), __ldcg(xgp + 2 * Rp + 3 + 2 * e))
                    : __ldcg(&g_gb[e]);
      }
      double2 gg = zmul(gae, gbe);
      if (r == q) {
        gg.x += a.lam;
        gda[r] = gae.x;
        gdb[r] = gbe.x;
      }
      G[e] = gg;
      if (!TIGHT) {
        gaf[r * R + q] = gae;
        gaf[q * R + r] = zconj(gae);
        gbf[r * R + q] = gbe;
        gbf[q * R + r] = zconj(gbe);
      }
    }
    __syncthreads();
    if (warp == 0) {  // ||Bh||^2 = trace(GB); ||Ah||^2 from the column norms (phase 2: from the payload)
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
        if (phase == 0) scal[1] = w;
      }
    }
    STAMP(11);

    double mu_used = 0.0, alpha = 0.0, cost;
    // the step is global: a rank whose rows hold no samples this frame still solves and scales them
    const bool update = Sglob > 0;
    if (update) {
      {
        // Gauss-Jordan (R parallel steps, no back substitution) up to R = 32; the 2x2-blocked
        // LDL^H has fewer flops per step and wins beyond (profiles/tools/ubench_gj.cu)
        // (few instantiations: every inlined variant costs instruction-cache lines in the frame loop)
        if (SOLV == 1) block_gj_solve<1>(G, hv, gam, colb, R);
        else if (SOLV == 2) block_gj_solve<2>(G, hv, gam, colb, R);
        else if (SOLV == 5) block_gj_solve<5>(G, hv, gam, colb, R);
        else block_ldl2_solve<9>(G, hv, gam, colb, blk, zf, R);
      }
      STAMP(12);
      if (warp == 0) {
        double gh = 0.0, gg = 0.0, top = 0.0;
        for (int r = lane; r < R; r += 32) {
          const double2 g = gam[r], h = hsave[r];
          gh += g.x * h.x + g.y * h.y;  // Re(conj(g) h)
          const double g2 = g.x * g.x + g.y * g.y;
          gg += g2;
          top = fmax(top, g2 * fmax(gda[r], gdb[r]));
          gamf[r] = to_f2(g);
        }
        gh = warp_sum(gh);
        gg = warp_sum(gg);
        top = warp_max(top);
        if (lane == 0) {
          scal[3] = gh;
          scal[4] = gg;
          scal[5] = top;
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
      __syncthreads();
      if (tid < R) {
        gam[tid] = make_double2(0.0, 0.0);
        gamf[tid] = make_float2(0.f, 0.f);
      }
      cost = 0.5 * lt * (scal[1] + scal[2]);
      __syncthreads();
    }
    if (a.resid_out != nullptr) write_residual(a, pl, f, s, S, j0, nJ, rows, g_ahs, gamf, bhl, ys, ahs);
    STAMP(13);

    // ======== (e) updates (k-space): Bh <- cfac Bh + mu conj(g) (W - Bh diag(g) GA^T)
    //                                 Ah_S <- cfac Ah_S + mu conj(g) (Z - Ah_S diag(g) GB^T)
    if (update) {
      const double cfac_d = 1.0 - mu_used * lt;
      if (TIGHT) {
        // one correction at a time, the gamma scaling moved onto the R x R factor:
        // corr[m][r] = sum_q X[m][q] conj(conj(g_q) G[q][r]) with (X, G) = (Bh, GA) then (Ah, GB)
        // (the P GEMM runs over every local row; its epilogue keeps the sampled ones)
        float2* mq = (float2*)(smem + pl.o_u1);  // the solver workspace is free now
        for (int gsel = 0; gsel < 2; ++gsel) {
          const bool q = gsel == 0;
          for (int e = tid; e < Rp; e += NT) {
            const int ij = tab[e];
            const int r = ij >> 8, qq = ij & 255;
            double2 gv;
            if (q && phase == 2) {
              gv.x = xg_at(2 * e);
              gv.y = xg_at(2 * e + 1);
            } else {
              const double2* src = q ? g_ga : g_gb;
              gv.x = __ldcg(&src[e].x);
              gv.y = __ldcg(&src[e].y);
            }
            const float2 g = to_f2(gv);
            mq[r * R + qq] = cmul(cconj(gamf[r]), g);
            mq[qq * R + r] = cmul(cconj(gamf[qq]), cconj(g));
          }
          __syncthreads();
          const int M = q ? nJ : (nown > 0 ? nI : 0);
          const RowsEpi epi{q ? EPI_Q_UPDATE : EPI_P_MAPPED, R, wacc, bhl, gam, cfac_d, mu_used, flags,
                            own_k, g_zp, Smax * R, CL * zks, zs32};
          cgemm_tile<GTM, GTN, false, true>(M, R, R, q ? bhl : ahl, R, 1, mq, R, 1, 1, red2, epi);
          __syncthreads();
        }
      } else {
        // the corrections on the fp64 tensor-core path, exact fp32 operands, the gamma scaling on the
        // fp64 R x R factor: corr[m][r] = sum_q X[m][q] conj(conj(g_q) G[q][r]) with (X, G) = (Bh, GA) for
        // Q and (the owned sampled Ah rows, GB) for P
        double2* gqa = gaf;  // scaled in place: GA, GB are not read again this frame
        double2* gqb = gbf;
        float2* aown = vop;
        for (int o = tid; o < R * R; o += NT) {
          const double2 cg = zconj(gam[idiv(o, R)]);
          gqa[o] = zmul(cg, gaf[o]);
          gqb[o] = zmul(cg, gbf[o]);
        }
        for (int o = tid; o < nown * R; o += NT) {
          const int m = idiv(o, R), q = o - m * R;
          aown[o] = ahl[own_li[m] * R + q];
        }
        __syncthreads();
        STAMP(21);
        {  // both products in one pass (disjoint outputs): one barrier
          const RowsEpi eq{EPI_Q_UPDATE, R, wacc, bhl, gam, cfac_d, mu_used, nullptr};
          const RowsEpi ep{EPI_P_UPDATE, R, zs, bhl, gam, cfac_d, mu_used, nullptr};
          zgemm_dmma<ZG>(nJ, R, R, bhl, R, 1, gqa, R, 1, eq);
          zgemm_dmma<ZG>(nown, R, R, aown, R, 1, gqb, R, 1, ep);
          __syncthreads();
        }
      }
      STAMP(22);
      STAMP(23);
      for (int o = tid; o < nI * R; o += NT) {
        const int li = idiv(o, R), r = o - li * R;
        double2 v = zscale(to_d2(ahl[o]), cfac_d);
        const int m = flags[li];
        if (m >= 0) v = zadd(v, TIGHT ? to_d2(zs32[m * R + r]) : zs[m * R + r]);
        ahl[o] = to_f2(v);
      }
      for (int o = tid; o < nJ * R; o += NT) {
        const float2 v = to_f2(wacc[o]);  // the state is fp32; the fp64 copy holds the same values
        bhl[o] = v;
        if (!TIGHT) bh64[o] = to_d2(v);
      }
      __syncthreads();
    }
    STAMP(14);

    // ======== outputs
    const size_t fs = (size_t)f * a.nslices + s;
    if (a.norm_out && !shard && c == 0 && tid == 0 && f > 0)  // the previous frame's post-update norms
      a.norm_out[fs - a.nslices] = (prev_upd && (scal[1] > ncap2 || scal[2] > ncap2)) ? 1 : 0;
    prev_upd = update;
    if (c == 0 && lead) {
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
    if (a.ah_hist) {
      float2* dst = (float2*)a.ah_hist + (multi ? (size_t)f * nx + i0 : fs * nxs + aoff) * R;
      for (int o = tid; o < nI * R; o += NT) dst[o] = ahl[o];
    }
    if (a.bh_hist && lead) {
      float2* dst = (float2*)a.bh_hist + (fs * ny + j0) * R;
      for (int o = tid; o < nJ * R; o += NT) dst[o] = bhl[o];
    }
    __syncthreads();
    STAMP(15);
  }
#undef STAMP

  // ---- write back resident state
  {
    float2* dst = (float2*)a.ah_out + arow * R;
    for (int o = tid; o < nI * R; o += NT) dst[o] = ahl[o];
    float2* dsb = (float2*)a.bh_out + ((size_t)s * ny + j0) * R;
    for (int o = tid; lead && o < nJ * R; o += NT) dsb[o] = bhl[o];
  }
  if (c == 0 && tid == 0 && lead) {
    if (a.alpha_bar) a.alpha_bar[s] = alpha_bar;
    if (a.policy == TT_POLICY_INFORMATIVE && a.philox_pos) a.philox_pos[s] = ppos;
  }
  if (status && tid == 0 && a.status) atomicOr(&a.status[s], status);
  if (a.norm_out && !shard && a.frames > 0) {  // the last frame's post-update norms
    const double2 nn = cluster_state_norms(ahl, nI * R, bhl, nJ * R, g_hp, c, CL, red);
    if (c == 0 && tid == 0)
      a.norm_out[(size_t)(a.frames - 1) * a.nslices + s] = (prev_upd && (nn.x > ncap2 || nn.y > ncap2)) ? 1 : 0;
  }
  // keep the cluster alive until every CTA is done with the shared scratch
  cluster_barrier();
}

// ---------------------------------------------------------------- host side
static int rows_choose_cluster(int nx, int ny, int R, int Smax, int want, RowsPlan* pl) {
  const int cands[5] = {16, 8, 4, 2, 1};
  if (want > 0) {
    if (want != 1 && want != 2 && want != 4 && want != 8 && want != 16)
      return tt_fail(TT_EINVAL, "cluster size must be 1, 2, 4, 8 or 16 (got %d)", want);
    if (!rows_make_plan(nx, ny, R, Smax, want, pl))
      return tt_fail(TT_EUNSUPPORTED, "row-mask step does not fit shared memory at cluster %d", want);
    return TT_OK;
  }
  // default: the smallest cluster that fits, grown to 16 for single-slice latency
  for (int i = 4; i >= 0; --i) {
    if (rows_make_plan(nx, ny, R, Smax, cands[i], pl)) return TT_OK;
  }
  return tt_fail(TT_EUNSUPPORTED, "row-mask step (nx=%d ny=%d R=%d rows=%d) does not fit", nx, ny, R, Smax);
}

// the instantiation: solver by Gauss-Jordan entries per thread, sharding phases only when sharded
typedef void (*RowsFn)(const tt_rows_args, const RowsPlan);
static const RowsFn rows_fns[10] = {tt_rows_kernel<1, false>, tt_rows_kernel<2, false>, tt_rows_kernel<5, false>,
                                    tt_rows_kernel<9, false>, tt_rows_kernel<1, true>,  tt_rows_kernel<2, true>,
                                    tt_rows_kernel<5, true>,  tt_rows_kernel<9, true>,
                                    tt_rows_kernel<5, false, true>, tt_rows_kernel<9, false, true>};
static int rows_which(int rank, bool sharded, bool tight) {
  const int ept = gj_ept(rank, ROWS_NT);
  const int solv = ept <= 1 ? 0 : ept <= 2 ? 1 : ept <= 5 ? 2 : 3;
  if (!tight) return solv + (sharded ? 4 : 0);
  // the tight plan is needed only at large N x R (R = 64 at 1024^2); compiled for the two wide solvers
  if (sharded || solv < 2) return -1;
  return 8 + (solv - 2);
}

// How many clusters of `cluster` CTAs of the row-mask kernel the device holds at once
// (cudaOccupancyMaxActiveClusters): on the B200's 8 GPCs of 16-20 SMs fewer than 148 / cluster for
// clusters of 8 and 16, so a launch with more slices than this runs in waves.
extern "C" int tt_rows_max_clusters(int nx, int ny, int rank, int max_rows, int cluster, int* nclusters) {
  if (!nclusters || nx < 1 || ny < 1 || rank < 1 || max_rows < 1 || cluster < 1)
    return tt_fail(TT_EINVAL, "tt_rows_max_clusters: bad args");
  RowsPlan pl;
  int rc = rows_choose_cluster(nx, ny, rank, max_rows, cluster, &pl);
  if (rc) return rc;
  const int which = rows_which(rank, false, pl.tight);
  if (which < 0) return tt_fail(TT_EUNSUPPORTED, "tt_rows_max_clusters: no kernel for this shape");
  const RowsFn fn = rows_fns[which];
  TT_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaFuncAttributes fa;
  TT_CUDA_TRY(cudaFuncGetAttributes(&fa, fn));
  if (fa.maxDynamicSharedSizeBytes < (int)pl.smem)  // only ever raised (the launch path caches the size it set)
    TT_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(148 * pl.CL), 1, 1);
  cfg.blockDim = dim3(ROWS_NT, 1, 1);
  cfg.dynamicSmemBytes = (size_t)pl.smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)pl.CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  TT_CUDA_TRY(cudaOccupancyMaxActiveClusters(&n, fn, &cfg));
  *nclusters = n;
  return TT_OK;
}

extern "C" int tt_rows_plan(int nx, int ny, int rank, int max_rows, int policy, int* cluster, size_t* smem_bytes) {
  (void)policy;
  if (nx < 1 || ny < 1 || rank < 1 || max_rows < 1 || !cluster)
    return tt_fail(TT_EINVAL, "tt_rows_plan: bad shape");
  RowsPlan pl;
  int rc = rows_choose_cluster(nx, ny, rank, max_rows, *cluster, &pl);
  if (rc) return rc;
  *cluster = pl.CL;
  if (smem_bytes) *smem_bytes = (size_t)pl.smem;
  return TT_OK;
}

extern "C" size_t tt_rows_shard_xg_len(int rank) { return (size_t)rank * (rank + 1) + 2; }

// Shared-memory plan of a row-mask launch at a given cluster size (diagnostics / tests): out[0..5] =
// cluster, rows per k tile (KT), smem bytes, tight (1/0), padded Y row stride, K-split buffer entries.
extern "C" int tt_rows_plan_info(int nx, int ny, int rank, int max_rows, int cluster, int* out) {
  if (!out || nx < 1 || ny < 1 || rank < 1 || max_rows < 1) return tt_fail(TT_EINVAL, "tt_rows_plan_info: bad args");
  RowsPlan pl;
  int rc = rows_choose_cluster(nx, ny, rank, max_rows, cluster, &pl);
  if (rc) return rc;
  out[0] = pl.CL;
  out[1] = pl.KT;
  out[2] = pl.smem;
  out[3] = pl.tight;
  out[4] = pl.ysr;
  out[5] = pl.red_cap;
  return TT_OK;
}

// Sum the payload slots of a local multi-rank launch into slot 0 (fixed order over ranks): the
// on-device counterpart of the all-reduce between the two phases.
__global__ void shard_reduce_kernel(int world, size_t nw, size_t ng, double* __restrict__ xw, double* __restrict__ xg) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nw + ng; i += (size_t)gridDim.x * blockDim.x) {
    if (i < nw) {
      double v = xw[i];
      for (int r = 1; r < world; ++r) v += xw[(size_t)r * nw + i];
      xw[i] = v;
    } else {
      const size_t k = i - nw;
      double v = xg[k];
      for (int r = 1; r < world; ++r) v += xg[(size_t)r * ng + k];
      xg[k] = v;
    }
  }
}

extern "C" int tt_rows_shard_reduce(void* stream, int world, int ny, int rank, double* xw, double* xg) {
  if (world < 1 || ny < 1 || rank < 1 || !xw || !xg) return tt_fail(TT_EINVAL, "tt_rows_shard_reduce: bad args");
  if (world == 1) return TT_OK;
  const size_t nw = 2 * (size_t)ny * rank, ng = (size_t)rank * (rank + 1) + 2;
  int blocks = (int)((nw + ng + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  shard_reduce_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(world, nw, ng, xw, xg);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

// ---------------------------------------------------------------- informative draws under row sharding
__global__ void shard_energy_kernel(int nx, int R, int r0, int nrows, const float2* __restrict__ a,
                                    double* __restrict__ e) {
  const int n = nx * R;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int row = i / R;
    double v = 0.0;
    if (row >= r0 && row < r0 + nrows) {
      const float2 x = a[(size_t)(row - r0) * R + (i - row * R)];
      v = (double)x.x * x.x + (double)x.y * x.y;
    }
    e[i] = v;
  }
}

extern "C" int tt_rows_shard_energy(void* stream, int nx, int rank, int r0, int nrows, const float* ah_rows,
                                    double* energy) {
  if (nx < 1 || rank < 1 || r0 < 0 || nrows < 0 || r0 + nrows > nx || !energy || (nrows > 0 && !ah_rows))
    return tt_fail(TT_EINVAL, "tt_rows_shard_energy: bad args");
  const int n = nx * rank;
  shard_energy_kernel<<<(n + 255) / 256 < 592 ? (n + 255) / 256 : 592, 256, 0, (cudaStream_t)stream>>>(
      nx, rank, r0, nrows, (const float2*)ah_rows, energy);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

// one CTA: column sums of the energy matrix in a fixed order (thread (r, part) sums rows part, part + P, ...,
// then the parts in order), then every row's raw score with the rows kernel's formula
__global__ void __launch_bounds__(256) shard_scores_kernel(int nx, int ny, int R, const double* __restrict__ e,
                                                           double* __restrict__ sraw, int32_t* status) {
  __shared__ double part[256];
  __shared__ double inrm[64];
  const int tid = threadIdx.x, P = blockDim.x / R;
  if (tid < P * R) {
    const int r = tid % R, p = tid / R;
    double acc = 0.0;
    for (int i = p; i < nx; i += P) acc += e[(size_t)i * R + r];
    part[p * R + r] = acc;
  }
  __syncthreads();
  if (tid < R) {
    double n2 = 0.0;
    for (int p = 0; p < P; ++p) n2 += part[p * R + tid];
    inrm[tid] = n2 > 0.0 ? fast_rcp(n2) : 0.0;
    if (n2 == 0.0 && status) atomicOr(status, TT_ST_ZEROCOL);
  }
  __syncthreads();
  const double cs = (double)ny, cr = (double)R, cd = 1.0 / ((double)R * (double)(nx + ny));
  for (int i = tid; i < nx; i += blockDim.x) {
    double acc = 0.0;
    for (int r = 0; r < R; ++r) acc = fma(e[(size_t)i * R + r], inrm[r], acc);
    sraw[i] = (cs * acc + cr) * cd;
  }
}

extern "C" int tt_rows_shard_scores(void* stream, int nx, int ny, int rank, const double* energy, double* sraw,
                                    int32_t* status) {
  if (nx < 1 || ny < 1 || rank < 1 || rank > 64 || !energy || !sraw)
    return tt_fail(TT_EINVAL, "tt_rows_shard_scores: bad args");
  shard_scores_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(nx, ny, rank, energy, sraw, status);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

extern "C" size_t tt_rows_scratch_bytes(int nslices, int nx, int ny, int rank, int max_rows, int cluster) {
  if (cluster < 1) cluster = 16;
  return rows_scratch_layout(nx, ny, rank, max_rows, cluster).per_slice * (size_t)(nslices > 0 ? nslices : 1);
}

extern "C" int tt_track_rows(void* stream, const tt_rows_args* a) {
  if (!a) return tt_fail(TT_EINVAL, "null args");
  if (a->nslices < 1 || a->nx < 1 || a->ny < 1 || a->rank < 1 || a->rank > 64 || a->frames < 0 || a->max_rows < 1)
    return tt_fail(TT_EINVAL, "tt_track_rows: bad shape (nslices=%d nx=%d ny=%d rank=%d frames=%d max_rows=%d)",
                   a->nslices, a->nx, a->ny, a->rank, a->frames, a->max_rows);
  if (a->max_rows > a->nx) return tt_fail(TT_EINVAL, "max_rows exceeds nx");
  if (!a->ah_in || !a->bh_in || !a->ah_out || !a->bh_out || !a->scratch || !a->ysrc)
    return tt_fail(TT_EINVAL, "tt_track_rows: null buffer");
  if (a->policy == TT_POLICY_STATIC && (!a->rows_tab || !a->rows_cnt))
    return tt_fail(TT_EINVAL, "static policy needs rows_tab/rows_cnt");
  if (a->policy == TT_POLICY_INFORMATIVE) {
    if (a->k_draws < 1 || a->k_draws > a->max_rows || a->nforced < 0 || a->nforced > a->k_draws)
      return tt_fail(TT_EINVAL, "informative policy: need 1 <= k <= max_rows and nforced <= k");
    if (!(a->beta >= 0.0 && a->beta < 1.0)) return tt_fail(TT_EINVAL, "uniform blend weight must be in [0, 1)");
    if (a->nforced > 0 && !a->forced) return tt_fail(TT_EINVAL, "null forced list");
  }
  if (a->lam < 0) return tt_fail(TT_EINVAL, "lambda must be nonnegative");
  if (a->shard_world > 0) {
    if (a->shard_rank < 0 || a->shard_rank >= a->shard_world || (a->shard_phase != 1 && a->shard_phase != 2))
      return tt_fail(TT_EINVAL, "row sharding: need 0 <= rank < world and phase 1 or 2");
    const bool fused = a->shard_local && a->shard_fused;
    const bool inf_ok = a->policy == TT_POLICY_INFORMATIVE && a->shard_phase == 1 && a->sraw_in && !a->shard_local;
    if ((a->policy != TT_POLICY_STATIC && !inf_ok) || a->nslices != 1 || (a->frames != 1 && !fused) ||
        a->y_mode != TT_Y_GATHER)
      return tt_fail(TT_EUNSUPPORTED, "row sharding supports static row tables (informative draws in phase 1 "
                                      "with sraw_in, one GPU per rank), one slice, one frame per launch (any "
                                      "number when fused), gathered measurements");
    if (a->shard_fused && (!a->shard_local || !a->grid_sync))
      return tt_fail(TT_EINVAL, "fused row sharding needs shard_local and a grid_sync counter");
    if (!a->xw || !a->xg) return tt_fail(TT_EINVAL, "row sharding: null payload buffers");
    if (a->resid_out) return tt_fail(TT_EUNSUPPORTED, "row sharding: residual output not supported");
    if (a->norm_out) return tt_fail(TT_EUNSUPPORTED, "row sharding: norm_cap flags not supported");
  }
  if (a->t0 < 1) return tt_fail(TT_EINVAL, "t must be >= 1");
  if (a->frames == 0) return TT_OK;
  {
    // the mirrored kernel (tt_rows2.cu) when the whole Ah fits every CTA at the requested cluster size
    const int cands[5] = {16, 8, 4, 2, 1};
    MirrorPlan mp;
    if (a->cluster > 0) {
      if (tt_rows_mirror_plan(a, a->cluster, &mp)) return tt_rows_mirror_launch(stream, a, mp);
    } else {
      for (int i = 0; i < 5; ++i)
        if (a->nslices * cands[i] <= 148 && tt_rows_mirror_plan(a, cands[i], &mp))
          return tt_rows_mirror_launch(stream, a, mp);
    }
  }
  RowsPlan pl;
  int rc = rows_choose_cluster(a->nx, a->ny, a->rank, a->max_rows, a->cluster, &pl);
  if (rc) return rc;
  if (a->cluster > 0 && a->cluster != pl.CL) return tt_fail(TT_EINVAL, "cluster mismatch");
  // the instantiation: solver by Gauss-Jordan entries per thread, sharding phases only when sharded
  static size_t configured_smem[10][TT_MAXDEV] = {{0}};
  const int which = rows_which(a->rank, a->shard_world > 0, pl.tight);
  if (which < 0)
    return tt_fail(TT_EUNSUPPORTED, "row-mask step (nx=%d R=%d rows=%d) needs the tight shared-memory plan, "
                                    "which is not built for this solver / sharding", a->nx, a->rank, a->max_rows);
  const RowsFn fn = rows_fns[which];
  {
    int dev = 0;
    TT_CUDA_TRY(cudaGetDevice(&dev));
    if (dev >= TT_MAXDEV || configured_smem[which][dev] < (size_t)pl.smem) {
      TT_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      TT_CUDA_TRY(tt_smem_attr((const void*)fn, (size_t)pl.smem, configured_smem[which]));
    }
  }
  cudaLaunchConfig_t cfg = {};
  const int nclusters = (a->shard_world > 0 && a->shard_local) ? a->shard_world : a->nslices;
  cfg.gridDim = dim3((unsigned)(nclusters * pl.CL), 1, 1);
  cfg.blockDim = dim3(ROWS_NT, 1, 1);
  cfg.dynamicSmemBytes = (size_t)pl.smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)pl.CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (a->shard_world > 0 && a->shard_local && a->shard_fused) {
    // the in-kernel inter-cluster barriers need every CTA resident: a cooperative launch, which fails
    // cleanly (TT_ECUDA) when the ranks' clusters do not fit the GPU at once
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.numAttrs = 2;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, fn, *a, pl);
    if (e == cudaErrorCooperativeLaunchTooLarge) {
      (void)cudaGetLastError();  // not sticky: clear it so the caller's fallback launches run
      return tt_fail(TT_ECUDA, "fused row sharding: %d ranks x %d CTAs do not fit the GPU at once "
                               "(cooperative launch too large)", a->shard_world, pl.CL);
    }
    TT_CUDA_TRY(e);
    return TT_OK;
  }
  TT_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, *a, pl));
  return TT_OK;
}
