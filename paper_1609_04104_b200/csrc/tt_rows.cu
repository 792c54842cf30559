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

#include "tt_block.cuh"

namespace cg = cooperative_groups;

#define ROWS_NT 256

struct RowsPlan {
  int CL, KT, nIm, nJm, Rp;
  int o_ahl, o_bhl, o_u1, o_ga32, o_gb32, o_vec, o_tab, o_flags, o_rows, o_forced, o_wacc, o_u2, o_red;
  int smem;
};

struct RowsScratch {
  size_t cn, gbp, gb, ga, sraw, ahs, zp, hp, yn, per_slice;
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
  s.zp = o;   o = al16(o + sizeof(float2) * (size_t)CL * Smax * R);
  s.hp = o;   o = al16(o + sizeof(double2) * CL * R);
  s.yn = o;   o = al16(o + sizeof(double) * CL);
  s.per_slice = al16(o + 256);
  (void)ny;
  return s;
}

static bool rows_make_plan(int nx, int ny, int R, int Smax, int CL, RowsPlan* p) {
  const int maxsmem = 227 * 1024;
  if (R > 64) return false;
  p->CL = CL;
  p->nIm = (nx + CL - 1) / CL;
  p->nJm = (ny + CL - 1) / CL;
  p->Rp = R * (R + 1) / 2;
  size_t o = 0;
  p->o_ahl = (int)o;    o = al16(o + sizeof(float2) * p->nIm * R);
  p->o_bhl = (int)o;    o = al16(o + sizeof(float2) * p->nJm * R);
  p->o_u1 = (int)o;     // packed fp64 Gram / LDL workspace  |  p + cdf (draw phase)
  {
    size_t g = sizeof(double2) * (size_t)p->Rp;
    size_t d = sizeof(double) * 2 * (size_t)nx;
    o = al16(o + (g > d ? g : d));
  }
  p->o_ga32 = (int)o;   o = al16(o + sizeof(float2) * p->Rp);  // packed lower, fp32
  p->o_gb32 = (int)o;   o = al16(o + sizeof(float2) * p->Rp);
  // vec: gam, hv, hsave (double2 R); nrm, inrm, inv, gda, gdb (double R); gamf (float2 R); 16 scalars
  // + LDL scratch: colb 4 (R+1) double2, blk 4 (R/2+1) double, zf R double2
  p->o_vec = (int)o;    o = al16(o + sizeof(double2) * R * 3 + sizeof(double) * R * 5 + sizeof(float2) * R + 128 +
                                 sizeof(double2) * 4 * (R + 1) + sizeof(double) * 4 * (R / 2 + 1) + sizeof(double2) * R);
  p->o_tab = (int)o;    o = al16(o + sizeof(unsigned short) * p->Rp);
  p->o_flags = (int)o;  o = al16(o + sizeof(int) * (nx > p->nIm ? nx : p->nIm));
  p->o_rows = (int)o;   o = al16(o + sizeof(int) * Smax);
  p->o_forced = (int)o; o = al16(o + sizeof(int) * Smax);
  p->o_wacc = (int)o;   o = al16(o + sizeof(float2) * p->nJm * R);
  p->o_u2 = (int)o;
  size_t fixed = o + sizeof(double) * 64;
  if (fixed > (size_t)maxsmem) return false;
  // U2: k-tiles (ys KT x nJm, ahs KT x R)  |  P rows nIm x R
  size_t other = sizeof(float2) * (size_t)R * p->nIm;
  size_t avail = maxsmem - fixed;
  int KT = (int)(avail / (sizeof(float2) * (size_t)(p->nJm + R)));
  if (KT > Smax) KT = Smax;
  if (KT > 128) KT = 128;
  if (KT < 1) return false;
  p->KT = KT;
  size_t tiles = sizeof(float2) * (size_t)KT * (p->nJm + R);
  size_t u2 = tiles > other ? tiles : other;
  if (fixed + u2 > (size_t)maxsmem) return false;
  o = al16(o + u2);
  p->o_red = (int)o;
  o += sizeof(double) * 64;
  p->smem = (int)o;
  return true;
}

// Hermitian R x R from a packed lower triangle: M[r][q]
TT_DEV float2 herm_at(const float2* P, int r, int q) {
  return r >= q ? P[r * (r + 1) / 2 + q] : cconj(P[q * (q + 1) / 2 + r]);
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
      ys[kk * pl.nJm + jj] = src[jj];
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
      float2 e = ys[kk * pl.nJm + jj];
      float2 sacc = make_float2(0.f, 0.f);
      for (int r = 0; r < R; ++r) sacc = cfma(ahs[kk * R + r], bhl[jj * R + r], sacc);
      float2* dst = (float2*)a.resid_out + (((size_t)f * a.nslices + s) * Smax + k0 + kk) * ny + j0 + jj;
      *dst = csub(e, sacc);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(ROWS_NT, 1) tt_rows_kernel(const __grid_constant__ tt_rows_args a,
                                                             const __grid_constant__ RowsPlan pl) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, NT = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;
  const int CL = pl.CL;
  const int c = (int)(blockIdx.x % CL);
  const int s = (int)(blockIdx.x / CL);
  const int nx = a.nx, ny = a.ny, R = a.rank, Smax = a.max_rows, Rp = pl.Rp;
  const int i0 = part_begin(nx, CL, c), nI = part_begin(nx, CL, c + 1) - i0;
  const int j0 = part_begin(ny, CL, c), nJ = part_begin(ny, CL, c + 1) - j0;
  const int KT = pl.KT;

  float2* ahl = (float2*)(smem + pl.o_ahl);
  float2* bhl = (float2*)(smem + pl.o_bhl);
  double2* G = (double2*)(smem + pl.o_u1);
  double* pbuf = (double*)(smem + pl.o_u1);
  double* cdf = pbuf + nx;
  float2* ga32 = (float2*)(smem + pl.o_ga32);
  float2* gb32 = (float2*)(smem + pl.o_gb32);
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
  float2* wacc = (float2*)(smem + pl.o_wacc);
  float2* ys = (float2*)(smem + pl.o_u2);
  float2* ahs = ys + (size_t)KT * pl.nJm;
  float2* prow = (float2*)(smem + pl.o_u2);
  double* red = (double*)(smem + pl.o_red);
  __shared__ int sh_S, sh_flag, sh_err;
  long long* pclk = (a.phase_clock != nullptr && blockIdx.x == 0) ? (long long*)a.phase_clock : nullptr;
#define STAMP(k)                                                             \
  do {                                                                       \
    if (pclk != nullptr && tid == 0) pclk[(size_t)f * 32 + (k)] = clock64(); \
  } while (0)

  // global scratch for this slice
  const RowsScratch L = rows_scratch_layout(nx, ny, R, Smax, CL);
  unsigned char* sb = (unsigned char*)a.scratch + (size_t)s * L.per_slice;
  double* g_cn = (double*)(sb + L.cn);
  double2* g_gbp = (double2*)(sb + L.gbp);
  double2* g_gb = (double2*)(sb + L.gb);
  double2* g_ga = (double2*)(sb + L.ga);
  double* g_sraw = (double*)(sb + L.sraw);
  float2* g_ahs = (float2*)(sb + L.ahs);
  float2* g_zp = (float2*)(sb + L.zp);
  double2* g_hp = (double2*)(sb + L.hp);
  double* g_yn = (double*)(sb + L.yn);

  // ---- load resident state and constants once
  {
    const float2* src = (const float2*)a.ah_in + ((size_t)s * nx + i0) * R;
    for (int o = tid; o < nI * R; o += NT) ahl[o] = src[o];
    const float2* srb = (const float2*)a.bh_in + ((size_t)s * ny + j0) * R;
    for (int o = tid; o < nJ * R; o += NT) bhl[o] = srb[o];
    if (a.policy == TT_POLICY_INFORMATIVE)
      for (int m = tid; m < a.nforced; m += NT) forced[m] = a.forced[m];
  }
  ldl_table_init(tab, R);
  double alpha_bar = a.alpha_bar ? a.alpha_bar[s] : 0.0;
  uint64_t ppos = (a.policy == TT_POLICY_INFORMATIVE && a.philox_pos) ? a.philox_pos[s] : 0ull;
  int status = 0;
  const int eb = part_begin(Rp, CL, c), ee = part_begin(Rp, CL, c + 1);
  __syncthreads();

  for (int f = 0; f < a.frames; ++f) {
    const long long t = a.t0 + f;
    const double lt = a.lam / (double)t;
    STAMP(0);
    // ======== (a) column-norm partials of Ah (own rows) and packed GB partials
    for (int r = warp; r < R; r += nwarps) {
      double acc = 0.0;
      for (int i = lane; i < nI; i += 32) {
        const float2 v = ahl[i * R + r];
        acc += (double)v.x * v.x + (double)v.y * v.y;
      }
      acc = warp_sum(acc);
      if (lane == 0) __stcg(&g_cn[c * R + r], acc);
    }
    for (int e = tid; e < Rp; e += NT) {
      const int ij = tab[e];
      const int r = ij >> 8, q = ij & 255;
      double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
      int jj = 0;
      for (; jj + 1 < nJ; jj += 2) {
        acc = zfma_cj(bhl[jj * R + r], bhl[jj * R + q], acc);
        acc2 = zfma_cj(bhl[(jj + 1) * R + r], bhl[(jj + 1) * R + q], acc2);
      }
      if (jj < nJ) acc = zfma_cj(bhl[jj * R + r], bhl[jj * R + q], acc);
      acc = zadd(acc, acc2);
      __stcg(&g_gbp[(size_t)c * Rp + e].x, acc.x);
      __stcg(&g_gbp[(size_t)c * Rp + e].y, acc.y);
    }
    STAMP(1);
    cluster_barrier();  // ---------------------------------------------- B1
    STAMP(2);
    for (int e = eb + tid - 32; tid >= 32 && e < ee; e += NT - 32) {
      const double2 g = sum_parts2(g_gbp + e, (size_t)Rp, CL);
      __stcg(&g_gb[e].x, g.x);
      __stcg(&g_gb[e].y, g.y);
    }
    for (int r = tid; r < R && tid < 32; r += 32) {
      const double n2 = sum_parts(g_cn + r, (size_t)R, CL);
      nrm[r] = n2;
      inrm[r] = n2 > 0.0 ? fast_rcp(n2) : 0.0;
    }
    if (tid == 0) sh_err = 0;
    __syncthreads();
    if (warp == 0) {  // ||Ah||^2, fixed order
      double v = 0.0;
      for (int r = lane; r < R; r += 32) v += nrm[r];
      v = warp_sum(v);
      if (lane == 0) scal[1] = v;
    }

    int S = 0;
    if (a.policy == TT_POLICY_INFORMATIVE) {
      // raw row scores for own rows (sampler.py:77-85, :126)
      const double cs = (double)ny, cr = (double)R, cd = 1.0 / ((double)R * (double)(nx + ny));
      for (int i = tid; i < nI; i += NT) {
        double e = 0.0;
        for (int r = 0; r < R; ++r) {
          const float2 v = ahl[i * R + r];
          e = fma((double)v.x * v.x + (double)v.y * v.y, inrm[r], e);
        }
        __stcg(&g_sraw[i0 + i], (cs * e + cr) * cd);
      }
      if (tid < R && nrm[tid] == 0.0) atomicOr(&sh_err, TT_ST_ZEROCOL);
      STAMP(3);
      cluster_barrier();  // -------------------------------------------- B2
      STAMP(4);
      // probabilities: normalise, blend with the uniform law (sampler.py:88-92);
      // the final renormalisation is folded into cdf /= cdf[-1] of the draw.
      const int chunk = (nx + NT - 1) / NT;
      const int q0 = min(nx, tid * chunk), q1 = min(nx, q0 + chunk);
      double loc = 0.0;
      for (int i = q0; i < q1; ++i) {
        const double v = __ldcg(&g_sraw[i]);
        pbuf[i] = v;
        loc += v;
      }
      const double S1 = block_sum(loc, red);
      const double w1 = (1.0 - a.beta) / S1, w0 = a.beta / (double)nx;
      for (int i = q0; i < q1; ++i) pbuf[i] = fma(pbuf[i], w1, w0);
      __syncthreads();
      STAMP(20);
      const int ndraw = a.k_draws - a.nforced;
      int Sd;
      draw_with_replacement_block<false>(pbuf, cdf, flags, rows, Sd, nx, ndraw > 0 ? ndraw : 0, forced, a.nforced,
                                  a.key0, a.key1 + (uint64_t)s, ppos, red, &sh_flag);
      ppos += (uint64_t)(ndraw > 0 ? ndraw : 0);
      S = Sd;
    } else {
      S = load_static_rows(a, f, s, rows, flags, &sh_err);
    }
    if (tid == 0) sh_S = S;
    __syncthreads();
    STAMP(5);
    S = sh_S;
    status |= sh_err;

    // ======== (b) publish own sampled rows of Ah; prefetch the first Y tile
    for (int o = tid; o < S * R; o += NT) {
      const int k = o / R, r = o - k * R;
      const int i = rows[k];
      if (i >= i0 && i < i0 + nI) {
        const float2 v = ahl[(i - i0) * R + r];
        __stcg(&g_ahs[(size_t)k * R + r].x, v.x);
        __stcg(&g_ahs[(size_t)k * R + r].y, v.y);
      }
    }
    STAMP(6);
    cluster_arrive();  // ------------------------------------------------ B3 (split)
    const float2* ybase = a.y_mode == TT_Y_GATHER
                              ? (const float2*)a.ysrc + (size_t)f * a.y_frame_stride + (size_t)s * a.y_slice_stride + j0
                              : (const float2*)a.ysrc + ((size_t)f * a.nslices + s) * Smax * ny + j0;
    const bool gather = a.y_mode == TT_Y_GATHER;
    {
      const int kt = min(KT, S);
      for (int o = tid; o < kt * nJ; o += NT) {
        const int kk = o / nJ, jj = o - kk * nJ;
        cp_async8(&ys[kk * pl.nJm + jj], ybase + (size_t)(gather ? rows[kk] : kk) * ny + jj);
      }
    }
    for (int o = tid; o < nJ * R; o += NT) wacc[o] = make_float2(0.f, 0.f);
    for (int e = eb + tid; e < ee; e += NT) G[e - eb] = make_double2(0.0, 0.0);
    cluster_wait();
    STAMP(7);

    // ======== (c) heavy phase over k tiles: W, Z partials, GA (own entries), ||Y||^2
    double ysq = 0.0;
    for (int k0 = 0; k0 < S; k0 += KT) {
      const int kt = min(KT, S - k0);
      if (k0 > 0) {
        for (int o = tid; o < kt * nJ; o += NT) {
          const int kk = o / nJ, jj = o - kk * nJ;
          cp_async8(&ys[kk * pl.nJm + jj], ybase + (size_t)(gather ? rows[k0 + kk] : k0 + kk) * ny + jj);
        }
      }
      for (int o = tid; o < kt * R; o += NT) {
        float2 v;
        v.x = __ldcg(&g_ahs[(size_t)k0 * R + o].x);
        v.y = __ldcg(&g_ahs[(size_t)k0 * R + o].y);
        ahs[o] = v;
      }
      cp_async_wait_all();
      __syncthreads();
      if (k0 == 0) STAMP(16);
      for (int o = tid; o < kt * nJ; o += NT) {
        const int kk = o / nJ, jj = o - kk * nJ;
        const float2 v = ys[kk * pl.nJm + jj];
        ysq += (double)v.x * v.x + (double)v.y * v.y;
      }
      // W[jj][r] += sum_k Y[k][jj] conj(Ah_S[k][r])   (thread-owned smem accumulators)
      for (int o = tid; o < nJ * R; o += 2 * NT) {
        const int o2 = o + NT;
        const bool two = o2 < nJ * R;
        const int jj = o / R, r = o - jj * R;
        const int jj2 = two ? o2 / R : jj, r2 = two ? o2 - jj2 * R : r;
        float2 w = wacc[o], w2 = two ? wacc[o2] : make_float2(0.f, 0.f);
#pragma unroll 4
        for (int kk = 0; kk < kt; ++kk) {
          w = cfma_conj(ys[kk * pl.nJm + jj], ahs[kk * R + r], w);
          w2 = cfma_conj(ys[kk * pl.nJm + jj2], ahs[kk * R + r2], w2);
        }
        wacc[o] = w;
        if (two) wacc[o2] = w2;
      }
      if (k0 == 0) STAMP(17);
      // Z partial over own columns
      for (int ob = tid; ob < kt * R; ob += 4 * NT) {
        int kq[4], rq[4];
        float2 z[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int o = min(ob + u * NT, kt * R - 1);
          kq[u] = o / R;
          rq[u] = o - kq[u] * R;
          z[u] = make_float2(0.f, 0.f);
        }
#pragma unroll 2
        for (int jj = 0; jj < nJ; ++jj) {
#pragma unroll
          for (int u = 0; u < 4; ++u) z[u] = cfma_conj(ys[kq[u] * pl.nJm + jj], bhl[jj * R + rq[u]], z[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (ob + u * NT < kt * R) {
            float2* dst = &g_zp[((size_t)c * Smax + k0 + kq[u]) * R + rq[u]];
            __stcg(&dst->x, z[u].x);
            __stcg(&dst->y, z[u].y);
          }
        }
      }
      if (k0 == 0) STAMP(18);
      // GA own packed entries
      const int nq = 4 * (ee - eb);
      for (int base = tid & ~31; base < nq; base += NT) {  // warp-uniform trip count
        const int eq = base + lane;
        const int e = eb + (eq >> 2), part = eq & 3;
        double2 g = make_double2(0.0, 0.0);
        if (eq < nq) {
          const int ij = tab[e];
          const int r = ij >> 8, q = ij & 255;
          for (int kk = part; kk < kt; kk += 4) g = zfma_cj(ahs[kk * R + r], ahs[kk * R + q], g);
        }
        // lanes 4m..4m+3 hold the parts of one entry: (p0 + p1) + (p2 + p3)
        g.x += __shfl_xor_sync(0xffffffffu, g.x, 1);
        g.y += __shfl_xor_sync(0xffffffffu, g.y, 1);
        g.x += __shfl_xor_sync(0xffffffffu, g.x, 2);
        g.y += __shfl_xor_sync(0xffffffffu, g.y, 2);
        if (part == 0 && eq < nq) G[e - eb] = zadd(G[e - eb], g);
      }
      if (k0 == 0) STAMP(19);
      __syncthreads();
    }
    STAMP(8);
    // h partial: sum_jj conj(Bh[jj][r]) W[jj][r]
    if (tid < R) {
      double2 h = make_double2(0.0, 0.0);
      for (int jj = 0; jj < nJ; ++jj) h = zfma_cj(bhl[jj * R + tid], wacc[jj * R + tid], h);
      __stcg(&g_hp[c * R + tid].x, h.x);
      __stcg(&g_hp[c * R + tid].y, h.y);
    }
    for (int e = eb + tid; e < ee; e += NT) {
      __stcg(&g_ga[e].x, G[e - eb].x);
      __stcg(&g_ga[e].y, G[e - eb].y);
    }
    {
      const double yt = block_sum(ysq, red);
      if (tid == 0) __stcg(&g_yn[c], yt);
    }
    STAMP(9);
    cluster_barrier();  // ---------------------------------------------- B4
    STAMP(10);

    // ======== (d) redundant fp64 solve (every cross-CTA read is one parallel round trip)
    for (int e = tid; e < Rp; e += NT) {
      const int ij = tab[e];
      const int r = ij >> 8, q = ij & 255;
      double2 gae, gbe;
      gae.x = __ldcg(&g_ga[e].x);
      gae.y = __ldcg(&g_ga[e].y);
      gbe.x = __ldcg(&g_gb[e].x);
      gbe.y = __ldcg(&g_gb[e].y);
      double2 gg = zmul(gae, gbe);
      if (r == q) {
        gg.x += a.lam;
        gda[r] = gae.x;
        gdb[r] = gbe.x;
      }
      G[e] = gg;
      ga32[e] = to_f2(gae);
      gb32[e] = to_f2(gbe);
    }
    if (tid < R) {
      const double2 h = sum_parts2(g_hp + tid, (size_t)R, CL);
      hv[tid] = h;
      hsave[tid] = h;
    }
    if (tid == 32) scal[0] = sum_parts(g_yn, 1, CL);
    __syncthreads();
    if (warp == 0) {  // ||Bh||^2 = trace(GB)
      double v = 0.0;
      for (int r = lane; r < R; r += 32) v += gdb[r];
      v = warp_sum(v);
      if (lane == 0) scal[2] = v;
    }
    STAMP(11);

    double mu_used = 0.0, alpha = 0.0, cost;
    const bool update = S > 0;
    if (update) {
      {
        const int E = Rp + R;  // augmented entries; registers per thread
        if (E <= 2 * ROWS_NT) block_ldl2_solve<2>(G, hv, gam, colb, blk, zf, R);
        else if (E <= 4 * ROWS_NT) block_ldl2_solve<4>(G, hv, gam, colb, blk, zf, R);
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

    // ======== (e) updates (k-space): Ah <- cfac Ah + mu conj(g) P_S ; Bh <- cfac Bh + mu conj(g) Q
    if (update) {
      const float cfac = (float)(1.0 - mu_used * lt);
      const float muf = (float)mu_used;
      for (int li = tid; li < nI; li += NT) flags[li] = -1;
      __syncthreads();
      for (int k = tid; k < S; k += NT) {
        const int i = rows[k];
        if (i >= i0 && i < i0 + nI) flags[i - i0] = k;
      }
      __syncthreads();
      // P_S rows owned here: Z (summed over the cluster) - Ah_S diag(gamma) GB^T
      for (int o = tid; o < nI * R; o += NT) {
        const int li = o / R, r = o - li * R;
        const int k = flags[li];
        if (k >= 0) {
          const float2 z = sum_parts_f2(g_zp + (size_t)k * R + r, (size_t)Smax * R, CL);
          float2 corr = make_float2(0.f, 0.f);
          for (int q = 0; q < R; ++q) corr = cfma(cmul(ahl[li * R + q], gamf[q]), herm_at(gb32, r, q), corr);
          prow[o] = csub(z, corr);
        }
      }
      // Q = W - Bh diag(gamma) GA^T ; new Bh into wacc (W is consumed in place)
      for (int o = tid; o < nJ * R; o += NT) {
        const int jj = o / R, r = o - jj * R;
        float2 corr = make_float2(0.f, 0.f);
        for (int q = 0; q < R; ++q) corr = cfma(cmul(bhl[jj * R + q], gamf[q]), herm_at(ga32, r, q), corr);
        const float2 qv = csub(wacc[o], corr);
        wacc[o] = cadd(cscale(bhl[o], cfac), cscale(cmul(cconj(gamf[r]), qv), muf));
      }
      __syncthreads();
      for (int o = tid; o < nI * R; o += NT) {
        const int li = o / R, r = o - li * R;
        float2 v = cscale(ahl[o], cfac);
        if (flags[li] >= 0) v = cadd(v, cscale(cmul(cconj(gamf[r]), prow[o]), muf));
        ahl[o] = v;
      }
      for (int o = tid; o < nJ * R; o += NT) bhl[o] = wacc[o];
      __syncthreads();
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
    if (a.ah_hist) {
      float2* dst = (float2*)a.ah_hist + (fs * nx + i0) * R;
      for (int o = tid; o < nI * R; o += NT) dst[o] = ahl[o];
    }
    if (a.bh_hist) {
      float2* dst = (float2*)a.bh_hist + (fs * ny + j0) * R;
      for (int o = tid; o < nJ * R; o += NT) dst[o] = bhl[o];
    }
    __syncthreads();
    STAMP(15);
  }
#undef STAMP

  // ---- write back resident state
  {
    float2* dst = (float2*)a.ah_out + ((size_t)s * nx + i0) * R;
    for (int o = tid; o < nI * R; o += NT) dst[o] = ahl[o];
    float2* dsb = (float2*)a.bh_out + ((size_t)s * ny + j0) * R;
    for (int o = tid; o < nJ * R; o += NT) dsb[o] = bhl[o];
  }
  if (c == 0 && tid == 0) {
    if (a.alpha_bar) a.alpha_bar[s] = alpha_bar;
    if (a.policy == TT_POLICY_INFORMATIVE && a.philox_pos) a.philox_pos[s] = ppos;
  }
  if (status && tid == 0 && a.status) atomicOr(&a.status[s], status);
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
  if (a->t0 < 1) return tt_fail(TT_EINVAL, "t must be >= 1");
  if (a->frames == 0) return TT_OK;
  RowsPlan pl;
  int rc = rows_choose_cluster(a->nx, a->ny, a->rank, a->max_rows, a->cluster, &pl);
  if (rc) return rc;
  if (a->cluster > 0 && a->cluster != pl.CL) return tt_fail(TT_EINVAL, "cluster mismatch");
  static int configured_smem = -1;
  if (configured_smem < pl.smem) {
    TT_CUDA_TRY(cudaFuncSetAttribute(tt_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem));
    TT_CUDA_TRY(cudaFuncSetAttribute(tt_rows_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured_smem = pl.smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a->nslices * pl.CL), 1, 1);
  cfg.blockDim = dim3(ROWS_NT, 1, 1);
  cfg.dynamicSmemBytes = (size_t)pl.smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)pl.CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TT_CUDA_TRY(cudaLaunchKernelEx(&cfg, tt_rows_kernel, *a, pl));
  return TT_OK;
}
