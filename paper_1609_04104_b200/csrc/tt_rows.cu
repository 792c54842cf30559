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
#define ROWS_WPT 16

struct RowsPlan {
  int CL, KT, nIm, nJm, Rp;
  int o_ahl, o_bhl, o_u1, o_ga32, o_gb32, o_vec, o_flags, o_rows, o_u2, o_red;
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
  p->CL = CL;
  p->nIm = (nx + CL - 1) / CL;
  p->nJm = (ny + CL - 1) / CL;
  p->Rp = R * (R + 1) / 2;
  if (p->nJm * R > ROWS_WPT * ROWS_NT) return false;
  size_t o = 0;
  p->o_ahl = (int)o;   o = al16(o + sizeof(float2) * p->nIm * R);
  p->o_bhl = (int)o;   o = al16(o + sizeof(float2) * p->nJm * R);
  p->o_u1 = (int)o;    // packed fp64 Gram / LDL workspace  |  p + cdf (draw phase)
  {
    size_t g = sizeof(double2) * (size_t)p->Rp;
    size_t d = sizeof(double) * 2 * (size_t)nx;
    o = al16(o + (g > d ? g : d));
  }
  p->o_ga32 = (int)o;  o = al16(o + sizeof(float2) * R * R);
  p->o_gb32 = (int)o;  o = al16(o + sizeof(float2) * R * R);
  p->o_vec = (int)o;   o = al16(o + sizeof(double2) * R * 2 + sizeof(double) * R + sizeof(float2) * R + 64);
  p->o_flags = (int)o; o = al16(o + sizeof(int) * (nx > p->nIm ? nx : p->nIm));
  p->o_rows = (int)o;  o = al16(o + sizeof(int) * (Smax > 0 ? Smax : 1));
  p->o_u2 = (int)o;
  size_t fixed = o + sizeof(double) * 64;
  if (fixed > (size_t)maxsmem) return false;
  // U2: k-tiles (ys KT x nJm, ahs KT x R)  |  W buffer nJm x R  |  P rows nIm x R
  size_t other = sizeof(float2) * (size_t)R * (p->nJm > p->nIm ? p->nJm : p->nIm);
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

  float2* ahl = (float2*)(smem + pl.o_ahl);
  float2* bhl = (float2*)(smem + pl.o_bhl);
  double2* G = (double2*)(smem + pl.o_u1);
  double* pbuf = (double*)(smem + pl.o_u1);
  double* cdf = pbuf + nx;
  float2* ga32 = (float2*)(smem + pl.o_ga32);
  float2* gb32 = (float2*)(smem + pl.o_gb32);
  double2* gam = (double2*)(smem + pl.o_vec);
  double2* hv = gam + R;
  double* nrm = (double*)(hv + R);
  float2* gamf = (float2*)(nrm + R);
  double* scal = (double*)(gamf + R);  // 8 scalars
  int* flags = (int*)(smem + pl.o_flags);
  int* rows = (int*)(smem + pl.o_rows);
  float2* ys = (float2*)(smem + pl.o_u2);
  float2* ahs = ys + (size_t)pl.KT * pl.nJm;
  float2* wbuf = (float2*)(smem + pl.o_u2);
  float2* prow = (float2*)(smem + pl.o_u2);
  double* red = (double*)(smem + pl.o_red);
  int* ired = (int*)red;
  __shared__ int sh_S, sh_flag, sh_err;

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

  // ---- load resident state
  {
    const float2* src = (const float2*)a.ah_in + ((size_t)s * nx + i0) * R;
    for (int o = tid; o < nI * R; o += NT) ahl[o] = src[o];
    const float2* srb = (const float2*)a.bh_in + ((size_t)s * ny + j0) * R;
    for (int o = tid; o < nJ * R; o += NT) bhl[o] = srb[o];
  }
  double alpha_bar = a.alpha_bar ? a.alpha_bar[s] : 0.0;
  uint64_t ppos = (a.policy == TT_POLICY_INFORMATIVE && a.philox_pos) ? a.philox_pos[s] : 0ull;
  int status = 0;
  const int eb = part_begin(Rp, CL, c), ee = part_begin(Rp, CL, c + 1);
  __syncthreads();

  for (int f = 0; f < a.frames; ++f) {
    const long long t = a.t0 + f;
    const double lt = a.lam / (double)t;
    // ======== (a) column norms of Ah (own rows) and packed GB partials
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
      int r, q;
      tri_decode(e, r, q);
      double2 acc = make_double2(0.0, 0.0);
      for (int jj = 0; jj < nJ; ++jj) acc = zfma_cj(bhl[jj * R + r], bhl[jj * R + q], acc);
      __stcg(&g_gbp[(size_t)c * Rp + e].x, acc.x);
      __stcg(&g_gbp[(size_t)c * Rp + e].y, acc.y);
    }
    cluster_barrier();  // ---------------------------------------------- B1
    for (int e = eb + tid; e < ee; e += NT) {
      double2 acc = make_double2(0.0, 0.0);
      for (int cc = 0; cc < CL; ++cc) {
        acc.x += __ldcg(&g_gbp[(size_t)cc * Rp + e].x);
        acc.y += __ldcg(&g_gbp[(size_t)cc * Rp + e].y);
      }
      __stcg(&g_gb[e].x, acc.x);
      __stcg(&g_gb[e].y, acc.y);
    }
    if (tid < R) {
      double acc = 0.0;
      for (int cc = 0; cc < CL; ++cc) acc += __ldcg(&g_cn[cc * R + tid]);
      nrm[tid] = acc;
    }
    if (tid == 0) sh_err = 0;
    __syncthreads();
    double anorm2 = 0.0;
    for (int r = 0; r < R; ++r) anorm2 += nrm[r];

    int S = 0;
    if (a.policy == TT_POLICY_INFORMATIVE) {
      // raw row scores for own rows (sampler.py:77-85, :126)
      for (int i = tid; i < nI; i += NT) {
        double e = 0.0;
        for (int r = 0; r < R; ++r) {
          const float2 v = ahl[i * R + r];
          const double n2 = nrm[r];
          if (n2 > 0.0) e += ((double)v.x * v.x + (double)v.y * v.y) / n2;
        }
        const double sc = ((double)ny * e + (double)R) / ((double)R * (double)(nx + ny));
        __stcg(&g_sraw[i0 + i], sc);
      }
      if (tid < R && nrm[tid] == 0.0) sh_err = TT_ST_ZEROCOL;
      cluster_barrier();  // -------------------------------------------- B2
      double loc = 0.0;
      for (int i = tid; i < nx; i += NT) {
        const double v = __ldcg(&g_sraw[i]);
        pbuf[i] = v;
      }
      __syncthreads();
      // deterministic sums over contiguous chunks
      const int chunk = (nx + NT - 1) / NT;
      const int q0 = min(nx, tid * chunk), q1 = min(nx, q0 + chunk);
      loc = 0.0;
      for (int i = q0; i < q1; ++i) loc += pbuf[i];
      const double S1 = block_sum(loc, red);
      loc = 0.0;
      for (int i = q0; i < q1; ++i) {
        const double v = (1.0 - a.beta) * (pbuf[i] / S1) + a.beta / (double)nx;  // sampler.py:88-92
        pbuf[i] = v;
        loc += v;
      }
      const double S2 = block_sum(loc, red);
      for (int i = q0; i < q1; ++i) pbuf[i] = pbuf[i] / S2;
      __syncthreads();
      const int ndraw = a.k_draws - a.nforced;
      int Sd;
      draw_with_replacement_block(pbuf, cdf, flags, rows, Sd, nx, ndraw > 0 ? ndraw : 0, a.forced, a.nforced,
                                  a.key0, a.key1 + (uint64_t)s, ppos, red, &sh_flag);
      ppos += (uint64_t)(ndraw > 0 ? ndraw : 0);
      S = Sd;
    } else {
      const int* tab = a.rows_tab + ((size_t)f * a.nslices + s) * Smax;
      const int cnt = a.rows_cnt[(size_t)f * a.nslices + s];
      for (int i = tid; i < nx; i += NT) flags[i] = 0;
      __syncthreads();
      if (cnt < 0 || cnt > Smax) {
        if (tid == 0) sh_err |= TT_ST_OVERFLOW;
        S = 0;
      } else {
        for (int k = tid; k < cnt; k += NT) {
          const int i = tab[k];
          rows[k] = i;
          if (i < 0 || i >= nx) atomicOr(&sh_err, TT_ST_BADROW);
          else if (atomicAdd(&flags[i], 1) > 0) atomicOr(&sh_err, TT_ST_DUPROW);
        }
        S = cnt;
      }
      __syncthreads();
      if (sh_err & (TT_ST_BADROW | TT_ST_DUPROW | TT_ST_OVERFLOW)) S = 0;
    }
    if (tid == 0) sh_S = S;
    __syncthreads();
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
    cluster_arrive();  // ------------------------------------------------ B3 (split)
    auto yptr = [&](int k) -> const float2* {
      if (a.y_mode == TT_Y_GATHER)
        return (const float2*)a.ysrc + (size_t)f * a.y_frame_stride + (size_t)s * a.y_slice_stride +
               (size_t)rows[k] * ny + j0;
      return (const float2*)a.ysrc + (((size_t)f * a.nslices + s) * Smax + k) * ny + j0;
    };
    const int KT = pl.KT;
    {
      const int kt = min(KT, S);
      for (int o = tid; o < kt * nJ; o += NT) {
        const int kk = o / nJ, jj = o - kk * nJ;
        cp_async8(&ys[kk * pl.nJm + jj], yptr(kk) + jj);
      }
    }
    cluster_wait();

    // ======== (c) heavy phase over k tiles: W, Z partials, GA (own entries), ||Y||^2
    float2 acc[ROWS_WPT];
#pragma unroll
    for (int m = 0; m < ROWS_WPT; ++m) acc[m] = make_float2(0.f, 0.f);
    for (int e = eb + tid; e < ee; e += NT) G[e - eb] = make_double2(0.0, 0.0);
    double ysq = 0.0;
    for (int k0 = 0; k0 < S; k0 += KT) {
      const int kt = min(KT, S - k0);
      if (k0 > 0) {
        for (int o = tid; o < kt * nJ; o += NT) {
          const int kk = o / nJ, jj = o - kk * nJ;
          cp_async8(&ys[kk * pl.nJm + jj], yptr(k0 + kk) + jj);
        }
      }
      for (int o = tid; o < kt * R; o += NT) {
        float2 v;
        v.x = __ldcg(&g_ahs[(size_t)(k0) * R + o].x);
        v.y = __ldcg(&g_ahs[(size_t)(k0) * R + o].y);
        ahs[o] = v;
      }
      cp_async_wait_all();
      __syncthreads();
      for (int o = tid; o < kt * nJ; o += NT) {
        const int kk = o / nJ, jj = o - kk * nJ;
        const float2 v = ys[kk * pl.nJm + jj];
        ysq += (double)v.x * v.x + (double)v.y * v.y;
      }
      // W[jj][r] += sum_k Y[k][jj] conj(Ah_S[k][r])
#pragma unroll
      for (int m = 0; m < ROWS_WPT; ++m) {
        const int o = tid + m * NT;
        if (o < nJ * R) {
          const int jj = o / R, r = o - jj * R;
          float2 w = acc[m];
          for (int kk = 0; kk < kt; ++kk) w = cfma_conj(ys[kk * pl.nJm + jj], ahs[kk * R + r], w);
          acc[m] = w;
        }
      }
      // Z partial over own columns
      for (int o = tid; o < kt * R; o += NT) {
        const int kk = o / R, r = o - kk * R;
        float2 z = make_float2(0.f, 0.f);
        for (int jj = 0; jj < nJ; ++jj) z = cfma_conj(ys[kk * pl.nJm + jj], bhl[jj * R + r], z);
        float2* dst = &g_zp[((size_t)c * Smax + k0 + kk) * R + r];
        __stcg(&dst->x, z.x);
        __stcg(&dst->y, z.y);
      }
      // GA own packed entries
      for (int e = eb + tid; e < ee; e += NT) {
        int r, q;
        tri_decode(e, r, q);
        double2 g = G[e - eb];
        for (int kk = 0; kk < kt; ++kk) g = zfma_cj(ahs[kk * R + r], ahs[kk * R + q], g);
        G[e - eb] = g;
      }
      __syncthreads();
    }
    // h partial: sum_jj conj(Bh[jj][r]) W[jj][r]
#pragma unroll
    for (int m = 0; m < ROWS_WPT; ++m) {
      const int o = tid + m * NT;
      if (o < nJ * R) wbuf[o] = acc[m];
    }
    __syncthreads();
    if (tid < R) {
      double2 h = make_double2(0.0, 0.0);
      for (int jj = 0; jj < nJ; ++jj) h = zfma_cj(bhl[jj * R + tid], wbuf[jj * R + tid], h);
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
    cluster_barrier();  // ---------------------------------------------- B4

    // ======== (d) redundant fp64 solve
    for (int e = tid; e < Rp; e += NT) {
      int r, q;
      tri_decode(e, r, q);
      double2 gae, gbe;
      gae.x = __ldcg(&g_ga[e].x);
      gae.y = __ldcg(&g_ga[e].y);
      gbe.x = __ldcg(&g_gb[e].x);
      gbe.y = __ldcg(&g_gb[e].y);
      double2 gg = zmul(gae, gbe);
      if (r == q) gg.x += a.lam;
      G[e] = gg;
      ga32[r * R + q] = to_f2(gae);
      ga32[q * R + r] = to_f2(zconj(gae));
      gb32[r * R + q] = to_f2(gbe);
      gb32[q * R + r] = to_f2(zconj(gbe));
    }
    if (tid < R) {
      double2 h = make_double2(0.0, 0.0);
      for (int cc = 0; cc < CL; ++cc) {
        h.x += __ldcg(&g_hp[cc * R + tid].x);
        h.y += __ldcg(&g_hp[cc * R + tid].y);
      }
      hv[tid] = h;
    }
    if (tid == 0) {
      double yn = 0.0;
      for (int cc = 0; cc < CL; ++cc) yn += __ldcg(&g_yn[cc]);
      scal[0] = yn;
    }
    __syncthreads();
    double bnorm2 = 0.0;  // ||Bh||^2 = trace(GB)
    for (int r = 0; r < R; ++r) bnorm2 += __ldcg(&g_gb[tri_idx(r, r)].x);
    const double energy = anorm2 + bnorm2;

    double mu_used = 0.0, alpha = 0.0, cost;
    bool update = S > 0;
    if (update) {
      block_ldl_solve(G, hv, gam, R);
      // h was overwritten by the elimination: reload it for the cost
      if (tid < R) {
        double2 h = make_double2(0.0, 0.0);
        for (int cc = 0; cc < CL; ++cc) {
          h.x += __ldcg(&g_hp[cc * R + tid].x);
          h.y += __ldcg(&g_hp[cc * R + tid].y);
        }
        hv[tid] = h;
        gamf[tid] = to_f2(gam[tid]);
      }
      __syncthreads();
      double gh = 0.0, gg = 0.0, top = 0.0;
      for (int r = 0; r < R; ++r) {
        const double2 g = gam[r], h = hv[r];
        gh += g.x * h.x + g.y * h.y;  // Re(conj(g) h)
        const double g2 = g.x * g.x + g.y * g.y;
        gg += g2;
        const double da = __ldcg(&g_ga[tri_idx(r, r)].x), db = __ldcg(&g_gb[tri_idx(r, r)].x);
        top = fmax(top, g2 * fmax(da, db));
      }
      const double e2 = scal[0] - gh - a.lam * gg;
      cost = 0.5 * e2 + 0.5 * lt * energy;
      if (a.step_mode == TT_STEP_HESSIAN) {
        alpha = fmin(fmax(lt + top, a.c_floor), a.c_cap);  // tracker.py:364
        alpha_bar += alpha;
        mu_used = 1.0 / alpha_bar;
      } else {
        mu_used = a.mu;
      }
      if (!isfinite(cost) || !isfinite(gh)) status |= TT_ST_NONFINITE;
    } else {
      if (tid < R) {
        gam[tid] = make_double2(0.0, 0.0);
        gamf[tid] = make_float2(0.f, 0.f);
      }
      cost = 0.5 * lt * energy;
      __syncthreads();
    }

    // optional residual e = Y - Ah_S diag(gamma) Bh^T on own columns (pre-update)
    if (a.resid_out != nullptr) {
      for (int k0 = 0; k0 < S; k0 += KT) {
        const int kt = min(KT, S - k0);
        for (int o = tid; o < kt * nJ; o += NT) {
          const int kk = o / nJ, jj = o - kk * nJ;
          ys[kk * pl.nJm + jj] = yptr(k0 + kk)[jj];
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
          e = csub(e, sacc);
          float2* dst = (float2*)a.resid_out + (((size_t)f * a.nslices + s) * Smax + k0 + kk) * ny + j0 + jj;
          *dst = e;
        }
        __syncthreads();
      }
    }

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
      for (int o = tid; o < nI * R; o += NT) {
        const int li = o / R, r = o - li * R;
        const int k = flags[li];
        if (k >= 0) {
          float2 z = make_float2(0.f, 0.f);
          for (int cc = 0; cc < CL; ++cc) {
            const float2* src = &g_zp[((size_t)cc * Smax + k) * R + r];
            z.x += __ldcg(&src->x);
            z.y += __ldcg(&src->y);
          }
          float2 corr = make_float2(0.f, 0.f);
          for (int q = 0; q < R; ++q) corr = cfma(cmul(ahl[li * R + q], gamf[q]), gb32[r * R + q], corr);
          prow[o] = csub(z, corr);
        }
      }
      // new Bh values (need old Bh everywhere) into registers
      float2 nb[ROWS_WPT];
#pragma unroll
      for (int m = 0; m < ROWS_WPT; ++m) {
        const int o = tid + m * NT;
        nb[m] = make_float2(0.f, 0.f);
        if (o < nJ * R) {
          const int jj = o / R, r = o - jj * R;
          float2 corr = make_float2(0.f, 0.f);
          for (int q = 0; q < R; ++q) corr = cfma(cmul(bhl[jj * R + q], gamf[q]), ga32[r * R + q], corr);
          const float2 qv = csub(acc[m], corr);
          nb[m] = cadd(cscale(bhl[o], cfac), cscale(cmul(cconj(gamf[r]), qv), muf));
        }
      }
      __syncthreads();
      for (int o = tid; o < nI * R; o += NT) {
        const int li = o / R, r = o - li * R;
        float2 v = cscale(ahl[o], cfac);
        if (flags[li] >= 0) v = cadd(v, cscale(cmul(cconj(gamf[r]), prow[o]), muf));
        ahl[o] = v;
      }
#pragma unroll
      for (int m = 0; m < ROWS_WPT; ++m) {
        const int o = tid + m * NT;
        if (o < nJ * R) bhl[o] = nb[m];
      }
      __syncthreads();
    }

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
  }

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
