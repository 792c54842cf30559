// Generic online step for an arbitrary (i, j) index list (FourierMask /
// EntryMask, observation.py:58-90) on measurement-domain factors
// (Ah, Bh) = (F_x A, F_y B) for Fourier masks, (A, B) for entry masks — the
// two are the same iteration (test_mri.py:258-286).
//
//   1. ent_gram     Phi_l = Ah[i_l] .* Bh[j_l] (exact fp64 products), block
//                   partials of G = Phi^H Phi, h = Phi^H y, ||y||^2
//                   (build_phi observation.py:219-228; solve_gamma
//                   tracker.py:139-156 as normal equations)
//   2. ent_solve    fixed-order reduction, G + lam I, fp64 LDL^H -> gamma,
//                   cost (tracker.py:386-389)
//   3. ent_resid    e_l = y_l - Phi_l gamma, scattered into a dense residual
//                   image Xi and mask M (the scatter of _scatter_theta,
//                   tracker.py:176-188)
//   4. ent_backproj P = Xi conj(Bh), Q = Xi^T conj(Ah) and the closed-form
//                   curvature sums c0 = M |Bh|^2, c1 = M^T |Ah|^2
//                   (collapsed gradient data terms tracker.py:208-228;
//                   hessian_bound tracker.py:337-364)
//   5. ent_step     alpha / mu (tracker.py:391-400)
//   6. ent_update   Ah <- (1 - mu lam/t) Ah + mu conj(gamma) P, same for Bh
//                   (tracker.py:402-404)
// Everything is deterministic (fixed reduction orders, no float atomics).

#include "tt_block.cuh"

#define ENT_NT 256
#define ENT_NB 64
#define ENT_TL 32

struct EntScratch {
  size_t gp, hp, yp, gam, scal, xi, mk, P, Q, c0, c1, total;
};
static EntScratch ent_layout(int nx, int ny, int R) {
  EntScratch s;
  const size_t Rp = (size_t)R * (R + 1) / 2;
  size_t o = 0;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  s.gp = o;   o = al(o + sizeof(double2) * ENT_NB * Rp);
  s.hp = o;   o = al(o + sizeof(double2) * ENT_NB * R);
  s.yp = o;   o = al(o + sizeof(double) * ENT_NB);
  s.gam = o;  o = al(o + sizeof(double2) * R);
  s.scal = o; o = al(o + sizeof(double) * 16);
  s.xi = o;   o = al(o + sizeof(float2) * (size_t)nx * ny);
  s.mk = o;   o = al(o + sizeof(float) * (size_t)nx * ny);
  s.P = o;    o = al(o + sizeof(float2) * (size_t)nx * R);
  s.Q = o;    o = al(o + sizeof(float2) * (size_t)ny * R);
  s.c0 = o;   o = al(o + sizeof(float) * (size_t)nx * R);
  s.c1 = o;   o = al(o + sizeof(float) * (size_t)ny * R);
  s.total = o;
  return s;
}

__global__ void __launch_bounds__(ENT_NT) ent_gram_kernel(int nmeas, const int* __restrict__ nmeas_dev, int R,
                                                          const float2* __restrict__ ah,
                                                          const float2* __restrict__ bh, const int* __restrict__ idx,
                                                          const float2* __restrict__ y, double2* __restrict__ gp,
                                                          double2* __restrict__ hp, double* __restrict__ yp) {
  if (nmeas_dev) nmeas = min(*nmeas_dev, nmeas);
  extern __shared__ __align__(16) unsigned char smem[];
  double2* phi = (double2*)smem;                   // [TL][R]
  double2* yv = phi + ENT_TL * R;                  // [TL]
  double* red = (double*)(yv + ENT_TL);
  const int tid = threadIdx.x, NT = blockDim.x;
  const int Rp = R * (R + 1) / 2;
  const int b = blockIdx.x;
  const int l0 = (int)(((long long)nmeas * b) / gridDim.x), l1 = (int)(((long long)nmeas * (b + 1)) / gridDim.x);
  // per-thread accumulators for entries e = tid + m*NT (Rp <= 2080 -> m < 9)
  double2 acc[9];
#pragma unroll
  for (int m = 0; m < 9; ++m) acc[m] = make_double2(0.0, 0.0);
  double2 hacc = make_double2(0.0, 0.0);
  double ysq = 0.0;
  for (int t0 = l0; t0 < l1; t0 += ENT_TL) {
    const int tl = min(ENT_TL, l1 - t0);
    for (int o = tid; o < tl * R; o += NT) {
      const int ll = o / R, r = o - ll * R;
      const int i = idx[2 * (t0 + ll)], j = idx[2 * (t0 + ll) + 1];
      phi[o] = zmul(to_d2(ah[(size_t)i * R + r]), to_d2(bh[(size_t)j * R + r]));
    }
    for (int ll = tid; ll < tl; ll += NT) {
      const float2 v = y[t0 + ll];
      yv[ll] = to_d2(v);
      ysq += (double)v.x * v.x + (double)v.y * v.y;
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 9; ++m) {
      const int e = tid + m * NT;
      if (e < Rp) {
        int r, q;
        tri_decode(e, r, q);
        double2 g = acc[m];
        for (int ll = 0; ll < tl; ++ll) g = zfma_cj(phi[ll * R + r], phi[ll * R + q], g);
        acc[m] = g;
      }
    }
    if (tid < R)
      for (int ll = 0; ll < tl; ++ll) hacc = zfma_cj(phi[ll * R + tid], yv[ll], hacc);
    __syncthreads();
  }
#pragma unroll
  for (int m = 0; m < 9; ++m) {
    const int e = tid + m * NT;
    if (e < Rp) gp[(size_t)b * Rp + e] = acc[m];
  }
  if (tid < R) hp[(size_t)b * R + tid] = hacc;
  const double ys = block_sum(ysq, red);
  if (tid == 0) yp[b] = ys;
}

__global__ void __launch_bounds__(ENT_NT) ent_solve_kernel(int nx, int ny, int R, int nmeas,
                                                           const int* __restrict__ nmeas_dev, int nb, double lam,
                                                           long long t, const float2* __restrict__ ah,
                                                           const float2* __restrict__ bh, const double2* gp,
                                                           const double2* hp, const double* yp, double2* gam_out,
                                                           double* scal, float2* gamma_out, double* cost_out,
                                                           int32_t* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (nmeas_dev) nmeas = min(*nmeas_dev, nmeas);
  const int Rp = R * (R + 1) / 2;
  double2* G = (double2*)smem;
  double2* hv = G + Rp;
  double2* gam = hv + R;
  double* red = (double*)(gam + R);
  const int tid = threadIdx.x, NT = blockDim.x;
  double en = 0.0;
  for (int o = tid; o < nx * R; o += NT) {
    const float2 v = ah[o];
    en += (double)v.x * v.x + (double)v.y * v.y;
  }
  for (int o = tid; o < ny * R; o += NT) {
    const float2 v = bh[o];
    en += (double)v.x * v.x + (double)v.y * v.y;
  }
  const double energy = block_sum(en, red);
  const double lt = lam / (double)t;
  if (nmeas == 0) {
    if (tid < R) {
      gam_out[tid] = make_double2(0.0, 0.0);
      if (gamma_out) gamma_out[tid] = make_float2(0.f, 0.f);
    }
    if (tid == 0) {
      const double cost = 0.5 * lt * energy;
      scal[0] = cost;
      if (cost_out) cost_out[0] = cost;
    }
    return;
  }
  for (int e = tid; e < Rp; e += NT) {
    int r, q;
    tri_decode(e, r, q);
    double2 g = make_double2(0.0, 0.0);
    int b = 0;
    for (; b + 4 <= nb; b += 4) {  // four loads in flight, fixed association order
      const double2 v0 = gp[(size_t)b * Rp + e], v1 = gp[(size_t)(b + 1) * Rp + e];
      const double2 v2 = gp[(size_t)(b + 2) * Rp + e], v3 = gp[(size_t)(b + 3) * Rp + e];
      g = zadd(g, zadd(zadd(v0, v1), zadd(v2, v3)));
    }
    for (; b < nb; ++b) g = zadd(g, gp[(size_t)b * Rp + e]);
    if (r == q) g.x += lam;
    G[e] = g;
  }
  double yn = 0.0;
  if (tid < R) {
    double2 h = make_double2(0.0, 0.0);
    for (int b = 0; b < nb; ++b) h = zadd(h, hp[(size_t)b * R + tid]);
    hv[tid] = h;
  }
  for (int b = 0; b < nb; ++b) yn += yp[b];
  __syncthreads();
  {
    double2* colb = (double2*)(red + 64);  // 4 (R+1) double2 after the reduction buffer
    const int ept = gj_ept(R, blockDim.x);
    if (ept <= 1) block_gj_solve<1>(G, hv, gam, colb, R);
    else if (ept <= 2) block_gj_solve<2>(G, hv, gam, colb, R);
    else if (ept <= 3) block_gj_solve<3>(G, hv, gam, colb, R);
    else if (ept <= 5) block_gj_solve<5>(G, hv, gam, colb, R);
    else block_ldl_solve(G, hv, gam, R);
  }
  // reload h (eliminated in place) for the cost
  if (tid < R) {
    double2 h = make_double2(0.0, 0.0);
    for (int b = 0; b < nb; ++b) h = zadd(h, hp[(size_t)b * R + tid]);
    hv[tid] = h;
    gam_out[tid] = gam[tid];
    if (gamma_out) gamma_out[tid] = to_f2(gam[tid]);
  }
  __syncthreads();
  if (tid == 0) {
    double gh = 0.0, gg = 0.0;
    for (int r = 0; r < R; ++r) {
      gh += gam[r].x * hv[r].x + gam[r].y * hv[r].y;
      gg += gam[r].x * gam[r].x + gam[r].y * gam[r].y;
    }
    const double cost = 0.5 * (yn - gh - lam * gg) + 0.5 * lt * energy;
    scal[0] = cost;
    if (cost_out) cost_out[0] = cost;
    if (!isfinite(cost) && status) atomicOr(status, TT_ST_NONFINITE);
  }
}

__global__ void ent_resid_kernel(int nmeas, const int* __restrict__ nmeas_dev, int ny, int R,
                                 const float2* __restrict__ ah, const float2* __restrict__ bh,
                                 const int* __restrict__ idx, const float2* __restrict__ y, const double2* gam,
                                 float2* __restrict__ xi, float* __restrict__ mk, float2* __restrict__ resid) {
  if (nmeas_dev) nmeas = min(*nmeas_dev, nmeas);
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nmeas; l += gridDim.x * blockDim.x) {
    const int i = idx[2 * l], j = idx[2 * l + 1];
    double2 s = make_double2(0.0, 0.0);
    for (int r = 0; r < R; ++r) {
      const double2 ph = zmul(to_d2(ah[(size_t)i * R + r]), to_d2(bh[(size_t)j * R + r]));
      s = zfma(ph, gam[r], s);
    }
    const float2 e = make_float2((float)((double)y[l].x - s.x), (float)((double)y[l].y - s.y));
    xi[(size_t)i * ny + j] = e;
    mk[(size_t)i * ny + j] = 1.f;
    if (resid) resid[l] = e;
  }
}

// role 0 (blockIdx.y = 0): rows i of P and c0; role 1: rows j of Q and c1. Block = 32 outputs x 8 parts
// of the contraction index; the 8 parts are summed in fixed order through shared memory.
#define BP_O 32
#define BP_K 8
__global__ void __launch_bounds__(BP_O * BP_K) ent_backproj_kernel(int nx, int ny, int R,
                                                                   const float2* __restrict__ ah,
                                                                   const float2* __restrict__ bh,
                                                                   const float2* __restrict__ xi,
                                                                   const float* __restrict__ mk,
                                                                   float2* __restrict__ P, float2* __restrict__ Q,
                                                                   float* __restrict__ c0, float* __restrict__ c1) {
  __shared__ float2 sacc[BP_K][BP_O];
  __shared__ float scs[BP_K][BP_O];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int o = blockIdx.x * BP_O + tx;
  const bool rows = blockIdx.y == 0;
  const int m = rows ? nx * R : ny * R;
  float2 acc = make_float2(0.f, 0.f);
  float cs = 0.f;
  if (o < m) {
    if (rows) {
      const int i = o / R, r = o - i * R;
      for (int j = ty; j < ny; j += BP_K) {
        const float2 b = bh[(size_t)j * R + r];
        acc = cfma_conj(xi[(size_t)i * ny + j], b, acc);
        cs = fmaf(mk[(size_t)i * ny + j], cabs2(b), cs);
      }
    } else {
      const int j = o / R, r = o - j * R;
      for (int i = ty; i < nx; i += BP_K) {
        const float2 a = ah[(size_t)i * R + r];
        acc = cfma_conj(xi[(size_t)i * ny + j], a, acc);
        cs = fmaf(mk[(size_t)i * ny + j], cabs2(a), cs);
      }
    }
  }
  sacc[ty][tx] = acc;
  scs[ty][tx] = cs;
  __syncthreads();
  if (ty == 0 && o < m) {
    for (int k = 1; k < BP_K; ++k) {
      acc = cadd(acc, sacc[k][tx]);
      cs += scs[k][tx];
    }
    if (rows) {
      P[o] = acc;
      c0[o] = cs;
    } else {
      Q[o] = acc;
      c1[o] = cs;
    }
  }
}

__global__ void __launch_bounds__(ENT_NT) ent_step_kernel(int nx, int ny, int R, int nmeas,
                                                          const int* __restrict__ nmeas_dev, double lam, long long t,
                                                          int step_mode, double mu, double c_floor, double c_cap,
                                                          const double2* gam, const float* c0, const float* c1,
                                                          double* alpha_bar, double* scal, double* mu_out,
                                                          double* alpha_out) {
  __shared__ double red[64];
  if (nmeas_dev) nmeas = min(*nmeas_dev, nmeas);
  const int tid = threadIdx.x, NT = blockDim.x;
  double top = 0.0;
  for (int o = tid; o < nx * R; o += NT) {
    const int r = o % R;
    const double g2 = gam[r].x * gam[r].x + gam[r].y * gam[r].y;
    top = fmax(top, g2 * (double)c0[o]);
  }
  for (int o = tid; o < ny * R; o += NT) {
    const int r = o % R;
    const double g2 = gam[r].x * gam[r].x + gam[r].y * gam[r].y;
    top = fmax(top, g2 * (double)c1[o]);
  }
  top = warp_max(top);
  if ((tid & 31) == 0) red[tid >> 5] = top;
  __syncthreads();
  if (tid == 0) {
    double tt = 0.0;
    for (int w = 0; w < (NT >> 5); ++w) tt = fmax(tt, red[w]);
    double m = 0.0, alpha = 0.0;
    if (nmeas > 0) {
      if (step_mode == TT_STEP_HESSIAN) {
        alpha = fmin(fmax(lam / (double)t + tt, c_floor), c_cap);
        const double ab = alpha_bar[0] + alpha;
        alpha_bar[0] = ab;
        m = 1.0 / ab;
      } else {
        m = mu;
      }
    }
    scal[1] = m;
    if (mu_out) mu_out[0] = m;
    if (alpha_out) alpha_out[0] = alpha;
  }
}

__global__ void ent_update_kernel(int nx, int ny, int R, double lam, long long t, const double* scal,
                                  const double2* gam, const float2* __restrict__ ah, const float2* __restrict__ bh,
                                  const float2* __restrict__ P, const float2* __restrict__ Q, float2* ah_out,
                                  float2* bh_out) {
  const double m = scal[1];
  const float cfac = (float)(1.0 - m * lam / (double)t);
  const float muf = (float)m;
  const int na = nx * R, nbb = ny * R;
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < na + nbb; o += gridDim.x * blockDim.x) {
    if (o < na) {
      const int r = o % R;
      const float2 g = cconj(to_f2(gam[r]));
      ah_out[o] = cadd(cscale(ah[o], cfac), cscale(cmul(g, P[o]), muf));
    } else {
      const int k = o - na, r = k % R;
      const float2 g = cconj(to_f2(gam[r]));
      bh_out[k] = cadd(cscale(bh[k], cfac), cscale(cmul(g, Q[k]), muf));
    }
  }
}

extern "C" size_t tt_entries_scratch_bytes(int nx, int ny, int rank, int nmeas) {
  (void)nmeas;
  return ent_layout(nx, ny, rank).total;
}

extern "C" int tt_track_entries(void* stream, const tt_entries_args* a) {
  if (!a) return tt_fail(TT_EINVAL, "null args");
  const int nx = a->nx, ny = a->ny, R = a->rank, L = a->nmeas;
  const int* Ld = a->nmeas_dev;  // device count (capacity L), graph-capturable chain
  if (nx < 1 || ny < 1 || R < 1 || L < 0) return tt_fail(TT_EINVAL, "tt_track_entries: bad shape");
  if (R > 64) return tt_fail(TT_EUNSUPPORTED, "rank > 64 is not supported");
  if (a->t < 1) return tt_fail(TT_EINVAL, "t must be >= 1");
  if (a->lam < 0) return tt_fail(TT_EINVAL, "lambda must be nonnegative");
  if (!a->ah_in || !a->bh_in || !a->ah_out || !a->bh_out || !a->scratch || !a->alpha_bar)
    return tt_fail(TT_EINVAL, "tt_track_entries: null buffer");
  if (L > 0 && (!a->idx || !a->y)) return tt_fail(TT_EINVAL, "tt_track_entries: null idx/y");
  cudaStream_t st = (cudaStream_t)stream;
  const EntScratch S = ent_layout(nx, ny, R);
  unsigned char* sb = (unsigned char*)a->scratch;
  double2* gp = (double2*)(sb + S.gp);
  double2* hp = (double2*)(sb + S.hp);
  double* yp = (double*)(sb + S.yp);
  double2* gam = (double2*)(sb + S.gam);
  double* scal = (double*)(sb + S.scal);
  float2* xi = (float2*)(sb + S.xi);
  float* mk = (float*)(sb + S.mk);
  float2* P = (float2*)(sb + S.P);
  float2* Q = (float2*)(sb + S.Q);
  float* c0 = (float*)(sb + S.c0);
  float* c1 = (float*)(sb + S.c1);
  const int Rp = R * (R + 1) / 2;
  const float2* ah = (const float2*)a->ah_in;
  const float2* bh = (const float2*)a->bh_in;
  int nb = 0;
  if (L > 0) {
    nb = (L + 255) / 256;
    if (nb > ENT_NB) nb = ENT_NB;
    const size_t sm = sizeof(double2) * (ENT_TL * (size_t)R + ENT_TL) + sizeof(double) * 64;
    static int set_gram = -1;
    if (set_gram < (int)sm) {
      TT_CUDA_TRY(cudaFuncSetAttribute(ent_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      set_gram = (int)sm;
    }
    ent_gram_kernel<<<nb, ENT_NT, sm, st>>>(L, Ld, R, ah, bh, a->idx, (const float2*)a->y, gp, hp, yp);
  }
  {
    const size_t sm = sizeof(double2) * (Rp + 2 * (size_t)R) + sizeof(double) * 64 + sizeof(double2) * 4 * (R + 1);
    static int set_solve = -1;
    if (set_solve < (int)sm) {
      TT_CUDA_TRY(cudaFuncSetAttribute(ent_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      set_solve = (int)sm;
    }
    ent_solve_kernel<<<1, ENT_NT, sm, st>>>(nx, ny, R, L, Ld, nb, a->lam, (long long)a->t, ah, bh, gp, hp, yp, gam, scal,
                                            (float2*)a->gamma_out, a->cost_out, a->status);
  }
  if (L == 0) {
    // empty batch: no update (tracker.py:380-384)
    ent_step_kernel<<<1, ENT_NT, 0, st>>>(0, 0, R, 0, nullptr, a->lam, (long long)a->t, a->step_mode, a->mu, a->c_floor,
                                          a->c_cap, gam, c0, c1, a->alpha_bar, scal, a->mu_out, a->alpha_out);
    if (a->ah_out != a->ah_in)
      TT_CUDA_TRY(cudaMemcpyAsync(a->ah_out, a->ah_in, sizeof(float2) * (size_t)nx * R, cudaMemcpyDeviceToDevice, st));
    if (a->bh_out != a->bh_in)
      TT_CUDA_TRY(cudaMemcpyAsync(a->bh_out, a->bh_in, sizeof(float2) * (size_t)ny * R, cudaMemcpyDeviceToDevice, st));
    TT_CUDA_TRY(cudaGetLastError());
    return TT_OK;
  }
  TT_CUDA_TRY(cudaMemsetAsync(xi, 0, sizeof(float2) * (size_t)nx * ny, st));
  TT_CUDA_TRY(cudaMemsetAsync(mk, 0, sizeof(float) * (size_t)nx * ny, st));
  {
    int blocks = (L + 255) / 256;
    if (blocks > 1184) blocks = 1184;
    ent_resid_kernel<<<blocks, 256, 0, st>>>(L, Ld, ny, R, ah, bh, a->idx, (const float2*)a->y, gam, xi, mk,
                                             (float2*)a->resid_out);
  }
  {
    const int m = (nx > ny ? nx : ny) * R;
    dim3 grid((m + BP_O - 1) / BP_O, 2);
    ent_backproj_kernel<<<grid, dim3(BP_O, BP_K), 0, st>>>(nx, ny, R, ah, bh, xi, mk, P, Q, c0, c1);
  }
  ent_step_kernel<<<1, ENT_NT, 0, st>>>(nx, ny, R, L, Ld, a->lam, (long long)a->t, a->step_mode, a->mu, a->c_floor,
                                        a->c_cap, gam, c0, c1, a->alpha_bar, scal, a->mu_out, a->alpha_out);
  {
    const int n = (nx + ny) * R;
    int blocks = (n + 255) / 256;
    if (blocks > 1184) blocks = 1184;
    ent_update_kernel<<<blocks, 256, 0, st>>>(nx, ny, R, a->lam, (long long)a->t, scal, gam, ah, bh, P, Q,
                                              (float2*)a->ah_out, (float2*)a->bh_out);
  }
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

// Acquisition at drawn entries (sampler.py:204-206 truth lookup): flat index -> (i, j), y = frame[i][j].
__global__ void ent_gather_kernel(int ny, const float2* __restrict__ frame, const int* __restrict__ omega,
                                  const int* __restrict__ count, int cap, int* __restrict__ idx, float2* __restrict__ y) {
  const int n = min(*count, cap);
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < n; m += gridDim.x * blockDim.x) {
    const int w = omega[m];
    const int i = w / ny;
    idx[2 * m] = i;
    idx[2 * m + 1] = w - i * ny;
    y[m] = frame[w];
  }
}

extern "C" int tt_gather_entries(void* stream, int nx, int ny, const float* frame, const int32_t* omega,
                                 const int32_t* count, int cap, int32_t* idx_out, float* y_out) {
  if (nx < 1 || ny < 1 || cap < 0) return tt_fail(TT_EINVAL, "tt_gather_entries: bad shape");
  if (cap == 0) return TT_OK;
  if (!frame || !omega || !count || !idx_out || !y_out) return tt_fail(TT_EINVAL, "tt_gather_entries: null buffer");
  int blocks = (cap + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  ent_gather_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(ny, (const float2*)frame, omega, count, cap, idx_out,
                                                             (float2*)y_out);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}
