// Generic online step for an arbitrary (i, j) index list (FourierMask /
// EntryMask, observation.py:58-90) on measurement-domain factors
// (Ah, Bh) = (F_x A, F_y B) for Fourier masks, (A, B) for entry masks — the
// two are the same iteration (test_mri.py:258-286).
//
//   1. ent_gram     thread-block clusters of 8 CTAs; each CTA stages its share of the entries
//                   and their regression rows Phi_l = Ah[i_l] .* Bh[j_l] in shared memory,
//                   accumulates G = Phi^H Phi, h = Phi^H y, ||y||^2 and its slice of
//                   ||Ah||^2 + ||Bh||^2 (fp32 products, fp64 sums), and the cluster sums its 8
//                   partials through distributed shared memory in fixed order
//                   (build_phi observation.py:219-228; solve_gamma tracker.py:139-156 as
//                   normal equations)
//   2. ent_solve    fixed-order sum of the cluster partials, G + lam I, fp64 Gauss-Jordan
//                   -> gamma, cost (tracker.py:386-389); advances the frame stamp
//   3. ent_resid    e_l = y_l - Phi_l gamma, written into the dense residual image Xi with
//                   the frame's stamp (the scatter of _scatter_theta, tracker.py:176-188)
//   4. ent_backproj P = Xi conj(Bh), Q = Xi^T conj(Ah) over this frame's stamped entries
//                   (collapsed gradient data terms, tracker.py:208-228); for HessianBound the
//                   closed-form curvature max_{m,r} |gamma_r|^2 c_m[., r] (hessian_bound
//                   tracker.py:337-364) as an order-free atomic max
//   5. ent_update   alpha / mu (tracker.py:391-400) and Ah <- (1 - mu lam/t) Ah + mu conj(gamma) P,
//                   same for Bh (tracker.py:402-404)
// Everything is deterministic (fixed reduction orders; the only atomic is a max). The stamps
// replace a per-frame clear of Xi: the scratch must be zero-filled before its first use.

#include <cooperative_groups.h>

#include "tt_block.cuh"

namespace cg = cooperative_groups;

#define ENT_NT 256
#define EG_CL 8       // CTAs per gram cluster
#define EG_NCL 16     // clusters at most (= partials the solve sums)
#define EG_TL 256     // entries staged per tile
#define EG_PER 128    // target entries per CTA
#define EG_MI 9       // items per thread (R <= 64: R(R+1)/2 + R + 1 <= 2145 <= 9 * 256)

// scal slots (8 bytes each): [0] cost, [1] mu, [2] curvature max (double bits, atomic max),
// [3] frame stamp counter (int64), [4] alpha_bar at the step's start
struct EntScratch {
  size_t gp, gam, scal, xi, st, P, Q, total;
};
static EntScratch ent_layout(int nx, int ny, int R) {
  EntScratch s;
  const size_t NI2 = (size_t)R * (R + 1) / 2 + R + 1;
  size_t o = 0;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  s.gp = o;   o = al(o + sizeof(double2) * EG_NCL * NI2);
  s.gam = o;  o = al(o + sizeof(double2) * R);
  s.scal = o; o = al(o + sizeof(double) * 16);
  s.xi = o;   o = al(o + sizeof(float2) * (size_t)nx * ny);
  s.st = o;   o = al(o + sizeof(int) * (size_t)nx * ny);
  s.P = o;    o = al(o + sizeof(float2) * (size_t)nx * R);
  s.Q = o;    o = al(o + sizeof(float2) * (size_t)ny * R);
  s.total = o;
  return s;
}
static size_t gram_smem(int R) {
  const size_t NI2 = (size_t)R * (R + 1) / 2 + R + 1;
  return sizeof(float2) * (size_t)EG_TL * (R + 1) + sizeof(int2) * EG_TL + sizeof(double2) * NI2 + sizeof(double) * 64;
}

// entry l of the step: (i, j) and y from the index list, or from the flat index into the resident frame
struct EntSrc {
  const int* idx;
  const float2* y;
  const int* omega;
  const float2* frame;
  int ny;
  TT_DEV void get(int l, int& i, int& j, float2& v) const {
    if (omega) {
      const int w = omega[l];
      i = w / ny;
      j = w - i * ny;
      v = frame[w];
    } else {
      i = idx[2 * l];
      j = idx[2 * l + 1];
      v = y[l];
    }
  }
};

__global__ void __cluster_dims__(EG_CL, 1, 1) __launch_bounds__(ENT_NT)
    ent_gram_kernel(int nmeas, const int* __restrict__ nmeas_dev, int nx, int ny, int R,
                    const float2* __restrict__ ah, const float2* __restrict__ bh, const EntSrc src,
                    double2* __restrict__ gp) {
  pdl_wait_and_trigger();
  if (nmeas_dev) nmeas = min(*nmeas_dev, nmeas);
  extern __shared__ __align__(16) unsigned char smem[];
  float2* phi = (float2*)smem;                   // [TL][R]
  float2* yv = phi + (size_t)EG_TL * R;          // [TL]
  int2* ij = (int2*)(yv + EG_TL);                // [TL]
  double2* part = (double2*)(ij + EG_TL);        // [NI2] this CTA's partial items
  const int Rp = R * (R + 1) / 2, NI = Rp + R, NI2 = NI + 1;
  double* red = (double*)(part + NI2);
  const int tid = threadIdx.x, NT = blockDim.x;
  const int b = blockIdx.x;
  const int l0 = (int)(((long long)nmeas * b) / gridDim.x), l1 = (int)(((long long)nmeas * (b + 1)) / gridDim.x);
  double2 acc[EG_MI];
#pragma unroll
  for (int m = 0; m < EG_MI; ++m) acc[m] = make_double2(0.0, 0.0);
  double ysq = 0.0;
  for (int t0 = l0; t0 < l1; t0 += EG_TL) {
    const int tl = min(EG_TL, l1 - t0);
    for (int ll = tid; ll < tl; ll += NT) {
      int i, j;
      float2 v;
      src.get(t0 + ll, i, j, v);
      ij[ll] = make_int2(i, j);
      yv[ll] = v;
      ysq += (double)v.x * v.x + (double)v.y * v.y;
    }
    __syncthreads();
    {  // gathered factor rows: eight iterations' loads in flight before any use
      constexpr int UP = 8;
      for (int o0 = tid; o0 < tl * R; o0 += NT * UP) {
        float2 av[UP], bv[UP];
#pragma unroll
        for (int u = 0; u < UP; ++u) {
          const int o = o0 + u * NT;
          if (o < tl * R) {
            const int ll = idiv(o, R), r = o - ll * R;
            const int2 q = ij[ll];
            av[u] = ah[(size_t)q.x * R + r];
            bv[u] = bh[(size_t)q.y * R + r];
          }
        }
#pragma unroll
        for (int u = 0; u < UP; ++u) {
          const int o = o0 + u * NT;
          if (o < tl * R) phi[o] = cmul(av[u], bv[u]);
        }
      }
    }
    __syncthreads();
    // item-outer: one guard per item, none per entry
#pragma unroll
    for (int m = 0; m < EG_MI; ++m) {
      const int it = tid + m * NT;
      if (it >= NI) break;
      double2 g = acc[m];
      if (it < Rp) {
        int r, q;
        tri_decode(it, r, q);
        for (int ll = 0; ll < tl; ++ll) {
          const float2 u = phi[ll * R + r], v = phi[ll * R + q];
          g.x += (double)fmaf(u.x, v.x, u.y * v.y);
          g.y += (double)fmaf(u.x, v.y, -u.y * v.x);
        }
      } else {
        const int r = it - Rp;
        for (int ll = 0; ll < tl; ++ll) {
          const float2 u = phi[ll * R + r], v = yv[ll];
          g.x += (double)fmaf(u.x, v.x, u.y * v.y);
          g.y += (double)fmaf(u.x, v.y, -u.y * v.x);
        }
      }
      acc[m] = g;
    }
    __syncthreads();
  }
  // this CTA's slice of ||Ah||^2 + ||Bh||^2 (the cost's regulariser, tracker.py:389)
  double en = 0.0;
  {
    const int E = (nx + ny) * R;
    const int e0 = (int)(((long long)E * b) / gridDim.x), e1 = (int)(((long long)E * (b + 1)) / gridDim.x);
    for (int e = e0 + tid; e < e1; e += NT) en += (double)cabs2(e < nx * R ? ah[e] : bh[e - nx * R]);
  }
  const double ys = block_sum(ysq, red);
  const double es = block_sum(en, red + 32);
#pragma unroll
  for (int m = 0; m < EG_MI; ++m) {
    const int it = tid + m * NT;
    if (it < NI) part[it] = acc[m];
  }
  if (tid == 0) part[NI] = make_double2(ys, es);
  // cluster sum of the 8 partials in fixed rank order, each CTA taking a slice of the items
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  const int rank = (int)cl.block_rank();
  const int per = (NI2 + EG_CL - 1) / EG_CL;
  const int i0 = rank * per, i1 = min(NI2, i0 + per);
  double2* dst = gp + (size_t)(b / EG_CL) * NI2;
  for (int it = i0 + tid; it < i1; it += NT) {
    double2 sum = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < EG_CL; ++c) sum = zadd(sum, cl.map_shared_rank(part, c)[it]);
    dst[it] = sum;
  }
  cl.sync();  // no CTA leaves while its partials are read
}

__global__ void __launch_bounds__(ENT_NT) ent_solve_kernel(int R, int nmeas, const int* __restrict__ nmeas_dev, int ncl,
                                                           double lam, long long t, const double2* __restrict__ gp,
                                                           const double* __restrict__ alpha_bar, double2* gam_out,
                                                           double* scal, float2* gamma_out, double* cost_out,
                                                           int32_t* status) {
  pdl_wait_and_trigger();
  extern __shared__ __align__(16) unsigned char smem[];
  if (nmeas_dev) nmeas = min(*nmeas_dev, nmeas);
  const int Rp = R * (R + 1) / 2, NI = Rp + R, NI2 = NI + 1;
  double2* G = (double2*)smem;   // [NI2]: G packed, h, (||y||^2, energy)
  double2* gam = G + NI2;
  double2* colb = gam + R;       // 4 (R + 1)
  const int tid = threadIdx.x, NT = blockDim.x;
  for (int it = tid; it < NI2; it += NT) {  // fixed-order sum of the cluster partials, loads in flight
    double2 v[EG_NCL];
#pragma unroll
    for (int c = 0; c < EG_NCL; ++c) v[c] = c < ncl ? gp[(size_t)c * NI2 + it] : make_double2(0.0, 0.0);
    double2 g = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < EG_NCL; ++c) g = zadd(g, v[c]);
    if (it < Rp) {
      int r, q;
      tri_decode(it, r, q);
      if (r == q) g.x += lam;
    }
    G[it] = g;
  }
  __syncthreads();
  const double yn = G[NI].x, energy = G[NI].y;
  const double lt = lam / (double)t;
  if (tid == 0) {
    long long* sl = (long long*)scal;
    sl[2] = 0;           // curvature max (bits of +0.0)
    sl[3] += 1;          // this frame's stamp
    scal[4] = alpha_bar[0];
  }
  if (nmeas == 0) {  // tracker.py:380-384
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
  double2 hsave = make_double2(0.0, 0.0);
  if (tid < R) hsave = G[Rp + tid];
  {
    const int ept = gj_ept(R, blockDim.x);
    if (ept <= 1) block_gj_solve<1>(G, G + Rp, gam, colb, R);
    else if (ept <= 2) block_gj_solve<2>(G, G + Rp, gam, colb, R);
    else if (ept <= 3) block_gj_solve<3>(G, G + Rp, gam, colb, R);
    else if (ept <= 5) block_gj_solve<5>(G, G + Rp, gam, colb, R);
    else block_ldl_solve(G, G + Rp, gam, R);
  }
  double gh = 0.0, gg = 0.0;
  if (tid < R) {
    const double2 g = gam[tid];
    gam_out[tid] = g;
    if (gamma_out) gamma_out[tid] = to_f2(g);
    gh = g.x * hsave.x + g.y * hsave.y;
    gg = g.x * g.x + g.y * g.y;
  }
  __shared__ double rgh[64], rgg[64];
  if (tid < 64) {
    rgh[tid] = tid < R ? gh : 0.0;
    rgg[tid] = tid < R ? gg : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    double sgh = 0.0, sgg = 0.0;
    for (int r = 0; r < R; ++r) {
      sgh += rgh[r];
      sgg += rgg[r];
    }
    const double cost = 0.5 * (yn - sgh - lam * sgg) + 0.5 * lt * energy;
    scal[0] = cost;
    if (cost_out) cost_out[0] = cost;
    if (!isfinite(cost) && status) atomicOr(status, TT_ST_NONFINITE);
  }
}

__global__ void ent_resid_kernel(int nmeas, const int* __restrict__ nmeas_dev, int ny, int R,
                                 const float2* __restrict__ ah, const float2* __restrict__ bh, const EntSrc src,
                                 const double2* gam, const double* scal, float2* __restrict__ xi,
                                 int* __restrict__ st, float2* __restrict__ resid) {
  pdl_wait_and_trigger();
  if (nmeas_dev) nmeas = min(*nmeas_dev, nmeas);
  const int cur = (int)((const long long*)scal)[3];
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nmeas; l += gridDim.x * blockDim.x) {
    int i, j;
    float2 yl;
    src.get(l, i, j, yl);
    double2 s = make_double2(0.0, 0.0);
    const float2* ar = ah + (size_t)i * R;
    const float2* br = bh + (size_t)j * R;
    int r = 0;
    for (; r + 8 <= R; r += 8) {  // eight row entries in flight
      float2 av[8], bv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        av[u] = ar[r + u];
        bv[u] = br[r + u];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) s = zfma(zmul(to_d2(av[u]), to_d2(bv[u])), gam[r + u], s);
    }
    for (; r < R; ++r) s = zfma(zmul(to_d2(ar[r]), to_d2(br[r])), gam[r], s);
    const float2 e = make_float2((float)((double)yl.x - s.x), (float)((double)yl.y - s.y));
    xi[(size_t)i * ny + j] = e;
    st[(size_t)i * ny + j] = cur;
    if (resid) resid[l] = e;
  }
}

// role 0 (blockIdx.y = 0): rows i of P; role 1: rows j of Q. Block = 32 outputs x 8 parts of the
// contraction index, summed in fixed order through shared memory. HessianBound: the block's max of
// |gamma_r|^2 sum_{stamped} |other factor|^2 joins the frame's max (order-free).
#define BP_O 32
#define BP_K 8
__global__ void __launch_bounds__(BP_O * BP_K) ent_backproj_kernel(int nx, int ny, int R, int hess,
                                                                   const float2* __restrict__ ah,
                                                                   const float2* __restrict__ bh,
                                                                   const float2* __restrict__ xi,
                                                                   const int* __restrict__ st, const double2* gam,
                                                                   double* scal, float2* __restrict__ P,
                                                                   float2* __restrict__ Q) {
  pdl_wait_and_trigger();
  __shared__ float2 sacc[BP_K][BP_O];
  __shared__ float scs[BP_K][BP_O];
  __shared__ double smax[BP_O * BP_K / 32];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int cur = (int)((const long long*)scal)[3];
  const int o = blockIdx.x * BP_O + tx;
  const bool rows = blockIdx.y == 0;
  const int m = rows ? nx * R : ny * R;
  float2 acc = make_float2(0.f, 0.f);
  float cs = 0.f;
  if (o < m) {
    const int x = o / R, r = o - x * R;
    const int K = rows ? ny : nx;
    const size_t xs = rows ? 1 : (size_t)ny, base = rows ? (size_t)x * ny : (size_t)x;
    const float2* F = rows ? bh : ah;
    int k = ty;
    for (; k + 3 * BP_K < K; k += 4 * BP_K) {  // four entries in flight
      float2 tv[4], fv[4];
      bool in[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const size_t kk = base + (size_t)(k + u * BP_K) * xs;
        in[u] = st[kk] == cur;
        tv[u] = xi[kk];
        fv[u] = F[(size_t)(k + u * BP_K) * R + r];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc = cfma_conj(in[u] ? tv[u] : make_float2(0.f, 0.f), fv[u], acc);
        cs += in[u] ? cabs2(fv[u]) : 0.f;
      }
    }
    for (; k < K; k += BP_K) {
      const size_t kk = base + (size_t)k * xs;
      const bool in = st[kk] == cur;
      const float2 fv = F[(size_t)k * R + r];
      acc = cfma_conj(in ? xi[kk] : make_float2(0.f, 0.f), fv, acc);
      cs += in ? cabs2(fv) : 0.f;
    }
  }
  sacc[ty][tx] = acc;
  scs[ty][tx] = cs;
  __syncthreads();
  double top = 0.0;
  if (ty == 0 && o < m) {
    for (int k = 1; k < BP_K; ++k) {
      acc = cadd(acc, sacc[k][tx]);
      cs += scs[k][tx];
    }
    (rows ? P : Q)[o] = acc;
    if (hess) {
      const double2 g = gam[o % R];
      top = (g.x * g.x + g.y * g.y) * (double)cs;
    }
  }
  if (hess) {
    const int w = (ty * BP_O + tx) >> 5, lane = tx & 31;
    top = warp_max(top);
    if (lane == 0) smax[w] = top;
    __syncthreads();
    if (ty == 0 && tx == 0) {
      double t2 = 0.0;
      for (int k = 0; k < BP_O * BP_K / 32; ++k) t2 = fmax(t2, smax[k]);
      // non-negative doubles order like their bit patterns
      atomicMax((unsigned long long*)&scal[2], (unsigned long long)__double_as_longlong(t2));
    }
  }
}

// step size (tracker.py:391-400) computed identically by every block from the step-start alpha_bar;
// block 0 publishes it. Then Ah <- (1 - mu lam/t) Ah + mu conj(gamma) P, likewise Bh.
__global__ void ent_update_kernel(int nx, int ny, int R, int nmeas, const int* __restrict__ nmeas_dev, double lam,
                                  long long t, int step_mode, double mu_fixed, double c_floor, double c_cap,
                                  double* scal, double* alpha_bar, const double2* gam, const float2* ah,
                                  const float2* bh, const float2* __restrict__ P, const float2* __restrict__ Q,
                                  float2* ah_out, float2* bh_out, double* mu_out, double* alpha_out) {
  pdl_wait_and_trigger();
  if (nmeas_dev) nmeas = min(*nmeas_dev, nmeas);
  const double lt = lam / (double)t;
  double m = 0.0, alpha = 0.0, ab = scal[4];
  if (nmeas > 0) {
    if (step_mode == TT_STEP_HESSIAN) {
      const double top = __longlong_as_double(((const long long*)scal)[2]);
      alpha = fmin(fmax(lt + top, c_floor), c_cap);
      ab += alpha;
      m = 1.0 / ab;
    } else {
      m = mu_fixed;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    alpha_bar[0] = ab;
    scal[1] = m;
    if (mu_out) mu_out[0] = m;
    if (alpha_out) alpha_out[0] = alpha;
  }
  const float cfac = (float)(1.0 - m * lt);
  const float muf = (float)m;
  const int na = nx * R, nbb = ny * R;
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < na + nbb; o += gridDim.x * blockDim.x) {
    if (o < na) {
      const int r = o % R;
      const float2 g = cconj(to_f2(gam[r]));
      ah_out[o] = nmeas > 0 ? cadd(cscale(ah[o], cfac), cscale(cmul(g, P[o]), muf)) : ah[o];
    } else {
      const int k = o - na, r = k % R;
      const float2 g = cconj(to_f2(gam[r]));
      bh_out[k] = nmeas > 0 ? cadd(cscale(bh[k], cfac), cscale(cmul(g, Q[k]), muf)) : bh[k];
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
  if (L > 0 && !a->omega && (!a->idx || !a->y)) return tt_fail(TT_EINVAL, "tt_track_entries: null idx/y");
  if (a->omega && !a->frame) return tt_fail(TT_EINVAL, "tt_track_entries: omega without frame");
  const EntSrc src{a->idx, (const float2*)a->y, a->omega, (const float2*)a->frame, ny};
  cudaStream_t st = (cudaStream_t)stream;
  const EntScratch S = ent_layout(nx, ny, R);
  unsigned char* sb = (unsigned char*)a->scratch;
  double2* gp = (double2*)(sb + S.gp);
  double2* gam = (double2*)(sb + S.gam);
  double* scal = (double*)(sb + S.scal);
  float2* xi = (float2*)(sb + S.xi);
  int* stp = (int*)(sb + S.st);
  float2* P = (float2*)(sb + S.P);
  float2* Q = (float2*)(sb + S.Q);
  const int Rp = R * (R + 1) / 2, NI2 = Rp + R + 1;
  const float2* ah = (const float2*)a->ah_in;
  const float2* bh = (const float2*)a->bh_in;
  // gram: clusters of 8 CTAs, about EG_PER entries per CTA, at most EG_NCL clusters
  int ncl = (L + EG_CL * EG_PER - 1) / (EG_CL * EG_PER);
  if (ncl < 1) ncl = 1;
  if (ncl > EG_NCL) ncl = EG_NCL;
  {
    const size_t sm = gram_smem(R);
    static size_t set_gram[TT_MAXDEV] = {0};
    TT_CUDA_TRY(tt_smem_attr((const void*)ent_gram_kernel, sm, set_gram));
    TT_CUDA_TRY(tt_launch_pdl(ent_gram_kernel, dim3(ncl * EG_CL), dim3(ENT_NT), sm, st,
        L, Ld, nx, ny, R, ah, bh, src, gp));
  }
  {
    const size_t sm = sizeof(double2) * ((size_t)NI2 + R + 4 * (size_t)(R + 1));
    static size_t set_solve[TT_MAXDEV] = {0};
    TT_CUDA_TRY(tt_smem_attr((const void*)ent_solve_kernel, sm, set_solve));
    TT_CUDA_TRY(tt_launch_pdl(ent_solve_kernel, dim3(1), dim3(ENT_NT), sm, st,
        R, L, Ld, ncl, a->lam, (long long)a->t, gp, a->alpha_bar, gam, scal, (float2*)a->gamma_out, a->cost_out,
        a->status));
  }
  if (L > 0) {
    int blocks = (L + 255) / 256;
    if (blocks > 1184) blocks = 1184;
    TT_CUDA_TRY(tt_launch_pdl(ent_resid_kernel, dim3(blocks), dim3(256), 0, st,
        L, Ld, ny, R, ah, bh, src, gam, scal, xi, stp, (float2*)a->resid_out));
    const int m = (nx > ny ? nx : ny) * R;
    dim3 grid((m + BP_O - 1) / BP_O, 2);
    TT_CUDA_TRY(tt_launch_pdl(ent_backproj_kernel, grid, dim3(BP_O, BP_K), 0, st,
        nx, ny, R, a->step_mode == TT_STEP_HESSIAN, ah, bh, xi, stp, gam, scal, P, Q));
  }
  {
    const int n = (nx + ny) * R;
    int blocks = (n + 255) / 256;
    if (blocks > 1184) blocks = 1184;
    TT_CUDA_TRY(tt_launch_pdl(ent_update_kernel, dim3(blocks), dim3(256), 0, st,
        nx, ny, R, L, Ld, a->lam, (long long)a->t, a->step_mode, a->mu, a->c_floor, a->c_cap, scal, a->alpha_bar,
        gam, ah, bh, P, Q, (float2*)a->ah_out, (float2*)a->bh_out, a->mu_out, a->alpha_out));
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
