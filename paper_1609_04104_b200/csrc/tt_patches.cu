// Per-patch independent trackers (experiment._run_tracking_patched, experiment.py:332-441;
// mri.PatchGrid / patch_partition / patch_assemble, mri.py:48-177).
//
// The frame is tiled into k1 x k2 non-overlapping n1 x n2 patches, each tracked by its own
// rank-rho EntryMask tracker (track_step, tracker.py:367-411, on the patch's entries in local
// coordinates). Patches are independent, so the device layout is one CTA per patch, persistent
// over a whole epoch of frames: the patch factors, the dense residual scatter Theta and the
// staged regression rows stay in shared memory, and a step is a handful of block barriers.
//
//   patch_bin_kernel    one CTA per frame: the frame's entry list split into per-patch lists in
//                       measurement order (patch_batches' stable filter, experiment.py:352-370),
//                       values read from the frame (StreamingProvider.entries, :105-108)
//   patch_track_kernel  one CTA per patch: the schedule's steps in order (Gram + ridge solve +
//                       residual + back-projection + update), or, with `project`, the ridge
//                       re-projection of every frame onto the final subspace with the tile written
//                       straight into the assembled frame (experiment.py:419-431)
#include <math.h>

#include "tt_block.cuh"
#include "tt_common.cuh"

#define PT_NT 256
#define PT_MAXR 16

#define PT_SCH 1024  // schedule steps staged in shared memory at a time

struct PtLayout {
  size_t g, h, gam, colb, red, sc, cn, a, b, p, q, th, st, phi, ry, ri, total;
};
static __host__ __device__ inline size_t pt_al(size_t x) { return (x + 15) & ~(size_t)15; }
static __host__ __device__ inline PtLayout pt_layout(int n1, int n2, int R) {
  PtLayout s;
  const size_t cap = (size_t)n1 * n2;
  size_t o = 0;
  s.g = o;    o = pt_al(o + 16 * (size_t)(R * (R + 1) / 2));
  s.h = o;    o = pt_al(o + 16 * (size_t)R);
  s.gam = o;  o = pt_al(o + 16 * (size_t)R);
  s.colb = o; o = pt_al(o + 16 * 4 * (size_t)(R + 1));
  s.red = o;  o = pt_al(o + 8 * 32);
  s.sc = o;   o = pt_al(o + 4 * PT_SCH);  // schedule chunk: frame index per step
  s.cn = o;   o = pt_al(o + 4 * PT_SCH);  // ... and this patch's entry count per step
  s.a = o;    o = pt_al(o + 8 * (size_t)n1 * R);
  s.b = o;    o = pt_al(o + 8 * (size_t)n2 * R);
  s.p = o;    o = pt_al(o + 8 * (size_t)n1 * R);
  s.q = o;    o = pt_al(o + 8 * (size_t)n2 * R);
  s.th = o;   o = pt_al(o + 8 * cap);
  s.st = o;   o = pt_al(o + 4 * cap);
  s.phi = o;  o = pt_al(o + 8 * cap * R);
  s.ry = o;   o = pt_al(o + 2 * 8 * cap);  // [2][cap] complex64 values (double-buffered across steps)
  s.ri = o;   o = pt_al(o + 2 * 4 * cap);  // [2][cap] packed local (i << 16) | j
  s.total = o;
  return s;
}

TT_DEV double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
TT_DEV double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------- binning
// Stable split of each frame's entries by patch: within a chunk of 256 entries, lanes of a warp with
// the same patch rank themselves with __match_any_sync; the warps then take their per-patch base
// counts in warp order. Out-of-range entries raise TT_ST_BADROW, more entries than a patch holds
// (only possible with duplicates) TT_ST_OVERFLOW.
__global__ void __launch_bounds__(PT_NT) patch_bin_kernel(int nx, int ny, int n1, int n2,
                                                          const float2* __restrict__ frames,
                                                          const int2* __restrict__ ent, const int64_t* __restrict__ off,
                                                          int32_t* __restrict__ pidx, float2* __restrict__ py,
                                                          int32_t* __restrict__ pcnt, int32_t* __restrict__ status) {
  extern __shared__ int pc[];
  const int f = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k2 = ny / n2, np = (nx / n1) * k2, cap = n1 * n2;
  for (int q = tid; q < np; q += PT_NT) pc[q] = 0;
  __syncthreads();
  const long long l0 = off[f], l1 = off[f + 1];
  const int Lf = l1 > l0 ? (int)min(l1 - l0, (long long)INT32_MAX) : 0;
  const int2* e = ent + l0;
  int bad = 0;
  for (int base = 0; base < Lf; base += PT_NT) {
    const int l = base + tid;
    int pid = -1, loc = 0, i = 0, j = 0;
    if (l < Lf) {
      const int2 v = e[l];
      i = v.x;
      j = v.y;
      if (i >= 0 && i < nx && j >= 0 && j < ny) {
        const int pi = i / n1, qj = j / n2;
        pid = pi * k2 + qj;
        loc = ((i - pi * n1) << 16) | (j - qj * n2);
      } else {
        bad |= TT_ST_BADROW;
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, pid);
    const int rk = __popc(peers & ((1u << lane) - 1u));
    const int leader = __ffs(peers) - 1;
    int bc = 0;
    for (int w = 0; w < PT_NT / 32; ++w) {
      if (warp == w && pid >= 0) bc = pc[pid];
      __syncwarp();
      if (warp == w && pid >= 0 && lane == leader) pc[pid] = bc + __popc(peers);
      __syncthreads();
    }
    if (pid >= 0) {
      const int pos = bc + rk;
      if (pos < cap) {
        const size_t o = ((size_t)f * np + pid) * cap + pos;
        pidx[o] = loc;
        py[o] = frames[((size_t)f * nx + i) * ny + j];
      } else {
        bad |= TT_ST_OVERFLOW;
      }
    }
  }
  __syncthreads();
  for (int q = tid; q < np; q += PT_NT) pcnt[(size_t)f * np + q] = min(pc[q], cap);
  if (bad) atomicOr(status, bad);
}

// ---------------------------------------------------------------- tracking
// IPW = Gram / rhs items per warp (compile time: the item loop is branch-free; padding items are
// computed on index 0 and discarded)
template <int IPW>
__global__ void __launch_bounds__(PT_NT) patch_track_kernel(tt_patches_args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n1 = a.pn1, n2 = a.pn2, R = a.rank, cap = n1 * n2;
  const int k2 = a.ny / n2, np = (a.nx / n1) * k2;
  const int pl = blockIdx.x, p = a.patch0 + pl, nloc = gridDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const PtLayout S = pt_layout(n1, n2, R);
  double2* G = (double2*)(smem + S.g);
  double2* h = (double2*)(smem + S.h);
  double2* gam = (double2*)(smem + S.gam);
  double2* colb = (double2*)(smem + S.colb);
  double* red = (double*)(smem + S.red);
  float2* A = (float2*)(smem + S.a);
  float2* B = (float2*)(smem + S.b);
  float2* P = (float2*)(smem + S.p);
  float2* Q = (float2*)(smem + S.q);
  float2* th = (float2*)(smem + S.th);
  int* st = (int*)(smem + S.st);
  float2* phi = (float2*)(smem + S.phi);
  float2* ry = (float2*)(smem + S.ry);
  int* rin = (int*)(smem + S.ri);
  int* sc = (int*)(smem + S.sc);
  int* cn = (int*)(smem + S.cn);

  float2* gA = (float2*)a.a + (size_t)pl * n1 * R;
  float2* gB = (float2*)a.b + (size_t)pl * n2 * R;
  for (int e = tid; e < n1 * R; e += PT_NT) A[e] = gA[e];
  for (int e = tid; e < n2 * R; e += PT_NT) B[e] = gB[e];
  for (int e = tid; e < cap; e += PT_NT) st[e] = 0;
  long long t = a.t[pl];
  double ab = a.alpha_bar[pl];
  int status = 0;
  // this warp's Gram / rhs items it = warp + 8 m: packed lower triangle (i >= j) first, then the rhs
  const int nG = R * (R + 1) / 2, NI = nG + R;
  int ri[IPW], rj[IPW];
#pragma unroll
  for (int m = 0; m < IPW; ++m) {
    const int it = warp + 8 * m;
    ri[m] = 0;
    rj[m] = 0;
    if (it < nG) {
      int i = (int)((sqrtf(8.0f * it + 1.0f) - 1.0f) * 0.5f);
      while (i * (i + 1) / 2 > it) --i;
      while ((i + 1) * (i + 2) / 2 <= it) ++i;
      ri[m] = i;
      rj[m] = it - i * (i + 1) / 2;
    } else if (it < NI) {
      ri[m] = it - nG;
      rj[m] = -1;
    }
  }
  const bool hess = a.step_mode == 1;
  // the entries of step s are staged into buffer s & 1 with cp.async while step s - 1 computes;
  // every thread copies, and later reads first, the entries l = tid + k * PT_NT
  auto load_chunk = [&](int base) {  // the schedule and this patch's counts for steps [base, base + PT_SCH)
    for (int k = tid; k < min(PT_SCH, a.nsteps - base); k += PT_NT) {
      const int fr = a.sched[base + k];
      sc[k] = fr;
      cn[k] = min(a.pcnt[(size_t)fr * np + p], cap);
    }
  };
  auto prefetch = [&](int s, int buf) -> int {
    const size_t slot = (size_t)sc[s % PT_SCH] * np + p;
    const int Ln = cn[s % PT_SCH];
    const int32_t* gi = a.pidx + slot * cap;
    const float2* gy = (const float2*)a.py + slot * cap;
    for (int l = tid; l < Ln; l += PT_NT) {
      cp_async4(&rin[buf * cap + l], gi + l);
      cp_async8(&ry[buf * cap + l], gy + l);
    }
    return Ln;
  };
  load_chunk(0);
  __syncthreads();
  int Lnext = a.nsteps > 0 ? prefetch(0, 0) : 0;
  __syncthreads();

  for (int s = 0; s < a.nsteps; ++s) {
    const int buf = s & 1;
    const int f = sc[s % PT_SCH];
    const int Lc = Lnext;
    const int* li = rin + buf * cap;
    const float2* ly = ry + buf * cap;
    cp_async_wait_all();
    // regression rows Phi[l, r] = A[i, r] B[j, r] (observation.py:219-223)
    for (int l = tid; l < Lc; l += PT_NT) {
      const int pk = li[l];
      const int i = pk >> 16, j = pk & 0xffff;
      for (int r = 0; r < R; ++r) phi[l * R + r] = cmul(A[i * R + r], B[j * R + r]);
    }
    if (s + 1 < a.nsteps) {  // buffer buf ^ 1 was last read in step s - 1
      if ((s + 1) % PT_SCH == 0) {
        __syncthreads();
        load_chunk(s + 1);
        __syncthreads();
      }
      Lnext = prefetch(s + 1, buf ^ 1);
    }
    if (!a.project) {  // ||A||^2 + ||B||^2 for the cost (tracker.py:389)
      double en = 0.0;
      for (int e = tid; e < (n1 + n2) * R; e += PT_NT) en += (double)cabs2(e < n1 * R ? A[e] : B[e - n1 * R]);
      en = warp_sum_d(en);
      if (lane == 0) red[warp] = en;
    }
    __syncthreads();
    // Gram Phi^H Phi + lam I (packed lower triangle) and rhs Phi^H y: products in fp32, sums in fp64;
    // the lanes of a warp split the entries, a shuffle tree sums them
    {
      double2 acc[IPW];
#pragma unroll
      for (int m = 0; m < IPW; ++m) acc[m] = make_double2(0.0, 0.0);
      for (int l = lane; l < Lc; l += 32) {
        const float2* ph = phi + l * R;
        const float2 y = ly[l];
#pragma unroll
        for (int m = 0; m < IPW; ++m) {
          const float2 u = ph[ri[m]];
          const float2 w = ph[max(rj[m], 0)];
          const float2 v = rj[m] >= 0 ? w : y;
          acc[m].x += (double)fmaf(u.x, v.x, u.y * v.y);
          acc[m].y += (double)fmaf(u.x, v.y, -u.y * v.x);
        }
      }
#pragma unroll
      for (int m = 0; m < IPW; ++m) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          acc[m].x += __shfl_xor_sync(0xffffffffu, acc[m].x, o);
          acc[m].y += __shfl_xor_sync(0xffffffffu, acc[m].y, o);
        }
      }
      if (lane == 0) {
#pragma unroll
        for (int m = 0; m < IPW; ++m) {
          const int it = warp + 8 * m;
          double2 v = acc[m];
          if (it < nG) {
            if (ri[m] == rj[m]) v.x += a.lam;
            G[it] = v;
          } else if (it < NI) {
            h[ri[m]] = v;
          }
        }
      }
    }
    __syncthreads();
    // ridge solve (G + lam I) gamma = h (the SVD ridge of tracker.py:139-156 via the normal equations)
    block_gj_solve<2>(G, h, gam, colb, R);
    const bool empty = Lc == 0;  // tracker.py:380-384: gamma = 0, no update, t advances

    if (a.project) {  // re-projection + tile into the assembled frame (experiment.py:419-431)
      if (tid < R) ((float2*)a.gamma_out)[((size_t)s * nloc + pl) * R + tid] = empty ? make_float2(0.f, 0.f) : to_f2(gam[tid]);
      if (a.recon_out) {
        const int p1 = p / k2, q = p - p1 * k2;
        float2* X = (float2*)a.recon_out + (size_t)f * a.nx * a.ny;
        for (int e = tid; e < cap; e += PT_NT) {
          const int i = e / n2, j = e - (e / n2) * n2;
          float2 x = make_float2(0.f, 0.f);
          if (!empty)
            for (int r = 0; r < R; ++r) x = cfma(cmul(A[i * R + r], to_f2(gam[r])), B[j * R + r], x);
          X[(size_t)(p1 * n1 + i) * a.ny + q * n2 + j] = x;
        }
      }
      __syncthreads();
      continue;
    }

    // residual e = y - Phi gamma (fp64), scattered into Theta; the stamp marks this step's entries
    // (a second write to a stamped entry is a duplicate index, observation.py:41-55)
    const int cur = s + 1;
    {
      double ee = 0.0;
      for (int l = tid; l < Lc; l += PT_NT) {
        const float2* ph = phi + l * R;
        const float2 y = ly[l];
        double ex = y.x, ey = y.y;
        for (int r = 0; r < R; ++r) {
          const double2 g = gam[r];
          const double px = ph[r].x, py_ = ph[r].y;
          ex -= px * g.x - py_ * g.y;
          ey -= px * g.y + py_ * g.x;
        }
        const int pk = li[l];
        const int id = (pk >> 16) * n2 + (pk & 0xffff);
        if (atomicExch(&st[id], cur) == cur) status |= TT_ST_DUPROW;
        const float2 ef = make_float2((float)ex, (float)ey);
        th[id] = ef;
        if (a.resid_out) ((float2*)a.resid_out)[((size_t)s * nloc + pl) * cap + l] = ef;
        ee += ex * ex + ey * ey;
      }
      ee = warp_sum_d(ee);
      if (lane == 0) red[8 + warp] = ee;
    }
    __syncthreads();
    // back-projection P = Theta conj(B), Q = Theta^T conj(A) over this step's entries (the entry
    // branch of _gradient_data_terms, tracker.py:211-222), and for HessianBound the closed-form
    // per-(mode, r) curvature max_i sum_{j in Omega_i} |B[j, r]|^2
    {
      double am = 0.0;
      for (int o = tid; o < (n1 + n2) * R; o += PT_NT) {
        float2 acc = make_float2(0.f, 0.f);
        float c = 0.f;
        const bool rowA = o < n1 * R;
        const int o2 = rowA ? o : o - n1 * R;
        const int x = o2 / R, r = o2 - x * R;
        const int K = rowA ? n2 : n1;
        const int kst = rowA ? 1 : n2, k0 = rowA ? x * n2 : x;
        const float2* F = rowA ? B : A;
        for (int k = 0; k < K; ++k) {
          const int kk = k0 + k * kst;
          const bool in = st[kk] == cur;
          const float2 fv = F[k * R + r];
          const float2 tv = in ? th[kk] : make_float2(0.f, 0.f);
          acc = cfma_conj(tv, fv, acc);
          c += in ? cabs2(fv) : 0.f;
        }
        (rowA ? P : Q)[o2] = acc;
        if (hess) {
          const double2 g = gam[r];
          am = fmax(am, (g.x * g.x + g.y * g.y) * (double)c);
        }
      }
      if (hess) {
        am = warp_max_d(am);
        if (lane == 0) red[16 + warp] = am;
      }
    }
    __syncthreads();
    // step scalars, computed identically by every thread (tracker.py:386-398)
    double etot = 0.0, ee = 0.0, am = 0.0;
#pragma unroll
    for (int w = 0; w < PT_NT / 32; ++w) {
      etot += red[w];
      ee += red[8 + w];
      if (hess) am = fmax(am, red[16 + w]);
    }
    const double lt = a.lam / (double)t;
    const double cost = 0.5 * ee + 0.5 * lt * etot;
    double mu = 0.0;
    if (!empty) {
      if (hess) {
        const double alpha = fmin(fmax(lt + am, a.c_floor), a.c_cap);
        ab += alpha;
        mu = 1.0 / ab;
      } else {
        mu = a.mu;
      }
      // A <- A - mu ((lam / t) A - conj(gamma) P), likewise B (tracker.py:262, :402-404)
      const float c = (float)(1.0 - mu * lt);
      for (int e = tid; e < (n1 + n2) * R; e += PT_NT) {
        const bool inA = e < n1 * R;
        const int e2 = inA ? e : e - n1 * R;
        const int r = e2 - (e2 / R) * R;
        const double2 g = gam[r];
        const float2 w = make_float2((float)(mu * g.x), (float)(-mu * g.y));  // mu conj(gamma_r)
        float2* F = inA ? A : B;
        const float2 d = inA ? P[e2] : Q[e2];
        F[e2] = cfma(w, d, cscale(F[e2], c));
      }
    }
    if (tid < R) {
      const double2 g = gam[tid];
      if (!isfinite(g.x) || !isfinite(g.y)) status |= TT_ST_NONFINITE;
      if (a.gamma_out) ((float2*)a.gamma_out)[((size_t)s * nloc + pl) * R + tid] = empty ? make_float2(0.f, 0.f) : to_f2(g);
    }
    if (tid == 0) {
      if (a.cost_out) a.cost_out[(size_t)s * nloc + pl] = cost;
      if (a.mu_out) a.mu_out[(size_t)s * nloc + pl] = mu;
    }
    t += 1;
    __syncthreads();
  }
  if (!a.project) {
    for (int e = tid; e < n1 * R; e += PT_NT) gA[e] = A[e];
    for (int e = tid; e < n2 * R; e += PT_NT) gB[e] = B[e];
    if (tid == 0) {
      a.t[pl] = t;
      a.alpha_bar[pl] = ab;
    }
  }
  if (status) atomicOr(&a.status[pl], status);  // rare path: one atomic per offending thread
}

// ---------------------------------------------------------------- host
extern "C" size_t tt_patches_smem_bytes(int pn1, int pn2, int rank) {
  if (pn1 < 1 || pn2 < 1 || rank < 1) return 0;
  return pt_layout(pn1, pn2, rank).total;
}

extern "C" int tt_patch_bin(void* stream, int nx, int ny, int pn1, int pn2, int frames, const float* frame_data,
                            const int32_t* entries, const int64_t* offsets, int32_t* pidx, float* py, int32_t* pcnt,
                            int32_t* status) {
  if (nx < 1 || ny < 1 || pn1 < 1 || pn2 < 1 || frames < 0) return tt_fail(TT_EINVAL, "tt_patch_bin: bad sizes");
  if (nx % pn1 || ny % pn2) return tt_fail(TT_EINVAL, "patch size does not tile the frame");
  if (frames == 0) return TT_OK;
  if (!frame_data || !entries || !offsets || !pidx || !py || !pcnt || !status)
    return tt_fail(TT_EINVAL, "tt_patch_bin: null pointer");
  const size_t np = (size_t)(nx / pn1) * (ny / pn2);
  const size_t sm = sizeof(int) * np;
  if (sm > 200 * 1024) return tt_fail(TT_EUNSUPPORTED, "too many patches for the binning kernel");
  if (sm > 48 * 1024) TT_CUDA_TRY(cudaFuncSetAttribute(patch_bin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  patch_bin_kernel<<<frames, PT_NT, sm, (cudaStream_t)stream>>>(nx, ny, pn1, pn2, (const float2*)frame_data,
                                                                 (const int2*)entries, (const int64_t*)offsets, pidx,
                                                                 (float2*)py, pcnt, status);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}

extern "C" int tt_track_patches(void* stream, const tt_patches_args* a) {
  if (!a) return tt_fail(TT_EINVAL, "tt_track_patches: null args");
  if (a->nx < 1 || a->ny < 1 || a->pn1 < 1 || a->pn2 < 1 || a->nx % a->pn1 || a->ny % a->pn2)
    return tt_fail(TT_EINVAL, "patch size does not tile the frame");
  if (a->rank < 1) return tt_fail(TT_EINVAL, "rank must be positive");
  if (a->rank > PT_MAXR) return tt_fail(TT_EUNSUPPORTED, "patch rank above 16 is not supported by the patch kernel");
  const int np = (a->nx / a->pn1) * (a->ny / a->pn2);
  if (a->patch0 < 0 || a->npatch_local < 0 || a->patch0 + a->npatch_local > np)
    return tt_fail(TT_EINVAL, "patch range outside the grid");
  if (a->nsteps < 0 || a->frames < 0) return tt_fail(TT_EINVAL, "negative step / frame count");
  if (a->nsteps == 0 || a->npatch_local == 0) return TT_OK;
  if (!a->pidx || !a->py || !a->pcnt || !a->sched || !a->a || !a->b || !a->t || !a->alpha_bar || !a->status)
    return tt_fail(TT_EINVAL, "tt_track_patches: null pointer");
  if (a->project && !a->gamma_out) return tt_fail(TT_EINVAL, "projection needs gamma_out");
  if (a->step_mode != 0 && a->step_mode != 1) return tt_fail(TT_EINVAL, "unknown step mode");
  const size_t sm = pt_layout(a->pn1, a->pn2, a->rank).total;
  int dev = 0, optin = 0;
  TT_CUDA_TRY(cudaGetDevice(&dev));
  TT_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (sm > (size_t)optin)
    return tt_fail(TT_EUNSUPPORTED, "patch too large for the fused patch kernel (shared memory)");
  if (a->pn1 > 32767 || a->pn2 > 65535) return tt_fail(TT_EUNSUPPORTED, "patch extent too large");
  // items per warp: ceil((R (R + 1) / 2 + R) / 8), rounded up to an instantiated size
  const int R = a->rank, need = (R * (R + 1) / 2 + R + 7) / 8;
  static const int sizes[] = {1, 2, 3, 4, 6, 8, 12, 19};
  static void (*const fns[])(tt_patches_args) = {patch_track_kernel<1>, patch_track_kernel<2>, patch_track_kernel<3>,
                                                  patch_track_kernel<4>, patch_track_kernel<6>, patch_track_kernel<8>,
                                                  patch_track_kernel<12>, patch_track_kernel<19>};
  static size_t set_bytes[8][TT_MAXDEV] = {{0}};
  int which = 7;
  for (int k = 0; k < 8; ++k)
    if (sizes[k] >= need) {
      which = k;
      break;
    }
  if (sm > 48 * 1024) TT_CUDA_TRY(tt_smem_attr((const void*)fns[which], sm, set_bytes[which]));
  fns[which]<<<a->npatch_local, PT_NT, sm, (cudaStream_t)stream>>>(*a);
  TT_CUDA_TRY(cudaGetLastError());
  return TT_OK;
}
