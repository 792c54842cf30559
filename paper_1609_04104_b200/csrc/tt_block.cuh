// Block-level building blocks shared by the tensortrack kernels:
// deterministic scans, the numpy-exact weighted draw, and the fp64 LDL^H
// ridge solve. All functions must be called by every thread of the block.
#pragma once

#include "tt_common.cuh"

// ---------------------------------------------------------------- PTX helpers
TT_DEV void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
TT_DEV void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
TT_DEV void cluster_barrier() {
  cluster_arrive();
  cluster_wait();
}
TT_DEV void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
TT_DEV void cp_async4(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
TT_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// mbarrier + bulk-copy (TMA) helpers: a row of Y is one cp.async.bulk of contiguous bytes into shared
// memory, completion counted in bytes on an mbarrier (one arrival per phase: the issuing lane's
// arrive.expect_tx), every consumer thread waits on the phase parity.
TT_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
TT_DEV void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
TT_DEV void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
TT_DEV void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "TT_MBW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TT_MBW_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// generic-proxy accesses of shared memory ordered before later async-proxy (bulk copy) accesses
TT_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
TT_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// packed lower-triangular index helpers (r >= q)
TT_DEV void tri_decode(int e, int& r, int& q) {
  int rr = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
  while (rr * (rr + 1) / 2 > e) --rr;
  while ((rr + 1) * (rr + 2) / 2 <= e) ++rr;
  r = rr;
  q = e - rr * (rr + 1) / 2;
}
TT_DEV int tri_idx(int r, int q) { return r * (r + 1) / 2 + q; }

// fp64 reciprocal without the IEEE division sequence on the critical path:
// MUFU approximation + two Newton steps (error ~ 1 ulp), for LDL pivots.
TT_DEV double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-x, r, 2.0);
  r = r * fma(-x, r, 2.0);
  return r;
}

// ---------------------------------------------------------------- scans
// Block-wide exclusive scan of per-thread integer counts (deterministic).
TT_DEV int block_excl_scan_int(int v, int* red, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) red[warp] = x;
  __syncthreads();
  int off = 0;
  total = 0;
  for (int w = 0; w < nw; ++w) {
    if (w < warp) off += red[w];
    total += red[w];
  }
  __syncthreads();
  return off + x - v;
}
// Block-wide exclusive scan of per-thread doubles (fixed association order).
TT_DEV double block_excl_scan_dbl(double v, double* red, double& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) red[warp] = x;
  __syncthreads();
  double off = 0.0;
  total = 0.0;
  for (int w = 0; w < nw; ++w) {
    if (w < warp) off += red[w];
    total += red[w];
  }
  __syncthreads();
  return off + (x - v);
}

// Sum of p[0..n) over the block (chunked, fixed order); every thread receives the total.
TT_DEV double block_sum_range(const double* p, int n, double* red, double& total) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int chunk = (n + NT - 1) / NT;
  const int c0 = min(n, tid * chunk), c1 = min(n, c0 + chunk);
  double local = 0.0;
  for (int i = c0; i < c1; ++i) local += p[i];
  return block_excl_scan_dbl(local, red, total);
}

TT_DEV int upper_bound_d(const double* cdf, int n, double u) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (cdf[mid] <= u) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Inclusive prefix sums of p[0..n) into cdf with the chunked parallel order;
// `exact` selects numpy's sequential add.accumulate order (thread 0 only).
TT_DEV void block_cumsum(const double* p, double* cdf, int n, bool exact, double* red) {
  const int tid = threadIdx.x, NT = blockDim.x;
  if (exact) {
    if (tid == 0) {
      double c = 0.0;
      for (int i = 0; i < n; ++i) {
        c += p[i];
        cdf[i] = c;
      }
    }
    __syncthreads();
    return;
  }
  const int chunk = (n + NT - 1) / NT;
  const int c0 = min(n, tid * chunk), c1 = min(n, c0 + chunk);
  double local = 0.0;
  for (int i = c0; i < c1; ++i) local += p[i];
  double total;
  double run = block_excl_scan_dbl(local, red, total);
  for (int i = c0; i < c1; ++i) {
    run += p[i];
    cdf[i] = run;
  }
  __syncthreads();
}

// ---------------------------------------------------------------- weighted draws
// numpy Generator.choice(n, size, replace=True, p) semantics
// (sampler.py:160-162): cdf = cumsum(p); cdf /= cdf[-1];
// idx = searchsorted(cdf, u, 'right') for u = Generator.random().
// A parallel scan is used first; if any uniform lands within 1e-12 of a CDF
// boundary the exact sequential cumsum is recomputed and every draw redone, so
// the result is bit-identical to numpy for identical probabilities.
// Marks flags[idx] = 1 (flags cleared here), then adds forced indices and
// compacts the flags into sorted unique rows (np.union1d semantics).
template <bool EXACT_DIV = true>
TT_DEV void draw_with_replacement_block(const double* p, double* cdf, int* flags, int* rows, int& S, int n,
                                        int ndraw, const int* forced, int nforced, uint64_t k0, uint64_t k1,
                                        uint64_t pos, double* red, int* sh_flag,
                                        const double* utab = nullptr) {
  const int tid = threadIdx.x, NT = blockDim.x;
  for (int i = tid; i < n; i += NT) flags[i] = 0;
  if (tid == 0) *sh_flag = 0;
  for (int exact = 0; exact < 2; ++exact) {
    block_cumsum(p, cdf, n, exact != 0, red);
    const double last = cdf[n - 1];
    __syncthreads();
    if (EXACT_DIV || exact) {
      for (int i = tid; i < n; i += NT) cdf[i] = cdf[i] / last;
    } else {
      const double il = fast_rcp(last);
      for (int i = tid; i < n; i += NT) cdf[i] = cdf[i] * il;
    }
    __syncthreads();
    for (int m = tid; m < ndraw; m += NT) {
      const double u = draw_uniform(utab, k0, k1, pos, (uint64_t)m);
      int idx = upper_bound_d(cdf, n, u);
      if (!exact) {
        const double lo = idx > 0 ? cdf[idx - 1] : -1.0;
        const double hi = idx < n ? cdf[idx] : 2.0;
        if (u - lo <= 1e-12 || hi - u <= 1e-12) *sh_flag = 1;
      }
      flags[idx < n ? idx : n - 1] = 1;
    }
    __syncthreads();
    const int redo = *sh_flag;
    __syncthreads();
    if (exact || !redo) break;
    for (int i = tid; i < n; i += NT) flags[i] = 0;
    __syncthreads();
  }
  for (int m = tid; m < nforced; m += NT) {
    const int f = forced[m];
    if (f >= 0 && f < n) flags[f] = 1;
  }
  __syncthreads();
  const int chunk = (n + NT - 1) / NT;
  const int c0 = min(n, tid * chunk), c1 = min(n, c0 + chunk);
  int cnt = 0;
  for (int i = c0; i < c1; ++i) cnt += flags[i];
  int tot;
  int o = block_excl_scan_int(cnt, (int*)red, tot);
  for (int i = c0; i < c1; ++i)
    if (flags[i]) rows[o++] = i;
  S = tot;
  __syncthreads();
}

// ---------------------------------------------------------------- fp64 ridge solve
// Solves (G) gamma = h for Hermitian G given as a packed lower triangle
// (overwritten) by a right-looking LDL^H with the right-hand side eliminated
// alongside (one barrier per column), then a warp back-substitution.
// Non-positive pivots are dropped (their component is set to zero), which
// reproduces the reference's s > 0 filter (tracker.py:154-155) for exactly
// rank-deficient systems at lam = 0. `hv` is overwritten.
TT_DEV void block_ldl_solve(double2* G, double2* hv, double2* gam, int R) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5;
  __syncthreads();
  for (int k = 0; k < R; ++k) {
    const double d = G[tri_idx(k, k)].x;
    const double inv = d > 0.0 ? 1.0 / d : 0.0;
    const int m = R - k - 1;
    for (int o = tid; o < m * m + m; o += NT) {
      if (o < m * m) {
        const int ii = k + 1 + o / m, jj = k + 1 + o % m;
        if (jj <= ii) {
          const double2 lik = G[tri_idx(ii, k)], ljk = G[tri_idx(jj, k)];
          double2 g = G[tri_idx(ii, jj)];
          const double2 pr = zmul(lik, zconj(ljk));
          g.x -= pr.x * inv;
          g.y -= pr.y * inv;
          G[tri_idx(ii, jj)] = g;
        }
      } else {
        const int ii = k + 1 + (o - m * m);
        const double2 pr = zmul(G[tri_idx(ii, k)], hv[k]);
        hv[ii].x -= pr.x * inv;
        hv[ii].y -= pr.y * inv;
      }
    }
    __syncthreads();
  }
  if (warp == 0) {
    for (int k = R - 1; k >= 0; --k) {
      const double d = G[tri_idx(k, k)].x;
      const double inv = d > 0.0 ? 1.0 / d : 0.0;
      double2 acc = make_double2(0.0, 0.0);
      for (int j = k + 1 + lane; j < R; j += 32) acc = zfma_cj(G[tri_idx(j, k)], gam[j], acc);
      acc.x = warp_sum(acc.x);
      acc.y = warp_sum(acc.y);
      if (lane == 0) gam[k] = make_double2((hv[k].x - acc.x) * inv, (hv[k].y - acc.y) * inv);
      __syncwarp();
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- cluster-part sums
// Sum of CL (<= 16) values at p, p+stride, ... read with ld.global.cg. All
// loads are issued before the adds (one L2 round trip, not CL dependent ones);
// the fixed 0..CL-1 order keeps every CTA bit-identical.
TT_DEV double sum_parts(const double* p, size_t stride, int CL) {
  double v[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) v[c] = c < CL ? __ldcg(p + c * stride) : 0.0;
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 16; ++c) s += v[c];
  return s;
}
TT_DEV double2 sum_parts2(const double2* p, size_t stride, int CL) {
  double2 v[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    v[c].x = c < CL ? __ldcg(&p[c * stride].x) : 0.0;
    v[c].y = c < CL ? __ldcg(&p[c * stride].y) : 0.0;
  }
  double2 s = make_double2(0.0, 0.0);
#pragma unroll
  for (int c = 0; c < 16; ++c) s = zadd(s, v[c]);
  return s;
}
// Any number of parts (the Z partials: CL CTAs x K parts): batches of 16 loads in flight, fixed order.
TT_DEV double2 sum_parts2n(const double2* p, size_t stride, int n) {
  double2 s = make_double2(0.0, 0.0);
  for (int c0 = 0; c0 < n; c0 += 16) {
    double2 v[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      v[c].x = c0 + c < n ? __ldcg(&p[(size_t)(c0 + c) * stride].x) : 0.0;
      v[c].y = c0 + c < n ? __ldcg(&p[(size_t)(c0 + c) * stride].y) : 0.0;
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) s = zadd(s, v[c]);
  }
  return s;
}
TT_DEV float2 sum_parts_f2(const float2* p, size_t stride, int CL) {
  float2 v[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    v[c].x = c < CL ? __ldcg(&p[c * stride].x) : 0.f;
    v[c].y = c < CL ? __ldcg(&p[c * stride].y) : 0.f;
  }
  float2 s = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 16; ++c) s = cadd(s, v[c]);
  return s;
}

// ---------------------------------------------------------------- fast fp64 LDL^H solve
// Same factorisation as block_ldl_solve, organised for latency: `tab[e]`
// holds the pre-decoded (i << 8 | j) of packed entry e, the owner of the next
// diagonal publishes its reciprocal pivot inside the step (one barrier per
// column), and the back substitution is column-oriented in warp 0 (one
// shuffle broadcast per step). R <= 64.
TT_DEV void ldl_table_init(unsigned short* tab, int R) {
  const int Rp = R * (R + 1) / 2;
  for (int e = threadIdx.x; e < Rp; e += blockDim.x) {
    int r, q;
    tri_decode(e, r, q);
    tab[e] = (unsigned short)((r << 8) | q);
  }
}

TT_DEV void block_ldl_solve_fast(double2* G, double2* hv, double2* gam, double* inv, const unsigned short* tab,
                                 int R) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int Rp = R * (R + 1) / 2;
  if (tid == 0) {
    const double d = G[0].x;
    inv[0] = d > 0.0 ? fast_rcp(d) : 0.0;
  }
  __syncthreads();
  for (int k = 0; k < R - 1; ++k) {
    const double ik = inv[k];
    const int e0 = (k + 1) * (k + 2) / 2;  // first entry of row k+1; rows <= k never change
    for (int e = e0 + tid; e < Rp; e += NT) {
      const int ij = tab[e];
      const int i = ij >> 8, j = ij & 255;
      if (j > k) {
        const double2 lik = G[i * (i + 1) / 2 + k], ljk = G[j * (j + 1) / 2 + k];
        double2 g = G[e];
        g.x -= (lik.x * ljk.x + lik.y * ljk.y) * ik;
        g.y -= (lik.y * ljk.x - lik.x * ljk.y) * ik;
        G[e] = g;
        if (i == k + 1 && j == k + 1) inv[k + 1] = g.x > 0.0 ? fast_rcp(g.x) : 0.0;
      }
    }
    if (tid > k && tid < R) {
      const double2 lik = G[tid * (tid + 1) / 2 + k], hk = hv[k];
      hv[tid].x -= (lik.x * hk.x - lik.y * hk.y) * ik;
      hv[tid].y -= (lik.x * hk.y + lik.y * hk.x) * ik;
    }
    __syncthreads();
  }
  if (tid < 32) {
    double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
    for (int k = R - 1; k >= 0; --k) {
      const int own = k & 31;
      double gx = 0.0, gy = 0.0;
      if (tid == own) {
        const double2 a = k < 32 ? a0 : a1;
        gx = (hv[k].x - a.x) * inv[k];
        gy = (hv[k].y - a.y) * inv[k];
        gam[k] = make_double2(gx, gy);
      }
      gx = __shfl_sync(0xffffffffu, gx, own);
      gy = __shfl_sync(0xffffffffu, gy, own);
      const int kb = k * (k + 1) / 2;
      if (tid < k) {
        const double2 g = G[kb + tid];
        a0.x += g.x * gx + g.y * gy;
        a0.y += g.x * gy - g.y * gx;
      }
      if (tid + 32 < k) {
        const double2 g = G[kb + tid + 32];
        a1.x += g.x * gx + g.y * gy;
        a1.y += g.x * gy - g.y * gx;
      }
    }
  }
  __syncthreads();
}

// Warp-synchronous variant for the fused per-frame kernel: warp 0 alone runs
// the factorisation (no CTA barriers between columns, only __syncwarp), every
// lane recomputing the reciprocal pivot itself. Other warps only meet the
// closing __syncthreads. Same arithmetic as block_ldl_solve_fast.
TT_DEV void warp_ldl_solve(double2* G, double2* hv, double2* gam, const unsigned short* tab, int R) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    const int lane = tid;
    const int Rp = R * (R + 1) / 2;
    for (int k = 0; k < R - 1; ++k) {
      const double d = G[k * (k + 1) / 2 + k].x;
      const double ik = d > 0.0 ? fast_rcp(d) : 0.0;
      const int e0 = (k + 1) * (k + 2) / 2;
#pragma unroll 2
      for (int e = e0 + lane; e < Rp; e += 32) {
        const int ij = tab[e];
        const int i = ij >> 8, j = ij & 255;
        if (j > k) {
          const double2 lik = G[i * (i + 1) / 2 + k], ljk = G[j * (j + 1) / 2 + k];
          double2 g = G[e];
          g.x -= (lik.x * ljk.x + lik.y * ljk.y) * ik;
          g.y -= (lik.y * ljk.x - lik.x * ljk.y) * ik;
          G[e] = g;
        }
      }
      for (int i = k + 1 + lane; i < R; i += 32) {
        const double2 lik = G[i * (i + 1) / 2 + k], hk = hv[k];
        hv[i].x -= (lik.x * hk.x - lik.y * hk.y) * ik;
        hv[i].y -= (lik.x * hk.y + lik.y * hk.x) * ik;
      }
      __syncwarp();
    }
    double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
    for (int k = R - 1; k >= 0; --k) {
      const int own = k & 31;
      const double d = G[k * (k + 1) / 2 + k].x;
      const double ik = d > 0.0 ? fast_rcp(d) : 0.0;
      double gx = 0.0, gy = 0.0;
      if (lane == own) {
        const double2 a = k < 32 ? a0 : a1;
        gx = (hv[k].x - a.x) * ik;
        gy = (hv[k].y - a.y) * ik;
        gam[k] = make_double2(gx, gy);
      }
      gx = __shfl_sync(0xffffffffu, gx, own);
      gy = __shfl_sync(0xffffffffu, gy, own);
      const int kb = k * (k + 1) / 2;
      if (lane < k) {
        const double2 g = G[kb + lane];
        a0.x += g.x * gx + g.y * gy;
        a0.y += g.x * gy - g.y * gx;
      }
      if (lane + 32 < k) {
        const double2 g = G[kb + lane + 32];
        a1.x += g.x * gx + g.y * gy;
        a1.y += g.x * gy - g.y * gx;
      }
    }
  }
  __syncthreads();
}

// value of row `row` held by lane row % 32 in (a0: rows < 32, a1: rows >= 32), broadcast to the warp
TT_DEV double2 shfl_d2_sel(double2 a0, double2 a1, int row) {
  const double2 v = row < 32 ? a0 : a1;
  double2 o;
  o.x = __shfl_sync(0xffffffffu, v.x, row & 31);
  o.y = __shfl_sync(0xffffffffu, v.y, row & 31);
  return o;
}

// ---------------------------------------------------------------- 2x2-blocked register LDL^H
// Solves (G) gamma = h for Hermitian positive (semi)definite G given as a
// packed lower triangle, with 2x2 pivot blocks: R/2 elimination steps and
// R/2 back-substitution steps instead of R each (the per-step latency of a
// barrier-synchronised chain dominates at R <= 64). Thread t owns entries
// e = t + m*NT of the augmented system (packed lower entries 0..Rp-1, then the
// rhs "column" R as entries Rp + i) in registers. The two pivot columns of
// each step are final after the previous step; their owners publish them to a
// double-buffered column buffer (slot R holds conj(h)). Singular pivot blocks
// (det <= 0) drop their components, mirroring the s > 0 filter of the
// reference SVD ridge (tracker.py:154-155).
//   scratch: colb 2*2*(R+1) double2 | blk (R/2+1)*4 double | zf R double2
//   Gio: packed lower in / final factor out. Ends with __syncthreads.
template <int EPT>
TT_DEV void block_ldl2_solve(double2* Gio, const double2* hin, double2* gam, double2* colb, double* blk, double2* zf,
                             int R) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int Rp = R * (R + 1) / 2, E = Rp + R, W = R + 1;
  // Entries are handed out in column-major order (column j has rows j..R-1), so the
  // columns eliminated first sit at the low thread indices: as the elimination proceeds
  // whole warps retire and skip the update (warp-uniform branch).
  int ri[EPT], rj[EPT];
  double2 g[EPT];
#pragma unroll
  for (int m = 0; m < EPT; ++m) {
    const int e = tid + m * NT;
    ri[m] = -1;
    rj[m] = -1;
    g[m] = make_double2(0.0, 0.0);
    if (e < Rp) {
      int q = 0, off = 0;
      while (off + (R - q) <= e) {
        off += R - q;
        ++q;
      }
      const int r = q + (e - off);
      ri[m] = r;
      rj[m] = q;
      g[m] = Gio[r * (r + 1) / 2 + q];
    } else if (e < E) {
      ri[m] = e - Rp;
      rj[m] = R;
      g[m] = hin[e - Rp];
    }
    // publish block 0 columns (0, 1) into buffer 0
    if (rj[m] == 0 || rj[m] == 1) colb[rj[m] * W + ri[m]] = g[m];
    if (rj[m] == R && ri[m] < 2) colb[ri[m] * W + R] = zconj(g[m]);
  }
  __syncthreads();
  const int nb = (R + 1) / 2;
  for (int b = 0; b < nb; ++b) {
    const int k = 2 * b;
    const bool pair = k + 1 < R;
    const double2* c0 = colb + (b & 1) * 2 * W;
    const double2* c1 = c0 + W;
    double2* n0 = colb + ((b + 1) & 1) * 2 * W;
    double2* n1 = n0 + W;
    const double a = c0[k].x;
    const double2 c = pair ? c0[k + 1] : make_double2(0.0, 0.0);
    const double bb = pair ? c1[k + 1].x : 0.0;
    double id;  // 1 / det (pair) or 1 / a (single)
    if (pair) {
      const double det = a * bb - (c.x * c.x + c.y * c.y);
      id = det > 0.0 ? fast_rcp(det) : 0.0;
    } else {
      id = a > 0.0 ? fast_rcp(a) : 0.0;
    }
    if (tid == 0) {
      blk[4 * b + 0] = a;
      blk[4 * b + 1] = bb;
      blk[4 * b + 2] = id;
      zf[k] = zconj(c0[R]);
      if (pair) zf[k + 1] = zconj(c1[R]);
    }
    // B^-1 = (1/det) [[bb, -conj(c)], [-c, a]]; row projection w_i = (G_ik, G_i,k+1) B^-1, then
    // G_ij -= w_i0 conj(G_jk) + w_i1 conj(G_j,k+1): 16 fp64 ops per entry
    const double2 x00 = make_double2(bb * id, 0.0), x11 = make_double2(a * id, 0.0);
    const double2 x01 = make_double2(-c.x * id, c.y * id);   // -conj(c)/det
    const double2 x10 = make_double2(-c.x * id, -c.y * id);  // -c/det
#pragma unroll
    for (int m = 0; m < EPT; ++m) {
      const int i = ri[m], j = rj[m];
      if ((j >= k + 2 && j < R && i >= j) || (j == R && i >= k + 2)) {  // trailing lower entry or rhs row
        const double2 u0 = c0[i], v0 = c0[j];
        double2 upd;
        if (pair) {
          const double2 u1 = c1[i], v1 = c1[j];
          const double2 w0 = zfma(u1, x10, zmul(u0, x00));
          const double2 w1 = zfma(u1, x11, zmul(u0, x01));
          upd = zfma(w1, zconj(v1), zmul(w0, zconj(v0)));
          g[m] = zsub(g[m], upd);
        } else {
          upd = zmul(u0, zconj(v0));
          g[m].x -= upd.x * id;
          g[m].y -= upd.y * id;
        }
        if (j == k + 2 || j == k + 3) n0[(j - k - 2) * W + i] = g[m];  // next pivot columns
        if (j == R && (i == k + 2 || i == k + 3)) n0[(i - k - 2) * W + R] = zconj(g[m]);
      }
      // entries of the two pivot columns are final now: keep them for the back substitution
      if (j == k || (pair && j == k + 1)) Gio[i * (i + 1) / 2 + j] = g[m];
    }
    (void)n1;
    __syncthreads();
  }
  // back substitution (warp 0): blocks from last to first
  //   [gk, gk1] = Bk^-1 ([zk, zk1] - [acc_k, acc_k1]),  acc_i = sum_{j > block} conj(G_ji) gamma_j
  if (tid < 32) {
    const int lane = tid;
    double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);  // acc for rows lane, lane+32
    for (int b = nb - 1; b >= 0; --b) {
      const int k = 2 * b;
      const bool pair = k + 1 < R;
      const double2 acck = shfl_d2_sel(a0, a1, k);
      const double2 acck1 = pair ? shfl_d2_sel(a0, a1, k + 1) : make_double2(0.0, 0.0);
      const double a = blk[4 * b + 0], bb = blk[4 * b + 1], id = blk[4 * b + 2];
      const double2 r0 = zsub(zf[k], acck);
      double2 gk, gk1 = make_double2(0.0, 0.0);
      if (pair) {
        const double2 c = Gio[(k + 1) * (k + 2) / 2 + k];  // G_k+1,k
        // B^-1 r = (1/det) [bb r0 - conj(c) r1 ; -c r0 + a r1]
        const double2 r1 = zsub(zf[k + 1], acck1);
        gk = zscale(zsub(zscale(r0, bb), zmul(zconj(c), r1)), id);
        gk1 = zscale(zsub(zscale(r1, a), zmul(c, r0)), id);
      } else {
        gk = zscale(r0, id);
      }
      if (lane == 0) {
        gam[k] = gk;
        if (pair) gam[k + 1] = gk1;
      }
      // rows i < k: acc_i += conj(G_k,i) gk + conj(G_k+1,i) gk1 (rows k, k+1 of the factor, contiguous)
      const double2* rk = Gio + k * (k + 1) / 2;
      const double2* rk1 = Gio + (k + 1) * (k + 2) / 2;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = lane + 32 * h;
        if (i < k) {
          double2 acc = h ? a1 : a0;
          acc = zfma_cj(rk[i], gk, acc);
          if (pair) acc = zfma_cj(rk1[i], gk1, acc);
          if (h) a1 = acc; else a0 = acc;
        }
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- Gauss-Jordan ridge solve
// Solves G gamma = h for Hermitian positive (semi)definite G (packed lower
// triangle) by Gauss-Jordan elimination of the full augmented R x (R+1)
// system without pivoting: R fully parallel steps, one barrier each, and no
// back substitution (the latency of a serial triangular solve dominates a
// blocked LDL^H at R <= 32). Thread t owns entries e = t + m*NT, column-major
// (column j = e / R, row i = e % R; column R is h), in registers; step k only
// touches columns j > k, so retired columns idle whole warps. The pivot
// column and row of the next step are published to a double-buffered scratch
// right after they are updated. Non-positive pivots drop their component
// (gamma_k = 0), mirroring the s > 0 filter of the reference SVD ridge
// (tracker.py:154-155).
//   scratch: colb 2*2*(R+1) double2. Ends with __syncthreads.
TT_DEV uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
TT_DEV double2 lds_d2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
TT_DEV double lds_d(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
TT_DEV void sts_d2(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
// clock stamp stored by one thread, without a branch
TT_DEV void stamp_if(bool p, long long* dst) {
  const long long v = clock64();
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.s64 [%0], %1;\n\t}" ::"l"(dst), "l"(v),
               "r"((unsigned)p)
               : "memory");
}
// clock stamp taken once a shared load issued after the preceding barrier has returned
TT_DEV void stamp_after(bool p, long long* dst, const int* dep) {
  const int v = *(const volatile int*)dep;
  if (v == 0x7fffffff) asm volatile("trap;");
  stamp_if(p, dst);
}
// predicated store without a branch
TT_DEV void sts_d2_if(bool p, uint32_t a, double2 v) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q st.shared.v2.f64 [%0], {%1, %2};\n\t}" ::"r"(a),
      "d"(v.x), "d"(v.y), "r"((unsigned)p)
      : "memory");
}
// opaque copy: keeps a value in a register (stops rematerialisation of the shared window base)
TT_DEV uint32_t pin_u32(uint32_t x) {
  uint32_t y;
  asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// registers per thread needed by block_gj_solve: ceil((R + 1) / (NT / R))
__host__ __device__ inline int gj_ept(int R, int NT) {
  const int ng = NT / R;
  return ng > 0 ? (R + ng) / ng : 1 << 20;
}

template <int EPT>
TT_DEV void block_gj_solve(const double2* G, const double2* hin, double2* gam, double2* colb, int R) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int W = R + 1;
  // thread = (row i, column group): columns j = grp + m * ng. One pivot-column load per
  // step serves all of a thread's entries, and the pivot-row loads are near-broadcasts.
  const int ng = NT / R, grp = tid / R, i = tid - grp * R;
  const bool live = grp < ng;
  int rj[EPT];  // 0 for unused slots: column 0 is never updated
  double2 g[EPT];
  double idk = 0.0;
#pragma unroll
  for (int m = 0; m < EPT; ++m) {
    const int j = grp + m * ng;
    rj[m] = 0;
    g[m] = make_double2(0.0, 0.0);
    if (live && j < W) {
      rj[m] = j;
      if (j == R) g[m] = hin[i];
      else if (i >= j) g[m] = G[i * (i + 1) / 2 + j];
      else g[m] = zconj(G[j * (j + 1) / 2 + i]);
      if (j == 0) colb[i] = g[m];               // pivot column 0
      else if (i == 0) colb[W + j] = g[m];      // pivot row 0
    }
  }
  __syncthreads();
  // byte addresses into the double-buffered pivot column/row scratch (buffer b at b * 32 W)
  const uint32_t base = smem_addr(colb);
  const uint32_t oc = base + 16u * (live ? i : 0);
  uint32_t orr[EPT];
#pragma unroll
  for (int m = 0; m < EPT; ++m) orr[m] = base + 16u * (W + rj[m]);
  const uint32_t bstride = 32u * W;
  for (int k = 0; k < R; ++k) {
    const uint32_t cur = (k & 1) ? bstride : 0u, nxt = bstride - cur;
    // operands first: the products a_ik a_kj do not depend on the pivot inverse
    const double2 aik = lds_d2(oc + cur);
    double2 u[EPT];
#pragma unroll
    for (int m = 0; m < EPT; ++m) u[m] = zmul(aik, lds_d2(orr[m] + cur));
    const double d = lds_d(base + cur + 16u * k);
    const double id = d > 0.0 ? fast_rcp(d) : 0.0;
    const double sc = i != k ? id : 0.0;
#pragma unroll
    for (int m = 0; m < EPT; ++m) {
      const int j = rj[m];
      const bool act = j > k;
      const double s = act ? sc : 0.0;
      g[m].x = fma(-u[m].x, s, g[m].x);
      g[m].y = fma(-u[m].y, s, g[m].y);
      const bool pc_next = act && j == k + 1;  // next pivot column (row k included: final)
      sts_d2_if(pc_next || (act && i == k + 1), (pc_next ? oc : orr[m]) + nxt, g[m]);
    }
    if (i == k) idk = id;
    __syncthreads();
#ifdef TT_GJ_STAMPS
    if (tid == 0) tt_gj_stamps[k] = clock64();
#endif
  }
#pragma unroll
  for (int m = 0; m < EPT; ++m)
    if (live && rj[m] == R) gam[i] = zscale(g[m], idk);
  __syncthreads();
}

// ---------------------------------------------------------------- register-tiled complex GEMM
// C(m, n) = sum_{k<K} opA(A[m*a_m + k*a_k]) * opB(B[k*b_k + n*b_n]) over shared
// memory operands (complex fp32). Work item = (TM x TN output tile, k part);
// with KS > 1 the parts are summed in fixed order through `red`
// (KS * M * N float2) after a barrier, so results are deterministic. Every
// (m, n) is delivered once to out(m, n, value). Callers synchronise after.
template <int TM, int TN, bool CA, bool CB, typename Out>
TT_DEV void cgemm_tile(int M, int N, int K, const float2* A, int a_m, int a_k, const float2* B, int b_k, int b_n,
                       int KS, float2* red, Out out) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int tn = (N + TN - 1) / TN, tiles = ((M + TM - 1) / TM) * tn;
  const int items = tiles * KS;
  for (int it = tid; it < items; it += NT) {
    const int ks = idiv(it, tiles), tile = it - ks * tiles;
    const int mt = idiv(tile, tn);
    const int m0 = mt * TM, n0 = (tile - mt * tn) * TN;
    const int k0 = idiv(K * ks, KS), k1 = idiv(K * (ks + 1), KS);
    float2 acc[TM][TN];
#pragma unroll
    for (int u = 0; u < TM; ++u)
#pragma unroll
      for (int v = 0; v < TN; ++v) acc[u][v] = make_float2(0.f, 0.f);
    const float2* Ap[TM];
    const float2* Bp[TN];
#pragma unroll
    for (int u = 0; u < TM; ++u) Ap[u] = A + (size_t)min(m0 + u, M - 1) * a_m;
#pragma unroll
    for (int v = 0; v < TN; ++v) Bp[v] = B + (size_t)min(n0 + v, N - 1) * b_n;
#pragma unroll 2
    for (int k = k0; k < k1; ++k) {
      float2 a[TM], b[TN];
#pragma unroll
      for (int u = 0; u < TM; ++u) {
        a[u] = Ap[u][(size_t)k * a_k];
        if (CA) a[u].y = -a[u].y;
      }
#pragma unroll
      for (int v = 0; v < TN; ++v) {
        b[v] = Bp[v][(size_t)k * b_k];
        if (CB) b[v].y = -b[v].y;
      }
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; ++v) acc[u][v] = cfma(a[u], b[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < TM; ++u)
#pragma unroll
      for (int v = 0; v < TN; ++v) {
        const int m = m0 + u, n = n0 + v;
        if (m < M && n < N) {
          if (KS == 1) out(m, n, acc[u][v]);
          else red[((size_t)ks * M + m) * N + n] = acc[u][v];
        }
      }
  }
  if (KS > 1) {
    __syncthreads();
    for (int o = tid; o < M * N; o += NT) {
      float2 s = red[o];
#pragma unroll
      for (int ks = 1; ks < 8; ++ks)  // KS <= 8 (gemm_split): all partial loads in flight, fixed order
        if (ks < KS) s = cadd(s, red[(size_t)ks * M * N + o]);
      const int om = idiv(o, N);
      out(om, o - om * N, s);
    }
  }
}

// Mixed-precision variant for the data GEMMs of the rows kernel (W = Y^T conj(Ah_S), Z = Y conj(Bh)):
// fp32 complex operands in shared memory, converted on load, products and accumulation in fp64, so
// every product of two fp32 values is exact and only the fp64 sums round. The updates subtract the
// model part from W and Z (Q = W - Bh diag(g) GA^T, P = Z - Ah_S diag(g) GB^T); with a good fit the
// difference is ~1e-2 of W, Z, so fp32 sums would lose two digits there. Same item /
// K-split structure as cgemm_tile; `red` holds KS * M * N double2.
template <int TM, int TN, bool CA, bool CB, typename Out>
TT_DEV void zgemm_tile(int M, int N, int K, const float2* A, int a_m, int a_k, const float2* B, int b_k, int b_n,
                       int KS, double2* red, Out out) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int tn = (N + TN - 1) / TN, tiles = ((M + TM - 1) / TM) * tn;
  const int items = tiles * KS;
  for (int it = tid; it < items; it += NT) {
    const int ks = idiv(it, tiles), tile = it - ks * tiles;
    const int mt = idiv(tile, tn);
    const int m0 = mt * TM, n0 = (tile - mt * tn) * TN;
    const int k0 = idiv(K * ks, KS), k1 = idiv(K * (ks + 1), KS);
    double2 acc[TM][TN];
#pragma unroll
    for (int u = 0; u < TM; ++u)
#pragma unroll
      for (int v = 0; v < TN; ++v) acc[u][v] = make_double2(0.0, 0.0);
    const float2* Ap[TM];
    const float2* Bp[TN];
#pragma unroll
    for (int u = 0; u < TM; ++u) Ap[u] = A + (size_t)min(m0 + u, M - 1) * a_m;
#pragma unroll
    for (int v = 0; v < TN; ++v) Bp[v] = B + (size_t)min(n0 + v, N - 1) * b_n;
#pragma unroll 2
    for (int k = k0; k < k1; ++k) {
      double2 a[TM], b[TN];
#pragma unroll
      for (int u = 0; u < TM; ++u) {
        a[u] = to_d2(Ap[u][(size_t)k * a_k]);
        if (CA) a[u].y = -a[u].y;
      }
#pragma unroll
      for (int v = 0; v < TN; ++v) {
        b[v] = to_d2(Bp[v][(size_t)k * b_k]);
        if (CB) b[v].y = -b[v].y;
      }
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; ++v) acc[u][v] = zfma(a[u], b[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < TM; ++u)
#pragma unroll
      for (int v = 0; v < TN; ++v) {
        const int m = m0 + u, n = n0 + v;
        if (m < M && n < N) {
          if (KS == 1) out(m, n, acc[u][v]);
          else red[((size_t)ks * M + m) * N + n] = acc[u][v];
        }
      }
  }
  if (KS > 1) {
    __syncthreads();
    for (int o = tid; o < M * N; o += NT) {
      double2 s = red[o];
#pragma unroll
      for (int ks = 1; ks < 8; ++ks)  // KS <= 8 (gemm_split): all partial loads in flight, fixed order
        if (ks < KS) s = zadd(s, red[(size_t)ks * M * N + o]);
      const int om = idiv(o, N);
      out(om, o - om * N, s);
    }
  }
}

// zgemm_tile with the B operand already in fp64 (the rows kernel keeps fp64 copies of the resident Bh
// rows and of the frame's Ah_S rows, so only the Y operand is converted on load: TM conversions per k step
// for TM * TN complex products). PARTS: every K part is delivered as it is, out(m, n, ks, value), for a
// consumer that sums the parts later in a fixed order (the cluster's Z partials); otherwise the KS > 1
// parts are summed through `red` (KS * M * N double2) and delivered once, out(m, n, 0, value).
TT_DEV double2 ld_d2(const double2* p) { return *p; }
TT_DEV double2 ld_d2(const float2* p) { return to_d2(*p); }
template <int TM, int TN, bool CB, bool PARTS, typename BT, typename Out>
TT_DEV void zgemm_fd(int M, int N, int K, const float2* A, int a_m, int a_k, const BT* B, int b_k, int b_n,
                     int KS, double2* red, Out out) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int tn = (N + TN - 1) / TN, tiles = ((M + TM - 1) / TM) * tn;
  const int items = tiles * KS;
  for (int it = tid; it < items; it += NT) {
    const int ks = idiv(it, tiles), tile = it - ks * tiles;
    const int mt = idiv(tile, tn);
    const int m0 = mt * TM, n0 = (tile - mt * tn) * TN;
    const int k0 = idiv(K * ks, KS), k1 = idiv(K * (ks + 1), KS);
    double2 acc[TM][TN];
#pragma unroll
    for (int u = 0; u < TM; ++u)
#pragma unroll
      for (int v = 0; v < TN; ++v) acc[u][v] = make_double2(0.0, 0.0);
    const float2* Ap[TM];
    const BT* Bp[TN];
#pragma unroll
    for (int u = 0; u < TM; ++u) Ap[u] = A + (size_t)min(m0 + u, M - 1) * a_m + (size_t)k0 * a_k;
#pragma unroll
    for (int v = 0; v < TN; ++v) Bp[v] = B + (size_t)min(n0 + v, N - 1) * b_n + (size_t)k0 * b_k;
    // software pipeline: the shared-memory loads of step k+1 are in flight while step k's DFMAs issue
    // (two resident warps per scheduler cannot hide the load + F2F latency on their own)
    float2 an[TM];
    BT bn[TN];
    if (k0 < k1) {
#pragma unroll
      for (int u = 0; u < TM; ++u) an[u] = *Ap[u];
#pragma unroll
      for (int v = 0; v < TN; ++v) bn[v] = *Bp[v];
    }
    for (int k = k0; k < k1; ++k) {
      double2 a[TM], b[TN];
#pragma unroll
      for (int u = 0; u < TM; ++u) a[u] = to_d2(an[u]);
#pragma unroll
      for (int v = 0; v < TN; ++v) {
        b[v] = ld_d2(&bn[v]);
        if (CB) b[v].y = -b[v].y;
      }
      if (k + 1 < k1) {
#pragma unroll
        for (int u = 0; u < TM; ++u) {
          Ap[u] += a_k;
          an[u] = *Ap[u];
        }
#pragma unroll
        for (int v = 0; v < TN; ++v) {
          Bp[v] += b_k;
          bn[v] = *Bp[v];
        }
      }
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; ++v) acc[u][v] = zfma(a[u], b[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < TM; ++u)
#pragma unroll
      for (int v = 0; v < TN; ++v) {
        const int m = m0 + u, n = n0 + v;
        if (m < M && n < N) {
          if (PARTS || KS == 1) out(m, n, PARTS ? ks : 0, acc[u][v]);
          else red[((size_t)ks * M + m) * N + n] = acc[u][v];
        }
      }
  }
  if (!PARTS && KS > 1) {
    __syncthreads();
    for (int o = tid; o < M * N; o += NT) {
      double2 s = red[o];
#pragma unroll
      for (int ks = 1; ks < 8; ++ks)
        if (ks < KS) s = zadd(s, red[(size_t)ks * M * N + o]);
      const int om = idiv(o, N);
      out(om, o - om * N, 0, s);
    }
  }
}

// ---------------------------------------------------------------- fp64 tensor-core (DMMA) complex GEMM
// C(m, r) = sum_k A(m, k) conj(B(k, r)) with A fp32 complex (converted: products exact), B fp64 complex,
// on mma.sync m8n8k4 f64 (the B200's fp64 matrix path: the same peak as DFMA at a fraction of the issued
// instructions). The complex product is a real GEMM with interleaved (re, im) K and N: output column
// n = 2r + q; for k = 4t + kq two K slots per complex k, the A (re) slot with B coefficient (b.x, -b.y)
// and the A (im) slot with (b.y, b.x) — so a lane loads one float2 of A and one double2 of B per complex
// k and feeds two DMMAs. A lane of an 8x8 output block then holds C(m0 + lane/4, r0 + lane%4) as one
// complex value. Work item = (group of G 8-row M blocks, one 4-wide r block, K part); warps take items
// round-robin. PARTS: each K part delivered as it is, out(m, r, ks, value); else KS must be 1.
TT_DEV void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
template <int G, typename AT, typename Out>
TT_DEV void zgemm_dmma_v1(int M, int R, int K, const AT* A, int a_m, int a_k, const double2* B, int b_k, int KS,
                          Out out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int row = lane >> 2, kq = lane & 3;
  const int MB = (M + 7) >> 3, NB = (R + 3) >> 2, MG = (MB + G - 1) / G;
  const int kpairs = (K + 3) >> 2;
  const int items = MG * NB * KS;
  for (int it = warp; it < items; it += nw) {
    const int ks = idiv(it, MG * NB), rest = it - ks * MG * NB;
    const int mg = idiv(rest, NB), nb = rest - mg * NB;
    const int gcount = min(G, MB - mg * G);  // warp-uniform: empty 8-row blocks issue no DMMA
    const int t0 = idiv(kpairs * ks, KS), t1 = idiv(kpairs * (ks + 1), KS);
    const int rb = nb * 4 + (row >> 1), q = row & 1;  // B fragment column n = nb * 8 + row = 2 rb + q
    const bool rok = rb < R;
    const AT* ap[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int m = ((mg * G + g) << 3) + row;
      ap[g] = A + (size_t)min(m, M - 1) * a_m;
    }
    double acc[G][2];
#pragma unroll
    for (int g = 0; g < G; ++g) acc[g][0] = acc[g][1] = 0.0;
    const double2* bp = B + min(rb, R - 1);
    for (int t = t0; t < t1; ++t) {
      const int k = 4 * t + kq;
      const bool kok = k < K;
      const int kc = min(k, K - 1);  // loads always in range (no branches around them), invalid ones zeroed
      const double2 braw = bp[(size_t)kc * b_k];
      const bool bv = kok && rok;
      const double2 b = make_double2(bv ? braw.x : 0.0, bv ? braw.y : 0.0);
      double ar[G], ai[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int m = ((mg * G + g) << 3) + row;
        const AT a = ap[g][(size_t)kc * a_k];
        const bool av = kok && m < M;
        ar[g] = av ? (double)a.x : 0.0;
        ai[g] = av ? (double)a.y : 0.0;
      }
      const double b0 = q == 0 ? b.x : -b.y, b1 = q == 0 ? b.y : b.x;
      // the re slots of all blocks before the im slots: consecutive DMMAs never chain on one accumulator
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (g < gcount) dmma_m8n8k4(acc[g][0], acc[g][1], ar[g], b0);
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (g < gcount) dmma_m8n8k4(acc[g][0], acc[g][1], ai[g], b1);
    }
    const int r = nb * 4 + kq;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int m = ((mg * G + g) << 3) + row;
      if (g < gcount && m < M && r < R) out(m, r, ks, make_double2(acc[g][0], acc[g][1]));
    }
  }
}

// zgemm_dmma (the round-2 form; zgemm_dmma_v1 above is the round-1 loop, kept for
// profiles/tools/ubench_dmma_shapes.cu): fewer issue slots per DMMA (the loop is issue-bound: a DMMA every ~16 SMSP cycles leaves
// ~8 slots per DMMA per warp at two warps per SMSP): every one of the G blocks of an item issues its DMMAs
// unpredicated (blocks past the item's last one, rows past M and columns past R compute on clamped, finite
// operands into accumulators that are never stored: a row of A only reaches its own output row, a column
// of B its own output column), the operand pointers advance by increments, and only the K tail step (K not a
// multiple of 4) selects zeros. Same products and K order per output as zgemm_dmma.
template <int G, typename AT, typename Out>
TT_DEV void zgemm_dmma(int M, int R, int K, const AT* A, int a_m, int a_k, const double2* B, int b_k, int KS,
                       Out out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int row = lane >> 2, kq = lane & 3;
  const int MB = (M + 7) >> 3, NB = (R + 3) >> 2, MG = (MB + G - 1) / G;
  const int kfull = K >> 2;                 // steps with all 4 k valid
  const int kpairs = (K + 3) >> 2;
  const int items = MG * NB * KS;
  for (int it = warp; it < items; it += nw) {
    const int ks = idiv(it, MG * NB), rest = it - ks * MG * NB;
    const int mg = idiv(rest, NB), nb = rest - mg * NB;
    const int gcount = min(G, MB - mg * G);
    const int t0 = idiv(kpairs * ks, KS), t1 = idiv(kpairs * (ks + 1), KS);
    const int rb = nb * 4 + (row >> 1), q = row & 1;
    const AT* ap[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int m = ((mg * G + g) << 3) + row;
      ap[g] = A + (size_t)min(m, M - 1) * a_m + (size_t)(4 * t0 + kq) * a_k;
    }
    const double2* bp = B + min(rb, R - 1) + (size_t)(4 * t0 + kq) * b_k;
    const size_t astep = (size_t)4 * a_k, bstep = (size_t)4 * b_k;
    double acc[G][2];
#pragma unroll
    for (int g = 0; g < G; ++g) acc[g][0] = acc[g][1] = 0.0;
    const int tf = min(t1, kfull);
    for (int t = t0; t < tf; ++t) {
      const double2 b = *bp;
      bp += bstep;
      const double b0 = q == 0 ? b.x : -b.y, b1 = q == 0 ? b.y : b.x;
      double ar[G], ai[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const AT a = *ap[g];
        ap[g] += astep;
        ar[g] = (double)a.x;
        ai[g] = (double)a.y;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) dmma_m8n8k4(acc[g][0], acc[g][1], ar[g], b0);
#pragma unroll
      for (int g = 0; g < G; ++g) dmma_m8n8k4(acc[g][0], acc[g][1], ai[g], b1);
    }
    if (tf < t1) {  // the K tail: k >= K contributes zero
      const bool kok = 4 * tf + kq < K;
      const double2 b = kok ? *bp : make_double2(0.0, 0.0);
      const double b0 = q == 0 ? b.x : -b.y, b1 = q == 0 ? b.y : b.x;
      double ar[G], ai[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const AT a = kok ? *ap[g] : AT{0, 0};
        ar[g] = (double)a.x;
        ai[g] = (double)a.y;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) dmma_m8n8k4(acc[g][0], acc[g][1], ar[g], b0);
#pragma unroll
      for (int g = 0; g < G; ++g) dmma_m8n8k4(acc[g][0], acc[g][1], ai[g], b1);
    }
    const int r = nb * 4 + kq;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int m = ((mg * G + g) << 3) + row;
      if (g < gcount && m < M && r < R) out(m, r, ks, make_double2(acc[g][0], acc[g][1]));
    }
  }
}

// Two independent GEMMs of the same shape class in one pass (cgemm_tile's items of both problems
// spread over the block, one barrier, one fixed-order reduction pass for both): problem p is
// C_p(m, n) = sum_k A_p[m*a_m + k] * conj(B_p[k*b_k + n]) (CB) with common N, K, strides and split KS;
// red holds KS * (M0 + M1) * N partials.
template <int TM, int TN, bool CA, bool CB, typename Out>
TT_DEV void cgemm_tile_pair(int M0, int M1, int N, int K, const float2* A0, const float2* A1, int a_m, int a_k,
                            const float2* B0, const float2* B1, int b_k, int b_n, int KS, float2* red,
                            const Out& out0, const Out& out1) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int tn = (N + TN - 1) / TN;
  const int tiles0 = ((M0 + TM - 1) / TM) * tn, tiles1 = ((M1 + TM - 1) / TM) * tn;
  const int items0 = tiles0 * KS, items = items0 + tiles1 * KS;
  for (int it = tid; it < items; it += NT) {
    const bool p1 = it >= items0;
    const int jt = p1 ? it - items0 : it, tiles = p1 ? tiles1 : tiles0, M = p1 ? M1 : M0;
    const float2* A = p1 ? A1 : A0;
    const float2* B = p1 ? B1 : B0;
    float2* rp = p1 ? red + (size_t)KS * M0 * N : red;
    const int ks = idiv(jt, tiles), tile = jt - ks * tiles;
    const int mt = idiv(tile, tn);
    const int m0 = mt * TM, n0 = (tile - mt * tn) * TN;
    const int k0 = idiv(K * ks, KS), k1 = idiv(K * (ks + 1), KS);
    float2 acc[TM][TN];
#pragma unroll
    for (int u = 0; u < TM; ++u)
#pragma unroll
      for (int v = 0; v < TN; ++v) acc[u][v] = make_float2(0.f, 0.f);
    const float2* Ap[TM];
    const float2* Bp[TN];
#pragma unroll
    for (int u = 0; u < TM; ++u) Ap[u] = A + (size_t)min(m0 + u, M - 1) * a_m;
#pragma unroll
    for (int v = 0; v < TN; ++v) Bp[v] = B + (size_t)min(n0 + v, N - 1) * b_n;
#pragma unroll 2
    for (int k = k0; k < k1; ++k) {
      float2 a[TM], b[TN];
#pragma unroll
      for (int u = 0; u < TM; ++u) {
        a[u] = Ap[u][(size_t)k * a_k];
        if (CA) a[u].y = -a[u].y;
      }
#pragma unroll
      for (int v = 0; v < TN; ++v) {
        b[v] = Bp[v][(size_t)k * b_k];
        if (CB) b[v].y = -b[v].y;
      }
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; ++v) acc[u][v] = cfma(a[u], b[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < TM; ++u)
#pragma unroll
      for (int v = 0; v < TN; ++v) {
        const int m = m0 + u, n = n0 + v;
        if (m < M && n < N) {
          if (KS == 1) (p1 ? out1 : out0)(m, n, acc[u][v]);
          else rp[((size_t)ks * M + m) * N + n] = acc[u][v];
        }
      }
  }
  if (KS > 1) {
    __syncthreads();
    const int n0s = M0 * N;
    for (int o = tid; o < (M0 + M1) * N; o += NT) {
      const bool p1 = o >= n0s;
      const int oo = p1 ? o - n0s : o, MN = p1 ? M1 * N : n0s;
      const float2* rp = p1 ? red + (size_t)KS * n0s : red;
      float2 s = rp[oo];
#pragma unroll
      for (int ks = 1; ks < 8; ++ks)
        if (ks < KS) s = cadd(s, rp[(size_t)ks * MN + oo]);
      const int om = idiv(oo, N);
      (p1 ? out1 : out0)(om, oo - om * N, s);
    }
  }
}

// Register-tiled complex GEMM, K split across adjacent lanes: C(m, n) = sum_k opA(A[m*a_m + k*a_k]) *
// opB(B[k*b_k + n*b_n]) over shared-memory operands. Work item = (TM x TN tile, k part); the KS parts of
// a tile sit on adjacent lanes and are summed by a fixed-order shuffle butterfly (deterministic, no
// reduction buffer, no barrier). Every (m, n) is delivered once to out(m, n, value) by the part-0 lane.
// KS must be a power of two <= 32. Callers synchronise after.
template <int TM, int TN, int KS, bool CA, bool CB, typename Out>
TT_DEV void cgemm_v2(int M, int N, int K, const float2* A, int a_m, int a_k, const float2* B, int b_k, int b_n,
                     Out out) {
  static_assert(KS >= 1 && KS <= 32 && (KS & (KS - 1)) == 0, "KS: power of two <= 32");
  const int tid = threadIdx.x, NT = blockDim.x;
  const int tn = (N + TN - 1) / TN, tiles = ((M + TM - 1) / TM) * tn;
  const int items = tiles * KS;
  const int kc = (K + KS - 1) / KS;
  for (int base = 0; base < items; base += NT) {  // uniform trip count: the butterfly stays convergent
    const int it = base + tid;
    const bool live = it < items;
    const int tile = it / KS, part = it & (KS - 1);
    const int mt = tile / tn, nt = tile - mt * tn;
    const int m0 = mt * TM, n0 = nt * TN;
    const int k0 = part * kc, k1 = min(K, k0 + kc);
    float2 acc[TM][TN];
#pragma unroll
    for (int u = 0; u < TM; ++u)
#pragma unroll
      for (int v = 0; v < TN; ++v) acc[u][v] = make_float2(0.f, 0.f);
    if (live) {
      int ao[TM], bo[TN];
#pragma unroll
      for (int u = 0; u < TM; ++u) ao[u] = min(m0 + u, M - 1) * a_m + k0 * a_k;
#pragma unroll
      for (int v = 0; v < TN; ++v) bo[v] = min(n0 + v, N - 1) * b_n + k0 * b_k;
#pragma unroll 4
      for (int k = k0; k < k1; ++k) {
        float2 a[TM], b[TN];
#pragma unroll
        for (int u = 0; u < TM; ++u) {
          a[u] = A[ao[u]];
          ao[u] += a_k;
          if (CA) a[u].y = -a[u].y;
        }
#pragma unroll
        for (int v = 0; v < TN; ++v) {
          b[v] = B[bo[v]];
          bo[v] += b_k;
          if (CB) b[v].y = -b[v].y;
        }
#pragma unroll
        for (int u = 0; u < TM; ++u)
#pragma unroll
          for (int v = 0; v < TN; ++v) acc[u][v] = cfma(a[u], b[v], acc[u][v]);
      }
    }
#pragma unroll
    for (int o = 1; o < KS; o <<= 1)
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; ++v) {
          acc[u][v].x += __shfl_xor_sync(0xffffffffu, acc[u][v].x, o);
          acc[u][v].y += __shfl_xor_sync(0xffffffffu, acc[u][v].y, o);
        }
    if (live && part == 0) {
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; ++v) {
          const int m = m0 + u, n = n0 + v;
          if (m < M && n < N) out(m, n, acc[u][v]);
        }
    }
  }
}

// K-split factor that fills the block without exceeding the reduction buffer
TT_DEV int gemm_split(int M, int N, int K, int TM, int TN, int red_cap) {
  const int tiles = ((M + TM - 1) / TM) * ((N + TN - 1) / TN);
  int ks = idiv((int)blockDim.x, tiles > 0 ? tiles : 1);
  if (ks > K / 4) ks = K / 4;
  if (ks > 8) ks = 8;
  while (ks > 1 && ks * M * N > red_cap) --ks;
  return ks < 1 ? 1 : ks;
}

// ---------------------------------------------------------------- warp-level draw (fused kernel)
// Same semantics as draw_with_replacement_block<false> but executed by one
// warp only (no CTA barriers): chunked warp scan, parallel Philox draws with
// the 1e-12 ambiguity check and exact sequential fallback, flag compaction.
// `p` may be unnormalised (the CDF is normalised by its last element).
TT_DEV void warp_draw_with_replacement(const double* p, double* cdf, int* flags, int* rows, int* S_out, int n,
                                       int ndraw, const int* forced, int nforced, uint64_t k0, uint64_t k1,
                                       uint64_t pos) {
  const int lane = threadIdx.x & 31;
  const int chunk = (n + 31) / 32;
  const int c0 = min(n, lane * chunk), c1 = min(n, c0 + chunk);
  for (int exact = 0; exact < 2; ++exact) {
    if (!exact) {
      double loc = 0.0;
      for (int i = c0; i < c1; ++i) loc += p[i];
      double x = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const double total = __shfl_sync(0xffffffffu, x, 31);
      const double il = fast_rcp(total);
      double run = x - loc;
      for (int i = c0; i < c1; ++i) {
        run += p[i];
        cdf[i] = run * il;
      }
    } else {
      if (lane == 0) {
        double cacc = 0.0;
        for (int i = 0; i < n; ++i) {
          cacc += p[i];
          cdf[i] = cacc;
        }
        const double last = cdf[n - 1];
        for (int i = 0; i < n; ++i) cdf[i] = cdf[i] / last;
      }
    }
    for (int i = c0; i < c1; ++i) flags[i] = 0;
    __syncwarp();
    int amb = 0;
    for (int m = lane; m < ndraw; m += 32) {
      const double u = philox_uniform(k0, k1, pos + (uint64_t)m);
      const int idx = upper_bound_d(cdf, n, u);
      if (!exact) {
        const double lo = idx > 0 ? cdf[idx - 1] : -1.0;
        const double hi = idx < n ? cdf[idx] : 2.0;
        if (u - lo <= 1e-12 || hi - u <= 1e-12) amb = 1;
      }
      flags[idx < n ? idx : n - 1] = 1;
    }
    __syncwarp();
    if (exact || !__any_sync(0xffffffffu, amb)) break;
  }
  for (int m = lane; m < nforced; m += 32) {
    const int f = forced[m];
    if (f >= 0 && f < n) flags[f] = 1;
  }
  __syncwarp();
  int cnt = 0;
  for (int i = c0; i < c1; ++i) cnt += flags[i];
  int x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  int o = x - cnt;
  for (int i = c0; i < c1; ++i)
    if (flags[i]) rows[o++] = i;
  if (lane == 31) *S_out = x;
  __syncwarp();
}
