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
TT_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// packed lower-triangular index helpers (r >= q)
TT_DEV void tri_decode(int e, int& r, int& q) {
  int rr = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
  while (rr * (rr + 1) / 2 > e) --rr;
  while ((rr + 1) * (rr + 2) / 2 <= e) ++rr;
  r = rr;
  q = e - rr * (rr + 1) / 2;
}
TT_DEV int tri_idx(int r, int q) { return r * (r + 1) / 2 + q; }

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
TT_DEV void draw_with_replacement_block(const double* p, double* cdf, int* flags, int* rows, int& S, int n,
                                        int ndraw, const int* forced, int nforced, uint64_t k0, uint64_t k1,
                                        uint64_t pos, double* red, int* sh_flag) {
  const int tid = threadIdx.x, NT = blockDim.x;
  for (int i = tid; i < n; i += NT) flags[i] = 0;
  if (tid == 0) *sh_flag = 0;
  for (int exact = 0; exact < 2; ++exact) {
    block_cumsum(p, cdf, n, exact != 0, red);
    const double last = cdf[n - 1];
    __syncthreads();
    for (int i = tid; i < n; i += NT) cdf[i] = cdf[i] / last;
    __syncthreads();
    for (int m = tid; m < ndraw; m += NT) {
      const double u = philox_uniform(k0, k1, pos + (uint64_t)m);
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
