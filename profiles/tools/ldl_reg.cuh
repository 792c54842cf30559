__device__ long long g_t_fwd;
// Register-resident right-looking LDL^H over the augmented system [G | h].
// Thread t owns entries e = t + m*NT (m < EPT) of the packed lower triangle
// (entries 0..Rp-1, row-major) followed by the rhs "column" (entries Rp + i,
// i < R). Column k is final after step k-1; its owners publish it to a
// double-buffered column buffer (colb[par][0..R], slot R holds conj(h_k)),
// and the owner of (k+1, k+1) publishes the reciprocal pivot. One barrier per
// column. The final L (scaled by D) goes to Gout (packed) for the warp
// back-substitution; z (eliminated rhs) to hv.
template <int EPT>
TT_DEV void ldl_reg_solve(const double2* Gin, const double2* hin, double2* Gout, double2* hv, double2* colb,
                          double* invb, double2* gam, int R) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int Rp = R * (R + 1) / 2, E = Rp + R;
  int ri[EPT], rj[EPT];
  double2 g[EPT];
#pragma unroll
  for (int m = 0; m < EPT; ++m) {
    const int e = tid + m * NT;
    ri[m] = -1;
    rj[m] = -1;
    g[m] = make_double2(0.0, 0.0);
    if (e < Rp) {
      int r, q;
      tri_decode(e, r, q);
      ri[m] = r;
      rj[m] = q;
      g[m] = Gin[e];
    } else if (e < E) {
      ri[m] = e - Rp;
      rj[m] = R;  // rhs column
      g[m] = hin[e - Rp];
    }
  }
  // publish column 0 and pivot 0
  double2* c0 = colb;              // colb[0][0..R]
#pragma unroll
  for (int m = 0; m < EPT; ++m) {
    if (rj[m] == 0) c0[ri[m]] = g[m];
    if (rj[m] == R && ri[m] == 0) c0[R] = zconj(g[m]);

  }
  __syncthreads();
  for (int k = 0; k < R; ++k) {
    const double2* ck = colb + (k & 1) * (R + 1);
    double2* cn = colb + ((k + 1) & 1) * (R + 1);
    const double dk = ck[k].x;
    const double ik = dk > 0.0 ? fast_rcp(dk) : 0.0;
    if (tid == 0) invb[2 + k] = ik;
#pragma unroll
    for (int m = 0; m < EPT; ++m) {
      const int i = ri[m], j = rj[m];
      if (j > k && i > k) {  // (i, j) with j > k; rhs rows i > k
        const double2 lik = ck[i];
        const double2 ljk = ck[j];  // slot R = conj(h_k)
        g[m].x -= (lik.x * ljk.x + lik.y * ljk.y) * ik;
        g[m].y -= (lik.y * ljk.x - lik.x * ljk.y) * ik;
        if (j == k + 1) cn[i] = g[m];                               // column k+1 now final
        if (j == R && i == k + 1) cn[R] = zconj(g[m]);               // h_{k+1} final

      }
    }
    __syncthreads();
  }
  if (tid == 0) g_t_fwd = clock64();
#pragma unroll
  for (int m = 0; m < EPT; ++m) {
    const int e = tid + m * NT;
    if (e < Rp) Gout[e] = g[m];
    else if (e < E) hv[e - Rp] = g[m];
  }
  __syncthreads();
  // back substitution (warp 0): gamma_k = (z_k - sum_{j>k} conj(G_jk) gamma_j) / d_k
  if (tid < 32) {
    const int lane = tid;
    double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
    for (int k = R - 1; k >= 0; --k) {
      const int own = k & 31;
      const double2* gk = Gout + k * (k + 1) / 2;   // row k, contiguous
      const double2 p0 = lane < k ? gk[lane] : make_double2(0.0, 0.0);
      const double2 p1 = lane + 32 < k ? gk[lane + 32] : make_double2(0.0, 0.0);
      double gx = 0.0, gy = 0.0;
      const double iv = invb[2 + k];
      if (lane == own) {
        const double2 a = k < 32 ? a0 : a1;
        gx = (hv[k].x - a.x) * iv;
        gy = (hv[k].y - a.y) * iv;
        gam[k] = make_double2(gx, gy);
      }
      gx = __shfl_sync(0xffffffffu, gx, own);
      gy = __shfl_sync(0xffffffffu, gy, own);
      a0.x += p0.x * gx + p0.y * gy;
      a0.y += p0.x * gy - p0.y * gx;
      a1.x += p1.x * gx + p1.y * gy;
      a1.y += p1.x * gy - p1.y * gx;
    }
  }
  __syncthreads();
}
