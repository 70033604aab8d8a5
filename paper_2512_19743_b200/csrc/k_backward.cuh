// k_backward.cuh -- reverse pass over the same sparse graph.
//
// Discrete choices of the forward (support, argmin, second argmin) are frozen; the gap
// clamp zeroes the gradient through g.  With grad_loss gl = dL/dloss_b:
//
//   k_sinkhorn_bwd (full mode, CTA per pair, k_sinkhorn.cuh) -- reverse of the scaling-vector Sinkhorn:
//     abar = gl sum_j P0 b^L c,  bbar = gl sum_i a^L P0 c,  then for l = L..1
//       row step  a^l = a^{l-1} / (a^{l-1} R^l + eps):
//         Rbar^l = -abar (a^l)^2,  abar <- abar eps (a^l / a^{l-1})^2,  bbar += P0^T Rbar^l
//       column step b^l = b^{l-1} / (b^{l-1} Q^l + eps):
//         Qbar^l = -bbar (b^l)^2,  bbar <- bbar eps (b^l / b^{l-1})^2,  abar += P0 Qbar^l
//     storing Rbar^l [B][N][L], Qbar^l [B][M][L].
//   k_pbar_rowsoft (thread per row) -- P0bar_ij = gl a^L_i b^L_j c_ij
//       + sum_l (Rbar^l_i b^l_j + Qbar^l_j a^{l-1}_i); then the row softmax reverse with
//     Pbar_row = P0bar/2: S = sum P Pbar, zbar = P (Pbar - S), Tbar = -sum zbar (c-m),
//     mbar = T sum zbar, gbar = -Tbar T / g (0 if clamped); the argmin entry receives
//     mbar - gbar and the second-argmin entry gbar (g = c2 - m + delta, T = Lambda / g).
//   k_colsoft (thread per column) -- the same for the column softmax.
//   k_grad (thread per row) -- cbar_t = gl v_t + (-T zbar_row) + (-T' zbar_col) + T-path
//     terms, then Eq. (5): xbar_i = sum_t cbar_t (x_i - y_j) / (c_t + eps_dist).
//   Plan-detached mode: cbar_t = gl v_t only.
// All sums are per-line sequential in sorted order (deterministic), accumulated in fp64.
#pragma once
#include "common.cuh"

namespace apml {

// Thread per row: P0bar per entry, then the row-softmax reverse -> LineBack.
__global__ void k_pbar_rowsoft(int N, int M, int L, const unsigned* __restrict__ cursor,
                               uint32_t cap, const unsigned* __restrict__ row_ptr,
                               const uint32_t* __restrict__ csr_jf, const float* __restrict__ cs,
                               const float* __restrict__ prow, const float* __restrict__ a_hist,
                               const float* __restrict__ b_hist, const float* __restrict__ Rbar,
                               const float* __restrict__ Qbar, const float* __restrict__ grad_loss,
                               const LineB* __restrict__ rowB, float* __restrict__ pbar,
                               LineBack* __restrict__ rowback) {
  const int b = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N || pair_overflow(cursor, b, cap)) return;
  const size_t pb = (size_t)b * cap;
  const float gl = grad_loss[b];
  const float* ai = a_hist + ((size_t)b * N + i) * (L + 1);
  const float* ri = Rbar + ((size_t)b * N + i) * L;
  const uint32_t beg = row_ptr[(size_t)b * (N + 1) + i], end = row_ptr[(size_t)b * (N + 1) + i + 1];
  const LineB lb = rowB[(size_t)b * N + i];
  double S = 0.0;
  for (uint32_t p = beg; p < end; ++p) {
    const uint32_t jf = csr_jf[pb + p];
    const uint32_t j = jf & kIdxMask;
    const float* bj = b_hist + ((size_t)b * M + j) * (L + 1);
    const float* qj = Qbar + ((size_t)b * M + j) * L;
    double v = (double)gl * (double)ai[L] * (double)bj[L] * (double)cs[pb + p];
    for (int l = 1; l <= L; ++l) v += (double)ri[l - 1] * (double)bj[l] + (double)qj[l - 1] * (double)ai[l - 1];
    const float pv = (float)v;
    pbar[pb + p] = pv;
    if (jf & kFlagRow) S += (double)prow[pb + p] * 0.5 * (double)pv;
  }
  LineBack out = {(float)S, 0.f, 0.f, lb.T};
  if (!(lb.flags & kLineK1)) {
    double szb = 0.0, Tbar = 0.0;
    for (uint32_t p = beg; p < end; ++p) {
      const uint32_t jf = csr_jf[pb + p];
      if (!(jf & kFlagRow)) continue;
      const double zb = (double)prow[pb + p] * (0.5 * (double)pbar[pb + p] - S);
      szb += zb;
      Tbar -= zb * ((double)cs[pb + p] - (double)lb.m);
    }
    const double mbar = (double)lb.T * szb;
    const double gbar = (lb.flags & kLineClamped) ? 0.0 : -Tbar * (double)lb.T / (double)lb.g;
    out.ca = (float)(mbar - gbar);
    out.cb = (float)gbar;
  } else {
    out.T = 0.f;
  }
  rowback[(size_t)b * N + i] = out;
}

// Thread per column: column-softmax reverse -> LineBack.
__global__ void k_colsoft(int N, int M, const unsigned* __restrict__ cursor, uint32_t cap,
                          const unsigned* __restrict__ col_ptr, const uint32_t* __restrict__ csc_perm,
                          const uint32_t* __restrict__ csr_jf, const float* __restrict__ cs,
                          const float* __restrict__ pcol, const float* __restrict__ pbar,
                          const LineB* __restrict__ colB, LineBack* __restrict__ colback) {
  const int b = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M || pair_overflow(cursor, b, cap)) return;
  const size_t pb = (size_t)b * cap;
  const uint32_t beg = col_ptr[(size_t)b * (M + 1) + j], end = col_ptr[(size_t)b * (M + 1) + j + 1];
  const LineB lb = colB[(size_t)b * M + j];
  double S = 0.0;
  for (uint32_t q = beg; q < end; ++q) {
    const uint32_t p = csc_perm[pb + q];
    if (csr_jf[pb + p] & kFlagCol) S += (double)pcol[pb + p] * 0.5 * (double)pbar[pb + p];
  }
  LineBack out = {(float)S, 0.f, 0.f, lb.T};
  if (!(lb.flags & kLineK1)) {
    double szb = 0.0, Tbar = 0.0;
    for (uint32_t q = beg; q < end; ++q) {
      const uint32_t p = csc_perm[pb + q];
      if (!(csr_jf[pb + p] & kFlagCol)) continue;
      const double zb = (double)pcol[pb + p] * (0.5 * (double)pbar[pb + p] - S);
      szb += zb;
      Tbar -= zb * ((double)cs[pb + p] - (double)lb.m);
    }
    const double mbar = (double)lb.T * szb;
    const double gbar = (lb.flags & kLineClamped) ? 0.0 : -Tbar * (double)lb.T / (double)lb.g;
    out.ca = (float)(mbar - gbar);
    out.cb = (float)gbar;
  } else {
    out.T = 0.f;
  }
  colback[(size_t)b * M + j] = out;
}

// Thread per row: cbar per entry and the Eq. (5) scatter into grad_pred (overwrites).
__global__ void k_grad(int N, int M, int L, int full, float eps_dist,
                       const unsigned* __restrict__ cursor, uint32_t cap,
                       const float4* __restrict__ pred4, const float4* __restrict__ gt4,
                       const unsigned* __restrict__ row_ptr, const uint32_t* __restrict__ csr_jf,
                       const float* __restrict__ cs, const float* __restrict__ P0,
                       const float* __restrict__ prow, const float* __restrict__ pcol,
                       const float* __restrict__ pbar, const float* __restrict__ a_hist,
                       const float* __restrict__ b_hist, const float* __restrict__ grad_loss,
                       const LineBack* __restrict__ rowback, const LineBack* __restrict__ colback,
                       const int2* __restrict__ rowidx, const int2* __restrict__ colidx,
                       float* __restrict__ grad_pred) {
  const int b = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  float* g = grad_pred + ((size_t)b * N + i) * 3;
  if (pair_overflow(cursor, b, cap)) {
    const float nan = __int_as_float(0x7fc00000);
    g[0] = nan; g[1] = nan; g[2] = nan;
    return;
  }
  const size_t pb = (size_t)b * cap;
  const float gl = grad_loss[b];
  const float4 x = pred4[(size_t)b * N + i];
  const float aL = a_hist[((size_t)b * N + i) * (L + 1) + L];
  const uint32_t beg = row_ptr[(size_t)b * (N + 1) + i], end = row_ptr[(size_t)b * (N + 1) + i + 1];
  LineBack rbk = {0.f, 0.f, 0.f, 0.f};
  int2 ri = make_int2(-1, -1);
  if (full) { rbk = rowback[(size_t)b * N + i]; ri = rowidx[(size_t)b * N + i]; }
  double gx = 0.0, gy = 0.0, gz = 0.0;
  for (uint32_t p = beg; p < end; ++p) {
    const uint32_t jf = csr_jf[pb + p];
    const uint32_t j = jf & kIdxMask;
    const float bL = b_hist[((size_t)b * M + j) * (L + 1) + L];
    const double c = (double)cs[pb + p];
    double cbar = (double)gl * (double)aL * (double)P0[pb + p] * (double)bL;
    if (full) {
      const double hp = 0.5 * (double)pbar[pb + p];
      if (jf & kFlagRow) cbar -= (double)rbk.T * (double)prow[pb + p] * (hp - (double)rbk.S);
      if ((int)j == ri.x) cbar += rbk.ca;
      if ((int)j == ri.y) cbar += rbk.cb;
      const bool cf = (jf & kFlagCol) != 0;
      const int2 ci = colidx[(size_t)b * M + j];
      if (cf || ci.x == i || ci.y == i) {
        const LineBack cbk = colback[(size_t)b * M + j];
        if (cf) cbar -= (double)cbk.T * (double)pcol[pb + p] * (hp - (double)cbk.S);
        if (ci.x == i) cbar += cbk.ca;
        if (ci.y == i) cbar += cbk.cb;
      }
    }
    const float4 y = gt4[(size_t)b * M + j];
    const double w = cbar / (c + (double)eps_dist);  // Eq. (5)
    gx += w * ((double)x.x - (double)y.x);
    gy += w * ((double)x.y - (double)y.y);
    gz += w * ((double)x.z - (double)y.z);
  }
  g[0] = (float)gx; g[1] = (float)gy; g[2] = (float)gz;
}

}  // namespace apml
