// k_bwd2.cuh -- full-mode backward of one pair per cluster, on
// shared-memory slices loaded with coalesced bulk copies from the forward's CSR / CSC arrays.
//
// Differences from k_sparse_bwd (k_mega.cuh), which it replaces for the full gradient after
// k_sparse_fwd2:
//   * set-up: the CTA's CSR slice (j | flags, P0, c) and CSC slice (i | flags, P0, c -- the
//     forward writes the CSC-order copies) are copied into shared memory with cp.async, a^L
//     (all rows) and b^L (all columns) too, so the initial adjoints
//        abar_i = g sum_j P0_ij b^L_j c_ij,  bbar_j = g sum_i a^L_i P0_ij c_ij,
//        P0bar_ij = g a^L_i b^L_j c_ij
//     need no global gathers;
//   * reverse Sinkhorn: sinkhorn_bwd of k_mega.cuh on those slices;
//   * column softmax reverse: reads its CSC-order inputs (flags, c, P_col) contiguously and
//     gathers only P0bar through the CSC -> CSR permutation (1 load per entry instead of 4).
// The row softmax reverse and the Eq. (5) scatter are k_mega.cuh's (row_soft_rev, grad_rows).

#pragma once
#include "k_fwd2.cuh"

namespace apml {

// Column softmax reverse (thread per column <= kRegLine entries, warp per longer column):
// S = sum_kept P_col Pbar/2, zbar = P_col (Pbar/2 - S), Tbar = -sum zbar (c - m),
// gbar = -Tbar T / g (0 if clamped) -> LineBack {S, mbar - gbar, gbar, T} (as col_soft_rev).
template <int G>
__device__ void col_soft_rev2(const SparseArgs& A, int b, Slice s, const unsigned* off, const float* cc,
                              uint32_t gc, const LongList& ll) {
  const int M = A.M;
  const size_t pb = (size_t)b * A.cap;
  const int lane = threadIdx.x & 31;
  auto body = [&](int j) {
    const int k = j - s.lo;
    const uint32_t beg = off[k], end = off[k + 1];
    const LineB lb = A.colB[(size_t)b * M + j];
    LineBack out = {0.f, 0.f, 0.f, 0.f};
    if (!(lb.flags & kLineK1)) {
      double S = 0.0, szb = 0.0, Tbar = 0.0;
      if (G == 1) {
        float pc[kRegLine], pbv[kRegLine], cv[kRegLine];
        uint32_t fl = 0u;
        const uint32_t L = end - beg;
        uint32_t pp[kRegLine];
#pragma unroll
        for (uint32_t u = 0; u < kRegLine; ++u) {
          const bool v = u < L;
          pp[u] = v ? A.csc_perm[pb + gc + beg + u] : 0u;
          fl |= (v && (A.csc_if[pb + gc + beg + u] & kFlagCol)) ? (1u << u) : 0u;
          pc[u] = v ? A.csc_pc[pb + gc + beg + u] : 0.f;
          cv[u] = v ? cc[beg + u] : 0.f;
        }
#pragma unroll
        for (uint32_t u = 0; u < kRegLine; ++u) pbv[u] = u < L ? A.pbar[pb + pp[u]] : 0.f;
#pragma unroll
        for (uint32_t u = 0; u < kRegLine; ++u)
          if (fl >> u & 1u) S += (double)pc[u] * 0.5 * (double)pbv[u];
#pragma unroll
        for (uint32_t u = 0; u < kRegLine; ++u) {
          if (!(fl >> u & 1u)) continue;
          const double zb = (double)pc[u] * (0.5 * (double)pbv[u] - S);
          szb += zb;
          Tbar -= zb * ((double)cv[u] - (double)lb.m);
        }
      } else {
        for (uint32_t q = beg + lane; q < end; q += 32)
          if (A.csc_if[pb + gc + q] & kFlagCol)
            S += (double)A.csc_pc[pb + gc + q] * 0.5 * (double)A.pbar[pb + A.csc_perm[pb + gc + q]];
        S = gsum<32>(S);
        for (uint32_t q = beg + lane; q < end; q += 32) {
          if (!(A.csc_if[pb + gc + q] & kFlagCol)) continue;
          const double zb =
              (double)A.csc_pc[pb + gc + q] * (0.5 * (double)A.pbar[pb + A.csc_perm[pb + gc + q]] - S);
          szb += zb;
          Tbar -= zb * ((double)cc[q] - (double)lb.m);
        }
        szb = gsum<32>(szb);
        Tbar = gsum<32>(Tbar);
      }
      const double mbar = (double)lb.T * szb;
      const double gbar = (lb.flags & kLineClamped) ? 0.0 : -Tbar * (double)lb.T / (double)lb.g;
      out = {(float)S, (float)(mbar - gbar), (float)gbar, lb.T};
    }
    if (G == 1 || lane == 0) A.colback[(size_t)b * M + j] = out;
  };
  if (G == 1) {
    for (int j = s.lo + threadIdx.x; j < s.hi; j += blockDim.x)
      if (off[j - s.lo + 1] - off[j - s.lo] <= kRegLine) body(j);
  } else {
    for (int q = threadIdx.x >> 5; q < ll.count(); q += blockDim.x >> 5) {
      const int j = ll.line(q);
      if (off[j - s.lo + 1] - off[j - s.lo] > kRegLine) body(j);
    }
  }
}

// cbar per entry and the Eq. (5) scatter (as grad_rows<1, U>) for the rows of <= kRegLine
// entries, reading the CTA's shared-memory CSR slice (16-bit j, c, P0, P0bar) instead of the
// global copies; flags / P_row / P_col stay global (contiguous per row).
template <int U>
__device__ void grad_rows_sm(const SparseArgs& A, int b, Slice s, const unsigned* off, const uint16_t* j16,
                             const float* cs, const float* p0s, const float* pbs, uint32_t gr) {
  const int N = A.N, M = A.M, L = A.L;
  const size_t pb = (size_t)b * A.cap;
  const float gl = A.grad_loss[b];
  const float* aL = A.a_hist + ((size_t)b * (L + 1) + L) * N;
  const float* bL = A.b_hist + ((size_t)b * (L + 1) + L) * M;
  for (int i = s.lo + threadIdx.x; i < s.hi; i += blockDim.x) {
    const int k = i - s.lo;
    const uint32_t beg = off[k], end = off[k + 1];
    if (end - beg > kRegLine) continue;
    const float4 x = A.pred4[(size_t)b * N + i];
    const LineBack rbk = A.rowback[(size_t)b * N + i];
    const int2 ri = A.rowidx[(size_t)b * N + i];
    const double ai = (double)aL[i];
    double gx = 0.0, gy = 0.0, gz = 0.0;
    for (uint32_t p0 = beg; p0 < end; p0 += U) {
      uint32_t jf[U], j[U];
      float cv[U], p0v[U], pbv[U], prv[U], pcv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t p = p0 + u;
        const bool v = p < end;
        j[u] = v ? (uint32_t)j16[p] : 0u;
        cv[u] = v ? cs[p] : 1.f;
        p0v[u] = v ? p0s[p] : 0.f;
        pbv[u] = v ? pbs[p] : 0.f;
        jf[u] = v ? A.csr_jf[pb + gr + p] : 0u;
        prv[u] = v ? A.prow[pb + gr + p] : 0.f;
        pcv[u] = v ? A.pcol[pb + gr + p] : 0.f;
      }
      float4 y[U];
      float bLv[U];
      int2 ci[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool v = p0 + u < end;
        y[u] = v ? A.gt4[(size_t)b * M + j[u]] : x;
        bLv[u] = v ? bL[j[u]] : 0.f;
        ci[u] = v ? A.colidx[(size_t)b * M + j[u]] : make_int2(-1, -1);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (p0 + u >= end) continue;
        double cbar = (double)gl * ai * (double)p0v[u] * (double)bLv[u];  // d loss / d c = v
        const double hp = 0.5 * (double)pbv[u];
        if (jf[u] & kFlagRow) cbar -= (double)rbk.T * (double)prv[u] * (hp - (double)rbk.S);
        if ((int)j[u] == ri.x) cbar += rbk.ca;
        if ((int)j[u] == ri.y) cbar += rbk.cb;
        const bool cf = (jf[u] & kFlagCol) != 0;
        if (cf || ci[u].x == i || ci[u].y == i) {
          const LineBack cbk = A.colback[(size_t)b * M + j[u]];
          if (cf) cbar -= (double)cbk.T * (double)pcv[u] * (hp - (double)cbk.S);
          if (ci[u].x == i) cbar += cbk.ca;
          if (ci[u].y == i) cbar += cbk.cb;
        }
        const double w = cbar / ((double)cv[u] + (double)A.eps_dist);  // Eq. (5)
        if (A.gw) A.gw[pb + gr + p0 + u] = (float)w;
        gx += w * ((double)x.x - (double)y[u].x);
        gy += w * ((double)x.y - (double)y[u].y);
        gz += w * ((double)x.z - (double)y[u].z);
      }
    }
    float* g = A.grad_pred + ((size_t)b * N + orig_row(A, b, (uint32_t)i)) * 3;
    g[0] = (float)gx; g[1] = (float)gy; g[2] = (float)gz;
  }
}

__device__ __forceinline__ void sparse_bwd2_body(const SparseArgs& A) {
  extern __shared__ __align__(16) uint8_t shm[];
  uint32_t* s_long_r = long_lists();
  uint32_t* s_long_c = s_long_r + kLongCap;
  __shared__ int s_nlong[2];
  __shared__ __align__(8) unsigned long long s_mbar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int CL = cl.num_blocks(), rank = cl.block_rank();
  const int b = blockIdx.x / CL;
  const int N = A.N, M = A.M, L = A.L;
  const size_t pb = (size_t)b * A.cap;
  const Slice sr = slice_of(N, rank, CL), sc = slice_of(M, rank, CL);
  const int nr = sr.hi - sr.lo, nc = sc.hi - sc.lo;
  pdl_trigger();
  pdl_wait();  // the forward's saved state (k_sparse_fwd2)
  if (A.cursor[b] > A.cap) {
    const float nan = __int_as_float(0x7fc00000);
    for (int i = sr.lo + threadIdx.x; i < sr.hi; i += blockDim.x) {
      float* g = A.grad_pred + ((size_t)b * N + orig_row(A, b, (uint32_t)i)) * 3;
      g[0] = nan; g[1] = nan; g[2] = nan;
    }
    return;
  }
  const unsigned* rp = A.row_ptr + (size_t)b * (N + 1);
  const unsigned* cp = A.col_ptr + (size_t)b * (M + 1);
  const LongList llr = collect_long(rp, sr, s_long_r, &s_nlong[0]);
  const LongList llc = collect_long(cp, sc, s_long_c, &s_nlong[1]);
  phase(A, 0);
  const float gl = A.grad_loss[b];
  const float* aLg = A.a_hist + ((size_t)b * (L + 1) + L) * N;
  const float* bLg = A.b_hist + ((size_t)b * (L + 1) + L) * M;
  const uint32_t gr = rp[sr.lo], gc = cp[sc.lo];
  const uint32_t nnzr = rp[sr.hi] - gr, nnzc = cp[sc.hi] - gc;

  // ---- shared memory: replicas (Rbar^l; Qbar^l), abar / bbar, b^l double buffer, offsets,
  // CSR slice {jf, P0, c, P0bar}, CSC slice {i|flags, P0, c}, own-row a history if it fits
  uint8_t* sm = shm;
  const size_t vN = 4 * (size_t)((N + 3) / 4 * 4 + 4), vM = 4 * (size_t)((M + 3) / 4 * 4 + 4);
  float* rcur = reinterpret_cast<float*>(carve(sm, vN));  // a^L during set-up
  float* qcur = reinterpret_cast<float*>(carve(sm, vM));
  float* ab = reinterpret_cast<float*>(carve(sm, 4 * (size_t)nr));
  float* bb = reinterpret_cast<float*>(carve(sm, 4 * (size_t)nc));
  float* bls = reinterpret_cast<float*>(carve(sm, 8 * (size_t)M));
  unsigned* roff = reinterpret_cast<unsigned*>(carve(sm, 4 * (size_t)(nr + 1)));
  unsigned* coff = reinterpret_cast<unsigned*>(carve(sm, 4 * (size_t)(nc + 1)));
  // line orders by length for the reverse Sinkhorn (single-CTA clusters, as the forward)
  uint16_t* rperm = (CL == 1 && nr <= 65536 && nc <= 65536) ? reinterpret_cast<uint16_t*>(carve(sm, 2 * (size_t)nr)) : nullptr;
  uint16_t* cperm = rperm ? reinterpret_cast<uint16_t*>(carve(sm, 2 * (size_t)nc)) : nullptr;
  __shared__ unsigned s_hist[kRegLine + 2];
  auto a16 = [](size_t v) { return (v + 15) & ~size_t(15); };
  const size_t ent = 4 * a16(4 * (size_t)nnzr) + 3 * a16(4 * (size_t)nnzc);
  const bool fit = (size_t)(sm - shm) + ent <= A.smem_bytes;  // (u16 indices need less)
  // shared-memory slices use 16-bit indices (flags stay in the global copies)
  const bool fit16 = fit && N <= 65536 && M <= 65536;
  uint32_t *rjf = nullptr, *cif = nullptr;
  uint16_t *r16 = nullptr, *c16 = nullptr;
  float *rP0, *rc, *racc, *cP0, *ccs;
  if (fit16) {
    r16 = reinterpret_cast<uint16_t*>(carve(sm, 2 * (size_t)nnzr));
    rP0 = reinterpret_cast<float*>(carve(sm, 4 * (size_t)nnzr));
    rc = reinterpret_cast<float*>(carve(sm, 4 * (size_t)nnzr));
    racc = reinterpret_cast<float*>(carve(sm, 4 * (size_t)nnzr));
    c16 = reinterpret_cast<uint16_t*>(carve(sm, 2 * (size_t)nnzc));
    cP0 = reinterpret_cast<float*>(carve(sm, 4 * (size_t)nnzc));
    ccs = reinterpret_cast<float*>(carve(sm, 4 * (size_t)nnzc));
    g2s_async(rP0, A.P0 + pb + gr, nnzr);
    g2s_async(rc, A.cs + pb + gr, nnzr);
    g2s_async(cP0, A.P0c + pb + gc, nnzc);
    g2s_async(ccs, A.csc_c + pb + gc, nnzc);
    constexpr int kU = 8;
    const uint32_t bd = blockDim.x;
    for (uint32_t k0 = threadIdx.x; k0 < nnzr; k0 += kU * bd) {
      uint32_t v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = k0 + u * bd < nnzr ? A.csr_jf[pb + gr + k0 + u * bd] : 0u;
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (k0 + u * bd < nnzr) r16[k0 + u * bd] = (uint16_t)(v[u] & kIdxMask);
    }
    for (uint32_t k0 = threadIdx.x; k0 < nnzc; k0 += kU * bd) {
      uint32_t v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = k0 + u * bd < nnzc ? A.csc_i[pb + gc + k0 + u * bd] : 0u;
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (k0 + u * bd < nnzc) c16[k0 + u * bd] = (uint16_t)v[u];
    }
  } else {
    rjf = A.csr_jf + pb + gr;
    rP0 = A.P0 + pb + gr;
    rc = A.cs + pb + gr;
    racc = A.pbar + pb + gr;
    cif = A.csc_if + pb + gc;
    cP0 = A.P0c + pb + gc;
    ccs = A.csc_c + pb + gc;
  }
  // own rows' a history [L+1][nr] and the whole b history [L+1][M] when they fit (else
  // sinkhorn_bwd reads them from global memory, b^l staged per iteration in bls)
  float *ahs = nullptr, *bhs = nullptr;
  if (fit16 && (size_t)(sm - shm) + 4 * (size_t)(L + 1) * nr + 16 <= A.smem_bytes) {
    ahs = reinterpret_cast<float*>(carve(sm, 4 * (size_t)(L + 1) * nr));
    const float* ahg = A.a_hist + (size_t)b * (L + 1) * N;
    for (int l = 0; l <= L; ++l) g2s_async(ahs + (size_t)l * nr, ahg + (size_t)l * N + sr.lo, nr);
    if (A.bhs_stage && (size_t)(sm - shm) + 4 * (size_t)(L + 1) * M + 16 <= A.smem_bytes) {
      bhs = reinterpret_cast<float*>(carve(sm, 4 * (size_t)(L + 1) * M));
      g2s_async(bhs, A.b_hist + (size_t)b * (L + 1) * M, (size_t)(L + 1) * M);
    }
  }
  g2s_async(rcur, aLg, N);                 // a^L, all rows (bbar)
  g2s_async(bls + (L & 1) * M, bLg, M);    // b^L, all columns (abar, P0bar)
  for (int k = threadIdx.x; k <= nr; k += blockDim.x) roff[k] = rp[sr.lo + k] - gr;
  for (int k = threadIdx.x; k <= nc; k += blockDim.x) coff[k] = cp[sc.lo + k] - gc;
  if (threadIdx.x == 0) {
    mbar_init(smem_addr(&s_mbar[0]));
    mbar_init(smem_addr(&s_mbar[1]));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cp_async_wait_all();
  __syncthreads();
  Xchg xr{rcur, smem_addr(&s_mbar[0]), N, true, 0u};
  Xchg xq{qcur, smem_addr(&s_mbar[1]), M, true, 0u};
  xchg_arm(xr);  // peers push Rbar^L only after the cluster barrier below
  xchg_arm(xq);
  phase(A, 1);

  // ---- initial adjoints (loss = sum a P0 b c): abar, bbar, P0bar (rows by thread / warp)
  const float* bL = bls + (L & 1) * M;
  const float* aL = rcur;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  auto row_init = [&](int i, int G) {
    const int k = i - sr.lo;
    const uint32_t p0 = roff[k], p1 = roff[k + 1];
    const float ga = gl * aL[i];
    double t = 0.0;
    for (uint32_t p = p0 + (G == 1 ? 0 : lane); p < p1; p += G) {
      const float bj = bL[r16 ? (uint32_t)r16[p] : (rjf[p] & kIdxMask)], c = rc[p];
      t += (double)rP0[p] * (double)bj * (double)c;
      racc[p] = ga * bj * c;
    }
    if (G == 32) t = gsum<32>(t);
    if (G == 1 || lane == 0) ab[k] = (float)((double)gl * t);
  };
  auto col_init = [&](int j, int G) {
    const int k = j - sc.lo;
    const uint32_t q0 = coff[k], q1 = coff[k + 1];
    double t = 0.0;
    for (uint32_t q = q0 + (G == 1 ? 0 : lane); q < q1; q += G)
      t += (double)aL[c16 ? (uint32_t)c16[q] : (cif[q] & kIdxMask)] * (double)cP0[q] * (double)ccs[q];
    if (G == 32) t = gsum<32>(t);
    if (G == 1 || lane == 0) bb[k] = (float)((double)gl * t);
  };
  for (int k = threadIdx.x; k < nr; k += blockDim.x)
    if (roff[k + 1] - roff[k] <= kRegLine) row_init(sr.lo + k, 1);
  for (int k = threadIdx.x; k < nc; k += blockDim.x)
    if (coff[k + 1] - coff[k] <= kRegLine) col_init(sc.lo + k, 1);
  for (int q = w; q < llr.count(); q += nw) {
    const int i = llr.line(q);
    if (roff[i - sr.lo + 1] - roff[i - sr.lo] > kRegLine) row_init(i, 32);
  }
  for (int q = w; q < llc.count(); q += nw) {
    const int j = llc.line(q);
    if (coff[j - sc.lo + 1] - coff[j - sc.lo] > kRegLine) col_init(j, 32);
  }
  if (rperm) {
    line_perm(roff, nr, rperm, s_hist);
    line_perm(coff, nc, cperm, s_hist);
  }
  csync(cl);  // every CTA is done with its a^L copy before Rbar^L arrives in it
  phase(A, 2);

  // ---- reverse Sinkhorn (P0bar accumulated per CSR entry)
  {
    if (fit16) {
      const SliceView<uint16_t> R{roff, r16, rP0, racc};
      const SliceView<uint16_t> C{coff, c16, cP0, nullptr};
      sinkhorn_bwd<uint16_t, true>(cl, A, b, sr, sc, R, C, ab, bb, xr, xq, (bhs || M > kPf * (int)blockDim.x) ? nullptr : bls, ahs, bhs, llr, llc,
                                    rperm, cperm);
    } else {
      const SliceView<uint32_t> R{roff, rjf, rP0, racc};
      const SliceView<uint32_t> C{coff, cif, cP0, nullptr};
      sinkhorn_bwd<uint32_t, false>(cl, A, b, sr, sc, R, C, ab, bb, xr, xq, (bhs || M > kPf * (int)blockDim.x) ? nullptr : bls, ahs, bhs, llr, llc);
    }
  }
  if (fit16)
    for (uint32_t p = threadIdx.x; p < nnzr; p += blockDim.x) A.pbar[pb + gr + p] = racc[p];
  __syncthreads();
  phase(A, 3);
  // ---- row softmax reverse (own rows; global CSR arrays, contiguous per row)
  row_soft_rev<1, 8>(A, b, sr, llr);
  row_soft_rev<32, 1>(A, b, sr, llr);
  csync(cl);  // P0bar of every row visible to the column owners
  phase(A, 4);
  // ---- column softmax reverse (own columns; CSC-order inputs + P0bar through csc_perm)
  col_soft_rev2<1>(A, b, sc, coff, ccs, gc, llc);
  col_soft_rev2<32>(A, b, sc, coff, ccs, gc, llc);
  csync(cl);  // column adjoints visible to the row owners
  phase(A, 5);
  // ---- cbar per entry and the Eq. (5) scatter into grad_pred
  if (fit16) grad_rows_sm<4>(A, b, sr, roff, r16, rc, rP0, racc, gr);
  else grad_rows<1, 4>(A, b, sr, llr);
  grad_rows<32, 1>(A, b, sr, llr);
  phase(A, 6);
}

__global__ void __launch_bounds__(kMegaThreads, 1) k_sparse_bwd2(const SparseArgs A) { sparse_bwd2_body(A); }

// Forward + backward in ONE launch (apml_plan_forward_backward: the training step with
// grad_loss known before the launch).  Each cluster runs its pair's sparse forward, one
// cluster barrier (release / acquire at cluster scope: the pair's CSR / CSC arrays, history and
// line data written by any CTA of the cluster are visible to all of them), then the backward:
// no kernel boundary between them, and a pair whose forward finishes early goes straight on
// instead of waiting for the slowest pair of the batch.
__global__ void __launch_bounds__(kMegaThreads, 1) k_sparse_fwdbwd2(const SparseArgs A) {
  sparse_fwd2_body(A);
  cg::cluster_group cl = cg::this_cluster();
  csync(cl);
  sparse_bwd2_body(A);
}

}  // namespace apml
