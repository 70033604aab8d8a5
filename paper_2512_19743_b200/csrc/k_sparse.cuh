// k_sparse.cuh -- O(B * nnz) stages of the forward.
//
//   k_scan        per-pair exclusive scan of row / column counts -> CSR row_ptr, CSC col_ptr
//                 ("an exclusive prefix sum converts these counts into write offsets")
//   k_scatter     bucket the emitted entries by row and by column (counting sort)
//   k_sort_rows   order each row segment by j (deterministic), record entry -> CSR position
//   k_sort_cols   order each column segment by i; CSC perm = CSR position of the same (i, j)
//                 -- together the key-sort / merge of P:99, Alg. 1 line 3; each
//                 (i, j) is emitted once with its direction flags, so the "duplicates" of
//                 the paper's concatenated streams are merged by construction.
//   k_row_norm    c = sqrt(d2), s = exp(-T (c - m)) on row-kept entries, Z = sum, P_row = s/Z
//                 (Eq. (2), "normalizes ... by the sum of kept similarities");
//                 argmin / second argmin = first entries whose d2 equals m2 / s2 (R12).
//   k_col_norm    the same over CSC -> P_col; P0 = (P_row + P_col)/2, a missing direction
//                 counting as 0 (reading R8); P0 stored in CSR and CSC order.
//   (Sinkhorn + loss: k_sinkhorn.cuh)
//
// Per-pair arrays are [B][cap] (cap = emit capacity per pair); positions inside a pair are
// 32-bit.  A pair whose emission overflowed its capacity is skipped (loss = NaN).
#pragma once
#include "common.cuh"

namespace apml {

// Block-wide exclusive scan of cnt[0..n] -> ptr[0..n] for pair blockIdx.x; also zeroes cnt
// (reused as the fill cursor by k_scatter).  1024 threads.
__global__ void __launch_bounds__(1024)
k_scan(unsigned* __restrict__ cnt, unsigned* __restrict__ ptr, int n) {
  const int b = blockIdx.x;
  unsigned* c = cnt + (size_t)b * (n + 1);
  unsigned* p = ptr + (size_t)b * (n + 1);
  const int len = n + 1;
  const int per = (len + blockDim.x - 1) / blockDim.x;
  const int beg = threadIdx.x * per, end = min(len, beg + per);
  unsigned sum = 0;
  for (int k = beg; k < end; ++k) sum += c[k];
  __shared__ unsigned warp_tot[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) warp_tot[w] = inc;
  __syncthreads();
  if (w == 0) {
    unsigned t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += v;
    }
    warp_tot[lane] = t;
  }
  __syncthreads();
  unsigned run = inc - sum + (w ? warp_tot[w - 1] : 0u);
  for (int k = beg; k < end; ++k) {
    const unsigned v = c[k];
    p[k] = run;
    run += v;
    c[k] = 0u;
  }
}

__global__ void k_scatter(const uint2* __restrict__ ebuf, const unsigned* __restrict__ cursor,
                          uint32_t cap, int N, int M, const unsigned* __restrict__ row_ptr,
                          unsigned* __restrict__ row_fill, const unsigned* __restrict__ col_ptr,
                          unsigned* __restrict__ col_fill, uint32_t* __restrict__ csr_t,
                          uint32_t* __restrict__ csc_t) {
  const int b = blockIdx.y;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned total = cursor[b];
  if (total > cap || t >= total) return;
  const uint2 e = ebuf[(size_t)b * cap + t];
  const uint32_t i = e.x, j = e.y & kIdxMask;
  const size_t rb = (size_t)b * (N + 1), cb = (size_t)b * (M + 1);
  const uint32_t p = row_ptr[rb + i] + atomicAdd(row_fill + rb + i, 1u);
  const uint32_t q = col_ptr[cb + j] + atomicAdd(col_fill + cb + j, 1u);
  csr_t[(size_t)b * cap + p] = t;
  csc_t[(size_t)b * cap + q] = t;
}

// Warp per line: rank-sort a segment of entry ids by their key (j for rows, i for columns).
// Keys inside a line are distinct, so rank = #keys smaller.  Segments are short (~5 on
// average, <= ~170 in practice); a long degenerate line costs O(L^2 / 32) per warp.
template <bool kRows>
__global__ void k_sort_lines(const uint2* __restrict__ ebuf, const unsigned* __restrict__ cursor,
                             uint32_t cap, int nlines, const unsigned* __restrict__ ptr,
                             const uint32_t* __restrict__ seg_t, uint32_t* __restrict__ out_key,
                             uint32_t* __restrict__ inv_or_perm_in, uint32_t* __restrict__ perm_out) {
  const int b = blockIdx.y;
  const int line = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (line >= nlines || pair_overflow(cursor, b, cap)) return;
  const size_t pb = (size_t)b * cap;
  const uint32_t beg = ptr[(size_t)b * (nlines + 1) + line];
  const uint32_t end = ptr[(size_t)b * (nlines + 1) + line + 1];
  const uint32_t L = end - beg;
  auto key_of = [&](uint32_t t) -> uint32_t {
    const uint2 e = ebuf[pb + t];
    return kRows ? (e.y & kIdxMask) : e.x;
  };
  auto place = [&](uint32_t t, uint32_t rank) {
    const uint2 e = ebuf[pb + t];
    const uint32_t pos = beg + rank;
    if (kRows) {
      out_key[pb + pos] = e.y;                  // j | flags
      inv_or_perm_in[pb + t] = pos;             // entry id -> CSR position
    } else {
      out_key[pb + pos] = e.x;                  // i
      perm_out[pb + pos] = inv_or_perm_in[pb + t];  // CSC position -> CSR position
    }
  };
  if (L <= 32) {
    const uint32_t t = lane < (int)L ? seg_t[pb + beg + lane] : 0u;
    const uint32_t key = lane < (int)L ? key_of(t) : 0xffffffffu;
    uint32_t rank = 0;
    for (uint32_t k = 0; k < L; ++k) rank += (__shfl_sync(0xffffffffu, key, k) < key) ? 1u : 0u;
    if (lane < (int)L) place(t, rank);
  } else {
    for (uint32_t e = beg + lane; e < end; e += 32) {
      const uint32_t t = seg_t[pb + e];
      const uint32_t key = key_of(t);
      uint32_t rank = 0;
      for (uint32_t f = beg; f < end; ++f) rank += (key_of(seg_t[pb + f]) < key) ? 1u : 0u;
      place(t, rank);
    }
  }
}

// Thread per row.  Writes d2, c, P_row (0 where the row flag is absent) per CSR entry and the
// row's argmin / second-argmin column (-1 if absent).
__global__ void k_row_norm(const float4* __restrict__ pred4, const float4* __restrict__ gt4,
                           int N, int M, const unsigned* __restrict__ cursor, uint32_t cap,
                           const unsigned* __restrict__ row_ptr, const uint32_t* __restrict__ csr_jf,
                           const LineA* __restrict__ rowA, const LineB* __restrict__ rowB,
                           float* __restrict__ d2s, float* __restrict__ cs,
                           float* __restrict__ prow, int2* __restrict__ rowidx) {
  const int b = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N || pair_overflow(cursor, b, cap)) return;
  const size_t pb = (size_t)b * cap;
  const uint32_t beg = row_ptr[(size_t)b * (N + 1) + i], end = row_ptr[(size_t)b * (N + 1) + i + 1];
  const float4 x = pred4[(size_t)b * N + i];
  const LineA la = rowA[(size_t)b * N + i];
  const LineB lb = rowB[(size_t)b * N + i];
  int ia = -1, ib = -1;
  float Z = 0.f;
  for (uint32_t p = beg; p < end; ++p) {
    const uint32_t jf = csr_jf[pb + p];
    const uint32_t j = jf & kIdxMask;
    const float4 y = gt4[(size_t)b * M + j];
    const float d2 = dist2(x.x, x.y, x.z, y.x, y.y, y.z);
    const float c = __fsqrt_rn(d2);
    d2s[pb + p] = d2;
    cs[pb + p] = c;
    if (ia < 0 && d2 == la.m2) ia = (int)j;
    else if (ib < 0 && d2 == la.s2) ib = (int)j;
    float s = 0.f;
    if (jf & kFlagRow) {
      s = (lb.flags & kLineK1) ? 1.f : expf(-lb.T * (c - lb.m));
      Z += s;
    }
    prow[pb + p] = s;
  }
  const float iz = 1.f / Z;
  for (uint32_t p = beg; p < end; ++p) prow[pb + p] *= iz;
  rowidx[(size_t)b * N + i] = make_int2(ia, ib);
}

// Thread per column.  P_col, P0 (CSR and CSC order), column argmin / second-argmin row.
__global__ void k_col_norm(int N, int M, const unsigned* __restrict__ cursor, uint32_t cap,
                           const unsigned* __restrict__ col_ptr, const uint32_t* __restrict__ csc_i,
                           const uint32_t* __restrict__ csc_perm, const uint32_t* __restrict__ csr_jf,
                           const LineA* __restrict__ colA, const LineB* __restrict__ colB,
                           const float* __restrict__ d2s, const float* __restrict__ cs,
                           const float* __restrict__ prow, float* __restrict__ pcol,
                           float* __restrict__ P0, float* __restrict__ P0c,
                           int2* __restrict__ colidx) {
  const int b = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M || pair_overflow(cursor, b, cap)) return;
  const size_t pb = (size_t)b * cap;
  const uint32_t beg = col_ptr[(size_t)b * (M + 1) + j], end = col_ptr[(size_t)b * (M + 1) + j + 1];
  const LineA la = colA[(size_t)b * M + j];
  const LineB lb = colB[(size_t)b * M + j];
  int ia = -1, ib = -1;
  float Z = 0.f;
  for (uint32_t q = beg; q < end; ++q) {
    const uint32_t p = csc_perm[pb + q];
    const float d2 = d2s[pb + p];
    const uint32_t i = csc_i[pb + q];
    if (ia < 0 && d2 == la.m2) ia = (int)i;
    else if (ib < 0 && d2 == la.s2) ib = (int)i;
    if (csr_jf[pb + p] & kFlagCol)
      Z += (lb.flags & kLineK1) ? 1.f : expf(-lb.T * (cs[pb + p] - lb.m));
  }
  const float iz = 1.f / Z;
  for (uint32_t q = beg; q < end; ++q) {
    const uint32_t p = csc_perm[pb + q];
    float pc = 0.f;
    if (csr_jf[pb + p] & kFlagCol)
      pc = ((lb.flags & kLineK1) ? 1.f : expf(-lb.T * (cs[pb + p] - lb.m))) * iz;
    pcol[pb + p] = pc;
    const float p0 = 0.5f * (prow[pb + p] + pc);
    P0[pb + p] = p0;
    P0c[pb + q] = p0;
  }
  colidx[(size_t)b * M + j] = make_int2(ia, ib);
}

}  // namespace apml
