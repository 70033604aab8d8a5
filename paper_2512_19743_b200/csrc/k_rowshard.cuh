// k_rowshard.cuh -- the sparse stage when one cloud's pred rows are sharded over GPUs
// (north_star "pred rows shard and per-iteration column sums are
// all-reduced").  Rank r owns pred rows [row_offset, row_offset + N) of every pair and all M
// gt points.  Row quantities are local; every column quantity is a sum over the column's
// entries, which are spread over the ranks, so each one is formed as a local partial and
// all-reduced by the caller's collective (apml_comm, NCCL over NVLink in practice) between
// the kernels below.  Per forward: column (min, second) all-gather (X2), column softmax sum,
// column argmin candidates, L_iter column sums Q_j (X3), the loss.  Per backward: bbar init,
// L_iter column sums P0^T Rbar^l, column softmax reverse sums.  Every kernel is grid-wide
// (no cluster), reusing the per-line device functions of k_mega.cuh.
#pragma once
#include "k_nvls.cuh"
#include "k_mega.cuh"

namespace apml {

constexpr int kRsThreads = 512;

// ---------------------------------------------------------------- column statistics (X2)

// Collapse the S column-split partials of Pass A into one (min, second) per column.
__global__ void k_top2_collapse(const float2* __restrict__ part, int S, int B, int Mp, int M,
                                float2* __restrict__ out) {
  const int b = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M) return;
  float m = __int_as_float(0x7f800000), s = m;
  for (int k = 0; k < S; ++k) {
    const float2 p = part[((size_t)k * B + b) * Mp + j];
    top2_merge(m, s, p.x, p.y);
  }
  out[(size_t)b * M + j] = make_float2(m, s);
}

// ---------------------------------------------------------------- CSR / CSC (local entries)

// Batched multi-CTA exclusive scan of count arrays (CSR/CSC pointers, Morton-cell starts):
// per-tile sums, a per-array scan of the tile sums, then a rescan of every tile with its
// offset.  Loads and stores are coalesced; blockIdx.z selects one of two jobs, blockIdx.y
// the pair.  The counts are zeroed on the way (they are reused as scatter cursors).
constexpr int kScanThreads = 256, kScanPer = 8, kScanTile = kScanThreads * kScanPer;
struct ScanJob {
  unsigned* cnt;   // [B][stride], len used
  unsigned* ptr;   // [B][stride] exclusive prefix sums
  unsigned* tsum;  // [B][ntiles] tile sums, then tile offsets
  size_t stride;
  int len, ntiles;
};
struct ScanJobs { ScanJob j[2]; };

__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned* s_warp, unsigned* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_warp[w] = inc;
  __syncthreads();
  if (w == 0) {
    unsigned t = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    s_warp[lane] = t;
  }
  __syncthreads();
  const unsigned r = inc - v + (w ? s_warp[w - 1] : 0u);
  if (total) *total = s_warp[(blockDim.x >> 5) - 1];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const ScanJobs J) {
  const ScanJob jb = blockIdx.z ? J.j[1] : J.j[0];
  const int b = blockIdx.y, tile = blockIdx.x;
  if (tile >= jb.ntiles) return;
  const unsigned* c = jb.cnt + (size_t)b * jb.stride;
  unsigned v = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int idx = tile * kScanTile + k * kScanThreads + threadIdx.x;
    if (idx < jb.len) v += c[idx];
  }
  v = __reduce_add_sync(0xffffffffu, v);
  __shared__ unsigned s_w[kScanThreads / 32];
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) t += s_w[w];
    jb.tsum[(size_t)b * jb.ntiles + tile] = t;
  }
}

__global__ void __launch_bounds__(1024) k_scan_tiles(const ScanJobs J) {
  const ScanJob jb = blockIdx.z ? J.j[1] : J.j[0];
  __shared__ unsigned s_warp[32];
  unsigned* t = jb.tsum + (size_t)blockIdx.y * jb.ntiles;
  unsigned carry = 0;
  for (int base = 0; base < jb.ntiles; base += blockDim.x) {
    const int k = base + threadIdx.x;
    const unsigned v = k < jb.ntiles ? t[k] : 0u;
    unsigned tot;
    const unsigned e = block_excl_scan(v, s_warp, &tot);
    if (k < jb.ntiles) t[k] = carry + e;
    carry += tot;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const ScanJobs J) {
  const ScanJob jb = blockIdx.z ? J.j[1] : J.j[0];
  const int b = blockIdx.y, tile = blockIdx.x;
  if (tile >= jb.ntiles) return;
  __shared__ unsigned s_v[kScanTile + kScanTile / 32];
  __shared__ unsigned s_warp[32];
  unsigned* c = jb.cnt + (size_t)b * jb.stride;
  unsigned* out = jb.ptr + (size_t)b * jb.stride;
  const int base = tile * kScanTile;
  const int len = jb.len;
  unsigned v[kScanPer];
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {  // all loads in flight before any store
    const int idx = base + k * kScanThreads + threadIdx.x;
    v[k] = idx < len ? c[idx] : 0u;
  }
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int e = k * kScanThreads + threadIdx.x;
    if (base + e < len) c[base + e] = 0u;
    s_v[e + (e >> 5)] = v[k];
  }
  __syncthreads();
  unsigned loc[kScanPer], sum = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int e = threadIdx.x * kScanPer + k;
    loc[k] = sum;
    sum += s_v[e + (e >> 5)];
  }
  const unsigned off = block_excl_scan(sum, s_warp, nullptr) + jb.tsum[(size_t)b * jb.ntiles + tile];
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int e = threadIdx.x * kScanPer + k;
    s_v[e + (e >> 5)] = off + loc[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    const int e = k * kScanThreads + threadIdx.x, idx = base + e;
    if (idx < jb.len) out[idx] = s_v[e + (e >> 5)];
  }
}

__global__ void k_rs_scatter(const SparseArgs A) {
  const int b = blockIdx.y;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned total = A.cursor[b];
  if (total > A.cap || t >= total) return;
  const size_t pb = (size_t)b * A.cap;
  const uint2 e = ebuf_of(A, b)[t];
  const uint32_t i = e.x, j = e.y & kIdxMask;
  const size_t rb = (size_t)b * (A.N + 1), cb = (size_t)b * (A.M + 1);
  A.csr_t[pb + A.row_ptr[rb + i] + atomicAdd(A.row_cnt + rb + i, 1u)] = t;
  A.csc_t[pb + A.col_ptr[cb + j] + atomicAdd(A.col_cnt + cb + j, 1u)] = t;
}

__device__ __forceinline__ Slice block_slice(int n) {
  return Slice{min(n, (int)(blockIdx.x * blockDim.x)), min(n, (int)((blockIdx.x + 1) * blockDim.x))};
}

// Rows: sort by j + row softmax (everything row-local).
__global__ void __launch_bounds__(kRsThreads, 2) k_rs_rows(const SparseArgs A) {
  __shared__ uint32_t s_long[kLongCap];
  __shared__ int s_n;
  const int b = blockIdx.y;
  if (A.cursor[b] > A.cap) return;
  const Slice s = block_slice(A.N);
  // rows of up to 8 entries by a thread in registers (64 registers: two CTAs per SM), longer
  // ones by a warp (C4 / C5: ~4 entries per row)
  constexpr uint32_t kTh = 8;
  const LongList ll = collect_long(A.row_ptr + (size_t)b * (A.N + 1), s, s_long, &s_n, kTh);
  row_sort_norm_regs<kTh>(A, b, s);
  __syncthreads();
  sort_lines<true, kTh>(A, b, s, ll);
  __syncthreads();
  row_norm<kTh>(A, b, s, ll);
}

// Columns, pass 1: sort by i; partial column-softmax sum over this rank's entries and this
// rank's argmin / second-argmin candidates (global row indices, or -1):
//   cand = {first entry with d2 == m2, second entry with d2 == m2, first entry with d2 == s2}.
// CSC order of one short column by ORIGINAL row index (R12): csc_i and the CSR position of each
// entry (csc_perm), from the unsorted emit ids of the column (csc_t).
template <uint32_t KR>
__device__ __forceinline__ void col_rank_sort(const SparseArgs& A, int b, uint32_t beg, uint32_t L) {
  const size_t pb = (size_t)b * A.cap;
  uint32_t t[KR], ex[KR], key[KR], pp[KR];
#pragma unroll
  for (uint32_t k = 0; k < KR; ++k) t[k] = k < L ? A.csc_t[pb + beg + k] : 0u;
#pragma unroll
  for (uint32_t k = 0; k < KR; ++k) {
    ex[k] = k < L ? ebuf_of(A, b)[t[k]].x : 0u;
    pp[k] = k < L ? A.inv[pb + t[k]] : 0u;
  }
#pragma unroll
  for (uint32_t k = 0; k < KR; ++k) key[k] = k < L ? orig_row(A, b, ex[k]) : 0xffffffffu;
#pragma unroll
  for (uint32_t k = 0; k < KR; ++k) {
    uint32_t r = 0;
#pragma unroll
    for (uint32_t f = 0; f < KR; ++f) r += (key[f] < key[k]) ? 1u : 0u;
    if (k < L) {
      A.csc_i[pb + beg + r] = ex[k];
      A.csc_perm[pb + beg + r] = pp[k];
    }
  }
}

__global__ void __launch_bounds__(kRsThreads) k_rs_cols_a(const SparseArgs A) {
  __shared__ uint32_t s_long[kLongCap];
  __shared__ int s_n;
  const int b = blockIdx.y, M = A.M;
  if (A.cursor[b] > A.cap) return;
  const Slice s = block_slice(M);
  const unsigned* cp = A.col_ptr + (size_t)b * (M + 1);
  const LongList ll = collect_long(cp, s, s_long, &s_n);
  // short columns sorted in registers by col_sort_norm_regs would also normalise; here the
  // warp rank sort handles every column (long lists only cover long ones), so sort all:
  for (int j = s.lo + threadIdx.x; j < s.hi; j += blockDim.x) {
    const uint32_t beg = cp[j], end = cp[j + 1];
    if (end - beg > kRegLine) continue;
    // rank sort by (original) i in registers (all loads of the column in flight at once; an
    // in-place insertion sort through global memory chained two dependent loads per step)
    if (end - beg <= 8) col_rank_sort<8>(A, b, beg, end - beg);
    else col_rank_sort<kRegLine>(A, b, beg, end - beg);
  }
  __syncthreads();
  sort_lines<false>(A, b, s, ll);
  __syncthreads();
  const size_t pb = (size_t)b * A.cap;
  for (int j = s.lo + threadIdx.x; j < s.hi; j += blockDim.x) {
    const LineA la = A.colA[(size_t)b * M + j];
    const LineB lb = A.colB[(size_t)b * M + j];
    int x1 = -1, x2 = -1, y1 = -1;
    float Z = 0.f;
    for (uint32_t q = cp[j]; q < cp[j + 1]; ++q) {
      const uint32_t p = A.csc_perm[pb + q];
      const float d2 = A.d2s[pb + p];
      const int gi = A.row_offset + (int)orig_row(A, b, A.csc_i[pb + q]);  // global ORIGINAL row
      if (d2 == la.m2) { if (x1 < 0) x1 = gi; else if (x2 < 0) x2 = gi; }
      if (d2 == la.s2 && y1 < 0) y1 = gi;
      if (A.csr_jf[pb + p] & kFlagCol) Z += (lb.flags & kLineK1) ? 1.f : expf(-lb.T * (A.cs[pb + p] - lb.m));
    }
    float* red = A.colred + ((size_t)b * M + j) * 3;
    red[0] = Z; red[1] = 0.f; red[2] = 0.f;
    int* c = A.cand + ((size_t)b * M + j) * 3;
    c[0] = x1; c[1] = x2; c[2] = y1;
  }
}

// Columns, pass 2 (after the all-reduce of Z and the all-gather of the candidates):
// P_col, P0 in CSR and CSC order, and the global argmin / second argmin of the column.
__global__ void __launch_bounds__(kRsThreads) k_rs_cols_b(const SparseArgs A, const int* __restrict__ gcand,
                                                          int world) {
  const int b = blockIdx.y, M = A.M, B = gridDim.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (A.cursor[b] > A.cap || j >= M) return;
  const size_t pb = (size_t)b * A.cap;
  const unsigned* cp = A.col_ptr + (size_t)b * (M + 1);
  const LineA la = A.colA[(size_t)b * M + j];
  const LineB lb = A.colB[(size_t)b * M + j];
  // merge candidates over ranks: argmin = lowest index with d2 == m2; second = second-lowest
  // such index when s2 == m2, else the lowest index with d2 == s2
  int a1 = -1, a2 = -1, y = -1;
  auto ins = [&](int v) {
    if (v < 0) return;
    if (a1 < 0 || v < a1) { a2 = a1; a1 = v; }
    else if (a2 < 0 || v < a2) a2 = v;
  };
  for (int r = 0; r < world; ++r) {
    const int* c = gcand + (((size_t)r * B + b) * M + j) * 3;
    ins(c[0]);
    ins(c[1]);
    if (c[2] >= 0 && (y < 0 || c[2] < y)) y = c[2];
  }
  int second = (la.s2 == la.m2) ? a2 : y;
  if (A.ipperm) {  // relabelled (one rank, row_offset 0): back to sorted positions
    a1 = a1 >= 0 ? A.ipperm[(size_t)b * A.N + a1] : -1;
    second = second >= 0 ? A.ipperm[(size_t)b * A.N + second] : -1;
  }
  A.colidx[(size_t)b * M + j] = make_int2(a1, second);
  const float iz = 1.f / A.colred[((size_t)b * M + j) * 3];
  for (uint32_t q = cp[j]; q < cp[j + 1]; ++q) {
    const uint32_t p = A.csc_perm[pb + q];
    float pc = 0.f;
    if (A.csr_jf[pb + p] & kFlagCol) pc = ((lb.flags & kLineK1) ? 1.f : expf(-lb.T * (A.cs[pb + p] - lb.m))) * iz;
    A.pcol[pb + p] = pc;
    const float p0 = 0.5f * (A.prow[pb + p] + pc);
    A.P0[pb + p] = p0;
    A.P0c[pb + q] = p0;
  }
}

// ---------------------------------------------------------------- warp-cooperative lines
// The per-iteration kernels below run 256-thread blocks, one warp per 32 consecutive lines:
// the warp walks the lines' contiguous entry range in chunks of kWChunk entries, staging the
// per-entry factors with coalesced loads (entry-parallel), then every lane folds its own
// line's staged factors in entry order -- the same sequential fma chain as a thread-per-line
// loop, without its uncoalesced, latency-serialised loads.
constexpr int kWChunk = 128;
constexpr int kWWarps = 8;  // warps per 256-thread block

struct WarpLines {
  uint32_t beg, end;  // this lane's line [beg, end) (empty past the last line)
  uint32_t e0, e1;    // the warp's entry range
};
__device__ __forceinline__ WarpLines warp_lines(const unsigned* ptr, int line, int n) {
  WarpLines w;
  w.beg = ptr[min(line, n)];
  w.end = ptr[min(line + 1, n)];
  w.e0 = __shfl_sync(0xffffffffu, w.beg, 0);
  w.e1 = __shfl_sync(0xffffffffu, w.end, 31);
  return w;
}

// stage(k, q): entry-parallel, k = slot in the chunk, q = entry; line(k): the owning lane,
// in entry order; post(k, q): entry-parallel again with s_own[k] = owning lane.
template <class Stage, class Line, class Post>
__device__ __forceinline__ void warp_walk(const WarpLines& w, unsigned char* s_own, Stage stage, Line line,
                                          Post post) {
  const int lane = threadIdx.x & 31;
  for (uint32_t base = w.e0; base < w.e1; base += kWChunk) {
#pragma unroll
    for (int k0 = 0; k0 < kWChunk; k0 += 32) {
      const uint32_t q = base + k0 + lane;
      if (q < w.e1) stage(k0 + lane, q);
    }
    __syncwarp();
    const uint32_t lo = max(w.beg, base), hi = min(w.end, base + kWChunk);
    for (uint32_t q = lo; q < hi; ++q) {
      if (s_own) s_own[q - base] = (unsigned char)lane;
      line((int)(q - base));
    }
    __syncwarp();
#pragma unroll
    for (int k0 = 0; k0 < kWChunk; k0 += 32) {
      const uint32_t q = base + k0 + lane;
      if (q < w.e1) post(k0 + lane, q);
    }
    __syncwarp();
  }
}
struct NoPost {
  __device__ void operator()(int, uint32_t) const {}
};

// ---------------------------------------------------------------- Sinkhorn (X3)

// Other-cloud index of an entry in the Sinkhorn loops: 16-bit copies when N, M <= 65536
// (k_rs_idx16): 6 instead of 8 bytes per entry and half-step, which keeps C4's CSR + CSC of a
// forward iteration (64 pairs x 65k entries) inside one die's L2 (ncu before: 46 MB from DRAM
// per half-step).
__device__ __forceinline__ uint32_t rs_cidx(const SparseArgs& A, size_t pb, uint32_t q) {
  return A.csc16 ? (uint32_t)A.csc16[pb + q] : A.csc_i[pb + q];
}
__device__ __forceinline__ uint32_t rs_ridx(const SparseArgs& A, size_t pb, uint32_t q) {
  return A.csr16 ? (uint32_t)A.csr16[pb + q] : (A.csr_jf[pb + q] & kIdxMask);
}
__global__ void k_rs_idx16(const SparseArgs A) {
  const int b = blockIdx.y;
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (A.cursor[b] > A.cap) return;
  const size_t pb = (size_t)b * A.cap;
  if (p < A.row_ptr[(size_t)b * (A.N + 1) + A.N]) A.csr16[pb + p] = (uint16_t)(A.csr_jf[pb + p] & kIdxMask);
  if (p < A.col_ptr[(size_t)b * (A.M + 1) + A.M]) A.csc16[pb + p] = (uint16_t)A.csc_i[pb + p];
}

// Per-group bodies (one warp, 32 consecutive lines of pair b; `line` = this lane's line),
// shared by the per-step kernels (row sharding: a collective between the steps) and the
// persistent single-GPU kernels further down.  sx / sy / sv / own: the warp's shared memory.

// sum over this rank's entries of column j of w[i] * P0_ij  (w: pair b's N-vector)
__device__ __forceinline__ float grp_colsum(const SparseArgs& A, int b, int j, const float* wb, float* sx,
                                            float* sy) {
  const size_t pb = (size_t)b * A.cap;
  const WarpLines wl = warp_lines(A.col_ptr + (size_t)b * (A.M + 1), j, A.M);
  float t = 0.f;
  warp_walk(wl, nullptr,
            [&](int k, uint32_t q) { sx[k] = wb[rs_cidx(A, pb, q)]; sy[k] = A.P0c[pb + q]; },
            [&](int k) { t = __fmaf_rn(sx[k], sy[k], t); }, NoPost{});
  return t;
}

// Column step of Eq. (3): b_j <- b_j / (b_j Q_j + eps)
__device__ __forceinline__ void grp_bstep(const SparseArgs& A, int b, int j, int l, float Q) {
  if (j >= A.M) return;
  float* bv = A.gvec + (size_t)b * 2 * (A.N + A.M) + A.N;
  float nb = 1.f;
  if (l > 0) {
    const float bj = bv[j];
    nb = __fdividef(bj, __fmaf_rn(bj, Q, A.eps));
  }
  bv[j] = nb;
  A.b_hist[((size_t)b * (A.L + 1) + l) * A.M + j] = nb;
}

// Row step of Eq. (4) (local rows): a_i <- a_i / (a_i R_i + eps), R_i = sum_j P0_ij b_j
__device__ __forceinline__ void grp_astep(const SparseArgs& A, int b, int i, int l, float* sx, float* sy) {
  const int N = A.N;
  const size_t pb = (size_t)b * A.cap;
  float* a = A.gvec + (size_t)b * 2 * (N + A.M);
  const float* bv = a + N;
  float na = 1.f;
  if (l > 0) {
    const WarpLines wl = warp_lines(A.row_ptr + (size_t)b * (N + 1), i, N);
    float Rs = 0.f;
    warp_walk(wl, nullptr,
              [&](int k, uint32_t q) { sx[k] = A.P0[pb + q]; sy[k] = bv[rs_ridx(A, pb, q)]; },
              [&](int k) { Rs = __fmaf_rn(sx[k], sy[k], Rs); }, NoPost{});
    if (i < N) {
      const float ai = a[i];
      na = __fdividef(ai, __fmaf_rn(ai, Rs, A.eps));
    }
  }
  if (i < N) {
    a[i] = na;
    A.a_hist[((size_t)b * (A.L + 1) + l) * N + i] = na;
  }
}

// Reverse of the row step at iteration l (local rows): Rbar, abar, P0bar += Rbar^l_i b^l_j
__device__ __forceinline__ void grp_rowrev(const SparseArgs& A, int b, int i, int l, float* sv,
                                           unsigned char* own) {
  const int N = A.N, M = A.M, L = A.L, lane = threadIdx.x & 31;
  const size_t pb = (size_t)b * A.cap;
  float* ab = A.gvec + (size_t)b * 2 * (N + M);
  float* rcur = ab + N + M;
  float Rb = 0.f;
  if (i < N) {
    const float al = A.a_hist[((size_t)b * (L + 1) + l) * N + i];
    const float alm = A.a_hist[((size_t)b * (L + 1) + l - 1) * N + i];
    const float r = al / alm;
    Rb = -ab[i] * al * al;
    ab[i] = ab[i] * A.eps * r * r;
    rcur[i] = Rb;
  }
  sv[lane] = Rb;
  const float* bl = A.b_hist + ((size_t)b * (L + 1) + l) * M;
  const WarpLines wl = warp_lines(A.row_ptr + (size_t)b * (N + 1), i, N);
  warp_walk(wl, own, [&](int, uint32_t) {}, [&](int) {},
            [&](int k, uint32_t q) { A.pbar[pb + q] += sv[own[k]] * bl[rs_ridx(A, pb, q)]; });
}

// Column step reverse on t = P0^T Rbar^l (summed over the ranks)
__device__ __forceinline__ void grp_colrev(const SparseArgs& A, int b, int j, int l, float t) {
  const int N = A.N, M = A.M, L = A.L;
  if (j >= M) return;
  float* bb = A.gvec + (size_t)b * 2 * (N + M) + N;
  float* qcur = bb + M + N;
  const float bsum = bb[j] + t;
  const float bl = A.b_hist[((size_t)b * (L + 1) + l) * M + j];
  const float blm = A.b_hist[((size_t)b * (L + 1) + l - 1) * M + j];
  const float r = bl / blm;
  bb[j] = bsum * A.eps * r * r;
  qcur[j] = -bsum * bl * bl;
}

// abar += P0 Qbar^l; P0bar_ij += Qbar^l_j a^{l-1}_i (local rows)
__device__ __forceinline__ void grp_rowrev2(const SparseArgs& A, int b, int i, int l, float* sx, float* sy,
                                            float* sv, unsigned char* own) {
  const int N = A.N, M = A.M, L = A.L, lane = threadIdx.x & 31;
  const size_t pb = (size_t)b * A.cap;
  float* ab = A.gvec + (size_t)b * 2 * (N + M);
  const float* qcur = ab + N + M + N;
  sv[lane] = i < N ? A.a_hist[((size_t)b * (L + 1) + l - 1) * N + i] : 0.f;
  const WarpLines wl = warp_lines(A.row_ptr + (size_t)b * (N + 1), i, N);
  float t = 0.f;
  warp_walk(wl, own,
            [&](int k, uint32_t q) { sx[k] = qcur[rs_ridx(A, pb, q)]; sy[k] = A.P0[pb + q]; },
            [&](int k) { t = __fmaf_rn(sx[k], sy[k], t); },
            [&](int k, uint32_t q) { A.pbar[pb + q] += sx[k] * sv[own[k]]; });
  if (i < N) ab[i] += t;
}

// Row step 2 of reverse iteration l (abar += P0 Qbar^l, P0bar += Qbar^l_j a^{l-1}_i) fused with
// the row step of iteration l - 1 (Rbar^{l-1} = -abar (a^{l-1})^2, P0bar += Rbar^{l-1}_i
// b^{l-1}_j), l > 1: a first walk folds the row sums, a second one applies BOTH P0bar terms in
// one read-modify-write (the two walks of grp_rowrev2 + grp_rowrev each rewrote P0bar).
__device__ __forceinline__ void grp_rowrev2_fused(const SparseArgs& A, int b, int i, int l, float* sx, float* sy,
                                                  float* sv, float* sv2, unsigned char* own) {
  const int N = A.N, M = A.M, L = A.L, lane = threadIdx.x & 31;
  const size_t pb = (size_t)b * A.cap;
  float* ab = A.gvec + (size_t)b * 2 * (N + M);
  float* rcur = ab + N + M;
  const float* qcur = ab + N + M + N;
  const float alm = i < N ? A.a_hist[((size_t)b * (L + 1) + l - 1) * N + i] : 0.f;  // a^{l-1}
  const WarpLines wl = warp_lines(A.row_ptr + (size_t)b * (N + 1), i, N);
  float t = 0.f;
  warp_walk(wl, nullptr,
            [&](int k, uint32_t q) { sx[k] = qcur[rs_ridx(A, pb, q)]; sy[k] = A.P0[pb + q]; },
            [&](int k) { t = __fmaf_rn(sx[k], sy[k], t); }, NoPost{});
  float Rb = 0.f;
  if (i < N) {
    const float abi = ab[i] + t;
    const float almm = A.a_hist[((size_t)b * (L + 1) + l - 2) * N + i];  // a^{l-2}
    const float r = alm / almm;
    Rb = -abi * alm * alm;
    ab[i] = abi * A.eps * r * r;
    rcur[i] = Rb;
  }
  sv[lane] = alm;
  sv2[lane] = Rb;
  const float* bprev = A.b_hist + ((size_t)b * (L + 1) + l - 1) * M;  // b^{l-1}
  __syncwarp();
  warp_walk(wl, own,
            [&](int k, uint32_t q) {
              const uint32_t j = rs_ridx(A, pb, q);
              sx[k] = qcur[j];
              sy[k] = bprev[j];
            },
            [&](int) {},
            [&](int k, uint32_t q) {
              const float p1 = __fmaf_rn(sx[k], sv[own[k]], A.pbar[pb + q]);
              A.pbar[pb + q] = __fmaf_rn(sv2[own[k]], sy[k], p1);
            });
}

// Shared memory of one 256-thread block of the group kernels.
struct GrpSmem {
  float x[kWWarps][kWChunk], y[kWWarps][kWChunk], v[kWWarps][32], v2[kWWarps][32];
  unsigned char own[kWWarps][kWChunk];
};

// ---- per-step kernels (grid (lines / 256, B); a collective may follow each one)

__global__ void __launch_bounds__(256) k_rs_colsum(const SparseArgs A, const float* __restrict__ w,
                                                   size_t w_stride, float* __restrict__ out, size_t out_stride) {
  __shared__ GrpSmem S;
  const int b = blockIdx.y, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = (blockIdx.x * kWWarps + wid) * 32 + lane;
  if (A.cursor[b] > A.cap || j - lane >= A.M) return;  // warp-uniform
  const float t = grp_colsum(A, b, j, w + (size_t)b * w_stride, S.x[wid], S.y[wid]);
  if (j < A.M) out[(size_t)b * out_stride + j] = t;
}

// Single GPU (world 1: nothing to all-reduce between them): the column sum and the column step
// of Eq. (3) in one launch (the column step needs only its own column's sum).
__global__ void __launch_bounds__(256) k_rs_colsum_bstep(const SparseArgs A, int l) {
  __shared__ GrpSmem S;
  const int b = blockIdx.y, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = (blockIdx.x * kWWarps + wid) * 32 + lane;
  if (A.cursor[b] > A.cap || j - lane >= A.M) return;  // warp-uniform
  const float t = grp_colsum(A, b, j, A.gvec + (size_t)b * 2 * (A.N + A.M), S.x[wid], S.y[wid]);
  grp_bstep(A, b, j, l, t);
}

// Column step of Eq. (3) on the all-reduced Q (every rank).
__global__ void k_rs_bstep(const SparseArgs A, int l, const float* __restrict__ Q) {
  const int b = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
  grp_bstep(A, b, j, l, (l > 0 && j < A.M) ? Q[(size_t)b * A.M + j] : 0.f);
}

__global__ void __launch_bounds__(256) k_rs_astep(const SparseArgs A, int l) {
  __shared__ GrpSmem S;
  const int b = blockIdx.y, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = (blockIdx.x * kWWarps + wid) * 32 + lane;
  if (A.cursor[b] > A.cap || i - lane >= A.N) return;  // warp-uniform
  grp_astep(A, b, i, l, S.x[wid], S.y[wid]);
}

// This rank's part of loss_b = sum_i a_i sum_j P0_ij b_j c_ij: per-block partials in fp64
// (k_rs_loss_part, grid over rows), then a fixed-order per-pair sum (k_rs_loss_fin).
constexpr int kLossThreads = 256;
__global__ void __launch_bounds__(kLossThreads) k_rs_loss_part(const SparseArgs A, double* __restrict__ part) {
  __shared__ double red[kLossThreads / 32];
  const int b = blockIdx.y, N = A.N;
  const int i = blockIdx.x * kLossThreads + threadIdx.x;
  double acc = 0.0;
  if (A.cursor[b] <= A.cap && i < N) {
    const size_t pb = (size_t)b * A.cap;
    const unsigned* rp = A.row_ptr + (size_t)b * (N + 1);
    const float* a = A.gvec + (size_t)b * 2 * (N + A.M);
    const float* bv = a + N;
    float t = 0.f;
    for (uint32_t p = rp[i]; p < rp[i + 1]; ++p)
      t = __fmaf_rn(__fmul_rn(A.P0[pb + p], bv[A.csr_jf[pb + p] & kIdxMask]), A.cs[pb + p], t);
    acc = (double)a[i] * (double)t;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kLossThreads / 32; ++w) t += red[w];
    part[(size_t)b * gridDim.x + blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(256) k_rs_loss_fin(const SparseArgs A, const double* __restrict__ part, int nblk) {
  __shared__ double red[8];
  const int b = blockIdx.x;
  double acc = 0.0;
  for (int k = threadIdx.x; k < nblk; k += blockDim.x) acc += part[(size_t)b * nblk + k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    A.loss[b] = A.cursor[b] > A.cap ? __int_as_float(0x7fc00000) : (float)t;
  }
}

// ---------------------------------------------------------------- backward

// abar_i = gl sum_j P0 b^L c (local rows); P0bar_ij = gl a^L_i b^L_j c_ij (direct term).
__global__ void k_rs_bwd_init_rows(const SparseArgs A) {
  const int b = blockIdx.y, N = A.N, M = A.M, L = A.L;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N || A.cursor[b] > A.cap) return;
  const size_t pb = (size_t)b * A.cap;
  const unsigned* rp = A.row_ptr + (size_t)b * (N + 1);
  const float* aL = A.a_hist + ((size_t)b * (L + 1) + L) * N;
  const float* bL = A.b_hist + ((size_t)b * (L + 1) + L) * M;
  const float gl = A.grad_loss[b];
  double t = 0.0;
  for (uint32_t p = rp[i]; p < rp[i + 1]; ++p) {
    const uint32_t j = A.csr_jf[pb + p] & kIdxMask;
    t += (double)A.P0[pb + p] * (double)bL[j] * (double)A.cs[pb + p];
    A.pbar[pb + p] = gl * aL[i] * bL[j] * A.cs[pb + p];
  }
  A.gvec[(size_t)b * 2 * (N + M) + i] = (float)((double)gl * t);  // abar
}

// Partial bbar_j = sum over local entries of a^L_i P0_ij c_ij (times gl after the reduce).
__global__ void k_rs_bwd_init_cols(const SparseArgs A, float* __restrict__ out) {
  const int b = blockIdx.y, N = A.N, M = A.M, L = A.L;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M || A.cursor[b] > A.cap) return;
  const size_t pb = (size_t)b * A.cap;
  const unsigned* cp = A.col_ptr + (size_t)b * (M + 1);
  const float* aL = A.a_hist + ((size_t)b * (L + 1) + L) * N;
  float t = 0.f;
  for (uint32_t q = cp[j]; q < cp[j + 1]; ++q)
    t = __fmaf_rn(aL[A.csc_i[pb + q]] * A.P0c[pb + q], A.cs[pb + A.csc_perm[pb + q]], t);
  out[(size_t)b * M + j] = t;
}

__global__ void k_rs_bwd_set_bbar(const SparseArgs A, const float* __restrict__ red) {
  const int b = blockIdx.y, N = A.N, M = A.M;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M) return;
  A.gvec[(size_t)b * 2 * (N + M) + N + j] = A.grad_loss[b] * red[(size_t)b * M + j];
}

__global__ void __launch_bounds__(256) k_rs_bwd_rowrev(const SparseArgs A, int l) {
  __shared__ GrpSmem S;
  const int b = blockIdx.y, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = (blockIdx.x * kWWarps + wid) * 32 + lane;
  if (A.cursor[b] > A.cap || i - lane >= A.N) return;  // warp-uniform
  grp_rowrev(A, b, i, l, S.v[wid], S.own[wid]);
}

// Single GPU: P0^T Rbar^l and the column step reverse in one launch.
__global__ void __launch_bounds__(256) k_rs_colsum_colrev(const SparseArgs A, int l) {
  __shared__ GrpSmem S;
  const int b = blockIdx.y, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = (blockIdx.x * kWWarps + wid) * 32 + lane;
  if (A.cursor[b] > A.cap || j - lane >= A.M) return;  // warp-uniform
  const float t = grp_colsum(A, b, j, A.gvec + (size_t)b * 2 * (A.N + A.M) + A.N + A.M, S.x[wid], S.y[wid]);
  grp_colrev(A, b, j, l, t);
}

__global__ void k_rs_bwd_colrev(const SparseArgs A, int l, const float* __restrict__ t) {
  const int b = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < A.M) grp_colrev(A, b, j, l, t[(size_t)b * A.M + j]);
}

// ---- NVLS variants of the X3 reductions (k_nvls.cuh): the producer writes this rank's
// column sums into its copy of the team buffer and every CTA bumps every rank's flag once (no
// early return: the consumer counts all CTAs of all ranks); the consumer waits for the count
// and reads each sum over the ranks with one multimem.ld_reduce.
template <bool kMc>
__global__ void __launch_bounds__(256) k_rs_colsum_nvls(const SparseArgs A, const float* __restrict__ w,
                                                        size_t w_stride, float* __restrict__ part,
                                                        unsigned* flag_mc) {
  __shared__ GrpSmem S;
  const int b = blockIdx.y, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = (blockIdx.x * kWWarps + wid) * 32 + lane;
  if (A.cursor[b] <= A.cap && j - lane < A.M) {  // warp-uniform
    const float t = grp_colsum(A, b, j, w + (size_t)b * w_stride, S.x[wid], S.y[wid]);
    if (j < A.M) part[(size_t)b * A.M + j] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) nvls_signal<kMc>(flag_mc);
}
// Eq. (3) column step on the sums over the ranks
template <bool kMc>
__global__ void k_rs_bstep_nvls(const SparseArgs A, int l, const float* part_mc, const unsigned* flag_uc,
                                unsigned target) {
  if (threadIdx.x == 0) nvls_wait(flag_uc, target);
  __syncthreads();
  const int b = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < A.M) grp_bstep(A, b, j, l, nvls_ld_sum<kMc>(part_mc + (size_t)b * A.M + j));
}
// Reverse column step on t = P0^T Rbar^l summed over the ranks
template <bool kMc>
__global__ void k_rs_bwd_colrev_nvls(const SparseArgs A, int l, const float* part_mc, const unsigned* flag_uc,
                                     unsigned target) {
  if (threadIdx.x == 0) nvls_wait(flag_uc, target);
  __syncthreads();
  const int b = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < A.M) grp_colrev(A, b, j, l, nvls_ld_sum<kMc>(part_mc + (size_t)b * A.M + j));
}

__global__ void __launch_bounds__(256) k_rs_bwd_rowrev2(const SparseArgs A, int l) {
  __shared__ GrpSmem S;
  const int b = blockIdx.y, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = (blockIdx.x * kWWarps + wid) * 32 + lane;
  if (A.cursor[b] > A.cap || i - lane >= A.N) return;  // warp-uniform
  grp_rowrev2(A, b, i, l, S.x[wid], S.y[wid], S.v[wid], S.own[wid]);
}

// Row step 2 of reverse iteration l fused with the row step of iteration l - 1 (both touch
// only the warp's own rows; no collective between them): one launch per iteration fewer.
__global__ void __launch_bounds__(256) k_rs_bwd_rowrev2_rowrev(const SparseArgs A, int l, int env_fused_rowrev) {
  __shared__ GrpSmem S;
  const int b = blockIdx.y, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = (blockIdx.x * kWWarps + wid) * 32 + lane;
  if (A.cursor[b] > A.cap || i - lane >= A.N) return;  // warp-uniform
  if (l > 1 && env_fused_rowrev) {
    grp_rowrev2_fused(A, b, i, l, S.x[wid], S.y[wid], S.v[wid], S.v2[wid], S.own[wid]);
    return;
  }
  grp_rowrev2(A, b, i, l, S.x[wid], S.y[wid], S.v[wid], S.own[wid]);
  if (l > 1) {
    __syncwarp();  // P0bar entries and the warp's scratch are shared by the lanes of both walks
    grp_rowrev(A, b, i, l - 1, S.v[wid], S.own[wid]);
  }
}

// Row softmax reverse (local rows).
__global__ void __launch_bounds__(kRsThreads) k_rs_row_soft(const SparseArgs A) {
  __shared__ uint32_t s_long[kLongCap];
  __shared__ int s_n;
  const int b = blockIdx.y;
  if (A.cursor[b] > A.cap) return;
  const Slice s = block_slice(A.N);
  const LongList ll = collect_long(A.row_ptr + (size_t)b * (A.N + 1), s, s_long, &s_n);
  row_soft_rev<1, 8>(A, b, s, ll);
  row_soft_rev<32, 1>(A, b, s, ll);
}

// Column softmax reverse, partial sums over local entries (two passes, each all-reduced):
// pass 0: S_j = sum P_col Pbar/2;  pass 1: (sum zbar, -sum zbar (c - m)) with zbar = P (Pbar/2 - S).
__global__ void k_rs_col_soft_part(const SparseArgs A, int pass, int rank) {
  const int b = blockIdx.y, M = A.M;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M || A.cursor[b] > A.cap) return;
  const size_t pb = (size_t)b * A.cap;
  const unsigned* cp = A.col_ptr + (size_t)b * (M + 1);
  const LineB lb = A.colB[(size_t)b * M + j];
  float* red = A.colred + ((size_t)b * M + j) * 3;
  if (pass == 0) {
    float S = 0.f;
    for (uint32_t q = cp[j]; q < cp[j + 1]; ++q) {
      const uint32_t p = A.csc_perm[pb + q];
      if (A.csr_jf[pb + p] & kFlagCol) S = __fmaf_rn(A.pcol[pb + p], 0.5f * A.pbar[pb + p], S);
    }
    red[0] = S; red[1] = 0.f; red[2] = 0.f;
  } else {
    const float S = red[0];
    float szb = 0.f, Tb = 0.f;
    for (uint32_t q = cp[j]; q < cp[j + 1]; ++q) {
      const uint32_t p = A.csc_perm[pb + q];
      if (!(A.csr_jf[pb + p] & kFlagCol)) continue;
      const float zb = A.pcol[pb + p] * (0.5f * A.pbar[pb + p] - S);
      szb += zb;
      Tb -= zb * (A.cs[pb + p] - lb.m);
    }
    red[0] = rank == 0 ? S : 0.f;  // S is already global: keep it through the next all-reduce
    red[1] = szb;
    red[2] = Tb;
  }
}

__global__ void k_rs_col_soft_fin(const SparseArgs A) {
  const int b = blockIdx.y, M = A.M;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M) return;
  const LineB lb = A.colB[(size_t)b * M + j];
  const float* red = A.colred + ((size_t)b * M + j) * 3;
  LineBack out = {0.f, 0.f, 0.f, 0.f};
  if (!(lb.flags & kLineK1)) {
    const double mbar = (double)lb.T * (double)red[1];
    const double gbar = (lb.flags & kLineClamped) ? 0.0 : -(double)red[2] * (double)lb.T / (double)lb.g;
    out = {red[0], (float)(mbar - gbar), (float)gbar, lb.T};
  }
  A.colback[(size_t)b * M + j] = out;
}

__global__ void __launch_bounds__(256, 3) k_rs_grad(const SparseArgs A) {
  __shared__ uint32_t s_long[kLongCap];
  __shared__ int s_n;
  const int b = blockIdx.y;
  const Slice s = block_slice(A.N);
  if (A.cursor[b] > A.cap) {
    const float nan = __int_as_float(0x7fc00000);
    for (int i = s.lo + threadIdx.x; i < s.hi; i += blockDim.x) {
      float* g = A.grad_pred + ((size_t)b * A.N + i) * 3;
      g[0] = nan; g[1] = nan; g[2] = nan;
    }
    return;
  }
  const LongList ll = collect_long(A.row_ptr + (size_t)b * (A.N + 1), s, s_long, &s_n);
  grad_rows<1, 4>(A, b, s, ll);
  grad_rows<32, 1>(A, b, s, ll);
}

}  // namespace apml
