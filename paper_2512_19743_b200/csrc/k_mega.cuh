// k_mega.cuh -- the O(nnz) sparse stage of one pair as ONE kernel per direction of the pass,
// run by a thread-block CLUSTER per pair.
//
// Every CTA of the cluster owns a contiguous slice of the pair's rows and of its columns.
// Phases are separated by cluster barriers (barrier.cluster release/acquire), so the whole
// sparse forward (or backward) of a batch is a single launch of B x CL CTAs instead of ~10
// grid-wide launches:
//
//   forward  k_sparse_fwd:  scan (cluster-wide, slice totals exchanged through DSMEM) ->
//            scatter -> rank-sort rows -> rank-sort columns (CSR + CSC) ->
//            row softmax on the kept support -> column softmax +
//            symmetrisation P0 = (P_row + P_col)/2 -> Sinkhorn, L_iter x
//            {Eq. (3), Eq. (4)} -> loss.
//   backward k_sparse_bwd:  reverse Sinkhorn with P0bar accumulated in shared memory ->
//            row softmax reverse -> column softmax reverse -> cbar + Eq. (5).
//
// Sinkhorn runs in scaling-vector form P = diag(a) P0 diag(b) (see k_sinkhorn.cuh).  Each
// CTA keeps a full REPLICA of the current scaling vector (a, b forward; Rbar^l, Qbar^l
// backward) in its shared memory and, after computing its own slice, pushes the new values
// into every replica of the cluster through distributed shared memory (st.shared::cluster);
// all gathers of a half-step are then local shared-memory reads.  Its own CSR / CSC slice
// (16-bit indices when N, M <= 65536) and P0 also sit in shared memory.  When the replicas do
// not fit (N + M too large) they live in global memory, and a CTA whose own slice does not
// fit reads it from global memory -- same loop, L2-resident operands.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace apml {

namespace cg = cooperative_groups;

constexpr int kMegaThreads = 512;
constexpr int kMaxCluster = 16;

struct SparseArgs {
  int N, M, L, full;
  uint32_t cap;    // per-pair stride of the per-entry arrays (>= every pair's emitted count, or
                   // the pair is skipped as overflowed)
  uint32_t cap_e;  // per-pair stride of the emit buffer (the emit capacity, >= cap)
  float eps, eps_dist;
  const float4* pred4;
  const float4* gt4;
  const LineA* rowA;
  const LineB* rowB;
  const LineA* colA;
  const LineB* colB;
  const uint2* ebuf;  // [B][cap_e]
  const unsigned* cursor;
  unsigned* row_cnt;  // counts from k_emit; zeroed here and reused as fill cursors
  unsigned* col_cnt;
  unsigned* row_ptr;
  unsigned* col_ptr;
  uint32_t* csr_t;
  uint32_t* csc_t;
  uint32_t* inv;
  uint32_t* csr_jf;
  uint32_t* csc_i;
  uint32_t* csc_perm;
  uint32_t* csc_if;  // CSC order (k_sparse_fwd2): i | flags, c, P_col
  uint16_t* csr16;   // grid path, N, M <= 65536: 16-bit other-cloud indices for Sinkhorn (or NULL)
  uint16_t* csc16;
  float* csc_c;
  float* csc_pc;
  float* d2s;
  float* cs;
  float* prow;
  float* pcol;
  float* P0;
  float* P0c;
  float* pbar;
  int2* rowidx;
  int2* colidx;
  float* a_hist;  // [B][L+1][N]
  float* b_hist;  // [B][L+1][M]
  float* gvec;    // [B][2 (N + M)] replica scratch when replicas are not in shared memory
  LineBack* rowback;
  LineBack* colback;
  float* loss;
  const float* grad_loss;
  float* grad_pred;
  float* gw;       // optional [B][cap]: Eq. (5) weight cbar / (c + eps_dist) per CSR entry (grad_gt)
  float* grad_gt;  // optional [B][M][3]
  size_t smem_bytes;
  int rep_smem;
  int bhs_stage;  // k_sparse_bwd2: stage the whole b history in shared memory (APML_BHS, default 1)
  unsigned long long* dbg;  // optional phase timestamps [grid][16] (APML_PHASES=1), else NULL
  // row-sharded mode (k_rowshard.cuh): global index of local row 0, column partial sums /
  // argmin candidates exchanged through the caller's collectives
  int row_offset;
  float* colred;  // [B][M][3]
  int* cand;      // [B][M][3]
  // Morton-relabelled index space (culled sweeps, one GPU per cloud): every line index in
  // the sparse stage is a SORTED position; pperm / gperm [B][perm_np / perm_mp] give the
  // original index (lines are still ordered, and ties broken, by ORIGINAL index, so the
  // results equal the unrelabelled ones), ipperm [B][N] the inverse for pred.  NULL: identity.
  const int* pperm;
  const int* gperm;
  const int* ipperm;
  int perm_np, perm_mp;
};

__device__ __forceinline__ const uint2* ebuf_of(const SparseArgs& A, int b) { return A.ebuf + (size_t)b * A.cap_e; }

__device__ __forceinline__ uint32_t orig_row(const SparseArgs& A, int b, uint32_t i) {
  return A.pperm ? (uint32_t)A.pperm[(size_t)b * A.perm_np + i] : i;
}
__device__ __forceinline__ uint32_t orig_col(const SparseArgs& A, int b, uint32_t j) {
  return A.gperm ? (uint32_t)A.gperm[(size_t)b * A.perm_mp + j] : j;
}

__device__ __forceinline__ void phase(const SparseArgs& A, int k) {
  if (A.dbg && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    A.dbg[blockIdx.x * 16 + k] = t;
  }
}

// Cluster barrier, or a CTA barrier when the cluster is a single CTA (barrier.cluster also
// invalidates L1, which a single CTA does not need: its own global writes are coherent to it).
__device__ __forceinline__ void csync(cg::cluster_group& cl) {
  if (cl.num_blocks() == 1) __syncthreads();
  else cl.sync();
}

struct Slice {
  int lo, hi;
};
// Slice boundaries are multiples of 4 lines so that every slice of a replica is 16-byte
// aligned for the bulk DSMEM exchange.
__device__ __forceinline__ int slice_lo(int n, int rank, int cl) {
  return rank >= cl ? n : (int)(((long long)n * rank / cl) & ~3LL);
}
__device__ __forceinline__ Slice slice_of(int n, int rank, int cl) {
  return Slice{slice_lo(n, rank, cl), rank + 1 >= cl ? n : slice_lo(n, rank + 1, cl)};
}

// ---------------------------------------------------------------- CSR / CSC construction

// Exclusive scan of cnt[lo, hi) (block-wide) offset by the totals of lower-ranked slices;
// writes ptr[lo, hi) (+ ptr[n] by the last rank) and zeroes cnt[lo, hi) (fill cursors).
__device__ void cluster_scan(cg::cluster_group& cl, unsigned* cnt, unsigned* ptr, int n, Slice s,
                             unsigned* s_tot, unsigned* s_warp) {
  const int rank = cl.block_rank(), CL = cl.num_blocks();
  const int len = s.hi - s.lo;
  const int per = (len + blockDim.x - 1) / blockDim.x;
  const int beg = s.lo + threadIdx.x * per, end = min(s.hi, beg + per);
  unsigned sum = 0;
  for (int k = beg; k < end; ++k) sum += cnt[k];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) s_warp[w] = inc;
  __syncthreads();
  if (w == 0) {
    unsigned t = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += v;
    }
    s_warp[lane] = t;
  }
  __syncthreads();
  const unsigned slice_total = s_warp[(blockDim.x >> 5) - 1];
  if (threadIdx.x < CL) {
    unsigned* remote = cl.map_shared_rank(s_tot, (int)threadIdx.x);
    remote[rank] = slice_total;
  }
  csync(cl);
  unsigned off = 0;
  for (int r = 0; r < rank; ++r) off += s_tot[r];
  unsigned run = off + inc - sum + (w ? s_warp[w - 1] : 0u);
  for (int k = beg; k < end; ++k) {
    const unsigned v = cnt[k];
    ptr[k] = run;
    run += v;
    cnt[k] = 0u;
  }
  if (rank == CL - 1 && threadIdx.x == 0) ptr[n] = off + slice_total;
  __syncthreads();  // s_tot / s_warp reused by the next scan
}

constexpr uint32_t kRegLine = 16;  // lines up to this length are sorted in registers by one thread
constexpr int kLongCap = 1024;     // per-CTA list of longer lines (warp per line)

// The two long-line lists of a CTA (rows, columns) in ONE static shared allocation, shared by
// every kernel body that calls this (the fused forward + backward reuses it: 8 KB once).
__device__ __forceinline__ uint32_t* long_lists() {
  __shared__ uint32_t buf[2 * kLongCap];
  return buf;
}

// The lines of a slice longer than kRegLine, collected once so that warp-per-line passes do
// not walk (and load the offsets of) every line of the slice.
struct LongList {
  const uint32_t* idx;
  int n, lo, hi;
  bool all;  // list overflowed: walk the whole slice
  __device__ __forceinline__ int count() const { return all ? hi - lo : n; }
  __device__ __forceinline__ int line(int k) const { return all ? lo + k : (int)idx[k]; }
};

__device__ LongList collect_long(const unsigned* ptr, Slice s, uint32_t* list, int* cnt, uint32_t th = kRegLine) {
  if (threadIdx.x == 0) *cnt = 0;
  __syncthreads();
  for (int i = s.lo + threadIdx.x; i < s.hi; i += blockDim.x)
    if (ptr[i + 1] - ptr[i] > th) {
      const int k = atomicAdd(cnt, 1);
      if (k < kLongCap) list[k] = (uint32_t)i;
    }
  __syncthreads();
  const int n = *cnt;
  return LongList{list, n < kLongCap ? n : kLongCap, s.lo, s.hi, n > kLongCap};
}

// G == 1: thread per line over the whole slice (short lines are its business);
// G == 32: warp per line over the long-line list.
#define APML_FOR_LINES(G, s, ll, var)                                                              \
  for (int _k = (G == 1 ? (int)threadIdx.x : (int)(threadIdx.x >> 5)),                             \
           _n = (G == 1 ? (s).hi - (s).lo : (ll).count());                                         \
       _k < _n; _k += (G == 1 ? (int)blockDim.x : (int)(blockDim.x >> 5)))                         \
    if (const int var = (G == 1 ? (s).lo + _k : (ll).line(_k)); true)

// Warp per line rank sort of the lines longer than TH (keys inside a line are distinct).
template <bool kRows, uint32_t TH = kRegLine>
__device__ void sort_lines(const SparseArgs& A, int b, Slice s, const LongList& ll) {
  const size_t pb = (size_t)b * A.cap;
  const int n = kRows ? A.N : A.M;
  const unsigned* ptr = (kRows ? A.row_ptr : A.col_ptr) + (size_t)b * (n + 1);
  const uint32_t* seg_t = (kRows ? A.csr_t : A.csc_t) + pb;
  const uint2* e = ebuf_of(A, b);
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  (void)nw;
  APML_FOR_LINES(32, s, ll, line) {
    const uint32_t beg = ptr[line], end = ptr[line + 1], L = end - beg;
    if (L <= TH) continue;
    auto key_of = [&](uint32_t t) -> uint32_t {  // ORIGINAL index of the other cloud
      return kRows ? orig_col(A, b, e[t].y & kIdxMask) : orig_row(A, b, e[t].x);
    };
    auto place = [&](uint32_t t, uint32_t rank) {
      const uint32_t pos = beg + rank;
      if (kRows) {
        A.csr_jf[pb + pos] = e[t].y;
        A.inv[pb + t] = pos;
      } else {
        A.csc_i[pb + pos] = e[t].x;
        A.csc_perm[pb + pos] = A.inv[pb + t];
      }
    };
    if (L <= 32) {
      const uint32_t t = lane < (int)L ? seg_t[beg + lane] : 0u;
      const uint32_t key = lane < (int)L ? key_of(t) : 0xffffffffu;
      uint32_t rank = 0;
      for (uint32_t k = 0; k < L; ++k) rank += (__shfl_sync(0xffffffffu, key, k) < key) ? 1u : 0u;
      if (lane < (int)L) place(t, rank);
    } else {
      for (uint32_t q = beg + lane; q < end; q += 32) {
        const uint32_t t = seg_t[q];
        const uint32_t key = key_of(t);
        uint32_t rank = 0;
        for (uint32_t f = beg; f < end; ++f) rank += (key_of(seg_t[f]) < key) ? 1u : 0u;
        place(t, rank);
      }
    }
  }
}

// ---------------------------------------------------------------- normalisation

// Deterministic sum over a group of G lanes (butterfly: every lane ends with the same bits).
template <int G, typename T>
__device__ __forceinline__ T gsum(T v) {
  if (G > 1) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;
}

// First and second match in sorted line order (argmin = first entry with d2 == m2; second
// argmin = first other entry with d2 == s2), warp-cooperative over a 32-entry chunk.
__device__ __forceinline__ void first_two(unsigned bal_m, unsigned bal_s, int& ka, int& kb, int chunk0) {
  if (ka < 0 && bal_m) {
    const int f = __ffs(bal_m) - 1;
    ka = chunk0 + f;
    bal_s &= ~(1u << f);
  }
  if (kb < 0 && bal_s) kb = chunk0 + __ffs(bal_s) - 1;
}

// Row softmax on the kept support for rows longer than kRegLine: one warp per row, 32
// entries per step (the short rows are done in registers by row_sort_norm_regs).
template <uint32_t TH = kRegLine>
__device__ void row_norm(const SparseArgs& A, int b, Slice s, const LongList& ll) {
  const int N = A.N, M = A.M;
  const size_t pb = (size_t)b * A.cap;
  const unsigned* rp = A.row_ptr + (size_t)b * (N + 1);
  const int lane = threadIdx.x & 31;
  APML_FOR_LINES(32, s, ll, i) {
    const uint32_t beg = rp[i], end = rp[i + 1];
    if (end - beg <= TH) continue;
    const float4 x = A.pred4[(size_t)b * N + i];
    const LineA la = A.rowA[(size_t)b * N + i];
    const LineB lb = A.rowB[(size_t)b * N + i];
    int ka = -1, kb = -1;
    float Z = 0.f;
    for (uint32_t p0 = beg; p0 < end; p0 += 32) {
      const uint32_t p = p0 + lane;
      const bool v = p < end;
      uint32_t jf = 0;
      float d2 = 0.f, sv = 0.f;
      if (v) {
        jf = A.csr_jf[pb + p];
        const float4 y = A.gt4[(size_t)b * M + (jf & kIdxMask)];
        d2 = dist2(x.x, x.y, x.z, y.x, y.y, y.z);
        const float c = __fsqrt_rn(d2);
        A.d2s[pb + p] = d2;
        A.cs[pb + p] = c;
        if (jf & kFlagRow) sv = (lb.flags & kLineK1) ? 1.f : expf(-lb.T * (c - lb.m));
        A.prow[pb + p] = sv;
        Z += sv;
      }
      first_two(__ballot_sync(0xffffffffu, v && d2 == la.m2), __ballot_sync(0xffffffffu, v && d2 == la.s2),
                ka, kb, (int)(p0 - beg));
    }
    const float iz = 1.f / gsum<32>(Z);
    for (uint32_t p = beg + lane; p < end; p += 32) A.prow[pb + p] *= iz;
    if (lane == 0) {
      const int ja = ka >= 0 ? (int)(A.csr_jf[pb + beg + ka] & kIdxMask) : -1;
      const int jb = kb >= 0 ? (int)(A.csr_jf[pb + beg + kb] & kIdxMask) : -1;
      A.rowidx[(size_t)b * N + i] = make_int2(ja, jb);
    }
  }
}

// Column softmax + symmetrisation for columns longer than kRegLine (warp per column).
__device__ void col_norm(const SparseArgs& A, int b, Slice s, const LongList& ll) {
  const int M = A.M;
  const size_t pb = (size_t)b * A.cap;
  const unsigned* cp = A.col_ptr + (size_t)b * (M + 1);
  const int lane = threadIdx.x & 31;
  APML_FOR_LINES(32, s, ll, j) {
    const uint32_t beg = cp[j], end = cp[j + 1];
    if (end - beg <= kRegLine) continue;
    const LineA la = A.colA[(size_t)b * M + j];
    const LineB lb = A.colB[(size_t)b * M + j];
    int ka = -1, kb = -1;
    float Z = 0.f;
    for (uint32_t q0 = beg; q0 < end; q0 += 32) {
      const uint32_t q = q0 + lane;
      const bool v = q < end;
      float d2 = 0.f;
      if (v) {
        const uint32_t p = A.csc_perm[pb + q];
        d2 = A.d2s[pb + p];
        if (A.csr_jf[pb + p] & kFlagCol) Z += (lb.flags & kLineK1) ? 1.f : expf(-lb.T * (A.cs[pb + p] - lb.m));
      }
      first_two(__ballot_sync(0xffffffffu, v && d2 == la.m2), __ballot_sync(0xffffffffu, v && d2 == la.s2),
                ka, kb, (int)(q0 - beg));
    }
    const float iz = 1.f / gsum<32>(Z);
    for (uint32_t q = beg + lane; q < end; q += 32) {
      const uint32_t p = A.csc_perm[pb + q];
      float pc = 0.f;
      if (A.csr_jf[pb + p] & kFlagCol)
        pc = ((lb.flags & kLineK1) ? 1.f : expf(-lb.T * (A.cs[pb + p] - lb.m))) * iz;
      A.pcol[pb + p] = pc;
      const float p0 = 0.5f * (A.prow[pb + p] + pc);
      A.P0[pb + p] = p0;
      A.P0c[pb + q] = p0;
    }
    if (lane == 0) {
      const int ia = ka >= 0 ? (int)A.csc_i[pb + beg + ka] : -1;
      const int ib = kb >= 0 ? (int)A.csc_i[pb + beg + kb] : -1;
      A.colidx[(size_t)b * M + j] = make_int2(ia, ib);
    }
  }
}

// Register paths (thread per line, length <= kRegLine), in two passes that each keep at
// most ~3 arrays of kRegLine registers live (no spills under the 128-register cap):
//   pass 1  the entries, in the order the scatter left them (csr_t / csc_t, arbitrary), are
//           ranked in the line by ORIGINAL index of the other cloud and their index arrays
//           written at beg + rank (CSR / CSC order);
//   pass 2  the line is re-read in sorted order (same thread: its own stores are visible),
//           every gather is issued before any store (stores could alias them as far as the
//           compiler knows, which would serialise one L2 round trip per entry), then the
//           softmax runs in sorted order (deterministic sums; argmin / second argmin = the
//           first matches, R12).

// Row softmax on the kept support (S5) + CSR order by j.
template <uint32_t TH = kRegLine>
__device__ void row_sort_norm_regs(const SparseArgs& A, int b, Slice s) {
  const int N = A.N, M = A.M;
  const size_t pb = (size_t)b * A.cap;
  const unsigned* rp = A.row_ptr + (size_t)b * (N + 1);
  for (int i = s.lo + threadIdx.x; i < s.hi; i += blockDim.x) {
    const uint32_t beg = rp[i], L = rp[i + 1] - beg;
    if (L > TH) continue;
    const float4 x = A.pred4[(size_t)b * N + i];
    const LineA la = A.rowA[(size_t)b * N + i];
    const LineB lb = A.rowB[(size_t)b * N + i];
    {
      uint32_t t[TH], jf[TH], ok[TH];
#pragma unroll
      for (uint32_t k = 0; k < TH; ++k) t[k] = k < L ? A.csr_t[pb + beg + k] : 0u;
#pragma unroll
      for (uint32_t k = 0; k < TH; ++k) jf[k] = k < L ? ebuf_of(A, b)[t[k]].y : 0u;
#pragma unroll
      for (uint32_t k = 0; k < TH; ++k) ok[k] = k < L ? orig_col(A, b, jf[k] & kIdxMask) : 0xffffffffu;
#pragma unroll
      for (uint32_t k = 0; k < TH; ++k) {
        uint32_t r = 0;
#pragma unroll
        for (uint32_t f = 0; f < TH; ++f) r += (ok[f] < ok[k]) ? 1u : 0u;
        if (k < L) {  // padded entries (key = ~0) never precede a real key
          A.csr_jf[pb + beg + r] = jf[k];
          A.inv[pb + t[k]] = beg + r;
        }
      }
    }
    uint32_t sj[TH];
#pragma unroll
    for (uint32_t r = 0; r < TH; ++r) sj[r] = r < L ? A.csr_jf[pb + beg + r] : 0u;
    float d2v[TH], cv[TH];
#pragma unroll
    for (uint32_t r = 0; r < TH; ++r) {
      if (r < L) {
        const float4 y = A.gt4[(size_t)b * M + (sj[r] & kIdxMask)];
        d2v[r] = dist2(x.x, x.y, x.z, y.x, y.y, y.z);
        cv[r] = __fsqrt_rn(d2v[r]);
      }
    }
    int ia = -1, ib = -1;
    float Z = 0.f;
#pragma unroll
    for (uint32_t r = 0; r < TH; ++r) {
      if (r < L) {
        const int j = (int)(sj[r] & kIdxMask);
        if (ia < 0 && d2v[r] == la.m2) ia = j;
        else if (ib < 0 && d2v[r] == la.s2) ib = j;
        float sv = 0.f;
        if (sj[r] & kFlagRow) {
          sv = (lb.flags & kLineK1) ? 1.f : expf(-lb.T * (cv[r] - lb.m));
          Z += sv;
        }
        A.d2s[pb + beg + r] = d2v[r];
        A.cs[pb + beg + r] = cv[r];
        cv[r] = sv;  // reuse: unnormalised similarity
      }
    }
    const float iz = 1.f / Z;
#pragma unroll
    for (uint32_t r = 0; r < TH; ++r)
      if (r < L) A.prow[pb + beg + r] = cv[r] * iz;
    A.rowidx[(size_t)b * N + i] = make_int2(ia, ib);
  }
}

// Column softmax + symmetrisation P0 = (P_row + P_col)/2 in both orders + CSC
// order by i (+ CSR position of each entry).
__device__ void col_sort_norm_regs(const SparseArgs& A, int b, Slice s) {
  const int M = A.M;
  const size_t pb = (size_t)b * A.cap;
  const unsigned* cp = A.col_ptr + (size_t)b * (M + 1);
  for (int j = s.lo + threadIdx.x; j < s.hi; j += blockDim.x) {
    const uint32_t beg = cp[j], L = cp[j + 1] - beg;
    if (L > kRegLine) continue;
    const LineA la = A.colA[(size_t)b * M + j];
    const LineB lb = A.colB[(size_t)b * M + j];
    {
      uint32_t t[kRegLine], key[kRegLine], pp[kRegLine];
#pragma unroll
      for (uint32_t k = 0; k < kRegLine; ++k) t[k] = k < L ? A.csc_t[pb + beg + k] : 0u;
#pragma unroll
      for (uint32_t k = 0; k < kRegLine; ++k) {
        key[k] = k < L ? ebuf_of(A, b)[t[k]].x : 0xffffffffu;
        pp[k] = k < L ? A.inv[pb + t[k]] : 0u;
      }
#pragma unroll
      for (uint32_t k = 0; k < kRegLine; ++k) t[k] = k < L ? orig_row(A, b, key[k]) : 0xffffffffu;  // t <- ok
#pragma unroll
      for (uint32_t k = 0; k < kRegLine; ++k) {
        uint32_t r = 0;
#pragma unroll
        for (uint32_t f = 0; f < kRegLine; ++f) r += (t[f] < t[k]) ? 1u : 0u;
        if (k < L) {
          A.csc_i[pb + beg + r] = key[k];
          A.csc_perm[pb + beg + r] = pp[k];
        }
      }
    }
    uint32_t sp[kRegLine];
#pragma unroll
    for (uint32_t r = 0; r < kRegLine; ++r) sp[r] = r < L ? A.csc_perm[pb + beg + r] : 0u;
    float d2v[kRegLine], prv[kRegLine];
    uint32_t colf = 0u;  // bit r: entry r kept by the column softmax
#pragma unroll
    for (uint32_t r = 0; r < kRegLine; ++r) {
      if (r < L) {
        d2v[r] = A.d2s[pb + sp[r]];
        prv[r] = A.prow[pb + sp[r]];
        colf |= (A.csr_jf[pb + sp[r]] & kFlagCol) ? (1u << r) : 0u;
      }
    }
    int ra = -1, rb = -1;
    float Z = 0.f;
#pragma unroll
    for (uint32_t r = 0; r < kRegLine; ++r) {
      if (r < L) {
        const float d2 = d2v[r];
        if (ra < 0 && d2 == la.m2) ra = (int)r;
        else if (rb < 0 && d2 == la.s2) rb = (int)r;
        float e = 0.f;
        if (colf >> r & 1u) {
          e = (lb.flags & kLineK1) ? 1.f : expf(-lb.T * (__fsqrt_rn(d2) - lb.m));
          Z += e;
        }
        d2v[r] = e;  // reuse: unnormalised similarity
      }
    }
    const float iz = 1.f / Z;
#pragma unroll
    for (uint32_t r = 0; r < kRegLine; ++r) {
      if (r < L) {
        const float pc = d2v[r] * iz;
        const float p0 = 0.5f * (prv[r] + pc);
        A.pcol[pb + sp[r]] = pc;
        A.P0[pb + sp[r]] = p0;
        A.P0c[pb + beg + r] = p0;
      }
    }
    A.colidx[(size_t)b * M + j] = make_int2(ra >= 0 ? (int)A.csc_i[pb + beg + ra] : -1,
                                            rb >= 0 ? (int)A.csc_i[pb + beg + rb] : -1);
  }
}

// ---------------------------------------------------------------- shared-memory views

// One CTA's slice of the CSR (or CSC) structure: entries of local line k are
// [off[k], off[k+1]) in idx / val (and acc, backward).
template <typename IdxT>
struct SliceView {
  const unsigned* off;
  const IdxT* idx;
  const float* val;
  float* acc;
  __device__ __forceinline__ uint32_t col(uint32_t p) const { return (uint32_t)idx[p] & kIdxMask; }
};

__device__ __forceinline__ uint8_t* carve(uint8_t*& sm, size_t bytes) {
  uint8_t* p = sm;
  sm += (bytes + 15) & ~size_t(15);
  return p;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// Global -> shared copy of n floats by the whole CTA with cp.async (LDGSTS): every thread
// keeps all of its copies in flight, no register round trip per element.  16-byte copies
// when both ends are 16-byte aligned.  Completion: cp_async_wait_all() in every thread,
// then a CTA (or cluster) barrier.
__device__ __forceinline__ void g2s_async(float* dst, const float* src, size_t n) {
  size_t k0 = 0;
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    const size_t n4 = n / 4;
    for (size_t k = threadIdx.x; k < n4; k += blockDim.x)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst + 4 * k)), "l"(src + 4 * k)
                   : "memory");
    k0 = n4 * 4;
  }
  for (size_t k = k0 + threadIdx.x; k < n; k += blockDim.x)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst + k)), "l"(src + k) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Stage a line slice [s.lo, s.hi) of a CSR/CSC structure into shared memory (relative offsets).
// Values by cp.async; offsets and indices (converted) with kU loads in flight per thread.
template <typename IdxT>
__device__ SliceView<IdxT> stage_slice(uint8_t*& sm, const unsigned* ptr, Slice s,
                                       const uint32_t* idx_g, const float* val_g, bool with_acc) {
  constexpr int kU = 8;
  const int nl = s.hi - s.lo;
  const uint32_t base = ptr[s.lo], cnt = ptr[s.hi] - base;
  unsigned* off = reinterpret_cast<unsigned*>(carve(sm, 4 * (size_t)(nl + 1)));
  IdxT* idx = reinterpret_cast<IdxT*>(carve(sm, sizeof(IdxT) * (size_t)cnt));
  float* val = reinterpret_cast<float*>(carve(sm, 4 * (size_t)cnt));
  float* acc = with_acc ? reinterpret_cast<float*>(carve(sm, 4 * (size_t)cnt)) : nullptr;
  g2s_async(val, val_g + base, cnt);
  const uint32_t bd = blockDim.x;
  for (uint32_t k0 = threadIdx.x; k0 <= (uint32_t)nl; k0 += kU * bd) {
    unsigned v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) v[u] = k0 + u * bd <= (uint32_t)nl ? ptr[s.lo + k0 + u * bd] : 0u;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (k0 + u * bd <= (uint32_t)nl) off[k0 + u * bd] = v[u] - base;
  }
  for (uint32_t k0 = threadIdx.x; k0 < cnt; k0 += kU * bd) {
    uint32_t v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) v[u] = k0 + u * bd < cnt ? idx_g[base + k0 + u * bd] : 0u;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (k0 + u * bd < cnt) idx[k0 + u * bd] = (IdxT)(v[u] & kIdxMask);
  }
  cp_async_wait_all();
  return SliceView<IdxT>{off, idx, val, acc};
}

__device__ __forceinline__ size_t slice_bytes(int nl, uint32_t cnt, size_t idx_bytes, bool acc) {
  return ((4 * (size_t)(nl + 1) + 15) & ~size_t(15)) + ((idx_bytes * cnt + 15) & ~size_t(15)) +
         ((4 * (size_t)cnt + 15) & ~size_t(15)) + (acc ? ((4 * (size_t)cnt + 15) & ~size_t(15)) : 0);
}

// ---------------------------------------------------------------- replica exchange
//
// After a CTA computes the new values of its own slice of a scaling vector it writes them
// into the replica of every CTA of the cluster with st.async (DSMEM), each store signalling
// the destination's mbarrier (complete_tx); a CTA then waits on its own mbarrier for the
// whole vector (4 n bytes).  No cluster barrier (and hence no MEMBAR.GPU) per half-step.
// Reuse safety is causal: a CTA's push of the next vector depends on its reads of the
// current replica, and nobody can produce vector v+1 before receiving all of vector v.
// When the replicas live in global memory the exchange degrades to a store + cluster
// barrier.

__device__ __forceinline__ uint32_t map_rank(uint32_t addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

struct Xchg {
  float* rep;      // replica (shared; 16-byte aligned, length padded to a multiple of 4 + 4)
                   // or the single global copy
  uint32_t mbar;   // shared address of this CTA's mbarrier for the vector
  int n;           // vector length
  bool smem;
  uint32_t phase;  // parity of the next completion
};

__device__ __forceinline__ void mbar_init(uint32_t mbar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mbar) : "memory");
}
// Arm this CTA's mbarrier for the next use of the vector (4 n bytes: every element of the
// vector, own slice included, arrives through st.async).  Arming must precede any peer's
// pushes for that use: xchg_arm runs at set-up (before a cluster barrier) and at the end of
// every xchg_end (followed by a CTA barrier), so a peer -- which can only push the next
// round after receiving this CTA's pushes of the other vector, issued after that barrier --
// never sends bytes before the arm.
__device__ __forceinline__ void xchg_arm(const Xchg& x) {
  if (x.smem && threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(x.mbar), "r"(4u * (uint32_t)x.n) : "memory");
}
// Write element k of the vector into the replica of every CTA of the cluster (st.async, DSMEM),
// each store signalling the destination's mbarrier.
__device__ __forceinline__ void xchg_put(const Xchg& x, int CL, int k, float v) {
  if (!x.smem || CL == 1) { x.rep[k] = v; return; }  // one CTA: its replica is the vector
  const uint32_t a = smem_addr(x.rep + k);
  for (int r = 0; r < CL; ++r)
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
                 :: "r"(map_rank(a, r)), "r"(__float_as_uint(v)), "r"(map_rank(x.mbar, r)) : "memory");
}
// Wait until the whole vector has arrived, then re-arm for its next use.
__device__ __forceinline__ void xchg_end(cg::cluster_group& cl, Xchg& x, int CL, int me) {
  (void)me;
  if (!x.smem) { csync(cl); return; }
  if (CL == 1) { __syncthreads(); return; }  // no peers: a CTA barrier publishes the stores
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(x.mbar), "r"(x.phase) : "memory");
  x.phase ^= 1u;
  xchg_arm(x);
  __syncthreads();
}

// Segment dot product sum_{p in [p0, p1)} vec[col(p)] * val[p] with four independent
// accumulators (4x shorter dependent chain on long lines; fixed order -> deterministic).
// Segments of up to kDotShort entries are loaded with one predicated, fully unrolled batch
// (every gather in flight at once: one dependent chain off -> idx -> vec instead of one per 4
// entries); same accumulator assignment (entry u -> s[u % 4]) and final combination, so the
// result is bit-identical to the loop.
constexpr uint32_t kDotShort = 16;
template <typename IdxT>
__device__ __forceinline__ float seg_dot(const SliceView<IdxT>& V, uint32_t p0, uint32_t p1, const float* vec) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if (p1 - p0 <= kDotShort) {
    const uint32_t L = p1 - p0;
    float g[kDotShort], v[kDotShort];
#pragma unroll
    for (uint32_t u = 0; u < kDotShort; ++u) {
      g[u] = u < L ? vec[V.col(p0 + u)] : 0.f;
      v[u] = u < L ? V.val[p0 + u] : 0.f;
    }
#pragma unroll
    for (uint32_t u = 0; u < kDotShort; u += 4) {
      if (u < L) s0 = __fmaf_rn(g[u], v[u], s0);
      if (u + 1 < L) s1 = __fmaf_rn(g[u + 1], v[u + 1], s1);
      if (u + 2 < L) s2 = __fmaf_rn(g[u + 2], v[u + 2], s2);
      if (u + 3 < L) s3 = __fmaf_rn(g[u + 3], v[u + 3], s3);
    }
    return (s0 + s1) + (s2 + s3);
  }
  uint32_t p = p0;
  for (; p + 4 <= p1; p += 4) {
    s0 = __fmaf_rn(vec[V.col(p)], V.val[p], s0);
    s1 = __fmaf_rn(vec[V.col(p + 1)], V.val[p + 1], s1);
    s2 = __fmaf_rn(vec[V.col(p + 2)], V.val[p + 2], s2);
    s3 = __fmaf_rn(vec[V.col(p + 3)], V.val[p + 3], s3);
  }
  if (p < p1) s0 = __fmaf_rn(vec[V.col(p)], V.val[p], s0);
  if (p + 1 < p1) s1 = __fmaf_rn(vec[V.col(p + 1)], V.val[p + 1], s1);
  if (p + 2 < p1) s2 = __fmaf_rn(vec[V.col(p + 2)], V.val[p + 2], s2);
  return (s0 + s1) + (s2 + s3);
}

// seg_dot with a compile-time batch of KB predicated loads (lines of <= KB entries; same
// accumulator assignment as seg_dot, hence the same bits), and the choice of KB from the
// warp's longest line: with lines ordered by length (line_perm) most warps issue 4 or 8
// loads per array instead of 16.
template <int KB, typename IdxT>
__device__ __forceinline__ float seg_dot_n(const SliceView<IdxT>& V, uint32_t p0, uint32_t p1, const float* vec) {
  const uint32_t L = p1 - p0;
  float g[KB], v[KB];
#pragma unroll
  for (uint32_t u = 0; u < KB; ++u) {
    g[u] = u < L ? vec[V.col(p0 + u)] : 0.f;
    v[u] = u < L ? V.val[p0 + u] : 0.f;
  }
  float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (uint32_t u = 0; u < KB; ++u)
    if (u < L) s[u & 3] = __fmaf_rn(g[u], v[u], s[u & 3]);
  return (s[0] + s[1]) + (s[2] + s[3]);
}
template <typename IdxT>
__device__ __forceinline__ float seg_dot_adapt(const SliceView<IdxT>& V, uint32_t p0, uint32_t p1, const float* vec,
                                               uint32_t wmax) {
  if (wmax <= 4) return seg_dot_n<4>(V, p0, p1, vec);
  if (wmax <= 8) return seg_dot_n<8>(V, p0, p1, vec);
  return seg_dot_n<16>(V, p0, p1, vec);
}

// Lines of a slice ordered by length (counting sort: 0..kRegLine, then longer), so that the
// 32 lines of a warp have similar lengths (seg_dot_adapt).  The order inside a length class
// is arbitrary: every line's result is independent of the thread that computes it.
__device__ void line_perm(const unsigned* off, int n, uint16_t* perm, unsigned* hist /*[kRegLine + 2]*/) {
  constexpr int kB = kRegLine + 2;
  if (threadIdx.x < kB) hist[threadIdx.x] = 0u;
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const uint32_t L = off[k + 1] - off[k];
    atomicAdd(hist + (L <= kRegLine ? L : kRegLine + 1), 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned run = 0;
    for (int q = 0; q < kB; ++q) { const unsigned v = hist[q]; hist[q] = run; run += v; }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const uint32_t L = off[k + 1] - off[k];
    perm[atomicAdd(hist + (L <= kRegLine ? L : kRegLine + 1), 1u)] = (uint16_t)k;
  }
  __syncthreads();
}

// ---------------------------------------------------------------- forward Sinkhorn + loss
//
// A half-step costs one replica exchange (~0.6 us, scripts/micro/xchg_bench.cu) plus the
// slowest line of any CTA of the cluster.  Lines of up to kRegLine entries are one thread's
// (seg_dot: one batched gather); longer lines -- the CTA's long-line list -- are done by a
// warp each (lane-strided gathers, butterfly sum), so one long line no longer gates the step.

static_assert(kDotShort == kRegLine, "short-line threshold of the Sinkhorn loops = long-line list threshold");

template <typename IdxT>
__device__ __forceinline__ float warp_dot(const SliceView<IdxT>& V, uint32_t p0, uint32_t p1, const float* vec) {
  float s = 0.f;
  for (uint32_t p = p0 + (threadIdx.x & 31); p < p1; p += 32) s = __fmaf_rn(vec[V.col(p)], V.val[p], s);
  return gsum<32>(s);  // every lane holds the same bits
}

// kSm: slices and replicas are all in shared memory -- asserted to the compiler so that the
// gathers through these (struct-held, generic) pointers compile to LDS rather than generic
// LD, whose long-scoreboard latency dominated the half-steps.
#define APML_ASSUME_SMEM(p) __builtin_assume(__isShared((const void*)(p)))
template <typename IdxT>
__device__ __forceinline__ void assume_smem(const SliceView<IdxT>& V) {
  APML_ASSUME_SMEM(V.off);
  APML_ASSUME_SMEM(V.idx);
  APML_ASSUME_SMEM(V.val);
}

template <typename IdxT, bool kSm>
__device__ void sinkhorn_fwd(cg::cluster_group& cl, const SparseArgs& A, int b, Slice sr, Slice sc,
                             const SliceView<IdxT>& R, const SliceView<IdxT>& C, Xchg& xa, Xchg& xb,
                             const LongList& llr, const LongList& llc, const uint16_t* rperm = nullptr,
                             const uint16_t* cperm = nullptr) {
  const int N = A.N, M = A.M, L = A.L, CL = cl.num_blocks(), me = cl.block_rank();
  float* ah = A.a_hist + (size_t)b * (L + 1) * N;
  float* bh = A.b_hist + (size_t)b * (L + 1) * M;
  const float* a = xa.rep;
  const float* bv = xb.rep;
  if (kSm) {
    assume_smem(R);
    assume_smem(C);
    APML_ASSUME_SMEM(a);
    APML_ASSUME_SMEM(bv);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // Eq. (3): colsum_j = b_j Q_j, b_j <- b_j / (colsum_j + eps)
  // an EMPTY line (the padding lines of a ragged pair; a real line always holds its argmin)
  // keeps its scale: Eq. (3)/(4) would divide by eps alone and overflow
  auto col_upd = [&](int j, float Q, int l, bool empty = false) {
    const float bj = bv[j];
    const float nb = empty ? bj : __fdividef(bj, __fmaf_rn(bj, Q, A.eps));
    xchg_put(xb, CL, j, nb);
    bh[(size_t)l * M + j] = nb;
  };
  // Eq. (4): rowsum_i = a_i R_i, a_i <- a_i / (rowsum_i + eps)
  auto row_upd = [&](int i, float Rs, int l, bool empty = false) {
    const float ai = a[i];
    const float na = empty ? ai : __fdividef(ai, __fmaf_rn(ai, Rs, A.eps));
    xchg_put(xa, CL, i, na);
    ah[(size_t)l * N + i] = na;
  };
  const int nr = sr.hi - sr.lo, nc = sc.hi - sc.lo;
  for (int l = 1; l <= L; ++l) {
    if (cperm) {  // lines ordered by length: the warp's longest line sets the batch
      for (int t = threadIdx.x; t < nc; t += blockDim.x) {
        const int k = cperm[t], j = sc.lo + k;
        const uint32_t p0 = C.off[k], p1 = C.off[k + 1], Ln = p1 - p0;
        const uint32_t wmax = __reduce_max_sync(__activemask(), Ln <= kRegLine ? Ln : 0u);
        if (Ln <= kRegLine) col_upd(j, seg_dot_adapt(C, p0, p1, a, wmax), l, Ln == 0);
      }
    } else {
      for (int j = sc.lo + threadIdx.x; j < sc.hi; j += blockDim.x) {
        const int k = j - sc.lo;
        const uint32_t p0 = C.off[k], p1 = C.off[k + 1];
        if (p1 - p0 <= kRegLine) col_upd(j, seg_dot(C, p0, p1, a), l, p1 == p0);
      }
    }
    for (int q = w; q < llc.count(); q += nw) {
      const int j = llc.line(q), k = j - sc.lo;
      const uint32_t p0 = C.off[k], p1 = C.off[k + 1];
      if (p1 - p0 <= kRegLine) continue;  // (overflowed list: whole slice)
      const float Q = warp_dot(C, p0, p1, a);
      if (lane == 0) col_upd(j, Q, l);
    }
    xchg_end(cl, xb, CL, me);
    if (rperm) {
      for (int t = threadIdx.x; t < nr; t += blockDim.x) {
        const int k = rperm[t], i = sr.lo + k;
        const uint32_t p0 = R.off[k], p1 = R.off[k + 1], Ln = p1 - p0;
        const uint32_t wmax = __reduce_max_sync(__activemask(), Ln <= kRegLine ? Ln : 0u);
        if (Ln <= kRegLine) row_upd(i, seg_dot_adapt(R, p0, p1, bv, wmax), l, Ln == 0);
      }
    } else {
      for (int i = sr.lo + threadIdx.x; i < sr.hi; i += blockDim.x) {
        const int k = i - sr.lo;
        const uint32_t p0 = R.off[k], p1 = R.off[k + 1];
        if (p1 - p0 <= kRegLine) row_upd(i, seg_dot(R, p0, p1, bv), l, p1 == p0);
      }
    }
    for (int q = w; q < llr.count(); q += nw) {
      const int i = llr.line(q), k = i - sr.lo;
      const uint32_t p0 = R.off[k], p1 = R.off[k + 1];
      if (p1 - p0 <= kRegLine) continue;
      const float Rs = warp_dot(R, p0, p1, bv);
      if (lane == 0) row_upd(i, Rs, l);
    }
    xchg_end(cl, xa, CL, me);
  }
}

// ---------------------------------------------------------------- the forward kernel

template <typename IdxT>
__global__ void __launch_bounds__(kMegaThreads, 1) k_sparse_fwd(const SparseArgs A) {
  pdl_trigger();
  pdl_wait();  // launched with programmatic dependent launch: the emit's output first
  extern __shared__ __align__(16) uint8_t shm[];
  __shared__ unsigned s_tot_r[kMaxCluster], s_tot_c[kMaxCluster];  // one per scan (no reuse race)
  __shared__ unsigned s_warp[32];
  __shared__ double s_part[kMaxCluster];
  __shared__ uint32_t s_long_r[kLongCap], s_long_c[kLongCap];
  __shared__ int s_nlong[2];
  cg::cluster_group cl = cg::this_cluster();
  const int CL = cl.num_blocks(), rank = cl.block_rank();
  const int b = blockIdx.x / CL;
  const int N = A.N, M = A.M, L = A.L;
  const size_t pb = (size_t)b * A.cap;
  const unsigned total = A.cursor[b];
  if (total > A.cap) {  // overflowed pair: uniform across the cluster, no barrier follows
    if (rank == 0 && threadIdx.x == 0) A.loss[b] = __int_as_float(0x7fc00000);
    return;
  }
  const Slice sr = slice_of(N, rank, CL), sc = slice_of(M, rank, CL);
  unsigned* rc = A.row_cnt + (size_t)b * (N + 1);
  unsigned* cc = A.col_cnt + (size_t)b * (M + 1);
  unsigned* rp = A.row_ptr + (size_t)b * (N + 1);
  unsigned* cp = A.col_ptr + (size_t)b * (M + 1);
  phase(A, 0);
  // S4: counts -> offsets ("exclusive prefix sum"), then bucket the entries
  cluster_scan(cl, rc, rp, N, sr, s_tot_r, s_warp);
  cluster_scan(cl, cc, cp, M, sc, s_tot_c, s_warp);
  csync(cl);
  phase(A, 1);
  {
    // kSc entries per thread per step: loads, then all atomics, then the stores, so a step
    // costs ~3 L2 round trips instead of 3 per entry
    constexpr int kSc = 4;
    const uint32_t stride = CL * blockDim.x;
    for (uint32_t t0 = rank * blockDim.x + threadIdx.x; t0 < total; t0 += kSc * stride) {
      uint32_t ii[kSc], jj[kSc], pr[kSc], pc[kSc];
#pragma unroll
      for (int u = 0; u < kSc; ++u) {
        const uint32_t t = t0 + u * stride;
        const uint2 e = t < total ? ebuf_of(A, b)[t] : make_uint2(0u, 0u);
        ii[u] = e.x;
        jj[u] = e.y & kIdxMask;
      }
#pragma unroll
      for (int u = 0; u < kSc; ++u) {
        if (t0 + u * stride < total) {
          pr[u] = rp[ii[u]] + atomicAdd(rc + ii[u], 1u);
          pc[u] = cp[jj[u]] + atomicAdd(cc + jj[u], 1u);
        }
      }
#pragma unroll
      for (int u = 0; u < kSc; ++u) {
        const uint32_t t = t0 + u * stride;
        if (t < total) {
          A.csr_t[pb + pr[u]] = t;
          A.csc_t[pb + pc[u]] = t;
        }
      }
    }
  }
  csync(cl);
  phase(A, 2);
  // rows: sort by j (registers for short rows, warp rank sort for long ones) and the row
  // softmax (S5) on the kept support
  const LongList llr = collect_long(rp, sr, s_long_r, &s_nlong[0]);
  const LongList llc = collect_long(cp, sc, s_long_c, &s_nlong[1]);
  phase(A, 3);
  row_sort_norm_regs(A, b, sr);
  __syncthreads();
  phase(A, 4);
  sort_lines<true>(A, b, sr, llr);
  __syncthreads();
  phase(A, 5);
  row_norm(A, b, sr, llr);
  csync(cl);
  phase(A, 6);
  // columns: sort by i, column softmax, symmetrisation P0 = (P_row + P_col)/2
  col_sort_norm_regs(A, b, sc);
  __syncthreads();
  phase(A, 7);
  sort_lines<false>(A, b, sc, llc);
  __syncthreads();
  phase(A, 8);
  col_norm(A, b, sc, llc);
  csync(cl);
  phase(A, 9);
  // S6: Sinkhorn.  Replicas of a and b (full length) + own CSR / CSC slices in shared memory.
  uint8_t* sm = shm;
  float *a, *bv;
  __shared__ __align__(8) unsigned long long s_mbar[2];
  if (A.rep_smem) {
    a = reinterpret_cast<float*>(carve(sm, 4 * (size_t)((N + 3) / 4 * 4 + 4)));
    bv = reinterpret_cast<float*>(carve(sm, 4 * (size_t)((M + 3) / 4 * 4 + 4)));
    for (int k = threadIdx.x; k < N; k += blockDim.x) a[k] = 1.f;
    for (int k = threadIdx.x; k < M; k += blockDim.x) bv[k] = 1.f;
    if (threadIdx.x == 0) {
      mbar_init(smem_addr(&s_mbar[0]));
      mbar_init(smem_addr(&s_mbar[1]));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  } else {
    a = A.gvec + (size_t)b * 2 * (N + M);
    bv = a + N;
    for (int k = sr.lo + threadIdx.x; k < sr.hi; k += blockDim.x) a[k] = 1.f;
    for (int k = sc.lo + threadIdx.x; k < sc.hi; k += blockDim.x) bv[k] = 1.f;
  }
  float* ah = A.a_hist + (size_t)b * (L + 1) * N;
  float* bh = A.b_hist + (size_t)b * (L + 1) * M;
  for (int k = sr.lo + threadIdx.x; k < sr.hi; k += blockDim.x) ah[k] = 1.f;
  for (int k = sc.lo + threadIdx.x; k < sc.hi; k += blockDim.x) bh[k] = 1.f;
  Xchg xa{a, smem_addr(&s_mbar[0]), N, A.rep_smem != 0, 0u};
  Xchg xb{bv, smem_addr(&s_mbar[1]), M, A.rep_smem != 0, 0u};
  xchg_arm(xa);  // first use of each mbarrier; peers start pushing after the next cl.sync
  xchg_arm(xb);
  const size_t used = (size_t)(sm - shm);
  const bool fit = used + slice_bytes(sr.hi - sr.lo, rp[sr.hi] - rp[sr.lo], sizeof(IdxT), false) +
                       slice_bytes(sc.hi - sc.lo, cp[sc.hi] - cp[sc.lo], sizeof(IdxT), false) <= A.smem_bytes;
  if (fit) {
    const SliceView<IdxT> R = stage_slice<IdxT>(sm, rp, sr, A.csr_jf + pb, A.P0 + pb, false);
    const SliceView<IdxT> C = stage_slice<IdxT>(sm, cp, sc, A.csc_i + pb, A.P0c + pb, false);
    csync(cl);
    phase(A, 10);
    if (A.rep_smem) sinkhorn_fwd<IdxT, true>(cl, A, b, sr, sc, R, C, xa, xb, llr, llc);
    else sinkhorn_fwd<IdxT, false>(cl, A, b, sr, sc, R, C, xa, xb, llr, llc);
  } else {
    const SliceView<uint32_t> R{rp + sr.lo, A.csr_jf + pb, A.P0 + pb, nullptr};
    const SliceView<uint32_t> C{cp + sc.lo, A.csc_i + pb, A.P0c + pb, nullptr};
    csync(cl);
    phase(A, 10);
    sinkhorn_fwd<uint32_t, false>(cl, A, b, sr, sc, R, C, xa, xb, llr, llc);
  }
  phase(A, 11);
  // S7: loss_b = sum_i a_i sum_j P0_ij b_j c_ij over own rows, then cluster reduction in rank order
  double acc = 0.0;
  for (int i = sr.lo + threadIdx.x; i < sr.hi; i += blockDim.x) {
    float t = 0.f;
    for (uint32_t p = rp[i]; p < rp[i + 1]; ++p)
      t = __fmaf_rn(__fmul_rn(A.P0[pb + p], bv[A.csr_jf[pb + p] & kIdxMask]), A.cs[pb + p], t);
    acc += (double)a[i] * (double)t;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  __shared__ double s_red[32];
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
    cl.map_shared_rank(s_part, 0)[rank] = t;
  }
  csync(cl);
  if (rank == 0 && threadIdx.x == 0) {
    double t = 0.0;
    for (int r = 0; r < CL; ++r) t += s_part[r];
    A.loss[b] = (float)t;
  }
  phase(A, 12);
}

// ---------------------------------------------------------------- backward

constexpr int kPf = 8;  // b^l prefetch registers per thread (bls staging needs M <= kPf * blockDim)

// acc[p] += s * vec[col(p)] over a short segment (<= kRegLine entries): one batched gather.
template <typename IdxT>
__device__ __forceinline__ void seg_axpy(const SliceView<IdxT>& V, uint32_t p0, uint32_t p1, float s, const float* vec) {
  const uint32_t n = p1 - p0;
  float g[kRegLine], c[kRegLine];
#pragma unroll
  for (uint32_t u = 0; u < kRegLine; ++u) {
    g[u] = u < n ? vec[V.col(p0 + u)] : 0.f;
    c[u] = u < n ? V.acc[p0 + u] : 0.f;
  }
#pragma unroll
  for (uint32_t u = 0; u < kRegLine; ++u)
    if (u < n) V.acc[p0 + u] = c[u] + s * g[u];
}
// Returns sum_p vec[col(p)] val[p] (accumulators as seg_dot) and does acc[p] += vec[col(p)] * s,
// over a short segment.
template <typename IdxT>
__device__ __forceinline__ float seg_dot_axpy(const SliceView<IdxT>& V, uint32_t p0, uint32_t p1, const float* vec,
                                              float s) {
  const uint32_t n = p1 - p0;
  float g[kRegLine], v[kRegLine], c[kRegLine];
#pragma unroll
  for (uint32_t u = 0; u < kRegLine; ++u) {
    g[u] = u < n ? vec[V.col(p0 + u)] : 0.f;
    v[u] = u < n ? V.val[p0 + u] : 0.f;
    c[u] = u < n ? V.acc[p0 + u] : 0.f;
  }
  float t[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (uint32_t u = 0; u < kRegLine; ++u)
    if (u < n) t[u & 3] = __fmaf_rn(g[u], v[u], t[u & 3]);
#pragma unroll
  for (uint32_t u = 0; u < kRegLine; ++u)
    if (u < n) V.acc[p0 + u] = c[u] + g[u] * s;
  return (t[0] + t[1]) + (t[2] + t[3]);
}

// Row step 2 of reverse iteration l fused with the row step of iteration l - 1 for one short
// row (<= kRegLine entries, one batched gather each):
//   t = sum_j P0_ij Qbar^l_j;  abar_i += t;
//   (l > 1) Rbar^{l-1}_i = -abar_i (a^{l-1}_i)^2, abar_i <- abar_i eps (a^{l-1}_i / a^{l-2}_i)^2;
//   P0bar_ij += Qbar^l_j a^{l-1}_i  (+ Rbar^{l-1}_i b^{l-1}_j)
// Returns Rbar^{l-1}_i (0 when l == 1); the caller pushes it.
template <int KB, typename IdxT>
__device__ __forceinline__ float seg_rev_fused_n(const SliceView<IdxT>& V, uint32_t p0, uint32_t p1, const float* q,
                                                 const float* bprev, float alm, float almm, float& abk, float eps) {
  const uint32_t n = p1 - p0;
  uint32_t ix[KB];
  float g[KB];
  float t[4] = {0.f, 0.f, 0.f, 0.f};
  {
    float v[KB];
#pragma unroll
    for (uint32_t u = 0; u < KB; ++u) {
      ix[u] = u < n ? V.col(p0 + u) : 0u;
      v[u] = u < n ? V.val[p0 + u] : 0.f;
    }
#pragma unroll
    for (uint32_t u = 0; u < KB; ++u) g[u] = u < n ? q[ix[u]] : 0.f;
#pragma unroll
    for (uint32_t u = 0; u < KB; ++u)
      if (u < n) t[u & 3] = __fmaf_rn(g[u], v[u], t[u & 3]);
  }
  abk += (t[0] + t[1]) + (t[2] + t[3]);
  float Rb = 0.f;
  if (bprev) {
    const float r = alm / almm;
    Rb = -abk * alm * alm;
    abk = abk * eps * r * r;
  }
  float bp[KB], c[KB];
#pragma unroll
  for (uint32_t u = 0; u < KB; ++u) {
    bp[u] = (u < n && bprev) ? bprev[ix[u]] : 0.f;
    c[u] = u < n ? V.acc[p0 + u] : 0.f;
  }
#pragma unroll
  for (uint32_t u = 0; u < KB; ++u)
    if (u < n) V.acc[p0 + u] = (c[u] + g[u] * alm) + Rb * bp[u];
  return Rb;
}
template <typename IdxT>
__device__ __forceinline__ float seg_rev_fused(const SliceView<IdxT>& V, uint32_t p0, uint32_t p1, const float* q,
                                               const float* bprev, float alm, float almm, float& abk, float eps,
                                               uint32_t wmax = kRegLine) {
  if (wmax <= 4) return seg_rev_fused_n<4>(V, p0, p1, q, bprev, alm, almm, abk, eps);
  if (wmax <= 8) return seg_rev_fused_n<8>(V, p0, p1, q, bprev, alm, almm, abk, eps);
  return seg_rev_fused_n<kRegLine>(V, p0, p1, q, bprev, alm, almm, abk, eps);
}

// Reverse Sinkhorn in scaling form; P0bar accumulated per CSR entry of the own
// rows in shared memory (R.acc).  Short lines by a thread, long lines by a warp (as forward).
template <typename IdxT, bool kSm>
__device__ void sinkhorn_bwd(cg::cluster_group& cl, const SparseArgs& A, int b, Slice sr, Slice sc,
                             const SliceView<IdxT>& R, const SliceView<IdxT>& C, float* ab, float* bb,
                             Xchg& xr, Xchg& xq, float* bls, const float* ahs, const float* bhs,
                             const LongList& llr, const LongList& llc, const uint16_t* rperm = nullptr,
                             const uint16_t* cperm = nullptr) {
  // kSm: slices (+ acc), replicas, abar / bbar and the staged history all in shared memory
  if (kSm) {
    assume_smem(R);
    assume_smem(C);
    APML_ASSUME_SMEM(R.acc);
    APML_ASSUME_SMEM(xr.rep);
    APML_ASSUME_SMEM(xq.rep);
    APML_ASSUME_SMEM(ab);
    APML_ASSUME_SMEM(bb);
    if (ahs) APML_ASSUME_SMEM(ahs);
    if (bhs) APML_ASSUME_SMEM(bhs);
    if (bls) APML_ASSUME_SMEM(bls);
  }
  const int N = A.N, M = A.M, L = A.L, CL = cl.num_blocks(), me = cl.block_rank();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // ahs: own rows' a history [L+1][nr] and bhs: full b history [L+1][M], staged in shared
  // memory when they fit (else read from global memory, b^l optionally staged via bls).
  const int nr = sr.hi - sr.lo;
  const float* ah = ahs ? ahs - sr.lo : A.a_hist + (size_t)b * (L + 1) * N;
  const size_t ald = ahs ? (size_t)nr : (size_t)N;
  const float* bh = bhs ? bhs : A.b_hist + (size_t)b * (L + 1) * M;
  if (bhs) bls = nullptr;
  const float* rcur = xr.rep;
  const float* qcur = xq.rep;
  // bls (2 x M floats, shared memory, optional): b^l staged for the P0bar gathers, double
  // buffered -- b^{l-1} is loaded into registers at the top of iteration l and stored after it.
  if (bls) {
    for (int k = threadIdx.x; k < M; k += blockDim.x) bls[(L & 1) * M + k] = bh[(size_t)L * M + k];
    __syncthreads();
  }
  // row step reverse of iteration l: Rbar^l = -abar (a^l)^2, abar <- abar eps (a^l/a^{l-1})^2,
  // P0bar_ij += Rbar^l_i b^l_j.  Iteration L's runs here; iteration l-1's runs fused with
  // row step 2 of iteration l (seg_rev_fused / the warp loop below): one row pass fewer.
  {
    const float* bL = bls ? bls + (L & 1) * M : bh + (size_t)L * M;
    auto row_rev = [&](int i, int k, float abk, bool writer) -> float {
      const float al = ah[(size_t)L * ald + i], alm = ah[(size_t)(L - 1) * ald + i];
      const float r = al / alm;
      const float Rb = -abk * al * al;
      if (writer) {
        ab[k] = abk * A.eps * r * r;
        xchg_put(xr, CL, i, Rb);
      }
      return Rb;
    };
    for (int i = sr.lo + threadIdx.x; i < sr.hi; i += blockDim.x) {
      const int k = i - sr.lo;
      const uint32_t p0 = R.off[k], p1 = R.off[k + 1];
      if (p1 - p0 > kRegLine) continue;
      seg_axpy(R, p0, p1, row_rev(i, k, ab[k], true), bL);
    }
    for (int q = w; q < llr.count(); q += nw) {
      const int i = llr.line(q), k = i - sr.lo;
      const uint32_t p0 = R.off[k], p1 = R.off[k + 1];
      if (p1 - p0 <= kRegLine) continue;
      const float abk = ab[k];
      __syncwarp();
      const float Rb = row_rev(i, k, abk, lane == 0);
      for (uint32_t p = p0 + lane; p < p1; p += 32) R.acc[p] += Rb * bL[R.col(p)];
      __syncwarp();
    }
  }
  for (int l = L; l >= 1; --l) {
    float pf[kPf];
    if (bls && l > 1) {
#pragma unroll
      for (int u = 0; u < kPf; ++u) {
        const int k = threadIdx.x + u * blockDim.x;
        pf[u] = k < M ? bh[(size_t)(l - 1) * M + k] : 0.f;
      }
    }
    const float* bcur = bls ? bls + (l & 1) * M : bh + (size_t)l * M;  // b^l
    // b^{l-1} of this thread's first kOwnPf columns, loaded now so that the column step does
    // not wait on it when the history is not in shared memory
    constexpr int kOwnPf = 2;
    float blm_pf[kOwnPf];
#pragma unroll
    for (int u = 0; u < kOwnPf; ++u) {
      const int j = sc.lo + threadIdx.x + u * blockDim.x;
      blm_pf[u] = j < sc.hi ? bh[(size_t)(l - 1) * M + j] : 1.f;
    }
    xchg_end(cl, xr, CL, me);
    // column step reverse: bbar += P0^T Rbar^l; Qbar^l = -bbar (b^l)^2; bbar <- bbar eps (..)^2
    auto col_rev = [&](int j, int k, float t, float blm) {
      const float bsum = bb[k] + t;
      const float bl = bcur[j];
      const float r = bl / blm;
      bb[k] = bsum * A.eps * r * r;
      xchg_put(xq, CL, j, -bsum * bl * bl);
    };
    if (cperm) {  // lines ordered by length (single-CTA clusters): adaptive batch
      for (int t = threadIdx.x; t < sc.hi - sc.lo; t += blockDim.x) {
        const int k = cperm[t], j = sc.lo + k;
        const uint32_t p0 = C.off[k], p1 = C.off[k + 1], Ln = p1 - p0;
        const uint32_t wmax = __reduce_max_sync(__activemask(), Ln <= kRegLine ? Ln : 0u);
        if (Ln <= kRegLine) col_rev(j, k, seg_dot_adapt(C, p0, p1, rcur, wmax), bh[(size_t)(l - 1) * M + j]);
      }
    } else {
      int u = 0;
      for (int j = sc.lo + threadIdx.x; j < sc.hi; j += blockDim.x, ++u) {
        const int k = j - sc.lo;
        const uint32_t p0 = C.off[k], p1 = C.off[k + 1];
        float blm = 0.f;
#pragma unroll
        for (int v = 0; v < kOwnPf; ++v) blm = u == v ? blm_pf[v] : blm;
        if (u >= kOwnPf) blm = bh[(size_t)(l - 1) * M + j];
        if (p1 - p0 <= kRegLine) col_rev(j, k, seg_dot(C, p0, p1, rcur), blm);
      }
    }
    for (int q = w; q < llc.count(); q += nw) {
      const int j = llc.line(q), k = j - sc.lo;
      const uint32_t p0 = C.off[k], p1 = C.off[k + 1];
      if (p1 - p0 <= kRegLine) continue;
      const float t = warp_dot(C, p0, p1, rcur);
      if (lane == 0) col_rev(j, k, t, bh[(size_t)(l - 1) * M + j]);
    }
    // b^{l-1} into the other staging buffer (it held b^{l+1}, last read by the column step of
    // iteration l+1); published by the barrier inside xchg_end below
    if (bls && l > 1) {
#pragma unroll
      for (int u = 0; u < kPf; ++u) {
        const int k = threadIdx.x + u * blockDim.x;
        if (k < M) bls[((l - 1) & 1) * M + k] = pf[u];
      }
    }
    xchg_end(cl, xq, CL, me);
    // row step 2 of l: abar += P0 Qbar^l, P0bar_ij += Qbar^l_j a^{l-1}_i -- fused with the
    // row step of l-1 (Rbar^{l-1} pushed for the next column step)
    const float* bprev = l > 1 ? (bls ? bls + ((l - 1) & 1) * M : bh + (size_t)(l - 1) * M) : nullptr;
    if (rperm) {
      for (int t = threadIdx.x; t < sr.hi - sr.lo; t += blockDim.x) {
        const int k = rperm[t], i = sr.lo + k;
        const uint32_t p0 = R.off[k], p1 = R.off[k + 1], Ln = p1 - p0;
        const uint32_t wmax = __reduce_max_sync(__activemask(), Ln <= kRegLine ? Ln : 0u);
        if (Ln > kRegLine) continue;
        const float alm = ah[(size_t)(l - 1) * ald + i];
        const float almm = l > 1 ? ah[(size_t)(l - 2) * ald + i] : 1.f;
        float abk = ab[k];
        const float Rb = seg_rev_fused(R, p0, p1, qcur, bprev, alm, almm, abk, A.eps, wmax);
        ab[k] = abk;
        if (l > 1) xchg_put(xr, CL, i, Rb);
      }
    } else {
      for (int i = sr.lo + threadIdx.x; i < sr.hi; i += blockDim.x) {
        const int k = i - sr.lo;
        const uint32_t p0 = R.off[k], p1 = R.off[k + 1];
        if (p1 - p0 > kRegLine) continue;
        const float alm = ah[(size_t)(l - 1) * ald + i];
        const float almm = l > 1 ? ah[(size_t)(l - 2) * ald + i] : 1.f;
        float abk = ab[k];
        const float Rb = seg_rev_fused_n<kRegLine>(R, p0, p1, qcur, bprev, alm, almm, abk, A.eps);
        ab[k] = abk;
        if (l > 1) xchg_put(xr, CL, i, Rb);
      }
    }
    for (int q = w; q < llr.count(); q += nw) {
      const int i = llr.line(q), k = i - sr.lo;
      const uint32_t p0 = R.off[k], p1 = R.off[k + 1];
      if (p1 - p0 <= kRegLine) continue;
      const float alm = ah[(size_t)(l - 1) * ald + i];
      float t = 0.f;
      for (uint32_t p = p0 + lane; p < p1; p += 32) t = __fmaf_rn(qcur[R.col(p)], R.val[p], t);
      t = gsum<32>(t);
      float abk = ab[k] + t;
      float Rb = 0.f;
      if (l > 1) {
        const float almm = ah[(size_t)(l - 2) * ald + i];
        const float r = alm / almm;
        Rb = -abk * alm * alm;
        abk = abk * A.eps * r * r;
      }
      for (uint32_t p = p0 + lane; p < p1; p += 32) {
        const uint32_t j = R.col(p);
        R.acc[p] = (R.acc[p] + qcur[j] * alm) + (l > 1 ? Rb * bprev[j] : 0.f);
      }
      __syncwarp();
      if (lane == 0) {
        ab[k] = abk;
        if (l > 1) xchg_put(xr, CL, i, Rb);
      }
      __syncwarp();
    }
  }
  csync(cl);
}

// ---- per-line loops of the backward, run by groups of G lanes: G = 1 (thread per line,
// lines of length <= kRegLine, U entries loaded per step) and G = 32 (warp per longer line).
// Loads of a step are issued together so a line costs ~2 round trips per G*U entries.

template <int G>
__device__ __forceinline__ bool line_mine(uint32_t L) { return G == 1 ? L <= kRegLine : L > kRegLine; }

// Row softmax reverse -> LineBack (two passes: S = sum P Pbar/2, then zbar = P (Pbar/2 - S)).
template <int G, int U>
__device__ void row_soft_rev(const SparseArgs& A, int b, Slice s, const LongList& ll) {
  const int N = A.N;
  const size_t pb = (size_t)b * A.cap;
  const unsigned* rp = A.row_ptr + (size_t)b * (N + 1);
  const int mem = G == 1 ? 0 : (threadIdx.x & 31);
  APML_FOR_LINES(G, s, ll, i) {
    const uint32_t beg = rp[i], end = rp[i + 1];
    if (!line_mine<G>(end - beg)) continue;
    const LineB lb = A.rowB[(size_t)b * N + i];
    LineBack out = {0.f, 0.f, 0.f, 0.f};
    if (!(lb.flags & kLineK1)) {
      double S = 0.0;
      for (uint32_t p0 = beg; p0 < end; p0 += G * U) {
        uint32_t jf[U];
        float pr[U], pbv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t p = p0 + u * G + mem;
          jf[u] = p < end ? A.csr_jf[pb + p] : 0u;
          pr[u] = p < end ? A.prow[pb + p] : 0.f;
          pbv[u] = p < end ? A.pbar[pb + p] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (jf[u] & kFlagRow) S += (double)pr[u] * 0.5 * (double)pbv[u];
      }
      S = gsum<G>(S);
      double szb = 0.0, Tbar = 0.0;
      for (uint32_t p0 = beg; p0 < end; p0 += G * U) {
        uint32_t jf[U];
        float pr[U], pbv[U], cv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t p = p0 + u * G + mem;
          jf[u] = p < end ? A.csr_jf[pb + p] : 0u;
          pr[u] = p < end ? A.prow[pb + p] : 0.f;
          pbv[u] = p < end ? A.pbar[pb + p] : 0.f;
          cv[u] = p < end ? A.cs[pb + p] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!(jf[u] & kFlagRow)) continue;
          const double zb = (double)pr[u] * (0.5 * (double)pbv[u] - S);
          szb += zb;
          Tbar -= zb * ((double)cv[u] - (double)lb.m);
        }
      }
      szb = gsum<G>(szb);
      Tbar = gsum<G>(Tbar);
      const double mbar = (double)lb.T * szb;
      const double gbar = (lb.flags & kLineClamped) ? 0.0 : -Tbar * (double)lb.T / (double)lb.g;
      out = {(float)S, (float)(mbar - gbar), (float)gbar, lb.T};
    }
    if (mem == 0) A.rowback[(size_t)b * N + i] = out;
  }
}

template <int G, int U>
__device__ void col_soft_rev(const SparseArgs& A, int b, Slice s, const LongList& ll) {
  const int M = A.M;
  const size_t pb = (size_t)b * A.cap;
  const unsigned* cp = A.col_ptr + (size_t)b * (M + 1);
  const int mem = G == 1 ? 0 : (threadIdx.x & 31);
  APML_FOR_LINES(G, s, ll, j) {
    const uint32_t beg = cp[j], end = cp[j + 1];
    if (!line_mine<G>(end - beg)) continue;
    const LineB lb = A.colB[(size_t)b * M + j];
    LineBack out = {0.f, 0.f, 0.f, 0.f};
    if (!(lb.flags & kLineK1)) {
      double S = 0.0;
      for (uint32_t q0 = beg; q0 < end; q0 += G * U) {
        uint32_t pp[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t q = q0 + u * G + mem;
          pp[u] = q < end ? A.csc_perm[pb + q] : 0xffffffffu;
        }
        uint32_t jf[U];
        float pc[U], pbv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool v = pp[u] != 0xffffffffu;
          jf[u] = v ? A.csr_jf[pb + pp[u]] : 0u;
          pc[u] = v ? A.pcol[pb + pp[u]] : 0.f;
          pbv[u] = v ? A.pbar[pb + pp[u]] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (jf[u] & kFlagCol) S += (double)pc[u] * 0.5 * (double)pbv[u];
      }
      S = gsum<G>(S);
      double szb = 0.0, Tbar = 0.0;
      for (uint32_t q0 = beg; q0 < end; q0 += G * U) {
        uint32_t pp[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t q = q0 + u * G + mem;
          pp[u] = q < end ? A.csc_perm[pb + q] : 0xffffffffu;
        }
        uint32_t jf[U];
        float pc[U], pbv[U], cv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool v = pp[u] != 0xffffffffu;
          jf[u] = v ? A.csr_jf[pb + pp[u]] : 0u;
          pc[u] = v ? A.pcol[pb + pp[u]] : 0.f;
          pbv[u] = v ? A.pbar[pb + pp[u]] : 0.f;
          cv[u] = v ? A.cs[pb + pp[u]] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!(jf[u] & kFlagCol)) continue;
          const double zb = (double)pc[u] * (0.5 * (double)pbv[u] - S);
          szb += zb;
          Tbar -= zb * ((double)cv[u] - (double)lb.m);
        }
      }
      szb = gsum<G>(szb);
      Tbar = gsum<G>(Tbar);
      const double mbar = (double)lb.T * szb;
      const double gbar = (lb.flags & kLineClamped) ? 0.0 : -Tbar * (double)lb.T / (double)lb.g;
      out = {(float)S, (float)(mbar - gbar), (float)gbar, lb.T};
    }
    if (mem == 0) A.colback[(size_t)b * M + j] = out;
  }
}

// cbar per entry and the Eq. (5) scatter into grad_pred (overwrites).
template <int G, int U>
__device__ void grad_rows(const SparseArgs& A, int b, Slice s, const LongList& ll) {
  const int N = A.N, M = A.M, L = A.L;
  const size_t pb = (size_t)b * A.cap;
  const unsigned* rp = A.row_ptr + (size_t)b * (N + 1);
  const float gl = A.grad_loss[b];
  const float* aL = A.a_hist + ((size_t)b * (L + 1) + L) * N;
  const float* bL = A.b_hist + ((size_t)b * (L + 1) + L) * M;
  const int mem = G == 1 ? 0 : (threadIdx.x & 31);
  APML_FOR_LINES(G, s, ll, i) {
    const uint32_t beg = rp[i], end = rp[i + 1];
    if (!line_mine<G>(end - beg)) continue;
    const float4 x = A.pred4[(size_t)b * N + i];
    LineBack rbk = {0.f, 0.f, 0.f, 0.f};
    int2 ri = make_int2(-1, -1);
    if (A.full) { rbk = A.rowback[(size_t)b * N + i]; ri = A.rowidx[(size_t)b * N + i]; }
    const double ai = (double)aL[i];
    double gx = 0.0, gy = 0.0, gz = 0.0;
    for (uint32_t p0 = beg; p0 < end; p0 += G * U) {
      uint32_t jf[U];
      float cv[U], p0v[U], pbv[U], prv[U], pcv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t p = p0 + u * G + mem;
        const bool v = p < end;
        jf[u] = v ? A.csr_jf[pb + p] : 0u;
        cv[u] = v ? A.cs[pb + p] : 1.f;
        p0v[u] = v ? A.P0[pb + p] : 0.f;
        if (A.full) {
          pbv[u] = v ? A.pbar[pb + p] : 0.f;
          prv[u] = v ? A.prow[pb + p] : 0.f;
          pcv[u] = v ? A.pcol[pb + p] : 0.f;
        }
      }
      float4 y[U];
      float bLv[U];
      int2 ci[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool v = p0 + u * G + mem < end;
        const uint32_t j = jf[u] & kIdxMask;
        y[u] = v ? A.gt4[(size_t)b * M + j] : x;
        bLv[u] = v ? bL[j] : 0.f;
        ci[u] = (v && A.full) ? A.colidx[(size_t)b * M + j] : make_int2(-1, -1);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (p0 + u * G + mem >= end) continue;
        const uint32_t j = jf[u] & kIdxMask;
        double cbar = (double)gl * ai * (double)p0v[u] * (double)bLv[u];  // d loss / d c = v
        if (A.full) {
          const double hp = 0.5 * (double)pbv[u];
          if (jf[u] & kFlagRow) cbar -= (double)rbk.T * (double)prv[u] * (hp - (double)rbk.S);
          if ((int)j == ri.x) cbar += rbk.ca;
          if ((int)j == ri.y) cbar += rbk.cb;
          const bool cf = (jf[u] & kFlagCol) != 0;
          const int gi = i + A.row_offset;  // colidx holds global row indices
          if (cf || ci[u].x == gi || ci[u].y == gi) {
            const LineBack cbk = A.colback[(size_t)b * M + j];
            if (cf) cbar -= (double)cbk.T * (double)pcv[u] * (hp - (double)cbk.S);
            if (ci[u].x == gi) cbar += cbk.ca;
            if (ci[u].y == gi) cbar += cbk.cb;
          }
        }
        const double w = cbar / ((double)cv[u] + (double)A.eps_dist);  // Eq. (5)
        if (A.gw) A.gw[pb + p0 + u * G + mem] = (float)w;
        gx += w * ((double)x.x - (double)y[u].x);
        gy += w * ((double)x.y - (double)y[u].y);
        gz += w * ((double)x.z - (double)y[u].z);
      }
    }
    gx = gsum<G>(gx);
    gy = gsum<G>(gy);
    gz = gsum<G>(gz);
    if (mem == 0) {
      float* g = A.grad_pred + ((size_t)b * N + orig_row(A, b, (uint32_t)i)) * 3;
      g[0] = (float)gx; g[1] = (float)gy; g[2] = (float)gz;
    }
  }
}

// abar_i = gl sum_j P0 b^L c (rows) and bbar_j = gl sum_i a^L P0 c (columns), own slices.
template <int G, int U>
__device__ void bwd_init_rows(const SparseArgs& A, int b, Slice s, const LongList& ll, float* ab) {
  const int N = A.N, M = A.M, L = A.L;
  const size_t pb = (size_t)b * A.cap;
  const unsigned* rp = A.row_ptr + (size_t)b * (N + 1);
  const float* bL = A.b_hist + ((size_t)b * (L + 1) + L) * M;
  const double gl = (double)A.grad_loss[b];
  const int mem = G == 1 ? 0 : (threadIdx.x & 31);
  APML_FOR_LINES(G, s, ll, i) {
    const uint32_t beg = rp[i], end = rp[i + 1];
    if (!line_mine<G>(end - beg)) continue;
    double t = 0.0;
    for (uint32_t p0 = beg; p0 < end; p0 += G * U) {
      uint32_t jf[U];
      float pv[U], cv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t p = p0 + u * G + mem;
        const bool v = p < end;
        jf[u] = v ? A.csr_jf[pb + p] : 0u;
        pv[u] = v ? A.P0[pb + p] : 0.f;
        cv[u] = v ? A.cs[pb + p] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (p0 + u * G + mem < end) t += (double)pv[u] * (double)bL[jf[u] & kIdxMask] * (double)cv[u];
    }
    t = gsum<G>(t);
    if (mem == 0) ab[i - s.lo] = (float)(gl * t);
  }
}

template <int G, int U>
__device__ void bwd_init_cols(const SparseArgs& A, int b, Slice s, const LongList& ll, float* bb) {
  const int N = A.N, M = A.M, L = A.L;
  const size_t pb = (size_t)b * A.cap;
  const unsigned* cp = A.col_ptr + (size_t)b * (M + 1);
  const float* aL = A.a_hist + ((size_t)b * (L + 1) + L) * N;
  const double gl = (double)A.grad_loss[b];
  const int mem = G == 1 ? 0 : (threadIdx.x & 31);
  APML_FOR_LINES(G, s, ll, j) {
    const uint32_t beg = cp[j], end = cp[j + 1];
    if (!line_mine<G>(end - beg)) continue;
    double t = 0.0;
    for (uint32_t q0 = beg; q0 < end; q0 += G * U) {
      uint32_t ii[U], pp[U];
      float pv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t q = q0 + u * G + mem;
        const bool v = q < end;
        ii[u] = v ? A.csc_i[pb + q] : 0u;
        pp[u] = v ? A.csc_perm[pb + q] : 0u;
        pv[u] = v ? A.P0c[pb + q] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q0 + u * G + mem < end) t += (double)aL[ii[u]] * (double)pv[u] * (double)A.cs[pb + pp[u]];
    }
    t = gsum<G>(t);
    if (mem == 0) bb[j - s.lo] = (float)(gl * t);
  }
}

template <typename IdxT>
__global__ void __launch_bounds__(kMegaThreads, 1) k_sparse_bwd(const SparseArgs A) {
  pdl_trigger();
  pdl_wait();  // the forward's saved state first
  extern __shared__ __align__(16) uint8_t shm[];
  cg::cluster_group cl = cg::this_cluster();
  const int CL = cl.num_blocks(), rank = cl.block_rank();
  const int b = blockIdx.x / CL;
  const int N = A.N, M = A.M, L = A.L;
  const size_t pb = (size_t)b * A.cap;
  const Slice sr = slice_of(N, rank, CL), sc = slice_of(M, rank, CL);
  if (A.cursor[b] > A.cap) {
    const float nan = __int_as_float(0x7fc00000);
    for (int i = sr.lo + threadIdx.x; i < sr.hi; i += blockDim.x) {
      float* g = A.grad_pred + ((size_t)b * N + i) * 3;
      g[0] = nan; g[1] = nan; g[2] = nan;
    }
    return;
  }
  __shared__ uint32_t s_long_r[kLongCap], s_long_c[kLongCap];
  __shared__ int s_nlong[2];
  const LongList llr = collect_long(A.row_ptr + (size_t)b * (N + 1), sr, s_long_r, &s_nlong[0]);
  const LongList llc = collect_long(A.col_ptr + (size_t)b * (M + 1), sc, s_long_c, &s_nlong[1]);
  phase(A, 0);
  if (A.full) {
    const unsigned* rp = A.row_ptr + (size_t)b * (N + 1);
    const unsigned* cp = A.col_ptr + (size_t)b * (M + 1);
    const float gl = A.grad_loss[b];
    const float* aL = A.a_hist + ((size_t)b * (L + 1) + L) * N;
    const float* bL = A.b_hist + ((size_t)b * (L + 1) + L) * M;
    uint8_t* sm = shm;
    float *rcur, *qcur;
    __shared__ __align__(8) unsigned long long s_mbar[2];
    if (A.rep_smem) {
      rcur = reinterpret_cast<float*>(carve(sm, 4 * (size_t)((N + 3) / 4 * 4 + 4)));
      qcur = reinterpret_cast<float*>(carve(sm, 4 * (size_t)((M + 3) / 4 * 4 + 4)));
      if (threadIdx.x == 0) {
        mbar_init(smem_addr(&s_mbar[0]));
        mbar_init(smem_addr(&s_mbar[1]));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
    } else {
      rcur = A.gvec + (size_t)b * 2 * (N + M);
      qcur = rcur + N;
    }
    // abar / bbar of the own slices: shared memory when they fit, else the second half of
    // the pair's global scratch (the first half holds the replicas in global mode)
    float *ab, *bb;
    const bool ab_sm = (size_t)(sm - shm) + 4 * (size_t)(sr.hi - sr.lo + sc.hi - sc.lo) + 64 <= A.smem_bytes;
    if (ab_sm) {
      ab = reinterpret_cast<float*>(carve(sm, 4 * (size_t)(sr.hi - sr.lo)));
      bb = reinterpret_cast<float*>(carve(sm, 4 * (size_t)(sc.hi - sc.lo)));
    } else {
      float* g = A.gvec + (size_t)b * 2 * (N + M) + (N + M);
      ab = g + sr.lo;
      bb = g + N + sc.lo;
    }
    Xchg xr{rcur, smem_addr(&s_mbar[0]), N, A.rep_smem != 0, 0u};
    Xchg xq{qcur, smem_addr(&s_mbar[1]), M, A.rep_smem != 0, 0u};
    xchg_arm(xr);
    xchg_arm(xq);
    float* bls = nullptr;
    if (A.rep_smem && M <= kPf * (int)blockDim.x) bls = reinterpret_cast<float*>(carve(sm, 8 * (size_t)M));
    // abar = gl sum_j P0 b^L c, bbar = gl sum_i a^L P0 c   (loss = sum a P0 b c)
    bwd_init_rows<1, 8>(A, b, sr, llr, ab);
    bwd_init_rows<32, 1>(A, b, sr, llr, ab);
    bwd_init_cols<1, 8>(A, b, sc, llc, bb);
    bwd_init_cols<32, 1>(A, b, sc, llc, bb);
    const size_t used = (size_t)(sm - shm);
    const bool fit = used + slice_bytes(sr.hi - sr.lo, rp[sr.hi] - rp[sr.lo], sizeof(IdxT), true) +
                         slice_bytes(sc.hi - sc.lo, cp[sc.hi] - cp[sc.lo], sizeof(IdxT), false) <= A.smem_bytes;
    // P0bar accumulator starts at the direct term gl a^L_i b^L_j c_ij
    if (fit) {
      const SliceView<IdxT> R = stage_slice<IdxT>(sm, rp, sr, A.csr_jf + pb, A.P0 + pb, true);
      const SliceView<IdxT> C = stage_slice<IdxT>(sm, cp, sc, A.csc_i + pb, A.P0c + pb, false);
      __syncthreads();  // offsets staged by other threads
      const float* csl = A.cs + pb + rp[sr.lo];
      for (int i = sr.lo + threadIdx.x; i < sr.hi; i += blockDim.x) {
        const int k = i - sr.lo;
        const float ga = gl * aL[i];
        for (uint32_t p0 = R.off[k], p1 = R.off[k + 1]; p0 < p1; p0 += 8) {
          float bv[8], cv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            bv[u] = p0 + u < p1 ? bL[R.col(p0 + u)] : 0.f;
            cv[u] = p0 + u < p1 ? csl[p0 + u] : 0.f;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (p0 + u < p1) R.acc[p0 + u] = ga * bv[u] * cv[u];
        }
      }
      // stage the Sinkhorn history (own rows of a, all of b) when it fits
      float *ahs = nullptr, *bhs = nullptr;
      const int nr = sr.hi - sr.lo;
      if ((size_t)(sm - shm) + 4 * (size_t)(L + 1) * (nr + M) + 64 <= A.smem_bytes) {
        ahs = reinterpret_cast<float*>(carve(sm, 4 * (size_t)(L + 1) * nr));
        bhs = reinterpret_cast<float*>(carve(sm, 4 * (size_t)(L + 1) * M));
        const float* ahg = A.a_hist + (size_t)b * (L + 1) * N;
        const float* bhg = A.b_hist + (size_t)b * (L + 1) * M;
        for (int l = 0; l <= L; ++l) g2s_async(ahs + (size_t)l * nr, ahg + (size_t)l * N + sr.lo, nr);
        g2s_async(bhs, bhg, (size_t)(L + 1) * M);
        cp_async_wait_all();
      }
      csync(cl);
      phase(A, 1);
      const bool all_sm = A.rep_smem && ahs && bhs && ab_sm;
      if (all_sm) sinkhorn_bwd<IdxT, true>(cl, A, b, sr, sc, R, C, ab, bb, xr, xq, bls, ahs, bhs, llr, llc);
      else sinkhorn_bwd<IdxT, false>(cl, A, b, sr, sc, R, C, ab, bb, xr, xq, bls, ahs, bhs, llr, llc);
      const uint32_t base = rp[sr.lo], cnt = rp[sr.hi] - base;
      for (uint32_t k = threadIdx.x; k < cnt; k += blockDim.x) A.pbar[pb + base + k] = R.acc[k];
    } else {
      const SliceView<uint32_t> R{rp + sr.lo, A.csr_jf + pb, A.P0 + pb, A.pbar + pb};
      const SliceView<uint32_t> C{cp + sc.lo, A.csc_i + pb, A.P0c + pb, nullptr};
      for (int i = sr.lo + threadIdx.x; i < sr.hi; i += blockDim.x)
        for (uint32_t p = rp[i]; p < rp[i + 1]; ++p)
          A.pbar[pb + p] = gl * aL[i] * bL[A.csr_jf[pb + p] & kIdxMask] * A.cs[pb + p];
      csync(cl);
      phase(A, 1);
      sinkhorn_bwd<uint32_t, false>(cl, A, b, sr, sc, R, C, ab, bb, xr, xq, bls, nullptr, nullptr, llr, llc);
    }
    __syncthreads();
    phase(A, 2);
    row_soft_rev<1, 8>(A, b, sr, llr);
    row_soft_rev<32, 1>(A, b, sr, llr);
    csync(cl);
    phase(A, 3);
    col_soft_rev<1, 8>(A, b, sc, llc);
    col_soft_rev<32, 1>(A, b, sc, llc);
    csync(cl);
    phase(A, 4);
  }
  grad_rows<1, 4>(A, b, sr, llr);
  grad_rows<32, 1>(A, b, sr, llr);
  phase(A, 5);
}

// Gradient with respect to gt: the loss depends on y only through the costs
// c_ij, so by Eq. (5) with the roles of x and y exchanged (dc/dy_j = -(x_i - y_j) / c_ij),
//   ybar_j = - sum_i w_ij (x_i - y_j),   w_ij = cbar_ij / (c_ij + eps_dist),
// with the per-entry weights w written by grad_rows (CSR order) and summed here over each
// column's CSC segment in sorted order (deterministic).  Thread per column, all pairs.
__global__ void __launch_bounds__(256) k_grad_gt(const SparseArgs A) {
  const int b = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
  const int N = A.N, M = A.M;
  if (j >= M) return;
  float* g = A.grad_gt + ((size_t)b * M + orig_col(A, b, (uint32_t)j)) * 3;
  if (A.cursor[b] > A.cap) {
    const float nan = __int_as_float(0x7fc00000);
    g[0] = nan; g[1] = nan; g[2] = nan;
    return;
  }
  const size_t pb = (size_t)b * A.cap;
  const unsigned* cp = A.col_ptr + (size_t)b * (M + 1);
  const float4 y = A.gt4[(size_t)b * M + j];
  double gx = 0.0, gy = 0.0, gz = 0.0;
  for (unsigned q = cp[j]; q < cp[j + 1]; ++q) {
    const float4 x = A.pred4[(size_t)b * N + A.csc_i[pb + q]];
    const double w = (double)A.gw[pb + A.csc_perm[pb + q]];
    gx -= w * ((double)x.x - (double)y.x);
    gy -= w * ((double)x.y - (double)y.y);
    gz -= w * ((double)x.z - (double)y.z);
  }
  g[0] = (float)gx; g[1] = (float)gy; g[2] = (float)gz;
}

}  // namespace apml
