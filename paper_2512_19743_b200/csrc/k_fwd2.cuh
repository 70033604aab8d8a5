// k_fwd2.cuh -- the sparse forward of one pair per thread-block cluster,
// built in SHARED memory.
//
// Every CTA of the cluster owns a slice of the pair's rows and of its columns (as k_mega.cuh).
// Instead of a global counting sort (atomics on global counters, scattered 4-byte stores) and
// per-entry gathers between the row and column phases through global memory, each CTA
//   1. scans the emit counts of its own lines (block scan; slice totals exchanged via DSMEM),
//   2. reads ALL emitted entries of its pair (coalesced) and buckets the ones of its own rows
//      (CSR) and own columns (CSC) into shared memory with shared-memory atomics,
//   3. sorts every line by the ORIGINAL index of the other cloud (deterministic order, R12),
//   4. runs the row softmax of its rows and the column softmax of its columns in ONE phase
//      (both read only coordinates and line constants) and exchanges the normalisers 1/Z,
//      1/Z' as replicated vectors through DSMEM (the same mechanism as the Sinkhorn vectors),
//   5. forms P0 = (P_row + P_col)/2 for its CSR entries AND its CSC entries, each
//      side re-evaluating the other side's similarity exp(-T (c - m)) from the same fp32
//      operands with the same rounding (explicit _rn intrinsics, one shared helper), so the two
//      copies are bitwise equal without any per-entry exchange,
//   6. runs Sinkhorn (sinkhorn_fwd of k_mega.cuh) on the shared-memory slices and the loss,
//   7. writes the CSR / CSC arrays the backward and the introspection calls read (coalesced).
// Per-entry global traffic drops from ~12 scattered transactions to ~4 coordinate / line-
// constant gathers (L1/L2-resident) + coalesced copies.  A CTA whose slice does not fit in
// shared memory runs the same code on the global arrays.

#pragma once
#include "k_mega.cuh"

namespace apml {

// Unnormalised similarity of an entry on a line (Eq. (1)): exp(-T (c - m)), or 1 on a
// K = 1 line.  ONE definition for both sides of P0 (bitwise-equal CSR and CSC copies).
__device__ __forceinline__ float line_sim(float c, const LineB& lb) {
  return (lb.flags & kLineK1) ? 1.f : expf(__fmul_rn(-lb.T, __fsub_rn(c, lb.m)));
}
__device__ __forceinline__ float sym_p0(float prow, float pcol) {  // (P_row + P_col) / 2
  return __fmul_rn(0.5f, __fadd_rn(prow, pcol));
}

// Exclusive block scan of cnt[0, n) into off[0, n]; returns the total (all threads).
__device__ unsigned block_scan(const unsigned* cnt, int n, unsigned* off, unsigned* s_warp) {
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int beg = threadIdx.x * per, end = min(n, beg + per);
  unsigned v[8];
  unsigned sum = 0;
  if (per <= 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = beg + u < end ? cnt[beg + u] : 0u;
#pragma unroll
    for (int u = 0; u < 8; ++u) sum += v[u];
  } else {
    for (int k = beg; k < end; ++k) sum += cnt[k];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_warp[w] = inc;
  __syncthreads();
  if (w == 0) {
    unsigned t = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned q = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += q;
    }
    s_warp[lane] = t;
  }
  __syncthreads();
  unsigned run = inc - sum + (w ? s_warp[w - 1] : 0u);
  if (per <= 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (beg + u < end) { off[beg + u] = run; run += v[u]; }
  } else {
    for (int k = beg; k < end; ++k) { off[k] = run; run += cnt[k]; }
  }
  const unsigned total = s_warp[(blockDim.x >> 5) - 1];
  if (threadIdx.x == 0) off[n] = total;
  __syncthreads();  // s_warp reused by the next scan; off complete
  return total;
}

// Lines of a slice longer than kRegLine (local offsets), as collect_long.
__device__ LongList collect_long_local(const unsigned* off, Slice s, uint32_t* list, int* cnt,
                                       uint32_t thresh = kRegLine) {
  if (threadIdx.x == 0) *cnt = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < s.hi - s.lo; k += blockDim.x)
    if (off[k + 1] - off[k] > thresh) {
      const int q = atomicAdd(cnt, 1);
      if (q < kLongCap) list[q] = (uint32_t)(s.lo + k);
    }
  __syncthreads();
  const int n = *cnt;
  return LongList{list, n < kLongCap ? n : kLongCap, s.lo, s.hi, n > kLongCap};
}

// One side (CSR rows or CSC columns) of a CTA's slice.  idx: other-cloud index | flags;
// t: emit-buffer index (only until the CSC side has read the CSR positions), reused as c;
// val: P0; pr: unnormalised similarity of this side's softmax, then this side's P (CSR:
// P_row, CSC: P_col).
struct Side {
  unsigned* off;  // [n + 1] local offsets
  uint32_t* idx;
  uint32_t* t;
  float* c;       // aliases t
  float* val;
  float* pr;
};

// In-place sort of the entries [beg, beg + L) of a line by ORIGINAL index of the other cloud
// (keys are distinct on a line).  kRows: key = orig_col(j), also records the CSR position of
// each entry in A.inv (by emit index).  G == 1: L <= kRegLine, registers; G == 32: warp, L <= 32
// by a shuffle rank count, up to 256 with 8 entries per lane in registers, longer by bitonic sort.
template <bool kRows>
__device__ __forceinline__ uint32_t sort_key(const SparseArgs& A, int b, uint32_t idx) {
  return kRows ? orig_col(A, b, idx & kIdxMask) : orig_row(A, b, idx & kIdxMask);
}

template <bool kRows, uint32_t KR = kRegLine>
__device__ void sort_line_regs(const SparseArgs& A, int b, const Side& S, uint32_t beg, uint32_t L, uint32_t gbase) {
  uint32_t ix[KR], tt[KR], ok[KR];
#pragma unroll
  for (uint32_t k = 0; k < KR; ++k) {
    ix[k] = k < L ? S.idx[beg + k] : 0u;
    tt[k] = k < L ? S.t[beg + k] : 0u;
  }
#pragma unroll
  for (uint32_t k = 0; k < KR; ++k) ok[k] = k < L ? sort_key<kRows>(A, b, ix[k]) : 0xffffffffu;
#pragma unroll
  for (uint32_t k = 0; k < KR; ++k) {
    uint32_t r = 0;
#pragma unroll
    for (uint32_t f = 0; f < KR; ++f) r += (ok[f] < ok[k]) ? 1u : 0u;
    if (k < L) {
      S.idx[beg + r] = ix[k];
      S.t[beg + r] = tt[k];
      if (kRows) A.inv[(size_t)b * A.cap + tt[k]] = gbase + beg + r;
    }
  }
}

template <bool kRows>
__device__ void sort_line_warp(const SparseArgs& A, int b, const Side& S, uint32_t beg, uint32_t L, uint32_t gbase) {
  const int lane = threadIdx.x & 31;
  if (L <= 32) {
    const uint32_t ix = lane < (int)L ? S.idx[beg + lane] : 0u;
    const uint32_t tt = lane < (int)L ? S.t[beg + lane] : 0u;
    const uint32_t key = lane < (int)L ? sort_key<kRows>(A, b, ix) : 0xffffffffu;
    uint32_t r = 0;
    for (uint32_t k = 0; k < L; ++k) r += (__shfl_sync(0xffffffffu, key, k) < key) ? 1u : 0u;
    __syncwarp();
    if (lane < (int)L) {
      S.idx[beg + r] = ix;
      S.t[beg + r] = tt;
      if (kRows) A.inv[(size_t)b * A.cap + tt] = gbase + beg + r;
    }
    __syncwarp();
    return;
  }
  constexpr uint32_t kSlots = 8;  // entries per lane held in registers: L <= 256
  if (L <= 32 * kSlots) {
    uint32_t ix[kSlots], tt[kSlots], rk[kSlots], key[kSlots];
#pragma unroll
    for (uint32_t u = 0; u < kSlots; ++u) {
      const uint32_t p = lane + 32 * u;
      ix[u] = p < L ? S.idx[beg + p] : 0u;
      tt[u] = p < L ? S.t[beg + p] : 0u;
      key[u] = p < L ? sort_key<kRows>(A, b, ix[u]) : 0xffffffffu;
      rk[u] = 0u;
    }
    // rank = number of smaller keys on the line; the keys are broadcast 32 at a time
#pragma unroll
    for (uint32_t v = 0; v < kSlots; ++v) {
      if (32 * v >= L) break;
      for (uint32_t q = 0; q < 32 && 32 * v + q < L; ++q) {
        const uint32_t kq = __shfl_sync(0xffffffffu, key[v], q);
#pragma unroll
        for (uint32_t u = 0; u < kSlots; ++u) rk[u] += (kq < key[u]) ? 1u : 0u;
      }
    }
    __syncwarp();
#pragma unroll
    for (uint32_t u = 0; u < kSlots; ++u) {
      if (lane + 32 * u < L) {
        S.idx[beg + rk[u]] = ix[u];
        S.t[beg + rk[u]] = tt[u];
        if (kRows) A.inv[(size_t)b * A.cap + tt[u]] = gbase + beg + rk[u];
      }
    }
    __syncwarp();
    return;
  }
  // > 256 entries (outlier points whose line is nearly flat; seen at C3): in-place bitonic
  // sort over the next power of two with ascending comparators only, so the virtual +inf
  // elements beyond L never move (O(L log^2 L), deterministic)
  uint32_t n2 = 1;
  while (n2 < L) n2 <<= 1;
  for (uint32_t k = 2; k <= n2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t q = lane; q < n2 / 2; q += 32) {
        // q-th pair of this step: i has bit j clear; partner = i ^ (k - 1) (flip) or i ^ j
        const uint32_t i = ((q & ~(j - 1)) << 1) | (q & (j - 1));
        const uint32_t pi = (j == (k >> 1)) ? (i ^ (k - 1)) : (i ^ j);
        const uint32_t lo = min(i, pi), hi = max(i, pi);
        if (hi < L) {
          const uint32_t a = S.idx[beg + lo], c = S.idx[beg + hi];
          if (sort_key<kRows>(A, b, a) > sort_key<kRows>(A, b, c)) {
            const uint32_t ta = S.t[beg + lo];
            S.idx[beg + lo] = c;
            S.idx[beg + hi] = a;
            S.t[beg + lo] = S.t[beg + hi];
            S.t[beg + hi] = ta;
          }
        }
      }
      __syncwarp();
    }
  }
  if (kRows)
    for (uint32_t k = lane; k < L; k += 32) A.inv[(size_t)b * A.cap + S.t[beg + k]] = gbase + beg + k;
  __syncwarp();
}

// Softmax of one line on its kept support, entries in sorted order.  kRows:
// row i of pred (other cloud gt, flag kFlagRow); else column j of gt.  Writes c and the
// unnormalised similarity per entry, the argmin / second-argmin indices (R12) and returns Z.
// G == 1: thread per line (L <= kRegLine, one batched gather); G == 32: warp per line.
template <bool kRows, int G>
__device__ float line_softmax(const SparseArgs& A, int b, const Side& S, int line, int k, int2* argidx) {
  const int N = A.N, M = A.M;
  const uint32_t beg = S.off[k], L = S.off[k + 1] - beg;
  const float4 own = kRows ? A.pred4[(size_t)b * N + line] : A.gt4[(size_t)b * M + line];
  const LineA la = kRows ? A.rowA[(size_t)b * N + line] : A.colA[(size_t)b * M + line];
  const LineB lb = kRows ? A.rowB[(size_t)b * N + line] : A.colB[(size_t)b * M + line];
  const uint32_t fl = kRows ? kFlagRow : kFlagCol;
  auto d2_of = [&](uint32_t ix) {
    const uint32_t o = ix & kIdxMask;
    if (kRows) {
      const float4 y = A.gt4[(size_t)b * M + o];
      return dist2(own.x, own.y, own.z, y.x, y.y, y.z);
    }
    const float4 x = A.pred4[(size_t)b * N + o];
    return dist2(x.x, x.y, x.z, own.x, own.y, own.z);  // same operand order as the rows
  };
  if (G == 1) {
    // chunks of 8 entries in sorted order (one batched gather each; most lines need one):
    // half the unrolled code of a 16-wide batch -- this phase runs once per launch, so its
    // instruction fetch (ncu: no_instruction stalls) matters more than a second round trip
    constexpr uint32_t kC = 8;
    int ia = -1, ib = -1;
    float Z = 0.f;
    for (uint32_t r0 = 0; r0 < L; r0 += kC) {
      uint32_t ix[kC];
      float d2[kC];
#pragma unroll
      for (uint32_t r = 0; r < kC; ++r) ix[r] = r0 + r < L ? S.idx[beg + r0 + r] : 0u;
#pragma unroll
      for (uint32_t r = 0; r < kC; ++r) d2[r] = r0 + r < L ? d2_of(ix[r]) : 0.f;
#pragma unroll
      for (uint32_t r = 0; r < kC; ++r) {
        if (r0 + r < L) {
          const int o = (int)(ix[r] & kIdxMask);
          if (ia < 0 && d2[r] == la.m2) ia = o;
          else if (ib < 0 && d2[r] == la.s2) ib = o;
          const float c = __fsqrt_rn(d2[r]);
          float s = 0.f;
          if (ix[r] & fl) {
            s = line_sim(c, lb);
            Z += s;
          }
          S.c[beg + r0 + r] = c;
          S.pr[beg + r0 + r] = s;
        }
      }
    }
    *argidx = make_int2(ia, ib);
    return Z;
  }
  const int lane = threadIdx.x & 31;
  int ka = -1, kb = -1;
  float Z = 0.f;
  for (uint32_t p0 = 0; p0 < L; p0 += 32) {
    const uint32_t p = p0 + lane;
    const bool v = p < L;
    float d2 = 0.f;
    if (v) {
      const uint32_t ix = S.idx[beg + p];
      d2 = d2_of(ix);
      const float c = __fsqrt_rn(d2);
      const float s = (ix & fl) ? line_sim(c, lb) : 0.f;
      Z += s;
      S.c[beg + p] = c;
      S.pr[beg + p] = s;
    }
    first_two(__ballot_sync(0xffffffffu, v && d2 == la.m2), __ballot_sync(0xffffffffu, v && d2 == la.s2), ka, kb,
              (int)p0);
  }
  __syncwarp();
  if (lane == 0)
    *argidx = make_int2(ka >= 0 ? (int)(S.idx[beg + ka] & kIdxMask) : -1,
                        kb >= 0 ? (int)(S.idx[beg + kb] & kIdxMask) : -1);
  return gsum<32>(Z);
}

// P0 of the entries of one line (chunks of 8, gathers before stores).  kRows: CSR entries of
// row i -- own P_row = s * iz_i, P_col re-evaluated from colB[j] and 1/Z'_j; writes P_row and
// P_col (CSR order, global, for the backward) and P0.  Else CSC entries of column j.
// G == 1: one thread per line; G == 32: one warp per (long) line, lane-strided entries.
template <bool kRows, int G = 1>
__device__ void line_p0(const SparseArgs& A, int b, const Side& S, int line, int k, const float* iz_own,
                        const float* iz_oth, uint32_t gbase) {
  const int N = A.N, M = A.M;
  const size_t pb = (size_t)b * A.cap;
  const uint32_t beg = S.off[k], end = S.off[k + 1];
  const uint32_t mem = G == 1 ? 0u : (threadIdx.x & 31);
  const float izl = iz_own[line];
  const uint32_t fo = kRows ? kFlagCol : kFlagRow;  // the OTHER side's flag
  for (uint32_t p0 = beg; p0 < end; p0 += 8 * G) {
    uint32_t ix[8];
    float c[8], s[8];
    LineB lo[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t p = p0 + u * G + mem;
      const bool v = p < end;
      ix[u] = v ? S.idx[p] : 0u;
      c[u] = v ? S.c[p] : 0.f;
      s[u] = v ? S.pr[p] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t o = ix[u] & kIdxMask;
      lo[u] = (p0 + u * G + mem < end && (ix[u] & fo))
                  ? (kRows ? A.colB[(size_t)b * M + o] : A.rowB[(size_t)b * N + o])
                  : LineB{0.f, 0.f, 0.f, 0};
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t p = p0 + u * G + mem;
      if (p >= end) continue;
      const uint32_t o = ix[u] & kIdxMask;
      const float pown = __fmul_rn(s[u], izl);
      const float poth = (ix[u] & fo) ? __fmul_rn(line_sim(c[u], lo[u]), iz_oth[o]) : 0.f;
      const float prow = kRows ? pown : poth, pcol = kRows ? poth : pown;
      S.val[p] = sym_p0(prow, pcol);
      S.pr[p] = pown;  // this side's probability (CSR: P_row, CSC: P_col)
      if (kRows) A.pcol[pb + gbase + p] = pcol;
    }
  }
}

template <typename IdxT, bool kSm>
__device__ void fwd2_sinkhorn(cg::cluster_group& cl, const SparseArgs& A, int b, Slice sr, Slice sc,
                              const unsigned* roff, const IdxT* ridx, const float* rval, const unsigned* coff,
                              const IdxT* cidx, const float* cval, Xchg& xa, Xchg& xb, const LongList& llr,
                              const LongList& llc, const uint16_t* rperm, const uint16_t* cperm) {
  const SliceView<IdxT> RV{roff, ridx, rval, nullptr};
  const SliceView<IdxT> CV{coff, cidx, cval, nullptr};
  sinkhorn_fwd<IdxT, kSm>(cl, A, b, sr, sc, RV, CV, xa, xb, llr, llc, rperm, cperm);
}

__device__ __forceinline__ void sparse_fwd2_body(const SparseArgs& A) {
  extern __shared__ __align__(16) uint8_t shm[];
  __shared__ unsigned s_tot[2][kMaxCluster];
  __shared__ unsigned s_warp[32];
  __shared__ double s_part[kMaxCluster];
  uint32_t* s_long_r = long_lists();
  uint32_t* s_long_c = s_long_r + kLongCap;
  __shared__ int s_nlong[2];
  __shared__ __align__(8) unsigned long long s_mbar[4];
  cg::cluster_group cl = cg::this_cluster();
  const int CL = cl.num_blocks(), rank = cl.block_rank();
  const int b = blockIdx.x / CL;
  const int N = A.N, M = A.M, L = A.L;
  const size_t pb = (size_t)b * A.cap;
  pdl_trigger();
  pdl_wait();  // the emitted support (k_emit)
  const unsigned total = A.cursor[b];
  if (total > A.cap) {  // overflowed pair: uniform across the cluster, no barrier follows
    if (rank == 0 && threadIdx.x == 0) A.loss[b] = __int_as_float(0x7fc00000);
    return;
  }
  const Slice sr = slice_of(N, rank, CL), sc = slice_of(M, rank, CL);
  const int nr = sr.hi - sr.lo, nc = sc.hi - sc.lo;
  unsigned* rp = A.row_ptr + (size_t)b * (N + 1);
  unsigned* cp = A.col_ptr + (size_t)b * (M + 1);
  phase(A, 0);

  // ---- shared memory: 4 replicated line vectors (a, b, 1/Z, 1/Z'), offsets, fill cursors
  uint8_t* sm = shm;
  const size_t vN = 4 * (size_t)((N + 3) / 4 * 4 + 4), vM = 4 * (size_t)((M + 3) / 4 * 4 + 4);
  float* va = reinterpret_cast<float*>(carve(sm, vN));
  float* vb = reinterpret_cast<float*>(carve(sm, vM));
  float* viz = reinterpret_cast<float*>(carve(sm, vN));
  float* vizc = reinterpret_cast<float*>(carve(sm, vM));
  unsigned* roff = reinterpret_cast<unsigned*>(carve(sm, 4 * (size_t)(nr + 1)));
  unsigned* coff = reinterpret_cast<unsigned*>(carve(sm, 4 * (size_t)(nc + 1)));
  unsigned* rcur = reinterpret_cast<unsigned*>(carve(sm, 4 * (size_t)nr));
  unsigned* ccur = reinterpret_cast<unsigned*>(carve(sm, 4 * (size_t)nc));
  // line orders by length for Sinkhorn (slices of <= 65536 lines)
  uint16_t* rperm = (nr <= 65536 && nc <= 65536) ? reinterpret_cast<uint16_t*>(carve(sm, 2 * (size_t)nr)) : nullptr;
  uint16_t* cperm = rperm ? reinterpret_cast<uint16_t*>(carve(sm, 2 * (size_t)nc)) : nullptr;
  __shared__ unsigned s_hist[kRegLine + 2];
  for (int k = threadIdx.x; k < N; k += blockDim.x) va[k] = 1.f;
  for (int k = threadIdx.x; k < M; k += blockDim.x) vb[k] = 1.f;
  for (int k = threadIdx.x; k < nr; k += blockDim.x) rcur[k] = 0u;
  for (int k = threadIdx.x; k < nc; k += blockDim.x) ccur[k] = 0u;
  if (threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q) mbar_init(smem_addr(&s_mbar[q]));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  Xchg xa{va, smem_addr(&s_mbar[0]), N, true, 0u};
  Xchg xb{vb, smem_addr(&s_mbar[1]), M, true, 0u};
  Xchg xz{viz, smem_addr(&s_mbar[2]), N, true, 0u};
  Xchg xzc{vizc, smem_addr(&s_mbar[3]), M, true, 0u};
  xchg_arm(xa);  // first use of each mbarrier; peers start pushing after the next cl.sync
  xchg_arm(xb);
  xchg_arm(xz);
  xchg_arm(xzc);

  // ---- S4a: local scans of the emit counts; slice totals to every CTA of the cluster
  const unsigned nnzr = block_scan(A.row_cnt + (size_t)b * (N + 1) + sr.lo, nr, roff, s_warp);
  const unsigned nnzc = block_scan(A.col_cnt + (size_t)b * (M + 1) + sc.lo, nc, coff, s_warp);
  if (threadIdx.x < CL) {
    cl.map_shared_rank(&s_tot[0][0], (int)threadIdx.x)[rank] = nnzr;
    cl.map_shared_rank(&s_tot[1][0], (int)threadIdx.x)[rank] = nnzc;
  }
  csync(cl);
  unsigned gr = 0, gc = 0;  // global CSR / CSC offsets of this CTA's slices
  for (int r = 0; r < rank; ++r) { gr += s_tot[0][r]; gc += s_tot[1][r]; }
  for (int k = threadIdx.x; k < nr; k += blockDim.x) rp[sr.lo + k] = gr + roff[k];
  for (int k = threadIdx.x; k < nc; k += blockDim.x) cp[sc.lo + k] = gc + coff[k];
  if (rank == CL - 1 && threadIdx.x == 0) { rp[N] = gr + nnzr; cp[M] = gc + nnzc; }
  phase(A, 1);

  // per-entry arrays: shared memory when both sides fit, else the global arrays at the
  // slices' global offsets (csr_jf / csr_t / P0 / prow; csc_i / csc_t / P0c / pbar as scratch)
  const size_t used = (size_t)(sm - shm);
  auto a16 = [](size_t v) { return (v + 15) & ~size_t(15); };
  const bool fit = used + 4 * (a16(4 * (size_t)nnzr) + a16(4 * (size_t)nnzc)) <= A.smem_bytes;
  Side R, C;
  R.off = roff;
  C.off = coff;
  if (fit) {
    R.idx = reinterpret_cast<uint32_t*>(carve(sm, 4 * (size_t)nnzr));
    R.t = reinterpret_cast<uint32_t*>(carve(sm, 4 * (size_t)nnzr));
    R.val = reinterpret_cast<float*>(carve(sm, 4 * (size_t)nnzr));
    R.pr = reinterpret_cast<float*>(carve(sm, 4 * (size_t)nnzr));
    C.idx = reinterpret_cast<uint32_t*>(carve(sm, 4 * (size_t)nnzc));
    C.t = reinterpret_cast<uint32_t*>(carve(sm, 4 * (size_t)nnzc));
    C.val = reinterpret_cast<float*>(carve(sm, 4 * (size_t)nnzc));
    C.pr = reinterpret_cast<float*>(carve(sm, 4 * (size_t)nnzc));
  } else {
    R.idx = A.csr_jf + pb + gr;
    R.t = reinterpret_cast<uint32_t*>(A.cs + pb + gr);  // emit indices, then c (R.c aliases R.t)
    R.val = A.P0 + pb + gr;
    R.pr = A.prow + pb + gr;
    C.idx = A.csc_i + pb + gc;
    C.t = reinterpret_cast<uint32_t*>(A.csc_c + pb + gc);
    C.val = A.P0c + pb + gc;
    C.pr = A.pbar + pb + gc;
  }
  R.c = reinterpret_cast<float*>(R.t);
  C.c = reinterpret_cast<float*>(C.t);

  // ---- S4b: bucket every emitted entry of the pair into own rows / own columns
  {
    constexpr int kU = 4;
    const uint32_t bd = blockDim.x;
    for (uint32_t t0 = threadIdx.x; t0 < total; t0 += kU * bd) {
      uint2 e[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) e[u] = t0 + u * bd < total ? ebuf_of(A, b)[t0 + u * bd] : make_uint2(~0u, ~0u);
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t t = t0 + u * bd;
        if (t >= total) continue;
        const uint32_t li = e[u].x - (uint32_t)sr.lo, lj = (e[u].y & kIdxMask) - (uint32_t)sc.lo;
        if (li < (uint32_t)nr) {
          const uint32_t p = roff[li] + atomicAdd(rcur + li, 1u);
          R.idx[p] = e[u].y;
          R.t[p] = t;
        }
        if (lj < (uint32_t)nc) {
          const uint32_t q = coff[lj] + atomicAdd(ccur + lj, 1u);
          C.idx[q] = e[u].x | (e[u].y & ~kIdxMask);
          C.t[q] = t;
        }
      }
    }
  }
  __syncthreads();
  phase(A, 2);

  // ---- S4c: order every line by original index of the other cloud (CSR: also A.inv).
  // Lines of <= 8 entries (most) by one thread in registers (8 x 8 rank counts: a quarter of
  // the once-per-launch code of 16 x 16), longer ones by a warp.
  // (mean line length > 6 entries, e.g. the MM-Fi columns of C3: the 16-wide register path,
  // so that the warp path stays rare)
  {
    const bool narrow = (uint64_t)(nnzr + nnzc) <= 6ull * (uint64_t)(nr + nc);
    const uint32_t kSortReg = narrow ? 8u : kRegLine;
    const LongList slr = collect_long_local(roff, sr, s_long_r, &s_nlong[0], kSortReg);
    const LongList slc = collect_long_local(coff, sc, s_long_c, &s_nlong[1], kSortReg);
    for (int k = threadIdx.x; k < nr; k += blockDim.x) {
      const uint32_t beg = roff[k], Ln = roff[k + 1] - beg;
      if (Ln > kSortReg) continue;
      if (narrow) sort_line_regs<true, 8>(A, b, R, beg, Ln, gr);
      else sort_line_regs<true>(A, b, R, beg, Ln, gr);
    }
    for (int k = threadIdx.x; k < nc; k += blockDim.x) {
      const uint32_t beg = coff[k], Ln = coff[k + 1] - beg;
      if (Ln > kSortReg) continue;
      if (narrow) sort_line_regs<false, 8>(A, b, C, beg, Ln, gc);
      else sort_line_regs<false>(A, b, C, beg, Ln, gc);
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int q = w; q < slr.count(); q += nw) {
      const int k = slr.line(q) - sr.lo;
      const uint32_t beg = roff[k], Ln = roff[k + 1] - beg;
      if (Ln > kSortReg) sort_line_warp<true>(A, b, R, beg, Ln, gr);
    }
    for (int q = w; q < slc.count(); q += nw) {
      const int k = slc.line(q) - sc.lo;
      const uint32_t beg = coff[k], Ln = coff[k + 1] - beg;
      if (Ln > kSortReg) sort_line_warp<false>(A, b, C, beg, Ln, gc);
    }
  }
  csync(cl);  // A.inv complete for the whole pair
  // the long-line lists of the later phases (lines of more than kRegLine entries)
  const LongList llr = collect_long_local(roff, sr, s_long_r, &s_nlong[0]);
  const LongList llc = collect_long_local(coff, sc, s_long_c, &s_nlong[1]);
  phase(A, 3);
  // CSR position of every CSC entry (the backward's column passes); frees C.t for c
  for (uint32_t q0 = threadIdx.x; q0 < nnzc; q0 += 4 * blockDim.x) {
    uint32_t tt[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) tt[u] = q0 + u * blockDim.x < nnzc ? C.t[q0 + u * blockDim.x] : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) tt[u] = q0 + u * blockDim.x < nnzc ? A.inv[pb + tt[u]] : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (q0 + u * blockDim.x < nnzc) A.csc_perm[pb + gc + q0 + u * blockDim.x] = tt[u];
  }
  __syncthreads();
  phase(A, 4);

  // ---- S5: row softmax of own rows and column softmax of own columns; 1/Z exchanged
  {
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
    for (int k = threadIdx.x; k < nr; k += blockDim.x) {
      if (roff[k + 1] - roff[k] > kRegLine) continue;
      const int i = sr.lo + k;
      int2 ai;
      const float Z = line_softmax<true, 1>(A, b, R, i, k, &ai);
      A.rowidx[(size_t)b * N + i] = ai;
      xchg_put(xz, CL, i, 1.f / Z);
    }
    for (int k = threadIdx.x; k < nc; k += blockDim.x) {
      if (coff[k + 1] - coff[k] > kRegLine) continue;
      const int j = sc.lo + k;
      int2 ai;
      const float Z = line_softmax<false, 1>(A, b, C, j, k, &ai);
      A.colidx[(size_t)b * M + j] = ai;
      xchg_put(xzc, CL, j, 1.f / Z);
    }
    for (int q = w; q < llr.count(); q += nw) {
      const int i = llr.line(q), k = i - sr.lo;
      if (roff[k + 1] - roff[k] <= kRegLine) continue;
      int2 ai;
      const float Z = line_softmax<true, 32>(A, b, R, i, k, &ai);
      if (lane == 0) {
        A.rowidx[(size_t)b * N + i] = ai;
        xchg_put(xz, CL, i, 1.f / Z);
      }
    }
    for (int q = w; q < llc.count(); q += nw) {
      const int j = llc.line(q), k = j - sc.lo;
      if (coff[k + 1] - coff[k] <= kRegLine) continue;
      int2 ai;
      const float Z = line_softmax<false, 32>(A, b, C, j, k, &ai);
      if (lane == 0) {
        A.colidx[(size_t)b * M + j] = ai;
        xchg_put(xzc, CL, j, 1.f / Z);
      }
    }
  }
  xchg_end(cl, xz, CL, rank);
  xchg_end(cl, xzc, CL, rank);
  phase(A, 5);
  // P0 = (P_row + P_col) / 2 on both sides (bitwise-equal copies)
  for (int k = threadIdx.x; k < nr; k += blockDim.x)
    if (roff[k + 1] - roff[k] <= kRegLine) line_p0<true>(A, b, R, sr.lo + k, k, viz, vizc, gr);
  for (int k = threadIdx.x; k < nc; k += blockDim.x)
    if (coff[k + 1] - coff[k] <= kRegLine) line_p0<false>(A, b, C, sc.lo + k, k, vizc, viz, gc);
  {
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int q = w; q < llr.count(); q += nw) {
      const int k = llr.line(q) - sr.lo;
      if (roff[k + 1] - roff[k] > kRegLine) line_p0<true, 32>(A, b, R, sr.lo + k, k, viz, vizc, gr);
    }
    for (int q = w; q < llc.count(); q += nw) {
      const int k = llc.line(q) - sc.lo;
      if (coff[k + 1] - coff[k] > kRegLine) line_p0<false, 32>(A, b, C, sc.lo + k, k, vizc, viz, gc);
    }
  }
  // Sinkhorn history at l = 0
  float* ah = A.a_hist + (size_t)b * (L + 1) * N;
  float* bh = A.b_hist + (size_t)b * (L + 1) * M;
  for (int k = sr.lo + threadIdx.x; k < sr.hi; k += blockDim.x) ah[k] = 1.f;
  for (int k = sc.lo + threadIdx.x; k < sc.hi; k += blockDim.x) bh[k] = 1.f;
  __syncthreads();
  // this side's probabilities are final: write them now and reuse their shared memory for
  // 16-bit copies of the indices (half the shared-memory bytes per gather in Sinkhorn)
  const bool idx16 = fit && N <= 65536 && M <= 65536;
  if (fit) {
    for (uint32_t p = threadIdx.x; p < nnzr; p += blockDim.x) A.prow[pb + gr + p] = R.pr[p];
    for (uint32_t q = threadIdx.x; q < nnzc; q += blockDim.x) A.csc_pc[pb + gc + q] = C.pr[q];
    __syncthreads();
  }
  uint16_t* r16 = reinterpret_cast<uint16_t*>(R.pr);
  uint16_t* c16 = reinterpret_cast<uint16_t*>(C.pr);
  if (idx16) {
    for (uint32_t p = threadIdx.x; p < nnzr; p += blockDim.x) r16[p] = (uint16_t)(R.idx[p] & kIdxMask);
    for (uint32_t q = threadIdx.x; q < nnzc; q += blockDim.x) c16[q] = (uint16_t)(C.idx[q] & kIdxMask);
    __syncthreads();
  }
  // (single-CTA clusters only: with DSMEM peers the pushes of a warp must stay on consecutive
  // addresses -- scattered st.async made the exchange slower than the saved loads, measured)
  if (CL > 1) rperm = cperm = nullptr;
  if (rperm) {
    line_perm(roff, nr, rperm, s_hist);
    line_perm(coff, nc, cperm, s_hist);
  }
  phase(A, 6);

  // ---- S6: Sinkhorn, L_iter x {Eq. (3), Eq. (4)}
  if (idx16) fwd2_sinkhorn<uint16_t, true>(cl, A, b, sr, sc, roff, r16, R.val, coff, c16, C.val, xa, xb, llr, llc, rperm, cperm);
  else if (fit) fwd2_sinkhorn<uint32_t, true>(cl, A, b, sr, sc, roff, R.idx, R.val, coff, C.idx, C.val, xa, xb, llr, llc, rperm, cperm);
  else fwd2_sinkhorn<uint32_t, false>(cl, A, b, sr, sc, roff, R.idx, R.val, coff, C.idx, C.val, xa, xb, llr, llc, rperm, cperm);
  phase(A, 7);

  // ---- S7: loss_b = sum_i a_i sum_j P0_ij b_j c_ij, own rows, then cluster sum
  double acc = 0.0;
  for (int k = threadIdx.x; k < nr; k += blockDim.x) {
    float t = 0.f;
    for (uint32_t p = roff[k]; p < roff[k + 1]; ++p)
      t = __fmaf_rn(__fmul_rn(R.val[p], vb[R.idx[p] & kIdxMask]), R.c[p], t);
    acc += (double)va[sr.lo + k] * (double)t;
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
  // ---- the arrays the backward / introspection read (CSR: csr_jf, P0, cs, prow; CSC:
  // csc_i, P0c; pcol and csc_perm were written above)
  if (fit) {
    for (uint32_t p = threadIdx.x; p < nnzr; p += blockDim.x) {
      A.csr_jf[pb + gr + p] = R.idx[p];
      A.P0[pb + gr + p] = R.val[p];
      A.cs[pb + gr + p] = R.c[p];
    }
    for (uint32_t q = threadIdx.x; q < nnzc; q += blockDim.x) {
      A.csc_i[pb + gc + q] = C.idx[q] & kIdxMask;
      A.csc_if[pb + gc + q] = C.idx[q];
      A.P0c[pb + gc + q] = C.val[q];
      A.csc_c[pb + gc + q] = C.c[q];
    }
  } else {
    for (uint32_t p = threadIdx.x; p < nnzr; p += blockDim.x) A.cs[pb + gr + p] = R.c[p];
    for (uint32_t q = threadIdx.x; q < nnzc; q += blockDim.x) {
      A.csc_if[pb + gc + q] = C.idx[q];
      A.csc_c[pb + gc + q] = C.c[q];
      A.csc_pc[pb + gc + q] = C.pr[q];
      C.idx[q] &= kIdxMask;  // = csc_i
    }
  }
  csync(cl);
  if (rank == 0 && threadIdx.x == 0) {
    double t = 0.0;
    for (int r = 0; r < CL; ++r) t += s_part[r];
    A.loss[b] = (float)t;
  }
  phase(A, 8);
}

__global__ void __launch_bounds__(kMegaThreads, 1) k_sparse_fwd2(const SparseArgs A) { sparse_fwd2_body(A); }

}  // namespace apml
