// k_sinkhorn.cuh -- Sinkhorn forward (S6) + loss (S7) and its reverse (S8), one CTA per pair,
// SHARED-MEMORY RESIDENT: the pair's CSR / CSC structure (16-bit indices when N, M < 65536)
// and P0 in both orders are copied into shared memory once, then all 2 L half-steps run out
// of shared memory with deterministic per-line sums (no float atomics, no per-entry writes
// per half-step).  A pair whose structure does not fit the dynamic shared memory the kernel
// was launched with falls back to the same loop over global (L2-resident) arrays.
//
// Forward (Eqs. (3)-(4)), scaling-vector form P = diag(a) P0 diag(b):
//   b_j <- b_j / (b_j Q_j + eps),  Q_j = sum_i a_i P0_ij        (column scaling, Eq. (3))
//   a_i <- a_i / (a_i R_i + eps),  R_i = sum_j P0_ij b_j        (row scaling, Eq. (4))
//   loss = sum_i a_i sum_j P0_ij b_j c_ij
// Reverse (see k_backward.cuh for the derivation), with r = a^l / a^{l-1}:
//   Rbar^l = -abar (a^l)^2, abar <- abar eps r^2, bbar += P0^T Rbar^l,
//   Qbar^l = -bbar (b^l)^2, bbar <- bbar eps r'^2, abar += P0 Qbar^l.
#pragma once
#include "common.cuh"

namespace apml {

constexpr int kSkThreads = 1024;

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

// Shared-memory bytes a pair with nnz entries needs (idx_bytes = 2 or 4; extra vectors =
// number of N- and M-sized float vectors beyond the structure).
__host__ __device__ inline size_t sk_smem_bytes(size_t N, size_t M, size_t nnz, size_t idx_bytes,
                                                int vec_sets) {
  return align16(4 * (N + 1)) + align16(4 * (M + 1)) + 2 * align16(idx_bytes * nnz) +
         2 * align16(4 * nnz) + (size_t)vec_sets * (align16(4 * N) + align16(4 * M));
}

struct SkPair {
  const unsigned* rp;  // [N+1] pair-local CSR offsets
  const unsigned* cp;  // [M+1] pair-local CSC offsets
  const void* cj;      // CSR column index (IdxT; u32 global arrays carry flags above bit 30)
  const float* p0;     // P0 in CSR order
  const void* ci;      // CSC row index
  const float* p0c;    // P0 in CSC order
};

// Copy one pair's structure into shared memory; returns views into it.
template <typename IdxT>
__device__ SkPair sk_stage_smem(uint8_t* sm, int N, int M, uint32_t nnz, const unsigned* rp,
                                const unsigned* cp, const uint32_t* csr_jf, const float* P0,
                                const uint32_t* csc_i, const float* P0c, uint8_t** rest) {
  unsigned* s_rp = reinterpret_cast<unsigned*>(sm);
  sm += align16(4 * (N + 1));
  unsigned* s_cp = reinterpret_cast<unsigned*>(sm);
  sm += align16(4 * (M + 1));
  IdxT* s_cj = reinterpret_cast<IdxT*>(sm);
  sm += align16(sizeof(IdxT) * nnz);
  IdxT* s_ci = reinterpret_cast<IdxT*>(sm);
  sm += align16(sizeof(IdxT) * nnz);
  float* s_p0 = reinterpret_cast<float*>(sm);
  sm += align16(4 * nnz);
  float* s_p0c = reinterpret_cast<float*>(sm);
  sm += align16(4 * nnz);
  for (int k = threadIdx.x; k <= N; k += blockDim.x) s_rp[k] = rp[k];
  for (int k = threadIdx.x; k <= M; k += blockDim.x) s_cp[k] = cp[k];
  for (uint32_t k = threadIdx.x; k < nnz; k += blockDim.x) {
    s_cj[k] = (IdxT)(csr_jf[k] & kIdxMask);
    s_p0[k] = P0[k];
    s_ci[k] = (IdxT)csc_i[k];
    s_p0c[k] = P0c[k];
  }
  *rest = sm;
  return SkPair{s_rp, s_cp, s_cj, s_p0, s_ci, s_p0c};
}

template <typename IdxT>
__device__ __forceinline__ uint32_t sk_idx(const void* base, uint32_t k) {
  return (uint32_t)(reinterpret_cast<const IdxT*>(base)[k]) & kIdxMask;
}

template <typename IdxT>
__device__ void sk_forward_body(const SkPair v, int N, int M, int L, float eps, float* a,
                                float* bv, float* ah, float* bh) {
  for (int i = threadIdx.x; i < N; i += blockDim.x) { a[i] = 1.f; ah[(size_t)i * (L + 1)] = 1.f; }
  for (int j = threadIdx.x; j < M; j += blockDim.x) { bv[j] = 1.f; bh[(size_t)j * (L + 1)] = 1.f; }
  __syncthreads();
  for (int l = 1; l <= L; ++l) {
    for (int j = threadIdx.x; j < M; j += blockDim.x) {  // Eq. (3): colsum_j = b_j Q_j
      float Q = 0.f;
      for (uint32_t q = v.cp[j]; q < v.cp[j + 1]; ++q) Q = __fmaf_rn(a[sk_idx<IdxT>(v.ci, q)], v.p0c[q], Q);
      const float bj = bv[j];
      const float nb = __fdiv_rn(bj, __fmaf_rn(bj, Q, eps));
      bv[j] = nb;
      bh[(size_t)j * (L + 1) + l] = nb;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += blockDim.x) {  // Eq. (4): rowsum_i = a_i R_i
      float Rs = 0.f;
      for (uint32_t p = v.rp[i]; p < v.rp[i + 1]; ++p) Rs = __fmaf_rn(v.p0[p], bv[sk_idx<IdxT>(v.cj, p)], Rs);
      const float ai = a[i];
      const float na = __fdiv_rn(ai, __fmaf_rn(ai, Rs, eps));
      a[i] = na;
      ah[(size_t)i * (L + 1) + l] = na;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  }
  return t;
}

// Forward Sinkhorn + loss.  grid = B, block = kSkThreads, dynamic smem = smem_bytes.
template <typename IdxT>
__global__ void __launch_bounds__(kSkThreads)
k_sinkhorn(int N, int M, int L, float eps, const unsigned* __restrict__ cursor, uint32_t cap,
           const unsigned* __restrict__ row_ptr, const uint32_t* __restrict__ csr_jf,
           const unsigned* __restrict__ col_ptr, const uint32_t* __restrict__ csc_i,
           const float* __restrict__ P0, const float* __restrict__ P0c,
           const float* __restrict__ cs, float* __restrict__ a_hist, float* __restrict__ b_hist,
           float* __restrict__ gscratch, size_t smem_bytes, float* __restrict__ loss) {
  extern __shared__ __align__(16) uint8_t shm[];
  __shared__ double red[32];
  const int b = blockIdx.x;
  if (pair_overflow(cursor, b, cap)) {
    if (threadIdx.x == 0) loss[b] = __int_as_float(0x7fc00000);
    return;
  }
  const size_t pb = (size_t)b * cap;
  const unsigned* rp = row_ptr + (size_t)b * (N + 1);
  const unsigned* cp = col_ptr + (size_t)b * (M + 1);
  const uint32_t nnz = rp[N];
  float* ah = a_hist + (size_t)b * N * (L + 1);
  float* bh = b_hist + (size_t)b * M * (L + 1);
  const bool fits = sk_smem_bytes(N, M, nnz, sizeof(IdxT), 1) <= smem_bytes;
  SkPair v;
  float *a, *bv;
  if (fits) {
    uint8_t* rest;
    v = sk_stage_smem<IdxT>(shm, N, M, nnz, rp, cp, csr_jf + pb, P0 + pb, csc_i + pb, P0c + pb, &rest);
    a = reinterpret_cast<float*>(rest);
    bv = a + align16(4 * N) / 4;
    __syncthreads();
    sk_forward_body<IdxT>(v, N, M, L, eps, a, bv, ah, bh);
  } else {
    v = SkPair{rp, cp, csr_jf + pb, P0 + pb, csc_i + pb, P0c + pb};
    a = gscratch + (size_t)b * (N + M);
    bv = a + N;
    sk_forward_body<uint32_t>(v, N, M, L, eps, a, bv, ah, bh);
  }
  // loss_b = sum_i a_i sum_j P0_ij b_j c_ij  (c in CSR order, global)
  double acc = 0.0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    float t = 0.f;
    for (uint32_t p = v.rp[i]; p < v.rp[i + 1]; ++p) {
      const uint32_t j = fits ? sk_idx<IdxT>(v.cj, p) : sk_idx<uint32_t>(v.cj, p);
      t = __fmaf_rn(__fmul_rn(v.p0[p], bv[j]), cs[pb + p], t);
    }
    acc += (double)a[i] * (double)t;
  }
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) loss[b] = (float)tot;
}

template <typename IdxT>
__device__ void sk_backward_body(const SkPair v, int N, int M, int L, float eps, const float* ah,
                                 const float* bh, float* ab, float* bb, float* rcur, float* qcur,
                                 float* rb, float* qb) {
  for (int l = L; l >= 1; --l) {
    // row step reverse (a^l = a^{l-1} / (a^{l-1} R^l + eps)) ... (the P0 Qbar^{l+1} sum of the
    // previous iteration has already been folded into abar)
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const float al = ah[(size_t)i * (L + 1) + l], alm = ah[(size_t)i * (L + 1) + l - 1];
      const float r = al / alm;
      const float R = -ab[i] * al * al;
      rcur[i] = R;
      rb[(size_t)i * L + (l - 1)] = R;
      ab[i] = ab[i] * eps * r * r;
    }
    __syncthreads();
    // bbar += P0^T Rbar^l, then the column step reverse (b^l = b^{l-1} / (b^{l-1} Q^l + eps))
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
      double t = 0.0;
      for (uint32_t q = v.cp[j]; q < v.cp[j + 1]; ++q) t += (double)rcur[sk_idx<IdxT>(v.ci, q)] * (double)v.p0c[q];
      const float bsum = (float)((double)bb[j] + t);
      const float bl = bh[(size_t)j * (L + 1) + l], blm = bh[(size_t)j * (L + 1) + l - 1];
      const float r = bl / blm;
      const float Q = -bsum * bl * bl;
      qcur[j] = Q;
      qb[(size_t)j * L + (l - 1)] = Q;
      bb[j] = bsum * eps * r * r;
    }
    __syncthreads();
    // abar += P0 Qbar^l
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      double t = 0.0;
      for (uint32_t p = v.rp[i]; p < v.rp[i + 1]; ++p) t += (double)qcur[sk_idx<IdxT>(v.cj, p)] * (double)v.p0[p];
      ab[i] = (float)((double)ab[i] + t);
    }
    __syncthreads();
  }
}

// Reverse Sinkhorn (full mode).  Writes Rbar [B][N][L], Qbar [B][M][L].
template <typename IdxT>
__global__ void __launch_bounds__(kSkThreads)
k_sinkhorn_bwd(int N, int M, int L, float eps, const unsigned* __restrict__ cursor, uint32_t cap,
               const unsigned* __restrict__ row_ptr, const uint32_t* __restrict__ csr_jf,
               const unsigned* __restrict__ col_ptr, const uint32_t* __restrict__ csc_i,
               const uint32_t* __restrict__ csc_perm, const float* __restrict__ P0,
               const float* __restrict__ P0c, const float* __restrict__ cs,
               const float* __restrict__ a_hist, const float* __restrict__ b_hist,
               const float* __restrict__ grad_loss, float* __restrict__ Rbar,
               float* __restrict__ Qbar, float* __restrict__ gscratch, size_t smem_bytes) {
  extern __shared__ __align__(16) uint8_t shm[];
  const int b = blockIdx.x;
  if (pair_overflow(cursor, b, cap)) return;
  const size_t pb = (size_t)b * cap;
  const float gl = grad_loss[b];
  const unsigned* rp = row_ptr + (size_t)b * (N + 1);
  const unsigned* cp = col_ptr + (size_t)b * (M + 1);
  const uint32_t nnz = rp[N];
  const float* ah = a_hist + (size_t)b * N * (L + 1);
  const float* bh = b_hist + (size_t)b * M * (L + 1);
  float* rb = Rbar + (size_t)b * N * L;
  float* qb = Qbar + (size_t)b * M * L;
  const bool fits = sk_smem_bytes(N, M, nnz, sizeof(IdxT), 2) <= smem_bytes;
  SkPair v;
  float *ab, *bb, *rcur, *qcur;
  if (fits) {
    uint8_t* rest;
    v = sk_stage_smem<IdxT>(shm, N, M, nnz, rp, cp, csr_jf + pb, P0 + pb, csc_i + pb, P0c + pb, &rest);
    ab = reinterpret_cast<float*>(rest);
    bb = ab + align16(4 * N) / 4;
    rcur = bb + align16(4 * M) / 4;
    qcur = rcur + align16(4 * N) / 4;
  } else {
    v = SkPair{rp, cp, csr_jf + pb, P0 + pb, csc_i + pb, P0c + pb};
    ab = gscratch + (size_t)b * 2 * (N + M);
    bb = ab + N;
    rcur = bb + M;
    qcur = rcur + N;
  }
  // abar = gl sum_j P0 b^L c,  bbar = gl sum_i a^L P0 c   (loss = sum a P0 b c)
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    double t = 0.0;
    for (uint32_t p = rp[i]; p < rp[i + 1]; ++p)
      t += (double)P0[pb + p] * (double)bh[(size_t)(csr_jf[pb + p] & kIdxMask) * (L + 1) + L] * (double)cs[pb + p];
    ab[i] = (float)((double)gl * t);
  }
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    double t = 0.0;
    for (uint32_t q = cp[j]; q < cp[j + 1]; ++q)
      t += (double)ah[(size_t)csc_i[pb + q] * (L + 1) + L] * (double)P0c[pb + q] * (double)cs[pb + csc_perm[pb + q]];
    bb[j] = (float)((double)gl * t);
  }
  __syncthreads();
  if (fits) sk_backward_body<IdxT>(v, N, M, L, eps, ah, bh, ab, bb, rcur, qcur, rb, qb);
  else sk_backward_body<uint32_t>(v, N, M, L, eps, ah, bh, ab, bb, rcur, qcur, rb, qb);
}

}  // namespace apml
