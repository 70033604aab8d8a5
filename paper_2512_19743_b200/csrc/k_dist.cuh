// k_dist.cuh -- the O(B N M) distance sweeps of the hot path.
//
//   k_stage      S0: AoS [B][n][3] -> padded SoA [B][3][np] (sentinel-padded, so the sweeps
//                    need no bounds checks) + float4 copy [B][n] for the sparse gathers.
//   k_line_top2  S1 (Pass A): for every owned point, the min and second min (multiset) of
//                    d2 against all streamed points -- "tracks the minimum and second
//                    minimum" (Alg. 1).  Launched twice (rows: own = pred,
//                    stream = gt; columns: roles swapped).  Column range split across
//                    blockIdx.y; partial (min, second) per split are merged in k_line_info.
//   k_line_info  S2: merge partials, m = sqrt(m2), c2 = sqrt(s2), g = max(c2 - m + delta,
//                    eps_g), T = Lambda_K / g (Eq. (1)), kept radius
//                    R = m + rho_K g with rho_K = ln(1/tau)/Lambda_K, so s >= tau <=> c <= R
//                     -- no exp / sqrt per pair in the sweeps.
//   k_emit       S3 (Pass B): recompute d2, keep (i, j) iff d2 <= R_i^2 (row) or d2 <= R'_j^2
//                    (column), append (i, j | flags) to the pair's segment (P:90 union
//                    support, "rescans ... writes the kept COO triples").
//
// Thread mapping of the sweeps: a CTA of 128 threads owns 128*R points (R per thread, kept
// in registers as negated packed pairs) and streams the other cloud through shared memory
// in tiles of kTQ points; per 4 streamed points a thread issues 3 broadcast LDS.128 and, per
// owned point, 2 x 6 packed FADD2/FMUL2/FFMA2 + 2 x 5 FMNMX(3) -- FP32 / ALU issue bound
// (DESIGN.md "Roofline").
#pragma once
#include "common.cuh"

namespace apml {

constexpr int kSweepThreads = 128;
constexpr int kTQ = 128;  // streamed points per shared-memory tile

// nb (ragged batches, else NULL): pair b has nb[b] <= n real points; the rest of its n slots
// are staged as sentinels (never a minimum, never emitted).
__device__ __forceinline__ void stage_point(const float* __restrict__ pts, int n, int np, float sentinel,
                                            float* __restrict__ soa, float4* __restrict__ p4,
                                            const int* __restrict__ nb, int b, int k) {
  if (k >= np) return;
  float x = sentinel, y = sentinel, z = sentinel;
  if (k < n) {
    if (!nb || k < nb[b]) {
      const float* p = pts + ((size_t)b * n + k) * 3;
      x = p[0]; y = p[1]; z = p[2];
    }
    p4[(size_t)b * n + k] = make_float4(x, y, z, 0.f);
  }
  float* s = soa + (size_t)b * 3 * np;
  s[k] = x; s[np + k] = y; s[2 * np + k] = z;
}
// pred and gt of every pair in ONE launch (grid.z = 2 B: pred, then gt)
__global__ void k_stage_both(const float* __restrict__ pred, int N, int Np, float* __restrict__ predS,
                             float4* __restrict__ pred4, const int* __restrict__ nb, const float* __restrict__ gt,
                             int M, int Mp, float* __restrict__ gtS, float4* __restrict__ gt4,
                             const int* __restrict__ mb, int B) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  pdl_trigger();
  if ((int)blockIdx.z < B) stage_point(pred, N, Np, kPadPred, predS, pred4, nb, blockIdx.z, k);
  else stage_point(gt, M, Mp, kPadGt, gtS, gt4, mb, blockIdx.z - B, k);
}

__global__ void k_stage(const float* __restrict__ pts, int n, int np, float sentinel,
                        float* __restrict__ soa, float4* __restrict__ p4, const int* __restrict__ nb) {
  const int b = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  float x = sentinel, y = sentinel, z = sentinel;
  if (k < n) {
    if (!nb || k < nb[b]) {
      const float* p = pts + ((size_t)b * n + k) * 3;
      x = p[0]; y = p[1]; z = p[2];
    }
    p4[(size_t)b * n + k] = make_float4(x, y, z, 0.f);
  }
  if (!soa) return;  // culled mode: the SoA copy is written in Morton order by k_cell_scatter
  float* s = soa + (size_t)b * 3 * np;
  s[k] = x; s[np + k] = y; s[2 * np + k] = z;
}

// ---- TMA (bulk-copy engine) staging of the streamed tiles: one elected thread issues three
// 1-D cp.async.bulk copies (x, y, z: 3 x kTQ floats, contiguous in the SoA staging, 512-byte
// aligned) per tile into a 2-deep shared-memory ring, each completing on the ring slot's
// mbarrier (expect-tx); the tile after next is issued as soon as every warp has left a slot,
// so the copy of tile t+1 overlaps the distance work of tile t (north_star (1): "stages gt /
// pred tiles in shared memory via TMA bulk copies").
struct TileRing {
  float v[2][3][kTQ];
  unsigned long long bar[2];
};
__device__ __forceinline__ uint32_t sptr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ring_init(TileRing& r) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 2; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sptr(&r.bar[k])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}
// (one thread) tile at streamed index j0 into slot k
__device__ __forceinline__ void ring_issue(TileRing& r, int k, const float* __restrict__ str, int str_np, int j0) {
  const uint32_t bar = sptr(&r.bar[k]);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(3u * kTQ * 4u) : "memory");
#pragma unroll
  for (int c = 0; c < 3; ++c)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sptr(&r.v[k][c][0])),
                 "l"(str + (size_t)c * str_np + j0), "r"(kTQ * 4u), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void ring_wait(TileRing& r, int k, uint32_t parity) {
  const uint32_t bar = sptr(&r.bar[k]);
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(bar), "r"(parity)
                 : "memory");
}

// The emit's ring: the streamed coordinates AND the streamed columns' radii (R'^2, E'^2: SoA
// copies written by line_info) per tile, five bulk copies completing on one mbarrier.
struct TileRing5 {
  float v[2][5][kTQ];
  unsigned long long bar[2];
};
__device__ __forceinline__ void ring5_init(TileRing5& r) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 2; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sptr(&r.bar[k])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}
__device__ __forceinline__ void ring5_issue(TileRing5& r, int k, const float* __restrict__ str, int str_np,
                                            const float* __restrict__ R2s, const float* __restrict__ E2s, int j0) {
  const uint32_t bar = sptr(&r.bar[k]);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(5u * kTQ * 4u) : "memory");
  const float* src[5] = {str + j0, str + (size_t)str_np + j0, str + 2 * (size_t)str_np + j0, R2s + j0, E2s + j0};
#pragma unroll
  for (int c = 0; c < 5; ++c)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sptr(&r.v[k][c][0])),
                 "l"(src[c]), "r"(kTQ * 4u), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void ring5_wait(TileRing5& r, int k, uint32_t parity) {
  const uint32_t bar = sptr(&r.bar[k]);
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(bar), "r"(parity)
                 : "memory");
}

// Load one kTQ-point tile of the streamed cloud (SoA) into shared memory.
__device__ __forceinline__ void load_tile(const float* __restrict__ str, int str_np, int j0,
                                          float* sx, float* sy, float* sz) {
  for (int t = threadIdx.x; t < kTQ; t += kSweepThreads) {
    sx[t] = __ldg(str + j0 + t);
    sy[t] = __ldg(str + str_np + j0 + t);
    sz[t] = __ldg(str + 2 * str_np + j0 + t);
  }
}

// One direction of Pass A (own points in registers, the other cloud streamed): block bx of
// the own points, column split `split`, pair b.
template <int R>
__device__ __forceinline__ void top2_block(const float* __restrict__ own_soa, int own_np,
                                           const float* __restrict__ str_soa, int str_np, int chunk, int B,
                                           float2* __restrict__ part, const int* __restrict__ nown,
                                           const int* __restrict__ nstr, int bx, int split, int b) {
  // ragged batches: blocks of padding rows have no line to serve (k_line_info ignores their
  // partials); streamed tiles past the pair's real points hold only sentinels
  if (nown && (int)(bx * kSweepThreads * R) >= nown[b]) return;
  const int str_end = nstr ? min(str_np, (nstr[b] + kTQ - 1) / kTQ * kTQ) : str_np;
  const float* own = own_soa + (size_t)b * 3 * own_np;
  const float* str = str_soa + (size_t)b * 3 * str_np;
  const int base = bx * kSweepThreads * R + threadIdx.x;
  __shared__ __align__(128) TileRing ring;
  const int j0 = split * chunk, j1 = min(str_end, j0 + chunk);
  ring_init(ring);
  pdl_trigger();
  pdl_wait();  // the staged SoA clouds (k_stage_both)
  if (threadIdx.x == 0) {
    if (j0 < j1) ring_issue(ring, 0, str, str_np, j0);
    if (j0 + kTQ < j1) ring_issue(ring, 1, str, str_np, j0 + kTQ);
  }

  f2_t nx[R], ny[R], nz[R];
  // two independent running (min, second) per owned point (streamed points 0,1 / 2,3 of each
  // group of 4), merged exactly at the end: twice the independent dependency chains
  float m[R], s[R], m2[R], s2[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int idx = base + r * kSweepThreads;
    const float x = -__ldg(own + idx), y = -__ldg(own + own_np + idx), z = -__ldg(own + 2 * own_np + idx);
    nx[r] = f2_pack(x, x); ny[r] = f2_pack(y, y); nz[r] = f2_pack(z, z);
    m[r] = __int_as_float(0x7f800000); s[r] = m[r];
    m2[r] = m[r]; s2[r] = m[r];
  }
  int t = 0;
  for (int jt = j0; jt < j1; jt += kTQ, ++t) {
    const int k = t & 1;
    ring_wait(ring, k, (uint32_t)(t >> 1) & 1u);
    const ulonglong2* px = reinterpret_cast<const ulonglong2*>(ring.v[k][0]);
    const ulonglong2* py = reinterpret_cast<const ulonglong2*>(ring.v[k][1]);
    const ulonglong2* pz = reinterpret_cast<const ulonglong2*>(ring.v[k][2]);
#pragma unroll 4
    for (int q = 0; q < kTQ / 4; ++q) {
      const ulonglong2 qx = px[q], qy = py[q], qz = pz[q];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const f2_t d01 = f2_dist2(qx.x, qy.x, qz.x, nx[r], ny[r], nz[r]);
        const f2_t d23 = f2_dist2(qx.y, qy.y, qz.y, nx[r], ny[r], nz[r]);
        float d0, d1, d2, d3;
        f2_unpack(d01, d0, d1);
        f2_unpack(d23, d2, d3);
        top2_pair(m[r], s[r], d0, d1);
        top2_pair(m2[r], s2[r], d2, d3);
      }
    }
    if (jt + 2 * kTQ < j1) {  // slot k is refilled with the tile after next once every warp left it
      __syncthreads();
      if (threadIdx.x == 0) ring_issue(ring, k, str, str_np, jt + 2 * kTQ);
    }
  }
  float2* out = part + ((size_t)split * B + b) * own_np;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    top2_merge(m[r], s[r], m2[r], s2[r]);
    out[base + r * kSweepThreads] = make_float2(m[r], s[r]);
  }
}

template <int R>
__global__ void __launch_bounds__(kSweepThreads)
k_line_top2(const float* __restrict__ own_soa, int own_np, const float* __restrict__ str_soa,
            int str_np, int chunk, int B, float2* __restrict__ part, const int* __restrict__ nown,
            const int* __restrict__ nstr) {
  top2_block<R>(own_soa, own_np, str_soa, str_np, chunk, B, part, nown, nstr, blockIdx.x, blockIdx.y, blockIdx.z);
}

// Both directions of Pass A in ONE launch (grid.z = 2 B: rows, then columns): the two sweeps
// share the waves, so neither pays a partly empty last wave (and one launch gap less).
struct Top2Dir {
  const float* own;
  int own_np;
  const float* str;
  int str_np, chunk, S, nblk;
  float2* part;
  const int* nown;
  const int* nstr;
};
template <int R>
__global__ void __launch_bounds__(kSweepThreads) k_line_top2_both(const Top2Dir d0, const Top2Dir d1, int B) {
  const int dir = blockIdx.z >= (unsigned)B;
  const Top2Dir& d = dir ? d1 : d0;
  if ((int)blockIdx.x >= d.nblk || (int)blockIdx.y >= d.S) return;
  top2_block<R>(d.own, d.own_np, d.str, d.str_np, d.chunk, B, d.part, d.nown, d.nstr, blockIdx.x, blockIdx.y,
                blockIdx.z - dir * B);
}

// S2: one thread per line.  lam = Lambda_K (fp64 on the host, rounded), rho = ln(1/tau) /
// Lambda_K (+inf for tau = 0).  K == 1 lines keep their single entry with P = 1.
// ufb (APML_FLAG_UNIFORM_FALLBACK, the stability mode of P:64 / P:97 instead of the clamp of
// P:140): a line whose gap c~(2) = c2 - m is below eps_g keeps ALL K entries with P = 1/K --
// T = 0 makes every similarity exp(-0 (c - m)) = 1, the infinite radii emit the whole line,
// and with T = 0 the softmax reverse passes no gradient (P constant), as the oracle does.
// Ragged batches (nown != NULL): pair b has nown[b] real lines of length K = kpair[b], with
// lam / rho = lr[4 b + lr_off], lr[4 b + lr_off + 1]; the padding lines are inactive (radii
// -1: nothing emitted; no entries downstream).
__device__ __forceinline__ void line_info(const float2* __restrict__ part, int S, int B, int own_np, int n,
                                          int K, float lam, float rho, float delta, float eps_g,
                                          LineA* __restrict__ A, LineB* __restrict__ Bo,
                                          unsigned long long* __restrict__ clamp_count, const int* __restrict__ nown,
                                          const int* __restrict__ kpair, const float* __restrict__ lr, int lr_off,
                                          int b, int k, int ufb, float* __restrict__ R2s = nullptr,
                                          float* __restrict__ E2s = nullptr, int re_np = 0) {
  // R2s / E2s (or NULL): SoA copies of the radii at [b][re_np] for the emit's tile copies
  if (k >= n) return;
  if (nown) {
    if (k >= nown[b]) {
      const float inf = __int_as_float(0x7f800000);
      A[(size_t)b * n + k] = LineA{inf, inf, -1.f, -1.f};
      Bo[(size_t)b * n + k] = LineB{0.f, 0.f, 0.f, 0};
      if (R2s) { R2s[(size_t)b * re_np + k] = -1.f; E2s[(size_t)b * re_np + k] = -1.f; }
      return;
    }
    K = kpair[b];
    lam = lr[4 * b + lr_off];
    rho = lr[4 * b + lr_off + 1];
  }
  float m2 = __int_as_float(0x7f800000), s2 = m2;
  for (int sp0 = 0; sp0 < S; sp0 += 8) {  // 8 partials in flight per step
    float2 p[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      p[u] = sp0 + u < S ? part[((size_t)(sp0 + u) * B + b) * own_np + k]
                         : make_float2(__int_as_float(0x7f800000), __int_as_float(0x7f800000));
#pragma unroll
    for (int u = 0; u < 8; ++u) top2_merge(m2, s2, p[u].x, p[u].y);
  }
  LineA a;
  LineB o;
  const float inf = __int_as_float(0x7f800000);
  if (K == 1) {
    a = {m2, inf, inf, inf};
    o = {__fsqrt_rn(m2), 0.f, 0.f, kLineK1};
  } else {
    const float m = __fsqrt_rn(m2), c2 = __fsqrt_rn(s2);
    const float gap = __fsub_rn(c2, m);                  // c~(2)
    if (ufb && gap < eps_g) {                            // uniform fallback
      a = {m2, s2, inf, inf};
      o = {m, 0.f, fmaxf(__fadd_rn(gap, delta), eps_g), kLineUniform};
      atomicAdd(clamp_count + 4, 1ull);
    } else {
      float g = __fadd_rn(gap, delta);                   // g = c~(2) + delta
      int flags = 0;
      if (g < eps_g) { g = eps_g; flags |= kLineClamped; } // max(gap, eps_g)
      const float T = __fdiv_rn(lam, g);                 // Eq. (1)
      const float R = __fadd_rn(m, __fmul_rn(rho, g));   // s >= tau <=> c <= R
      float R2 = fmaxf(__fmul_rn(R, R), m2);             // the argmin (s = 1) is always kept
      a = {m2, s2, R2, fmaxf(R2, s2)};
      o = {m, T, g, flags};
      if (flags & kLineClamped) atomicAdd(clamp_count, 1ull);
    }
  }
  A[(size_t)b * n + k] = a;
  Bo[(size_t)b * n + k] = o;
  if (R2s) { R2s[(size_t)b * re_np + k] = a.R2; E2s[(size_t)b * re_np + k] = a.E2; }
}

__global__ void k_line_info(const float2* __restrict__ part, int S, int B, int own_np, int n,
                            int K, float lam, float rho, float delta, float eps_g,
                            LineA* __restrict__ A, LineB* __restrict__ Bo,
                            unsigned long long* __restrict__ clamp_count, const int* __restrict__ nown,
                            const int* __restrict__ kpair, const float* __restrict__ lr, int lr_off, int ufb,
                            float* __restrict__ R2s = nullptr, float* __restrict__ E2s = nullptr, int re_np = 0) {
  line_info(part, S, B, own_np, n, K, lam, rho, delta, eps_g, A, Bo, clamp_count, nown, kpair, lr, lr_off,
            blockIdx.y, blockIdx.x * blockDim.x + threadIdx.x, ufb, R2s, E2s, re_np);
}

// Rows and columns in ONE launch (grid.z = 2: rows, columns; grid.y = pair).
struct LineInfoDir {
  const float2* part;
  int S, own_np, n, K;
  float lam, rho;
  LineA* A;
  LineB* Bo;
  const int* nown;
  const int* kpair;
  int lr_off;
  float* R2s = nullptr;  // SoA radii copies (columns of the full sweeps: the emit's tile copies)
  float* E2s = nullptr;
  int re_np = 0;         // their per-pair stride
};
__global__ void k_line_info_both(const LineInfoDir d0, const LineInfoDir d1, int B, float delta, float eps_g,
                                 unsigned long long* __restrict__ clamp_count, const float* __restrict__ lr, int ufb) {
  pdl_trigger();
  pdl_wait();  // Pass A's partials
  const LineInfoDir& d = blockIdx.z ? d1 : d0;
  line_info(d.part, d.S, B, d.own_np, d.n, d.K, d.lam, d.rho, delta, eps_g, d.A, d.Bo, clamp_count, d.nown,
            d.kpair, lr, d.lr_off, blockIdx.y, blockIdx.x * blockDim.x + threadIdx.x, ufb, d.R2s, d.E2s, d.re_np);
}

// Pass A with S2 fused (the full sweeps): every CTA of a (direction, pair, row block) writes
// its partial (min, second) and counts itself in; the LAST of the block's S column splits
// merges the S partials of its 512 lines into the line constants (line_info), so no separate
// launch (and no kernel boundary) is needed between Pass A and the emit.  Writers: stores,
// __threadfence, then the counter; the last CTA fences before reading the other partials.
struct FusedInfo {
  LineInfoDir li[2];  // rows, columns
  float delta, eps_g;
  unsigned long long* clamp;
  const float* lr;
  int ufb;
  unsigned* cnt;      // [2][B][nblk] arrivals, zeroed before every forward
  int nblk;           // row-block stride of cnt (the larger direction's)
};
template <int R>
__global__ void __launch_bounds__(kSweepThreads) k_line_top2_info(const Top2Dir d0, const Top2Dir d1, int B,
                                                                   const FusedInfo fi) {
  const int dir = blockIdx.z >= (unsigned)B;
  const Top2Dir& d = dir ? d1 : d0;
  if ((int)blockIdx.x >= d.nblk || (int)blockIdx.y >= d.S) return;
  const int b = blockIdx.z - dir * B;
  top2_block<R>(d.own, d.own_np, d.str, d.str_np, d.chunk, B, d.part, d.nown, d.nstr, blockIdx.x, blockIdx.y, b);
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0)
    s_last = atomicAdd(fi.cnt + ((size_t)dir * B + b) * fi.nblk + blockIdx.x, 1u) == (unsigned)d.S - 1u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const LineInfoDir& L = fi.li[dir];
  for (int k = threadIdx.x; k < kSweepThreads * R; k += blockDim.x)
    line_info(L.part, L.S, B, L.own_np, L.n, L.K, L.lam, L.rho, fi.delta, fi.eps_g, L.A, L.Bo, fi.clamp, L.nown,
              L.kpair, fi.lr, L.lr_off, b, (int)blockIdx.x * kSweepThreads * R + k, fi.ufb, L.R2s, L.E2s, L.re_np);
}

// Emission (S3).  Counts keep running past the capacity so the host can size a retry;
// overflowed pairs are skipped downstream; the per-line counts are non-returning reductions.
// Per-lane emission queues (k_emit, k_emit_cull): every lane appends its own hits to its own slots of a
// shared-memory queue with no cross-lane communication (the common case -- a warp with a hit
// somewhere in a 4-column step -- used to cost 4 ballots + popcounts + a serialised compaction
// per step); the warp flushes all queues with one shuffle scan and one returning atomic when a
// queue is nearly full and at the end.
constexpr int kLaneQ = 16;  // queue slots per lane
constexpr unsigned kCursorSat = 0x80000000u, kCursorPark = 0xC0000000u;

__device__ __forceinline__ void lane_flush(int b, const uint2* q, int cnt, uint32_t cap, uint2* __restrict__ ebuf,
                                           unsigned* __restrict__ cursor, unsigned* __restrict__ aux_cnt,
                                           unsigned* __restrict__ row_cnt, int N, unsigned* __restrict__ col_cnt,
                                           int M) {
  const int lane = threadIdx.x & 31;
  unsigned inc = (unsigned)cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  const unsigned total = __shfl_sync(0xffffffffu, inc, 31);
  if (total == 0) return;
  unsigned base = 0;
  if (lane == 31) {
    base = atomicAdd(cursor + b, total);
    // saturate: a count past 2^31 is parked at 3 * 2^30, so that no amount of emission
    // (tau = 0 on N M >= 2^32 pairs) wraps the 32-bit cursor back under the capacity; the
    // concurrent flushes between the add and the exchange total far less than 2^30
    if (base >= kCursorSat) atomicExch(cursor + b, kCursorPark);
  }
  base = __shfl_sync(0xffffffffu, base, 31) + inc - (unsigned)cnt;
  unsigned aux = 0;
  for (int k = 0; k < cnt; ++k) {
    const uint2 e = q[k * 32];
    const unsigned pos = base + k;
    if (pos < cap) ebuf[(size_t)b * cap + pos] = e;
    atomicAdd(row_cnt + (size_t)b * (N + 1) + e.x, 1u);
    atomicAdd(col_cnt + (size_t)b * (M + 1) + (e.y & kIdxMask), 1u);
    aux += (e.y & (kFlagRow | kFlagCol)) ? 0u : 1u;
  }
  aux = __reduce_add_sync(0xffffffffu, aux);
  if (lane == 0 && aux) atomicAdd(aux_cnt + b, aux);
}

// S3 (Pass B).  Rows own pred points; gt streamed with its column radii in shared memory.
template <int R>
__global__ void __launch_bounds__(kSweepThreads)
k_emit(const float* __restrict__ pred_soa, int np, int N, const LineA* __restrict__ rowA,
       const float* __restrict__ gt_soa, int mp, int M, const LineA* __restrict__ colA,
       int chunk, uint32_t cap, uint2* __restrict__ ebuf, unsigned* __restrict__ cursor,
       unsigned* __restrict__ aux_cnt, unsigned* __restrict__ row_cnt,
       unsigned* __restrict__ col_cnt, const int* __restrict__ nb, const int* __restrict__ mb,
       const float* __restrict__ colR2s, const float* __restrict__ colE2s) {
  const int b = blockIdx.z, split = blockIdx.y;
  const uint32_t nreal = nb ? (uint32_t)nb[b] : (uint32_t)N, mreal = mb ? (uint32_t)mb[b] : (uint32_t)M;
  if ((uint32_t)(blockIdx.x * kSweepThreads * R) >= nreal) return;  // a block of padding rows
  pdl_trigger();
  pdl_wait();  // the line constants (k_line_info_both)
  const int str_end = min(mp, (int)((mreal + kTQ - 1) / kTQ * kTQ));
  const float* own = pred_soa + (size_t)b * 3 * np;
  const float* str = gt_soa + (size_t)b * 3 * mp;
  const int base = blockIdx.x * kSweepThreads * R + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ __align__(128) TileRing5 ring;  // streamed coordinates + column radii (TMA bulk copies)
  __shared__ uint2 queue_all[kSweepThreads / 32][kLaneQ][32];  // [warp][slot][lane]: conflict-free
  uint2* q = &queue_all[w][0][lane];
  int qn = 0;  // this lane's queued entries
  const float* cR2 = colR2s + (size_t)b * mp;
  const float* cE2 = colE2s + (size_t)b * mp;

  f2_t nx[R], ny[R], nz[R];
  float rR2[R], rE2[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int idx = base + r * kSweepThreads;
    const float x = -__ldg(own + idx), y = -__ldg(own + np + idx), z = -__ldg(own + 2 * np + idx);
    nx[r] = f2_pack(x, x); ny[r] = f2_pack(y, y); nz[r] = f2_pack(z, z);
    if (idx < N) {
      const LineA a = rowA[(size_t)b * N + idx];
      rR2[r] = a.R2; rE2[r] = a.E2;
    } else {
      rR2[r] = -1.f; rE2[r] = -1.f;
    }
  }
  const int j0 = split * chunk, j1 = min(str_end, j0 + chunk);
  ring5_init(ring);
  if (threadIdx.x == 0) {
    if (j0 < j1) ring5_issue(ring, 0, str, mp, cR2, cE2, j0);
    if (j0 + kTQ < j1) ring5_issue(ring, 1, str, mp, cR2, cE2, j0 + kTQ);
  }
  int tix = 0;
  for (int jt = j0; jt < j1; jt += kTQ, ++tix) {
    const int slot = tix & 1;
    ring5_wait(ring, slot, (uint32_t)(tix >> 1) & 1u);
    const float* sx = ring.v[slot][0];
    const float* sy = ring.v[slot][1];
    const float* sz = ring.v[slot][2];
    const float* sR = ring.v[slot][3];
    const float* sE = ring.v[slot][4];
    const ulonglong2* px = reinterpret_cast<const ulonglong2*>(sx);
    const ulonglong2* py = reinterpret_cast<const ulonglong2*>(sy);
    const ulonglong2* pz = reinterpret_cast<const ulonglong2*>(sz);
    const float4* pE = reinterpret_cast<const float4*>(sE);
    const float4* pR = reinterpret_cast<const float4*>(sR);
    // Blocks of 32 columns: the hit test only sets bits of a per-(lane, owned point) mask
    // (no branch, no vote per 4 columns); after the block, the lanes with hits recompute
    // those few d2 (same operation sequence, same bits) and queue them, warp-synchronously so
    // that a nearly full queue can be flushed collectively.
    for (int blk = 0; blk < kTQ / 32; ++blk) {
      uint32_t mask[R];
#pragma unroll
      for (int r = 0; r < R; ++r) mask[r] = 0u;
#pragma unroll 2
      for (int qq = 8 * blk; qq < 8 * blk + 8; ++qq) {
        const ulonglong2 qx = px[qq], qy = py[qq], qz = pz[qq];
        const float4 ce = pE[qq];
        const int sh = 4 * (qq - 8 * blk);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const f2_t d01 = f2_dist2(qx.x, qy.x, qz.x, nx[r], ny[r], nz[r]);
          const f2_t d23 = f2_dist2(qx.y, qy.y, qz.y, nx[r], ny[r], nz[r]);
          float d[4];
          f2_unpack(d01, d[0], d[1]);
          f2_unpack(d23, d[2], d[3]);
          const uint32_t h = (d[0] <= fmaxf(rE2[r], ce.x) ? 1u : 0u) | (d[1] <= fmaxf(rE2[r], ce.y) ? 2u : 0u) |
                             (d[2] <= fmaxf(rE2[r], ce.z) ? 4u : 0u) | (d[3] <= fmaxf(rE2[r], ce.w) ? 8u : 0u);
          mask[r] |= h << sh;
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t i = base + r * kSweepThreads;
        uint32_t m = i < nreal ? mask[r] : 0u;
        float xr, yr, zr;  // -x of the owned point (exactly the packed operand)
        {
          float t;
          f2_unpack(nx[r], xr, t);
          f2_unpack(ny[r], yr, t);
          f2_unpack(nz[r], zr, t);
        }
        while (__any_sync(0xffffffffu, m)) {
          if (__any_sync(0xffffffffu, qn == kLaneQ)) {
            __syncwarp();
            lane_flush(b, q, qn, cap, ebuf, cursor, aux_cnt, row_cnt, N, col_cnt, M);
            qn = 0;
            __syncwarp();
          }
          if (m) {
            const int c = 32 * blk + __ffs(m) - 1;
            m &= m - 1;
            const uint32_t j = jt + c;
            if (j < mreal) {
              const float dx = __fadd_rn(sx[c], xr), dy = __fadd_rn(sy[c], yr), dz = __fadd_rn(sz[c], zr);
              float d2 = __fmul_rn(dx, dx);
              d2 = __fmaf_rn(dy, dy, d2);
              d2 = __fmaf_rn(dz, dz, d2);
              const uint32_t fl = (d2 <= rR2[r] ? kFlagRow : 0u) | (d2 <= sR[c] ? kFlagCol : 0u);
              q[qn * 32] = make_uint2(i, j | fl);
              ++qn;
            }
          }
        }
      }
    }
    if (jt + 2 * kTQ < j1) {  // slot refilled with the tile after next once every warp left it
      __syncthreads();
      if (threadIdx.x == 0) ring5_issue(ring, slot, str, mp, cR2, cE2, jt + 2 * kTQ);
    }
  }
  __syncwarp();
  lane_flush(b, q, qn, cap, ebuf, cursor, aux_cnt, row_cnt, N, col_cnt, M);
}

}  // namespace apml
