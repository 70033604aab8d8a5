// k_cull.cuh -- exact spatially-culled distance sweeps (the paper's future work,
// P:295 "restrict the candidate support, for example via neighborhood pruning").
//
// The result is IDENTICAL to the brute-force sweeps: min / second min of every line (Pass A)
// and the emitted union support (Pass B) are unchanged, only provably irrelevant (row block,
// column tile) pairs are skipped:
//   * both clouds of a pair are ordered by a Morton cell key of their joint bounding box
//     (counting sort; the order inside a cell is arbitrary -- it cannot change a min, a
//     threshold test or the emitted set, and all outputs are written at ORIGINAL indices);
//   * Pass A: a 128-point streamed tile whose bounding box is farther (squared) than the
//     largest current second minimum of the CTA's 512 owned points cannot change any of their
//     (min, second) -> skipped.  Tiles are visited in a ring around the CTA's own position in
//     Morton order so the bounds tighten after the first few tiles;
//   * Pass B: a tile farther than max(largest row emit radius of the block, largest column
//     emit radius of the tile) cannot contain an emitted entry -> skipped.
// Bounds carry a 1e-5 relative margin against fp32 rounding of the box distances.
#pragma once
#include "k_dist.cuh"

namespace apml {

constexpr float kCullMargin = 1.0f - 1e-5f;
constexpr int kSub = 32;                   // culling granularity of the streamed side
constexpr int kSubPerTile = kTQ / kSub;

// Joint bounding box of pred and gt of each pair: partial boxes over P chunks of the points
// (grid (P, B)), then bb[b] = {lo x,y,z, hi x,y,z} (min / max are exact in any order).
constexpr int kBoxThreads = 256;
__global__ void __launch_bounds__(kBoxThreads)
k_pair_bbox_part(const float* __restrict__ pred, int N, const float* __restrict__ gt, int M, float* __restrict__ part) {
  const int b = blockIdx.y, P = gridDim.x;
  float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
  for (int k = blockIdx.x * kBoxThreads + threadIdx.x; k < N + M; k += P * kBoxThreads) {
    const float* p = k < N ? pred + ((size_t)b * N + k) * 3 : gt + ((size_t)b * M + (k - N)) * 3;
#pragma unroll
    for (int d = 0; d < 3; ++d) { lo[d] = fminf(lo[d], p[d]); hi[d] = fmaxf(hi[d], p[d]); }
  }
  __shared__ float red[6][kBoxThreads / 32];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int d = 0; d < 3; ++d) { red[d][w] = lo[d]; red[3 + d][w] = hi[d]; }
  __syncthreads();
  if (threadIdx.x < 6) {
    float v = threadIdx.x < 3 ? 3e38f : -3e38f;
    for (int k = 0; k < kBoxThreads / 32; ++k)
      v = threadIdx.x < 3 ? fminf(v, red[threadIdx.x][k]) : fmaxf(v, red[threadIdx.x][k]);
    part[((size_t)b * P + blockIdx.x) * 6 + threadIdx.x] = v;
  }
}

__global__ void k_pair_bbox_fin(const float* __restrict__ part, int P, float* __restrict__ bb) {
  const int b = blockIdx.x, d = threadIdx.x;
  if (d >= 6) return;
  float v = d < 3 ? 3e38f : -3e38f;
  for (int k = 0; k < P; ++k) {
    const float u = part[((size_t)b * P + k) * 6 + d];
    v = d < 3 ? fminf(v, u) : fmaxf(v, u);
  }
  bb[b * 6 + d] = v;
}

__device__ __forceinline__ uint32_t spread_bits3(uint32_t v) {  // 10-bit v -> every third bit
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// Cell of one coordinate in a G-cell axis over [lo, hi] (and the fractional coordinate f):
// ONE definition for the sort (k_cell_count) and the cell sweeps (k_cells.cuh), so a point is
// always looked up in the cell it was sorted into.
__device__ __forceinline__ uint32_t cell_axis(float p, float lo, float hi, uint32_t G, float* frac) {
  const float ext = fmaxf(hi - lo, 1e-30f);
  const float f = (p - lo) / ext * (float)G;
  *frac = f;
  return (uint32_t)fminf(fmaxf(f, 0.f), (float)(G - 1));
}

// Morton cell key of every point (bits per axis), its rank in the cell (returning atomic: the
// scatter then needs no atomics) and the per-pair cell histogram.
__device__ void cell_count_body(const float* __restrict__ pts, int n, const float* __restrict__ bb, int bits,
                                uint32_t* __restrict__ key, uint32_t* __restrict__ hist, uint32_t* __restrict__ rank,
                                int b, int k) {
  if (k >= n) return;
  const float* p = pts + ((size_t)b * n + k) * 3;
  const float* box = bb + b * 6;
  const uint32_t cells_axis = 1u << bits;
  uint32_t c[3];
  float f;
#pragma unroll
  for (int d = 0; d < 3; ++d) c[d] = cell_axis(p[d], box[d], box[3 + d], cells_axis, &f);
  const uint32_t kk = spread_bits3(c[0]) | (spread_bits3(c[1]) << 1) | (spread_bits3(c[2]) << 2);
  key[(size_t)b * n + k] = kk;
  rank[(size_t)b * n + k] = atomicAdd(hist + (size_t)b * ((1u << (3 * bits)) + 1) + kk, 1u);
}
__global__ void k_cell_count(const float* __restrict__ pts, int n, const float* __restrict__ bb, int bits,
                             uint32_t* __restrict__ key, uint32_t* __restrict__ hist, uint32_t* __restrict__ rank) {
  cell_count_body(pts, n, bb, bits, key, hist, rank, blockIdx.y, blockIdx.x * blockDim.x + threadIdx.x);
}

// Both clouds in one launch each (grid.z = 2: pred, gt).
struct CellCloud {
  const float* pts;
  int n, np;
  float sentinel;
  uint32_t *key, *hist, *rank;
  const uint32_t* start;
  float* soa;
  int* perm;
  float4* p4;
  int* iperm;
};
__device__ void cell_count_body(const float* __restrict__ pts, int n, const float* __restrict__ bb, int bits,
                                uint32_t* __restrict__ key, uint32_t* __restrict__ hist, uint32_t* __restrict__ rank,
                                int b, int k);
__device__ void cell_scatter_body(const float* __restrict__ pts, int n, int np, float sentinel, int bits,
                                  const uint32_t* __restrict__ key, const uint32_t* __restrict__ start,
                                  const uint32_t* __restrict__ rank, float* __restrict__ soa, int* __restrict__ perm,
                                  float4* __restrict__ p4, int* __restrict__ iperm, int b, int k);

// Place every point at its sorted position: SoA coordinates (pads = sentinel) + perm.
// Relabelled mode (p4 != NULL): also the float4 copy and the inverse permutation (original
// -> sorted) at sorted positions.
__device__ void cell_scatter_body(const float* __restrict__ pts, int n, int np, float sentinel, int bits,
                                  const uint32_t* __restrict__ key, const uint32_t* __restrict__ start,
                                  const uint32_t* __restrict__ rank, float* __restrict__ soa, int* __restrict__ perm,
                                  float4* __restrict__ p4, int* __restrict__ iperm, int b, int k) {
  if (k >= np) return;
  float* s = soa ? soa + (size_t)b * 3 * np : nullptr;  // (NULL: the cell sweeps read the float4 copy)
  if (k >= n) {  // pads occupy the sorted positions [n, np)
    if (s) { s[k] = sentinel; s[np + k] = sentinel; s[2 * np + k] = sentinel; }
    perm[(size_t)b * np + k] = -1;
    return;
  }
  const size_t hb = (size_t)b * ((1u << (3 * bits)) + 1);
  const uint32_t kk = key[(size_t)b * n + k];
  const uint32_t pos = start[hb + kk] + rank[(size_t)b * n + k];
  const float* p = pts + ((size_t)b * n + k) * 3;
  if (s) { s[pos] = p[0]; s[np + pos] = p[1]; s[2 * np + pos] = p[2]; }
  perm[(size_t)b * np + pos] = k;
  if (p4) {
    p4[(size_t)b * n + pos] = make_float4(p[0], p[1], p[2], 0.f);
    if (iperm) iperm[(size_t)b * n + k] = (int)pos;
  }
}
__global__ void k_cell_scatter(const float* __restrict__ pts, int n, int np, float sentinel, int bits,
                               const uint32_t* __restrict__ key, const uint32_t* __restrict__ start,
                               const uint32_t* __restrict__ rank, float* __restrict__ soa, int* __restrict__ perm,
                               float4* __restrict__ p4, int* __restrict__ iperm) {
  cell_scatter_body(pts, n, np, sentinel, bits, key, start, rank, soa, perm, p4, iperm, blockIdx.y,
                    blockIdx.x * blockDim.x + threadIdx.x);
}
__global__ void k_cell_count_both(const CellCloud c0, const CellCloud c1, const float* __restrict__ bb, int bits) {
  const CellCloud& c = blockIdx.z ? c1 : c0;
  cell_count_body(c.pts, c.n, bb, bits, c.key, c.hist, c.rank, blockIdx.y, blockIdx.x * blockDim.x + threadIdx.x);
}
__global__ void k_cell_scatter_both(const CellCloud c0, const CellCloud c1, int bits) {
  const CellCloud& c = blockIdx.z ? c1 : c0;
  cell_scatter_body(c.pts, c.n, c.np, c.sentinel, bits, c.key, c.start, c.rank, c.soa, c.perm, c.p4, c.iperm,
                    blockIdx.y, blockIdx.x * blockDim.x + threadIdx.x);
}

// Bounding boxes of every kTQ-point tile (cb[b][t]) and of its kSub-point sub-tiles
// (fb[b][t * kSubPerTile + q]) of a sorted cloud, pads excluded (an all-pad box is empty:
// lo = +3e38, hi = -3e38, so its distance to anything is +inf).
__global__ void __launch_bounds__(kTQ)
k_tile_bbox(const float* __restrict__ soa, int np, int n, float* __restrict__ cb, float* __restrict__ fb) {
  const int b = blockIdx.y, t = blockIdx.x;
  const int k = t * kTQ + threadIdx.x;
  const float* s = soa + (size_t)b * 3 * np;
  float lo[3], hi[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const float v = k < n ? s[d * np + k] : 0.f;
    lo[d] = k < n ? v : 3e38f;
    hi[d] = k < n ? v : -3e38f;
  }
#pragma unroll
  for (int d = 0; d < 3; ++d)
    for (int o = 16; o > 0; o >>= 1) {
      lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  __shared__ float red[6][kTQ / 32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  static_assert(kSub == 32, "a sub-tile is one warp's worth of points");
  if (lane < 6) {
    const float v = lane < 3 ? lo[lane] : hi[lane - 3];
    fb[((size_t)b * (np / kSub) + t * kSubPerTile + w) * 6 + lane] = v;
    red[lane][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    float v = threadIdx.x < 3 ? 3e38f : -3e38f;
    for (int q = 0; q < kTQ / 32; ++q)
      v = threadIdx.x < 3 ? fminf(v, red[threadIdx.x][q]) : fmaxf(v, red[threadIdx.x][q]);
    cb[((size_t)b * (np / kTQ) + t) * 6 + threadIdx.x] = v;
  }
}

// Column radii in SORTED order (gre[b][k] = (R2, E2) of the gt point at sorted position k,
// (-1, -1) for pads) and the largest E2 of every tile (ce2) and sub-tile (fe2).
__global__ void __launch_bounds__(kTQ)
k_tile_re(const int* __restrict__ gperm, int mp, const LineA* __restrict__ colA, int M, int relabel,
          float2* __restrict__ gre, float* __restrict__ ce2, float* __restrict__ fe2) {
  const int b = blockIdx.y, t = blockIdx.x;
  const int k = t * kTQ + threadIdx.x;
  const int j = gperm[(size_t)b * mp + k];
  float2 re = make_float2(-1.f, -1.f);
  if (j >= 0) {
    const LineA a = colA[(size_t)b * M + (relabel ? k : j)];
    re = make_float2(a.R2, a.E2);
  }
  gre[(size_t)b * mp + k] = re;
  float e = re.y;
  for (int o = 16; o > 0; o >>= 1) e = fmaxf(e, __shfl_xor_sync(0xffffffffu, e, o));
  __shared__ float red[kTQ / 32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[w] = e;
    fe2[(size_t)b * (mp / kSub) + t * kSubPerTile + w] = e;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float v = -1.f;
    for (int q = 0; q < kTQ / 32; ++q) v = fmaxf(v, red[q]);
    ce2[(size_t)b * (mp / kTQ) + t] = v;
  }
}

// Super-tiles of 32 consecutive tiles (4096 sorted points): box = union of the tile boxes and,
// for the emit, the largest column emit radius of its tiles.  The candidate walks test a
// super-tile first and only its surviving tiles individually: the flat walk tested every
// tile of the cloud against every warp (ncu at C5: ~35 % of the culled Pass A samples in the
// tile-box tests, stalled on their global loads).  grid (ceil(nt / 32), B), 32 threads.
constexpr int kSuper = 32;
__global__ void __launch_bounds__(32) k_super_box(const float* __restrict__ cb, int nt, float* __restrict__ sb,
                                                  const float* __restrict__ ce2, float* __restrict__ sce2) {
  const int b = blockIdx.y, s = blockIdx.x, lane = threadIdx.x;
  const int nst = (nt + kSuper - 1) / kSuper;
  const int t = s * kSuper + lane;
  float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
  float e = -1.f;
  if (t < nt) {
    const float* tb = cb + ((size_t)b * nt + t) * 6;
#pragma unroll
    for (int d = 0; d < 3; ++d) { lo[d] = tb[d]; hi[d] = tb[3 + d]; }
    if (ce2) e = ce2[(size_t)b * nt + t];
  }
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
    e = fmaxf(e, __shfl_xor_sync(0xffffffffu, e, o));
  }
  if (lane < 6) sb[((size_t)b * nst + s) * 6 + lane] = lane < 3 ? lo[lane] : hi[lane - 3];
  if (sce2 && lane == 0) sce2[(size_t)b * nst + s] = e;
}

__device__ __forceinline__ float box_dist2(const float* a, const float* b) {
  float s = 0.f;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const float g = fmaxf(0.f, fmaxf(a[d] - b[3 + d], b[d] - a[3 + d]));
    s = fmaf(g, g, s);
  }
  return s;
}

// Warp-autonomous culling.  A warp owns R groups of 32 CONSECUTIVE sorted points (group r =
// positions base + 32 r + lane, a compact piece of the Morton curve) and walks the streamed
// tiles on its own, without block barriers: a candidate tile is tested against the warp's
// box (one tile per lane, 32 tiles per ballot), then each of its 4 sub-tiles against each
// group's box (one (group, sub-tile) pair per lane); only the surviving (group, sub-tile)
// pairs are evaluated, from the tile staged in the warp's own shared memory.
template <int R>
__device__ __forceinline__ int cull_idx(int blk, int r) {
  return blk * kSweepThreads * R + (threadIdx.x >> 5) * 32 * R + r * 32 + (threadIdx.x & 31);
}
__device__ __forceinline__ void warp_box(const float* lo_in, const float* hi_in, float* box) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    float lo = lo_in[d], hi = hi_in[d];
    for (int o = 16; o > 0; o >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    box[d] = lo;
    box[3 + d] = hi;
  }
}
__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Ring order around t0: t0, t0 + 1, t0 - 1, t0 + 2, ...; returns -1 for out-of-range steps.
__device__ __forceinline__ int ring_tile(int t0, int step, int nt) {
  const int d = (step + 1) >> 1;
  const int t = (step & 1) ? t0 + d : t0 - d;
  return (t >= 0 && t < nt) ? t : -1;
}

// Box of one group (the lane's point if valid) and its union into the warp box.
__device__ __forceinline__ void group_box(float x, float y, float z, bool valid, float* gb, float* wbox) {
  const float lo[3] = {valid ? x : 3e38f, valid ? y : 3e38f, valid ? z : 3e38f};
  const float hi[3] = {valid ? x : -3e38f, valid ? y : -3e38f, valid ? z : -3e38f};
  warp_box(lo, hi, gb);
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    wbox[d] = fminf(wbox[d], gb[d]);
    wbox[3 + d] = fmaxf(wbox[3 + d], gb[3 + d]);
  }
}

// Stage streamed tile t (coordinates, SoA) into the warp's shared memory: one float4 per lane.
__device__ __forceinline__ void stage_tile_xyz(const float* __restrict__ str, int str_np, int t, float* tx,
                                               float* ty, float* tz) {
  const int lane = threadIdx.x & 31;
  const size_t o = (size_t)t * kTQ;
  reinterpret_cast<float4*>(tx)[lane] = __ldg(reinterpret_cast<const float4*>(str + o) + lane);
  reinterpret_cast<float4*>(ty)[lane] = __ldg(reinterpret_cast<const float4*>(str + str_np + o) + lane);
  reinterpret_cast<float4*>(tz)[lane] = __ldg(reinterpret_cast<const float4*>(str + 2 * (size_t)str_np + o) + lane);
}

// Culled Pass A: (min, second) of d2 for every owned point, written at its ORIGINAL index.
// Tiles are visited in a ring around the warp's own position in Morton order so the bounds
// (largest current second minimum of each group) tighten after the first few tiles.
template <int R>
__device__ __forceinline__ void top2_cull_block(const float* __restrict__ own_soa, int own_np, int own_n,
                                                const int* __restrict__ own_perm, const float* __restrict__ str_soa,
                                                int str_np, const float* __restrict__ str_cb,
                                                const float* __restrict__ str_fb, const float* __restrict__ str_sb,
                                                int relabel, float2* __restrict__ out,
                                                unsigned long long* __restrict__ evals, const int blk, const int b) {
  constexpr int kW = kSweepThreads / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float* own = own_soa + (size_t)b * 3 * own_np;
  const float* str = str_soa + (size_t)b * 3 * str_np;
  const int nt = str_np / kTQ;
  const float* cb = str_cb + (size_t)b * nt * 6;
  const float* fb = str_fb + (size_t)b * nt * kSubPerTile * 6;
  __shared__ __align__(16) float s_t[kW][3][kTQ];
  __shared__ float s_gbox[kW][R][6], s_gmax[kW][R];
  float* tx = s_t[w][0];
  float* ty = s_t[w][1];
  float* tz = s_t[w][2];

  f2_t nx[R], ny[R], nz[R];
  float m[R], s[R], gmax[R];
  bool valid[R];
  float wbox[6] = {3e38f, 3e38f, 3e38f, -3e38f, -3e38f, -3e38f};
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int idx = cull_idx<R>(blk, r);
    valid[r] = idx < own_n;
    const float x = __ldg(own + idx), y = __ldg(own + own_np + idx), z = __ldg(own + 2 * own_np + idx);
    nx[r] = f2_pack(-x, -x); ny[r] = f2_pack(-y, -y); nz[r] = f2_pack(-z, -z);
    m[r] = __int_as_float(0x7f800000); s[r] = m[r];
    float gb[6];
    group_box(x, y, z, valid[r], gb, wbox);
    gmax[r] = __any_sync(0xffffffffu, valid[r]) ? 3e38f : -1.f;  // empty groups need nothing
#pragma unroll
    for (int d = 0; d < 6; ++d)
      if (lane == d) s_gbox[w][r][d] = gb[d];
    if (lane == 0) s_gmax[w][r] = gmax[r];
  }
  __syncwarp();
  float wmax = -1.f;
#pragma unroll
  for (int r = 0; r < R; ++r) wmax = fmaxf(wmax, gmax[r]);

  unsigned nev = 0;
  const int own_base = blk * kSweepThreads * R + w * 32 * R;
  const int t0 = min(nt - 1, (int)((long long)own_base * nt / own_np));
  // Candidate tiles come from a two-level generator: super-tiles (32 tiles) in a ring around
  // the warp's own super-tile, each tested against the warp bound with one broadcast box; the
  // 32 tiles of a surviving super-tile are tested one per lane (one ballot).  Inside the own
  // super-tile the candidates start at the own tile so the bound tightens first.  The data of
  // the NEXT candidate (its sub-tile box for this lane's (group, sub-tile) test and its
  // coordinates) is loaded into registers before the current one is evaluated, so the
  // dependent global round trips overlap the arithmetic.  A candidate chosen with an older,
  // larger bound is only a weaker filter: the result is unchanged.
  // Candidate tiles come from a generator (32 ring steps per ballot against the warp bound);
  // the data of the NEXT candidate (its sub-tile box for this lane's (group, sub-tile) test
  // and its coordinates) is loaded into registers before the current one is evaluated, so
  // the two dependent global round trips per tile overlap the arithmetic (the walk was
  // latency-bound: ncu 13 % occupancy, 45 % issue).  A candidate chosen with an older,
  // larger bound is only a weaker filter: the result is unchanged.  (A two-level walk over
  // super-tiles of 32 tiles, str_sb, measured slower here: C5 Pass A 0.57 -> 0.67 ms, C4
  // 0.88 -> 1.10 ms -- the ring order of single tiles tightens the bound sooner; the emit,
  // whose bound is fixed, does use it.)
  (void)str_sb;
  int gbase = 0, gT = -1;
  unsigned gcm = 0u;
  auto next_cand = [&]() -> int {
    while (!gcm) {
      if (gbase >= 2 * nt) return -1;
      gT = ring_tile(t0, gbase + lane, nt);
      const bool cand = gT >= 0 && box_dist2(wbox, cb + (size_t)gT * 6) * kCullMargin <= wmax;
      gcm = __ballot_sync(0xffffffffu, cand);
      gbase += 32;
    }
    const int l = __ffs(gcm) - 1;
    gcm &= gcm - 1;
    return __shfl_sync(0xffffffffu, gT, l);
  };
  const int sl_r = lane / kSubPerTile, sl_q = lane % kSubPerTile;  // this lane's (group, sub-tile)
  const bool sl_on = lane < kSubPerTile * R;
  float4 nxv, nyv, nzv;
  float nbox[6];
  auto prefetch = [&](int t) {
    const size_t o = (size_t)t * kTQ;
    nxv = __ldg(reinterpret_cast<const float4*>(str + o) + lane);
    nyv = __ldg(reinterpret_cast<const float4*>(str + str_np + o) + lane);
    nzv = __ldg(reinterpret_cast<const float4*>(str + 2 * (size_t)str_np + o) + lane);
    const float* fbp = fb + ((size_t)t * kSubPerTile + sl_q) * 6;
#pragma unroll
    for (int d = 0; d < 6; ++d) nbox[d] = sl_on ? __ldg(fbp + d) : 0.f;
  };
  int tn = next_cand();
  if (tn >= 0) prefetch(tn);
  while (tn >= 0) {
    const float4 cx = nxv, cy = nyv, cz = nzv;
    float cbx[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) cbx[d] = nbox[d];
    tn = next_cand();
    if (tn >= 0) prefetch(tn);
    bool need = false;
    if (sl_on) need = box_dist2(s_gbox[w][sl_r], cbx) * kCullMargin <= s_gmax[w][sl_r];
    const unsigned fm = __ballot_sync(0xffffffffu, need);
    if (!fm) continue;
    nev += (unsigned)__popc(fm);  // (group, sub-tile) blocks of 32 x kSub evaluations
    reinterpret_cast<float4*>(tx)[lane] = cx;
    reinterpret_cast<float4*>(ty)[lane] = cy;
    reinterpret_cast<float4*>(tz)[lane] = cz;
    __syncwarp();
    for (int q = 0; q < kSubPerTile; ++q) {
      const ulonglong2* px = reinterpret_cast<const ulonglong2*>(tx + q * kSub);
      const ulonglong2* py = reinterpret_cast<const ulonglong2*>(ty + q * kSub);
      const ulonglong2* pz = reinterpret_cast<const ulonglong2*>(tz + q * kSub);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!((fm >> (r * kSubPerTile + q)) & 1u)) continue;  // warp-uniform
#pragma unroll
        for (int k = 0; k < kSub / 4; ++k) {
          const ulonglong2 qx = px[k], qy = py[k], qz = pz[k];
          const f2_t d01 = f2_dist2(qx.x, qy.x, qz.x, nx[r], ny[r], nz[r]);
          const f2_t d23 = f2_dist2(qx.y, qy.y, qz.y, nx[r], ny[r], nz[r]);
          float d0, d1, d2, d3;
          f2_unpack(d01, d0, d1);
          f2_unpack(d23, d2, d3);
          top2_pair(m[r], s[r], d0, d1);
          top2_pair(m[r], s[r], d2, d3);
        }
      }
    }
    wmax = -1.f;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if ((fm >> (r * kSubPerTile)) & ((1u << kSubPerTile) - 1u)) gmax[r] = warp_max(valid[r] ? s[r] : -1.f);
      wmax = fmaxf(wmax, gmax[r]);
    }
    __syncwarp();  // every lane is done with the staged tile and the old bounds
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (lane == r) s_gmax[w][r] = gmax[r];
    __syncwarp();
  }
  if (evals && lane == 0 && nev) atomicAdd(evals, (unsigned long long)nev * 32ull * kSub);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int idx = cull_idx<R>(blk, r);
    if (valid[r])
      out[(size_t)b * own_n + (relabel ? idx : own_perm[(size_t)b * own_np + idx])] = make_float2(m[r], s[r]);
  }
}

template <int R>
__global__ void __launch_bounds__(kSweepThreads)
k_line_top2_cull(const float* __restrict__ own_soa, int own_np, int own_n, const int* __restrict__ own_perm,
                 const float* __restrict__ str_soa, int str_np, const float* __restrict__ str_cb,
                 const float* __restrict__ str_fb, const float* __restrict__ str_sb, int relabel,
                 float2* __restrict__ out, unsigned long long* __restrict__ evals) {
  top2_cull_block<R>(own_soa, own_np, own_n, own_perm, str_soa, str_np, str_cb, str_fb, str_sb, relabel, out,
                     evals, blockIdx.x, blockIdx.y);
}

// Both culled Pass A directions in ONE launch (grid.z = 2: rows, then columns).  At B = 1
// (C5) one direction alone fills under half of the GPU's warp slots, and the walk is
// latency-bound: the second direction's warps hide the first's latency instead of waiting
// for their own launch.
struct CullDir {
  const float* own;
  int own_np, own_n;
  const int* own_perm;
  const float* str;
  int str_np;
  const float* str_cb;
  const float* str_fb;
  float2* out;
  unsigned long long* evals;
  int nblk;
  const float* str_sb;  // super-tile boxes of the streamed cloud (k_super_box)
};
template <int R>
__global__ void __launch_bounds__(kSweepThreads) k_line_top2_cull_both(const CullDir d0, const CullDir d1,
                                                                       int relabel) {
  const CullDir& d = blockIdx.z ? d1 : d0;
  if ((int)blockIdx.x >= d.nblk) return;
  top2_cull_block<R>(d.own, d.own_np, d.own_n, d.own_perm, d.str, d.str_np, d.str_cb, d.str_fb, d.str_sb, relabel,
                     d.out, d.evals, blockIdx.x, blockIdx.y);
}

// Culled Pass B: as k_emit over the sorted clouds, evaluating only the (group, sub-tile)
// pairs within max(group's largest row emit radius, sub-tile's largest column emit radius);
// entries are emitted with ORIGINAL indices.
template <int R>
__global__ void __launch_bounds__(kSweepThreads)
k_emit_cull(const float* __restrict__ pred_soa, int np, int N, const int* __restrict__ pperm,
            const LineA* __restrict__ rowA, const float* __restrict__ gt_soa, int mp, int M,
            const int* __restrict__ gperm, int relabel, const float2* __restrict__ gre, const float* __restrict__ gcb,
            const float* __restrict__ gfb, const float* __restrict__ gce2, const float* __restrict__ gfe2,
            const float* __restrict__ gsb, const float* __restrict__ gsce2,
            uint32_t cap, uint2* __restrict__ ebuf, unsigned* __restrict__ cursor,
            unsigned* __restrict__ aux_cnt, unsigned* __restrict__ row_cnt, unsigned* __restrict__ col_cnt,
            unsigned long long* __restrict__ evals) {
  constexpr int kW = kSweepThreads / 32;
  const int b = blockIdx.y, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float* own = pred_soa + (size_t)b * 3 * np;
  const float* str = gt_soa + (size_t)b * 3 * mp;
  const int nt = mp / kTQ;
  const float* cb = gcb + (size_t)b * nt * 6;
  const float* fb = gfb + (size_t)b * nt * kSubPerTile * 6;
  const float* ce2 = gce2 + (size_t)b * nt;
  const float* fe2 = gfe2 + (size_t)b * nt * kSubPerTile;
  const float2* re = gre + (size_t)b * mp;
  const int* jp = gperm + (size_t)b * mp;
  __shared__ __align__(16) float s_t[kW][5][kTQ];
  __shared__ __align__(16) int s_j[kW][kTQ];
  __shared__ uint2 queue_all[kW][kLaneQ][32];  // per-lane emission queues (as k_emit)
  __shared__ float s_gbox[kW][R][6], s_ge[kW][R];
  float* tx = s_t[w][0];
  float* ty = s_t[w][1];
  float* tz = s_t[w][2];
  float* sR = s_t[w][3];
  float* sE = s_t[w][4];
  int* sJ = s_j[w];
  uint2* qp = &queue_all[w][0][lane];
  int qn = 0;

  f2_t nx[R], ny[R], nz[R];
  float rR2[R], rE2[R];
  int oi[R];
  float wE = -1.f;
  float wbox[6] = {3e38f, 3e38f, 3e38f, -3e38f, -3e38f, -3e38f};
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int idx = cull_idx<R>(blockIdx.x, r);
    const float x = __ldg(own + idx), y = __ldg(own + np + idx), z = __ldg(own + 2 * np + idx);
    nx[r] = f2_pack(-x, -x); ny[r] = f2_pack(-y, -y); nz[r] = f2_pack(-z, -z);
    oi[r] = pperm[(size_t)b * np + idx];
    if (relabel && oi[r] >= 0) oi[r] = idx;  // emit sorted positions
    rR2[r] = -1.f; rE2[r] = -1.f;
    if (oi[r] >= 0) {
      const LineA a = rowA[(size_t)b * N + oi[r]];
      rR2[r] = a.R2; rE2[r] = a.E2;
    }
    float gb[6];
    group_box(x, y, z, oi[r] >= 0, gb, wbox);
    const float ge = warp_max(rE2[r]);
    wE = fmaxf(wE, ge);
#pragma unroll
    for (int d = 0; d < 6; ++d)
      if (lane == d) s_gbox[w][r][d] = gb[d];
    if (lane == 0) s_ge[w][r] = ge;
  }
  __syncwarp();
  unsigned nev = 0;
  // two-level scan: 32 super-tiles per ballot (box + largest column emit radius), then the 32
  // tiles of each surviving super-tile (one per lane)
  const int nst = (nt + kSuper - 1) / kSuper;
  const float* sbx = gsb + (size_t)b * nst * 6;
  const float* sce = gsce2 + (size_t)b * nst;
  unsigned scm = 0u;
  int sbase = 0, ST = -1;
  for (;;) {
    while (!scm && sbase < nst) {
      ST = sbase + lane;
      bool sc = false;
      if (ST < nst) {
        const float lb = box_dist2(wbox, sbx + (size_t)ST * 6) * kCullMargin;
        sc = lb <= fmaxf(wE, sce[ST]) && lb < 3e38f;
      }
      scm = __ballot_sync(0xffffffffu, sc);
      sbase += 32;
    }
    if (!scm) break;
    const int sl = __ffs(scm) - 1;
    scm &= scm - 1;
    const int T = __shfl_sync(0xffffffffu, ST, sl) * kSuper + lane;
    bool cand = false;
    if (T < nt) {
      const float lb = box_dist2(wbox, cb + (size_t)T * 6) * kCullMargin;
      cand = lb <= fmaxf(wE, ce2[T]) && lb < 3e38f;
    }
    unsigned cm = __ballot_sync(0xffffffffu, cand);
    while (cm) {
      const int l = __ffs(cm) - 1;
      cm &= cm - 1;
      const int t = __shfl_sync(0xffffffffu, T, l);
      bool need = false;
      if (lane < kSubPerTile * R) {
        const int r = lane / kSubPerTile, sq = t * kSubPerTile + lane % kSubPerTile;
        need = box_dist2(s_gbox[w][r], fb + (size_t)sq * 6) * kCullMargin <= fmaxf(s_ge[w][r], fe2[sq]);
      }
      const unsigned fm = __ballot_sync(0xffffffffu, need);
      if (!fm) continue;
      nev += (unsigned)__popc(fm);
      stage_tile_xyz(str, mp, t, tx, ty, tz);
      {
        const float4* src = reinterpret_cast<const float4*>(re + (size_t)t * kTQ);
        const float4 a0 = __ldg(src + 2 * lane), a1 = __ldg(src + 2 * lane + 1);
        reinterpret_cast<float4*>(sR)[lane] = make_float4(a0.x, a0.z, a1.x, a1.z);
        reinterpret_cast<float4*>(sE)[lane] = make_float4(a0.y, a0.w, a1.y, a1.w);
        int4 jj = __ldg(reinterpret_cast<const int4*>(jp + (size_t)t * kTQ) + lane);
        if (relabel) {  // sorted positions of the real points
          const int k0 = t * kTQ + 4 * lane;
          jj = make_int4(jj.x >= 0 ? k0 : -1, jj.y >= 0 ? k0 + 1 : -1, jj.z >= 0 ? k0 + 2 : -1, jj.w >= 0 ? k0 + 3 : -1);
        }
        reinterpret_cast<int4*>(sJ)[lane] = jj;
      }
      __syncwarp();
      for (int q = 0; q < kSubPerTile; ++q) {
        const ulonglong2* px = reinterpret_cast<const ulonglong2*>(tx + q * kSub);
        const ulonglong2* py = reinterpret_cast<const ulonglong2*>(ty + q * kSub);
        const ulonglong2* pz = reinterpret_cast<const ulonglong2*>(tz + q * kSub);
        const float4* pE = reinterpret_cast<const float4*>(sE + q * kSub);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!((fm >> (r * kSubPerTile + q)) & 1u)) continue;  // warp-uniform
          // hit mask over the 32 points of the sub-tile (no branch / vote per 4 points), then
          // the lanes' hits recomputed (same bits) and queued warp-synchronously (as k_emit)
          uint32_t mask = 0u;
#pragma unroll 2
          for (int k = 0; k < kSub / 4; ++k) {
            const ulonglong2 qx = px[k], qy = py[k], qz = pz[k];
            const float4 ce = pE[k];
            const f2_t d01 = f2_dist2(qx.x, qy.x, qz.x, nx[r], ny[r], nz[r]);
            const f2_t d23 = f2_dist2(qx.y, qy.y, qz.y, nx[r], ny[r], nz[r]);
            float d[4];
            f2_unpack(d01, d[0], d[1]);
            f2_unpack(d23, d[2], d[3]);
            const uint32_t h = (d[0] <= fmaxf(rE2[r], ce.x) ? 1u : 0u) | (d[1] <= fmaxf(rE2[r], ce.y) ? 2u : 0u) |
                               (d[2] <= fmaxf(rE2[r], ce.z) ? 4u : 0u) | (d[3] <= fmaxf(rE2[r], ce.w) ? 8u : 0u);
            mask |= h << (4 * k);
          }
          uint32_t m = oi[r] >= 0 ? mask : 0u;
          if (!__any_sync(0xffffffffu, m)) continue;
          float xr, yr, zr, tmp;
          f2_unpack(nx[r], xr, tmp);
          f2_unpack(ny[r], yr, tmp);
          f2_unpack(nz[r], zr, tmp);
          while (__any_sync(0xffffffffu, m)) {
            if (__any_sync(0xffffffffu, qn == kLaneQ)) {
              __syncwarp();
              lane_flush(b, qp, qn, cap, ebuf, cursor, aux_cnt, row_cnt, N, col_cnt, M);
              qn = 0;
              __syncwarp();
            }
            if (m) {
              const int qq = q * kSub + __ffs(m) - 1;
              m &= m - 1;
              const int j = sJ[qq];
              if (j >= 0) {
                const float dx = __fadd_rn(tx[qq], xr), dy = __fadd_rn(ty[qq], yr), dz = __fadd_rn(tz[qq], zr);
                float d2 = __fmul_rn(dx, dx);
                d2 = __fmaf_rn(dy, dy, d2);
                d2 = __fmaf_rn(dz, dz, d2);
                const uint32_t fl = (d2 <= rR2[r] ? kFlagRow : 0u) | (d2 <= sR[qq] ? kFlagCol : 0u);
                qp[qn * 32] = make_uint2((uint32_t)oi[r], (uint32_t)j | fl);
                ++qn;
              }
            }
          }
        }
      }
      __syncwarp();  // every lane is done with the staged tile
    }
  }
  __syncwarp();
  lane_flush(b, qp, qn, cap, ebuf, cursor, aux_cnt, row_cnt, N, col_cnt, M);
  if (evals && lane == 0 && nev) atomicAdd(evals, (unsigned long long)nev * 32ull * kSub);
}

}  // namespace apml
