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

// Joint bounding box of pred and gt of each pair: bb[b] = {lo x,y,z, hi x,y,z}.
__global__ void __launch_bounds__(1024)
k_pair_bbox(const float* __restrict__ pred, int N, const float* __restrict__ gt, int M, float* __restrict__ bb) {
  const int b = blockIdx.x;
  float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
  for (int k = threadIdx.x; k < N + M; k += blockDim.x) {
    const float* p = k < N ? pred + ((size_t)b * N + k) * 3 : gt + ((size_t)b * M + (k - N)) * 3;
#pragma unroll
    for (int d = 0; d < 3; ++d) { lo[d] = fminf(lo[d], p[d]); hi[d] = fmaxf(hi[d], p[d]); }
  }
  __shared__ float red[6][32];
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
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k)
      v = threadIdx.x < 3 ? fminf(v, red[threadIdx.x][k]) : fmaxf(v, red[threadIdx.x][k]);
    bb[b * 6 + threadIdx.x] = v;
  }
}

__device__ __forceinline__ uint32_t spread_bits3(uint32_t v) {  // 10-bit v -> every third bit
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// Morton cell key of every point (bits per axis) and the per-pair cell histogram.
__global__ void k_cell_count(const float* __restrict__ pts, int n, const float* __restrict__ bb, int bits,
                             uint32_t* __restrict__ key, uint32_t* __restrict__ hist) {
  const int b = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const float* p = pts + ((size_t)b * n + k) * 3;
  const float* box = bb + b * 6;
  const uint32_t cells_axis = 1u << bits;
  uint32_t c[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const float ext = fmaxf(box[3 + d] - box[d], 1e-30f);
    float f = (p[d] - box[d]) / ext * (float)cells_axis;
    c[d] = (uint32_t)fminf(fmaxf(f, 0.f), (float)(cells_axis - 1));
  }
  const uint32_t kk = spread_bits3(c[0]) | (spread_bits3(c[1]) << 1) | (spread_bits3(c[2]) << 2);
  key[(size_t)b * n + k] = kk;
  atomicAdd(hist + (size_t)b * ((1u << (3 * bits)) + 1) + kk, 1u);
}

// Place every point at its sorted position: SoA coordinates (pads = sentinel) + perm.
__global__ void k_cell_scatter(const float* __restrict__ pts, int n, int np, float sentinel, int bits,
                               const uint32_t* __restrict__ key, const uint32_t* __restrict__ start,
                               uint32_t* __restrict__ fill, float* __restrict__ soa, int* __restrict__ perm) {
  const int b = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  float* s = soa + (size_t)b * 3 * np;
  if (k >= n) {  // pads occupy the sorted positions [n, np)
    s[k] = sentinel; s[np + k] = sentinel; s[2 * np + k] = sentinel;
    perm[(size_t)b * np + k] = -1;
    return;
  }
  const size_t hb = (size_t)b * ((1u << (3 * bits)) + 1);
  const uint32_t kk = key[(size_t)b * n + k];
  const uint32_t pos = start[hb + kk] + atomicAdd(fill + hb + kk, 1u);
  const float* p = pts + ((size_t)b * n + k) * 3;
  s[pos] = p[0]; s[np + pos] = p[1]; s[2 * np + pos] = p[2];
  perm[(size_t)b * np + pos] = k;
}

// Bounding box of every kTQ-point tile of a sorted cloud (pads excluded): tb[b][t] = 6 floats.
__global__ void k_tile_bbox(const float* __restrict__ soa, int np, int n, float* __restrict__ tb) {
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
  __shared__ float red[6][kTQ / 32];
#pragma unroll
  for (int d = 0; d < 3; ++d)
    for (int o = 16; o > 0; o >>= 1) {
      lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int d = 0; d < 3; ++d) { red[d][w] = lo[d]; red[3 + d][w] = hi[d]; }
  __syncthreads();
  if (threadIdx.x < 6) {
    float v = threadIdx.x < 3 ? 3e38f : -3e38f;
    for (int q = 0; q < kTQ / 32; ++q)
      v = threadIdx.x < 3 ? fminf(v, red[threadIdx.x][q]) : fmaxf(v, red[threadIdx.x][q]);
    tb[((size_t)b * (np / kTQ) + t) * 6 + threadIdx.x] = v;
  }
}

// Largest emit radius E2 of the columns of each gt tile (-1 for pads).
__global__ void k_tile_e2max(const int* __restrict__ gperm, int mp, const LineA* __restrict__ colA, int M,
                             float* __restrict__ e2max) {
  const int b = blockIdx.y, t = blockIdx.x;
  const int k = t * kTQ + threadIdx.x;
  const int j = gperm[(size_t)b * mp + k];
  float e = j >= 0 ? colA[(size_t)b * M + j].E2 : -1.f;
  for (int o = 16; o > 0; o >>= 1) e = fmaxf(e, __shfl_xor_sync(0xffffffffu, e, o));
  __shared__ float red[kTQ / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    float v = -1.f;
    for (int q = 0; q < kTQ / 32; ++q) v = fmaxf(v, red[q]);
    e2max[(size_t)b * (mp / kTQ) + t] = v;
  }
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

// Own block bounding box = union of its 4 (= kSweepThreads * R / kTQ) tiles.
template <int R>
__device__ __forceinline__ void own_block_box(const float* tb, int blk, float* box) {
  if (threadIdx.x < 6) {
    float v = threadIdx.x < 3 ? 3e38f : -3e38f;
    for (int q = 0; q < kSweepThreads * R / kTQ; ++q) {
      const float u = tb[(size_t)(blk * (kSweepThreads * R / kTQ) + q) * 6 + threadIdx.x];
      v = threadIdx.x < 3 ? fminf(v, u) : fmaxf(v, u);
    }
    box[threadIdx.x] = v;
  }
}

// Warp-level culling: in the culled kernels a warp owns R*32 CONSECUTIVE sorted points
// (idx = block base + warp*32R + r*32 + lane), i.e. a compact piece of the Morton curve, and
// skips a tile on its own bounds; the CTA loads a tile only if some warp may need it.
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

// Ring order around t0: t0, t0 + 1, t0 - 1, t0 + 2, ...; returns -1 for out-of-range steps.
__device__ __forceinline__ int ring_tile(int t0, int step, int nt) {
  const int d = (step + 1) >> 1;
  const int t = (step & 1) ? t0 + d : t0 - d;
  return (t >= 0 && t < nt) ? t : -1;
}

// Culled Pass A: (min, second) of d2 for every owned point, written at its ORIGINAL index.
template <int R>
__global__ void __launch_bounds__(kSweepThreads)
k_line_top2_cull(const float* __restrict__ own_soa, int own_np, int own_n, const int* __restrict__ own_perm,
                 const float* __restrict__ own_tb, const float* __restrict__ str_soa, int str_np,
                 const float* __restrict__ str_tb, float2* __restrict__ out) {
  const int b = blockIdx.y, blk = blockIdx.x;
  const float* own = own_soa + (size_t)b * 3 * own_np;
  const float* str = str_soa + (size_t)b * 3 * str_np;
  const int nt = str_np / kTQ;
  const float* stb = str_tb + (size_t)b * nt * 6;
  constexpr int kW = kSweepThreads / 32;
  const int w = threadIdx.x >> 5;
  __shared__ __align__(16) float sx[kTQ], sy[kTQ], sz[kTQ];
  __shared__ float s_box[6], s_wbox[kW][6], s_wmax[kW];
  own_block_box<R>(own_tb + (size_t)b * (own_np / kTQ) * 6, blk, s_box);

  f2_t nx[R], ny[R], nz[R];
  float m[R], s[R];
  bool valid[R];
  float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int idx = cull_idx<R>(blk, r);
    valid[r] = idx < own_n;
    const float x = __ldg(own + idx), y = __ldg(own + own_np + idx), z = __ldg(own + 2 * own_np + idx);
    if (valid[r]) {
      lo[0] = fminf(lo[0], x); lo[1] = fminf(lo[1], y); lo[2] = fminf(lo[2], z);
      hi[0] = fmaxf(hi[0], x); hi[1] = fmaxf(hi[1], y); hi[2] = fmaxf(hi[2], z);
    }
    nx[r] = f2_pack(-x, -x); ny[r] = f2_pack(-y, -y); nz[r] = f2_pack(-z, -z);
    m[r] = __int_as_float(0x7f800000); s[r] = m[r];
  }
  float wbox[6];
  warp_box(lo, hi, wbox);
  float wmax = __int_as_float(0x7f800000);  // this warp's largest current second minimum
  if ((threadIdx.x & 31) == 0) {
    for (int d = 0; d < 6; ++d) s_wbox[w][d] = wbox[d];
    s_wmax[w] = wmax;
  }
  __syncthreads();
  const int t0 = min(nt - 1, (int)(((long long)blk * kSweepThreads * R * str_np / own_np) / kTQ));
  for (int step = 0; step < 2 * nt; ++step) {
    const int t = ring_tile(t0, step, nt);
    if (t < 0) continue;
    const float* tbox = stb + (size_t)t * 6;
    // CTA: load the tile if any warp may need it (uniform decision from shared state)
    bool any = false;
    if (box_dist2(s_box, tbox) * kCullMargin <= 3e38f)
      for (int k = 0; k < kW; ++k) any |= box_dist2(s_wbox[k], tbox) * kCullMargin <= s_wmax[k];
    if (!any) continue;
    __syncthreads();
    load_tile(str, str_np, t * kTQ, sx, sy, sz);
    __syncthreads();
    if (box_dist2(wbox, tbox) * kCullMargin <= wmax) {  // warp-uniform
      const ulonglong2* px = reinterpret_cast<const ulonglong2*>(sx);
      const ulonglong2* py = reinterpret_cast<const ulonglong2*>(sy);
      const ulonglong2* pz = reinterpret_cast<const ulonglong2*>(sz);
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
          top2_pair(m[r], s[r], d2, d3);
        }
      }
      float mx = -1.f;
#pragma unroll
      for (int r = 0; r < R; ++r) mx = valid[r] ? fmaxf(mx, s[r]) : mx;
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      wmax = mx;
    }
    __syncthreads();  // every warp has finished reading the tile and the old bounds
    if ((threadIdx.x & 31) == 0) s_wmax[w] = wmax;
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int idx = cull_idx<R>(blk, r);
    if (valid[r]) out[(size_t)b * own_n + own_perm[(size_t)b * own_np + idx]] = make_float2(m[r], s[r]);
  }
}

// Culled Pass B: as k_emit over the sorted clouds, skipping tiles beyond the emit radii;
// entries are emitted with ORIGINAL indices.
template <int R>
__global__ void __launch_bounds__(kSweepThreads)
k_emit_cull(const float* __restrict__ pred_soa, int np, int N, const int* __restrict__ pperm,
            const LineA* __restrict__ rowA, const float* __restrict__ ptb,
            const float* __restrict__ gt_soa, int mp, int M, const int* __restrict__ gperm,
            const LineA* __restrict__ colA, const float* __restrict__ gtb, const float* __restrict__ ge2max,
            uint32_t cap, uint2* __restrict__ ebuf, unsigned* __restrict__ cursor,
            unsigned* __restrict__ aux_cnt, unsigned* __restrict__ row_cnt, unsigned* __restrict__ col_cnt) {
  const int b = blockIdx.y, blk = blockIdx.x;
  const float* own = pred_soa + (size_t)b * 3 * np;
  const float* str = gt_soa + (size_t)b * 3 * mp;
  const int nt = mp / kTQ;
  const float* stb = gtb + (size_t)b * nt * 6;
  const float* se2 = ge2max + (size_t)b * nt;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ __align__(16) float sx[kTQ], sy[kTQ], sz[kTQ], sR[kTQ], sE[kTQ];
  __shared__ int sJ[kTQ];
  __shared__ uint2 wbuf_all[kSweepThreads / 32][kWarpBuf];
  __shared__ float s_box[6], s_wmax[kSweepThreads / 32], s_rmax;
  uint2* wbuf = wbuf_all[w];
  int wcnt = 0;
  own_block_box<R>(ptb + (size_t)b * (np / kTQ) * 6, blk, s_box);

  f2_t nx[R], ny[R], nz[R];
  float rR2[R], rE2[R];
  int oi[R];
  float emax = -1.f;
  float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int idx = cull_idx<R>(blk, r);
    const float x = __ldg(own + idx), y = __ldg(own + np + idx), z = __ldg(own + 2 * np + idx);
    nx[r] = f2_pack(-x, -x); ny[r] = f2_pack(-y, -y); nz[r] = f2_pack(-z, -z);
    oi[r] = pperm[(size_t)b * np + idx];
    if (oi[r] >= 0) {
      const LineA a = rowA[(size_t)b * N + oi[r]];
      rR2[r] = a.R2; rE2[r] = a.E2;
      emax = fmaxf(emax, a.E2);
      lo[0] = fminf(lo[0], x); lo[1] = fminf(lo[1], y); lo[2] = fminf(lo[2], z);
      hi[0] = fmaxf(hi[0], x); hi[1] = fmaxf(hi[1], y); hi[2] = fmaxf(hi[2], z);
    } else {
      rR2[r] = -1.f; rE2[r] = -1.f;
    }
  }
  float wbox[6];
  warp_box(lo, hi, wbox);
  for (int o = 16; o > 0; o >>= 1) emax = fmaxf(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  if (lane == 0) s_wmax[w] = emax;
  __syncthreads();
  if (threadIdx.x == 0) {
    float v = -1.f;
    for (int k = 0; k < kSweepThreads / 32; ++k) v = fmaxf(v, s_wmax[k]);
    s_rmax = v;
  }
  __syncthreads();
  const float rmax = s_rmax;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int t = 0; t < nt; ++t) {
    if (box_dist2(s_box, stb + (size_t)t * 6) * kCullMargin > fmaxf(rmax, se2[t])) continue;  // uniform
    const bool wneed = box_dist2(wbox, stb + (size_t)t * 6) * kCullMargin <= fmaxf(emax, se2[t]);
    const int jt = t * kTQ;
    __syncthreads();
    load_tile(str, mp, jt, sx, sy, sz);
    for (int q = threadIdx.x; q < kTQ; q += kSweepThreads) {
      const int j = gperm[(size_t)b * mp + jt + q];
      sJ[q] = j;
      if (j >= 0) {
        const LineA a = colA[(size_t)b * M + j];
        sR[q] = a.R2; sE[q] = a.E2;
      } else {
        sR[q] = -1.f; sE[q] = -1.f;
      }
    }
    __syncthreads();
    const ulonglong2* px = reinterpret_cast<const ulonglong2*>(sx);
    const ulonglong2* py = reinterpret_cast<const ulonglong2*>(sy);
    const ulonglong2* pz = reinterpret_cast<const ulonglong2*>(sz);
    const float4* pE = reinterpret_cast<const float4*>(sE);
#pragma unroll 2
    for (int q = 0; q < (wneed ? kTQ / 4 : 0); ++q) {  // warp-uniform trip count
      const ulonglong2 qx = px[q], qy = py[q], qz = pz[q];
      const float4 ce = pE[q];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const f2_t d01 = f2_dist2(qx.x, qy.x, qz.x, nx[r], ny[r], nz[r]);
        const f2_t d23 = f2_dist2(qx.y, qy.y, qz.y, nx[r], ny[r], nz[r]);
        float d[4];
        f2_unpack(d01, d[0], d[1]);
        f2_unpack(d23, d[2], d[3]);
        const bool hit = (d[0] <= fmaxf(rE2[r], ce.x)) | (d[1] <= fmaxf(rE2[r], ce.y)) |
                         (d[2] <= fmaxf(rE2[r], ce.z)) | (d[3] <= fmaxf(rE2[r], ce.w));
        if (__any_sync(0xffffffffu, hit)) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int qq = 4 * q + c;
            const int j = sJ[qq];
            const bool h = d[c] <= fmaxf(rE2[r], sE[qq]) && oi[r] >= 0 && j >= 0;
            const unsigned bal = __ballot_sync(0xffffffffu, h);
            if (h) {
              const uint32_t fl = (d[c] <= rR2[r] ? kFlagRow : 0u) | (d[c] <= sR[qq] ? kFlagCol : 0u);
              wbuf[wcnt + __popc(bal & lt_mask)] = make_uint2((uint32_t)oi[r], (uint32_t)j | fl);
            }
            wcnt += __popc(bal);
          }
          if (wcnt > kFlushAt) {
            __syncwarp();
            warp_flush(b, wbuf, wcnt, cap, ebuf, cursor, aux_cnt, row_cnt, N, col_cnt, M);
            wcnt = 0;
          }
        }
      }
    }
  }
  __syncwarp();
  if (wcnt) warp_flush(b, wbuf, wcnt, cap, ebuf, cursor, aux_cnt, row_cnt, N, col_cnt, M);
}

}  // namespace apml
