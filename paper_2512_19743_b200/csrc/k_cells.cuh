// k_cells.cuh -- exact culled distance sweeps over the Morton CELL grid (the
// paper's future work, "restrict the candidate support, for example via neighborhood
// pruning"), the default culled mode (APML_CULL_MODE=0 selects the tile walk of k_cull.cuh).
//
// Both clouds of a pair are counting-sorted by the Morton key of their cell in a G^3 grid over
// the pair's joint bounding box (k_cell_count / k_cell_scatter of k_cull.cuh), so every cell's
// points are one contiguous range [start[key], start[key + 1]) of the sorted cloud.  A warp owns
// 32 consecutive sorted points (one per lane) and scans, cooperatively, the cells of a box
// around them: the box of the lanes' own cells grown by one cell (or, when that box is large, a
// 3x3x3 cube per distinct own cell, for the lanes of that cell only).  The cells' points are
// staged in the warp's shared memory and every lane evaluates all of them with the packed
// FADD2 / FMUL2 / FFMA2 distance of the full sweeps (identical d2 bits).  A lane is finished
// when its bound is inside the scanned box: every point outside the box is farther than the
// distance from the lane's point to the box faces (the faces on the grid boundary have no
// points beyond them), so
//   Pass A (top-2):    second min  <= face distance^2   (ties beyond cannot change values)
//   Pass B (emit):     emit radius^2 <  face distance^2
// otherwise the box grows by one shell of cells (only the new cells are scanned, so no point
// is counted twice for a lane) until every lane of the group is finished.  Face distances
// carry a margin for the rounding of the cell coordinates and of d2.
//
// Pass B is split into two passes so that the union support is emitted exactly once without a
// global candidate bound: the row pass (own = pred) emits (i, j) with d2 <= E_i^2; the column
// pass (own = gt) emits (i, j) with d2 <= E'_j^2 and d2 > E_i^2.  Together: d2 <= max(E_i^2,
// E'_j^2), the set (and the flags) of k_emit.
#pragma once
#include "k_cull.cuh"

namespace apml {

constexpr int kCellWarps = 4;        // warps per CTA (independent; no CTA barrier)
constexpr int kCellBuf = 256;        // staged points per warp
constexpr int kCellMaxBlock = 216;   // largest grown warp box (cells) scanned for all lanes at once
__constant__ int g_cell_maxblock = kCellMaxBlock;  // (tuning: APML_CELL_MAXBLOCK)

struct CellBox {
  int lo[3], hi[3];
};

// Diagnostics (a build with -DAPML_CELL_DIAG=1, printed with APML_CELL_STATS=1): [0] cell rounds,
// [1] staged points, [2] far lanes, [3] shells, [4] groups, [5] warps -- Pass A in [0, 8), the
// emit in [8, 16).  Compiled out by default (the flag load alone cost ~5 % of the emit).
#ifndef APML_CELL_DIAG
#define APML_CELL_DIAG 0
#endif
__device__ unsigned long long g_cell_stats[16];
// Bounds checks of the cell kernels (a build with -DAPML_CELL_CHECKS=1; compute-sanitizer is
// not available on the GPU pool): every staged slot, sorted position, cell key, queue slot and
// output index is checked, a violation traps the kernel (the test then fails loudly).
#ifndef APML_CELL_CHECKS
#define APML_CELL_CHECKS 0
#endif
#define CELL_CHECK(cond)                                                                        \
  do {                                                                                          \
    if (APML_CELL_CHECKS && !(cond)) {                                                          \
      printf("apml cell check failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);              \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
__device__ __forceinline__ void cell_stat(int k, unsigned long long v) {
  if (APML_CELL_DIAG && (threadIdx.x & 31) == 0 && v) atomicAdd(&g_cell_stats[k], v);
}

__device__ __forceinline__ uint32_t morton3(uint32_t x, uint32_t y, uint32_t z) {
  return spread_bits3(x) | (spread_bits3(y) << 1) | (spread_bits3(z) << 2);
}

// Per-lane cell coordinates (cell_axis of k_cull.cuh: the cell the point was sorted into), the
// fractional coordinates and the cell widths.
struct CellFrame {
  float lo[3], hi[3], h[3], ext[3];
  int G;
};
__device__ __forceinline__ CellFrame cell_frame(const float* bb, int bits) {
  CellFrame F;
  F.G = 1 << bits;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    F.lo[d] = bb[d];
    F.hi[d] = bb[3 + d];
    F.ext[d] = fmaxf(bb[3 + d] - bb[d], 1e-30f);
    F.h[d] = F.ext[d] / (float)F.G;
  }
  return F;
}

// Squared distance from a point (fractional cell coordinates f) to the outside of box B,
// shrunk by the rounding margins; +inf when B covers the grid.
__device__ __forceinline__ float face_bound2(const CellFrame& F, const float* f, const CellBox& B) {
  float d = 3e38f;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float mg = 4e-6f * F.ext[a];
    if (B.lo[a] > 0) d = fminf(d, (f[a] - (float)B.lo[a]) * F.h[a] - mg);
    if (B.hi[a] < F.G - 1) d = fminf(d, ((float)(B.hi[a] + 1) - f[a]) * F.h[a] - mg);
  }
  if (d >= 3e38f) return __int_as_float(0x7f800000);
  d = fmaxf(d, 0.f);
  return d * d * (1.0f - 1e-5f);
}

__device__ __forceinline__ bool box_covers_grid(const CellBox& B, int G) {
  return B.lo[0] == 0 && B.lo[1] == 0 && B.lo[2] == 0 && B.hi[0] == G - 1 && B.hi[1] == G - 1 && B.hi[2] == G - 1;
}
__device__ __forceinline__ CellBox box_grow(const CellBox& B, int G) {
  CellBox N;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    N.lo[a] = max(B.lo[a] - 1, 0);
    N.hi[a] = min(B.hi[a] + 1, G - 1);
  }
  return N;
}

// The warp's staging buffer (shared memory): coordinates, one radius and the output index of
// the other cloud's points (the radius / index only for the emit).
struct CellStage {
  float* x;
  float* y;
  float* z;
  float* r2;
  int* id;
};

// Enumerate the cells of box B that are not in box S (S = NULL: none), 32 per round (one per
// lane), and stage their points; eval(cnt) is called whenever the buffer is full and for the
// remainder.  str: sorted SoA of the streamed cloud; start: its cell starts [cells1].
// Staging is lane-parallel over the round's points: slot s (of the T points of the round) finds
// its cell by a binary search over the lanes' inclusive counts (5 shuffles), so the loads of
// 32 points are in flight together (a lane-serial copy of its own cell was latency-bound).
template <bool kEmit, typename Eval>
__device__ __forceinline__ void scan_box(const CellBox& B, const CellBox* S, const uint32_t* __restrict__ start,
                                         const float* __restrict__ str, int str_np, const float* __restrict__ r2src,
                                         const int* __restrict__ perm, int relabel, const CellStage& st, int& filled,
                                         Eval&& eval, const float4* __restrict__ s4 = nullptr) {
  // s4 (relabelled clouds): the float4 copy in sorted order -- one 16-byte load per point
  // instead of three from the SoA copy (which is then not written at all)
  const int lane = threadIdx.x & 31;
  // the box is enumerated in x-PAIRS of cells (2 px, 2 px + 1): x is the lowest bit of the
  // Morton key, so the two cells of a pair are consecutive keys and their points one contiguous
  // range -- one start lookup and one lane per pair (about half the rounds); a pair half outside
  // the box (or inside the skip box S) contributes its other cell only
  const int px0 = B.lo[0] >> 1;
  const int ex = (B.hi[0] >> 1) - px0 + 1, ey = B.hi[1] - B.lo[1] + 1, ez = B.hi[2] - B.lo[2] + 1;
  const int exy = ex * ey, V = exy * ez;
  // small-integer division by ex, ex * ey in fp32 (exact for V < 2^17: the quotient's true value
  // is at least 0.5 / ex away from an integer)
  const float rx = 1.0f / (float)ex, rxy = 1.0f / (float)exy;
  auto in_skip = [&](int ix, int iy, int iz) {
    return S && ix >= S->lo[0] && ix <= S->hi[0] && iy >= S->lo[1] && iy <= S->hi[1] && iz >= S->lo[2] &&
           iz <= S->hi[2];
  };
  // the cell starts of the NEXT round are loaded before this round's points are staged and
  // evaluated (their latency overlaps the work)
  auto cell_of = [&](int idx, uint32_t& cst, uint32_t& cnt) {
    cst = 0;
    cnt = 0;
    if (idx < V) {
      const int qz = (int)(((float)idx + 0.5f) * rxy), rem = idx - qz * exy;
      const int qy = (int)(((float)rem + 0.5f) * rx), qx = rem - qy * ex;
      const int x0 = 2 * (px0 + qx), iy = B.lo[1] + qy, iz = B.lo[2] + qz;
      const bool in0 = x0 >= B.lo[0] && !in_skip(x0, iy, iz);
      const bool in1 = x0 + 1 <= B.hi[0] && !in_skip(x0 + 1, iy, iz);
      if (in0 || in1) {
        const uint32_t key = morton3((uint32_t)(in0 ? x0 : x0 + 1), (uint32_t)iy, (uint32_t)iz);
        CELL_CHECK(x0 >= 0 && iy >= 0 && iz >= 0 && x0 < 1024 && iy < 1024 && iz < 1024);
        cst = __ldg(start + key);
        cnt = __ldg(start + key + ((in0 && in1) ? 2u : 1u));
        CELL_CHECK(cnt >= cst && cnt <= (uint32_t)str_np);
      }
    }
  };
  uint32_t ncst, ncnt;
  cell_of(lane, ncst, ncnt);
  for (int base = 0; base < V; base += 32) {
    cell_stat(8 * kEmit + 0, 1);
    const uint32_t cst = ncst, cnt = ncnt - ncst;
    if (base + 32 < V) cell_of(base + 32 + lane, ncst, ncnt);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t T = __shfl_sync(0xffffffffu, inc, 31);
    cell_stat(8 * kEmit + 1, T);
    const uint32_t bse = cst - (inc - cnt);  // sorted position of round slot s of this lane's cell: bse + s
    auto src_of = [&](uint32_t s) {
      int l = 0;
#pragma unroll
      for (int wd = 16; wd; wd >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, inc, l + wd - 1);
        if (v <= s) l += wd;
      }
      return __shfl_sync(0xffffffffu, bse, l & 31) + s;
    };
    for (uint32_t sb = 0; sb < T; sb += 64) {  // two slots per lane per step: 64 loads in flight
      if (filled > kCellBuf - 64) {
        __syncwarp();
        eval(filled);
        filled = 0;
      }
      const uint32_t s0 = sb + (uint32_t)lane, s1 = s0 + 32;
      const uint32_t src0 = src_of(s0), src1 = src_of(s1);
      const bool v0 = s0 < T, v1 = s1 < T;
      float x0 = 0.f, y0 = 0.f, z0 = 0.f, x1 = 0.f, y1 = 0.f, z1 = 0.f, r0 = 0.f, r1 = 0.f;
      int o0 = 0, o1 = 0;
      CELL_CHECK(!v0 || (src0 < (uint32_t)str_np && filled + lane < kCellBuf));
      CELL_CHECK(!v1 || (src1 < (uint32_t)str_np && filled + 32 + lane < kCellBuf));
      if (v0 && s4) {
        const float4 q = __ldg(s4 + src0);
        x0 = q.x; y0 = q.y; z0 = q.z;
        if (kEmit) { o0 = relabel ? (int)src0 : __ldg(perm + src0); }
      } else if (v0) {
        x0 = __ldg(str + src0); y0 = __ldg(str + str_np + src0); z0 = __ldg(str + 2 * (size_t)str_np + src0);
        if (kEmit) { o0 = relabel ? (int)src0 : __ldg(perm + src0); }
      }
      if (v1 && s4) {
        const float4 q = __ldg(s4 + src1);
        x1 = q.x; y1 = q.y; z1 = q.z;
        if (kEmit) { o1 = relabel ? (int)src1 : __ldg(perm + src1); }
      } else if (v1) {
        x1 = __ldg(str + src1); y1 = __ldg(str + str_np + src1); z1 = __ldg(str + 2 * (size_t)str_np + src1);
        if (kEmit) { o1 = relabel ? (int)src1 : __ldg(perm + src1); }
      }
      if (kEmit) {
        if (v0) r0 = __ldg(r2src + 4 * (size_t)o0);  // a field of the LineA at o
        if (v1) r1 = __ldg(r2src + 4 * (size_t)o1);
      }
      if (v0) {
        st.x[filled + lane] = x0; st.y[filled + lane] = y0; st.z[filled + lane] = z0;
        if (kEmit) { st.id[filled + lane] = o0; st.r2[filled + lane] = r0; }
      }
      if (v1) {
        st.x[filled + 32 + lane] = x1; st.y[filled + 32 + lane] = y1; st.z[filled + 32 + lane] = z1;
        if (kEmit) { st.id[filled + 32 + lane] = o1; st.r2[filled + 32 + lane] = r1; }
      }
      filled += (int)min(64u, T - sb);
    }
  }
}

// Pad the staged points [cnt, cnt rounded up to 4) with a far sentinel (d2 = +inf, index -1).
template <bool kEmit>
__device__ __forceinline__ int stage_pad(const CellStage& st, int cnt) {
  const int lane = threadIdx.x & 31;
  const int c4 = (cnt + 3) & ~3;
  if (lane < c4 - cnt) {
    st.x[cnt + lane] = 1e30f;
    st.y[cnt + lane] = 1e30f;
    st.z[cnt + lane] = 1e30f;
    if (kEmit) {
      st.id[cnt + lane] = -1;
      st.r2[cnt + lane] = -1.f;
    }
  }
  __syncwarp();
  return c4;
}
// Own points of a warp: 32 consecutive sorted positions (one per lane).
struct CellOwn {
  float x, y, z, f[3];
  int c[3];
  bool valid;
};
__device__ __forceinline__ CellOwn cell_own(const float* __restrict__ own, int own_np, int own_n, int k,
                                            const CellFrame& F, const float4* __restrict__ own4 = nullptr) {
  CellOwn o;
  o.valid = k < own_n;
  if (own4) {
    const float4 q = o.valid ? __ldg(own4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
    o.x = q.x; o.y = q.y; o.z = q.z;
  } else {
    o.x = o.valid ? __ldg(own + k) : 0.f;
    o.y = o.valid ? __ldg(own + own_np + k) : 0.f;
    o.z = o.valid ? __ldg(own + 2 * (size_t)own_np + k) : 0.f;
  }
  const float p[3] = {o.x, o.y, o.z};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    o.f[a] = 0.f;
    o.c[a] = o.valid ? (int)cell_axis(p[a], F.lo[a], F.hi[a], (uint32_t)F.G, &o.f[a]) : 0;
  }
  return o;
}

__device__ __forceinline__ CellBox cube_box(const int* c, int G) {
  CellBox B;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    B.lo[a] = max(c[a] - 1, 0);
    B.hi[a] = min(c[a] + 1, G - 1);
  }
  return B;
}
__device__ __forceinline__ int box_cells(const CellBox& B) {
  return (B.hi[0] - B.lo[0] + 1) * (B.hi[1] - B.lo[1] + 1) * (B.hi[2] - B.lo[2] + 1);
}
__device__ __forceinline__ int box_side(const CellBox& B) {
  return max(B.hi[0] - B.lo[0], max(B.hi[1] - B.lo[1], B.hi[2] - B.lo[2])) + 1;
}

// Box of cells holding every point within squared radius r2 of a lane's point (the face
// distance of the box exceeds the radius); ok = false if none of side <= max_side was found.
__device__ __forceinline__ CellBox radius_box(const CellFrame& F, const CellOwn& o, float r2, int max_side, bool* ok) {
  const float r = sqrtf(r2);
  CellBox B;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float q = r / F.h[a];
    B.lo[a] = min(o.c[a], max(0, (int)floorf(fmaxf(o.f[a] - q, -1.f))));
    B.hi[a] = max(o.c[a], min(F.G - 1, (int)floorf(fminf(o.f[a] + q, (float)F.G))));
  }
  *ok = false;
  for (int it = 0; it < 3; ++it) {
    if (box_side(B) > max_side) return B;
    if (r2 < face_bound2(F, o.f, B)) { *ok = true; return B; }
    B = box_grow(B, F.G);
  }
  return B;
}

// The groups of a warp: the union of the lanes' boxes for all lanes of `lanes` when it is
// small, else the two halves of the warp (consecutive sorted points: a Morton jump splits
// them), recursively, down to single lanes.  body(mask, box) scans a group.
template <typename Body>
__device__ __forceinline__ void for_groups(const CellOwn& o, unsigned lanes, const CellBox& lb, Body&& body) {
  (void)o;
  if (!lanes) return;
  const int lane = threadIdx.x & 31;
  auto unite = [&](unsigned m) {
    const bool mine = (m >> lane) & 1u;
    CellBox W;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      W.lo[a] = (int)__reduce_min_sync(0xffffffffu, mine ? (unsigned)lb.lo[a] : 0x7fffffffu);
      W.hi[a] = (int)__reduce_max_sync(0xffffffffu, mine ? (unsigned)lb.hi[a] : 0u);
    }
    return W;
  };
  unsigned done = ~lanes;
  for (int len = 32; len >= 1 && ~done; len >>= 1) {
    for (int s0 = 0; s0 < 32; s0 += len) {
      const unsigned seg = len == 32 ? 0xffffffffu : ((1u << len) - 1u) << s0;
      const unsigned m = seg & ~done;
      if (!m) continue;
      const CellBox W = unite(m);
      if (box_cells(W) <= g_cell_maxblock || len == 1) {
        body(m, W);
        done |= m;
      }
    }
  }
}

// Coarse scan for ONE lane l (the "far" lanes: a large radius, or a top-2 search that did not
// settle within the near boxes), all lanes cooperating: the coarsest-needed level of the Morton
// hierarchy (a level-lev cell is a contiguous key range, hence a contiguous range of sorted
// points), cells of that level within squared radius r2 of the point (r2 = +inf: all), their
// points lane-parallel.  fn(t, valid) is called warp-synchronously for every sorted position t.
template <typename Fn>
__device__ __forceinline__ void far_scan(const CellFrame& F, int bits, const uint32_t* __restrict__ start,
                                         const float* fl, float r2, Fn&& fn) {
  const int lane = threadIdx.x & 31;
  const float r = sqrtf(r2);
  const bool all = !(r2 < 3e38f);
  int lev = bits;
  CellBox B;
  float fc[3], Hc[3];
  for (;;) {
    const float sc = (float)(1 << (bits - lev));
    const int Gl = 1 << lev;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      fc[a] = fl[a] / sc;
      Hc[a] = F.h[a] * sc;
      if (all) {
        B.lo[a] = 0;
        B.hi[a] = Gl - 1;
      } else {
        const float q = r / Hc[a];
        B.lo[a] = max(0, (int)floorf(fmaxf(fc[a] - q, -1.f)) - 1);
        B.hi[a] = min(Gl - 1, (int)floorf(fminf(fc[a] + q, (float)Gl)) + 1);
      }
    }
    if (box_cells(B) <= 512 || lev == 0) break;
    --lev;
  }
  const int ex = B.hi[0] - B.lo[0] + 1, ey = B.hi[1] - B.lo[1] + 1;
  const int V = box_cells(B), sh = 3 * (bits - lev);
  for (int base = 0; base < V; base += 32) {
    const int idx = base + lane;
    bool keep = false;
    uint32_t a0 = 0, a1 = 0;
    if (idx < V) {
      const int c[3] = {B.lo[0] + idx % ex, B.lo[1] + (idx / ex) % ey, B.lo[2] + idx / (ex * ey)};
      float d2 = 0.f;
#pragma unroll
      for (int a = 0; a < 3; ++a) {  // conservative distance from the point to the cell
        float g = fmaxf((float)c[a] - fc[a], fc[a] - (float)(c[a] + 1));
        g = fmaxf(g * Hc[a] - 4e-6f * F.ext[a], 0.f);
        d2 = fmaf(g, g, d2);
      }
      keep = all || d2 * (1.0f - 1e-5f) <= r2;
      if (keep) {
        const uint32_t key = morton3((uint32_t)c[0], (uint32_t)c[1], (uint32_t)c[2]);
        CELL_CHECK(((key + 1) << sh) <= (1u << (3 * bits)));
        a0 = __ldg(start + (key << sh));
        a1 = __ldg(start + ((key + 1) << sh));
        CELL_CHECK(a1 >= a0);
        keep = a1 > a0;
      }
    }
    unsigned km = __ballot_sync(0xffffffffu, keep);
    while (km) {
      const int l = __ffs(km) - 1;
      km &= km - 1;
      const uint32_t s0 = __shfl_sync(0xffffffffu, a0, l), s1 = __shfl_sync(0xffffffffu, a1, l);
      for (uint32_t t0 = s0; t0 < s1; t0 += 32) fn(t0 + lane, t0 + lane < s1);
    }
  }
}

// ---------------------------------------------------------------- Pass A (S1)

constexpr int kFarSide = 9;  // a near box grows to at most this many cells per axis

struct CellDir {
  const float* own;
  int own_np, own_n;
  const int* own_perm;
  const float* str;
  int str_np;
  const uint32_t* str_start;  // [B][cells1]
  float2* out;                // (min2, second2) at the output index
  unsigned long long* evals;
  int nblk;
  const float4* own4 = nullptr;  // relabelled clouds: the float4 copies in sorted order [B][n]
  const float4* str4 = nullptr;  // (the SoA copies own / str are then NULL)
  int str_n = 0;
};

__device__ __forceinline__ void top2_cells_warp(const CellDir& d, const float* bb, int bits, int cells1,
                                                int relabel, int b, int k0) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ __align__(16) float s_buf[kCellWarps][3][kCellBuf + 4];
  const CellStage st{s_buf[w][0], s_buf[w][1], s_buf[w][2], nullptr, nullptr};
  const CellFrame F = cell_frame(bb + 6 * b, bits);
  const float* own = d.own ? d.own + (size_t)b * 3 * d.own_np : nullptr;
  const float* str = d.str ? d.str + (size_t)b * 3 * d.str_np : nullptr;
  const float4* own4 = d.own4 ? d.own4 + (size_t)b * d.own_n : nullptr;
  const float4* str4 = d.str4 ? d.str4 + (size_t)b * d.str_n : nullptr;
  // a point of the streamed cloud at sorted position t (float4 copy or SoA)
  auto str_pt = [&](uint32_t t) {
    if (str4) return __ldg(str4 + t);
    return make_float4(__ldg(str + t), __ldg(str + d.str_np + t), __ldg(str + 2 * (size_t)d.str_np + t), 0.f);
  };
  const uint32_t* start = d.str_start + (size_t)b * cells1;
  const int k = k0 + lane;
  const CellOwn o = cell_own(own, d.own_np, d.own_n, k, F, own4);
  const f2_t nx = f2_pack(-o.x, -o.x), ny = f2_pack(-o.y, -o.y), nz = f2_pack(-o.z, -o.z);
  const float inf = __int_as_float(0x7f800000);
  float m = inf, s = inf, m2 = inf, s2 = inf;
  unsigned long long nev = 0, nfar = 0;  // evaluations: near (warp-uniform), far (per lane)
  unsigned far = 0u;
  cell_stat(5, 1);
  const unsigned vm = __ballot_sync(0xffffffffu, o.valid);
  for_groups(o, vm, cube_box(o.c, F.G), [&](unsigned mask, CellBox Bx) {
    cell_stat(4, 1);
    const bool act = (mask >> lane) & 1u;
    const int nact = __popc(mask);
    int filled = 0;
    auto eval = [&](int cnt) {
      const int c4 = stage_pad<false>(st, cnt);
      nev += (unsigned long long)cnt * nact;
      if (act) {
        const ulonglong2* px = reinterpret_cast<const ulonglong2*>(st.x);
        const ulonglong2* py = reinterpret_cast<const ulonglong2*>(st.y);
        const ulonglong2* pz = reinterpret_cast<const ulonglong2*>(st.z);
#pragma unroll 4
        for (int q = 0; q < c4 / 4; ++q) {
          const ulonglong2 qx = px[q], qy = py[q], qz = pz[q];
          const f2_t d01 = f2_dist2(qx.x, qy.x, qz.x, nx, ny, nz);
          const f2_t d23 = f2_dist2(qx.y, qy.y, qz.y, nx, ny, nz);
          float v0, v1, v2, v3;
          f2_unpack(d01, v0, v1);
          f2_unpack(d23, v2, v3);
          top2_pair(m, s, v0, v1);
          top2_pair(m2, s2, v2, v3);
        }
      }
      __syncwarp();  // the buffer is refilled next
    };
    scan_box<false>(Bx, nullptr, start, str, d.str_np, nullptr, nullptr, relabel, st, filled, eval, str4);
    if (filled) { __syncwarp(); eval(filled); filled = 0; }
    for (;;) {
      float mm = m, ss = s;
      top2_merge(mm, ss, m2, s2);
      const bool need = act && !(ss <= face_bound2(F, o.f, Bx));
      const unsigned nm = __ballot_sync(0xffffffffu, need);
      if (!nm || box_covers_grid(Bx, F.G)) break;
      if (box_side(Bx) >= kFarSide) {  // the rest of this group: the coarse scan below
        far |= nm;
        break;
      }
      cell_stat(3, 1);
      const CellBox Nb = box_grow(Bx, F.G);
      scan_box<false>(Nb, &Bx, start, str, d.str_np, nullptr, nullptr, relabel, st, filled, eval, str4);
      if (filled) { __syncwarp(); eval(filled); filled = 0; }
      Bx = Nb;
    }
  });
  top2_merge(m, s, m2, s2);
  // lanes that did not settle: redo from scratch over every point within their current second
  // minimum (an upper bound of the true one), all lanes cooperating, one such lane at a time
  cell_stat(2, __popc(far));
  while (far) {
    const int l = __ffs(far) - 1;
    far &= far - 1;
    const float fl[3] = {__shfl_sync(0xffffffffu, o.f[0], l), __shfl_sync(0xffffffffu, o.f[1], l),
                         __shfl_sync(0xffffffffu, o.f[2], l)};
    const float r2 = __shfl_sync(0xffffffffu, s, l);
    const float xl = __shfl_sync(0xffffffffu, -o.x, l), yl = __shfl_sync(0xffffffffu, -o.y, l),
                zl = __shfl_sync(0xffffffffu, -o.z, l);
    float fm = inf, fs = inf;
    far_scan(F, bits, start, fl, r2, [&](uint32_t t, bool v) {
      if (!v) return;
      const float4 q = str_pt(t);
      const float dx = __fadd_rn(q.x, xl), dy = __fadd_rn(q.y, yl), dz = __fadd_rn(q.z, zl);
      float d2 = __fmul_rn(dx, dx);
      d2 = __fmaf_rn(dy, dy, d2);
      d2 = __fmaf_rn(dz, dz, d2);
      fs = fminf(fs, fmaxf(fm, d2));
      fm = fminf(fm, d2);
      ++nfar;
    });
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, fm, o2), os = __shfl_xor_sync(0xffffffffu, fs, o2);
      top2_merge(fm, fs, om, os);
    }
    if (lane == l) { m = fm; s = fs; }
  }
  CELL_CHECK(!o.valid || relabel || (d.own_perm[(size_t)b * d.own_np + k] >= 0 && d.own_perm[(size_t)b * d.own_np + k] < d.own_n));
  if (o.valid) d.out[(size_t)b * d.own_n + (relabel ? k : d.own_perm[(size_t)b * d.own_np + k])] = make_float2(m, s);
  nev += __reduce_add_sync(0xffffffffu, (unsigned)min(nfar, 0xffffffffull));
  if (d.evals && lane == 0 && nev) atomicAdd(d.evals, nev);
}

// Both directions in one launch: grid (blocks, B, 2).
__global__ void __launch_bounds__(32 * kCellWarps, 8) k_top2_cells(const CellDir d0, const CellDir d1, const float* bb,
                                                                int bits, int cells1, int relabel) {
  const CellDir& d = blockIdx.z ? d1 : d0;
  if ((int)blockIdx.x >= d.nblk) return;
  const int k0 = ((int)blockIdx.x * kCellWarps + (int)(threadIdx.x >> 5)) * 32;
  if (k0 >= d.own_n) return;  // warp-uniform
  top2_cells_warp(d, bb, bits, cells1, relabel, blockIdx.y, k0);
}

// ---------------------------------------------------------------- Pass B (S3)

constexpr int kNearSide = 5;  // emit radius boxes of more cells per axis go to the coarse scan

struct CellEmitDir {
  const float* own;
  int own_np, own_n;
  const int* own_perm;
  const LineA* ownA;          // own line constants at the output index
  const float* str;
  int str_np;
  const uint32_t* str_start;
  const int* str_perm;
  const LineA* strA;          // the other cloud's line constants at the output index
  int nblk;
  const float4* own4 = nullptr;  // relabelled clouds: the float4 copies in sorted order [B][n]
  const float4* str4 = nullptr;
  int str_n = 0;
};

__device__ __forceinline__ void emit_cells_warp(const CellEmitDir& d, int dir, const float* bb, int bits,
                                                int cells1, int relabel, int b, int k0, int N, int M, uint32_t cap,
                                                uint2* __restrict__ ebuf, unsigned* __restrict__ cursor,
                                                unsigned* __restrict__ aux_cnt, unsigned* __restrict__ row_cnt,
                                                unsigned* __restrict__ col_cnt, unsigned long long* evals) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ __align__(16) float s_buf[kCellWarps][4][kCellBuf + 4];
  __shared__ __align__(16) int s_id[kCellWarps][kCellBuf + 4];
  __shared__ uint2 queue_all[kCellWarps][kLaneQ][32];
  // r2: row pass -> R'^2 of the gt point (its column flag); column pass -> E^2 of the pred
  // point (an entry it already emits from its row is skipped)
  const CellStage st{s_buf[w][0], s_buf[w][1], s_buf[w][2], s_buf[w][3], s_id[w]};
  uint2* qp = &queue_all[w][0][lane];
  int qn = 0;
  const CellFrame F = cell_frame(bb + 6 * b, bits);
  const float* own = d.own ? d.own + (size_t)b * 3 * d.own_np : nullptr;
  const float* str = d.str ? d.str + (size_t)b * 3 * d.str_np : nullptr;
  const float4* own4 = d.own4 ? d.own4 + (size_t)b * d.own_n : nullptr;
  const float4* str4 = d.str4 ? d.str4 + (size_t)b * d.str_n : nullptr;
  // a point of the streamed cloud at sorted position t (float4 copy or SoA)
  auto str_pt = [&](uint32_t t) {
    if (str4) return __ldg(str4 + t);
    return make_float4(__ldg(str + t), __ldg(str + d.str_np + t), __ldg(str + 2 * (size_t)d.str_np + t), 0.f);
  };
  const uint32_t* start = d.str_start + (size_t)b * cells1;
  const int* sperm = d.str_perm + (size_t)b * d.str_np;
  const LineA* strA = d.strA + (size_t)b * (dir ? N : M);
  const float* r2src = reinterpret_cast<const float*>(strA) + (dir ? 3 : 2);
  const int k = k0 + lane;
  const CellOwn o = cell_own(own, d.own_np, d.own_n, k, F, own4);
  const int oi = o.valid ? (relabel ? k : d.own_perm[(size_t)b * d.own_np + k]) : -1;
  float oR2 = -1.f, oE2 = -1.f;
  if (oi >= 0) {
    const LineA a = d.ownA[(size_t)b * (dir ? M : N) + oi];
    oR2 = a.R2;
    oE2 = a.E2;
  }
  const f2_t nx = f2_pack(-o.x, -o.x), ny = f2_pack(-o.y, -o.y), nz = f2_pack(-o.z, -o.z);
  float xr, yr, zr;
  {
    float t;
    f2_unpack(nx, xr, t);
    f2_unpack(ny, yr, t);
    f2_unpack(nz, zr, t);
  }
  unsigned long long nev = 0, nfar = 0;  // evaluations: near (warp-uniform), far (per lane)
  cell_stat(13, 1);
  // near lanes: a box from the emit radius; far lanes (large or infinite radius): coarse scan
  bool ok = false;
  const bool active = o.valid && oE2 >= 0.f;
  CellBox lb = cube_box(o.c, F.G);
  if (active && oE2 < 3e38f) lb = radius_box(F, o, oE2, kNearSide, &ok);
  const unsigned near = __ballot_sync(0xffffffffu, active && ok);
  unsigned far = __ballot_sync(0xffffffffu, active && !ok);
  auto queue_hit = [&](int j, float d2, float r2o) {  // (r2o: the other point's R'^2, row pass)
    CELL_CHECK(qn < kLaneQ && j >= 0 && j < (dir ? N : M) && oi >= 0 && oi < (dir ? M : N));
    if (dir == 0) {
      const uint32_t fl = (d2 <= oR2 ? kFlagRow : 0u) | (d2 <= r2o ? kFlagCol : 0u);
      qp[qn * 32] = make_uint2((uint32_t)oi, (uint32_t)j | fl);
    } else {
      const uint32_t fl = d2 <= oR2 ? kFlagCol : 0u;
      qp[qn * 32] = make_uint2((uint32_t)j, (uint32_t)oi | fl);
    }
    ++qn;
  };
  auto flush_if_full = [&]() {
    if (__any_sync(0xffffffffu, qn == kLaneQ)) {
      __syncwarp();
      lane_flush(b, qp, qn, cap, ebuf, cursor, aux_cnt, row_cnt, N, col_cnt, M);
      qn = 0;
      __syncwarp();
    }
  };
  for_groups(o, near, lb, [&](unsigned mask, CellBox Bx) {
    cell_stat(12, 1);
    const bool act = (mask >> lane) & 1u;
    const int nact = __popc(mask);
    int filled = 0;
    auto eval = [&](int cnt) {
      const int c4 = stage_pad<true>(st, cnt);
      nev += (unsigned long long)cnt * nact;
      const ulonglong2* px = reinterpret_cast<const ulonglong2*>(st.x);
      const ulonglong2* py = reinterpret_cast<const ulonglong2*>(st.y);
      const ulonglong2* pz = reinterpret_cast<const ulonglong2*>(st.z);
      // blocks of 128 staged points: a candidate bit per group of 4 (min of the 4 d2 within
      // the own emit radius -- necessary for every hit of both passes), then the candidate
      // groups re-evaluated exactly (same d2 bits) and their hits queued
      for (int q0 = 0; q0 < c4; q0 += 128) {
        uint32_t gm = 0u;
        const int qe = min(c4, q0 + 128);
        if (act) {
#pragma unroll 2
          for (int q = q0 / 4; q < qe / 4; ++q) {
            const ulonglong2 qx = px[q], qy = py[q], qz = pz[q];
            const f2_t d01 = f2_dist2(qx.x, qy.x, qz.x, nx, ny, nz);
            const f2_t d23 = f2_dist2(qx.y, qy.y, qz.y, nx, ny, nz);
            float v0, v1, v2, v3;
            f2_unpack(d01, v0, v1);
            f2_unpack(d23, v2, v3);
            const float mn = fminf(fmin3(v0, v1, v2), v3);
            gm |= (mn <= oE2 ? 1u : 0u) << (q - q0 / 4);
          }
        }
        if (!__any_sync(0xffffffffu, gm)) continue;
        // room for 4 hits per candidate group in every lane's queue (else flush first; a lane
        // with more candidates than that checks before every group)
        if (__any_sync(0xffffffffu, qn + 4 * __popc(gm) > kLaneQ)) {
          __syncwarp();
          lane_flush(b, qp, qn, cap, ebuf, cursor, aux_cnt, row_cnt, N, col_cnt, M);
          qn = 0;
          __syncwarp();
        }
        const bool checked = __any_sync(0xffffffffu, 4 * __popc(gm) > kLaneQ);
        while (__any_sync(0xffffffffu, gm)) {
          if (checked && __any_sync(0xffffffffu, qn + 4 > kLaneQ)) {
            __syncwarp();
            lane_flush(b, qp, qn, cap, ebuf, cursor, aux_cnt, row_cnt, N, col_cnt, M);
            qn = 0;
            __syncwarp();
          }
          if (gm) {
            const int qb = q0 + 4 * (__ffs(gm) - 1);
            gm &= gm - 1;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int qq = qb + u;
              const int j = st.id[qq];
              const float dx = __fadd_rn(st.x[qq], xr), dy = __fadd_rn(st.y[qq], yr), dz = __fadd_rn(st.z[qq], zr);
              float d2 = __fmul_rn(dx, dx);
              d2 = __fmaf_rn(dy, dy, d2);
              d2 = __fmaf_rn(dz, dz, d2);
              const float r2o = st.r2[qq];
              if (j >= 0 && d2 <= oE2 && (dir == 0 || !(d2 <= r2o))) queue_hit(j, d2, r2o);
            }
          }
        }
      }
      __syncwarp();  // the buffer is refilled next
    };
    scan_box<true>(Bx, nullptr, start, str, d.str_np, r2src, sperm, relabel, st, filled, eval, str4);
    if (filled) { __syncwarp(); eval(filled); filled = 0; }
  });
  // far lanes, one at a time, all lanes cooperating (the hits go to the queue of the lane that
  // evaluated them)
  cell_stat(10, __popc(far));
  while (far) {
    const int l = __ffs(far) - 1;
    far &= far - 1;
    const float fl[3] = {__shfl_sync(0xffffffffu, o.f[0], l), __shfl_sync(0xffffffffu, o.f[1], l),
                         __shfl_sync(0xffffffffu, o.f[2], l)};
    const float E2l = __shfl_sync(0xffffffffu, oE2, l), R2l = __shfl_sync(0xffffffffu, oR2, l);
    const int oil = __shfl_sync(0xffffffffu, oi, l);
    const float xl = __shfl_sync(0xffffffffu, xr, l), yl = __shfl_sync(0xffffffffu, yr, l),
                zl = __shfl_sync(0xffffffffu, zr, l);
    far_scan(F, bits, start, fl, E2l, [&](uint32_t t, bool v) {
      bool hit = false;
      float d2 = 0.f, r2o = 0.f;
      int j = -1;
      if (v) {
        const float4 q = str_pt(t);
        const float dx = __fadd_rn(q.x, xl), dy = __fadd_rn(q.y, yl), dz = __fadd_rn(q.z, zl);
        d2 = __fmul_rn(dx, dx);
        d2 = __fmaf_rn(dy, dy, d2);
        d2 = __fmaf_rn(dz, dz, d2);
        ++nfar;
        if (d2 <= E2l) {
          j = relabel ? (int)t : __ldg(sperm + t);
          r2o = __ldg(r2src + 4 * (size_t)j);
          hit = dir == 0 || !(d2 <= r2o);
        }
      }
      flush_if_full();
      CELL_CHECK(!hit || (qn < kLaneQ && j >= 0 && j < (dir ? N : M)));
      if (hit) {
        if (dir == 0) {
          const uint32_t fl2 = (d2 <= R2l ? kFlagRow : 0u) | (d2 <= r2o ? kFlagCol : 0u);
          qp[qn * 32] = make_uint2((uint32_t)oil, (uint32_t)j | fl2);
        } else {
          const uint32_t fl2 = d2 <= R2l ? kFlagCol : 0u;
          qp[qn * 32] = make_uint2((uint32_t)j, (uint32_t)oil | fl2);
        }
        ++qn;
      }
    });
  }
  __syncwarp();
  lane_flush(b, qp, qn, cap, ebuf, cursor, aux_cnt, row_cnt, N, col_cnt, M);
  nev += __reduce_add_sync(0xffffffffu, (unsigned)min(nfar, 0xffffffffull));
  if (evals && lane == 0 && nev) atomicAdd(evals, nev);
}

// Row pass (z = 0, own = pred) and column pass (z = 1, own = gt) in one launch.
__global__ void __launch_bounds__(32 * kCellWarps, 6)
k_emit_cells(const CellEmitDir d0, const CellEmitDir d1, const float* bb, int bits, int cells1, int relabel, int N,
             int M, uint32_t cap, uint2* __restrict__ ebuf, unsigned* __restrict__ cursor,
             unsigned* __restrict__ aux_cnt, unsigned* __restrict__ row_cnt, unsigned* __restrict__ col_cnt,
             unsigned long long* evals) {
  const int dir = blockIdx.z;
  const CellEmitDir& d = dir ? d1 : d0;
  if ((int)blockIdx.x >= d.nblk) return;
  const int k0 = ((int)blockIdx.x * kCellWarps + (int)(threadIdx.x >> 5)) * 32;
  if (k0 >= d.own_n) return;  // warp-uniform
  emit_cells_warp(d, dir, bb, bits, cells1, relabel, blockIdx.y, k0, N, M, cap, ebuf, cursor, aux_cnt, row_cnt,
                  col_cnt, evals);
}

}  // namespace apml
