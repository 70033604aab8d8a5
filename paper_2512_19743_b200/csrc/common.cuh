// common.cuh -- shared device helpers of the sm_100a APML path.
//
// The one arithmetic fact every kernel must agree on bit-for-bit is the fp32 squared
// distance d2(i, j): line statistics (Pass A), the emit test (Pass B) and the tie search
// for argmin / second argmin (normalisation) all compare d2 values for equality, so they
// all evaluate exactly   dx = y - x; d = dx*dx; d = fma(dy, dy, d); d = fma(dz, dz, d)
// with round-to-nearest and no contraction other than the two explicit FMAs.  The packed
// f32x2 forms below (FADD2 / FMUL2 / FFMA2 on sm_100a) are element-wise identical to it.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace apml {

constexpr float kPadPred = 1.0e30f;   // sentinel coordinate of padded pred points
constexpr float kPadGt = -1.0e30f;    // ... of padded gt points (pred-pad vs gt-pad -> +inf)
constexpr uint32_t kFlagRow = 1u << 30;   // entry kept by the row softmax  (Omega_row)
constexpr uint32_t kFlagCol = 1u << 31;   // entry kept by the column softmax (Omega_col)
constexpr uint32_t kIdxMask = (1u << 30) - 1u;

// Line flags stored in LineB.w (as bits of a float via __int_as_float).
constexpr int kLineK1 = 1;       // K == 1 line: P = 1 on its single entry
constexpr int kLineClamped = 2;  // gap clamp active: no gradient through g
constexpr int kLineUniform = 4;  // uniform fallback: T = 0, all K entries, P = 1/K

// Per-line constants (S2).  LineA = {m2, s2, R2, E2}: squared min, squared second min,
// squared kept radius (s >= tau  <=>  d2 <= R2), squared emit radius (max(R2, s2): the
// second argmin is always emitted so the T-gradient can reach it, reading R14).
// LineB = {m, T, g, flags}.
struct __align__(16) LineA { float m2, s2, R2, E2; };
struct __align__(16) LineB { float m, T, g; int flags; };

// Backward per-line scalars: S = sum_kept P*Pbar, ca = coefficient added to cbar at the
// argmin entry, cb = ... at the second-argmin entry; T copied for the final sweep.
struct __align__(16) LineBack { float S, ca, cb, T; };

__device__ __forceinline__ float dist2(float xi0, float xi1, float xi2, float yj0, float yj1,
                                       float yj2) {
  float dx = __fsub_rn(yj0, xi0);
  float dy = __fsub_rn(yj1, xi1);
  float dz = __fsub_rn(yj2, xi2);
  float d = __fmul_rn(dx, dx);
  d = __fmaf_rn(dy, dy, d);
  d = __fmaf_rn(dz, dz, d);
  return d;
}

// ---- packed fp32x2 (sm_100a FADD2 / FMUL2 / FFMA2) -------------------------------------
typedef unsigned long long f2_t;

__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(f2_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
  f2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// d2 of one owned point (negated coords nx = -x packed twice) against two streamed points
// (qx = (y0x, y1x) ...): identical rounding to dist2 since y + (-x) == y - x exactly.
__device__ __forceinline__ f2_t f2_dist2(f2_t qx, f2_t qy, f2_t qz, f2_t nx, f2_t ny, f2_t nz) {
  f2_t dx = f2_add(qx, nx);
  f2_t dy = f2_add(qy, ny);
  f2_t dz = f2_add(qz, nz);
  f2_t d = f2_mul(dx, dx);
  d = f2_fma(dy, dy, d);
  d = f2_fma(dz, dz, d);
  return d;
}

// 3-input min (sm_100a FMNMX3)
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// Running (min, second min) of a multiset, updated with a pair of values (v0, v1):
//   lo = min(v0, v1), hi = max(v0, v1); s' = min(s, hi, max(m, lo)); m' = min(m, lo).
// Case lo < m: s' = min(m, hi) (s >= m); case lo >= m: s' = min(s, lo).  5 ALU ops / 2 values.
__device__ __forceinline__ void top2_pair(float& m, float& s, float v0, float v1) {
  float lo = fminf(v0, v1), hi = fmaxf(v0, v1);
  s = fmin3(s, hi, fmaxf(m, lo));
  m = fminf(m, lo);
}
// Merge two (min, second) summaries of disjoint multisets.
__device__ __forceinline__ void top2_merge(float& m, float& s, float m1, float s1) {
  float ns = fminf(fmaxf(m, m1), fminf(s, s1));
  m = fminf(m, m1);
  s = ns;
}

// A pair whose emission overflowed its capacity is skipped by every downstream kernel.
__device__ __forceinline__ bool pair_overflow(const unsigned* cursor, int b, uint32_t cap) {
  return cursor[b] > cap;
}

__device__ __forceinline__ int warp_lane() { return threadIdx.x & 31; }

// Programmatic dependent launch (PDL) along the forward / backward chain: every kernel lets
// its dependent be scheduled as soon as all of its own CTAs are running (launch_dependents),
// and a dependent runs its prologue (shared-memory carve-out, mbarrier set-up) before it waits
// for the whole predecessor grid and its memory (wait).  Both are no-ops for a kernel not
// launched with the programmatic-serialization attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

}  // namespace apml
