// Microbenchmark: the FP32 lane-op ceiling the distance sweeps are measured against
// (DESIGN.md "Roofline").  Measures, on every SM at once, the sustained rate of
//   FFMA   scalar fma.rn.f32            (1 lane-op per lane per instruction, FMA counted once)
//   FFMA2  packed fma.rn.f32x2          (2 lane-ops per lane per instruction)
//   FMNMX  min.f32 (ALU pipe)           (the top-2 bookkeeping of Pass A)
//   MIX    the Pass A inner-loop mix: 3 packed FP32 + 5 FMNMX per 2 (i, j) values
// with 8 independent chains per thread, 148 x 4 CTAs of 256 threads, timed with CUDA events.
// Prints one JSON line (copied to profiles/fp32_peak.json).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_peak fp32_peak.cu && ./fp32_peak
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk(float lo, float hi) {
  f2_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ float2 upk(f2_t v) {
  float2 r; asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v)); return r; }
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
  f2_t r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
  f2_t r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ float fma1(float a, float b, float c) {
  float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
__device__ __forceinline__ float mn(float a, float b) {
  float r; asm volatile("min.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float mx(float a, float b) {
  float r; asm volatile("max.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float mn3(float a, float b, float c) {
  float r; asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }

constexpr int kChains = 8;

__global__ void k_ffma(int iters, float* out) {
  float a[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) a[k] = threadIdx.x * 1e-3f + k;
  const float b = 0.999f, c = 1e-4f;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = fma1(a[k], b, c);
  float s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += a[k];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma2(int iters, float* out) {
  f2_t a[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) a[k] = pk(threadIdx.x * 1e-3f + k, k + 0.5f);
  const f2_t b = pk(0.999f, 0.998f), c = pk(1e-4f, 2e-4f);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = fma2(a[k], b, c);
  float s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) { const float2 v = upk(a[k]); s += v.x + v.y; }
  if (s == 12345.f) out[0] = s;
}

__global__ void k_fmnmx(int iters, float* out) {
  float a[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) a[k] = threadIdx.x * 1e-3f + k;
  const float b = 0.5f;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = (it & 1) ? mn(a[k], b + k) : mx(a[k], b - k);
  float s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += a[k];
  if (s == 12345.f) out[0] = s;
}

// Pass A's inner loop for 2 values per owned point: d2 = (y-x)^2 summed (3 packed ops: add2,
// mul2, fma2 x 2 = 4 packed?) -- here exactly the k_line_top2 sequence: dx = y - x (add2 x 3),
// d = dx*dx (mul2), d = fma(dy,dy,d), d = fma(dz,dz,d) (fma2 x 2) = 6 packed instructions per
// 2 values (12 lane-ops = 6 per value), then the running (min, second) of a multiset for the
// 2 values: lo/hi + 3 FMNMX.
__global__ void k_mix(int iters, float* out) {
  f2_t qx = pk(threadIdx.x * 1e-3f, 0.1f), qy = pk(0.2f, 0.3f), qz = pk(0.4f, 0.5f);
  float m[4], s2[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { m[k] = 1e30f; s2[k] = 1e30f; }
  f2_t nx = pk(-0.1f, -0.2f), ny = pk(-0.3f, -0.4f), nz = pk(-0.5f, -0.6f);
  const f2_t step = pk(1e-6f, 2e-6f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const f2_t dx = add2(qx, nx), dy = add2(qy, ny), dz = add2(qz, nz);
      f2_t d = mul2(dx, dx);
      d = fma2(dy, dy, d);
      d = fma2(dz, dz, d);
      const float2 v = upk(d);
      const float lo = mn(v.x, v.y), hi = mx(v.x, v.y);
      s2[k] = mn3(s2[k], hi, mx(m[k], lo));
      m[k] = mn(m[k], lo);
      nx = add2(nx, step);
    }
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += m[k] + s2[k];
  if (s == 12345.f) out[0] = s;
}

template <typename K>
double run(K k, int iters, int blocks, int threads, float* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<blocks, threads>>>(iters / 10, out);  // warm-up
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 16);
  const int threads = 256, blocks = sms * 8, iters = 1 << 16;
  const double lanes = (double)blocks * threads;
  const double t1 = run(k_ffma, iters, blocks, threads, out);
  const double t2 = run(k_ffma2, iters, blocks, threads, out);
  const double t3 = run(k_fmnmx, iters, blocks, threads, out);
  const double t4 = run(k_mix, iters, blocks, threads, out);
  const double ffma = lanes * iters * kChains / (t1 * 1e-3) / 1e12;       // lane-op/s (FMA = 1)
  const double ffma2 = lanes * iters * kChains * 2 / (t2 * 1e-3) / 1e12;
  const double fmnmx = lanes * iters * kChains / (t3 * 1e-3) / 1e12;      // ops/s
  const double mix_vals = lanes * (double)iters * 4 * 2 / (t4 * 1e-3);    // (i, j) values/s
  const double nominal = sms * 128.0 * clk_khz * 1e3 / 1e12;
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"nominal_lane_tops\": %.2f, \"ffma_lane_tops\": %.2f, "
         "\"ffma2_lane_tops\": %.2f, \"fmnmx_tops\": %.2f, \"passA_mix_values_per_s\": %.4g, "
         "\"passA_mix_lane_tops\": %.2f, \"ms\": [%.3f, %.3f, %.3f, %.3f]}\n",
         sms, clk_khz / 1e3, nominal, ffma, ffma2, fmnmx, mix_vals, mix_vals * 6 / 1e12, t1, t2, t3, t4);
  return 0;
}
