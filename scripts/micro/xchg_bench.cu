// Microbenchmark: cost of one replica-exchange round of an n-float vector across a cluster
// of CL CTAs (512 threads), the pattern of the Sinkhorn half-steps in k_mega.cuh.
//   mode 0: st.async per element to every replica + mbarrier complete_tx (current design)
//   mode 1: local stores + one bulk DSMEM copy per peer (cp.async.bulk shared::cluster)
//   mode 2: st.shared::cluster per element to every replica + barrier.cluster arrive/wait
//   mode 3: local stores + barrier.cluster + pull the peers' slices with ld.shared::cluster
//   mode 4: local stores + barrier.cluster only (lower bound: no data movement)
//   mode 5: mode 0 + a global store per element per round (the Sinkhorn history)
//   mode 6: mode 0 + a 6-entry gather dot product per element (idx/val in shared memory)
//   mode 7: mode 0 with v4 pushes: each group of 4 lanes gathers its 4 consecutive values by
//           shuffles and lane q of the group sends the 16-byte vector to rank q (one st.async
//           per lane instead of CL)
//   mode 8: mode 7 + the 6-entry gather dot product of mode 6
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xb xchg_bench.cu && ./xb
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) {
  uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void mwait(uint32_t mb, uint32_t ph) {
  uint32_t done = 0;
  while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(mb), "r"(ph) : "memory");
}
__device__ __forceinline__ void arm(uint32_t mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(bytes) : "memory"); }

template <int MODE>
__global__ void __launch_bounds__(512, 1) xb(int rounds, int n, unsigned long long* out, float* hist) {
  extern __shared__ __align__(16) float sm[];
  __shared__ __align__(8) unsigned long long mbar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int CL = cl.num_blocks(), me = cl.block_rank();
  const int per = n / CL, lo = me * per, hi = lo + per;
  float* rep[2] = {sm, sm + n};
  for (int k = threadIdx.x; k < 2 * n; k += blockDim.x) sm[k] = 1.f;
  if (MODE == 6 || MODE == 8) {
    unsigned short* ix = reinterpret_cast<unsigned short*>(sm + 2 * n);
    float* vv = sm + 2 * n + 3 * n;
    for (int k = threadIdx.x; k < 6 * per; k += blockDim.x) { ix[k] = (unsigned short)((k * 2654435761u) % n); vv[k] = 0.1f; }
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t e = (MODE == 0 || MODE >= 5) ? 4u * n : 4u * (n - per);  // modes 7/8: CL == 4
    arm(sa(&mbar[0]), e); arm(sa(&mbar[1]), e);
  }
  cl.sync();
  uint32_t ph[2] = {0, 0};
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int it = 0; it < rounds; ++it) {
    const int w = it & 1;  // vector written this round; the other is read
    float* dst = rep[w];
    const float* src = rep[w ^ 1];
    const uint32_t mb = sa(&mbar[w]);
    for (int k = lo + threadIdx.x; k < hi; k += blockDim.x) {
      float v = src[(k * 7) % n] * 0.5f + 1.f;
      if (MODE == 6) {
        const unsigned short* ix = reinterpret_cast<const unsigned short*>(sm + 2 * n);
        const float* vv = sm + 2 * n + 3 * n;
        float s = 0.f;
#pragma unroll
        for (int u = 0; u < 6; ++u) s = fmaf(src[ix[6 * (k - lo) + u]], vv[6 * (k - lo) + u], s);
        v = __fdividef(v, fmaf(v, s, 1e-8f));
      }
      if (MODE == 8) {
        const unsigned short* ix = reinterpret_cast<const unsigned short*>(sm + 2 * n);
        const float* vv = sm + 2 * n + 3 * n;
        float s = 0.f;
#pragma unroll
        for (int u = 0; u < 6; ++u) s = fmaf(src[ix[6 * (k - lo) + u]], vv[6 * (k - lo) + u], s);
        v = __fdividef(v, fmaf(v, s, 1e-8f));
      }
      if (MODE == 7 || MODE == 8) {  // (k - lo) % 4 == lane % 4: per multiple of 4, CL == 4
        const int lane = threadIdx.x & 31, q = lane & 3, g0 = lane & ~3;
        float4 v4;
        v4.x = __shfl_sync(0xffffffffu, v, g0);
        v4.y = __shfl_sync(0xffffffffu, v, g0 + 1);
        v4.z = __shfl_sync(0xffffffffu, v, g0 + 2);
        v4.w = __shfl_sync(0xffffffffu, v, g0 + 3);
        if (q < CL) {
          const uint32_t a = sa(dst + (k & ~3));
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
                       :: "r"(mapa(a, q)), "r"(__float_as_uint(v4.x)), "r"(__float_as_uint(v4.y)),
                          "r"(__float_as_uint(v4.z)), "r"(__float_as_uint(v4.w)), "r"(mapa(mb, q)) : "memory");
        }
      }
      if (MODE == 5) hist[(size_t)it * n + k] = v;
      if (MODE == 0 || MODE == 5 || MODE == 6) {
        const uint32_t a = sa(dst + k);
        for (int r = 0; r < CL; ++r)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
                       :: "r"(mapa(a, r)), "r"(__float_as_uint(v)), "r"(mapa(mb, r)) : "memory");
      } else if (MODE == 2) {
        const uint32_t a = sa(dst + k);
        for (int r = 0; r < CL; ++r)
          asm volatile("st.shared::cluster.f32 [%0], %1;" :: "r"(mapa(a, r)), "f"(v) : "memory");
      } else {
        dst[k] = v;
      }
    }
    if (MODE == 0 || MODE == 1 || MODE >= 5) {
      if (MODE == 1) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0)
          for (int r = 0; r < CL; ++r) if (r != me)
            asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         :: "r"(mapa(sa(dst + lo), r)), "r"(sa(dst + lo)), "r"(4u * per), "r"(mapa(mb, r)) : "memory");
      }
      mwait(mb, ph[w]);
      ph[w] ^= 1u;
      if (threadIdx.x == 0) arm(mb, (MODE == 0 || MODE >= 5) ? 4u * n : 4u * (n - per));
      __syncthreads();
    } else {
      cl_arrive(); cl_wait();
      if (MODE == 3) {
        for (int k = threadIdx.x; k < n; k += blockDim.x) {
          const int r = k / per;
          if (r == me) continue;
          float v;
          asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(mapa(sa(dst + k), r)) : "memory");
          dst[k] = v;
        }
        cl_arrive(); cl_wait();  // nobody overwrites a slice a peer is still pulling
      }
    }
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  cl.sync();
}

template <int MODE>
void run(int CL, int n, int B) {
  unsigned long long* d; cudaMalloc(&d, 8 * B * CL);
  float* hist; cudaMalloc(&hist, sizeof(float) * 200 * (size_t)n * 1);
  auto k = xb<MODE>;
  const int smem = 8 * n + ((MODE == 6 || MODE == 8) ? 4 * n * 6 : 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(B * CL); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; cfg.attrs = at; cfg.numAttrs = 1;
  const int rounds = 200;
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, k, rounds, n, d, hist);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[1024]; cudaMemcpy(h, d, 8 * B * CL, cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < B * CL; ++i) s += h[i];
  printf("mode %d CL %d n %5d B %3d : %7.3f us/round  (%s)\n", MODE, CL, n, B, s / (B * CL) / rounds / 1e3, cudaGetErrorString(e));
  cudaFree(d); cudaFree(hist);
}

int main() {
  for (int CL : {4}) for (int n : {2048}) {
    const int B = 128 / CL;
    run<0>(CL, n, B); run<1>(CL, n, B); run<4>(CL, n, B); run<5>(CL, n, B); run<6>(CL, n, B);
    run<7>(CL, n, B); run<8>(CL, n, B);
  }
  return 0;
}
