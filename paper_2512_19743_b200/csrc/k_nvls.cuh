// k_nvls.cuh -- in-kernel cross-GPU reduction over NVSwitch multicast memory (NVLS), for the
// per-iteration Sinkhorn column sums of the row-sharded mode (north_star: "pred
// rows shard and per-iteration column sums are allreduced over NVLink"; Eq. (3)).
//
// A team (apml_nvls, host side in nvls_host.cuh) is one multicast object bound to a buffer on
// every rank's GPU.  Layout of the buffer (the same on every rank):
//   [0, 256)           flag word (uint32) + padding
//   [256, ...)         two partial-sum buffers of B x M floats (alternating by use, so that
//                      one barrier per reduction suffices: a rank can only start writing use
//                      u + 2 after every rank has passed the barrier of use u + 1, i.e. after
//                      every rank finished reading use u)
// Per reduction: the producer kernel writes this rank's partial column sums into its own copy
// (plain stores through the unicast mapping), every CTA then bumps the flag of EVERY rank with
// one multicast red.add (release, system scope); the consumer kernel waits until its local flag
// has counted all CTAs of all ranks (acquire, system scope) and reads each reduced value with
// one multimem.ld_reduce through the multicast mapping: the switch returns the sum over ranks.
#pragma once
#include "common.cuh"

namespace apml {

constexpr size_t kNvlsHdr = 256;  // bytes before the partial-sum buffers

// kMc = false: a one-device team in plain device memory (a driver that rejects a multicast
// object of one device, e.g. a one-GPU box): the same kernels and barrier bookkeeping with
// ordinary atomics / loads in place of the multimem instructions (the sum over one rank).

// One thread per CTA, after a CTA barrier that orders the CTA's partial-sum stores: make them
// visible system-wide, then add 1 to the flag of every rank of the team.
template <bool kMc>
__device__ __forceinline__ void nvls_signal(unsigned* flag_mc) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  if (kMc) asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(flag_mc), "r"(1u) : "memory");
  else asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(flag_mc), "r"(1u) : "memory");
}

// One thread per CTA: wait until this rank's flag reaches `target` (modular counter).
__device__ __forceinline__ void nvls_wait(const unsigned* flag_uc, unsigned target) {
  unsigned v;
  do {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag_uc) : "memory");
  } while ((int)(v - target) < 0);
}

// Sum over the ranks of the float at this multicast address.
template <bool kMc>
__device__ __forceinline__ float nvls_ld_sum(const float* mc) {
  float r;
  if (kMc) asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(r) : "l"(mc) : "memory");
  else asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(r) : "l"(mc) : "memory");
  return r;
}

}  // namespace apml
