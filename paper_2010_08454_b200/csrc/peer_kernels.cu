// peer_kernels.cu — device-side exchange between the ranks of one node over peer memory
// (CUDA-IPC-mapped arenas, NVLink on a multi-GPU node): the two small per-step collectives of
// the multi-rank SMC filter (the all-reduce MAX of the log-weight stabiliser
// and the all-gather of the 32-byte rank records) without NCCL or the host, so a rank's whole
// run — K5, exchanges, K6 with its peer stores — can be captured in one CUDA graph.
//
// Each rank's arena holds, per exchange phase, a mailbox of world slots and world flag words.
// One 32-thread CTA per exchange: lane q < world stores this rank's payload into slot `rank`
// of peer q's mailbox, fences at system scope, then releases flag `rank` of peer q with the
// phase's epoch (a device counter this kernel increments, so graph replays stay ordered); then
// lane q acquires its own flag q until it reaches the epoch, and the mailbox — every rank's
// payload in rank order — is reduced (MAX over int32) or copied out. A rank writes phase P of
// step t + 1 only after its phase-P' exchanges of step t, each of which needed every peer's
// earlier writes, so a slot is never overwritten before its reader consumed it. K6's peer
// stores are ordered before the next exchange's flags by K6's and this kernel's system fences.
// A spin that exceeds the timeout sets a status word and gives up (no hang).
#include "capi_internal.cuh"
#include "cuppl_device.cuh"

namespace cuppl {

struct PeerArgs {
  const uint8_t* src;                  // this rank's payload (device)
  unsigned int nbytes;                 // <= 64
  int rank, world;
  const unsigned long long* bases;     // [world] arena base address of every rank (device)
  unsigned long long mbox_off;         // offset of this phase's mailbox ([world][64] bytes)
  unsigned long long flags_off;        // offset of this phase's flags ([world] u64)
  unsigned long long* epoch;           // this phase's local epoch counter
  int* max_out;                        // MAX over the int32 payloads (or NULL)
  uint8_t* gather_out;                 // [world][nbytes] copy of the mailbox (or NULL)
  unsigned int* status;                // 1 on timeout
  unsigned long long timeout_ns;
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(32) peer_exchange_kernel(PeerArgs a) {
  const int q = threadIdx.x;
  const unsigned long long e = *a.epoch + 1;  // every rank runs the same exchange sequence
  __syncwarp();
  if (q == 0) *a.epoch = e;
  uint8_t* own = reinterpret_cast<uint8_t*>(a.bases[a.rank]);
  if (q < a.world) {
    uint8_t* peer = reinterpret_cast<uint8_t*>(a.bases[q]);
    uint8_t* slot = peer + a.mbox_off + 64ull * a.rank;
    for (unsigned int b = 0; b < a.nbytes; ++b) slot[b] = a.src[b];
    __threadfence_system();
    st_release_sys(reinterpret_cast<unsigned long long*>(peer + a.flags_off) + a.rank, e);
  }
  bool ok = true;
  if (q < a.world) {
    const unsigned long long* f = reinterpret_cast<const unsigned long long*>(own + a.flags_off) + q;
    const unsigned long long t0 = now_ns();
    while (ld_acquire_sys(f) < e) {
      if (now_ns() - t0 > a.timeout_ns) {
        ok = false;
        break;
      }
      __nanosleep(64);
    }
  }
  if (!__all_sync(0xffffffffu, ok)) {
    if (q == 0) atomicOr(a.status, 1u);
    return;
  }
  __threadfence_system();
  const uint8_t* mbox = own + a.mbox_off;
  if (a.gather_out && q < a.world)
    for (unsigned int b = 0; b < a.nbytes; ++b) a.gather_out[a.nbytes * q + b] = mbox[64ull * q + b];
  if (a.max_out) {
    int v = q < a.world ? *reinterpret_cast<const int*>(mbox + 64ull * q) : INT_MIN;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (q == 0) *a.max_out = v;
  }
}

}  // namespace cuppl

using namespace cuppl;

extern "C" {

int cuppl_peer_exchange(const void* src, uint32_t nbytes, const uint64_t* peer_bases, uint64_t mbox_off,
                        uint64_t flags_off, int rank, int world, uint64_t* epoch, int32_t* max_out,
                        void* gather_out, uint32_t* status, uint64_t timeout_ns, void* stream) {
  if (!src || !peer_bases || !epoch || !status) return set_error(CUPPL_E_ARGUMENT, "peer_exchange: NULL buffer");
  if (nbytes == 0 || nbytes > 64) return set_error(CUPPL_E_ARGUMENT, "peer_exchange: 1..64 bytes per rank");
  if (world < 1 || world > 32 || rank < 0 || rank >= world)
    return set_error(CUPPL_E_ARGUMENT, "peer_exchange: rank %d / world %d (<= 32)", rank, world);
  if (max_out && nbytes < 4) return set_error(CUPPL_E_ARGUMENT, "peer_exchange: MAX needs int32 payloads");
  PeerArgs a;
  a.src = static_cast<const uint8_t*>(src);
  a.nbytes = nbytes;
  a.rank = rank;
  a.world = world;
  a.bases = reinterpret_cast<const unsigned long long*>(peer_bases);
  a.mbox_off = mbox_off;
  a.flags_off = flags_off;
  a.epoch = reinterpret_cast<unsigned long long*>(epoch);
  a.max_out = max_out;
  a.gather_out = static_cast<uint8_t*>(gather_out);
  a.status = status;
  a.timeout_ns = timeout_ns;
  peer_exchange_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return cuda_status(cudaGetLastError(), "peer_exchange");
}

}  // extern "C"
