// capi_resample.cu — extern "C" entry points of the generic resampling primitive
// (include/cuppl_gpu.h cuppl_resample, kernels in resample_kernels.cu).
#include <cstring>

#include "capi_internal.cuh"
#include "resample_kernels.cuh"

using namespace cuppl;

namespace {
size_t align256(size_t v) { return (v + 255) & ~static_cast<size_t>(255); }

// Workspace: [zeroed: counters, flags] [blk_max] [M, total] [tile_prefix] [tile_s]
struct RsWs {
  size_t counters, flags, zero_end, blk_max, scalars, tile_prefix, tile_s, total;
};
RsWs rs_layout(uint64_t n) {
  const uint64_t n_tiles = (n + kRsTile - 1) / kRsTile;
  const uint64_t n_blocks = (n_tiles + kRsScanTiles - 1) / kRsScanTiles;
  RsWs w;
  size_t o = 0;
  w.counters = o;
  o = align256(o + 16);
  w.flags = o;
  o = align256(o + n_blocks * 8);
  w.zero_end = o;
  w.blk_max = o;
  o = align256(o + kRsMaxG1 * 4);
  w.scalars = o;
  o = align256(o + 16);
  w.tile_prefix = o;
  o = align256(o + n_tiles * 8);
  w.tile_s = o;
  o = align256(o + n_blocks * 16);
  w.total = o;
  return w;
}
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
}  // namespace

extern "C" {

size_t cuppl_resample_workspace_bytes(uint64_t n) { return rs_layout(n < 1 ? 1 : n).total; }

int cuppl_resample(const float* lw, uint64_t n, const void* payload, uint64_t payload_bytes, uint64_t key,
                   uint32_t t, void* payload_out, uint64_t* ancestors_out, cuppl_resample_stats* stats_out,
                   void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 1 || n >= (1ull << 31)) return set_error(CUPPL_E_CAPACITY, "n=%llu outside [1, 2^31)", (unsigned long long)n);
  if (!lw || !stats_out) return set_error(CUPPL_E_ARGUMENT, "NULL lw / stats_out");
  if (payload_bytes && (!payload || !payload_out)) return set_error(CUPPL_E_ARGUMENT, "NULL payload buffer");
  if (payload_bytes > (1ull << 20)) return set_error(CUPPL_E_CAPACITY, "payload_bytes > 1 MiB");
  if (!aligned16(lw) || (payload_bytes && (!aligned16(payload) || !aligned16(payload_out))))
    return set_error(CUPPL_E_ARGUMENT, "lw / payload buffers must be 16-byte aligned");
  const RsWs L = rs_layout(n);
  if (!workspace || workspace_bytes < L.total)
    return set_error(CUPPL_E_CAPACITY, "workspace %zu < %zu bytes", workspace_bytes, L.total);
  int sm = 0;
  if (int s = device_sm_count(&sm)) return s;
  char* ws = static_cast<char*>(workspace);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(ws, 0, L.zero_end, st);
  if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync");
  RsArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n = n;
  a.lw = lw;
  a.payload = static_cast<const uint8_t*>(payload);
  a.P = payload_bytes;
  a.payload_out = static_cast<uint8_t*>(payload_out);
  a.anc_out = reinterpret_cast<unsigned long long*>(ancestors_out);
  a.key = key;
  a.t = t;
  a.tma = 1;  // every buffer is 16-byte aligned (checked above)
  a.word4 = (payload_bytes % 4) == 0;
  unsigned long long g1 = (n + 4ull * kRsThreads * 8 - 1) / (4ull * kRsThreads * 8);  // ~8 float4 per thread
  if (g1 > static_cast<unsigned long long>(4 * sm)) g1 = 4ull * sm;
  if (g1 > static_cast<unsigned long long>(kRsMaxG1)) g1 = kRsMaxG1;
  a.g1 = static_cast<unsigned int>(g1 ? g1 : 1);
  a.counters = reinterpret_cast<unsigned int*>(ws + L.counters);
  a.flags = reinterpret_cast<unsigned long long*>(ws + L.flags);
  a.blk_max = reinterpret_cast<float*>(ws + L.blk_max);
  a.M = reinterpret_cast<float*>(ws + L.scalars);
  a.total = reinterpret_cast<unsigned long long*>(ws + L.scalars + 8);
  a.tile_prefix = reinterpret_cast<unsigned long long*>(ws + L.tile_prefix);
  a.tile_s = reinterpret_cast<double*>(ws + L.tile_s);
  a.stats_out = stats_out;
  a.n_tiles = (n + kRsTile - 1) / kRsTile;
  a.n_scan_blocks = (a.n_tiles + kRsScanTiles - 1) / kRsScanTiles;
  return cuda_status(launch_resample(a, sm, st), "resample");
}

}  // extern "C"
