// dist_kernels.cu — K8 batch draws and scores for every built-in distribution.
//
// dist_sample / dist_score of SPEC.md:303-320 (the absent `vm` module) for the constructor
// set of pkg/src/cuppl/builtins.py:86-94 plus categorical. The draw
// algorithms restate cuppl/rng.py:43-117 on a Philox word stream:
//   uniform        rng.py:43-45   -> 23-bit mantissa uniform [0,1)
//   randint        rng.py:47-56   -> Lemire multiply-shift with exact rejection
//   normal         rng.py:58-71   -> Box-Muller, spare normal cached in the stream state
//   exponential    rng.py:73-77   -> -ln(u)/rate, u in (0,1]
//   gamma          rng.py:79-98   -> Marsaglia-Tsang, shape < 1 boosted by u^(1/shape)
//   beta           rng.py:100-103 -> X/(X+Y), X ~ gamma(a), Y ~ gamma(b)
//   poisson        rng.py:105-117 -> Knuth for lambda < 30, recursive halving otherwise
// Sample i consumes the words of Philox blocks (first_id + i, 0..), tag in order, so the
// oracle (oracle/cuppl_oracle.c) replays the same consumption exactly.
#include "cuppl_device.cuh"
#include "dist_kernels.cuh"
#include "draws.cuh"

namespace cuppl {

__device__ __forceinline__ int categorical_index(const uint64_t* thr, int K, uint32_t w) {
  // smallest k with w < thr[k]; K-1 if none (thresholds are non-decreasing)
  int lo = 0, hi = K - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (static_cast<uint64_t>(w) < thr[mid]) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

__global__ void dist_sample_kernel(DistArgs a, uint64_t key, uint32_t tag, uint64_t first_id,
                                   uint64_t count, void* out) {
  const PhiloxKey k = make_key(key);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    WordStream s;
    s.init(k, first_id + i, tag);
    float* fo = static_cast<float*>(out);
    int32_t* io = static_cast<int32_t*>(out);
    switch (a.tag) {
      case CUPPL_DIST_NORMAL:  // fp64 like the reference, rounded once to the fp32 output
        fo[i] = static_cast<float>(__dadd_rn(a.p0, __dmul_rn(a.p1, s.normal_d())));
        break;
      case CUPPL_DIST_BERNOULLI: io[i] = s.uniform() < a.p0 ? 1 : 0; break;
      case CUPPL_DIST_POISSON: io[i] = s.poisson(a.p0); break;
      case CUPPL_DIST_UNIFORM_DISCRETE:
        io[i] = a.ia + static_cast<int32_t>(s.randint(static_cast<uint32_t>(a.ib - a.ia)));
        break;
      case CUPPL_DIST_UNIFORM_CONTINUOUS:
        fo[i] = static_cast<float>(__dadd_rn(a.p0, __dmul_rn(__dsub_rn(a.p1, a.p0), s.uniform_d())));
        break;
      case CUPPL_DIST_BETA: fo[i] = s.beta(a.p0, a.p1); break;
      case CUPPL_DIST_EXPONENTIAL: fo[i] = s.exponential(a.p0); break;
      case CUPPL_DIST_CATEGORICAL: io[i] = categorical_index(a.table, a.K, s.next()); break;
      default: break;
    }
  }
}

__global__ void dist_score_kernel(DistArgs a, const void* x, uint64_t count, float* score) {
  const float ninf = neg_inf_f();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float* fx = static_cast<const float*>(x);
    const int32_t* ix = static_cast<const int32_t*>(x);
    float r = ninf;
    switch (a.tag) {
      case CUPPL_DIST_NORMAL: {
        const float z = (fx[i] - a.p0) / a.p1;
        r = -0.5f * z * z - logf(a.p1) - kHalfLog2Pi;
        break;
      }
      case CUPPL_DIST_BERNOULLI: r = ix[i] ? logf(a.p0) : log1pf(-a.p0); break;
      case CUPPL_DIST_POISSON: {
        const int k = ix[i];
        if (k >= 0) r = (k == 0 ? 0.f : k * logf(a.p0)) - a.p0 - lgammaf(k + 1.0f);
        break;
      }
      case CUPPL_DIST_UNIFORM_DISCRETE:
        if (ix[i] >= a.ia && ix[i] < a.ib) r = -logf(static_cast<float>(a.ib - a.ia));
        break;
      case CUPPL_DIST_UNIFORM_CONTINUOUS:
        if (fx[i] >= a.p0 && fx[i] <= a.p1) r = -logf(a.p1 - a.p0);
        break;
      case CUPPL_DIST_BETA: {
        const float v = fx[i];
        if (v >= 0.f && v <= 1.f)
          r = (a.p0 - 1.f) * logf(v) + (a.p1 - 1.f) * log1pf(-v) -
              (lgammaf(a.p0) + lgammaf(a.p1) - lgammaf(a.p0 + a.p1));
        break;
      }
      case CUPPL_DIST_EXPONENTIAL:
        if (fx[i] >= 0.f) r = logf(a.p0) - a.p0 * fx[i];
        break;
      case CUPPL_DIST_CATEGORICAL: {
        const int k = ix[i];
        if (k >= 0 && k < a.K) {
          const uint64_t hi = k < a.K - 1 ? a.table[k] : (1ull << 32);
          const uint64_t lo = k > 0 ? a.table[k - 1] : 0ull;
          if (hi > lo) r = logf(static_cast<float>(hi - lo)) - 32.0f * kLn2;
        }
        break;
      }
      default: break;
    }
    score[i] = r;
  }
}

__global__ void philox_blocks_kernel(uint64_t key, uint64_t first_id, uint32_t block,
                                     uint32_t tag, uint64_t count, uint4* out) {
  const PhiloxKey k = make_key(key);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = draw_block(k, first_id + i, block, tag);
}

static unsigned grid_for(uint64_t count, int threads, int sm_count) {
  uint64_t g = (count + threads - 1) / threads;
  const uint64_t cap = static_cast<uint64_t>(sm_count) * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

cudaError_t launch_dist_sample(const DistArgs& a, uint64_t key, uint32_t tag, uint64_t first_id,
                               uint64_t count, void* out, int sm_count, cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  dist_sample_kernel<<<grid_for(count, 256, sm_count), 256, 0, stream>>>(a, key, tag, first_id,
                                                                         count, out);
  return cudaGetLastError();
}

cudaError_t launch_dist_score(const DistArgs& a, const void* x, uint64_t count, float* score,
                              int sm_count, cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  dist_score_kernel<<<grid_for(count, 256, sm_count), 256, 0, stream>>>(a, x, count, score);
  return cudaGetLastError();
}

cudaError_t launch_philox_blocks(uint64_t key, uint64_t first_id, uint32_t block, uint32_t tag,
                                 uint64_t count, uint32_t* out, int sm_count,
                                 cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  philox_blocks_kernel<<<grid_for(count, 256, sm_count), 256, 0, stream>>>(
      key, first_id, block, tag, count, reinterpret_cast<uint4*>(out));
  return cudaGetLastError();
}

}  // namespace cuppl
