// is_accum.cuh — per-thread online log-sum-exp accumulator and the fused block / grid record
// epilogue of the importance-sampling kernels (shared with the runtime-compiled model kernels
// of frontend.py).
#pragma once
#include "cuppl_device.cuh"

namespace cuppl {

// Thread-level online accumulator (fp32 lanes; fp64 from the block level up, D10).
template <int NS, int NB>
struct ThreadAcc {
  float m, s, s2;
  float st[NS > 0 ? NS : 1];
  float bn[NB > 0 ? NB : 1];
  float amax_lw;
  uint64_t amax_pid;
  uint32_t n_fin, n_tot;

  __device__ __forceinline__ void init() {
    m = neg_inf_f();
    s = s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NS; ++k) st[k] = 0.f;
#pragma unroll
    for (int k = 0; k < NB; ++k) bn[k] = 0.f;
    amax_lw = neg_inf_f();
    amax_pid = ~0ull;
    n_fin = n_tot = 0;
  }

  // Add one particle: stats f[k] and discrete bin `bin` (ignored when NB == 0).
  __device__ __forceinline__ void add(float lw, uint64_t pid, const float* f, int bin) {
    ++n_tot;
    if (!(fabsf(lw) <= 3.402823466e38f)) return;  // excludes -inf, +inf, NaN (D9)
    ++n_fin;
    if (lw > amax_lw) {  // particles arrive in increasing pid per thread: ties keep the lowest
      amax_lw = lw;
      amax_pid = pid;
    }
    if (lw > m) {
      const float f0 = fast_ex2((m - lw) * kLog2e);
      s *= f0;
      s2 *= f0 * f0;
#pragma unroll
      for (int k = 0; k < NS; ++k) st[k] *= f0;
#pragma unroll
      for (int k = 0; k < NB; ++k) bn[k] *= f0;
      m = lw;
    }
    const float w = fast_ex2((lw - m) * kLog2e);
    s += w;
    s2 = fmaf(w, w, s2);
#pragma unroll
    for (int k = 0; k < NS; ++k) st[k] = fmaf(w, f[k], st[k]);
#pragma unroll
    for (int k = 0; k < NB; ++k) bn[k] += (bin == k) ? w : 0.f;
  }

  // record view (block_reduce_view)
  static constexpr int kStats = NS;
  static constexpr int kBins = NB;
  __device__ __forceinline__ unsigned long long n_finite() const { return n_fin; }
  __device__ __forceinline__ unsigned long long n_total() const { return n_tot; }
  __device__ __forceinline__ double max_lw() const { return m; }
  __device__ __forceinline__ double sum_w() const { return s; }
  __device__ __forceinline__ double sum_w2() const { return s2; }
  __device__ __forceinline__ double stat(int k) const { return st[k]; }
  __device__ __forceinline__ double bin(int k) const { return bn[k]; }
  __device__ __forceinline__ double argmax_lw() const { return amax_lw; }
  __device__ __forceinline__ unsigned long long argmax_pid() const { return amax_pid; }
};

// The same accumulator in fp64 (exact exp / log): fp64 models (enumeration, where the record
// holds exact path probabilities).
template <int NS, int NB>
struct ThreadAccF64 {
  double m, s, s2;
  double st[NS > 0 ? NS : 1];
  double bn[NB > 0 ? NB : 1];
  double amax_lw;
  uint64_t amax_pid;
  uint32_t n_fin, n_tot;

  __device__ __forceinline__ void init() {
    m = neg_inf_d();
    s = s2 = 0.0;
#pragma unroll
    for (int k = 0; k < NS; ++k) st[k] = 0.0;
#pragma unroll
    for (int k = 0; k < NB; ++k) bn[k] = 0.0;
    amax_lw = neg_inf_d();
    amax_pid = ~0ull;
    n_fin = n_tot = 0;
  }
  __device__ __forceinline__ void add(double lw, uint64_t pid, const double* f, int bin) {
    ++n_tot;
    if (!(fabs(lw) <= 1.7976931348623157e308)) return;  // excludes -inf, +inf, NaN (D9)
    ++n_fin;
    if (lw > amax_lw) {
      amax_lw = lw;
      amax_pid = pid;
    }
    if (lw > m) {
      const double f0 = exp(m - lw);
      s *= f0;
      s2 *= f0 * f0;
#pragma unroll
      for (int k = 0; k < NS; ++k) st[k] *= f0;
#pragma unroll
      for (int k = 0; k < NB; ++k) bn[k] *= f0;
      m = lw;
    }
    const double w = exp(lw - m);
    s += w;
    s2 = fma(w, w, s2);
#pragma unroll
    for (int k = 0; k < NS; ++k) st[k] = fma(w, f[k], st[k]);
#pragma unroll
    for (int k = 0; k < NB; ++k) bn[k] += (bin == k) ? w : 0.0;
  }
  static constexpr int kStats = NS;
  static constexpr int kBins = NB;
  __device__ __forceinline__ unsigned long long n_finite() const { return n_fin; }
  __device__ __forceinline__ unsigned long long n_total() const { return n_tot; }
  __device__ __forceinline__ double max_lw() const { return m; }
  __device__ __forceinline__ double sum_w() const { return s; }
  __device__ __forceinline__ double sum_w2() const { return s2; }
  __device__ __forceinline__ double stat(int k) const { return st[k]; }
  __device__ __forceinline__ double bin(int k) const { return bn[k]; }
  __device__ __forceinline__ double argmax_lw() const { return amax_lw; }
  __device__ __forceinline__ unsigned long long argmax_pid() const { return amax_pid; }
};

// Block reduce + grid combine epilogue shared by the eval kernels.
template <typename Acc>
__device__ __forceinline__ void is_epilogue(const Acc& acc, cuppl_is_record* block_recs,
                                            unsigned int* counter, cuppl_is_record* rec_out) {
  __shared__ BlockScratch sc;
  __shared__ cuppl_is_record brec;
  block_reduce_view(acc, &brec, sc);
  __syncthreads();
  grid_combine(block_recs, counter, rec_out, brec, sc);
}

}  // namespace cuppl
