// hist_kernels.cu — K3: normalize() of weighted samples into an empirical posterior
// (SPEC.md:417-425): log-sum-exp stabiliser, per-value (histogram bin) probability mass, ESS
// and mode (argmax log-weight, ties to the lowest index).
//
// Determinism without float atomics: pass 1 reduces the max with an integer
// atomicMax on the order-preserving key of the double; pass 2 accumulates each weight
// exp(lw - M) into its bin as an unsigned 64-bit fixed-point number (scale 2^s with
// s = 62 - ceil(log2 n), so no sum can overflow) with integer atomics, whose result is
// independent of the order. sum w^2 and the argmax go through per-block records folded in a
// fixed order by the last block. Values below 2^-s of the max weight are dropped from the bins
// (|error| <= n 2^-s <= 2^-(62 - 2 log2 n) of the max weight).
#include <climits>

#include "capi_internal.cuh"
#include "cuppl_device.cuh"

namespace cuppl {
namespace {

constexpr int kHistThreads = 256;
constexpr int kHistSmemBins = 2048;

struct HistBlockRec {
  double s2;
  double amax_lw;
  unsigned long long amax_idx;
  unsigned long long n_finite;
};

__device__ __forceinline__ long long d2key(double d) {
  const long long i = __double_as_longlong(d);
  return i ^ ((i >> 63) & 0x7FFFFFFFFFFFFFFFll);
}
__device__ __forceinline__ double key2d(long long k) {
  return __longlong_as_double(k ^ ((k >> 63) & 0x7FFFFFFFFFFFFFFFll));
}

template <typename T>
__global__ void __launch_bounds__(kHistThreads) hist_max_kernel(const T* lw, unsigned long long n,
                                                                long long* max_key) {
  double m = neg_inf_d();
  for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const double v = static_cast<double>(lw[i]);
    if (v > m && v < __longlong_as_double(0x7FF0000000000000ll)) m = v;  // finite (NaN fails)
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > neg_inf_d()) atomicMax(max_key, d2key(m));
}

template <typename T>
__global__ void __launch_bounds__(kHistThreads) hist_sum_kernel(
    const T* lw, const int* bin, unsigned long long n, int n_bins, const long long* max_key,
    double scale, unsigned long long* bins, HistBlockRec* block_recs, unsigned int* counter,
    double* out /* [6]: max, s2, amax_lw, amax_idx(bits), n_finite(bits), reserved */) {
  __shared__ unsigned long long sbin[kHistSmemBins];
  __shared__ BlockScratch sc;
  __shared__ bool s_last;
  const bool smem_bins = n_bins <= kHistSmemBins;
  if (smem_bins)
    for (int b = threadIdx.x; b < n_bins; b += blockDim.x) sbin[b] = 0ull;
  __syncthreads();
  const long long mk = *max_key;
  const double M = key2d(mk);
  const bool any = mk != LLONG_MIN;
  double s2 = 0.0, amax = neg_inf_d();
  unsigned long long aidx = ~0ull, nf = 0;
  if (any) {
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
      const double v = static_cast<double>(lw[i]);
      if (!(v > neg_inf_d() && v < __longlong_as_double(0x7FF0000000000000ll))) continue;
      ++nf;
      if (v > amax) {  // increasing index per thread: ties keep the lowest
        amax = v;
        aidx = i;
      }
      const double w = exp(v - M);
      s2 = fma(w, w, s2);
      const unsigned long long q = static_cast<unsigned long long>(w * scale);  // floor
      if (q) {
        const int b = bin ? bin[i] : 0;
        if (b >= 0 && b < n_bins) {
          if (smem_bins) atomicAdd(&sbin[b], q);
          else atomicAdd(&bins[b], q);
        }
      }
    }
  }
  __syncthreads();
  if (smem_bins)
    for (int b = threadIdx.x; b < n_bins; b += blockDim.x)
      if (sbin[b]) atomicAdd(&bins[b], sbin[b]);
  const double bs2 = block_sum_d(s2, sc);
  unsigned long long bnf = block_sum_u(nf, sc);
  double al = amax;
  unsigned long long ai = aidx;
  block_argmax(al, ai, sc);
  if (threadIdx.x == 0) {
    block_recs[blockIdx.x] = HistBlockRec{bs2, al, ai, bnf};
    __threadfence();
    s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double f2 = 0.0, fl = neg_inf_d();
  unsigned long long fi = ~0ull, fn = 0;
  for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    const HistBlockRec r = block_recs[b];
    f2 += r.s2;
    fn += r.n_finite;
    if (r.amax_lw > fl || (r.amax_lw == fl && r.amax_idx < fi)) {
      fl = r.amax_lw;
      fi = r.amax_idx;
    }
  }
  f2 = block_sum_d(f2, sc);
  fn = block_sum_u(fn, sc);
  block_argmax(fl, fi, sc);
  if (threadIdx.x == 0) {
    out[0] = any ? M : neg_inf_d();
    out[1] = f2;
    out[2] = fl;
    out[3] = __longlong_as_double(static_cast<long long>(fi));
    out[4] = __longlong_as_double(static_cast<long long>(fn));
    out[5] = 0.0;
    *counter = 0u;
  }
}

}  // namespace
}  // namespace cuppl

using namespace cuppl;

namespace {
constexpr int kHistMaxBlocks = 148 * 8;

size_t hist_ws_bytes() { return 256 + sizeof(HistBlockRec) * kHistMaxBlocks; }

template <typename T>
int normalize_impl(const T* lw, const int32_t* bin, uint64_t n, int n_bins, uint64_t* bins,
                   double* out, int* scale_bits, void* ws, size_t ws_bytes, void* stream) {
  if (n == 0) return set_error(CUPPL_E_ARGUMENT, "normalize of an empty sample");
  if (!lw || !bins || !out || !scale_bits) return set_error(CUPPL_E_ARGUMENT, "NULL buffer");
  if (n_bins < 1) return set_error(CUPPL_E_ARGUMENT, "n_bins must be >= 1");
  if (!ws || ws_bytes < hist_ws_bytes()) return set_error(CUPPL_E_CAPACITY, "workspace too small");
  int sm = 0;
  if (int s = device_sm_count(&sm)) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int lg = 0;
  while ((1ull << lg) < n) ++lg;
  const int s = 62 - lg;  // sum of n values < 2^s each fits in 62 bits
  *scale_bits = s;
  char* base = static_cast<char*>(ws);
  long long* max_key = reinterpret_cast<long long*>(base);
  unsigned int* counter = reinterpret_cast<unsigned int*>(base + 64);
  HistBlockRec* recs = reinterpret_cast<HistBlockRec*>(base + 256);
  const long long init = LLONG_MIN;
  cudaError_t e = cudaMemcpyAsync(max_key, &init, sizeof(init), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(counter, 0, 4, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(bins, 0, sizeof(uint64_t) * n_bins, st);
  if (e != cudaSuccess) return cuda_status(e, "normalize setup");
  unsigned long long g = (n + kHistThreads - 1) / kHistThreads;
  const unsigned long long cap = static_cast<unsigned long long>(sm) * 8 < kHistMaxBlocks ? sm * 8 : kHistMaxBlocks;
  if (g > cap) g = cap;
  hist_max_kernel<T><<<static_cast<unsigned>(g), kHistThreads, 0, st>>>(lw, n, max_key);
  hist_sum_kernel<T><<<static_cast<unsigned>(g), kHistThreads, 0, st>>>(
      lw, bin, n, n_bins, max_key, ldexp(1.0, s), reinterpret_cast<unsigned long long*>(bins), recs,
      counter, out);
  return cuda_status(cudaGetLastError(), "normalize");
}
}  // namespace

extern "C" {

size_t cuppl_normalize_workspace_bytes(void) { return hist_ws_bytes(); }

int cuppl_normalize_f64(const double* lw, const int32_t* bin, uint64_t n, int n_bins, uint64_t* bins,
                        double* out, int* scale_bits, void* workspace, size_t workspace_bytes,
                        void* stream) {
  return normalize_impl(lw, bin, n, n_bins, bins, out, scale_bits, workspace, workspace_bytes, stream);
}

int cuppl_normalize_f32(const float* lw, const int32_t* bin, uint64_t n, int n_bins, uint64_t* bins,
                        double* out, int* scale_bits, void* workspace, size_t workspace_bytes,
                        void* stream) {
  return normalize_impl(lw, bin, n, n_bins, bins, out, scale_bits, workspace, workspace_bytes, stream);
}

}  // extern "C"
