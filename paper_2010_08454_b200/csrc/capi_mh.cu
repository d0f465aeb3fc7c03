// capi_mh.cu — extern "C" entry points of the many-chain MH engine (include/cuppl_gpu.h).
#include <cmath>
#include <cstring>

#include "capi_internal.cuh"
#include "cuppl_device.cuh"
#include "mh_kernels.cuh"

using namespace cuppl;

namespace {
int padded(int D) {
  int M = 0, NT = 0;
  mh_shape(D, &M, &NT);
  return 8 * NT * M;
}
}  // namespace

extern "C" {

int cuppl_mh_padded_points(int D) { return padded(D < 1 ? 1 : D); }

int cuppl_mh_gmm(const float* y, int D, int K, float prior_sd, float sigma, uint32_t n_chains,
                 uint32_t chain_begin, uint32_t n_steps, uint32_t burn_in, uint32_t thin,
                 uint64_t key, float* mu_out, float* ll_out, double* stats_out, float* trace_out,
                 uint32_t n_rec, void* stream) {
  if (K < 1 || K > kMhMaxK) return set_error(CUPPL_E_CAPACITY, "K=%d outside [1, %d]", K, kMhMaxK);
  if (D < 1) return set_error(CUPPL_E_ARGUMENT, "D must be >= 1");
  if (!(prior_sd > 0.f) || !(sigma > 0.f) || !std::isfinite(prior_sd) || !std::isfinite(sigma))
    return set_error(CUPPL_E_INVALID_PARAM, "normal(mean, sd): sd must be > 0");
  if (thin < 1) return set_error(CUPPL_E_ARGUMENT, "thin must be >= 1");
  if (!y || !mu_out || !ll_out || !stats_out) return set_error(CUPPL_E_ARGUMENT, "NULL buffer");
  if (n_chains == 0) return CUPPL_OK;
  int M = 0, NT = 0;
  mh_shape(D, &M, &NT);
  if (M > kMhMaxGroupsPerThread)
    return set_error(CUPPL_E_CAPACITY, "D=%d exceeds %d points", D, 8 * kMhMaxThreads * kMhMaxGroupsPerThread);
  const int G = NT * M, D_pad = 8 * G;
  int dev = 0, max_smem = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  e = cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
  // chains per CTA: one wave over the SMs, at most one per lane of warp 0, within shared memory
  int cpc = static_cast<int>((n_chains + sms - 1) / sms);
  if (cpc > kMhMaxChainsPerCta) cpc = kMhMaxChainsPerCta;
  if (cpc < 1) cpc = 1;
  while (cpc > 1 && mh_smem_bytes(G, K, cpc, NT) > static_cast<size_t>(max_smem)) --cpc;
  if (mh_smem_bytes(G, K, cpc, NT) > static_cast<size_t>(max_smem))
    return set_error(CUPPL_E_CAPACITY, "D=%d does not fit in shared memory", D);
  MhArgs a;
  std::memset(&a, 0, sizeof(a));
  a.key = key;
  a.n_chains = n_chains;
  a.chain_begin = chain_begin;
  a.n_steps = n_steps;
  a.burn_in = burn_in;
  a.thin = thin;
  a.D = D;
  a.D_pad = D_pad;
  a.G = G;
  a.threads = NT;
  a.groups_per_thread = M;
  a.K = K;
  a.prior_sd = prior_sd;
  a.neg_half_inv_var = static_cast<float>(-0.5 / (static_cast<double>(sigma) * sigma));
  a.ll_const = static_cast<float>(-D * (std::log(static_cast<double>(sigma)) + 0.91893853320467274178));
  a.neg_half_inv_var64 = -0.5 / (static_cast<double>(sigma) * sigma);
  a.ll_const64 = -D * (std::log(static_cast<double>(sigma)) + 0.91893853320467274178);
  a.chains_per_cta = cpc;
  a.y = y;
  a.mu_out = mu_out;
  a.ll_out = ll_out;
  a.stats_out = stats_out;
  a.trace_out = trace_out;
  a.n_rec = n_rec;
  return cuda_status(launch_mh_gmm(a, static_cast<cudaStream_t>(stream)), "mh_gmm");
}

}  // extern "C"
