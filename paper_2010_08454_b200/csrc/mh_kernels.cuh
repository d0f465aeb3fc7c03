// mh_kernels.cuh — launch parameters of the many-chain lightweight Metropolis-Hastings kernel (K7).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/cuppl_gpu.h"

namespace cuppl {

constexpr int kMhMaxK = 7;            // mixture components (3-bit labels; code 7 is padding)
constexpr int kMhPadPoints = 256;     // data padded to 32 lanes x 8 points
constexpr int kMhMaxChainsPerCta = 28;

struct MhArgs {
  unsigned long long key;
  unsigned int n_chains;      // chains in this launch
  unsigned int chain_begin;   // global id of the first chain (Philox counter word 0)
  unsigned int n_steps;       // MH steps per chain
  unsigned int burn_in;       // steps not recorded
  unsigned int thin;          // record every thin-th step after burn-in
  int D;                      // data points
  int D_pad;                  // padded to a multiple of kMhPadPoints
  int K;                      // components
  float prior_sd;             // mu_k ~ normal(0, prior_sd)
  float neg_half_inv_var;     // -0.5 / sigma^2
  float ll_const;             // -D (ln sigma + 0.5 ln 2 pi)
  int chains_per_cta;
  const float* y;             // device [D_pad] (zero padded)
  float* mu_out;              // [n_chains][K] final state
  float* ll_out;              // [n_chains] final log-likelihood
  double* stats_out;          // [n_chains][2K + 2]: sum sorted mu, sum sorted mu^2, n_rec, n_acc
  float* trace_out;           // optional [n_chains][n_rec][K] sorted mu per recorded step
  unsigned int n_rec;         // recorded steps per chain (trace_out capacity)
  unsigned int pad_;
};

size_t mh_smem_bytes(int D_pad, int chains_per_cta);
cudaError_t launch_mh_gmm(const MhArgs& a, cudaStream_t st);

}  // namespace cuppl
