// mh_kernels.cuh — launch parameters of the many-chain lightweight Metropolis-Hastings kernel (K7).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/cuppl_gpu.h"

namespace cuppl {

constexpr int kMhMaxK = 7;            // mixture components (label K is padding)
constexpr int kMhMaxThreads = 640;    // threads per CTA (each holds 8-point groups of y)
constexpr int kMhMaxGroupsPerThread = 8;  // D <= 640 * 8 * 8 = 40960 points
constexpr int kMhMaxChainsPerCta = 32;    // one chain per lane of warp 0
constexpr int kMhTab = 64;                // pair-code table entries: K^2 + K + 1 <= 57 (K <= 7)

// Point groups per thread (M) and threads per CTA (NT) for D points: D is padded to 8 NT M.
inline void mh_shape(int D, int* M, int* NT) {
  const int g = (D + 7) / 8;
  int m = (g + kMhMaxThreads - 1) / kMhMaxThreads;
  if (m < 1) m = 1;
  int nt = ((g + m - 1) / m + 31) / 32 * 32;
  if (nt < 32) nt = 32;
  *M = m;
  *NT = nt;
}

struct MhArgs {
  unsigned long long key;
  unsigned int n_chains;      // chains in this launch
  unsigned int chain_begin;   // global id of the first chain (Philox counter word 0)
  unsigned int n_steps;       // MH steps per chain
  unsigned int burn_in;       // steps not recorded
  unsigned int thin;          // record every thin-th step after burn-in
  int D;                      // data points
  int D_pad;                  // 8 G
  int G;                      // 8-point groups = threads * groups_per_thread
  int threads;                // threads per CTA
  int groups_per_thread;      // M: y values per thread = 8 M (registers)
  int K;                      // components
  float prior_sd;             // mu_k ~ normal(0, prior_sd)
  float neg_half_inv_var;     // -0.5 / sigma^2
  float ll_const;             // -D (ln sigma + 0.5 ln 2 pi)
  double neg_half_inv_var64;  // the same in fp64: the chains' log-likelihood folds in fp64
  double ll_const64;
  int chains_per_cta;
  const float* y;             // device [D_pad] (zero padded)
  float* mu_out;              // [n_chains][K] final state
  float* ll_out;              // [n_chains] final log-likelihood
  double* stats_out;          // [n_chains][2K + 2]: sum sorted mu, sum sorted mu^2, n_rec, n_acc
  float* trace_out;           // optional [n_chains][n_rec][K] sorted mu per recorded step
  unsigned int n_rec;         // recorded steps per chain (trace_out capacity)
  unsigned int pad_;
};

size_t mh_smem_bytes(int G, int K, int chains_per_cta, int threads);
cudaError_t launch_mh_gmm(const MhArgs& a, cudaStream_t st);

}  // namespace cuppl
