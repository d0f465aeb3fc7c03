/* resample_oracle.c — TEST INFRASTRUCTURE ONLY (see cuppl_oracle.c's header): the CPU
 * restatement of the generic systematic-resampling primitive (csrc/resample_kernels.cu,
 * include/cuppl_gpu.h cuppl_resample).
 *
 * SMC is a non-goal of the reference, so, as for or_smc_step, this file DEFINES
 * the bits the GPU must reproduce (the same rule or_smc_step applies to
 * HMM populations) for an arbitrary population of N particles given fp32 log-weights lw[N] and
 * a fixed-size payload of P bytes per particle:
 *
 *   M        = max over finite-or-+inf lw_i (NaN ignored)
 *   e_i      = or_smc_e(lw_i, M)              (0 for -inf / NaN / lw - M < -87; exact fp32 sequence)
 *   w_i      = or_smc_w(e_i) = min(floor(e_i 2^31), 2^31)
 *   C        = inclusive u64 prefix of w, T = C[N-1]  (status 2 if T == 0)
 *   u        = or_comb_word(key, t)
 *   target_j = floor((j 2^32 + u) T / (N 2^32))        (or_comb_target, 128-bit)
 *   a_j      = min{i : C_i > target_j}
 *   out[j]   = payload[a_j] (P bytes), anc[j] = a_j
 *   s1 = sum e_i, s2 = sum e_i^2 in fp64, sequentially in index order.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

float or_smc_e(float lw, float M);
uint32_t or_smc_w(float e);
uint64_t or_comb_target(uint64_t j, uint32_t u, uint64_t T, uint64_t N);
uint32_t or_comb_word(uint64_t key, uint32_t t);

typedef struct or_resample_stats {
  float M;
  uint32_t status; /* 0 ok, 2 all-zero weights */
  uint64_t T;
  double s1, s2;
} or_resample_stats;

int or_resample(uint64_t N, const float* lw, const uint8_t* payload, uint64_t P, uint64_t key,
                uint32_t t, uint8_t* payload_out, uint64_t* anc, or_resample_stats* st) {
  float M = -INFINITY;
  for (uint64_t i = 0; i < N; ++i)
    if (lw[i] > M) M = lw[i];
  uint64_t* C = (uint64_t*)malloc(sizeof(uint64_t) * (N ? N : 1));
  float* E = (float*)malloc(sizeof(float) * (N ? N : 1));
  if (!C || !E) { free(C); free(E); return 1; }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)N; ++i) {
    E[i] = M > -INFINITY ? or_smc_e(lw[i], M) : 0.0f;
    C[i] = or_smc_w(E[i]);
  }
  uint64_t T = 0;
  double s1 = 0.0, s2 = 0.0;
  for (uint64_t i = 0; i < N; ++i) {
    const double e = (double)E[i];
    T += C[i];
    C[i] = T;
    s1 += e;
    s2 += e * e;
  }
  free(E);
  st->M = M;
  st->T = T;
  st->s1 = s1;
  st->s2 = s2;
  st->status = T == 0 ? 2 : 0;
  if (T == 0) { free(C); return 2; }
  const uint32_t u = or_comb_word(key, t);
#pragma omp parallel for schedule(static)
  for (int64_t jj = 0; jj < (int64_t)N; ++jj) {
    const uint64_t j = (uint64_t)jj;
    const uint64_t tj = or_comb_target(j, u, T, N);
    uint64_t lo = 0, hi = N - 1; /* smallest i with C[i] > tj (exists: C[N-1] = T > tj) */
    while (lo < hi) {
      const uint64_t mid = lo + ((hi - lo) >> 1);
      if (C[mid] > tj) hi = mid; else lo = mid + 1;
    }
    if (anc) anc[j] = lo;
    if (payload_out && P) memcpy(payload_out + j * P, payload + lo * P, (size_t)P);
  }
  free(C);
  return 0;
}
