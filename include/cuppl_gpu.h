/*
 * cuppl_gpu.h — C ABI of libcuppl_gpu.so, the sm_100a inference hot path.
 *
 * This is the drop-in boundary for CuPPL's (arXiv 2010.08454) inference engines. The
 * reference keeps these engines in Python (`cuppl.infer`, specified in SPEC.md:363-459, not
 * shipped) on top of `cuppl.rng.Rng` (pkg/src/cuppl/rng.py:23-117) and
 * `cuppl.values.DistValue` (pkg/src/cuppl/values.py:86-98). Every entry point below replaces
 * one piece of that path; the reference interface it replaces is cited next to it.
 *
 * Conventions:
 *   - plain C types only; device buffers are raw pointers the caller allocated (PyTorch);
 *   - `stream` is a cudaStream_t passed as void*; every call is stream-ordered and never
 *     synchronises the host unless documented;
 *   - the library keeps no allocations between calls; scratch comes from the caller's
 *     `workspace` sized by the matching *_workspace_bytes() query;
 *   - return value is a cuppl_status; cuppl_last_error() gives a thread-local message.
 *
 * Random numbers: Philox4x32-10 (Salmon et al. 2011) keyed by the 64-bit `Rng.key` of
 * cuppl/rng.py:27 (split as key_lo, key_hi). The counter of every draw is
 * (id_lo, id_hi, block, tag) where id is the 64-bit global particle / chain / sample index,
 * `block` the 128-bit block index within that id's stream and `tag` one of CUPPL_TAG_*.
 * This replaces Rng.split(i)/next_u64 (cuppl/rng.py:31-41): like split(i), a stream is a
 * pure function of (key, i).
 */
#ifndef CUPPL_GPU_H
#define CUPPL_GPU_H

#ifdef __CUDACC_RTC__  /* runtime-compiled model kernels (NVRTC): no libc headers */
typedef unsigned long long uint64_t;
typedef unsigned int uint32_t;
typedef int int32_t;
typedef unsigned char uint8_t;
#else
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define CUPPL_ABI_VERSION 1

#if defined(__GNUC__)
#define CUPPL_API __attribute__((visibility("default")))
#else
#define CUPPL_API
#endif

/* Status codes. Python maps them onto the reference exception classes of
 * pkg/src/cuppl/errors.py (InvalidDistParamError :135, AllZeroWeightError :119,
 * UnsupportedDistError :97, InferRuntimeError :123). */
typedef enum cuppl_status {
  CUPPL_OK = 0,
  CUPPL_E_INVALID_PARAM = 1, /* errors.py:135 InvalidDistParamError */
  CUPPL_E_ALL_ZERO = 2,      /* errors.py:119 AllZeroWeightError */
  CUPPL_E_CUDA = 3,          /* CUDA runtime failure (message in cuppl_last_error) */
  CUPPL_E_NCCL = 4,          /* reserved: collectives are issued by the host (torch.distributed) */
  CUPPL_E_CAPACITY = 5,      /* workspace / parameter-space too small */
  CUPPL_E_UNSUPPORTED = 6,   /* errors.py:97 UnsupportedDistError */
  CUPPL_E_ARGUMENT = 7       /* bad pointer / size argument */
} cuppl_status;

/* Philox counter tags (word 3 of the counter). */
#define CUPPL_TAG_IS 1u        /* importance-sampling prior draws            */
#define CUPPL_TAG_SMC_INIT 2u  /* SMC t = 0 draws                             */
#define CUPPL_TAG_SMC_STEP 3u  /* SMC transition draws (block = time step)    */
#define CUPPL_TAG_SMC_COMB 4u  /* SMC systematic-comb offset (one per step)   */
#define CUPPL_TAG_MH 5u        /* MH chains (block = step)                    */
#define CUPPL_TAG_MH_INIT 6u   /* MH initial trace                            */
#define CUPPL_TAG_DIST 7u      /* batch dist_sample                           */
#define CUPPL_TAG_DSL 8u       /* runtime-compiled CuPPL models (frontend.py)  */
#define CUPPL_TAG_DSL_MH 9u    /* compiled LMH chains: id = step << 32 | chain  */

/* Distribution tags: order of the constructors in pkg/src/cuppl/builtins.py:86-94, plus
 * categorical (absent from the reference catalog). */
#define CUPPL_DIST_NORMAL 0             /* normal(mean, sd)            builtins.py:87 */
#define CUPPL_DIST_BERNOULLI 1          /* bernoulli(p)                builtins.py:88 */
#define CUPPL_DIST_POISSON 2            /* poisson(lambda)             builtins.py:89 */
#define CUPPL_DIST_UNIFORM_DISCRETE 3   /* uniform-discrete(a, b) [a,b) builtins.py:90 */
#define CUPPL_DIST_UNIFORM_CONTINUOUS 4 /* uniform-continuous(a, b)    builtins.py:91 */
#define CUPPL_DIST_BETA 5               /* beta(a, b)                  builtins.py:93 */
#define CUPPL_DIST_EXPONENTIAL 6        /* exponential(rate)           builtins.py:94 */
#define CUPPL_DIST_CATEGORICAL 7        /* categorical(weights)      */

/* Fixed-size distribution value: the paper's {int32 tag, 3 x 64-bit payload} encoding
 * (cuppl/values.py:86-98). Categorical keeps its cumulative u64
 * thresholds in a device side table (like the SPEC's empirical kind). */
typedef struct cuppl_dist {
  int32_t tag;
  int32_t n_table;        /* categorical: number of categories K (>= 1) */
  double p0, p1, p2;      /* parameters in the reference's argument order */
  const uint64_t* table;  /* categorical: device pointer to K-1 thresholds in [0, 2^32] */
} cuppl_dist;

/* Per-rank importance-sampling record: the compact EmpiricalDistribution of SPEC.md:376-379
 * plus the normalize() state of SPEC.md:417-425 (log-sum-exp stabiliser M and rescaled sums).
 * All weights are exp(lw - max_lw). Records merge associatively (cuppl_is_record_merge). */
#define CUPPL_REC_STATS 16
#define CUPPL_REC_BINS 8
typedef struct cuppl_is_record {
  double max_lw;     /* M: max finite log-weight (-inf if none)                     */
  double sum_w;      /* sum exp(lw - M) over finite lw                              */
  double sum_w2;     /* sum exp(2 (lw - M))  (ESS = sum_w^2 / sum_w2)               */
  double argmax_lw;  /* log-weight of the posterior mode particle                   */
  uint64_t argmax_pid; /* its global particle id; ties go to the lowest id (D7)     */
  uint64_t n_finite; /* particles with a finite log-weight                          */
  uint64_t n_total;  /* particles evaluated                                         */
  uint64_t reserved;
  double stat_w[CUPPL_REC_STATS]; /* sum w * f_k(theta), model-defined statistics   */
  double bin_w[CUPPL_REC_BINS];   /* sum w per discrete bin of the return value     */
} cuppl_is_record;

/* ---- library ---------------------------------------------------------------------- */
CUPPL_API int cuppl_abi_version(void);
CUPPL_API const char* cuppl_last_error(void);
/* Number of SMs of the current device (grid sizing is a multiple of it). */
CUPPL_API int cuppl_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ---- K8: counter-based draws (replaces Rng.next_u64 / split, cuppl/rng.py:31-41) ---- */
/* out[4*i + w] = word w of Philox4x32-10(ctr = (id_lo, id_hi, block, tag), key) for
 * i in [0, count), id = first_id + i. Debug/test entry point for bit-exact parity. */
CUPPL_API int cuppl_philox_blocks(uint64_t key, uint64_t first_id, uint32_t block, uint32_t tag,
                        uint64_t count, uint32_t* out, void* stream);

/* ---- K8: batch dist_sample / dist_score (builtins.py:96-99) -------- */
/* Draw count samples: sample i uses the Philox stream (first_id + i, block 0.., tag).
 * Output is float for continuous kinds, int32 for discrete kinds (bernoulli: 0/1). */
CUPPL_API int cuppl_dist_sample(const cuppl_dist* d, uint64_t key, uint32_t tag, uint64_t first_id,
                      uint64_t count, void* out, void* stream);
/* score[i] = dist_score(d, x[i]) (natural log, -inf outside the support). x is float for
 * continuous kinds and int32 for discrete kinds. */
CUPPL_API int cuppl_dist_score(const cuppl_dist* d, const void* x, uint64_t count, float* score,
                     void* stream);

/* ---- K1 + K2: importance sampling (replaces run_importance) -------- */
/* Workspace bytes for an importance-sampling launch on the current device. */
CUPPL_API size_t cuppl_is_workspace_bytes(void);
/* The same for a data set of n_points: data sets larger than the kernel-parameter block
 * (> 3968 points for linear regression, > 64 for the polynomial model) are copied into the
 * workspace tail and read from device memory (up to 2^24 points). */
CUPPL_API size_t cuppl_is_workspace_bytes_n(int n_points);

/* Fig.1 polynomial model:
 *   n ~ uniform-discrete(2, 5); c_j ~ normal(0, 10), j < n; factor(-sum_i (y_i - sum_j c_j x_i^j)^2)
 * for global particle ids [pid_begin, pid_end). xs/ys are HOST arrays of n_points floats
 * (they are passed to the kernel by value). Optional device outputs (NULL to skip):
 *   lw_out[N], deg_out[N] (int32 n), coef_out[4N] (c_0..c_3, zero-padded), N = pid_end-pid_begin.
 * injected (device, NULL for Philox): 5 floats per particle (n, c_0..c_3) replacing the draws.
 * rec_out: device cuppl_is_record (bin_w[n-2] = posterior mass of degree n; stat_w holds
 * sum w*c_j per degree: n=2 -> [0,1], n=3 -> [2..4], n=4 -> [5..8]). */
CUPPL_API int cuppl_is_poly(const float* xs, const float* ys, int n_points, uint64_t pid_begin,
                  uint64_t pid_end, uint64_t key, const float* injected, float* lw_out,
                  int32_t* deg_out, float* coef_out, cuppl_is_record* rec_out, void* workspace,
                  size_t workspace_bytes, void* stream);

/* Bayesian linear regression: a, b ~ normal(0, 10);
 * observe(normal(a x_i + b, sigma), y_i) for each point (desugar.py:37-39).
 * injected: 2 floats per particle (a, b). coef_out[2N] = (a, b).
 * rec_out->stat_w = [sum w a, sum w b, sum w a^2, sum w b^2, sum w a b]. */
CUPPL_API int cuppl_is_linreg(const float* xs, const float* ys, int n_points, float sigma,
                    uint64_t pid_begin, uint64_t pid_end, uint64_t key, const float* injected,
                    float* lw_out, float* coef_out, cuppl_is_record* rec_out, void* workspace,
                    size_t workspace_bytes, void* stream);

/* ---- K4/K5/K6: SMC bootstrap particle filter (new: SPEC.md:455 lists SMC as a non-goal;
 *      semantics defined by SURVEY.md Appendix A D6 and oracle/cuppl_oracle.c or_smc_*) ---- */
typedef struct cuppl_smc_model {
  int32_t n_states;           /* S <= 256 (particle state is one byte)                    */
  float inv_sd;               /* emission y_t ~ normal(mu[x_t], sd): 1 / sd                */
  float c;                    /* -ln sd - 0.5 ln 2 pi                                       */
  int32_t reserved;
  const uint64_t* alias_trans; /* device [S][S] alias tables of the transition rows:      */
                               /*   entry = thr (bits 0..32, in [0, 2^32]) | alias << 40    */
  const uint64_t* alias_init;  /* device [S] alias table of the initial distribution       */
  const float* mu;            /* HOST [S] emission means (passed by value to the kernels)   */
  const uint64_t* key_dev;    /* optional DEVICE Philox key: when non-NULL, cuppl_smc_init /  */
                              /*   cuppl_smc_resample read the key here at run time and ignore */
                              /*   their `key` argument (one captured CUDA graph of the whole  */
                              /*   time-step loop then serves every seed)                      */
} cuppl_smc_model;

/* Scratch for one rank of n_local particles: segment offsets, look-back words, counters,
 * per-tile sums. Must be zeroed once before the first step (cuppl_smc_init does it). */
CUPPL_API size_t cuppl_smc_workspace_bytes(uint64_t n_local);

/* A population is its states x (u8 per particle); in this discrete-state HMM the log-weight is
 * a function of the state, lw = log N(y_t; mu[x], sd) (fp32, fixed op sequence), so the kernels
 * tabulate the S per-state weights of a step instead of storing log-weights. */

/* t = 0: x[j] ~ categorical(init) for local particles j_begin + [0, n_local) (j_begin multiple
 * of 16); atomicMax of lw_0 into *m_key (ordered int, caller initialises it to INT32_MIN).
 * Zeroes the workspace. */
CUPPL_API int cuppl_smc_init(const cuppl_smc_model* m, uint64_t n_local, uint64_t j_begin,
                             uint64_t key, float y0, uint8_t* x, int32_t* m_key, void* workspace,
                             size_t workspace_bytes, void* stream);

/* Weight scan of population t (K5) with observation y: quantised weights against max *m_key,
 * segment offsets and tile prefixes (single-pass decoupled look-back) into the workspace,
 * rank_rec[0] = T_r (integer weight total of this rank; rank_rec[1..3] untouched);
 * hist[S] (optional, zeroed by the caller) += integer weights per state. */
CUPPL_API int cuppl_smc_scan(const cuppl_smc_model* m, uint64_t n_local, float y, const uint8_t* x,
                             const int32_t* m_key, uint64_t* hist, uint64_t* rank_rec,
                             void* workspace, size_t workspace_bytes, void* stream);

/* Systematic resampling of population t (observation y_cur) + propagation to t+1 (y_next)
 * (K6). rank_recs: device [world][4] records of every rank (all-gathered); rank_begin: device
 * [world+1] global index of each rank's first particle (multiples of 16); x_out / anc_out:
 * device arrays of `world` destination pointers (peer-mapped for other ranks; anc_out NULL to
 * skip). The outputs whose ancestors live on this rank are written to their owners;
 * *m_key_next gets the atomicMax of the new log-weights written here; stats_out[2] (device
 * doubles) receives this rank's (sum exp(lw - M), sum exp(2 (lw - M))) of population t. */
CUPPL_API int cuppl_smc_resample(const cuppl_smc_model* m, uint64_t n_local, uint64_t n_total,
                                 uint64_t key, uint32_t t, int rank, int world, float y_cur,
                                 float y_next, const uint8_t* x, const int32_t* m_key,
                                 const uint64_t* rank_recs, const uint64_t* rank_begin,
                                 uint8_t* const* x_out, uint64_t* const* anc_out,
                                 int32_t* m_key_next, double* stats_out, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* lw[i] = log N(y; mu[x[i]], sd) (the per-particle log-weights of a population). */
CUPPL_API int cuppl_smc_log_weights(const cuppl_smc_model* m, float y, const uint8_t* x, uint64_t n,
                                    float* lw, void* stream);

/* Statistics of a population that is not resampled (the last step): stats_out[2] as in
 * cuppl_smc_resample, from the per-tile sums of the preceding cuppl_smc_scan. */
CUPPL_API int cuppl_smc_fold(uint64_t n_local, double* stats_out, void* workspace,
                             size_t workspace_bytes, void* stream);

/* ---- K3: normalize / empirical-posterior histogram and mode ------------ */
/* lw[n] (device, fp64 or fp32) and bin[n] (device int32 value ids, NULL = all 0) ->
 *   bins[n_bins] (device u64): sum over the bin of floor(exp(lw - M) 2^s), s = *scale_bits
 *     (host int, set by the call: 62 - ceil(log2 n), so sums never overflow);
 *   out[6] (device fp64): M = max finite lw (-inf if none), sum exp(2 (lw - M)), argmax lw,
 *     argmax index (u64 bits), number of finite lw (u64 bits), 0.
 * Integer bin sums make the result independent of the reduction order. */
CUPPL_API size_t cuppl_normalize_workspace_bytes(void);
CUPPL_API int cuppl_normalize_f64(const double* lw, const int32_t* bin, uint64_t n, int n_bins,
                                  uint64_t* bins, double* out, int* scale_bits, void* workspace,
                                  size_t workspace_bytes, void* stream);
CUPPL_API int cuppl_normalize_f32(const float* lw, const int32_t* bin, uint64_t n, int n_bins,
                                  uint64_t* bins, double* out, int* scale_bits, void* workspace,
                                  size_t workspace_bytes, void* stream);

/* ---- K7: many-chain lightweight Metropolis-Hastings (replaces run_lmh) -- */
/* Gaussian mixture: mu_k ~ normal(0, prior_sd), k < K <= 7;
 * z_i ~ categorical(1/K, ...); observe(normal(mu[z_i], sigma), y_i), i < D. One warp per chain;
 * each step picks one of the K + D sites uniformly, redraws it from its prior, re-executes the
 * model (full log-likelihood) and accepts with log a = l' - l.
 * chains [chain_begin, chain_begin + n_chains) (global ids, Philox counter word 0).
 * y: DEVICE pointer to cuppl_mh_padded_points(D) floats (data then zeros). Outputs (device):
 * mu_out [n_chains][K],
 * ll_out [n_chains], stats_out [n_chains][2K + 2] = sum of sorted mu, sum of sorted mu^2,
 * recorded steps, accepted steps; trace_out [n_chains][n_rec][K] optional (NULL to skip). */
CUPPL_API int cuppl_mh_padded_points(int D);
CUPPL_API int cuppl_mh_gmm(const float* y, int D, int K, float prior_sd, float sigma,
                           uint32_t n_chains, uint32_t chain_begin, uint32_t n_steps,
                           uint32_t burn_in, uint32_t thin, uint64_t key, float* mu_out,
                           float* ll_out, double* stats_out, float* trace_out, uint32_t n_rec,
                           void* stream);

/* ---- shareable device arenas (multi-process SMC peer stores) ----------------------------- */
/* cudaMalloc'd arena owned by the caller (free with cuppl_arena_free); its 64-byte IPC handle
 * (cuppl_ipc_handle) is exchanged between ranks, which map it with cuppl_ipc_open (NVLink peer
 * access enabled lazily) and unmap it with cuppl_ipc_close. */
#define CUPPL_IPC_HANDLE_BYTES 64
CUPPL_API int cuppl_arena_alloc(size_t bytes, void** ptr);
CUPPL_API int cuppl_arena_free(void* ptr);
CUPPL_API int cuppl_ipc_handle(const void* arena, void* handle_out);
CUPPL_API int cuppl_ipc_open(const void* handle, void** ptr);
CUPPL_API int cuppl_ipc_close(void* ptr);

/* ---- roofline calibration ---------------------------------------------------------- */
/* Pipe-rate microbenchmark, blocks x 256 threads, each thread runs `iters` iterations of:
 * kind 0: 128 FFMA2 (256 fp32 FMA), kind 1: 128 FFMA, kind 2: one Philox4x32-10 block,
 * kind 3: 32 MUFU.EX2 + 32 MUFU.LG2; kinds 4..8: 16 "points" of the linear-regression inner
 * loop on 8 particles (4: FADD2+2 FFMA2, 5: 3 FFMA2, 6: scalar FADD+2 FFMA, 7: 2 FADD2 chain,
 * 8: 2 FADD chain). `sink` is a device float[256] (never written in practice). */
CUPPL_API int cuppl_calibrate(int kind, int blocks, int iters, float* sink, void* stream);

/* Host-side ordered merge of n records (rank order). Pure host function. */
CUPPL_API int cuppl_is_record_merge(const cuppl_is_record* recs, int n, cuppl_is_record* out);

/* ---------------------------------------------------------------- generic resampling --------
 * Systematic resampling of ANY population (BASELINE north_star "resampling
 * and ancestor gather"): N particles with fp32 log-weights lw[N] and a fixed-size payload of
 * payload_bytes per particle (the particle state, opaque to the library). The reference has no
 * SMC (a non-goal), so oracle/resample_oracle.c or_resample DEFINES the result,
 * with the exact integer rule of SURVEY.md Appendix A D6 that cuppl_smc_resample applies to
 * HMM populations:
 *   M = max lw (NaN ignored), w_i = min(floor(exp(lw_i - M) 2^31), 2^31) (reproducible fp32 exp),
 *   C = inclusive u64 prefix of w, T = C[N-1], u = word 0 of Philox(key; t, 0, 0, CUPPL_TAG_SMC_COMB),
 *   target_j = floor((j 2^32 + u) T / (N 2^32)), a_j = min{i : C_i > target_j},
 *   payload_out[j] = payload[a_j], ancestors_out[j] = a_j.
 * Ancestors are bit-exact for any weights; stats are written to device memory: max_lw = M,
 * total = T (0 means every weight quantised to 0 and nothing else was written: the caller
 * raises AllZeroWeightError), sum_e / sum_e2 = sum and sum of squares of exp(lw - M) (fp64;
 * ESS = sum_e^2 / sum_e2, log-evidence increment = M + ln(sum_e / N)).
 * Requirements: 1 <= n < 2^31; lw, payload and payload_out 16-byte aligned (PyTorch allocations
 * are); payload may be NULL with payload_bytes == 0 (ancestors only); ancestors_out may be NULL.
 * The workspace (cuppl_resample_workspace_bytes) needs no initialisation. */
typedef struct cuppl_resample_stats {
  double max_lw;
  uint64_t total;
  double sum_e;
  double sum_e2;
} cuppl_resample_stats;

CUPPL_API size_t cuppl_resample_workspace_bytes(uint64_t n);
CUPPL_API int cuppl_resample(const float* lw, uint64_t n, const void* payload, uint64_t payload_bytes,
                             uint64_t key, uint32_t t, void* payload_out, uint64_t* ancestors_out,
                             cuppl_resample_stats* stats_out, void* workspace, size_t workspace_bytes,
                             void* stream);

/* ---------------------------------------------------------------- peer exchange -------------
 * The multi-rank SMC filter's two per-step collectives (all-reduce MAX of the
 * stabiliser, all-gather of the 32-byte rank records) over peer memory, in one kernel and
 * without the host: every rank's arena (cuppl_arena_alloc, CUDA-IPC mapped by the others)
 * holds a mailbox of `world` 64-byte slots at mbox_off and `world` u64 flags at flags_off (zero
 * on first use); peer_bases[q] is rank q's arena base as mapped here (device array). The call
 * writes this rank's payload (nbytes <= 64) into slot `rank` of every peer, releases flag
 * `rank` there with the next value of *epoch (a device counter per phase), waits for every
 * peer's flag, then writes the MAX of the int32 payloads to max_out and/or copies the world
 * payloads to gather_out [world][nbytes]. Stream-ordered and graph-capturable (the epoch lives
 * in device memory). A wait beyond timeout_ns sets *status to 1. Replaces the NCCL
 * all_reduce / all_gather of a multi-process run (smc.SmcRunner(exchange="peer")). */
CUPPL_API int cuppl_peer_exchange(const void* src, uint32_t nbytes, const uint64_t* peer_bases, uint64_t mbox_off,
                                  uint64_t flags_off, int rank, int world, uint64_t* epoch, int32_t* max_out,
                                  void* gather_out, uint32_t* status, uint64_t timeout_ns, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CUPPL_GPU_H */
