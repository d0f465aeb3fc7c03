/*
 * cuppl_oracle.c — CPU ORACLE for the CuPPL inference hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This file restates, in plain C and fp64, the reference
 * semantics the GPU library (paper_2010_08454_b200/csrc) implements. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may load it,
 * and only as the checker or the timed CPU baseline — never as the product path.
 *
 * What it restates (reference = /root/reference):
 *   - Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as 1, 2, 3";
 *     Random123 known-answer vectors are checked in tests/test_oracle.py) replacing the
 *     SplitMix keyed counter of pkg/src/cuppl/rng.py:16-45;
 *   - draw algorithms of pkg/src/cuppl/rng.py:43-117 on a Philox word stream;
 *   - dist_score of SPEC.md:312-320 and observe = factor(dist-score) (desugar.py:37-39);
 *   - run_importance / normalize of SPEC.md:399-407 / 417-425 (prior proposal, factor adds to
 *     the log-weight, log-sum-exp, ordered merge SPEC.md:449) for the Fig.1 polynomial model
 *      and Bayesian linear regression.
 * Parity status: Philox pinned by the Random123 KATs; distribution scores pinned by the SPEC
 * known-answer rows; the engines have no executable reference (the
 * reference ships no vm/infer) and are pinned by the SPEC engine KATs
 * and the closed-form posteriors in oracle/exact.py.
 *
 * Build: see oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define PH_M0 0xD2511F53u
#define PH_M1 0xCD9E8D57u
#define PH_W0 0x9E3779B9u
#define PH_W1 0xBB67AE85u

#define TAG_IS 1u
#define TAG_DIST 7u

/* ---------------------------------------------------------------- Philox4x32-10 ------- */
void or_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)PH_M0 * c0;
    const uint64_t p1 = (uint64_t)PH_M1 * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    const uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += PH_W0;
    k1 += PH_W1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static inline void block_of(uint64_t key, uint64_t id, uint32_t blk, uint32_t tag, uint32_t out[4]) {
  const uint32_t ctr[4] = {(uint32_t)id, (uint32_t)(id >> 32), blk, tag};
  const uint32_t k[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
  or_philox(ctr, k, out);
}

void or_philox_blocks(uint64_t key, uint64_t first_id, uint32_t block, uint32_t tag,
                      uint64_t count, uint32_t* out) {
  for (uint64_t i = 0; i < count; ++i) block_of(key, first_id + i, block, tag, out + 4 * i);
}

/* ---------------------------------------------------------------- transforms ---------- */
static inline float bits_f(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}
/* 23-bit uniforms from the mantissa, exact in both precisions */
double or_u01_open0(uint32_t w) { return 2.0 - (double)bits_f(0x3F800000u | (w >> 9)); }
double or_u01_closed0(uint32_t w) { return (double)bits_f(0x3F800000u | (w >> 9)) - 1.0; }

/* Lemire multiply-shift with exact rejection; returns 0 if w must be rejected */
/* the same on a b-bit word v < 2^b */
int or_lemire_bits(uint32_t v, uint32_t range, int bits, uint32_t* out) {
  const uint32_t m = v * range, mask = (1u << bits) - 1u;
  *out = m >> bits;
  const uint32_t lo = m & mask;
  if (lo < range) return lo >= ((1u << bits) % range);
  return 1;
}

int or_lemire(uint32_t w, uint32_t range, uint32_t* out) {
  const uint64_t m = (uint64_t)w * range;
  const uint32_t lo = (uint32_t)m;
  *out = (uint32_t)(m >> 32);
  if (lo < range) {
    const uint32_t t = (0u - range) % range;
    return lo >= t;
  }
  return 1;
}

/* u1 in (0, 1] from all 32 bits of wa: (wa + 1) 2^-32 (normals up to 6.66 sd); u2 in [0, 1)
 * from the top 23 bits of wb */
double or_u01_open0_32(uint32_t w) { return ((double)w + 1.0) * (1.0 / 4294967296.0); }

void or_box_muller(uint32_t wa, uint32_t wb, double* z0, double* z1) {
  const double u1 = or_u01_open0_32(wa), u2 = or_u01_closed0(wb);
  const double r = sqrt(-2.0 * log(u1));
  const double th = 2.0 * M_PI * u2;
  *z0 = r * cos(th);
  *z1 = r * sin(th);
}

/* ---------------------------------------------------------------- records ------------- */
/* Same field order as cuppl_is_record (include/cuppl_gpu.h), restated here. */
typedef struct or_record {
  double max_lw, sum_w, sum_w2, argmax_lw;
  uint64_t argmax_pid, n_finite, n_total, reserved;
  double stat_w[16];
  double bin_w[8];
} or_record;

static void rec_init(or_record* r) {
  memset(r, 0, sizeof(*r));
  r->max_lw = -INFINITY;
  r->argmax_lw = -INFINITY;
  r->argmax_pid = ~0ull;
}

/* online ordered accumulation of one particle (fp64) */
static void rec_add(or_record* r, double lw, uint64_t pid, const double* f, int nf, int bin) {
  r->n_total++;
  if (!isfinite(lw)) return;
  r->n_finite++;
  if (lw > r->argmax_lw || (lw == r->argmax_lw && pid < r->argmax_pid)) {
    r->argmax_lw = lw;
    r->argmax_pid = pid;
  }
  if (lw > r->max_lw) {
    const double s = exp(r->max_lw - lw);
    r->sum_w *= s;
    r->sum_w2 *= s * s;
    for (int k = 0; k < 16; ++k) r->stat_w[k] *= s;
    for (int k = 0; k < 8; ++k) r->bin_w[k] *= s;
    r->max_lw = lw;
  }
  const double w = exp(lw - r->max_lw);
  r->sum_w += w;
  r->sum_w2 += w * w;
  for (int k = 0; k < nf; ++k) r->stat_w[k] += w * f[k];
  if (bin >= 0 && bin < 8) r->bin_w[bin] += w;
}

void or_rec_merge(or_record* a, const or_record* b) {
  a->n_total += b->n_total;
  a->n_finite += b->n_finite;
  if (b->argmax_lw > a->argmax_lw || (b->argmax_lw == a->argmax_lw && b->argmax_pid < a->argmax_pid)) {
    a->argmax_lw = b->argmax_lw;
    a->argmax_pid = b->argmax_pid;
  }
  if (b->n_finite == 0) return;
  if (a->n_finite == b->n_finite) {
    a->max_lw = b->max_lw;
    a->sum_w = b->sum_w;
    a->sum_w2 = b->sum_w2;
    memcpy(a->stat_w, b->stat_w, sizeof(a->stat_w));
    memcpy(a->bin_w, b->bin_w, sizeof(a->bin_w));
    return;
  }
  const double m = a->max_lw > b->max_lw ? a->max_lw : b->max_lw;
  const double fa = exp(a->max_lw - m), fb = exp(b->max_lw - m);
  a->max_lw = m;
  a->sum_w = a->sum_w * fa + b->sum_w * fb;
  a->sum_w2 = a->sum_w2 * fa * fa + b->sum_w2 * fb * fb;
  for (int k = 0; k < 16; ++k) a->stat_w[k] = a->stat_w[k] * fa + b->stat_w[k] * fb;
  for (int k = 0; k < 8; ++k) a->bin_w[k] = a->bin_w[k] * fa + b->bin_w[k] * fb;
}

/* ---------------------------------------------------------------- Fig.1 polynomial ---- */
/* One Philox block per particle (csrc/is_kernels.cu poly_draw): (c0, c1) = 10 BM(w0, w1),
 * (c2, c3) = 10 BM(w2, w3) (normal(0, 10), D2; radius uniforms from all 32 bits of w0 / w2,
 * angles from the top 23 bits of w1 / w3); n ~ uniform-discrete(2,5) (support [2,5), D1) by
 * Lemire on the 18-bit v = w1[8:0] | w3[8:0] << 9 (the bits the angle uniforms do not use); a
 * rejected v is redrawn from word 0 of blocks 1, 2, ... (32-bit Lemire) */
uint32_t or_poly_degree_word(const uint32_t w[4]) {
  return (w[1] & 0x1FFu) | ((w[3] & 0x1FFu) << 9);
}

void or_poly_draw(uint64_t key, uint64_t pid, int* n, double c[4]) {
  uint32_t b0[4], k;
  block_of(key, pid, 0, TAG_IS, b0);
  if (!or_lemire_bits(or_poly_degree_word(b0), 3u, 18, &k)) {
    for (uint32_t blk = 1;; ++blk) {
      uint32_t bb[4];
      block_of(key, pid, blk, TAG_IS, bb);
      if (or_lemire(bb[0], 3u, &k)) break;
    }
  }
  *n = 2 + (int)k;
  double z0, z1, z2, z3;
  or_box_muller(b0[0], b0[1], &z0, &z1);
  or_box_muller(b0[2], b0[3], &z2, &z3);
  c[0] = 10.0 * z0;
  c[1] = 10.0 * z1;
  c[2] = *n > 2 ? 10.0 * z2 : 0.0;
  c[3] = *n > 3 ? 10.0 * z3 : 0.0;
}

/* factor(-distance(c, data)), distance = sum_i (y_i - sum_{j<n} c_j x_i^j)^2 (D3) */
double or_poly_lw(int n, const double* c, const float* xs, const float* ys, int D) {
  double acc = 0.0;
  for (int i = 0; i < D; ++i) {
    const double x = xs[i];
    double p = 0.0;
    for (int j = n - 1; j >= 0; --j) p = p * x + c[j];
    const double r = (double)ys[i] - p;
    acc += r * r;
  }
  return -acc;
}

static void poly_particle(const float* xs, const float* ys, int D, uint64_t key, uint64_t pid,
                          const float* inj, int* n, double c[4], double* lw) {
  if (inj) {
    *n = (int)inj[0];
    for (int j = 0; j < 4; ++j) c[j] = j < *n ? (double)inj[1 + j] : 0.0;
  } else {
    or_poly_draw(key, pid, n, c);
  }
  *lw = or_poly_lw(*n, c, xs, ys, D);
}

static int n_threads(int want) {
#ifdef _OPENMP
  return want > 0 ? want : omp_get_max_threads();
#else
  (void)want;
  return 1;
#endif
}

/* run_importance over global ids [pid_begin, pid_end): contiguous chunks per thread, chunk
 * records merged in chunk order. Optional traces (NULL to skip). */
int or_is_poly(const float* xs, const float* ys, int D, uint64_t pid_begin, uint64_t pid_end,
               uint64_t key, const float* injected, double* lw_out, int32_t* deg_out,
               double* coef_out, or_record* out, int threads) {
  const uint64_t N = pid_end - pid_begin;
  const int T = n_threads(threads);
  or_record* parts = (or_record*)malloc(sizeof(or_record) * (size_t)T);
  if (!parts) return 1;
#pragma omp parallel num_threads(T)
  {
#ifdef _OPENMP
    const int t = omp_get_thread_num();
#else
    const int t = 0;
#endif
    const uint64_t lo = N * (uint64_t)t / (uint64_t)T, hi = N * (uint64_t)(t + 1) / (uint64_t)T;
    or_record r;
    rec_init(&r);
    for (uint64_t i = lo; i < hi; ++i) {
      int n;
      double c[4], lw;
      poly_particle(xs, ys, D, key, pid_begin + i, injected ? injected + 5 * i : NULL, &n, c, &lw);
      double f[9] = {0};
      if (n == 2) { f[0] = c[0]; f[1] = c[1]; }
      else if (n == 3) { f[2] = c[0]; f[3] = c[1]; f[4] = c[2]; }
      else { f[5] = c[0]; f[6] = c[1]; f[7] = c[2]; f[8] = c[3]; }
      rec_add(&r, lw, pid_begin + i, f, 9, n - 2);
      if (lw_out) lw_out[i] = lw;
      if (deg_out) deg_out[i] = n;
      if (coef_out) for (int j = 0; j < 4; ++j) coef_out[4 * i + j] = c[j];
    }
    parts[t] = r;
  }
  rec_init(out);
  for (int t = 0; t < T; ++t) or_rec_merge(out, &parts[t]);
  free(parts);
  return 0;
}

/* ---------------------------------------------------------------- linear regression --- */
void or_linreg_draw(uint64_t key, uint64_t pid, double* a, double* b) {
  uint32_t w[4];
  block_of(key, pid, 0, TAG_IS, w);
  double z0, z1;
  or_box_muller(w[0], w[1], &z0, &z1);
  *a = 10.0 * z0;
  *b = 10.0 * z1;
}

/* sum_i dist_score(normal(a x_i + b, sigma), y_i) (desugar.py:37-39) */
double or_linreg_lw(double a, double b, const float* xs, const float* ys, int D, double sigma) {
  double acc = 0.0;
  const double c = -log(sigma) - 0.5 * log(2.0 * M_PI);
  for (int i = 0; i < D; ++i) {
    const double z = ((double)ys[i] - (a * (double)xs[i] + b)) / sigma;
    acc += -0.5 * z * z + c;
  }
  return acc;
}

int or_is_linreg(const float* xs, const float* ys, int D, double sigma, uint64_t pid_begin,
                 uint64_t pid_end, uint64_t key, const float* injected, double* lw_out,
                 double* coef_out, or_record* out, int threads) {
  const uint64_t N = pid_end - pid_begin;
  const int T = n_threads(threads);
  or_record* parts = (or_record*)malloc(sizeof(or_record) * (size_t)T);
  if (!parts) return 1;
#pragma omp parallel num_threads(T)
  {
#ifdef _OPENMP
    const int t = omp_get_thread_num();
#else
    const int t = 0;
#endif
    const uint64_t lo = N * (uint64_t)t / (uint64_t)T, hi = N * (uint64_t)(t + 1) / (uint64_t)T;
    or_record r;
    rec_init(&r);
    for (uint64_t i = lo; i < hi; ++i) {
      double a, b;
      if (injected) {
        a = injected[2 * i];
        b = injected[2 * i + 1];
      } else {
        or_linreg_draw(key, pid_begin + i, &a, &b);
      }
      const double lw = or_linreg_lw(a, b, xs, ys, D, sigma);
      const double f[5] = {a, b, a * a, b * b, a * b};
      rec_add(&r, lw, pid_begin + i, f, 5, -1);
      if (lw_out) lw_out[i] = lw;
      if (coef_out) { coef_out[2 * i] = a; coef_out[2 * i + 1] = b; }
    }
    parts[t] = r;
  }
  rec_init(out);
  for (int t = 0; t < T; ++t) or_rec_merge(out, &parts[t]);
  free(parts);
  return 0;
}

/* ---------------------------------------------------------------- dist_sample --------- */
/* Word-stream restatement of dist_kernels.cu (consumption order identical). */
typedef struct {
  uint64_t key, id;
  uint32_t tag, blk;
  uint32_t buf[4];
  int pos;
  int has_spare;
  double spare;
} wstream;

static void ws_init(wstream* s, uint64_t key, uint64_t id, uint32_t tag) {
  s->key = key; s->id = id; s->tag = tag; s->blk = 0; s->pos = 4; s->has_spare = 0; s->spare = 0;
}
static uint32_t ws_next(wstream* s) {
  if (s->pos == 4) {
    block_of(s->key, s->id, s->blk++, s->tag, s->buf);
    s->pos = 0;
  }
  return s->buf[s->pos++];
}
/* the reference's u64 generator (rng.py:39-41): two consecutive Philox words, first word high,
 * and its algorithms verbatim on that stream (rng.py:43-71) */
static uint64_t ws_next_u64(wstream* s) {
  const uint64_t hi = ws_next(s);
  return (hi << 32) | ws_next(s);
}
static double ws_uniform(wstream* s) { return (double)(ws_next_u64(s) >> 11) * (1.0 / 9007199254740992.0); }
static double ws_uniform_pos(wstream* s) {
  double u;
  do { u = ws_uniform(s); } while (!(u > 0.0));
  return u;
}
static double ws_normal(wstream* s) {
  if (s->has_spare) { s->has_spare = 0; return s->spare; }
  const double u1 = ws_uniform_pos(s);
  const double u2 = ws_uniform(s);
  const double r = sqrt(-2.0 * log(u1));
  s->spare = r * sin(2.0 * M_PI * u2);
  s->has_spare = 1;
  return r * cos(2.0 * M_PI * u2);
}
static uint32_t ws_randint(wstream* s, uint32_t range) {
  const uint64_t n = range, limit = UINT64_MAX - (UINT64_MAX % n);
  for (;;) {
    const uint64_t r = ws_next_u64(s);
    if (r < limit) return (uint32_t)(r % n);
  }
}
static double ws_gamma(wstream* s, double shape) {
  double boost = 1.0;
  if (shape < 1.0) {
    const double u = ws_uniform_pos(s);
    boost = pow(u, 1.0 / shape);
    shape += 1.0;
  }
  const double d = shape - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * d);
  for (;;) {
    const double x = ws_normal(s);
    double v = 1.0 + c * x;
    if (v <= 0.0) continue;
    v = v * v * v;
    const double u = ws_uniform(s);
    if (u < 1.0 - 0.0331 * (x * x) * (x * x)) return d * v * boost;
    if (u > 0.0 && log(u) < 0.5 * x * x + d * (1.0 - v + log(v))) return d * v * boost;
  }
}
static int ws_poisson(wstream* s, double lam) {
  double stack[64];
  int sp = 0, total = 0;
  stack[sp++] = lam;
  while (sp > 0) {
    const double l = stack[--sp];
    if (l < 30.0) {
      const double limit = exp(-l);
      int k = 0;
      double p = ws_uniform(s);
      while (p > limit) { ++k; p *= ws_uniform(s); }
      total += k;
    } else {
      const double half = floor(l / 2.0);
      stack[sp++] = l - half;
      stack[sp++] = half;
    }
  }
  return total;
}

/* tag: CUPPL_DIST_* ; params p0, p1 ; out_f (continuous) or out_i (discrete) */
int or_dist_sample(int dtag, double p0, double p1, const uint64_t* table, int K, uint64_t key,
                   uint32_t tag, uint64_t first_id, uint64_t count, double* out_f, int32_t* out_i) {
  for (uint64_t i = 0; i < count; ++i) {
    wstream s;
    ws_init(&s, key, first_id + i, tag);
    switch (dtag) {
      case 0: out_f[i] = p0 + p1 * ws_normal(&s); break;
      case 1: out_i[i] = ws_uniform(&s) < p0 ? 1 : 0; break;
      case 2: out_i[i] = ws_poisson(&s, p0); break;
      case 3: out_i[i] = (int32_t)p0 + (int32_t)ws_randint(&s, (uint32_t)((int64_t)p1 - (int64_t)p0)); break;
      case 4: out_f[i] = p0 + (p1 - p0) * ws_uniform(&s); break;
      case 5: {
        const double x = ws_gamma(&s, p0), y = ws_gamma(&s, p1);
        out_f[i] = x / (x + y);
        break;
      }
      case 6: out_f[i] = -log(ws_uniform_pos(&s)) / p0; break;
      case 7: {
        const uint32_t w = ws_next(&s);
        int k = 0;
        while (k < K - 1 && !((uint64_t)w < table[k])) ++k;
        out_i[i] = k;
        break;
      }
      default: return 1;
    }
  }
  return 0;
}

/* ---------------------------------------------------------------- SMC (bootstrap PF) -- */
/* HMM bootstrap particle filter with integer-exact systematic resampling (SURVEY.md §8(d)
 * C4, Appendix A D6; SMC has no reference semantics — SPEC.md:455 lists it as a non-goal —
 * so this restatement *defines* it, bit for bit, for the GPU kernels of csrc/smc_kernels.cu).
 *
 *   x_0 ~ categorical(pi0); lw_t = log N(y_t; mu[x_t], sd) (fp32, fixed op sequence);
 *   w_i = floor(exp_repro(lw_i - M_t) * 2^31) (u32), M_t = max lw_t, C = inclusive u64 scan;
 *   comb: u = word0(Philox(t, 0, 0, TAG_SMC_COMB)),
 *         target_j = floor((j 2^32 + u) T / (N 2^32))  (exact, unsigned 128-bit), a_j = upper_bound(C, target_j);
 *   x_{t+1}[j] ~ categorical(A[x_t[a_j]]) (alias draw) with word (j & 3) of
 *                Philox(j >> 2, t + 1, TAG_SMC_STEP).
 * Categorical draws of the filter use alias tables (or_alias_build / or_alias_draw: O(1) per
 * draw); every step is exact integer or IEEE fp32 arithmetic without contraction, so CPU and
 * GPU agree bit for bit. */
#define TAG_SMC_INIT 2u
#define TAG_SMC_STEP 3u
#define TAG_SMC_COMB 4u

static inline float f_bits(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

float or_exp_repro(float d) {
  const float t = d * 1.44269504f;
  const float k = rintf(t);
  float r = fmaf(k, -0.693145752f, d);
  r = fmaf(k, -1.42860677e-06f, r);
  float p = 1.38888893e-03f;
  p = fmaf(p, r, 8.33333377e-03f);
  p = fmaf(p, r, 4.16666679e-02f);
  p = fmaf(p, r, 1.66666672e-01f);
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  return p * f_bits((uint32_t)((int)k + 127) << 23);
}

/* e = exp(lw - M) for lw - M >= -87 (else 0); w = min(floor(e 2^31), 2^31) */
float or_smc_e(float lw, float M) {
  if (!(lw > -INFINITY)) return 0.0f;
  const float d = lw - M;
  if (!(d >= -87.0f)) return 0.0f;
  return or_exp_repro(d);
}
uint32_t or_smc_w(float e) {
  const float x = e * 2147483648.0f;
  uint32_t w = (uint32_t)x;
  return w > 0x80000000u ? 0x80000000u : w;
}

float or_emission(float y, float mu, float inv_sd, float c) {
  const float z = (y - mu) * inv_sd;
  return fmaf(-0.5f * z, z, c);
}

/* Walker / Vose alias table with exact integer masses (SMC categorical draws): column k keeps
 * k when the coin (low 32 bits of w K) is below thr_k in [0, 2^32], else yields alias_k.
 * Entry layout: thr (bits 0..32) | alias << 40. Construction: m_k = floor(w_k / W * K * 2^32)
 * (left-fold W), the rounding deficit added to the first largest m_k, then small / large stacks
 * popped LIFO in index order — restated verbatim by paper_2010_08454_b200/dists.py. */
void or_alias_build(const double* w, int K, uint64_t* out) {
  if (K <= 0) return;
  const uint64_t unit = 1ull << 32;
  double total = 0.0;
  for (int k = 0; k < K; ++k) total += w[k];
  int64_t* m = (int64_t*)malloc(sizeof(int64_t) * K);
  int* small = (int*)malloc(sizeof(int) * K);
  int* large = (int*)malloc(sizeof(int) * K);
  uint64_t* thr = (uint64_t*)malloc(sizeof(uint64_t) * K);
  int* alias = (int*)malloc(sizeof(int) * K);
  int64_t sum = 0;
  int kmax = 0;
  for (int k = 0; k < K; ++k) {
    m[k] = (int64_t)floor(w[k] / total * K * 4294967296.0);
    sum += m[k];
  }
  for (int k = 1; k < K; ++k)
    if (m[k] > m[kmax]) kmax = k;
  m[kmax] += (int64_t)K * (int64_t)unit - sum;
  int ns = 0, nl = 0;
  for (int k = 0; k < K; ++k) {
    if (m[k] < (int64_t)unit) small[ns++] = k; else large[nl++] = k;
  }
  while (ns && nl) {
    const int sm = small[--ns], lg = large[--nl];
    thr[sm] = (uint64_t)m[sm];
    alias[sm] = lg;
    m[lg] -= (int64_t)unit - m[sm];
    if (m[lg] < (int64_t)unit) small[ns++] = lg; else large[nl++] = lg;
  }
  while (nl) { const int k = large[--nl]; thr[k] = unit; alias[k] = k; }
  while (ns) { const int k = small[--ns]; thr[k] = unit; alias[k] = k; }
  for (int k = 0; k < K; ++k) out[k] = thr[k] | ((uint64_t)alias[k] << 40);
  free(m); free(small); free(large); free(thr); free(alias);
}

int or_alias_draw(const uint64_t* tab, int K, uint32_t w) {
  const uint64_t p = (uint64_t)w * (uint64_t)K;
  const int col = (int)(p >> 32);
  const uint32_t coin = (uint32_t)p;
  const uint64_t e = tab[col];
  return (uint64_t)coin < (e & 0x1FFFFFFFFull) ? col : (int)(e >> 40);
}

int or_categorical(const uint64_t* thr, int K, uint32_t w) {
  int lo = 0, hi = K - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((uint64_t)w < thr[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}

/* D6: target_j = floor((j 2^32 + u) T / (N 2^32)), in [0, T) for j < N. */
uint64_t or_comb_target(uint64_t j, uint32_t u, uint64_t T, uint64_t N) {
  const unsigned __int128 x = ((unsigned __int128)((j << 32) | u)) * (unsigned __int128)T;
  return (uint64_t)(x / ((unsigned __int128)N << 32));
}

static inline uint32_t smc_word(uint64_t key, uint64_t j, uint32_t blk, uint32_t tag) {
  uint32_t b[4];
  block_of(key, j >> 2, blk, tag, b);
  return b[j & 3];
}

uint32_t or_comb_word(uint64_t key, uint32_t t) {
  uint32_t b[4];
  block_of(key, (uint64_t)t, 0, TAG_SMC_COMB, b);
  return b[0];
}

typedef struct or_smc_stats {
  float M;
  uint32_t status; /* 0 ok, 2 all-zero weights */
  uint64_t T;
  double s1, s2;
} or_smc_stats;

void or_smc_init(uint64_t N, uint64_t key, const uint64_t* alias_pi0, int S, const float* mu,
                 float y0, float inv_sd, float c, int32_t* x, float* lw) {
  for (uint64_t j = 0; j < N; ++j) {
    const int k = or_alias_draw(alias_pi0, S, smc_word(key, j, 0, TAG_SMC_INIT));
    x[j] = k;
    lw[j] = or_emission(y0, mu[k], inv_sd, c);
  }
}

/* Statistics of population t (max, integer total, s1 = sum e, s2 = sum e^2, optional integer
 * filtering histogram), then — when x_out != NULL — resample + propagate to t + 1. */
int or_smc_step(uint64_t N, uint64_t key, uint32_t t, const uint64_t* aliasA, int S,
                const float* mu, float y_next, float inv_sd, float c, const int32_t* x,
                const float* lw, int32_t* x_out, float* lw_out, uint64_t* anc,
                or_smc_stats* st, uint64_t* hist) {
  float M = -INFINITY;
  for (uint64_t i = 0; i < N; ++i)
    if (lw[i] > M) M = lw[i];
  uint64_t* C = (uint64_t*)malloc(sizeof(uint64_t) * (N ? N : 1));
  float* E = (float*)malloc(sizeof(float) * (N ? N : 1));
  if (!C || !E) { free(C); free(E); return 1; }
  /* per-particle weights in parallel; the prefix and the fp64 sums sequentially (fixed order) */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)N; ++i) {
    E[i] = M > -INFINITY ? or_smc_e(lw[i], M) : 0.0f;
    C[i] = or_smc_w(E[i]);
  }
  uint64_t T = 0;
  double s1 = 0.0, s2 = 0.0;
  if (hist) memset(hist, 0, sizeof(uint64_t) * (size_t)S);
  for (uint64_t i = 0; i < N; ++i) {
    const uint64_t w = C[i];
    const double e = (double)E[i];
    T += w;
    C[i] = T;
    s1 += e;
    s2 += e * e;
    if (hist) hist[x[i]] += w;
  }
  free(E);
  st->M = M;
  st->T = T;
  st->s1 = s1;
  st->s2 = s2;
  st->status = T == 0 ? 2 : 0;
  if (T == 0 || !x_out) { free(C); return T == 0 ? 2 : 0; }
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
    const int k = or_alias_draw(aliasA + (size_t)x[lo] * (size_t)S, S,
                                smc_word(key, j, t + 1, TAG_SMC_STEP));
    x_out[j] = k;
    lw_out[j] = or_emission(y_next, mu[k], inv_sd, c);
  }
  free(C);
  return 0;
}

/* ---------------------------------------------------------------- LMH chains (GMM) ---- */
/* Many independent single-site lightweight MH chains on
 * the Gaussian mixture of SURVEY.md §8(d) C3, restating csrc/mh_kernels.cu in fp64:
 * each step picks one of the K + D sites uniformly (Lemire on word 0 of Philox(chain, step, 0,
 * TAG_MH); rejected words redrawn from sub-blocks 1, 2, ...), proposes from the site's prior
 * (mean: normal(0, prior_sd) by Box-Muller on words 1, 2; label: Lemire on word 1), re-executes
 * the model (full log-likelihood) and accepts iff log(u) < l' - l with u = u01_open0(word 3)
 * (the resampled site's prior cancels with the proposal). */
#define TAG_MH 5u
#define TAG_MH_INIT 6u

static inline void mh_block(uint64_t key, uint32_t chain, uint32_t step, uint32_t sub, uint32_t tag,
                            uint32_t out[4]) {
  const uint32_t ctr[4] = {chain, step, sub, tag};
  const uint32_t k[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
  or_philox(ctr, k, out);
}

static double gmm_ll(const float* y, const int32_t* z, const double* mu, int D, double sigma) {
  double s = 0.0;
  for (int i = 0; i < D; ++i) {
    const double r = ((double)y[i] - mu[z[i]]) / sigma;
    s += -0.5 * r * r;
  }
  return s - D * (log(sigma) + 0.5 * log(2.0 * M_PI));
}

/* One chain. stats[2K + 2] as the GPU's; trace (optional) [n_rec][K]; mu_out[K]; returns ll. */
double or_mh_gmm_chain(const float* y, int D, int K, double prior_sd, double sigma, uint32_t chain,
                       uint32_t n_steps, uint32_t burn_in, uint32_t thin, uint64_t key,
                       double* mu_out, double* stats, double* trace, uint32_t n_rec,
                       int32_t* z_init_out, double* ll_init_out) {
  int32_t* z = (int32_t*)malloc(sizeof(int32_t) * (size_t)D);
  double mu[8] = {0};
  for (int i = 0; i < D; ++i) {
    uint32_t b[4], lab;
    mh_block(key, chain, (uint32_t)i >> 2, 0, TAG_MH_INIT, b);
    if (!or_lemire(b[i & 3], (uint32_t)K, &lab)) {
      for (uint32_t r = 2;; ++r) {
        uint32_t bb[4];
        mh_block(key, chain, (uint32_t)i, r, TAG_MH_INIT, bb);
        if (or_lemire(bb[0], (uint32_t)K, &lab)) break;
      }
    }
    z[i] = (int32_t)lab;
  }
  for (int k = 0; k < K; ++k) {
    uint32_t b[4];
    double z0, z1, z2, z3;
    mh_block(key, chain, (uint32_t)k >> 2, 1, TAG_MH_INIT, b);
    or_box_muller(b[0], b[1], &z0, &z1);
    or_box_muller(b[2], b[3], &z2, &z3);
    const double zz[4] = {z0, z1, z2, z3};
    mu[k] = prior_sd * zz[k & 3];
  }
  if (z_init_out) memcpy(z_init_out, z, sizeof(int32_t) * (size_t)D);
  double ll = gmm_ll(y, z, mu, D, sigma);
  if (ll_init_out) *ll_init_out = ll;
  memset(stats, 0, sizeof(double) * (size_t)(2 * K + 2));
  const uint32_t n_sites = (uint32_t)(K + D);
  uint32_t rec = 0;
  for (uint32_t s = 0; s < n_steps; ++s) {
    uint32_t b[4], site = 0, zp = 0;
    mh_block(key, chain, s, 0, TAG_MH, b);
    if (!or_lemire(b[0], n_sites, &site)) {
      for (uint32_t r = 1;; ++r) {
        uint32_t bb[4];
        mh_block(key, chain, s, r, TAG_MH, bb);
        if (or_lemire(bb[0], n_sites, &site)) break;
      }
    }
    double old = 0.0;
    int32_t oldz = 0;
    if (site < (uint32_t)K) {
      double z0, z1;
      or_box_muller(b[1], b[2], &z0, &z1);
      old = mu[site];
      mu[site] = prior_sd * z0;
    } else {
      if (!or_lemire(b[1], (uint32_t)K, &zp)) {
        for (uint32_t r = 1;; ++r) {
          uint32_t bb[4];
          mh_block(key, chain, s, r, TAG_MH, bb);
          if (or_lemire(bb[1], (uint32_t)K, &zp)) break;
        }
      }
      oldz = z[site - K];
      z[site - K] = (int32_t)zp;
    }
    const double llp = gmm_ll(y, z, mu, D, sigma);
    const double logu = log(or_u01_open0(b[3]));
    const int accept = logu < llp - ll;
    if (accept) {
      ll = llp;
      stats[2 * K + 1] += 1.0;
    } else if (site < (uint32_t)K) {
      mu[site] = old;
    } else {
      z[site - K] = oldz;
    }
    if (s >= burn_in && (s - burn_in) % thin == 0) {
      double srt[8];
      for (int k = 0; k < K; ++k) {
        const double v = mu[k];
        int q = k;
        while (q > 0 && srt[q - 1] > v) { srt[q] = srt[q - 1]; --q; }
        srt[q] = v;
      }
      for (int k = 0; k < K; ++k) {
        stats[k] += srt[k];
        stats[K + k] += srt[k] * srt[k];
        if (trace && rec < n_rec) trace[(size_t)rec * K + k] = srt[k];
      }
      stats[2 * K] += 1.0;
      ++rec;
    }
  }
  for (int k = 0; k < K; ++k) mu_out[k] = mu[k];
  free(z);
  return ll;
}

/* n_chains chains [chain_begin, +n) in parallel (OpenMP); outputs per chain as the GPU's. */
int or_mh_gmm(const float* y, int D, int K, double prior_sd, double sigma, uint32_t n_chains,
              uint32_t chain_begin, uint32_t n_steps, uint32_t burn_in, uint32_t thin, uint64_t key,
              double* mu_out, double* ll_out, double* stats_out, int threads) {
  const int T = n_threads(threads);
#pragma omp parallel for num_threads(T) schedule(dynamic, 1)
  for (int64_t c = 0; c < (int64_t)n_chains; ++c) {
    ll_out[c] = or_mh_gmm_chain(y, D, K, prior_sd, sigma, chain_begin + (uint32_t)c, n_steps, burn_in,
                                thin, key, mu_out + (size_t)c * K, stats_out + (size_t)c * (2 * K + 2),
                                NULL, 0, NULL, NULL);
  }
  return 0;
}
