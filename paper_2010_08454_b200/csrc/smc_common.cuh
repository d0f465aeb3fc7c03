// smc_common.cuh — exact resampling arithmetic shared by the SMC kernels (K5/K6) and the
// generic resampling primitive (resample_kernels.cu): the reproducible exp and weight
// quantisation of SURVEY.md Appendix A D6 (bit-identical to oracle/cuppl_oracle.c or_smc_e /
// or_smc_w), ordered float keys for atomicMax, the decoupled look-back of the tile scan, and
// the integer comb (targets, exact 128-bit comparisons, fp64 rank estimates with exact fix-up).
#pragma once
#include "cuppl_device.cuh"

namespace cuppl {

// ------------------------------------------------------------------ exact helpers -------
// k = rint(t) by the 1.5 * 2^23 magic addition (round-half-even, exact for |t| < 2^22; here
// |t| <= 126): the same value as the oracle's rintf, and its integer is read from the sum's
// low bits — no FRND / F2I conversion-pipe instructions.
__device__ __forceinline__ float exp_repro(float d) {
  const float t = __fmul_rn(d, 1.44269504f);
  const float kb = __fadd_rn(t, 12582912.0f);
  const float k = __fsub_rn(kb, 12582912.0f);
  const int ki = __float_as_int(kb) - 0x4B400000;
  float r = __fmaf_rn(k, -0.693145752f, d);
  r = __fmaf_rn(k, -1.42860677e-06f, r);
  float p = 1.38888893e-03f;
  p = __fmaf_rn(p, r, 8.33333377e-03f);
  p = __fmaf_rn(p, r, 4.16666679e-02f);
  p = __fmaf_rn(p, r, 1.66666672e-01f);
  p = __fmaf_rn(p, r, 0.5f);
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  return __fmul_rn(p, __int_as_float((ki + 127) << 23));
}

// The same sequence on two values at once (fma.rn / add.rn / mul.rn .f32x2 round each lane as
// the scalar instructions do: bit-identical results, half the FMA-pipe instructions).
__device__ __forceinline__ f32x2 exp_repro2(float d0, float d1) {
  // the range reduction stays scalar: the packed add does not reproduce the scalar
  // round-half-even of the 1.5 * 2^23 magic addition at exact ties (measured)
  const float t0 = __fmul_rn(d0, 1.44269504f), t1 = __fmul_rn(d1, 1.44269504f);
  const float kb0 = __fadd_rn(t0, 12582912.0f), kb1 = __fadd_rn(t1, 12582912.0f);
  const f32x2 k = pack2(__fsub_rn(kb0, 12582912.0f), __fsub_rn(kb1, 12582912.0f));
  const int k0 = __float_as_int(kb0) - 0x4B400000, k1 = __float_as_int(kb1) - 0x4B400000;
  const f32x2 d = pack2(d0, d1);
  f32x2 r = fma2(k, pack2(-0.693145752f, -0.693145752f), d);
  r = fma2(k, pack2(-1.42860677e-06f, -1.42860677e-06f), r);
  f32x2 p = fma2(pack2(1.38888893e-03f, 1.38888893e-03f), r, pack2(8.33333377e-03f, 8.33333377e-03f));
  p = fma2(p, r, pack2(4.16666679e-02f, 4.16666679e-02f));
  p = fma2(p, r, pack2(1.66666672e-01f, 1.66666672e-01f));
  p = fma2(p, r, pack2(0.5f, 0.5f));
  p = fma2(p, r, pack2(1.0f, 1.0f));
  p = fma2(p, r, pack2(1.0f, 1.0f));
  return mul2(p, pack2(__int_as_float((k0 + 127) << 23), __int_as_float((k1 + 127) << 23)));
}

// e = exp(lw - M) for lw - M >= -87, else 0 (and 0 for lw = -inf / NaN): branch-free, the
// polynomial evaluated on the clamped difference and discarded outside the range (the same
// values as the oracle's or_smc_e)
__device__ __forceinline__ float smc_e(float lw, float M) {
  const float d = __fsub_rn(lw, M);
  const float e = exp_repro(fmaxf(d, -87.0f));
  return (lw > neg_inf_f() && d >= -87.0f) ? e : 0.0f;
}

// smc_e of two log-weights (exp_repro2)
__device__ __forceinline__ float2 smc_e2(float la, float lb, float M) {
  const float da = __fsub_rn(la, M), db = __fsub_rn(lb, M);
  const float2 e = unpack2(exp_repro2(fmaxf(da, -87.0f), fmaxf(db, -87.0f)));
  return make_float2((la > neg_inf_f() && da >= -87.0f) ? e.x : 0.0f, (lb > neg_inf_f() && db >= -87.0f) ? e.y : 0.0f);
}

__device__ __forceinline__ uint32_t smc_w(float e) {
  const uint32_t w = __float2uint_rz(__fmul_rn(e, 2147483648.0f));
  return w > 0x80000000u ? 0x80000000u : w;
}

// Monotone float <-> int key (signed compare == float compare), for atomicMax.
__device__ __forceinline__ int f2key(float f) {
  const int i = __float_as_int(f);
  return i ^ ((i >> 31) & 0x7FFFFFFF);
}
__device__ __forceinline__ float key2f(int k) { return __int_as_float(k ^ ((k >> 31) & 0x7FFFFFFF)); }

// ------------------------------------------------------------------ look-back -----------
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagIncl = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Warp-parallel decoupled look-back (Merrill & Garland): every lane inspects one predecessor
// per round; the window contributes up to the nearest inclusive prefix. Returns the exclusive
// prefix of `tile` (all lanes).
__device__ __forceinline__ unsigned long long warp_lookback(const unsigned long long* flags,
                                                            unsigned long long tile) {
  const int lane = threadIdx.x & 31;
  unsigned long long prefix = 0;
  long long k = static_cast<long long>(tile) - 1;
  while (k >= 0) {
    const long long idx = k - lane;
    const unsigned long long f = idx >= 0 ? ld_relaxed_u64(flags + idx) : kFlagIncl;
    const unsigned int st = static_cast<unsigned int>(f >> 62);
    const unsigned int incl = __ballot_sync(0xffffffffu, st == 2u);
    const int lim = incl ? __ffs(incl) - 1 : 31;  // lanes 0..lim contribute this round
    const unsigned int lim_mask = lim == 31 ? 0xffffffffu : ((2u << lim) - 1u);
    if (__ballot_sync(0xffffffffu, st == 0u) & lim_mask) continue;  // a predecessor is still running
    unsigned long long v = lane <= lim ? (f & kValMask) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    prefix += v;
    if (incl) break;
    k -= 32;
  }
  return prefix;
}

// Comb in integers (D6): with T = Q N + R0 and A = floor(u T / 2^32) = Qa N + Ra,
// target_j = floor((j 2^32 + u) T / (N 2^32)) = floor((j T + A) / N)
//          = j Q + Qa + floor((j R0 + Ra) / N),
// where j R0 + Ra < N^2 < 2^62 (N < 2^31); every per-index quantity fits 32 bits.
struct Comb {
  unsigned int N, Q, R0, Qa, Ra;
  unsigned long long T, A;
  double invN;              // 1 / N
  double n_over_t, a_over_t;  // N / T, A / T: fp64 rank estimates (exact fix-up below)
  unsigned int u;
};

// floor(num / N) for num < 2^62: fp64 estimate, exact correction.
__device__ __forceinline__ unsigned long long div_n(unsigned long long num, const Comb& cb,
                                                   unsigned int* rem) {
  long long q = static_cast<long long>(__dmul_rn(__ull2double_rn(num), cb.invN));
  long long r = static_cast<long long>(num) - q * static_cast<long long>(cb.N);
  while (r < 0) {
    --q;
    r += cb.N;
  }
  while (r >= static_cast<long long>(cb.N)) {
    ++q;
    r -= cb.N;
  }
  *rem = static_cast<unsigned int>(r);
  return static_cast<unsigned long long>(q);
}

__device__ __forceinline__ unsigned long long comb_target(unsigned int j, const Comb& cb) {
  unsigned int mod;
  const unsigned long long q = div_n(static_cast<unsigned long long>(j) * cb.R0 + cb.Ra, cb, &mod);
  return static_cast<unsigned long long>(j) * cb.Q + cb.Qa + q;
}

// target_j >= c  <=>  j T + A >= c N   (exact, 128-bit)
__device__ __forceinline__ bool comb_ge(unsigned int j, unsigned long long c, const Comb& cb) {
  const unsigned long long lo = static_cast<unsigned long long>(j) * cb.T;
  unsigned long long hi = __umul64hi(static_cast<unsigned long long>(j), cb.T);
  const unsigned long long lo2 = lo + cb.A;
  hi += lo2 < lo ? 1ull : 0ull;
  const unsigned long long rlo = c * cb.N;
  const unsigned long long rhi = __umul64hi(c, static_cast<unsigned long long>(cb.N));
  return hi > rhi || (hi == rhi && lo2 >= rlo);
}

// Rank of a weight coordinate in the comb: F(c) = min{j in [0, N] : target_j >= c}
// = clamp(ceil((c N - A) / T), 0, N). `est` is an fp64 estimate of (c N - A) / T with error
// < 2^-18; ceil(est) is exact unless est lies within 2^-14 of an integer, when the integer
// comparison decides (probability ~2^-13 per call: no divergence in practice).
static __device__ __noinline__ unsigned int comb_rank_exact(double est, unsigned long long c, const Comb& cb) {
  unsigned int j = est <= 0.0 ? 0u : est >= static_cast<double>(cb.N) ? cb.N
                                                                       : static_cast<unsigned int>(ceil(est));
  while (j > 0 && comb_ge(j - 1, c, cb)) --j;
  while (j < cb.N && !comb_ge(j, c, cb)) ++j;
  return j;
}
static __device__ __noinline__ unsigned int comb_rank_exact2(double est, unsigned long long c0, double cd,
                                                     const Comb& cb) {
  return comb_rank_exact(est, c0 + static_cast<unsigned long long>(cd), cb);
}
// Same, for the coordinate c0 + cd (cd an exact integer-valued double): the u64 coordinate is
// only formed on the rare exact path.
__device__ __forceinline__ unsigned int comb_rank(double est, unsigned long long c0, double cd,
                                                  const Comb& cb) {
  constexpr double kMagic = 6755399441055744.0;
  const double t = __dadd_ru(est, kMagic);
  const double frac = __dsub_rn(__dsub_rn(t, kMagic), est);
  unsigned int j = static_cast<unsigned int>(__double2loint(t));
  if (!(frac > 0x1p-14 && frac < 1.0 - 0x1p-14)) j = comb_rank_exact2(est, c0, cd, cb);
  return j;
}
__device__ __forceinline__ unsigned int comb_rank(double est, unsigned long long c, const Comb& cb) {
  // 1.5 * 2^52: doubles in [2^52, 2^53) are the integers, so for |est| < 2^51 rounding the sum
  // up gives 1.5 * 2^52 + ceil(est) exactly and its low word is ceil(est) (est > -1: >= 0)
  constexpr double kMagic = 6755399441055744.0;
  const double t = __dadd_ru(est, kMagic);
  const double frac = __dsub_rn(__dsub_rn(t, kMagic), est);  // ceil(est) - est, in [0, 1)
  unsigned int j = static_cast<unsigned int>(__double2loint(t));
  if (!(frac > 0x1p-14 && frac < 1.0 - 0x1p-14)) j = comb_rank_exact(est, c, cb);
  return j;
}
// The fast path alone: ceil(est), and whether the exact path must decide (callers batch the rare
// fix-ups after a loop instead of branching per source).
__device__ __forceinline__ unsigned int comb_rank_fast(double est, bool* exact) {
  constexpr double kMagic = 6755399441055744.0;
  const double t = __dadd_ru(est, kMagic);
  const double frac = __dsub_rn(__dsub_rn(t, kMagic), est);
  *exact = !(frac > 0x1p-14 && frac < 1.0 - 0x1p-14);
  return static_cast<unsigned int>(__double2loint(t));
}
__device__ __forceinline__ unsigned int comb_rank(unsigned long long c, const Comb& cb) {
  if (c == 0) return 0u;
  return comb_rank(__fma_rn(__ull2double_rn(c), cb.n_over_t, -cb.a_over_t), c, cb);
}

}  // namespace cuppl
