// draws.cuh — per-particle word streams and the distribution scores, shared by the batch
// dist kernels (dist_kernels.cu) and the runtime-compiled model kernels (frontend.py, NVRTC).
//
// A WordStream replays the reference draw algorithms (pkg/src/cuppl/rng.py:43-117) on the
// Philox words of blocks (id, 0..), tag: one stream per particle plays the role of
// Rng.split(i) (rng.py:31-37), and successive sample sites consume it in program order. The
// reference's generator yields u64 words (rng.py:39-41); here next_u64() is two consecutive
// Philox words (first word high), and every algorithm is the reference's on that u64 stream:
// uniform = (x >> 11) 2^-53 (rng.py:43-45), randint = rejection below MASK - MASK % n then
// x % n (rng.py:47-56), normal = Box-Muller with u1 redrawn while 0 and the cached spare
// (rng.py:58-71), exponential / gamma / beta / poisson as rng.py:73-117. The integer decisions
// are exact (poisson's products of uniforms run in fp64, as in the reference; so do the batch
// path's gamma / beta / exponential); the other real-valued transforms run in fp32 (the oracle
// restates them in fp64 and
// equals oracle/refstream.Algorithms bit for bit on the same u64 stream, tests/test_oracle.py).
#pragma once
#include "cuppl_device.cuh"

namespace cuppl {

struct WordStream {
  PhiloxKey key;
  uint64_t id;
  uint32_t tag, blk;
  uint32_t b0, b1, b2, b3;  // the current block, in registers (no dynamically indexed array)
  int pos;
  double spare;  // the reference's one cached Box-Muller spare, shared by the fp32 and fp64 paths
  bool has_spare;

  __device__ __forceinline__ void init(PhiloxKey k, uint64_t i, uint32_t t) {
    key = k;
    id = i;
    tag = t;
    blk = 0;
    pos = 4;
    has_spare = false;
    spare = 0.0;
  }
  __device__ __forceinline__ uint32_t next() {
    if (pos == 4) {
      const uint4 b = draw_block(key, id, blk++, tag);
      b0 = b.x;
      b1 = b.y;
      b2 = b.z;
      b3 = b.w;
      pos = 0;
    }
    const uint32_t w = pos == 0 ? b0 : pos == 1 ? b1 : pos == 2 ? b2 : b3;
    ++pos;
    return w;
  }
  __device__ __forceinline__ unsigned long long next_u64() {
    const unsigned long long hi = next();
    return (hi << 32) | next();
  }
  // (x >> 11) 2^-53, rounded toward zero to fp32: in [0, 1) like the reference's double
  __device__ __forceinline__ float uniform() { return __ull2float_rz(next_u64() >> 11) * 0x1p-53f; }
  // the reference's `while u <= 0: u = uniform()` (rng.py:73-77, 79-85): in (0, 1)
  __device__ __forceinline__ float uniform_pos() {
    unsigned long long m;
    do {
      m = next_u64() >> 11;
    } while (m == 0ull);
    return __ull2float_rz(m) * 0x1p-53f;
  }
  __device__ __forceinline__ float normal() {  // rng.py:58-71
    if (has_spare) {
      has_spare = false;
      return static_cast<float>(spare);
    }
    const float u1 = uniform_pos();
    const float u2 = uniform();
    const float r = fast_sqrt(-2.0f * kLn2 * fast_lg2(u1));
    const float th = fmaf(kTwoPi, u2, -kPi);  // 2 pi u2 - pi in [-pi, pi): signs flipped below
    spare = static_cast<double>(-r * fast_sin(th));
    has_spare = true;
    return -r * fast_cos(th);
  }
  // ---- fp64 paths, the reference's arithmetic op for op (the oracle is built with
  // -ffp-contract=off: every product and sum below is rounded on its own, no FMA contraction)
  __device__ __forceinline__ double uniform_pos_d() {  // rng.py:73-77: (0, 1)
    double u;
    do {
      u = uniform_d();
    } while (!(u > 0.0));
    return u;
  }
  __device__ __forceinline__ double normal_d() {  // rng.py:58-71 in fp64
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    const double u1 = uniform_pos_d();
    const double u2 = uniform_d();
    const double r = sqrt(__dmul_rn(-2.0, log(u1)));
    // sin / cos(2 pi u2) as sincospi(2 u2): exact argument reduction without the local-memory
    // slow path (vs the reference's sin(fl(2 pi u2)): a relative difference ~1e-16)
    double sn, cs;
    sincospi(__dmul_rn(2.0, u2), &sn, &cs);
    spare = __dmul_rn(r, sn);
    has_spare = true;
    return __dmul_rn(r, cs);
  }
  __device__ __forceinline__ uint32_t randint(uint32_t range) {  // rng.py:47-56
    const unsigned long long n = range;
    const unsigned long long limit = ~0ull - (~0ull % n);
    for (;;) {
      const unsigned long long r = next_u64();
      if (r < limit) return static_cast<uint32_t>(r % n);
    }
  }
  // Marsaglia-Tsang (cuppl/rng.py:79-98) in fp64 like the reference (the batch dist_sample
  // path): the same acceptance decisions as the oracle (so the same words consumed), reals to
  // double rounding
  __device__ double gamma_d(double shape) {
    double boost = 1.0;
    if (shape < 1.0) {
      const double u = uniform_pos_d();
      boost = pow(u, __ddiv_rn(1.0, shape));
      shape = __dadd_rn(shape, 1.0);
    }
    const double d = __dsub_rn(shape, 1.0 / 3.0);
    const double c = __ddiv_rn(1.0, sqrt(__dmul_rn(9.0, d)));
    for (;;) {
      const double x = normal_d();
      double v = __dadd_rn(1.0, __dmul_rn(c, x));
      if (v <= 0.0) continue;
      v = __dmul_rn(__dmul_rn(v, v), v);
      const double u = uniform_d();
      const double x2 = __dmul_rn(x, x);
      if (u < __dsub_rn(1.0, __dmul_rn(__dmul_rn(0.0331, x2), x2))) return __dmul_rn(__dmul_rn(d, v), boost);
      if (u > 0.0 &&
          log(u) < __dadd_rn(__dmul_rn(__dmul_rn(0.5, x), x), __dmul_rn(d, __dadd_rn(__dsub_rn(1.0, v), log(v)))))
        return __dmul_rn(__dmul_rn(d, v), boost);
    }
  }
  // the fp32 version for compiled models (per-lane draws in registers; accurate logf for the
  // acceptance test): the same algorithm, decisions equal to the fp64 ones except on rare draws
  __device__ float gamma(float shape) {
    float boost = 1.0f;
    if (shape < 1.0f) {
      const float u = uniform_pos();
      boost = powf(u, 1.0f / shape);
      shape += 1.0f;
    }
    const float d = shape - 1.0f / 3.0f;
    const float c = 1.0f / sqrtf(9.0f * d);
    for (;;) {
      const float x = normal();
      float v = 1.0f + c * x;
      if (v <= 0.0f) continue;
      v = v * v * v;
      const float u = uniform();
      if (u < 1.0f - 0.0331f * (x * x) * (x * x)) return d * v * boost;
      if (u > 0.0f && logf(u) < 0.5f * x * x + d * (1.0f - v + logf(v))) return d * v * boost;
    }
  }
  // beta = X / (X + Y) (rng.py:100-103) and exponential = -ln(u) / rate (rng.py:73-77), in fp64
  __device__ float beta(float a, float b) {
    const double x = gamma_d(static_cast<double>(a));
    const double y = gamma_d(static_cast<double>(b));
    return static_cast<float>(__ddiv_rn(x, __dadd_rn(x, y)));
  }
  __device__ float exponential(float rate) {
    return static_cast<float>(__ddiv_rn(-log(uniform_pos_d()), static_cast<double>(rate)));
  }
  // the reference's 53-bit uniform as the double it is (exact: (x >> 11) 2^-53)
  __device__ __forceinline__ double uniform_d() {
    return static_cast<double>(next_u64() >> 11) * 0x1p-53;
  }
  // rng.py:105-117 in fp64 like the reference (products of uniforms against exp(-lambda),
  // halving above 30): the integer draws equal the oracle's, which is the reference algorithm
  __device__ int poisson(float lam) {
    // explicit DFS over the halving tree: same leaf order as the reference recursion
    double stack[64];
    int sp = 0;
    stack[sp++] = static_cast<double>(lam);
    int total = 0;
    while (sp > 0) {
      const double l = stack[--sp];
      if (l < 30.0) {
        const double limit = exp(-l);
        int k = 0;
        double p = uniform_d();
        while (p > limit) {
          ++k;
          p = __dmul_rn(p, uniform_d());
        }
        total += k;
      } else if (sp < 62) {  // rates are checked < 2^31 (<= 27 levels); never overflow the stack
        const double half = floor(l / 2.0);
        stack[sp++] = l - half;  // processed second
        stack[sp++] = half;      // processed first
      }
    }
    return total;
  }
};

// Natural-log density / mass; -inf outside the support.
// normal: z = (x - m) * (1 / sd) with a correctly rounded reciprocal (|dz| <= 1 ulp of a
// division); 1/sd and ln sd depend on sd only, so they leave a data loop when sd does not vary
__device__ __forceinline__ float score_normal(float x, float m, float sd) {
  const float z = (x - m) * __frcp_rn(sd);
  return fmaf(-0.5f * z, z, -logf(sd) - kHalfLog2Pi);
}
__device__ __forceinline__ float score_bernoulli(bool v, float p) { return v ? logf(p) : log1pf(-p); }
__device__ __forceinline__ float score_poisson(int k, float lam) {
  return k < 0 ? neg_inf_f() : (k == 0 ? 0.f : k * logf(lam)) - lam - lgammaf(k + 1.0f);
}
__device__ __forceinline__ float score_uniform_discrete(int k, int a, int b) {
  return (k >= a && k < b) ? -logf(static_cast<float>(b - a)) : neg_inf_f();
}
__device__ __forceinline__ float score_uniform_continuous(float x, float a, float b) {
  return (x >= a && x <= b) ? -logf(b - a) : neg_inf_f();
}
__device__ __forceinline__ float score_beta(float x, float a, float b) {
  return (x >= 0.f && x <= 1.f)
             ? (a - 1.f) * logf(x) + (b - 1.f) * log1pf(-x) - (lgammaf(a) + lgammaf(b) - lgammaf(a + b))
             : neg_inf_f();
}
__device__ __forceinline__ float score_exponential(float x, float r) {
  return x >= 0.f ? logf(r) - r * x : neg_inf_f();
}

}  // namespace cuppl
