// dsl_lanes.cuh — lane-polymorphic value types for runtime-compiled model kernels (frontend.py).
//
// The model compiler emits one body text in terms of VF / VI / VB (real, int, bool), VF2 (a
// packed pair of reals) and helpers (sel, to_f, to_i, to_b, ud_draw, ...). With LANES == 1
// these are the plain scalar types and functions: one particle per thread. With LANES == P > 1
// every particle-dependent value is a Lane<T> holding P particles of the same thread and every
// operation is applied lane by lane, fully unrolled, so the P particles' instruction streams
// interleave (ILP) and each uniform operand — a data element read from the constant bank, a
// loop index — is loaded once for all P particles, as the hand-written kernels do with their P
// particles per thread (is_kernels.cu). Control flow on a lane value (`if (Lane<bool>)`, a loop
// bound that differs per particle) has no conversion and fails to compile: the host then
// compiles the same text with LANES == 1.
#pragma once
#include "draws.cuh"

#ifndef LANES
#define LANES 1
#endif
#ifndef MAXD
#error "define MAXD (the per-particle draw-record width) before including dsl_lanes.cuh"
#endif

namespace cuppl {

template <bool B, class T = void>
struct enable_if_ {};
template <class T>
struct enable_if_<true, T> {
  typedef T type;
};

template <class T>
struct Lane {
  T v[LANES];
  Lane() = default;
  __device__ __forceinline__ Lane(const T& x) {
#pragma unroll
    for (int p = 0; p < LANES; ++p) v[p] = x;
  }
  template <class U>
  __device__ __forceinline__ Lane(const Lane<U>& o) {
#pragma unroll
    for (int p = 0; p < LANES; ++p) v[p] = static_cast<T>(o.v[p]);
  }
  template <class U>
  __device__ __forceinline__ Lane& operator+=(const U& o);
};

template <class T>
struct is_lane {
  static constexpr bool v = false;
};
template <class T>
struct is_lane<Lane<T>> {
  static constexpr bool v = true;
};
template <class... A>
struct any_lane {
  static constexpr bool v = (is_lane<A>::v || ...);
};

template <class T>
__device__ __forceinline__ const T& lane_at(const T& x, int) {
  return x;
}
template <class T>
__device__ __forceinline__ const T& lane_at(const Lane<T>& x, int p) {
  return x.v[p];
}
template <class T>
__device__ __forceinline__ T& lane_ref(T& x, int) {
  return x;
}
template <class T>
__device__ __forceinline__ T& lane_ref(Lane<T>& x, int p) {
  return x.v[p];
}

template <class T>
template <class U>
__device__ __forceinline__ Lane<T>& Lane<T>::operator+=(const U& o) {
#pragma unroll
  for (int p = 0; p < LANES; ++p) v[p] += lane_at(o, p);
  return *this;
}

// f(lanes...) = Lane{ f(lane 0 of each argument), ..., f(lane P-1 ...) }; scalars broadcast
#define CUPPL_LIFT(fn)                                                                      \
  template <class... A, class = typename enable_if_<any_lane<A...>::v>::type>               \
  __device__ __forceinline__ auto fn(const A&... a) {                                       \
    Lane<decltype(fn(lane_at(a, 0)...))> r;                                                 \
    _Pragma("unroll") for (int p = 0; p < LANES; ++p) r.v[p] = fn(lane_at(a, p)...);       \
    return r;                                                                               \
  }

#define CUPPL_LANE_BINOP(op)                                                                \
  template <class A, class B, class = typename enable_if_<any_lane<A, B>::v>::type>         \
  __device__ __forceinline__ auto operator op(const A& a, const B& b) {                     \
    Lane<decltype(lane_at(a, 0) op lane_at(b, 0))> r;                                       \
    _Pragma("unroll") for (int p = 0; p < LANES; ++p) r.v[p] = lane_at(a, p) op lane_at(b, p); \
    return r;                                                                               \
  }

CUPPL_LANE_BINOP(+)
CUPPL_LANE_BINOP(-)
CUPPL_LANE_BINOP(*)
CUPPL_LANE_BINOP(/)
CUPPL_LANE_BINOP(%)
CUPPL_LANE_BINOP(<)
CUPPL_LANE_BINOP(<=)
CUPPL_LANE_BINOP(>)
CUPPL_LANE_BINOP(>=)
CUPPL_LANE_BINOP(==)
CUPPL_LANE_BINOP(!=)
CUPPL_LANE_BINOP(&&)
CUPPL_LANE_BINOP(||)

template <class T>
__device__ __forceinline__ Lane<T> operator-(const Lane<T>& a) {
  Lane<T> r;
#pragma unroll
  for (int p = 0; p < LANES; ++p) r.v[p] = -a.v[p];
  return r;
}
__device__ __forceinline__ Lane<bool> operator!(const Lane<bool>& a) {
  Lane<bool> r;
#pragma unroll
  for (int p = 0; p < LANES; ++p) r.v[p] = !a.v[p];
  return r;
}

// ------------------------------------------------------------------ scalar helpers ------
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(int x) { return static_cast<float>(x); }
__device__ __forceinline__ float to_f(bool x) { return x ? 1.f : 0.f; }
__device__ __forceinline__ int to_i(float x) { return static_cast<int>(x); }
__device__ __forceinline__ int to_i(int x) { return x; }
__device__ __forceinline__ int to_i(bool x) { return x ? 1 : 0; }
__device__ __forceinline__ bool to_b(float x) { return x != 0.f; }
__device__ __forceinline__ bool to_b(int x) { return x != 0; }
__device__ __forceinline__ bool to_b(bool x) { return x; }
__device__ __forceinline__ float hsum2(f32x2 v) {
  const float2 t = unpack2(v);
  return t.x + t.y;
}
#ifdef CUPPL_F64
template <class A, class B>  // fp64 models: the common type, so a double branch is never narrowed
__device__ __forceinline__ auto sel_(bool c, const A& a, const B& b) -> decltype(true ? a : b) {
  return c ? a : b;
}
#else
template <class A, class B>
__device__ __forceinline__ A sel_(bool c, const A& a, const B& b) {
  return c ? a : static_cast<A>(b);
}
#endif

// pure select: both operands are already evaluated (they are side-effect free)
template <class C, class A, class B>
__device__ __forceinline__ auto sel(const C& c, const A& a, const B& b) {
  if constexpr (any_lane<C, A, B>::v) {
    Lane<decltype(sel_(lane_at(c, 0), lane_at(a, 0), lane_at(b, 0)))> r;
#pragma unroll
    for (int p = 0; p < LANES; ++p) r.v[p] = sel_(lane_at(c, p), lane_at(a, p), lane_at(b, p));
    return r;
  } else {
    return sel_(c, a, b);
  }
}

// the CUDA math builtins live in the global namespace: make them visible next to their lifts
using ::expf;
using ::logf;
using ::log1pf;
using ::sqrtf;
using ::fabsf;
using ::floorf;
using ::fmodf;
using ::powf;
using ::fmaf;
using ::fminf;

CUPPL_LIFT(to_f)
CUPPL_LIFT(to_i)
CUPPL_LIFT(to_b)
CUPPL_LIFT(hsum2)
CUPPL_LIFT(pack2)
CUPPL_LIFT(fma2)
CUPPL_LIFT(add2)
CUPPL_LIFT(mul2)
CUPPL_LIFT(expf)
CUPPL_LIFT(logf)
CUPPL_LIFT(log1pf)
CUPPL_LIFT(sqrtf)
CUPPL_LIFT(fabsf)
CUPPL_LIFT(floorf)
CUPPL_LIFT(fmodf)
CUPPL_LIFT(powf)
CUPPL_LIFT(fmaf)
CUPPL_LIFT(fminf)
CUPPL_LIFT(score_normal)
CUPPL_LIFT(score_bernoulli)
CUPPL_LIFT(score_poisson)
CUPPL_LIFT(score_uniform_discrete)
CUPPL_LIFT(score_uniform_continuous)
CUPPL_LIFT(score_beta)
CUPPL_LIFT(score_exponential)

// ------------------------------------------------------------------ masks --------------
// Particle-dependent control flow in lane form: a bounded loop `i < n` or an `if` with side
// effects opens a mask m (bool, or Lane<bool> when the condition differs per particle) and an
// `if (lanes_any(m))` block; inside it draws consume a lane's stream only where its mask bit
// is set, factors add sel(m, x, 0) and outer accumulators are updated as sel(m, new, old).
// With LANES == 1 (or a uniform condition) m is true inside its block and this is plain code.
__device__ __forceinline__ bool lanes_any(bool m) { return m; }

// var = x in the lanes of mask m (a per-lane predicated move, which ptxas folds into the
// instruction producing x) — the masked-update form of the generated code
template <class T, class M, class X>
__device__ __forceinline__ void masked_set(T& var, const M& m, const X& x) {
  if constexpr (is_lane<T>::v) {
#pragma unroll
    for (int p = 0; p < LANES; ++p)
      if (lane_at(m, p)) var.v[p] = lane_at(x, p);
  } else {
    if (lane_at(m, 0)) var = x;
  }
}
template <class T, class M, class X>
__device__ __forceinline__ void masked_add(T& var, const M& m, const X& x) {
  if constexpr (is_lane<T>::v) {
#pragma unroll
    for (int p = 0; p < LANES; ++p)
      if (lane_at(m, p)) var.v[p] += lane_at(x, p);
  } else {
    if (lane_at(m, 0)) var += x;
  }
}

// ------------------------------------------------------------------ draws --------------
// uniform-discrete(lo, hi): support [lo, hi); an empty range raises
// InvalidDistParamError on the host (err word) and draws from [lo, lo + 1)
// parameter checks: flag bit of the error word; the smallest failing particle id is kept in
// first_bad (reported with InvalidDistParamError)
__device__ __forceinline__ unsigned ud_check(bool valid, int lo, int hi, unsigned long long pid,
                                             unsigned long long& first_bad) {
  const bool bad = valid && !(hi > lo);
  if (bad && pid < first_bad) first_bad = pid;
  return bad ? 1u : 0u;
}
__device__ __forceinline__ int ud_draw1(WordStream& ws, int lo, int hi) {
  return lo + static_cast<int>(ws.randint(static_cast<unsigned>(hi > lo ? hi - lo : 1)));
}
// one-stream draws: the enclosing block already holds the mask
template <class M>
__device__ __forceinline__ int ud_draw(WordStream& ws, int lo, int hi, const M&) {
  return ud_draw1(ws, lo, hi);
}
template <class M>
__device__ __forceinline__ float draw_normal(WordStream& ws, const M&) { return ws.normal(); }
template <class M>
__device__ __forceinline__ float draw_uniform(WordStream& ws, const M&) { return ws.uniform(); }
template <class M>
__device__ __forceinline__ float draw_uniform_pos(WordStream& ws, const M&) { return ws.uniform_pos(); }
template <class M>
__device__ __forceinline__ float draw_gamma(WordStream& ws, float a, const M&) { return ws.gamma(a); }
// poisson(rate): rate must be finite, >= 0 and < 2^31 (int count); a bad lane draws with rate 0
__device__ __forceinline__ float pois_rate(float lam) { return (lam >= 0.f && lam < 2147483648.f) ? lam : 0.f; }
__device__ __forceinline__ unsigned pois_check(bool valid, float lam, unsigned long long pid,
                                               unsigned long long& first_bad) {
  const bool bad = valid && !(lam >= 0.f && lam < 2147483648.f);
  if (bad && pid < first_bad) first_bad = pid;
  return bad ? 4u : 0u;
}
template <class M>
__device__ __forceinline__ int draw_poisson(WordStream& ws, float lam, const M&) { return ws.poisson(pois_rate(lam)); }
// categorical(w): P(k) = w_k / sum w; weights must be >= 0 and not all 0
__device__ __forceinline__ unsigned cat_check(bool valid, float tot, float wmin, unsigned long long pid,
                                              unsigned long long& first_bad) {
  const bool bad = valid && !(tot > 0.f && wmin >= 0.f);
  if (bad && pid < first_bad) first_bad = pid;
  return bad ? 2u : 0u;
}
__device__ __forceinline__ float score_categorical(int k, int n, float wk, float tot) {
  return (k >= 0 && k < n && wk > 0.f) ? logf(wk / tot) : neg_inf_f();
}
CUPPL_LIFT(score_categorical)
__device__ __forceinline__ void store_draw(float* out, unsigned long long idx, bool valid, int nd, float x) {
  if (out && valid && nd < MAXD) out[idx * MAXD + nd] = x;
}

#if LANES > 1
// P particles' word streams of one thread: draw k of lane p is draw k of particle p's stream
struct LaneStream {
  WordStream s[LANES];
  __device__ __forceinline__ void init(PhiloxKey k, const Lane<unsigned long long>& id, uint32_t t) {
#pragma unroll
    for (int p = 0; p < LANES; ++p) s[p].init(k, id.v[p], t);
  }
};
__device__ __forceinline__ bool lanes_any(const Lane<bool>& m) {
  bool r = false;
#pragma unroll
  for (int p = 0; p < LANES; ++p) r = r || m.v[p];
  return r;
}
// lane p draws from its own stream only where its mask bit is set (0 elsewhere)
#define CUPPL_LANE_DRAW0(T, name, fn)                                                       \
  template <class M>                                                                        \
  __device__ __forceinline__ Lane<T> name(LaneStream& ws, const M& m) {                     \
    Lane<T> r;                                                                              \
    _Pragma("unroll") for (int p = 0; p < LANES; ++p) r.v[p] = lane_at(m, p) ? ws.s[p].fn() : T(0); \
    return r;                                                                               \
  }
#define CUPPL_LANE_DRAW1(T, name, fn)                                                       \
  template <class A, class M>                                                               \
  __device__ __forceinline__ Lane<T> name(LaneStream& ws, const A& a, const M& m) {         \
    Lane<T> r;                                                                              \
    _Pragma("unroll") for (int p = 0; p < LANES; ++p)                                       \
      r.v[p] = lane_at(m, p) ? ws.s[p].fn(lane_at(a, p)) : T(0);                             \
    return r;                                                                               \
  }
CUPPL_LANE_DRAW0(float, draw_normal, normal)
CUPPL_LANE_DRAW0(float, draw_uniform, uniform)
CUPPL_LANE_DRAW0(float, draw_uniform_pos, uniform_pos)
CUPPL_LANE_DRAW1(float, draw_gamma, gamma)
#define poisson_checked(lam) poisson(pois_rate(lam))
CUPPL_LANE_DRAW1(int, draw_poisson, poisson_checked)
#undef poisson_checked
#undef CUPPL_LANE_DRAW0
#undef CUPPL_LANE_DRAW1
template <class A, class B>
__device__ __forceinline__ unsigned ud_check(const Lane<bool>& valid, const A& lo, const B& hi,
                                             const Lane<unsigned long long>& pid,
                                             unsigned long long& first_bad) {
  unsigned e = 0u;
#pragma unroll
  for (int p = 0; p < LANES; ++p)
    e |= ud_check(valid.v[p], lane_at(lo, p), lane_at(hi, p), pid.v[p], first_bad);
  return e;
}
template <class T>
__device__ __forceinline__ unsigned pois_check(const Lane<bool>& valid, const T& lam,
                                               const Lane<unsigned long long>& pid,
                                               unsigned long long& first_bad) {
  unsigned e = 0u;
#pragma unroll
  for (int p = 0; p < LANES; ++p) e |= pois_check(valid.v[p], lane_at(lam, p), pid.v[p], first_bad);
  return e;
}
template <class T, class W>
__device__ __forceinline__ unsigned cat_check(const Lane<bool>& valid, const T& tot, const W& wmin,
                                              const Lane<unsigned long long>& pid,
                                              unsigned long long& first_bad) {
  unsigned e = 0u;
#pragma unroll
  for (int p = 0; p < LANES; ++p)
    e |= cat_check(valid.v[p], lane_at(tot, p), lane_at(wmin, p), pid.v[p], first_bad);
  return e;
}
template <class A, class B, class M>
__device__ __forceinline__ Lane<int> ud_draw(LaneStream& ws, const A& lo, const B& hi, const M& m) {
  Lane<int> r;
#pragma unroll
  for (int p = 0; p < LANES; ++p)
    r.v[p] = lane_at(m, p) ? ud_draw1(ws.s[p], lane_at(lo, p), lane_at(hi, p)) : 0;
  return r;
}
template <class N, class X>
__device__ __forceinline__ void store_draw(float* out, const Lane<unsigned long long>& idx,
                                           const Lane<bool>& valid, const N& nd, const X& x) {
#pragma unroll
  for (int p = 0; p < LANES; ++p) store_draw(out, idx.v[p], valid.v[p], lane_at(nd, p), to_f(lane_at(x, p)));
}
typedef Lane<float> VF;
typedef Lane<int> VI;
typedef Lane<bool> VB;
typedef Lane<f32x2> VF2;
typedef Lane<unsigned long long> VU64;
typedef LaneStream VStream;
#else
#ifdef CUPPL_F64
typedef double VF;
#else
typedef float VF;
#endif
typedef int VI;
typedef bool VB;
typedef f32x2 VF2;
typedef unsigned long long VU64;
typedef WordStream VStream;
#endif


#ifdef CUPPL_F64
// ------------------------------------------------------------------ fp64 models ---------
// Enumeration (frontend.py): path log-masses, factors and the record are fp64, and the body's
// real-valued helpers resolve to these forms (the generated source also maps the C math names
// logf, log1pf, fmaf, ... to their double functions). One path per thread.
#if LANES != 1
#error "fp64 models run one path per thread"
#endif
__device__ __forceinline__ double to_d(double x) { return x; }
__device__ __forceinline__ double to_d(float x) { return static_cast<double>(x); }
__device__ __forceinline__ double to_d(int x) { return static_cast<double>(x); }
__device__ __forceinline__ double to_d(bool x) { return x ? 1.0 : 0.0; }
__device__ __forceinline__ int to_i(double x) { return static_cast<int>(x); }
__device__ __forceinline__ bool to_b(double x) { return x != 0.0; }
__device__ __forceinline__ double neg_inf_d_() { return -__longlong_as_double(0x7FF0000000000000ll); }
__device__ __forceinline__ double score_normal_d(double x, double m, double sd) {
  const double z = (x - m) / sd;
  return -0.5 * z * z - log(sd) - 0.91893853320467274178032973640562;
}
__device__ __forceinline__ double score_bernoulli_d(bool v, double p) { return v ? log(p) : log1p(-p); }
__device__ __forceinline__ double score_poisson_d(int k, double lam) {
  return k < 0 ? neg_inf_d_() : (k == 0 ? 0.0 : k * log(lam)) - lam - lgamma(k + 1.0);
}
__device__ __forceinline__ double score_uniform_discrete_d(int k, int a, int b) {
  return (k >= a && k < b) ? -log(static_cast<double>(b - a)) : neg_inf_d_();
}
__device__ __forceinline__ double score_uniform_continuous_d(double x, double a, double b) {
  return (x >= a && x <= b) ? -log(b - a) : neg_inf_d_();
}
__device__ __forceinline__ double score_beta_d(double x, double a, double b) {
  return (x >= 0.0 && x <= 1.0)
             ? (a - 1.0) * log(x) + (b - 1.0) * log1p(-x) - (lgamma(a) + lgamma(b) - lgamma(a + b))
             : neg_inf_d_();
}
__device__ __forceinline__ double score_exponential_d(double x, double r) {
  return x >= 0.0 ? log(r) - r * x : neg_inf_d_();
}
__device__ __forceinline__ double score_categorical_d(int k, int n, double wk, double tot) {
  return (k >= 0 && k < n && wk > 0.0) ? log(wk / tot) : neg_inf_d_();
}
#define to_f to_d
#define score_normal score_normal_d
#define score_bernoulli score_bernoulli_d
#define score_poisson score_poisson_d
#define score_uniform_discrete score_uniform_discrete_d
#define score_uniform_continuous score_uniform_continuous_d
#define score_beta score_beta_d
#define score_exponential score_exponential_d
#define score_categorical score_categorical_d
#endif

}  // namespace cuppl
