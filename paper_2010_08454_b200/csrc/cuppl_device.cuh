// cuppl_device.cuh — K8 device library: Philox4x32-10, draw transforms, packed-fp32 helpers
// and the log-sum-exp record algebra shared by every kernel.
//
// Draw semantics follow the reference distributions (pkg/src/cuppl/rng.py:43-117,
// SPEC.md:303-329) with the generator replaced by Philox. The CPU
// oracle (oracle/cuppl_oracle.c) restates every transform here from the same u32 words.
#pragma once
#ifndef __CUDACC_RTC__
#include <cstdint>
#include <cuda_runtime.h>
#endif
#include "../../include/cuppl_gpu.h"

namespace cuppl {

// ---------------------------------------------------------------- Philox4x32-10 --------
constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

// One 128-bit block. The key schedule is computed inline; with a launch-uniform key the
// additions land on the uniform datapath. Each round is 2 IMAD.WIDE.U32 + 2 LOP3.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    // explicit 32x32 -> 64 multiplies (one IMAD.WIDE.U32 each) split into (lo, hi)
    uint32_t lo0, hi0, lo1, hi1;
    asm("{\n\t.reg .b64 p;\n\tmul.wide.u32 p, %2, %3;\n\tmov.b64 {%0, %1}, p;\n\t}"
        : "=r"(lo0), "=r"(hi0) : "r"(c.x), "n"(kPhiloxM0));
    asm("{\n\t.reg .b64 p;\n\tmul.wide.u32 p, %2, %3;\n\tmov.b64 {%0, %1}, p;\n\t}"
        : "=r"(lo1), "=r"(hi1) : "r"(c.z), "n"(kPhiloxM1));
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  return c;
}

// The same block with the key schedule precomputed (ks[2r], ks[2r + 1] = key words of round r):
// a launch-uniform schedule in the kernel-parameter block feeds the LOP3s as constant-bank
// operands, so it costs neither registers nor key-schedule adds.
__device__ __forceinline__ uint4 philox4x32_10_ks(uint4 c, const uint32_t (&ks)[20]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t lo0, hi0, lo1, hi1;
    asm("{\n\t.reg .b64 p;\n\tmul.wide.u32 p, %2, %3;\n\tmov.b64 {%0, %1}, p;\n\t}"
        : "=r"(lo0), "=r"(hi0) : "r"(c.x), "n"(kPhiloxM0));
    asm("{\n\t.reg .b64 p;\n\tmul.wide.u32 p, %2, %3;\n\tmov.b64 {%0, %1}, p;\n\t}"
        : "=r"(lo1), "=r"(hi1) : "r"(c.z), "n"(kPhiloxM1));
    c = make_uint4(hi1 ^ c.y ^ ks[2 * r], lo1, hi0 ^ c.w ^ ks[2 * r + 1], lo0);
  }
  return c;
}
__host__ __device__ inline void philox_key_schedule(uint64_t key, uint32_t (&ks)[20]) {
  uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
  for (int r = 0; r < 10; ++r) {
    ks[2 * r] = k0;
    ks[2 * r + 1] = k1;
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
}
__device__ __forceinline__ uint4 draw_block_ks(const uint32_t (&ks)[20], uint64_t id, uint32_t blk,
                                               uint32_t tag) {
  return philox4x32_10_ks(
      make_uint4(static_cast<uint32_t>(id), static_cast<uint32_t>(id >> 32), blk, tag), ks);
}

struct PhiloxKey {
  uint32_t k0, k1;
};
__host__ __device__ inline PhiloxKey make_key(uint64_t key) {
  return PhiloxKey{static_cast<uint32_t>(key), static_cast<uint32_t>(key >> 32)};
}

// Block `blk` of the stream of global id `id` under `tag`.
__device__ __forceinline__ uint4 draw_block(PhiloxKey k, uint64_t id, uint32_t blk,
                                            uint32_t tag) {
  return philox4x32_10(
      make_uint4(static_cast<uint32_t>(id), static_cast<uint32_t>(id >> 32), blk, tag), k.k0,
      k.k1);
}

// ---------------------------------------------------------------- transforms -----------
// 23-bit uniforms built from the mantissa (no I2F): exact in fp32 and fp64, so the oracle
// reproduces them bit for bit.
__device__ __forceinline__ float u01_open0(uint32_t w) {  // (0, 1]
  return 2.0f - __uint_as_float(0x3F800000u | (w >> 9));
}
__device__ __forceinline__ float u01_closed0(uint32_t w) {  // [0, 1)
  return __uint_as_float(0x3F800000u | (w >> 9)) - 1.0f;
}

// Lemire's multiply-shift on a b-bit word v < 2^b (range * 2^b < 2^32): exact uniform integer
// in [0, range); false when v must be rejected.
__device__ __forceinline__ bool lemire_bits(uint32_t v, uint32_t range, int bits, uint32_t* out) {
  const uint32_t m = v * range;
  const uint32_t mask = (1u << bits) - 1u;
  *out = m >> bits;
  const uint32_t lo = m & mask;
  if (lo < range) return lo >= ((1u << bits) % range);
  return true;
}

// Lemire's multiply-shift: uniform integer in [0, range) for range >= 1. Returns false when
// the word must be rejected for exact uniformity (cuppl/rng.py:47-56 rejects too).
__device__ __forceinline__ bool lemire(uint32_t w, uint32_t range, uint32_t* out) {
  const uint64_t m = static_cast<uint64_t>(w) * range;
  const uint32_t lo = static_cast<uint32_t>(m);
  *out = static_cast<uint32_t>(m >> 32);
  if (lo < range) {
    const uint32_t t = (0u - range) % range;
    return lo >= t;
  }
  return true;
}

__device__ __forceinline__ float fast_lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_sqrt(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_sin(float x) {
  float y;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_cos(float x) {
  float y;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr float kLn2 = 0.69314718055994530942f;
constexpr float kLog2e = 1.44269504088896340736f;
constexpr float kTwoPi = 6.28318530717958647692f;
constexpr float kPi = 3.14159265358979323846f;
constexpr float kHalfLog2Pi = 0.91893853320467274178f;

// u1 in (0, 1] from all 32 bits of a word: (w + 1) 2^-32 (the I2F rounds w above 2^24 to 24
// bits; the tail region u1 -> 0 is exact). A 32-bit u1 caps Box-Muller normals at
// sqrt(64 ln 2) = 6.66 sd (a 23-bit one would cap them at 5.65 sd).
__device__ __forceinline__ float u01_open0_32(uint32_t w) {
  return fmaf(__uint2float_rn(w), 0x1p-32f, 0x1p-32f);
}

// Box-Muller pair (cuppl/rng.py:58-71 without the cached spare: both normals are used).
// u1 = u01_open0_32(wa); u2 in [0,1) from the top 23 bits of wb; r = sqrt(-2 ln u1);
// (r cos 2pi u2, r sin 2pi u2). The angle is taken as 2pi u2 - pi in [-pi, pi) — sin.approx /
// cos.approx meet their 2^-20.5 absolute-error bound only there (2pi u2 up to 2pi measured
// ~1.6e-5) — and the signs flipped: cos(t + pi) = -cos t, sin(t + pi) = -sin t.
__device__ __forceinline__ float2 box_muller(uint32_t wa, uint32_t wb) {
  const float u1 = u01_open0_32(wa);
  const float u2 = u01_closed0(wb);
  const float r = fast_sqrt(-2.0f * kLn2 * fast_lg2(u1));
  const float th = fmaf(kTwoPi, u2, -kPi);
  return make_float2(-r * fast_cos(th), -r * fast_sin(th));
}

// sd * (Box-Muller pair) with the constants folded (the prior-draw form of the IS kernels):
// r_sd = sqrt(-2 sd^2 ln2 lg2 u1) carries the scale, and the angle 2 pi u2 - pi is formed from
// the mantissa-trick float f = 1 + u2 in [1, 2) as fma(2 pi, f, -3 pi) (the same [-pi, pi)
// range; no u2 = f - 1 subtraction). Two FMA-pipe instructions fewer per normal than
// sd * box_muller(); the values agree to fp32 rounding (~1e-6 relative).
__device__ __forceinline__ float2 box_muller_sd(uint32_t wa, uint32_t wb, float neg2_sd2_ln2) {
  const float u1 = u01_open0_32(wa);
  const float f = __uint_as_float(0x3F800000u | (wb >> 9));
  const float r = fast_sqrt(neg2_sd2_ln2 * fast_lg2(u1));
  const float th = fmaf(kTwoPi, f, -3.0f * kPi);
  return make_float2(-r * fast_cos(th), -r * fast_sin(th));
}
constexpr float kNeg2Sd2Ln2Prior = -2.0f * 100.0f * kLn2;  // normal(0, 10) priors (D2)

// ---------------------------------------------------------------- packed fp32 ----------
// sm_100 executes fma.rn.f32x2 / add.rn.f32x2 as one FFMA2 / FADD2 on a register pair.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pack2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 unpack2(f32x2 v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// ---------------------------------------------------------------- records --------------
__device__ __forceinline__ double neg_inf_d() { return __longlong_as_double(0xFFF0000000000000LL); }
__device__ __forceinline__ float neg_inf_f() { return __int_as_float(0xFF800000); }

__device__ __forceinline__ void rec_clear(cuppl_is_record& r) {
  r.max_lw = neg_inf_d();
  r.sum_w = 0.0;
  r.sum_w2 = 0.0;
  r.argmax_lw = neg_inf_d();
  r.argmax_pid = ~0ull;
  r.n_finite = 0;
  r.n_total = 0;
  r.reserved = 0;
#pragma unroll
  for (int k = 0; k < CUPPL_REC_STATS; ++k) r.stat_w[k] = 0.0;
#pragma unroll
  for (int k = 0; k < CUPPL_REC_BINS; ++k) r.bin_w[k] = 0.0;
}

// a <- merge(a, b). Symmetric in its arguments (commutative adds and max), so any fixed
// reduction tree gives identical bytes run to run.
__host__ __device__ inline void rec_merge(cuppl_is_record& a, const cuppl_is_record& b) {
  a.n_total += b.n_total;
  a.n_finite += b.n_finite;
  if (b.argmax_lw > a.argmax_lw || (b.argmax_lw == a.argmax_lw && b.argmax_pid < a.argmax_pid)) {
    a.argmax_lw = b.argmax_lw;
    a.argmax_pid = b.argmax_pid;
  }
  if (b.n_finite == 0) return;
  if (a.n_finite == b.n_finite) {  // a was empty
    a.max_lw = b.max_lw;
    a.sum_w = b.sum_w;
    a.sum_w2 = b.sum_w2;
    for (int k = 0; k < CUPPL_REC_STATS; ++k) a.stat_w[k] = b.stat_w[k];
    for (int k = 0; k < CUPPL_REC_BINS; ++k) a.bin_w[k] = b.bin_w[k];
    return;
  }
  const double m = a.max_lw > b.max_lw ? a.max_lw : b.max_lw;
  const double fa = exp(a.max_lw - m), fb = exp(b.max_lw - m);
  a.max_lw = m;
  a.sum_w = a.sum_w * fa + b.sum_w * fb;
  a.sum_w2 = a.sum_w2 * (fa * fa) + b.sum_w2 * (fb * fb);
  for (int k = 0; k < CUPPL_REC_STATS; ++k) a.stat_w[k] = a.stat_w[k] * fa + b.stat_w[k] * fb;
  for (int k = 0; k < CUPPL_REC_BINS; ++k) a.bin_w[k] = a.bin_w[k] * fa + b.bin_w[k] * fb;
}

// ---------------------------------------------------------------- block reductions -----
// Field-by-field reductions keep at most one fp64 value per thread in flight (a whole
// record in registers would cost 64+ registers and halve occupancy of the eval kernels).
// All trees are fixed (shuffle-down within a warp, then warp 0 folds the warps in order),
// so results are bit-identical run to run for a given launch shape.
constexpr int kMaxWarps = 32;

struct BlockScratch {
  double d[kMaxWarps];
  unsigned long long u[kMaxWarps];
  float f[kMaxWarps];
  float m_block;
};

__device__ __forceinline__ double block_sum_d(double v, BlockScratch& sc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) sc.d[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < nw; ++w) r += sc.d[w];
  __syncthreads();
  return r;  // valid in thread 0
}

__device__ __forceinline__ unsigned long long block_sum_u(unsigned long long v, BlockScratch& sc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) sc.u[warp] = v;
  __syncthreads();
  unsigned long long r = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < nw; ++w) r += sc.u[w];
  __syncthreads();
  return r;
}

// Max over the block, broadcast to every thread.
__device__ __forceinline__ double block_max_d_all(double v, BlockScratch& sc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  if (lane == 0) sc.d[warp] = v;
  __syncthreads();
  double r = sc.d[0];
  for (int w = 1; w < nw; ++w) r = fmax(r, sc.d[w]);
  __syncthreads();
  return r;
}

// Lexicographic argmax of (lw desc, pid asc); result in thread 0.
__device__ __forceinline__ void block_argmax(double& lw, unsigned long long& pid, BlockScratch& sc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ol = __shfl_down_sync(0xffffffffu, lw, o);
    const unsigned long long op = __shfl_down_sync(0xffffffffu, pid, o);
    if (ol > lw || (ol == lw && op < pid)) {
      lw = ol;
      pid = op;
    }
  }
  if (lane == 0) {
    sc.d[warp] = lw;
    sc.u[warp] = pid;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int w = 1; w < nw; ++w)
      if (sc.d[w] > lw || (sc.d[w] == lw && sc.u[w] < pid)) {
        lw = sc.d[w];
        pid = sc.u[w];
      }
  __syncthreads();
}

// A "record view": how a thread exposes its partial record field by field. Implemented by
// the eval kernels' fp32 accumulators and by the grid combine's strided fold of block records.
// Reduce the block's partial records into `out` (written by thread 0).
template <typename View>
__device__ __forceinline__ void block_reduce_view(const View& v, cuppl_is_record* out,
                                                  BlockScratch& sc) {
  const bool has = v.n_finite() > 0;
  const double M = block_max_d_all(has ? v.max_lw() : neg_inf_d(), sc);
  const double f = (has && M > neg_inf_d()) ? exp(v.max_lw() - M) : 0.0;
  double t;
  t = block_sum_d(v.sum_w() * f, sc);
  if (threadIdx.x == 0) out->sum_w = t;
  t = block_sum_d(v.sum_w2() * (f * f), sc);
  if (threadIdx.x == 0) out->sum_w2 = t;
#pragma unroll
  for (int k = 0; k < View::kStats; ++k) {
    t = block_sum_d(v.stat(k) * f, sc);
    if (threadIdx.x == 0) out->stat_w[k] = t;
  }
#pragma unroll
  for (int k = 0; k < View::kBins; ++k) {
    t = block_sum_d(v.bin(k) * f, sc);
    if (threadIdx.x == 0) out->bin_w[k] = t;
  }
  unsigned long long u = block_sum_u(v.n_finite(), sc);
  if (threadIdx.x == 0) out->n_finite = u;
  u = block_sum_u(v.n_total(), sc);
  if (threadIdx.x == 0) out->n_total = u;
  double al = has ? v.argmax_lw() : neg_inf_d();
  unsigned long long ap = has ? v.argmax_pid() : ~0ull;
  block_argmax(al, ap, sc);
  if (threadIdx.x == 0) {
    out->max_lw = M;
    out->argmax_lw = al;
    out->argmax_pid = ap;
    out->reserved = 0;
    for (int k = View::kStats; k < CUPPL_REC_STATS; ++k) out->stat_w[k] = 0.0;
    for (int k = View::kBins; k < CUPPL_REC_BINS; ++k) out->bin_w[k] = 0.0;
  }
}

// Strided fold of block records (already published to global memory) held by one thread.
struct StridedRecView {
  static constexpr int kStats = CUPPL_REC_STATS;
  static constexpr int kBins = CUPPL_REC_BINS;
  const cuppl_is_record* recs;
  unsigned int n, first, stride;
  double M;  // common stabiliser: global max over all records
  // the fold is computed lazily per field (records stay in L2; the grid is small)
  __device__ double fold(int field, int k) const {
    double acc = 0.0;
    for (unsigned int b = first; b < n; b += stride) {
      const cuppl_is_record& r = recs[b];
      if (r.n_finite == 0) continue;
      const double f = exp(r.max_lw - M);
      const double v = field == 0 ? r.sum_w : field == 1 ? r.sum_w2 : field == 2 ? r.stat_w[k] : r.bin_w[k];
      acc += v * (field == 1 ? f * f : f);
    }
    return acc;
  }
};

// Grid-level single-pass combine: every block publishes its record; the last block to
// arrive folds them (thread t folds blocks t, t+blockDim, ... in order; then the fixed block
// tree). `counter` must be 0 on entry; the last block resets it.
__device__ __forceinline__ void grid_combine(cuppl_is_record* block_recs, unsigned int* counter,
                                             cuppl_is_record* out, const cuppl_is_record& mine,
                                             BlockScratch& sc) {
  __shared__ bool is_last;
  if (threadIdx.x == 0) {
    block_recs[blockIdx.x] = mine;
    __threadfence();
    const unsigned int prev = atomicAdd(counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const unsigned int n = gridDim.x;
  double m = neg_inf_d();
  unsigned long long nf = 0, nt = 0;
  double al = neg_inf_d();
  unsigned long long ap = ~0ull;
  for (unsigned int b = threadIdx.x; b < n; b += blockDim.x) {
    const cuppl_is_record& r = block_recs[b];
    nf += r.n_finite;
    nt += r.n_total;
    if (r.n_finite) m = fmax(m, r.max_lw);
    if (r.argmax_lw > al || (r.argmax_lw == al && r.argmax_pid < ap)) {
      al = r.argmax_lw;
      ap = r.argmax_pid;
    }
  }
  const double M = block_max_d_all(m, sc);
  StridedRecView v{block_recs, n, threadIdx.x, blockDim.x, M};
  double t;
  t = block_sum_d(v.fold(0, 0), sc);
  if (threadIdx.x == 0) out->sum_w = t;
  t = block_sum_d(v.fold(1, 0), sc);
  if (threadIdx.x == 0) out->sum_w2 = t;
#pragma unroll 1
  for (int k = 0; k < CUPPL_REC_STATS; ++k) {
    t = block_sum_d(v.fold(2, k), sc);
    if (threadIdx.x == 0) out->stat_w[k] = t;
  }
#pragma unroll 1
  for (int k = 0; k < CUPPL_REC_BINS; ++k) {
    t = block_sum_d(v.fold(3, k), sc);
    if (threadIdx.x == 0) out->bin_w[k] = t;
  }
  nf = block_sum_u(nf, sc);
  nt = block_sum_u(nt, sc);
  block_argmax(al, ap, sc);
  if (threadIdx.x == 0) {
    out->max_lw = M;
    out->n_finite = nf;
    out->n_total = nt;
    out->argmax_lw = al;
    out->argmax_pid = ap;
    out->reserved = 0;
    *counter = 0u;
  }
}

}  // namespace cuppl
