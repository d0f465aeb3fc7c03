// is_kernels.cu — K1a/K1b importance-sampling evaluation fused with the K2 log-sum-exp /
// ESS / moment / histogram / argmax reduction.
//
// Replaces run_importance's hot loop: for each particle i the reference
// splits the RNG (cuppl/rng.py:31-37), runs the model through sample (prior draw) and
// factor (log-weight += log_p), and normalize()
// log-sum-exps the weights. Here a thread owns P particles at a time:
// draws come from Philox keyed by the global particle id, the model runs in registers with
// packed-fp32 (FFMA2) arithmetic on two particles per instruction, the data lives in the
// kernel-parameter constant bank (or registers), and the weights never leave the SM unless
// traces are requested: each thread keeps an online (max, sum w, sum w^2, sum w f(theta))
// record that is merged per block and then once per grid by the last block to finish.
#include "cuppl_device.cuh"
#include "is_kernels.cuh"
#include "is_accum.cuh"

namespace cuppl {

// ------------------------------------------------------------------ linear regression --
// lw = -0.5/sigma^2 * sum_i (y_i - a x_i - b)^2 - D (ln sigma + 0.5 ln 2 pi)
// Per point and particle pair: FADD2 (y - b), FFMA2 (r = -a x + (y - b)), FFMA2 (acc += r r).
template <int P, bool INJ, int CAP, int V>
__global__ void __launch_bounds__(kIsThreads)
is_linreg_kernel(const __grid_constant__ LinregParams<CAP> prm) {
  static_assert(P % 2 == 0, "particles are processed in FFMA2 pairs");
  ThreadAcc<5, 0> acc;
  acc.init();
  const uint64_t n = prm.pid_end - prm.pid_begin;
  const uint64_t chunk = static_cast<uint64_t>(blockDim.x) * P;
  const uint64_t nchunks = (n + chunk - 1) / chunk;
  const int D = prm.n_points;

  for (uint64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const uint64_t base = ch * chunk + threadIdx.x;
    float a[P], b[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint64_t idx = base + static_cast<uint64_t>(p) * blockDim.x;
      if (INJ) {
        const bool ok = idx < n;
        a[p] = ok ? prm.injected[2 * idx] : 0.f;
        b[p] = ok ? prm.injected[2 * idx + 1] : 0.f;
      } else {
        const uint4 w = draw_block_ks(prm.ks, prm.pid_begin + idx, 0u, CUPPL_TAG_IS);
        const float2 z = box_muller_sd(w.x, w.y, kNeg2Sd2Ln2Prior);  // normal(0, 10) (D2)
        a[p] = z.x;
        b[p] = z.y;
      }
    }
    // sum_i r_i^2 per particle, two accumulators per particle (even / odd points)
    float ssum[P];
    if constexpr (V == 2) {
      // scalar: per point and particle FADD (y - b), FFMA (r), FFMA (acc); x_i, y_i read
      // straight from the constant bank as instruction operands
      float s0[P], s1[P];
#pragma unroll
      for (int p = 0; p < P; ++p) s0[p] = s1[p] = 0.f;
      int i = 0;
#pragma unroll 2
      for (; i + 1 < D; i += 2) {
        const float2 p0 = xy_at(prm, i), p1 = xy_at(prm, i + 1);
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const float r0 = fmaf(-a[p], p0.x, p0.y - b[p]);
          const float r1 = fmaf(-a[p], p1.x, p1.y - b[p]);
          s0[p] = fmaf(r0, r0, s0[p]);
          s1[p] = fmaf(r1, r1, s1[p]);
        }
      }
      if (i < D) {
        const float2 p0 = xy_at(prm, i);
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const float r0 = fmaf(-a[p], p0.x, p0.y - b[p]);
          s0[p] = fmaf(r0, r0, s0[p]);
        }
      }
#pragma unroll
      for (int p = 0; p < P; ++p) ssum[p] = s0[p] + s1[p];
    } else {
      // packed: particle pairs share one FFMA2 / FADD2; V == 1 issues the (y - b) add as an
      // FFMA2 with a runtime 1.0 so it can use both FMA sub-pipes
      f32x2 NA[P / 2], NB[P / 2], S0[P / 2], S1[P / 2];
      const f32x2 ONE = pack2(prm.one, prm.one);
#pragma unroll
      for (int q = 0; q < P / 2; ++q) {
        NA[q] = pack2(-a[2 * q], -a[2 * q + 1]);
        NB[q] = pack2(-b[2 * q], -b[2 * q + 1]);
        S0[q] = pack2(0.f, 0.f);
        S1[q] = pack2(0.f, 0.f);
      }
      // large data sets (device-memory path): fp32 sums over 512-point chunks, folded in fp64
      // (D10), so the absolute error of lw stays ~1e-3 at 1e4..1e5 points
      constexpr bool kChunked = LinregParams<CAP>::kCap == 0;
      constexpr int kChunk = kChunked ? 512 : (1 << 30);
      double T64[kChunked ? P : 1];
#pragma unroll
      for (int p = 0; p < (kChunked ? P : 1); ++p) T64[p] = 0.0;
      int i = 0;
      for (int cend = min(D, kChunk); ; cend = min(D, cend + kChunk)) {
#pragma unroll 2
        for (; i + 1 < cend; i += 2) {
          const float2 p0 = xy_at(prm, i), p1 = xy_at(prm, i + 1);
          const f32x2 X0 = pack2(p0.x, p0.x), Y0 = pack2(p0.y, p0.y);
          const f32x2 X1 = pack2(p1.x, p1.x), Y1 = pack2(p1.y, p1.y);
#pragma unroll
          for (int q = 0; q < P / 2; ++q) {
            const f32x2 c0 = V == 1 ? fma2(NB[q], ONE, Y0) : add2(Y0, NB[q]);
            const f32x2 c1 = V == 1 ? fma2(NB[q], ONE, Y1) : add2(Y1, NB[q]);
            const f32x2 r0 = fma2(NA[q], X0, c0);
            const f32x2 r1 = fma2(NA[q], X1, c1);
            S0[q] = fma2(r0, r0, S0[q]);
            S1[q] = fma2(r1, r1, S1[q]);
          }
        }
        if constexpr (!kChunked) {
          break;
        } else {
          if (cend >= D) break;
#pragma unroll
          for (int q = 0; q < P / 2; ++q) {  // fold the chunk (even chunk sizes: i == cend here)
            const float2 t = unpack2(add2(S0[q], S1[q]));
            T64[2 * q] += t.x;
            T64[2 * q + 1] += t.y;
            S0[q] = pack2(0.f, 0.f);
            S1[q] = pack2(0.f, 0.f);
          }
        }
      }
      if (i < D) {
        const float2 p0 = xy_at(prm, i);
        const f32x2 X0 = pack2(p0.x, p0.x), Y0 = pack2(p0.y, p0.y);
#pragma unroll
        for (int q = 0; q < P / 2; ++q) {
          const f32x2 c0 = V == 1 ? fma2(NB[q], ONE, Y0) : add2(Y0, NB[q]);
          const f32x2 r0 = fma2(NA[q], X0, c0);
          S0[q] = fma2(r0, r0, S0[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < P / 2; ++q) {
        const float2 t = unpack2(add2(S0[q], S1[q]));
        if constexpr (kChunked) {
          ssum[2 * q] = static_cast<float>(T64[(2 * q) % (kChunked ? P : 1)] + t.x);
          ssum[2 * q + 1] = static_cast<float>(T64[(2 * q + 1) % (kChunked ? P : 1)] + t.y);
        } else {
          ssum[2 * q] = t.x;
          ssum[2 * q + 1] = t.y;
        }
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint64_t idx = base + static_cast<uint64_t>(p) * blockDim.x;
      if (idx < n) {
        const float lw = fmaf(prm.neg_half_inv_var, ssum[p], prm.lw_const);
        const float f[5] = {a[p], b[p], a[p] * a[p], b[p] * b[p], a[p] * b[p]};
        acc.add(lw, prm.pid_begin + idx, f, 0);
        if (prm.lw_out) prm.lw_out[idx] = lw;
        if (prm.coef_out) reinterpret_cast<float2*>(prm.coef_out)[idx] = make_float2(a[p], b[p]);
      }
    }
  }
  is_epilogue(acc, prm.block_recs, prm.counter, prm.rec_out);
}

// ------------------------------------------------------------------ Fig.1 polynomial ----
// One Philox block per particle: (c0, c1) = 10 BM(w0, w1), (c2, c3) = 10 BM(w2, w3); each
// Box-Muller pair takes its radius uniform from all 32 bits of w0 / w2 and its angle from the
// top 23 bits of w1 / w3, and n ~ uniform-discrete(2,5) (D1) uses the angle words' otherwise
// unused low bits: v = w1[8:0] | w3[8:0] << 9, Lemire on 18 bits; a rejected v (3 / 2^18) is
// redrawn from word 0 of blocks 1, 2, ... (32-bit Lemire). c_j = 0 for j >= n (exact: Horner
// with zero leading terms). lw = -sum_i (y_i - p(x_i))^2 (D3).
__device__ __forceinline__ uint32_t poly_degree_word(uint4 w) {
  return (w.y & 0x1FFu) | ((w.w & 0x1FFu) << 9);
}

__device__ __forceinline__ void poly_draw(const uint32_t (&ks)[20], uint64_t pid, int& n, float c[4]) {
  const uint4 w = draw_block_ks(ks, pid, 0u, CUPPL_TAG_IS);
  uint32_t k;
  if (!lemire_bits(poly_degree_word(w), 3u, 18, &k)) {
    for (uint32_t blk = 1;; ++blk) {
      if (lemire(draw_block_ks(ks, pid, blk, CUPPL_TAG_IS).x, 3u, &k)) break;
    }
  }
  n = 2 + static_cast<int>(k);
  const float2 z01 = box_muller_sd(w.x, w.y, kNeg2Sd2Ln2Prior);  // normal(0, 10) (D2)
  const float2 z23 = box_muller_sd(w.z, w.w, kNeg2Sd2Ln2Prior);
  c[0] = z01.x;
  c[1] = z01.y;
  c[2] = n > 2 ? z23.x : 0.0f;
  c[3] = n > 3 ? z23.y : 0.0f;
}

// Pair-packed online accumulator of the Fig.1 record: the two halves of every f32x2 belong to
// the two particles of an FFMA2 pair, so the per-degree moments (sum w c_j for n = 2, 3, 4:
// 9 values), the degree bins and sum w / sum w^2 cost one FADD2 / FFMA2 per pair. One
// stabiliser m per thread (D10: fp32 lanes, fp64 from the block level up).
struct PolyAcc {
  static constexpr int kStats = 9;  // n=2 -> [0,1]; n=3 -> [2,3,4]; n=4 -> [5..8]
  static constexpr int kBins = 3;   // n = 2, 3, 4
  float m;
  f32x2 s, s2, st[kStats], bn[kBins];
  float amax_lw;
  uint64_t amax_pid;
  uint32_t n_fin, n_tot;

  __device__ __forceinline__ void init() {
    m = neg_inf_f();
    s = s2 = pack2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < kStats; ++k) st[k] = pack2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < kBins; ++k) bn[k] = pack2(0.f, 0.f);
    amax_lw = neg_inf_f();
    amax_pid = ~0ull;
    n_fin = n_tot = 0;
  }

  // Particles a (lower pid) and b: log-weights, degrees, packed coefficients, validity.
  __device__ __forceinline__ void add_pair(float la, float lb, int da, int db, f32x2 C0, f32x2 C1,
                                           f32x2 C2, f32x2 C3, bool va, bool vb, uint64_t pid_a,
                                           uint64_t pid_b) {
    n_tot += static_cast<uint32_t>(va) + static_cast<uint32_t>(vb);
    const bool fa = va && fabsf(la) <= 3.402823466e38f;  // excludes +-inf and NaN (D9)
    const bool fb = vb && fabsf(lb) <= 3.402823466e38f;
    n_fin += static_cast<uint32_t>(fa) + static_cast<uint32_t>(fb);
    const float ea = fa ? la : neg_inf_f(), eb = fb ? lb : neg_inf_f();
    const float lmax = fmaxf(ea, eb);
    if (lmax > amax_lw) {  // strict: earlier (lower) pids win ties; a before b
      amax_lw = lmax;
      amax_pid = ea >= eb ? pid_a : pid_b;
    }
    if (lmax > m) {
      const float f0 = fast_ex2((m - lmax) * kLog2e);
      const f32x2 F = pack2(f0, f0);
      s = mul2(s, F);
      s2 = mul2(s2, mul2(F, F));
#pragma unroll
      for (int k = 0; k < kStats; ++k) st[k] = mul2(st[k], F);
#pragma unroll
      for (int k = 0; k < kBins; ++k) bn[k] = mul2(bn[k], F);
      m = lmax;
    }
    const float wa = fa ? fast_ex2((la - m) * kLog2e) : 0.f;
    const float wb = fb ? fast_ex2((lb - m) * kLog2e) : 0.f;
    const f32x2 W = pack2(wa, wb);
    s = add2(s, W);
    s2 = fma2(W, W, s2);
    const f32x2 W2 = pack2(da == 2 ? wa : 0.f, db == 2 ? wb : 0.f);
    const f32x2 W3 = pack2(da == 3 ? wa : 0.f, db == 3 ? wb : 0.f);
    const f32x2 W4 = pack2(da == 4 ? wa : 0.f, db == 4 ? wb : 0.f);
    bn[0] = add2(bn[0], W2);
    bn[1] = add2(bn[1], W3);
    bn[2] = add2(bn[2], W4);
    st[0] = fma2(W2, C0, st[0]);
    st[1] = fma2(W2, C1, st[1]);
    st[2] = fma2(W3, C0, st[2]);
    st[3] = fma2(W3, C1, st[3]);
    st[4] = fma2(W3, C2, st[4]);
    st[5] = fma2(W4, C0, st[5]);
    st[6] = fma2(W4, C1, st[6]);
    st[7] = fma2(W4, C2, st[7]);
    st[8] = fma2(W4, C3, st[8]);
  }

  __device__ __forceinline__ static double hsum(f32x2 v) {
    const float2 t = unpack2(v);
    return static_cast<double>(t.x) + static_cast<double>(t.y);
  }
  // record view (block_reduce_view)
  __device__ __forceinline__ unsigned long long n_finite() const { return n_fin; }
  __device__ __forceinline__ unsigned long long n_total() const { return n_tot; }
  __device__ __forceinline__ double max_lw() const { return m; }
  __device__ __forceinline__ double sum_w() const { return hsum(s); }
  __device__ __forceinline__ double sum_w2() const { return hsum(s2); }
  __device__ __forceinline__ double stat(int k) const { return hsum(st[k]); }
  __device__ __forceinline__ double bin(int k) const { return hsum(bn[k]); }
  __device__ __forceinline__ double argmax_lw() const { return amax_lw; }
  __device__ __forceinline__ unsigned long long argmax_pid() const { return amax_pid; }
};

// One chunk of P particles per thread: particle p of the chunk is global id base + p * 256.
// FULL: every particle of the chunk is in range (no per-particle bounds checks).
template <int P, bool INJ, int DC, bool TR, bool FULL, int CAP>
__device__ __forceinline__ void poly_chunk(const PolyParams<CAP>& prm, PolyAcc& acc, PhiloxKey key,
                                           uint64_t n, uint64_t base) {
  const int D = DC > 0 ? DC : prm.n_points;
  float c[P][4];
  int deg[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const uint64_t idx = base + static_cast<uint64_t>(p) * kIsThreads;
    if (INJ) {
      const bool ok = FULL || idx < n;
      const float* src = prm.injected + 5 * (ok ? idx : 0);
      deg[p] = ok ? static_cast<int>(src[0]) : 2;
#pragma unroll
      for (int j = 0; j < 4; ++j) c[p][j] = (ok && j < deg[p]) ? src[1 + j] : 0.f;
    } else {
      poly_draw(prm.ks, prm.pid_begin + idx, deg[p], c[p]);
    }
  }
  f32x2 C0[P / 2], C1[P / 2], C2[P / 2], C3[P / 2], S[P / 2];
#pragma unroll
  for (int q = 0; q < P / 2; ++q) {
    C0[q] = pack2(c[2 * q][0], c[2 * q + 1][0]);
    C1[q] = pack2(c[2 * q][1], c[2 * q + 1][1]);
    C2[q] = pack2(c[2 * q][2], c[2 * q + 1][2]);
    C3[q] = pack2(c[2 * q][3], c[2 * q + 1][3]);
    S[q] = pack2(0.f, 0.f);
  }
#pragma unroll(DC > 0 ? DC : 4)
  for (int i = 0; i < D; ++i) {
    const float2 xy = xy_at(prm, i);  // warp-uniform constant-bank load (LDCU)
    const f32x2 X = pack2(xy.x, xy.x), NY = pack2(-xy.y, -xy.y);
#pragma unroll
    for (int q = 0; q < P / 2; ++q) {
      f32x2 t = fma2(C3[q], X, C2[q]);
      t = fma2(t, X, C1[q]);
      t = fma2(t, X, C0[q]);
      const f32x2 r = add2(t, NY);
      S[q] = fma2(r, r, S[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < P / 2; ++q) {
    const float2 sq = unpack2(S[q]);
    const uint64_t ia = base + static_cast<uint64_t>(2 * q) * kIsThreads;
    const uint64_t ib = ia + kIsThreads;
    const bool va = FULL || ia < n, vb = FULL || ib < n;
    acc.add_pair(-sq.x, -sq.y, deg[2 * q], deg[2 * q + 1], C0[q], C1[q], C2[q], C3[q], va, vb,
                 prm.pid_begin + ia, prm.pid_begin + ib);
    if (TR) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = 2 * q + h;
        const uint64_t idx = h ? ib : ia;
        if (FULL || idx < n) {
          if (prm.lw_out) prm.lw_out[idx] = -(h ? sq.y : sq.x);
          if (prm.deg_out) prm.deg_out[idx] = deg[p];
          if (prm.coef_out)
            reinterpret_cast<float4*>(prm.coef_out)[idx] = make_float4(c[p][0], c[p][1], c[p][2], c[p][3]);
        }
      }
    }
  }
}

template <int P, bool INJ, int DC, bool TR, int CAP, int MB = kPolyMinBlocks>
__global__ void __launch_bounds__(kIsThreads, MB)
is_poly_kernel(const __grid_constant__ PolyParams<CAP> prm) {
  static_assert(P % 2 == 0, "particles are processed in FFMA2 pairs");
  PolyAcc acc;
  acc.init();
  const PhiloxKey key{prm.k0, prm.k1};
  const uint64_t n = prm.pid_end - prm.pid_begin;
  constexpr uint64_t chunk = static_cast<uint64_t>(kIsThreads) * P;
  const uint64_t nfull = n / chunk;
  for (uint64_t ch = blockIdx.x; ch < nfull; ch += gridDim.x)
    poly_chunk<P, INJ, DC, TR, true>(prm, acc, key, n, ch * chunk + threadIdx.x);
  if (nfull * chunk < n && blockIdx.x == nfull % gridDim.x)
    poly_chunk<P, INJ, DC, TR, false>(prm, acc, key, n, nfull * chunk + threadIdx.x);
  is_epilogue(acc, prm.block_recs, prm.counter, prm.rec_out);
}

// ------------------------------------------------------------------ launchers ----------
template <typename KernelT, typename ParamT>
static cudaError_t launch_persistent(KernelT kernel, const ParamT& prm, int sm_count,
                                     uint64_t n_chunks, int max_blocks, cudaStream_t stream,
                                     int* grid_out) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kIsThreads, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = static_cast<uint64_t>(sm_count) * per_sm;
  if (grid > n_chunks) grid = n_chunks ? n_chunks : 1;
  if (grid > static_cast<uint64_t>(max_blocks)) grid = max_blocks;
  *grid_out = static_cast<int>(grid);
  kernel<<<static_cast<unsigned>(grid), kIsThreads, 0, stream>>>(prm);
  return cudaGetLastError();
}

template <int CAP, int V>
static cudaError_t launch_linreg_v(const LinregParams<CAP>& prm, bool injected, int sm_count,
                                   int max_blocks, cudaStream_t stream) {
  constexpr int P = kLinregP;
  const uint64_t n = prm.pid_end - prm.pid_begin;
  const uint64_t nchunks = (n + kIsThreads * P - 1) / (kIsThreads * P);
  int grid = 0;
  if (injected)
    return launch_persistent(is_linreg_kernel<P, true, CAP, V>, prm, sm_count, nchunks, max_blocks, stream, &grid);
  return launch_persistent(is_linreg_kernel<P, false, CAP, V>, prm, sm_count, nchunks, max_blocks, stream, &grid);
}

template <int CAP>
cudaError_t launch_linreg(const LinregParams<CAP>& prm, bool injected, int sm_count,
                          int max_blocks, cudaStream_t stream, int variant) {
  switch (variant) {
    case 1: return launch_linreg_v<CAP, 1>(prm, injected, sm_count, max_blocks, stream);
    case 2: return launch_linreg_v<CAP, 2>(prm, injected, sm_count, max_blocks, stream);
    default: return launch_linreg_v<CAP, 0>(prm, injected, sm_count, max_blocks, stream);
  }
}

template <int CAP>
cudaError_t launch_poly(const PolyParams<CAP>& prm, bool injected, int sm_count, int max_blocks,
                        cudaStream_t stream, int variant) {
  constexpr int P = kPolyP;
  const uint64_t n = prm.pid_end - prm.pid_begin;
  int grid = 0;
  auto chunks = [n](int p) { return (n + kIsThreads * p - 1) / (kIsThreads * p); };
  const bool tr = prm.lw_out || prm.deg_out || prm.coef_out;
  if (prm.n_points == 20 && !injected && !tr) {  // the benchmark configuration (C1/C5)
    switch (variant) {  // (particles per thread, min blocks per SM): tuning only
      case 1: return launch_persistent(is_poly_kernel<4, false, 20, false, CAP, 3>, prm, sm_count, chunks(4), max_blocks, stream, &grid);
      case 2: return launch_persistent(is_poly_kernel<2, false, 20, false, CAP, 4>, prm, sm_count, chunks(2), max_blocks, stream, &grid);
      case 3: return launch_persistent(is_poly_kernel<2, false, 20, false, CAP, 3>, prm, sm_count, chunks(2), max_blocks, stream, &grid);
      default: return launch_persistent(is_poly_kernel<P, false, 20, false, CAP>, prm, sm_count, chunks(P), max_blocks, stream, &grid);
    }
  }
  if (injected)
    return launch_persistent(is_poly_kernel<P, true, 0, true, CAP>, prm, sm_count, chunks(P), max_blocks, stream, &grid);
  if (!tr)
    return launch_persistent(is_poly_kernel<P, false, 0, false, CAP>, prm, sm_count, chunks(P), max_blocks, stream, &grid);
  return launch_persistent(is_poly_kernel<P, false, 0, true, CAP>, prm, sm_count, chunks(P), max_blocks, stream, &grid);
}

// the measured point-array placement (is_kernels.cuh kXyOffset)
#pragma nv_diag_suppress 1427
#pragma GCC diagnostic push
#pragma GCC diagnostic ignored "-Winvalid-offsetof"
static_assert(offsetof(LinregParams<kLinregCapSmall>, xy) == kXyOffset, "linreg xy offset");
static_assert(offsetof(LinregParams<kLinregCapLarge>, xy) == kXyOffset, "linreg xy offset");
static_assert(offsetof(PolyParams<kPolyCap>, xy) == kXyOffset, "poly xy offset");
#pragma GCC diagnostic pop
#pragma nv_diag_default 1427

template cudaError_t launch_linreg<kLinregCapSmall>(const LinregParams<kLinregCapSmall>&, bool, int, int, cudaStream_t, int);
template cudaError_t launch_linreg<kLinregCapLarge>(const LinregParams<kLinregCapLarge>&, bool, int, int, cudaStream_t, int);
template cudaError_t launch_poly<kPolyCap>(const PolyParams<kPolyCap>&, bool, int, int, cudaStream_t, int);
template cudaError_t launch_linreg<kIsCapGlobal>(const LinregParams<kIsCapGlobal>&, bool, int, int, cudaStream_t, int);
template cudaError_t launch_poly<kIsCapGlobal>(const PolyParams<kIsCapGlobal>&, bool, int, int, cudaStream_t, int);

}  // namespace cuppl
