// smc_kernels.cu — K4 init, K5 quantise + tile scan (decoupled look-back), K6 fused
// systematic resampling + ancestor gather + propagate + reweight, for the bootstrap particle
// filter. SMC has no reference semantics, so
// oracle/cuppl_oracle.c (or_smc_*) *defines* every bit these kernels must reproduce:
//
//   w_i      = min(floor(exp_repro(lw_i - M_t) * 2^31), 2^31)      (u32, exact fp32 sequence)
//   C        = inclusive u64 scan of w; T = C[N-1]
//   target_j = floor((j 2^32 + u) T / (N 2^32)), u = word 0 of Philox(t, 0, 0, TAG_SMC_COMB)
//   a_j      = min{i : C_i > target_j}
//   x'_j     ~ categorical(A[x_{a_j}]) with word (j & 3) of Philox(j >> 2, t + 1, TAG_SMC_STEP)
//   lw'_j    = log N(y_{t+1}; mu[x'_j], sd)
//
// Data layout per rank: x (u8, one byte per particle), lw (f32); segoff (u64 per 32
// particles, rank-local inclusive weight prefix) is the only scan output in HBM. Per step
// the algorithmic traffic is 4 B (K5 reads lw) + 4 + 1 (K6 stages lw, x of its sources) +
// 1 + 4 (K6 writes x', lw') = 14 B per particle (+0.25 B of segment offsets each way).
//
// K6 is output-balanced and source-streaming: CTA b owns an even share of the rank's output
// range, finds the ancestor of its first output once (warp-parallel 32-ary search on segoff),
// then streams its sources in order in batches of 2048. For each staged source with w_i > 0 it
// computes f_i = min{j : target_j >= C_{i-1}} with an incremental integer recurrence; since
// a_j = max{i : w_i > 0, f_i <= j}, a scatter of i into mark[f_i] followed by an inclusive
// max-scan yields every ancestor of the batch's outputs with no per-output search, whatever the
// offspring distribution.
#include "cuppl_device.cuh"
#include "smc_kernels.cuh"

namespace cuppl {

// ------------------------------------------------------------------ exact helpers -------
__device__ __forceinline__ float exp_repro(float d) {
  const float t = __fmul_rn(d, 1.44269504f);
  const float k = rintf(t);
  float r = __fmaf_rn(k, -0.693145752f, d);
  r = __fmaf_rn(k, -1.42860677e-06f, r);
  float p = 1.38888893e-03f;
  p = __fmaf_rn(p, r, 8.33333377e-03f);
  p = __fmaf_rn(p, r, 4.16666679e-02f);
  p = __fmaf_rn(p, r, 1.66666672e-01f);
  p = __fmaf_rn(p, r, 0.5f);
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  return __fmul_rn(p, __int_as_float((static_cast<int>(k) + 127) << 23));
}

__device__ __forceinline__ float smc_e(float lw, float M) {
  if (!(lw > neg_inf_f())) return 0.0f;
  const float d = __fsub_rn(lw, M);
  if (!(d >= -87.0f)) return 0.0f;
  return exp_repro(d);
}

__device__ __forceinline__ uint32_t smc_w(float e) {
  const uint32_t w = __float2uint_rz(__fmul_rn(e, 2147483648.0f));
  return w > 0x80000000u ? 0x80000000u : w;
}

__device__ __forceinline__ float emission(float y, float mu, float inv_sd, float c) {
  const float z = __fmul_rn(__fsub_rn(y, mu), inv_sd);
  return __fmaf_rn(__fmul_rn(-0.5f, z), z, c);
}

// Monotone float <-> int key (signed compare == float compare), for atomicMax.
__device__ __forceinline__ int f2key(float f) {
  const int i = __float_as_int(f);
  return i ^ ((i >> 31) & 0x7FFFFFFF);
}
__device__ __forceinline__ float key2f(int k) { return __int_as_float(k ^ ((k >> 31) & 0x7FFFFFFF)); }

__device__ __forceinline__ int categorical_u64(const unsigned long long* thr, int K, uint32_t w) {
  int lo = 0, hi = K - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (static_cast<unsigned long long>(w) < __ldg(thr + mid)) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// ------------------------------------------------------------------ K4: init ------------
// x_0[j] ~ categorical(pi0) with word (j & 3) of Philox(j >> 2, 0, TAG_SMC_INIT);
// lw_0[j] = log N(y_0; mu[x_0[j]], sd). One Philox block per 4 particles.
__global__ void __launch_bounds__(kSmcThreads) smc_init_kernel(const __grid_constant__ SmcModel m,
                                                               SmcInitArgs a) {
  __shared__ float s_mu[kMaxStates];
  for (int q = threadIdx.x; q < m.S; q += blockDim.x) s_mu[q] = m.mu[q];
  __syncthreads();
  const PhiloxKey key = make_key(a.key);
  float bmax = neg_inf_f();
  const unsigned long long nq = (a.n_local + 3) / 4;
  for (unsigned long long q = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
       q < nq; q += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const unsigned long long j = a.j_begin + 4 * q;  // global index, multiple of 4
    const uint4 w = draw_block(key, j >> 2, 0u, CUPPL_TAG_SMC_INIT);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const unsigned long long i = 4 * q + k;
      if (i < a.n_local) {
        const int s = categorical_u64(m.thr_pi0, m.S, ws[k]);
        const float lw = emission(a.y0, s_mu[s], m.inv_sd, m.c);
        a.x[i] = static_cast<uint8_t>(s);
        a.lw[i] = lw;
        bmax = fmaxf(bmax, lw);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
  if ((threadIdx.x & 31) == 0 && bmax > neg_inf_f()) atomicMax(a.m_key, f2key(bmax));
}

// ------------------------------------------------------------------ K5: scan ------------
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagIncl = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <bool HIST>
__global__ void __launch_bounds__(kSmcThreads) smc_scan_kernel(SmcScanArgs a) {
  __shared__ unsigned long long seg_sum[kTileSegs];
  __shared__ unsigned long long wtot[kSmcThreads / 32];
  __shared__ unsigned long long s_prefix;
  __shared__ unsigned int s_tile;
  __shared__ bool s_last;
  __shared__ BlockScratch sc;
  __shared__ unsigned long long shist[HIST ? kMaxStates : 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long n = a.n_local;
  const unsigned long long n_tiles = (n + kTile - 1) / kTile;
  const float M = key2f(*a.m_key);
  if (tid == 0) s_tile = atomicAdd(&a.counters[0], 1u);
  if (HIST)
    for (int s = tid; s < a.S; s += kSmcThreads) shist[s] = 0;
  __syncthreads();
  const unsigned long long tile = s_tile;
  const unsigned long long wbase = tile * kTile + static_cast<unsigned long long>(warp) * 1024;
  float s1 = 0.f, s2 = 0.f;
#pragma unroll 2
  for (int it = 0; it < 8; ++it) {
    const unsigned long long p0 = wbase + it * 128 + lane * 4;
    float v[4];
    uint8_t xv[4] = {0, 0, 0, 0};
    if (p0 + 3 < n) {
      const float4 f = __ldcs(reinterpret_cast<const float4*>(a.lw + p0));
      v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
      if (HIST) {
        const uchar4 c = *reinterpret_cast<const uchar4*>(a.x + p0);
        xv[0] = c.x; xv[1] = c.y; xv[2] = c.z; xv[3] = c.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[k] = p0 + k < n ? a.lw[p0 + k] : neg_inf_f();
        if (HIST) xv[k] = p0 + k < n ? a.x[p0 + k] : 0;
      }
    }
    unsigned long long ws = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float e = smc_e(v[k], M);
      const uint32_t w = smc_w(e);
      ws += w;
      s1 += e;
      s2 = fmaf(e, e, s2);
      if (HIST && w) atomicAdd(&shist[xv[k]], static_cast<unsigned long long>(w));
    }
    ws += __shfl_xor_sync(0xffffffffu, ws, 1);
    ws += __shfl_xor_sync(0xffffffffu, ws, 2);
    ws += __shfl_xor_sync(0xffffffffu, ws, 4);
    if ((lane & 7) == 0) seg_sum[warp * 32 + it * 4 + (lane >> 3)] = ws;
  }
  __syncthreads();
  // inclusive scan of the tile's 256 segment sums (thread tid <-> segment tid)
  unsigned long long incl = seg_sum[tid];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  unsigned long long wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += wtot[w];
  incl += wpre;
  if (tid == 0) {
    unsigned long long agg = 0;
    for (int w = 0; w < kSmcThreads / 32; ++w) agg += wtot[w];
    unsigned long long prefix = 0;
    if (tile == 0) {
      st_release_u64(a.flags, kFlagIncl | agg);
    } else {
      st_release_u64(a.flags + tile, kFlagAgg | agg);
      long long k = static_cast<long long>(tile) - 1;
      while (k >= 0) {
        const unsigned long long f = ld_volatile_u64(a.flags + k);
        const unsigned long long st = f >> 62;
        if (st == 0) continue;  // predecessor not published yet
        prefix += f & kValMask;
        if (st == 2) break;
        --k;
      }
      st_release_u64(a.flags + tile, kFlagIncl | (prefix + agg));
    }
    s_prefix = prefix;
  }
  __syncthreads();
  const unsigned long long gs = tile * kTileSegs + tid;
  if (gs * kSegment < n) a.segoff[gs] = s_prefix + incl;
  const double d1 = block_sum_d(static_cast<double>(s1), sc);
  const double d2 = block_sum_d(static_cast<double>(s2), sc);
  if (tid == 0) {
    a.tile_s[2 * tile] = d1;
    a.tile_s[2 * tile + 1] = d2;
  }
  if (HIST) {
    for (int s = tid; s < a.S; s += kSmcThreads)
      if (shist[s]) atomicAdd(&a.hist[s], shist[s]);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&a.counters[1], 1u) == n_tiles - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // last CTA: fixed-order fp64 fold of the tile sums -> rank record
  double f1 = 0.0, f2 = 0.0;
  for (unsigned long long tt = tid; tt < n_tiles; tt += kSmcThreads) {
    f1 += a.tile_s[2 * tt];
    f2 += a.tile_s[2 * tt + 1];
  }
  f1 = block_sum_d(f1, sc);
  f2 = block_sum_d(f2, sc);
  if (tid == 0) {
    const unsigned long long T = ld_volatile_u64(a.flags + n_tiles - 1) & kValMask;
    a.rank_rec[0] = T;
    a.rank_rec[1] = static_cast<unsigned long long>(__double_as_longlong(f1));
    a.rank_rec[2] = static_cast<unsigned long long>(__double_as_longlong(f2));
    a.rank_rec[3] = 0;
    a.counters[0] = 0;
    a.counters[1] = 0;
  }
}

// ------------------------------------------------------------------ K6: resample --------
// Comb in integers (D6): with T = Q N + R0 and A = floor(u T / 2^32) = Qa N + Ra,
// target_j = floor((j 2^32 + u) T / (N 2^32)) = j Q + Qa + floor((j R0 + Ra) / N),
// where j R0 + Ra < N^2 < 2^64 (N < 2^32).
struct Comb {
  unsigned long long N, Q, R0, Qa, Ra;
  double invN;
};

// floor(num / N) for num < 2^64: fp64 estimate, exact correction.
__device__ __forceinline__ unsigned long long div_n(unsigned long long num, const Comb& cb,
                                                   unsigned long long* rem) {
  unsigned long long q = static_cast<unsigned long long>(__dmul_rn(__ull2double_rn(num), cb.invN));
  long long r = static_cast<long long>(num - q * cb.N);
  while (r < 0) {
    --q;
    r += static_cast<long long>(cb.N);
  }
  while (r >= static_cast<long long>(cb.N)) {
    ++q;
    r -= static_cast<long long>(cb.N);
  }
  *rem = static_cast<unsigned long long>(r);
  return q;
}

// Cursor over consecutive targets: (j, target_j, (j R0 + Ra) mod N).
struct CombCursor {
  unsigned long long j, tgt, mod;
  __device__ __forceinline__ void seek(unsigned long long jj, const Comb& cb) {
    j = jj;
    unsigned long long r;
    const unsigned long long q = div_n(jj * cb.R0 + cb.Ra, cb, &r);
    tgt = jj * cb.Q + cb.Qa + q;
    mod = r;
  }
  __device__ __forceinline__ void next(const Comb& cb) {
    ++j;
    tgt += cb.Q;
    mod += cb.R0;
    if (mod >= cb.N) {
      mod -= cb.N;
      ++tgt;
    }
  }
  // advance to the smallest j' >= j with target_j' >= c (or N); big gaps jump by estimate
  __device__ __forceinline__ void advance_to(unsigned long long c, const Comb& cb, double step_inv) {
    if (j >= cb.N || tgt >= c) return;
    const unsigned long long gap = c - tgt;
    if (gap > 8 * (cb.Q + 1)) {
      // estimate j' ~ j + gap N / T, then settle exactly from below
      double est = __dmul_rn(__ull2double_rn(gap), step_inv);
      unsigned long long jj = j + (est > 2.0 ? static_cast<unsigned long long>(est) - 2 : 0);
      if (jj > cb.N) jj = cb.N;
      if (jj > j) {
        seek(jj, cb);
        // seek may overshoot only if the estimate was too large: back off exponentially
        unsigned long long back = 1;
        while (j > 0 && tgt >= c) {
          const unsigned long long jn = j > back ? j - back : 0;
          seek(jn, cb);
          back <<= 1;
        }
      }
    }
    while (j < cb.N && tgt < c) next(cb);
  }
};

__device__ __forceinline__ unsigned long long comb_target(unsigned long long j, const Comb& cb) {
  unsigned long long r;
  return j * cb.Q + cb.Qa + div_n(j * cb.R0 + cb.Ra, cb, &r);
}

// smallest j in [0, N] with target_j >= c (N if none)
__device__ unsigned long long first_j_at_least(unsigned long long c, const Comb& cb,
                                               double step_inv) {
  CombCursor cur;
  cur.seek(0, cb);
  cur.advance_to(c, cb, step_inv);
  return cur.j;
}

// Warp-cooperative rank-local upper bound: smallest local i with C_i > t (C = inclusive scan
// of the rank's weights, represented by segoff + the lw of one segment). Returns n_local if none.
// The segment is found with a 33-way search (5 rounds of one coalesced-ish probe per lane for
// 3e6 segments), then resolved inside the segment with a warp scan of its 32 weights.
__device__ unsigned long long warp_upper_bound(unsigned long long t, const SmcResampleArgs& a,
                                               float M) {
  const int lane = threadIdx.x & 31;
  const unsigned long long n_segs = (a.n_local + kSegment - 1) / kSegment;
  unsigned long long lo = 0, hi = n_segs;  // invariant: answer in [lo, hi]
  while (hi - lo > 32) {
    const unsigned long long span = hi - lo;
    const unsigned long long p = lo + span * (lane + 1) / 33;  // strictly increasing, < hi
    const unsigned int bal = __ballot_sync(0xffffffffu, a.segoff[p] > t);
    if (!bal) {
      lo = lo + span * 32 / 33 + 1;
    } else {
      const int fl = __ffs(bal) - 1;
      const unsigned long long new_hi = lo + span * (fl + 1) / 33;
      if (fl > 0) lo = lo + span * fl / 33 + 1;
      hi = new_hi;
    }
  }
  {
    const unsigned long long p = lo + lane;
    const unsigned int bal = __ballot_sync(0xffffffffu, p < hi && a.segoff[p] > t);
    hi = bal ? lo + (__ffs(bal) - 1) : hi;
  }
  const unsigned long long s = hi;
  if (s >= n_segs) return a.n_local;
  const unsigned long long base = s > 0 ? a.segoff[s - 1] : 0ull;
  const unsigned long long i = s * kSegment + lane;
  const uint32_t w = i < a.n_local ? smc_w(smc_e(a.lw[i], M)) : 0u;
  unsigned long long incl = w;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long u2 = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u2;
  }
  const unsigned int bal = __ballot_sync(0xffffffffu, i < a.n_local && base + incl > t);
  if (!bal) return a.n_local;
  return s * kSegment + (__ffs(bal) - 1);
}

__global__ void __launch_bounds__(kSmcThreads) smc_resample_kernel(const __grid_constant__ SmcModel m,
                                                                   SmcResampleArgs a) {
  __shared__ unsigned int mark[kChunk];
  __shared__ uint8_t xs[kBatch];
  __shared__ unsigned long long wsum[kSmcThreads / 32];
  __shared__ unsigned int wmax[kSmcThreads / 32];
  __shared__ unsigned int s_carry;
  __shared__ unsigned long long s_u64[4];
  __shared__ unsigned long long s_rank_begin[kMaxRanks + 1];
  __shared__ float s_mu[kMaxStates];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int q = tid; q < m.S; q += kSmcThreads) s_mu[q] = m.mu[q];

  // step constants (identical on every rank)
  unsigned long long T = 0, O = 0;
  for (int q = 0; q < a.world; ++q) {
    const unsigned long long Tq = a.rank_recs[4 * q];
    if (q < a.rank) O += Tq;
    T += Tq;
  }
  const unsigned long long Tr = a.rank_recs[4 * a.rank];
  for (int q = tid; q <= a.world; q += kSmcThreads) s_rank_begin[q] = a.rank_begin[q];
  // clear the look-back words for the next scan
  for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(kSmcThreads) + tid;
       i < a.n_tiles; i += static_cast<unsigned long long>(gridDim.x) * kSmcThreads)
    a.flags_to_clear[i] = 0ull;
  if (T == 0) return;  // all weights zero: the host raises AllZeroWeightError
  const float M = key2f(*a.m_key);
  const PhiloxKey key = make_key(a.key);
  const uint32_t u = draw_block(key, a.t, 0u, CUPPL_TAG_SMC_COMB).x;
  Comb cb;
  cb.N = a.n_total;
  cb.Q = T / cb.N;
  cb.R0 = T % cb.N;
  const unsigned long long A = __umul64hi(static_cast<unsigned long long>(u) << 32, T);  // floor(u T / 2^32)
  cb.Qa = A / cb.N;
  cb.Ra = A % cb.N;
  cb.invN = 1.0 / static_cast<double>(cb.N);
  const double step_inv = static_cast<double>(cb.N) / static_cast<double>(T);

  // this rank's outputs: J_r = {j : O <= target_j < O + Tr}; this CTA's even share of it
  if (tid == 0) {
    s_u64[0] = a.rank == 0 ? 0ull : first_j_at_least(O, cb, step_inv);
    s_u64[1] = a.rank == a.world - 1 ? cb.N : first_j_at_least(O + Tr, cb, step_inv);
  }
  __syncthreads();
  const unsigned long long jr_lo = s_u64[0], jr_hi = s_u64[1];
  const unsigned long long span = jr_hi - jr_lo;
  const unsigned long long jb_lo = jr_lo + span * blockIdx.x / gridDim.x;
  const unsigned long long jb_hi = jr_lo + span * (blockIdx.x + 1) / gridDim.x;
  if (jb_lo >= jb_hi) return;

  // ancestor of the first output -> first batch starts at its segment boundary
  if (warp == 0) {
    const unsigned long long tl = comb_target(jb_lo, cb) - O;
    const unsigned long long i0 = warp_upper_bound(tl, a, M);
    if (lane == 0) s_u64[2] = i0;
  }
  __syncthreads();
  unsigned long long batch_base = (s_u64[2] / kSegment) * kSegment;
  unsigned long long c_base = batch_base > 0 ? a.segoff[batch_base / kSegment - 1] : 0ull;
  unsigned long long j_cur = jb_lo;
  float bmax = neg_inf_f();

  while (j_cur < jb_hi && batch_base < a.n_local) {
    // ---- stage 2048 sources: thread tid owns [batch_base + 8 tid, +8)
    const unsigned long long i0 = batch_base + kBatchPerThread * tid;
    uint32_t w[kBatchPerThread];
    unsigned long long tw = 0;
    if (i0 + kBatchPerThread <= a.n_local) {
      const float4 f0 = __ldcs(reinterpret_cast<const float4*>(a.lw + i0));
      const float4 f1 = __ldcs(reinterpret_cast<const float4*>(a.lw + i0) + 1);
      const uint2 xx = *reinterpret_cast<const uint2*>(a.x + i0);
      const float v[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
#pragma unroll
      for (int k = 0; k < kBatchPerThread; ++k) {
        w[k] = smc_w(smc_e(v[k], M));
        tw += w[k];
      }
      *reinterpret_cast<uint2*>(xs + kBatchPerThread * tid) = xx;
    } else {
#pragma unroll
      for (int k = 0; k < kBatchPerThread; ++k) {
        const bool ok = i0 + k < a.n_local;
        w[k] = ok ? smc_w(smc_e(a.lw[i0 + k], M)) : 0u;
        xs[kBatchPerThread * tid + k] = ok ? a.x[i0 + k] : 0;
        tw += w[k];
      }
    }
    // block exclusive scan of the thread sums
    unsigned long long incl = tw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t2 = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t2;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    unsigned long long wpre = 0, btot = 0;
    for (int q = 0; q < kSmcThreads / 32; ++q) {
      if (q < warp) wpre += wsum[q];
      btot += wsum[q];
    }
    const unsigned long long texcl = c_base + wpre + incl - tw;  // C_{i0 - 1} (local)
    // f_k for each positive-weight source (global target units), monotone per thread
    unsigned long long f[kBatchPerThread];
    {
      CombCursor cur;
      bool init = false;
      unsigned long long c = texcl;
#pragma unroll
      for (int k = 0; k < kBatchPerThread; ++k) {
        f[k] = ~0ull;
        if (w[k]) {
          if (!init) {
            const unsigned long long jg = O + c == 0 ? 0 : first_j_at_least(O + c, cb, step_inv);
            cur.seek(jg < cb.N ? jg : cb.N - 1, cb);
            if (jg >= cb.N) cur.j = cb.N;
            init = true;
          } else {
            cur.advance_to(O + c, cb, step_inv);
          }
          f[k] = cur.j;
        }
        c += w[k];
      }
    }
    // outputs whose ancestors lie in this batch: [j_cur, j_next)
    if (tid == kSmcThreads - 1) {
      const unsigned long long c_end = c_base + btot;
      unsigned long long jn = c_end >= Tr ? jb_hi : first_j_at_least(O + c_end, cb, step_inv);
      s_u64[3] = jn < jb_hi ? jn : jb_hi;
    }
    __syncthreads();
    const unsigned long long j_next = s_u64[3];

    for (unsigned long long j0 = j_cur; j0 < j_next;) {
      const unsigned long long jbase = (j0 / kChunk) * kChunk;
      const unsigned long long j1 = jbase + kChunk < j_next ? jbase + kChunk : j_next;
#pragma unroll
      for (int k = 0; k < kOutPerThread; ++k) mark[kOutPerThread * tid + k] = 0u;
      if (tid == 0) s_carry = 0u;
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kBatchPerThread; ++k) {
        if (f[k] == ~0ull) continue;
        const unsigned int rel = kBatchPerThread * tid + k + 1;  // +1: 0 means "none"
        if (f[k] <= j0) atomicMax(&s_carry, rel);
        else if (f[k] < j1) atomicMax(&mark[f[k] - jbase], rel);
      }
      __syncthreads();
      // inclusive max-scan over this thread's 8 marks, then across threads
      unsigned int run[kOutPerThread];
      unsigned int tm = 0;
#pragma unroll
      for (int k = 0; k < kOutPerThread; ++k) {
        tm = max(tm, mark[kOutPerThread * tid + k]);
        run[k] = tm;
      }
      unsigned int im = tm;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t2 = __shfl_up_sync(0xffffffffu, im, o);
        if (lane >= o) im = max(im, t2);
      }
      if (lane == 31) wmax[warp] = im;
      __syncthreads();
      unsigned int carry = s_carry;
      for (int q = 0; q < warp; ++q) carry = max(carry, wmax[q]);
      const unsigned int prev = __shfl_up_sync(0xffffffffu, im, 1);
      if (lane > 0) carry = max(carry, prev);
      // propagate my outputs
      const unsigned long long jt = jbase + kOutPerThread * tid;
      uint8_t xo[kOutPerThread];
      float lo[kOutPerThread];
      bool any = false, all = true;
#pragma unroll
      for (int h = 0; h < kOutPerThread / 4; ++h) {
        const unsigned long long jq = jt + 4 * h;
        const bool need = jq + 3 >= j0 && jq < j1;
        uint4 wd = make_uint4(0, 0, 0, 0);
        if (need) wd = draw_block(key, jq >> 2, a.t + 1, CUPPL_TAG_SMC_STEP);
        const uint32_t wv[4] = {wd.x, wd.y, wd.z, wd.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int kk = 4 * h + k;
          const unsigned long long j = jq + k;
          const bool valid = j >= j0 && j < j1;
          xo[kk] = 0;
          lo[kk] = 0.f;
          if (valid) {
            const unsigned int anc = max(carry, run[kk]) - 1;  // relative to batch_base
            const int xa = xs[anc];
            const int s = categorical_u64(m.thrA + static_cast<size_t>(xa) * (m.S - 1), m.S, wv[k]);
            const float l = emission(a.y_next, s_mu[s], m.inv_sd, m.c);
            xo[kk] = static_cast<uint8_t>(s);
            lo[kk] = l;
            bmax = fmaxf(bmax, l);
            if (a.anc_out) {
              int q = 0;
              while (q + 1 < a.world && s_rank_begin[q + 1] <= j) ++q;
              a.anc_out[q][j - s_rank_begin[q]] = s_rank_begin[a.rank] + batch_base + anc;
            }
            any = true;
          } else {
            all = false;
          }
        }
      }
      if (any) {
        // owner rank of the first output of the run (ranks own contiguous index ranges)
        int q = 0;
        const unsigned long long jfirst = jt > j0 ? jt : j0;
        while (q + 1 < a.world && s_rank_begin[q + 1] <= jfirst) ++q;
        const unsigned long long dest = jt - s_rank_begin[q];
        const bool same_owner = q + 1 >= a.world || s_rank_begin[q + 1] >= jt + kOutPerThread;
        if (all && same_owner && (dest % kOutPerThread) == 0 && jt >= s_rank_begin[q]) {
          uint2 packed;
          packed.x = xo[0] | (xo[1] << 8) | (xo[2] << 16) | (static_cast<uint32_t>(xo[3]) << 24);
          packed.y = xo[4] | (xo[5] << 8) | (xo[6] << 16) | (static_cast<uint32_t>(xo[7]) << 24);
          *reinterpret_cast<uint2*>(a.x_out[q] + dest) = packed;
          float4* lp = reinterpret_cast<float4*>(a.lw_out[q] + dest);
          __stcs(lp, make_float4(lo[0], lo[1], lo[2], lo[3]));
          __stcs(lp + 1, make_float4(lo[4], lo[5], lo[6], lo[7]));
        } else {
#pragma unroll
          for (int k = 0; k < kOutPerThread; ++k) {
            const unsigned long long j = jt + k;
            if (j >= j0 && j < j1) {
              int qq = 0;
              while (qq + 1 < a.world && s_rank_begin[qq + 1] <= j) ++qq;
              a.x_out[qq][j - s_rank_begin[qq]] = xo[k];
              a.lw_out[qq][j - s_rank_begin[qq]] = lo[k];
            }
          }
        }
      }
      __syncthreads();  // mark / wmax reuse
      j0 = j1;
    }
    j_cur = j_next;
    c_base += btot;
    batch_base += kBatch;
    __syncthreads();  // xs / wsum / s_u64 reuse
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
  if (lane == 0 && bmax > neg_inf_f()) atomicMax(a.m_key_next, f2key(bmax));
}

// ------------------------------------------------------------------ launchers -----------
cudaError_t launch_smc_init(const SmcModel& m, const SmcInitArgs& a, int sm_count, cudaStream_t st) {
  const unsigned long long nq = (a.n_local + 3) / 4;
  unsigned long long g = (nq + kSmcThreads - 1) / kSmcThreads;
  const unsigned long long cap = static_cast<unsigned long long>(sm_count) * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  smc_init_kernel<<<static_cast<unsigned>(g), kSmcThreads, 0, st>>>(m, a);
  return cudaGetLastError();
}

cudaError_t launch_smc_scan(const SmcScanArgs& a, int sm_count, cudaStream_t st) {
  (void)sm_count;
  const unsigned long long n_tiles = (a.n_local + kTile - 1) / kTile;
  if (a.hist)
    smc_scan_kernel<true><<<static_cast<unsigned>(n_tiles), kSmcThreads, 0, st>>>(a);
  else
    smc_scan_kernel<false><<<static_cast<unsigned>(n_tiles), kSmcThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_smc_resample(const SmcModel& m, const SmcResampleArgs& a, int sm_count,
                                cudaStream_t st) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, smc_resample_kernel,
                                                                kSmcThreads, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  unsigned long long g = static_cast<unsigned long long>(sm_count) * per_sm;
  const unsigned long long want = (a.n_local + kBatch - 1) / kBatch;  // ~ one batch per CTA minimum
  if (g > want) g = want > 0 ? want : 1;
  smc_resample_kernel<<<static_cast<unsigned>(g), kSmcThreads, 0, st>>>(m, a);
  return cudaGetLastError();
}

}  // namespace cuppl
