// smc_kernels.cu — K4 init, K5 quantise + tile scan (single-pass decoupled look-back), K6 fused
// systematic resampling + ancestor gather + propagate + reweight, for the bootstrap particle
// filter. SMC has no reference semantics, so
// oracle/cuppl_oracle.c (or_smc_*) *defines* every bit these kernels must reproduce:
//
//   w_i      = min(floor(exp_repro(lw_i - M_t) * 2^31), 2^31)      (u32, exact fp32 sequence)
//   C        = inclusive u64 scan of w; T = C[N-1]
//   target_j = floor((j 2^32 + u) T / (N 2^32)), u = word 0 of Philox(t, 0, 0, TAG_SMC_COMB)
//   a_j      = min{i : C_i > target_j}
//   x'_j     ~ categorical(A[x_{a_j}]): alias draw with word (j & 3) of Philox(j >> 2, t+1, STEP)
//   lw'_j    = log N(y_{t+1}; mu[x'_j], sd)
//
// Data layout per rank: a population is its states x (u8, one byte per particle). In a
// discrete-state HMM the log-weight is a function of the state alone, so each kernel builds the
// S-entry per-step tables lw_s = emission(y_t, mu_s), e_s = exp_repro(lw_s - M_t) and
// w_s = floor(e_s 2^31) in shared memory (same fp32 op sequence as the oracle, which evaluates
// them per particle) and never stores a log-weight. segoff (u64 per 32 particles, tile-local
// inclusive weight prefix) and tile_prefix (u64 per 8192) are the scan outputs. Algorithmic HBM
// traffic per particle-step: K5 reads x (1 B); K6 reads x (1 B) and writes x' (1 B) = 3 B
// (+0.25 B of segment offsets each way).
//
// K6 is output-balanced and source-streaming: CTA b owns an even share of the rank's output
// range, finds the ancestor of its first output once (warp-parallel 33-ary search over the
// segment prefixes), then streams its sources in order in batches of 2048 staged in shared
// memory with their batch-relative inclusive weight prefix. The batch's outputs are exactly
// [F(C_start), F(C_end)) with F(c) = min{j : target_j >= c}; they are propagated in dense
// rounds of 1024 (4 consecutive outputs per thread share one Philox block and one integer comb
// cursor); each output's ancestor is a binary search over the staged prefix, so the work per
// output is uniform whatever the offspring counts.
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

// Alias draw (oracle or_alias_draw): column = high word of w K, coin = low word.
__device__ __forceinline__ int alias_draw(const unsigned long long* tab, int K, uint32_t w) {
  const unsigned long long p = static_cast<unsigned long long>(w) * static_cast<unsigned>(K);
  const int col = static_cast<int>(p >> 32);
  const unsigned long long e = __ldg(tab + col);
  return (p & 0xFFFFFFFFull) < (e & 0x1FFFFFFFFull) ? col : static_cast<int>(e >> 40);
}

// Per-step state tables (shared memory): log-weight, weight factor e and quantised weight of
// every state for observation y and stabiliser M (M = -inf: lw only).
__device__ __forceinline__ void build_tables(const SmcModel& m, float y, float M, float* lwS, float* eS,
                                             uint32_t* wS) {
  for (int s = threadIdx.x; s < m.S; s += blockDim.x) {
    const float l = emission(y, m.mu[s], m.inv_sd, m.c);
    if (lwS) lwS[s] = l;
    if (eS) {
      const float e = smc_e(l, M);
      eS[s] = e;
      wS[s] = smc_w(e);
    }
  }
}

// ------------------------------------------------------------------ K4: init ------------
// x_0[j] ~ categorical(pi0) with word (j & 3) of Philox(j >> 2, 0, TAG_SMC_INIT);
// lw_0[j] = log N(y_0; mu[x_0[j]], sd). One Philox block per 4 particles.
__global__ void __launch_bounds__(kSmcThreads) smc_init_kernel(const __grid_constant__ SmcModel m,
                                                               SmcInitArgs a) {
  __shared__ float lwS[kMaxStates];
  build_tables(m, a.y0, neg_inf_f(), lwS, nullptr, nullptr);
  __syncthreads();
  const PhiloxKey key = make_key(a.key);
  float bmax = neg_inf_f();
  const unsigned long long nq = (a.n_local + 3) / 4;
  for (unsigned long long q = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
       q < nq; q += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const unsigned long long j = a.j_begin + 4 * q;  // global index, multiple of 4
    const uint4 w = draw_block(key, j >> 2, 0u, CUPPL_TAG_SMC_INIT);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    uint32_t packed = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int s = alias_draw(m.alias_init, m.S, ws[k]);
      packed |= static_cast<uint32_t>(s) << (8 * k);
      if (4 * q + k < a.n_local) bmax = fmaxf(bmax, lwS[s]);
    }
    if (4 * q + 3 < a.n_local) {
      *reinterpret_cast<uint32_t*>(a.x + 4 * q) = packed;
    } else {
      for (int k = 0; k < 4; ++k)
        if (4 * q + k < a.n_local) a.x[4 * q + k] = static_cast<uint8_t>(packed >> (8 * k));
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

template <bool HIST>
__global__ void __launch_bounds__(kSmcThreads) smc_scan_kernel(const __grid_constant__ SmcModel m,
                                                               SmcScanArgs a) {
  __shared__ uint32_t wS[kMaxStates];
  __shared__ float eS[kMaxStates];
  __shared__ uint2 wes[kMaxStates];  // (w, bits(e)) in one 64-bit entry: one LDS per particle
  __shared__ unsigned long long wtot[kSmcThreads / 32];
  __shared__ double wpart[kSmcThreads / 32][2];
  __shared__ unsigned int s_tile;
  __shared__ unsigned int cnt[HIST ? kMaxStates : 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long n = a.n_local;
  const unsigned long long n_tiles = (n + kTile - 1) / kTile;
  if (tid == 0) s_tile = atomicAdd(&a.counters[0], 1u);  // launch-order tile ids: look-back is deadlock free
  build_tables(m, a.y, key2f(*a.m_key), nullptr, eS, wS);
  for (int s = tid; s < a.S; s += kSmcThreads) {
    wes[s] = make_uint2(wS[s], __float_as_uint(eS[s]));
    if (HIST) cnt[s] = 0u;
  }
  __syncthreads();
  const unsigned long long tile = s_tile;
  // thread tid owns segment tid of the tile: particles [tile * 8192 + 32 tid, +32)
  const unsigned long long p0 = tile * kTile + static_cast<unsigned long long>(tid) * kSegment;
  uint4 v0 = make_uint4(0, 0, 0, 0), v1 = make_uint4(0, 0, 0, 0);
  int valid = 0;
  if (p0 + kSegment <= n) {
    v0 = __ldcs(reinterpret_cast<const uint4*>(a.x + p0));
    v1 = __ldcs(reinterpret_cast<const uint4*>(a.x + p0) + 1);
    valid = kSegment;
  } else if (p0 < n) {
    valid = static_cast<int>(n - p0);
    uint8_t tmp[kSegment];
    for (int k = 0; k < kSegment; ++k) tmp[k] = k < valid ? a.x[p0 + k] : 0;
    v0 = *reinterpret_cast<const uint4*>(tmp);
    v1 = *reinterpret_cast<const uint4*>(tmp + 16);
  }
  const uint32_t words[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
  unsigned long long ws = 0;
  float s1 = 0.f, s2 = 0.f;
  if (!HIST && valid == kSegment) {  // fast path: a full segment, no per-particle checks
    uint32_t wsum_lo = 0, wsum_hi = 0;  // two u32 halves of 16 weights each never overflow 2^36
#pragma unroll
    for (int k = 0; k < kSegment; ++k) {
      const uint2 te = wes[(words[k >> 2] >> (8 * (k & 3))) & 0xFFu];
      const float e = __uint_as_float(te.y);
      if (k < 16) wsum_lo += te.x >> 4; else wsum_hi += te.x >> 4;
      ws += te.x & 15u;
      s1 += e;
      s2 = fmaf(e, e, s2);
    }
    ws += (static_cast<unsigned long long>(wsum_lo) + wsum_hi) << 4;
  } else {
#pragma unroll
  for (int k = 0; k < kSegment; ++k) {
    const uint32_t st = (words[k >> 2] >> (8 * (k & 3))) & 0xFFu;
    const bool ok = k < valid;
    const uint2 te = wes[st];
    const uint32_t w = ok ? te.x : 0u;
    const float e = ok ? __uint_as_float(te.y) : 0.f;
    ws += w;
    s1 += e;
    s2 = fmaf(e, e, s2);
    if (HIST) {
      // warp-aggregated state counts: one shared atomic per distinct state in the warp
      const unsigned int key = ok ? st : 0xFFFFFFFFu;
      const unsigned int grp = __match_any_sync(0xffffffffu, key);
      if (ok && lane == __ffs(grp) - 1) atomicAdd(&cnt[st], static_cast<unsigned int>(__popc(grp)));
    }
  }
  }
  double d1 = s1, d2 = s2;  // per-warp fp64 partials, fixed tree
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d1 += __shfl_down_sync(0xffffffffu, d1, o);
    d2 += __shfl_down_sync(0xffffffffu, d2, o);
  }
  if (lane == 0) {
    wpart[warp][0] = d1;
    wpart[warp][1] = d2;
  }
  // inclusive scan of the tile's 256 segment sums (thread tid <-> segment tid)
  unsigned long long incl = ws;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  unsigned long long wpre = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kSmcThreads / 32; ++w) {
    if (w < warp) wpre += wtot[w];
    agg += wtot[w];
  }
  const unsigned long long gs = tile * kTileSegs + tid;
  if (gs * kSegment < n) a.segoff[gs] = incl + wpre;  // tile-local; K6 adds tile_prefix
  if (HIST) {
    for (int s = tid; s < a.S; s += kSmcThreads)
      if (cnt[s]) atomicAdd(&a.hist[s], static_cast<unsigned long long>(cnt[s]) * wS[s]);
  }
  if (warp != 0) return;  // only warp 0 waits on the predecessors
  if (lane == 0) st_relaxed_u64(a.flags + tile, (tile == 0 ? kFlagIncl : kFlagAgg) | agg);
  const unsigned long long prefix = tile == 0 ? 0ull : warp_lookback(a.flags, tile);
  if (lane == 0) {
    if (tile != 0) st_relaxed_u64(a.flags + tile, kFlagIncl | (prefix + agg));
    a.tile_prefix[tile] = prefix;
    double t1 = 0.0, t2 = 0.0;
    for (int w = 0; w < kSmcThreads / 32; ++w) {
      t1 += wpart[w][0];
      t2 += wpart[w][1];
    }
    a.tile_s[2 * tile] = t1;
    a.tile_s[2 * tile + 1] = t2;
    if (tile == n_tiles - 1) a.rank_rec[0] = prefix + agg;  // T_r
  }
}

// ------------------------------------------------------------------ K6: resample --------
// Comb in integers (D6): with T = Q N + R0 and A = floor(u T / 2^32) = Qa N + Ra,
// target_j = floor((j 2^32 + u) T / (N 2^32)) = j Q + Qa + floor((j R0 + Ra) / N),
// where j R0 + Ra < N^2 < 2^62 (N < 2^31); every per-index quantity fits 32 bits.
struct Comb {
  unsigned int N, Q, R0, Qa, Ra;
  double invN, step_inv, a_over_t;  // 1/N, N/T, A/T
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

// Cursor over consecutive targets: (j, target_j, (j R0 + Ra) mod N).
struct CombCursor {
  unsigned int j, mod;
  unsigned long long tgt;
  __device__ __forceinline__ void seek(unsigned int jj, const Comb& cb) {
    j = jj;
    const unsigned long long q =
        div_n(static_cast<unsigned long long>(jj) * cb.R0 + cb.Ra, cb, &mod);
    tgt = static_cast<unsigned long long>(jj) * cb.Q + cb.Qa + q;
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
  // smallest j' >= j with target_j' >= c (N if none); long gaps re-seek from an estimate
  __device__ __forceinline__ void advance_to(unsigned long long c, const Comb& cb) {
    if (j >= cb.N || tgt >= c) return;
    if (c - tgt > 4ull * cb.Q + 4ull) {
      // target_j ~ (j + u/2^32) T / N  =>  j ~ c N / T - u / 2^32 (error << 1)
      const double e = __dmul_rn(__ull2double_rn(c), cb.step_inv) - 2.0;
      const unsigned int jj = e <= static_cast<double>(j) ? j
                             : e >= static_cast<double>(cb.N) ? cb.N - 1
                                                              : static_cast<unsigned int>(e);
      if (jj > j) {
        seek(jj, cb);
        while (j > 0 && tgt >= c) seek(j - 1, cb);  // never taken unless the estimate was high
      }
    }
    while (j < cb.N && tgt < c) next(cb);
  }
};

__device__ __forceinline__ unsigned long long comb_target(unsigned int j, const Comb& cb) {
  CombCursor c;
  c.seek(j, cb);
  return c.tgt;
}

// smallest j in [0, N] with target_j >= c (N if none). target_j >= c <=> j T + A >= c N, so
// F(c) = ceil((c N - A) / T): fp64 estimate, then exact fix-up on the integer targets.
__device__ __forceinline__ unsigned int first_j_at_least(unsigned long long c, const Comb& cb) {
  if (c == 0) return 0u;
  const double est = __dmul_rn(__ull2double_rn(c), cb.step_inv) - cb.a_over_t;
  unsigned int j = est <= 0.0 ? 0u : est >= static_cast<double>(cb.N) ? cb.N : static_cast<unsigned int>(ceil(est));
  while (j > 0 && comb_target(j - 1, cb) >= c) --j;
  while (j < cb.N && comb_target(j, cb) < c) ++j;
  return j;
}

// Rank-local inclusive weight prefix at the end of segment s (K5 writes tile-local values).
__device__ __forceinline__ unsigned long long seg_incl(const SmcResampleArgs& a, unsigned long long s) {
  return __ldg(a.tile_prefix + s / kTileSegs) + __ldg(a.segoff + s);
}

// Warp-cooperative rank-local upper bound: smallest local i with C_i > t (C = inclusive scan
// of the rank's weights, represented by the segment prefixes + the lw of one segment). Returns
// n_local if none. The segment is found with a 33-ary search (5 rounds for 3e6 segments), then
// resolved inside the segment with a warp scan of its 32 weights.
__device__ unsigned long long warp_upper_bound(unsigned long long t, const SmcResampleArgs& a,
                                               const uint32_t* wS) {
  const int lane = threadIdx.x & 31;
  const unsigned long long n_segs = (a.n_local + kSegment - 1) / kSegment;
  unsigned long long lo = 0, hi = n_segs;  // invariant: answer in [lo, hi]
  while (hi - lo > 32) {
    const unsigned long long span = hi - lo;
    const unsigned long long p = lo + span * (lane + 1) / 33;  // strictly increasing, < hi
    const unsigned int bal = __ballot_sync(0xffffffffu, seg_incl(a, p) > t);
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
    const unsigned int bal = __ballot_sync(0xffffffffu, p < hi && seg_incl(a, p) > t);
    hi = bal ? lo + (__ffs(bal) - 1) : hi;
  }
  const unsigned long long s = hi;
  if (s >= n_segs) return a.n_local;
  const unsigned long long base = s > 0 ? seg_incl(a, s - 1) : 0ull;
  const unsigned long long i = s * kSegment + lane;
  const uint32_t w = i < a.n_local ? wS[a.x[i]] : 0u;
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

template <bool MULTI, bool DEBUG>
__global__ void __launch_bounds__(kSmcThreads, 3) smc_resample_kernel(const __grid_constant__ SmcModel m,
                                                                      SmcResampleArgs a) {
  __shared__ unsigned long long cb_incl[kBatch];  // batch-relative inclusive weight prefix per source
  __shared__ uint8_t xs[kBatch];                  // staged source states
  __shared__ __align__(16) uint8_t obuf[kOutBuf + 16];  // new states, indexed from o0 & ~15
  __shared__ unsigned long long wsum[kSmcThreads / 32];
  __shared__ unsigned long long s_u64[4];
  __shared__ unsigned long long s_rank_begin[MULTI ? kMaxRanks + 1 : 1];
  __shared__ uint32_t wS[kMaxStates];   // quantised weights of population t per state
  __shared__ float lwS1[kMaxStates];    // log-weights of population t + 1 per state
  __shared__ BlockScratch sc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (MULTI)
    for (int q = tid; q <= a.world; q += kSmcThreads) s_rank_begin[q] = a.rank_begin[q];
  constexpr bool debug_anc = DEBUG;
  const unsigned long long n_tiles = a.n_tiles;

  // CTA 0: fixed-order fp64 fold of K5's per-tile sums -> rank (sum e, sum e^2); reset K5's
  // tile counter. Every CTA clears a slice of the look-back words for the next scan.
  if (blockIdx.x == 0) {
    double f1 = 0.0, f2 = 0.0;
    for (unsigned long long tt = tid; tt < n_tiles; tt += kSmcThreads) {
      f1 += a.tile_s[2 * tt];
      f2 += a.tile_s[2 * tt + 1];
    }
    f1 = block_sum_d(f1, sc);
    f2 = block_sum_d(f2, sc);
    if (tid == 0) {
      a.stats_out[0] = f1;
      a.stats_out[1] = f2;
      a.counters[0] = 0u;
    }
  }
  for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(kSmcThreads) + tid; i < n_tiles;
       i += static_cast<unsigned long long>(gridDim.x) * kSmcThreads)
    a.flags_to_clear[i] = 0ull;

  // step constants (identical on every rank)
  unsigned long long T = 0, O = 0;
  for (int q = 0; q < a.world; ++q) {
    const unsigned long long Tq = a.rank_recs[4 * q];
    if (q < a.rank) O += Tq;
    T += Tq;
  }
  const unsigned long long Tr = a.rank_recs[4 * a.rank];
  if (T == 0) return;  // all weights zero: the host raises AllZeroWeightError
  {
    __shared__ float eS[kMaxStates];
    build_tables(m, a.y_cur, key2f(*a.m_key), nullptr, eS, wS);
    build_tables(m, a.y_next, neg_inf_f(), lwS1, nullptr, nullptr);
  }
  __syncthreads();
  const PhiloxKey key = make_key(a.key);
  Comb cb;
  cb.u = draw_block(key, a.t, 0u, CUPPL_TAG_SMC_COMB).x;
  cb.N = static_cast<unsigned int>(a.n_total);
  cb.Q = static_cast<unsigned int>(T / cb.N);
  cb.R0 = static_cast<unsigned int>(T % cb.N);
  const unsigned long long A = __umul64hi(static_cast<unsigned long long>(cb.u) << 32, T);  // floor(u T / 2^32)
  cb.Qa = static_cast<unsigned int>(A / cb.N);
  cb.Ra = static_cast<unsigned int>(A % cb.N);
  cb.invN = 1.0 / static_cast<double>(cb.N);
  cb.step_inv = static_cast<double>(cb.N) / static_cast<double>(T);
  cb.a_over_t = static_cast<double>(A) / static_cast<double>(T);

  // this rank's outputs: J_r = {j : O <= target_j < O + Tr}; this CTA's even share of it
  if (tid == 0) {
    s_u64[0] = a.rank == 0 ? 0ull : first_j_at_least(O, cb);
    s_u64[1] = a.rank == a.world - 1 ? cb.N : first_j_at_least(O + Tr, cb);
  }
  __syncthreads();
  const unsigned long long jr_lo = s_u64[0], jr_hi = s_u64[1];
  const unsigned long long span = jr_hi - jr_lo;
  const unsigned long long jb_lo = jr_lo + span * blockIdx.x / gridDim.x;
  const unsigned long long jb_hi = jr_lo + span * (blockIdx.x + 1) / gridDim.x;
  if (jb_lo >= jb_hi) return;

  // ancestor of the first output -> first batch starts at its segment boundary
  if (warp == 0) {
    const unsigned long long tl = comb_target(static_cast<unsigned int>(jb_lo), cb) - O;
    const unsigned long long i0 = warp_upper_bound(tl, a, wS);
    if (lane == 0) s_u64[2] = i0;
  }
  __syncthreads();
  unsigned long long batch_base = (s_u64[2] / kSegment) * kSegment;
  unsigned long long c_base = batch_base > 0 ? seg_incl(a, batch_base / kSegment - 1) : 0ull;
  unsigned long long j_cur = jb_lo;
  float bmax = neg_inf_f();
  const unsigned int S = static_cast<unsigned int>(m.S);

  while (j_cur < jb_hi && batch_base < a.n_local) {
    // ---- stage 2048 sources: thread tid owns [batch_base + 8 tid, +8)
    const unsigned long long i0 = batch_base + kBatchPerThread * tid;
    uint32_t w[kBatchPerThread];
    unsigned long long tw = 0;
    if (i0 + kBatchPerThread <= a.n_local) {
      const uint4 xx = __ldcs(reinterpret_cast<const uint4*>(a.x + i0));
      *reinterpret_cast<uint4*>(xs + kBatchPerThread * tid) = xx;
      const uint32_t xw[4] = {xx.x, xx.y, xx.z, xx.w};
#pragma unroll
      for (int k = 0; k < kBatchPerThread; ++k) {
        w[k] = wS[(xw[k >> 2] >> (8 * (k & 3))) & 0xFFu];
        tw += w[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < kBatchPerThread; ++k) {
        const bool ok = i0 + k < a.n_local;
        const uint8_t st = ok ? a.x[i0 + k] : 0;
        w[k] = ok ? wS[st] : 0u;
        xs[kBatchPerThread * tid + k] = st;
        tw += w[k];
      }
    }
    // block exclusive scan of the thread sums -> batch-relative inclusive prefix per source
    unsigned long long incl = tw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t2 = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t2;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    unsigned long long run = 0, btot = 0;
#pragma unroll
    for (int q = 0; q < kSmcThreads / 32; ++q) {
      if (q < warp) run += wsum[q];
      btot += wsum[q];
    }
    run += incl - tw;
#pragma unroll
    for (int k = 0; k < kBatchPerThread; ++k) {
      run += w[k];
      cb_incl[kBatchPerThread * tid + k] = run;
    }
    // outputs whose ancestors lie in this batch: [j_cur, j_next), j_next = F(C at batch end)
    if (tid == kSmcThreads - 1) {
      const unsigned long long c_end = c_base + btot;
      const unsigned long long jn = c_end >= Tr ? jb_hi : first_j_at_least(O + c_end, cb);
      s_u64[3] = jn < jb_hi ? jn : jb_hi;
    }
    __syncthreads();
    const unsigned long long j_next = s_u64[3];
    const unsigned long long off = O + c_base;  // global target of batch-relative weight 0

    // propagate [j_cur, j_next) in sub-rounds of at most kOutBuf outputs; thread tid takes an
    // equal slice of consecutive outputs, finds the ancestor of its first by a branchless binary
    // search over the staged prefix and the rest with a monotone merge pointer (targets increase
    // with j); the new states are staged in shared memory and written out coalesced.
    for (unsigned long long o0 = j_cur; o0 < j_next; o0 += kOutBuf) {
      const unsigned long long o1 = o0 + kOutBuf < j_next ? o0 + kOutBuf : j_next;
      const unsigned int n_out = static_cast<unsigned int>(o1 - o0);
      const unsigned long long ob = o0 & ~15ull;  // obuf[j - ob]: same 16-byte phase as the owners' x
      // slices of consecutive outputs, 4-aligned in j so a thread's Philox blocks (4 outputs
      // each) are drawn at the same iteration by every lane
      const unsigned long long a4 = o0 & ~3ull;
      const unsigned int span4 = static_cast<unsigned int>(o1 - a4);
      const unsigned int per = ((span4 + kSmcThreads - 1) / kSmcThreads + 3) & ~3u;
      const unsigned long long q0 = a4 + static_cast<unsigned long long>(tid) * per;
      const unsigned long long q1 = q0 + per < o1 ? q0 + per : o1;
      const unsigned long long qs = q0 > o0 ? q0 : o0;
      if (qs < q1) {
        CombCursor cc;
        cc.seek(static_cast<unsigned int>(qs), cb);
        int k;
        {  // smallest k with cb_incl[k] > t (exists: t < batch total): branchless, 12 steps
          const unsigned long long t = cc.tgt - off;
          int kk = 0;
#pragma unroll
          for (int step = kBatch / 2; step >= 1; step >>= 1)
            kk += (cb_incl[kk + step - 1] <= t) ? step : 0;
          k = kk;
        }
        for (unsigned long long jg = q0; jg < q1; jg += 4) {
          const uint4 wd = draw_block(key, jg >> 2, a.t + 1, CUPPL_TAG_SMC_STEP);
          const uint32_t wv[4] = {wd.x, wd.y, wd.z, wd.w};
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const unsigned long long j = jg + h;
            if (j < qs || j >= q1) continue;
            const unsigned long long t = cc.tgt - off;  // batch-relative target, < btot
            while (cb_incl[k] <= t) ++k;
            const int xa = xs[k];
            const int st = alias_draw(m.alias_trans + static_cast<size_t>(xa) * S, m.S, wv[h]);
            obuf[j - ob] = static_cast<uint8_t>(st);
            bmax = fmaxf(bmax, lwS1[st]);
            if (debug_anc) {
              int r = 0;
              if (MULTI)
                while (r + 1 < a.world && s_rank_begin[r + 1] <= j) ++r;
              const unsigned long long rb = MULTI ? s_rank_begin[r] : 0ull;
              const unsigned long long my = MULTI ? s_rank_begin[a.rank] : 0ull;
              a.anc_out[r][j - rb] = my + batch_base + k;
            }
            cc.next(cb);
          }
        }
      }
      (void)n_out;
      __syncthreads();
      // coalesced copy-out of obuf[0, n_out) -> owners' x at global index o0 + i
      int r = 0;
      if (MULTI)
        while (r + 1 < a.world && s_rank_begin[r + 1] <= o0) ++r;
      unsigned long long g = o0;
      while (g < o1) {
        const unsigned long long rb = MULTI ? s_rank_begin[r] : 0ull;
        const unsigned long long re = MULTI ? (r + 1 < a.world ? s_rank_begin[r + 1] : cb.N) : o1;
        const unsigned long long e = re < o1 ? re : o1;
        uint8_t* dst = a.x_out[r] + (g - rb);
        const uint8_t* src = obuf + (g - ob);  // 16-byte phase of src == phase of dst
        const unsigned int len = static_cast<unsigned int>(e - g);
        // head bytes up to 16-byte alignment of dst, then uint4 chunks, then tail bytes
        const unsigned int head = static_cast<unsigned int>((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15);
        const unsigned int hb = head < len ? head : len;
        if (tid < hb) dst[tid] = src[tid];
        const unsigned int nv = (len - hb) / 16;
        for (unsigned int v = tid; v < nv; v += kSmcThreads)
          __stcs(reinterpret_cast<uint4*>(dst + hb) + v, reinterpret_cast<const uint4*>(src + hb)[v]);
        for (unsigned int i = hb + 16 * nv + tid; i < len; i += kSmcThreads) dst[i] = src[i];
        g = e;
        ++r;
      }
      __syncthreads();  // obuf reuse
    }
    __syncthreads();  // cb_incl / xs / wsum / s_u64 reuse
    j_cur = j_next;
    c_base += btot;
    batch_base += kBatch;
  }
  if (MULTI) __threadfence_system();  // peer stores performed before the next collective
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
  if (lane == 0 && bmax > neg_inf_f()) atomicMax(a.m_key_next, f2key(bmax));
}

// Fixed-order fold of K5's per-tile sums for a population that is not resampled (the last
// step): same arithmetic as K6's CTA 0.
__global__ void __launch_bounds__(kSmcThreads) smc_fold_kernel(const double* tile_s,
                                                               unsigned long long n_tiles,
                                                               double* stats_out,
                                                               unsigned int* counters) {
  __shared__ BlockScratch sc;
  double f1 = 0.0, f2 = 0.0;
  for (unsigned long long tt = threadIdx.x; tt < n_tiles; tt += kSmcThreads) {
    f1 += tile_s[2 * tt];
    f2 += tile_s[2 * tt + 1];
  }
  f1 = block_sum_d(f1, sc);
  f2 = block_sum_d(f2, sc);
  if (threadIdx.x == 0) {
    stats_out[0] = f1;
    stats_out[1] = f2;
    counters[0] = 0u;
  }
}

cudaError_t launch_smc_fold(const double* tile_s, unsigned long long n_tiles, double* stats_out,
                            unsigned int* counters, cudaStream_t st) {
  smc_fold_kernel<<<1, kSmcThreads, 0, st>>>(tile_s, n_tiles, stats_out, counters);
  return cudaGetLastError();
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

cudaError_t launch_smc_scan(const SmcModel& m, const SmcScanArgs& a, int sm_count, cudaStream_t st) {
  (void)sm_count;
  const unsigned long long n_tiles = (a.n_local + kTile - 1) / kTile;
  if (a.hist)
    smc_scan_kernel<true><<<static_cast<unsigned>(n_tiles), kSmcThreads, 0, st>>>(m, a);
  else
    smc_scan_kernel<false><<<static_cast<unsigned>(n_tiles), kSmcThreads, 0, st>>>(m, a);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kSmcThreads) smc_log_weights_kernel(const __grid_constant__ SmcModel m,
                                                                      float y, const uint8_t* x,
                                                                      unsigned long long n, float* lw) {
  __shared__ float lwS[kMaxStates];
  build_tables(m, y, neg_inf_f(), lwS, nullptr, nullptr);
  __syncthreads();
  for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<unsigned long long>(gridDim.x) * blockDim.x)
    lw[i] = lwS[x[i]];
}

cudaError_t launch_smc_log_weights(const SmcModel& m, float y, const uint8_t* x, unsigned long long n,
                                   float* lw, int sm_count, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  unsigned long long g = (n + kSmcThreads - 1) / kSmcThreads;
  const unsigned long long cap = static_cast<unsigned long long>(sm_count) * 8;
  if (g > cap) g = cap;
  smc_log_weights_kernel<<<static_cast<unsigned>(g), kSmcThreads, 0, st>>>(m, y, x, n, lw);
  return cudaGetLastError();
}

template <bool MULTI, bool DEBUG>
static cudaError_t launch_resample_t(const SmcModel& m, const SmcResampleArgs& a, int sm_count,
                                     cudaStream_t st) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, smc_resample_kernel<MULTI, DEBUG>,
                                                                kSmcThreads, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  unsigned long long g = static_cast<unsigned long long>(sm_count) * per_sm;
  const unsigned long long want = (a.n_local + kBatch - 1) / kBatch;  // >= one batch per CTA
  if (g > want) g = want > 0 ? want : 1;
  smc_resample_kernel<MULTI, DEBUG><<<static_cast<unsigned>(g), kSmcThreads, 0, st>>>(m, a);
  return cudaGetLastError();
}

cudaError_t launch_smc_resample(const SmcModel& m, const SmcResampleArgs& a, int sm_count,
                                cudaStream_t st) {
  if (a.anc_out)
    return a.world > 1 ? launch_resample_t<true, true>(m, a, sm_count, st)
                       : launch_resample_t<false, true>(m, a, sm_count, st);
  return a.world > 1 ? launch_resample_t<true, false>(m, a, sm_count, st)
                     : launch_resample_t<false, false>(m, a, sm_count, st);
}

}  // namespace cuppl
