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
// range, finds the tile holding the ancestor of its first output once (warp-parallel 33-ary
// search over the tile prefixes), then streams its source tiles (4096 states staged in shared
// memory, batch-relative exact integer weight prefix per thread). It RANKS EVERY SOURCE INTO
// THE COMB instead of searching per output: the targets are an arithmetic progression, so
// source k's children are exactly [F(C_{k-1}), F(C_k)) with F(c) = min{j : target_j >= c}, an
// fp64 estimate with an exact 128-bit fix-up near integers (smc_common.cuh comb_rank). A source
// with children in the current 8192-position output window marks its first child's position;
// an output's ancestor is the last mark at or before it (a block max-scan, since marks increase
// with the position). Thread t then draws outputs [wb + 16t, +16) and [wb + 16(t + 256), +16):
// 4 Philox blocks per 16 outputs, alias tables in shared memory, one 16-byte store. The work per
// source and per output is uniform whatever the offspring counts.
#include "cuppl_device.cuh"
#include "smc_common.cuh"
#include "smc_kernels.cuh"

namespace cuppl {

__device__ __forceinline__ float emission(float y, float mu, float inv_sd, float c) {
  const float z = __fmul_rn(__fsub_rn(y, mu), inv_sd);
  return __fmaf_rn(__fmul_rn(-0.5f, z), z, c);
}

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
  const PhiloxKey key = make_key(a.key_dev ? *a.key_dev : a.key);
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
template <bool HIST>
__global__ void __launch_bounds__(kSmcThreads) smc_scan_kernel(const __grid_constant__ SmcModel m,
                                                               SmcScanArgs a) {
  __shared__ uint32_t wS[kMaxStates];
  __shared__ float eS[kMaxStates];
  __shared__ uint2 wes[kMaxStates];  // (w, bits(e)) in one 64-bit entry: one LDS per particle
  __shared__ unsigned long long wtot[kScanTiles][kSmcThreads / 32];
  __shared__ double wpart[kSmcThreads / 32][2];
  __shared__ unsigned int s_blk;
  __shared__ unsigned int cnt[HIST ? kMaxStates : 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long n = a.n_local;
  const unsigned long long n_tiles = (n + kTile - 1) / kTile;
  const unsigned long long n_blocks = (n_tiles + kScanTiles - 1) / kScanTiles;
  if (tid == 0) s_blk = atomicAdd(&a.counters[0], 1u);  // launch-order ids: look-back is deadlock free
  build_tables(m, a.y, key2f(*a.m_key), nullptr, eS, wS);
  for (int s = tid; s < a.S; s += kSmcThreads) {
    wes[s] = make_uint2(wS[s], __float_as_uint(eS[s]));
    if (HIST) cnt[s] = 0u;
  }
  __syncthreads();
  const unsigned long long blk = s_blk;
  const unsigned long long tile0 = blk * kScanTiles;
  // thread tid owns particles [tile * 4096 + 16 tid, +16) of each of the CTA's 8 tiles: all
  // eight 16-byte loads are issued before any is used
  uint4 v[kScanTiles];
  int valid[kScanTiles];
#pragma unroll
  for (int u = 0; u < kScanTiles; ++u) {
    const unsigned long long p0 = (tile0 + u) * kTile + static_cast<unsigned long long>(tid) * kSegment;
    v[u] = make_uint4(0, 0, 0, 0);
    valid[u] = 0;
    if (p0 + kSegment <= n) {
      v[u] = __ldcs(reinterpret_cast<const uint4*>(a.x + p0));
      valid[u] = kSegment;
    } else if (p0 < n) {
      valid[u] = static_cast<int>(n - p0);
      uint8_t tmp[kSegment];
      for (int k = 0; k < kSegment; ++k) tmp[k] = k < valid[u] ? a.x[p0 + k] : 0;
      v[u] = *reinterpret_cast<const uint4*>(tmp);
    }
  }
  double d1 = 0.0, d2 = 0.0;  // fp32 over each 16-particle slice, fp64 across slices (D10)
#pragma unroll
  for (int u = 0; u < kScanTiles; ++u) {
    const uint32_t words[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
    unsigned long long ws = 0;
    float s1 = 0.f, s2 = 0.f;
    if (!HIST && valid[u] == kSegment) {  // fast path: a full thread slice, no per-particle checks
#pragma unroll
      for (int k = 0; k < kSegment; ++k) {
        const uint2 te = wes[(words[k >> 2] >> (8 * (k & 3))) & 0xFFu];
        const float e = __uint_as_float(te.y);
        ws += te.x;
        s1 += e;
        s2 = fmaf(e, e, s2);
      }
    } else {
#pragma unroll
      for (int k = 0; k < kSegment; ++k) {
        const uint32_t st = (words[k >> 2] >> (8 * (k & 3))) & 0xFFu;
        const bool ok = k < valid[u];
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
    d1 += s1;
    d2 += s2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ws += __shfl_down_sync(0xffffffffu, ws, o);
    if (lane == 0) wtot[u][warp] = ws;
  }
  // per-warp fp64 partials, fixed tree
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d1 += __shfl_down_sync(0xffffffffu, d1, o);
    d2 += __shfl_down_sync(0xffffffffu, d2, o);
  }
  if (lane == 0) {
    wpart[warp][0] = d1;
    wpart[warp][1] = d2;
  }
  __syncthreads();
  if (HIST) {
    for (int s = tid; s < a.S; s += kSmcThreads)
      if (cnt[s]) atomicAdd(&a.hist[s], static_cast<unsigned long long>(cnt[s]) * wS[s]);
  }
  if (warp != 0) return;  // only warp 0 waits on the predecessors
  // lane u < 8: aggregate of tile u, then the exclusive offsets of the tiles inside the block
  unsigned long long tagg = 0;
  if (lane < kScanTiles) {
#pragma unroll
    for (int w = 0; w < kSmcThreads / 32; ++w) tagg += wtot[lane][w];
  }
  unsigned long long tincl = tagg;
#pragma unroll
  for (int o = 1; o < kScanTiles; o <<= 1) {
    const unsigned long long t2 = __shfl_up_sync(0xffffffffu, tincl, o);
    if (lane >= o) tincl += t2;
  }
  const unsigned long long agg = __shfl_sync(0xffffffffu, tincl, kScanTiles - 1);
  if (lane == 0) st_relaxed_u64(a.flags + blk, (blk == 0 ? kFlagIncl : kFlagAgg) | agg);
  const unsigned long long prefix = blk == 0 ? 0ull : warp_lookback(a.flags, blk);
  if (lane == 0 && blk != 0) st_relaxed_u64(a.flags + blk, kFlagIncl | (prefix + agg));
  if (lane < kScanTiles && tile0 + lane < n_tiles) a.tile_prefix[tile0 + lane] = prefix + tincl - tagg;
  if (lane == 0) {
    double t1 = 0.0, t2 = 0.0;
    for (int w = 0; w < kSmcThreads / 32; ++w) {
      t1 += wpart[w][0];
      t2 += wpart[w][1];
    }
    a.tile_s[2 * blk] = t1;
    a.tile_s[2 * blk + 1] = t2;
    if (blk == n_blocks - 1) a.rank_rec[0] = prefix + agg;  // T_r
  }
}

// ------------------------------------------------------------------ K6: resample --------
// K6: CTA b owns an even share [jb_lo, jb_hi) of this rank's outputs. It stages its sources
// tile by tile (the 4096-particle K5 tiles: states in shared memory, batch-relative integer
// weight prefix in registers) and RANKS EVERY SOURCE INTO THE COMB: the comb targets are an
// arithmetic progression, so the first child of source k is F(C_{k-1}) and its children are
// [F(C_{k-1}), F(C_k)) -- O(1) arithmetic per source instead of a search per output. Each
// source with children marks its first child's position in a 4096-output window; an output's
// ancestor is the last mark at or before it (a block max-scan, since marks increase with the
// position). Thread t then draws the new states of outputs [wb + 16 t, +16) (4 Philox blocks,
// alias tables in shared memory) and stores them as one 16-byte write. No per-output search,
// no data-dependent loop: the work per output and per source is uniform whatever the
// offspring counts.
template <bool MULTI, bool DEBUG, bool SMEM_ALIAS>
#ifndef CUPPL_SMC_MINBLOCKS
#define CUPPL_SMC_MINBLOCKS 4
#endif
__global__ void __launch_bounds__(kSmcThreads, CUPPL_SMC_MINBLOCKS) smc_resample_kernel(const __grid_constant__ SmcModel m,
                                                                      SmcResampleArgs a) {
  extern __shared__ __align__(16) unsigned long long alias_s[];  // [S][S] (SMEM_ALIAS)
  __shared__ __align__(16) uint8_t xs[kBatch];         // staged source states
  __shared__ __align__(16) uint16_t marks[kWindow];    // batch index + 1 of a first child
  __shared__ uint8_t present[kMaxStates];              // states drawn into population t + 1
  __shared__ unsigned long long wsum[kSmcThreads / 32];
  __shared__ unsigned int wmax[2 * (kSmcThreads / 32)];  // warp totals of both window halves
  __shared__ unsigned long long s_u64[4];
  __shared__ unsigned int s_jn;
  __shared__ unsigned long long s_rank_begin[MULTI ? kMaxRanks + 1 : 1];
  __shared__ uint32_t wS[kMaxStates];   // quantised weights of population t per state
  __shared__ double wdS[kMaxStates];    // the same as doubles (exact)
  __shared__ float lwS1[kMaxStates];    // log-weights of population t + 1 per state
  __shared__ BlockScratch sc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (MULTI)
    for (int q = tid; q <= a.world; q += kSmcThreads) s_rank_begin[q] = a.rank_begin[q];
  const unsigned long long n_tiles = a.n_tiles;
  const unsigned int S = static_cast<unsigned int>(m.S);

  // CTA 0: fixed-order fp64 fold of K5's per-tile sums -> rank (sum e, sum e^2); reset K5's
  // tile counter. Every CTA clears a slice of the look-back words for the next scan.
  if (blockIdx.x == 0) {
    double f1 = 0.0, f2 = 0.0;
    for (unsigned long long tt = tid; tt < a.n_scan_blocks; tt += kSmcThreads) {
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
  for (int i = tid; i < kWindow / 8; i += kSmcThreads) reinterpret_cast<uint4*>(marks)[i] = make_uint4(0, 0, 0, 0);
  for (int s = tid; s < kMaxStates; s += kSmcThreads) present[s] = 0;
  if (SMEM_ALIAS) {
    // compact entries: low word thr - 1, high word (kept state) | (alias << 16), where the kept
    // state is the column, or the alias when thr == 0 (never kept): coin < thr <=> coin <= thr - 1
    const unsigned int nA = S * S;
    for (unsigned int i = tid; i < nA; i += kSmcThreads) {
      const unsigned long long e = __ldg(m.alias_trans + i);
      const unsigned long long thr = e & 0x1FFFFFFFFull;
      const unsigned int al = static_cast<unsigned int>(e >> 40), col = i % S;
      const unsigned int keep = thr == 0 ? al : col;
      alias_s[i] = (thr == 0 ? 0ull : thr - 1) | (static_cast<unsigned long long>(keep | (al << 16)) << 32);
    }
  }
  __syncthreads();
  for (int s = tid; s < m.S; s += kSmcThreads) wdS[s] = static_cast<double>(wS[s]);
  const PhiloxKey key = make_key(a.key_dev ? *a.key_dev : a.key);
  __shared__ Comb s_cb;  // step constants (the rare exact rank path reads them here)
  if (tid == 0) {
    Comb c;
    c.u = draw_block(key, a.t, 0u, CUPPL_TAG_SMC_COMB).x;
    c.N = static_cast<unsigned int>(a.n_total);
    c.T = T;
    c.Q = static_cast<unsigned int>(T / c.N);
    c.R0 = static_cast<unsigned int>(T % c.N);
    c.A = __umul64hi(static_cast<unsigned long long>(c.u) << 32, T);  // floor(u T / 2^32)
    c.Qa = static_cast<unsigned int>(c.A / c.N);
    c.Ra = static_cast<unsigned int>(c.A % c.N);
    c.invN = 1.0 / static_cast<double>(c.N);
    c.n_over_t = static_cast<double>(c.N) / static_cast<double>(T);
    c.a_over_t = static_cast<double>(c.A) / static_cast<double>(T);
    s_cb = c;
  }
  __syncthreads();
  const Comb& cb = s_cb;
  const double n_over_t = cb.n_over_t;

  // this rank's outputs: J_r = {j : O <= target_j < O + Tr}; this CTA's even share of it
  if (tid == 0) {
    s_u64[0] = a.rank == 0 ? 0ull : comb_rank(O, cb);
    s_u64[1] = a.rank == a.world - 1 ? cb.N : comb_rank(O + Tr, cb);
  }
  __syncthreads();
  const unsigned long long jr_lo = s_u64[0], jr_hi = s_u64[1];
  const unsigned long long span = jr_hi - jr_lo;
  const unsigned long long jb_lo = jr_lo + span * blockIdx.x / gridDim.x;
  const unsigned long long jb_hi = jr_lo + span * (blockIdx.x + 1) / gridDim.x;
  if (jb_lo >= jb_hi) return;

  // the tile holding the ancestor of the first output: the last tile whose exclusive prefix
  // is <= its (rank-local) target (warp-cooperative 33-ary search over the tile prefixes)
  if (warp == 0) {
    const unsigned long long tl = comb_target(static_cast<unsigned int>(jb_lo), cb) - O;
    unsigned long long lo = 0, hi = n_tiles;  // answer in [lo, hi): prefix[lo] <= tl
    while (hi - lo > 32) {
      const unsigned long long sp = hi - lo;
      const unsigned long long p = lo + sp * (lane + 1) / 33;  // increasing, in (lo, hi)
      const unsigned int bal = __ballot_sync(0xffffffffu, __ldg(a.tile_prefix + p) > tl);
      if (!bal) {
        lo = lo + sp * 32 / 33;
      } else {
        const int fl = __ffs(bal) - 1;  // first probe above tl
        hi = lo + sp * (fl + 1) / 33;
        if (fl > 0) lo = lo + sp * fl / 33;
      }
    }
    const unsigned long long p = lo + lane;
    const unsigned int bal = __ballot_sync(0xffffffffu, p < hi && __ldg(a.tile_prefix + p) <= tl);
    if (lane == 0) s_u64[2] = lo + (31 - __clz(bal));  // prefix[lo] <= tl: bal has bit 0
  }
  __syncthreads();
  unsigned long long batch_base = s_u64[2] * kBatch;
  unsigned long long c_base = __ldg(a.tile_prefix + s_u64[2]);
  unsigned long long j_cur = jb_lo;
  float bmax = neg_inf_f();  // max log-weight of population t + 1 over this CTA's outputs
  const unsigned long long my_begin = MULTI ? s_rank_begin[a.rank] : 0ull;

  while (j_cur < jb_hi && batch_base < a.n_local) {
    // ---- stage the tile: thread tid owns sources [batch_base + 16 tid, +16)
    const unsigned long long i0 = batch_base + kSegment * tid;
    const int nv = i0 >= a.n_local ? 0 : i0 + kSegment <= a.n_local ? kSegment : static_cast<int>(a.n_local - i0);
    uint4 xx;
    if (nv == kSegment) {
      xx = __ldcs(reinterpret_cast<const uint4*>(a.x + i0));
    } else {
      uint8_t tmp[kSegment];
#pragma unroll
      for (int k = 0; k < kSegment; ++k) tmp[k] = k < nv ? a.x[i0 + k] : 0;
      xx = *reinterpret_cast<const uint4*>(tmp);
    }
    reinterpret_cast<uint4*>(xs)[tid] = xx;
    const uint32_t xw[4] = {xx.x, xx.y, xx.z, xx.w};
    double twd = 0.0;  // exact: 16 weights < 2^35
    if (nv == kSegment) {
#pragma unroll
      for (int k = 0; k < kSegment; ++k) twd += wdS[(xw[k >> 2] >> (8 * (k & 3))) & 0xFFu];
    } else {
#pragma unroll
      for (int k = 0; k < kSegment; ++k)
        twd += k < nv ? wdS[(xw[k >> 2] >> (8 * (k & 3))) & 0xFFu] : 0.0;
    }
    const unsigned long long tw = static_cast<unsigned long long>(twd);
    // block exclusive scan of the thread sums -> this thread's batch-relative prefix
    unsigned long long incl = tw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t2 = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t2;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    unsigned long long ex = incl - tw, btot = 0;
#pragma unroll
    for (int q = 0; q < kSmcThreads / 32; ++q) {
      if (q < warp) ex += wsum[q];
      btot += wsum[q];
    }
    const unsigned long long c0 = O + c_base + ex;  // global weight coordinate of my source 0
    const double est0 = __fma_rn(__ull2double_rn(c0), n_over_t, -cb.a_over_t);
    const unsigned int f0 = c0 == 0 ? 0u : comb_rank(est0, c0, cb);

    // ---- outputs [j_cur, j_next) in 16-aligned windows of 8192 positions (one per batch
    // unless the batch has > 8177 outputs)
    unsigned long long o0 = j_cur;
    while (true) {
      const unsigned long long wb = o0 & ~15ull;
      const unsigned long long we = wb + kWindow;
      {  // rank my 16 sources into the comb. A source with children in the window marks the
         // position of its first child there (position 0 when its children straddle the
         // window start): every window is self-contained, an output's ancestor is the last
         // mark at or before it
        const unsigned int wb32 = static_cast<unsigned int>(wb);  // N < 2^31: positions fit u32
        unsigned int fp = f0;
        double cd = 0.0;  // exact prefix of my sources (integer sums < 2^53)
        const uint16_t mark0 = static_cast<uint16_t>(kSegment * tid + 1);
        if (f0 >= wb32) {  // my first child is in the window: fp - wb32 is the position
#pragma unroll
          for (int k = 0; k < kSegment; ++k) {
            const uint32_t st = (xw[k >> 2] >> (8 * (k & 3))) & 0xFFu;
            cd += (nv == kSegment || k < nv) ? wdS[st] : 0.0;
            const unsigned int fn = comb_rank(__fma_rn(cd, n_over_t, est0), c0, cd, cb);
            if (fp < fn && fp - wb32 < static_cast<unsigned int>(kWindow))
              marks[fp - wb32] = static_cast<uint16_t>(mark0 + k);
            fp = fn;
          }
        } else {
#pragma unroll
          for (int k = 0; k < kSegment; ++k) {
            const uint32_t st = (xw[k >> 2] >> (8 * (k & 3))) & 0xFFu;
            cd += (nv == kSegment || k < nv) ? wdS[st] : 0.0;
            const unsigned int fn = comb_rank(__fma_rn(cd, n_over_t, est0), c0, cd, cb);
            if (fp < fn && fn > wb32 && fp < wb32 + static_cast<unsigned int>(kWindow))
              marks[(fp > wb32 ? fp : wb32) - wb32] = static_cast<uint16_t>(mark0 + k);
            fp = fn;
          }
        }
        if (tid == kSmcThreads - 1) s_jn = fp;  // F(end of batch): first output of the next batch
      }
      __syncthreads();
      const unsigned long long j_next = s_jn < jb_hi ? s_jn : jb_hi;
      if (o0 >= j_next) break;  // no outputs (no marks were written either)
      const unsigned long long o1 = we < j_next ? we : j_next;
      // chunk c of this thread covers positions wb + 16 (tid + 256 c) + [0, 16)
      // the second half of the window holds outputs only when the batch's outputs reach it
      const bool two = o1 > wb + kWindow / 2;
      unsigned int cm[2] = {0u, 0u};
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (c == 1 && !two) break;
        const uint4* mp = reinterpret_cast<const uint4*>(marks) + 2 * (tid + kSmcThreads * c);
        const uint4 a0 = mp[0], a1 = mp[1];
        const unsigned int m8 = __vmaxu2(__vmaxu2(__vmaxu2(a0.x, a0.y), __vmaxu2(a0.z, a0.w)),
                                         __vmaxu2(__vmaxu2(a1.x, a1.y), __vmaxu2(a1.z, a1.w)));
        cm[c] = max(m8 & 0xFFFFu, m8 >> 16);  // per-u16 max of the chunk's 16 marks
      }
      // inclusive max-scans over the threads (position order), both halves of the window
      unsigned int pm0 = cm[0], pm1 = cm[1];
      if (two) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned int t0 = __shfl_up_sync(0xffffffffu, pm0, o);
          const unsigned int t1 = __shfl_up_sync(0xffffffffu, pm1, o);
          if (lane >= o) {
            pm0 = max(pm0, t0);
            pm1 = max(pm1, t1);
          }
        }
      } else {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned int t0 = __shfl_up_sync(0xffffffffu, pm0, o);
          if (lane >= o) pm0 = max(pm0, t0);
        }
      }
      if (lane == 31) {
        wmax[warp] = pm0;
        wmax[kSmcThreads / 32 + warp] = pm1;
      }
      __syncthreads();
      unsigned int run0 = 0, run1 = 0, tot0 = 0;
      {
        const unsigned int e0 = __shfl_up_sync(0xffffffffu, pm0, 1);
        const unsigned int e1 = __shfl_up_sync(0xffffffffu, pm1, 1);
        if (lane > 0) {
          run0 = max(run0, e0);
          run1 = max(run1, e1);
        }
      }
#pragma unroll
      for (int q = 0; q < kSmcThreads / 32; ++q) {
        if (q < warp) {
          run0 = max(run0, wmax[q]);
          run1 = max(run1, wmax[kSmcThreads / 32 + q]);
        }
        tot0 = max(tot0, wmax[q]);
      }
      run1 = max(run1, tot0);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const unsigned long long jc = wb + kSegment * (tid + kSmcThreads * c);  // my first position
        if (jc + kSegment <= o0 || jc >= o1) {  // chunk without outputs of this batch
          uint4* mp = reinterpret_cast<uint4*>(marks) + 2 * (tid + kSmcThreads * c);
          mp[0] = make_uint4(0, 0, 0, 0);
          mp[1] = make_uint4(0, 0, 0, 0);
          continue;
        }
        unsigned int run = c ? run1 : run0;
        const bool full = jc >= o0 && jc + kSegment <= o1;
        uint32_t mw[8];
        {
          uint4* mp = reinterpret_cast<uint4*>(marks) + 2 * (tid + kSmcThreads * c);
          const uint4 a0 = mp[0], a1 = mp[1];
          mp[0] = make_uint4(0, 0, 0, 0);
          mp[1] = make_uint4(0, 0, 0, 0);
          mw[0] = a0.x; mw[1] = a0.y; mw[2] = a0.z; mw[3] = a0.w;
          mw[4] = a1.x; mw[5] = a1.y; mw[6] = a1.z; mw[7] = a1.w;
        }
        uint32_t outw[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const uint4 wd = draw_block(key, (jc >> 2) + g, a.t + 1, CUPPL_TAG_SMC_STEP);
          const uint32_t wv[4] = {wd.x, wd.y, wd.z, wd.w};
          uint32_t packed = 0;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int i = 4 * g + h;
            run = max(run, (mw[i >> 1] >> (16 * (i & 1))) & 0xFFFFu);
            const unsigned int anc = (run - 1u) & (kBatch - 1);  // run >= 1 at every output
            const unsigned int xa = xs[anc];
            uint32_t st;
            if (SMEM_ALIAS) {
              const unsigned long long pp = static_cast<unsigned long long>(wv[h]) * S;
              const unsigned long long e = alias_s[xa * S + static_cast<unsigned int>(pp >> 32)];
              const bool keep = static_cast<uint32_t>(pp) <= static_cast<uint32_t>(e);
              st = __byte_perm(static_cast<uint32_t>(e >> 32), 0u, keep ? 0x4410u : 0x4432u);
            } else {
              st = static_cast<uint32_t>(alias_draw(m.alias_trans + static_cast<size_t>(xa) * S, m.S, wv[h]));
            }
            packed = h == 0 ? st : __byte_perm(packed, st, h == 1 ? 0x3240u : h == 2 ? 0x3410u : 0x4210u);
            if (full) present[st] = 1;
            if (DEBUG) {
              const unsigned long long j = jc + i;
              if (j >= o0 && j < o1) {
                int r = 0;
                if (MULTI)
                  while (r + 1 < a.world && s_rank_begin[r + 1] <= j) ++r;
                const unsigned long long rb = MULTI ? s_rank_begin[r] : 0ull;
                a.anc_out[r][j - rb] = my_begin + batch_base + anc;
              }
            }
          }
          outw[g] = packed;
        }
        // store: one 16-byte write when the whole chunk is in [o0, o1) (rank boundaries are
        // multiples of 16: a chunk never straddles two owners); bytes at the window edges
        int r = 0;
        if (MULTI)
          while (r + 1 < a.world && s_rank_begin[r + 1] <= jc) ++r;
        const unsigned long long rb = MULTI ? s_rank_begin[r] : 0ull;
        if (full) {
          __stcs(reinterpret_cast<uint4*>(a.x_out[r] + (jc - rb)),
                 make_uint4(outw[0], outw[1], outw[2], outw[3]));
        } else {
#pragma unroll
          for (int i = 0; i < kSegment; ++i) {
            const unsigned long long j = jc + i;
            if (j >= o0 && j < o1) {
              const uint8_t st = static_cast<uint8_t>(outw[i >> 2] >> (8 * (i & 3)));
              a.x_out[r][j - rb] = st;
              bmax = fmaxf(bmax, lwS1[st]);
            }
          }
        }
      }
      o0 = we;
      if (o0 >= j_next) break;  // the end-of-batch barrier below orders the reuse
      __syncthreads();          // wmax / marks / s_jn reuse by the next window
    }
    j_cur = s_jn < jb_hi ? s_jn : jb_hi;
    c_base += btot;
    batch_base += kBatch;
    __syncthreads();  // xs / wsum / s_jn reuse
  }
  if (MULTI) __threadfence_system();  // peer stores performed before the next collective
  __syncthreads();  // present[] complete
  for (int s = tid; s < m.S; s += kSmcThreads)
    if (present[s]) bmax = fmaxf(bmax, lwS1[s]);
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
  const unsigned long long n_blocks = (n_tiles + kScanTiles - 1) / kScanTiles;
  if (a.hist)
    smc_scan_kernel<true><<<static_cast<unsigned>(n_blocks), kSmcThreads, 0, st>>>(m, a);
  else
    smc_scan_kernel<false><<<static_cast<unsigned>(n_blocks), kSmcThreads, 0, st>>>(m, a);
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

template <bool MULTI, bool DEBUG, bool SA>
static cudaError_t launch_resample_t(const SmcModel& m, const SmcResampleArgs& a, int sm_count,
                                     cudaStream_t st) {
  const size_t smem = SA ? static_cast<size_t>(m.S) * m.S * sizeof(unsigned long long) : 0;
  auto kern = smc_resample_kernel<MULTI, DEBUG, SA>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSmcThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  unsigned long long g = static_cast<unsigned long long>(sm_count) * per_sm;
  const unsigned long long want = (a.n_local + kBatch - 1) / kBatch;  // >= one batch per CTA
  if (g > want) g = want > 0 ? want : 1;
  kern<<<static_cast<unsigned>(g), kSmcThreads, smem, st>>>(m, a);
  return cudaGetLastError();
}

template <bool MULTI, bool DEBUG>
static cudaError_t launch_resample_s(const SmcModel& m, const SmcResampleArgs& a, int sm_count,
                                     cudaStream_t st) {
  return m.S <= kSmemAliasMaxStates ? launch_resample_t<MULTI, DEBUG, true>(m, a, sm_count, st)
                                    : launch_resample_t<MULTI, DEBUG, false>(m, a, sm_count, st);
}

cudaError_t launch_smc_resample(const SmcModel& m, const SmcResampleArgs& a, int sm_count,
                                cudaStream_t st) {
  if (a.anc_out)
    return a.world > 1 ? launch_resample_s<true, true>(m, a, sm_count, st)
                       : launch_resample_s<false, true>(m, a, sm_count, st);
  return a.world > 1 ? launch_resample_s<true, false>(m, a, sm_count, st)
                     : launch_resample_s<false, false>(m, a, sm_count, st);
}

}  // namespace cuppl
