// resample_kernels.cu — the generic systematic-resampling primitive (cuppl_resample): any
// population of N particles given fp32 log-weights lw[N] and a fixed-size payload of P bytes
// per particle, resampled with the exact integer comb of SURVEY.md Appendix A D6 (the rule the
// HMM filter's K5/K6 apply to u8 states), restated bit for bit by oracle/resample_oracle.c:
//
//   M = max lw (NaN ignored); w_i = min(floor(exp_repro(lw_i - M) 2^31), 2^31) (smc_common.cuh);
//   C = inclusive u64 prefix of w, T = C[N-1]; u = word 0 of Philox(t, 0, 0, TAG_SMC_COMB);
//   target_j = floor((j 2^32 + u) T / (N 2^32)); a_j = min{i : C_i > target_j};
//   out[j] = payload[a_j], anc[j] = a_j; stats: M, T, sum e, sum e^2.
//
// Three kernels, all HBM-streaming (algorithmic traffic per particle: lw read three times,
// 12 B, plus the payload read once and written once, 2P, plus 8 B of optional ancestors):
//   RS1 rs_max_kernel     grid max of lw (float4 loads, last-CTA fold);
//   RS2 rs_scan_kernel    quantised weights, per-tile u64 sums and fp64 (sum e, sum e^2), a
//                         single-pass decoupled look-back (smc_common.cuh warp_lookback) giving
//                         each 2048-particle tile its exclusive weight prefix, and T;
//   RS3 rs_gather_kernel  output-balanced: CTA b owns an even share of the N outputs, finds the
//                         tile holding its first ancestor (warp 33-ary search over the tile
//                         prefixes), then streams source tiles staged in shared memory by TMA
//                         (cp.async.bulk of the tile's log-weights and payload, one mbarrier
//                         transaction), ranks every source into the comb (source k's children
//                         are [F(C_{k-1}), F(C_k)), smc_common.cuh comb_rank) and marks first
//                         children in a 4096-output window; a block max-scan resolves each
//                         output's ancestor, and the payload is copied with lane-consecutive
//                         (coalesced) stores. The work per output is uniform whatever the
//                         offspring counts.
#include "cuppl_device.cuh"
#include "smc_common.cuh"
#include "resample_kernels.cuh"

namespace cuppl {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned int bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned int phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}
// 1-D bulk copy global -> shared (TMA), completing `bytes` on the mbarrier
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned int bytes,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float block_max_f(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float r = red[0];
  for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) r = fmaxf(r, red[w]);
  __syncthreads();
  return r;
}

}  // namespace

// ------------------------------------------------------------------ RS1: max ------------
__global__ void __launch_bounds__(kRsThreads) rs_max_kernel(RsArgs a) {
  __shared__ float red[kRsThreads / 32];
  __shared__ bool last;
  float m = neg_inf_f();
  const unsigned long long n4 = a.n / 4;
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * kRsThreads;
  const float4* l4 = reinterpret_cast<const float4*>(a.lw);
  for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(kRsThreads) + threadIdx.x; i < n4;
       i += stride) {
    const float4 v = __ldg(l4 + i);
    m = fmaxf(m, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));  // fmaxf drops NaN like the oracle's >
  }
  for (unsigned long long i = 4 * n4 + blockIdx.x * static_cast<unsigned long long>(kRsThreads) + threadIdx.x;
       i < a.n; i += stride)
    m = fmaxf(m, a.lw[i]);
  m = block_max_f(m, red);
  if (threadIdx.x == 0) {
    a.blk_max[blockIdx.x] = m;
    __threadfence();
    last = atomicAdd(&a.counters[0], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  float r = neg_inf_f();
  for (unsigned int b = threadIdx.x; b < gridDim.x; b += kRsThreads) r = fmaxf(r, __ldcg(a.blk_max + b));
  r = block_max_f(r, red);
  if (threadIdx.x == 0) *a.M = r;
}

// ------------------------------------------------------------------ RS2: scan -----------
__global__ void __launch_bounds__(kRsThreads) rs_scan_kernel(RsArgs a) {
  __shared__ unsigned long long wtot[kRsScanTiles][kRsThreads / 32];
  __shared__ double wpart[kRsThreads / 32][2];
  __shared__ unsigned int s_blk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_blk = atomicAdd(&a.counters[1], 1u);  // launch-order ids: look-back is deadlock free
  __syncthreads();
  const float M = *a.M;
  const bool any = M > neg_inf_f();
  const unsigned long long n = a.n;
  const unsigned long long blk = s_blk;
  const unsigned long long tile0 = blk * kRsScanTiles;
  float v[kRsScanTiles][kRsSeg];
#pragma unroll
  for (int u = 0; u < kRsScanTiles; ++u) {
    const unsigned long long p0 = (tile0 + u) * kRsTile + static_cast<unsigned long long>(tid) * kRsSeg;
    if (p0 + kRsSeg <= n) {
      const float4 x0 = __ldcs(reinterpret_cast<const float4*>(a.lw + p0));
      const float4 x1 = __ldcs(reinterpret_cast<const float4*>(a.lw + p0) + 1);
      v[u][0] = x0.x; v[u][1] = x0.y; v[u][2] = x0.z; v[u][3] = x0.w;
      v[u][4] = x1.x; v[u][5] = x1.y; v[u][6] = x1.z; v[u][7] = x1.w;
    } else {
#pragma unroll
      for (int k = 0; k < kRsSeg; ++k) v[u][k] = p0 + k < n ? a.lw[p0 + k] : neg_inf_f();
    }
  }
  double d1 = 0.0, d2 = 0.0;  // fp32 over each thread's 8 particles, fp64 across (D10)
#pragma unroll
  for (int u = 0; u < kRsScanTiles; ++u) {
    unsigned long long ws = 0;
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < kRsSeg; k += 2) {
      const float2 ee = smc_e2(v[u][k], v[u][k + 1], M);
      const float e0 = any ? ee.x : 0.f, e1 = any ? ee.y : 0.f;
      ws += smc_w(e0);
      s1 += e0;
      s2 = fmaf(e0, e0, s2);
      ws += smc_w(e1);
      s1 += e1;
      s2 = fmaf(e1, e1, s2);
    }
    d1 += s1;
    d2 += s2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ws += __shfl_down_sync(0xffffffffu, ws, o);
    if (lane == 0) wtot[u][warp] = ws;
  }
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
  if (warp != 0) return;
  unsigned long long tagg = 0;
  if (lane < kRsScanTiles) {
#pragma unroll
    for (int w = 0; w < kRsThreads / 32; ++w) tagg += wtot[lane][w];
  }
  unsigned long long tincl = tagg;
#pragma unroll
  for (int o = 1; o < kRsScanTiles; o <<= 1) {
    const unsigned long long t2 = __shfl_up_sync(0xffffffffu, tincl, o);
    if (lane >= o) tincl += t2;
  }
  const unsigned long long agg = __shfl_sync(0xffffffffu, tincl, kRsScanTiles - 1);
  if (lane == 0) st_relaxed_u64(a.flags + blk, (blk == 0 ? kFlagIncl : kFlagAgg) | agg);
  const unsigned long long prefix = blk == 0 ? 0ull : warp_lookback(a.flags, blk);
  if (lane == 0 && blk != 0) st_relaxed_u64(a.flags + blk, kFlagIncl | (prefix + agg));
  if (lane < kRsScanTiles && tile0 + lane < a.n_tiles) a.tile_prefix[tile0 + lane] = prefix + tincl - tagg;
  if (lane == 0) {
    double t1 = 0.0, t2 = 0.0;
    for (int w = 0; w < kRsThreads / 32; ++w) {
      t1 += wpart[w][0];
      t2 += wpart[w][1];
    }
    a.tile_s[2 * blk] = t1;
    a.tile_s[2 * blk + 1] = t2;
    if (blk == a.n_scan_blocks - 1) *a.total = prefix + agg;
  }
}

// ------------------------------------------------------------------ RS3: gather ---------
template <bool STAGE_PAY>
__global__ void __launch_bounds__(kRsThreads, 3) rs_gather_kernel(RsArgs a) {
  extern __shared__ __align__(128) uint8_t pay_s2[];  // [2][kRsTile][P] staged payloads (STAGE_PAY)
  __shared__ __align__(128) float lws2[2][kRsTile];   // staged log-weights, double-buffered
  __shared__ __align__(16) uint16_t marks[kRsWin];  // tile index + 1 of a first child
  __shared__ __align__(16) uint16_t ancs[kRsWin];   // resolved ancestor (tile index + 1)
  __shared__ unsigned long long wsum[kRsThreads / 32];
  __shared__ unsigned int wmax[kRsThreads / 32];
  __shared__ unsigned long long s_u64[3];
  __shared__ unsigned int s_jn;
  __shared__ Comb s_cb;
  __shared__ __align__(8) unsigned long long mbar[2];
  __shared__ BlockScratch sc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long n = a.n;
  const unsigned long long P = a.P;
  const unsigned long long T = *a.total;
  const float M = *a.M;
  if (blockIdx.x == 0) {  // the step statistics: fixed-order fp64 fold of RS2's per-CTA sums
    double f1 = 0.0, f2 = 0.0;
    for (unsigned long long b = tid; b < a.n_scan_blocks; b += kRsThreads) {
      f1 += a.tile_s[2 * b];
      f2 += a.tile_s[2 * b + 1];
    }
    f1 = block_sum_d(f1, sc);
    f2 = block_sum_d(f2, sc);
    if (tid == 0) {
      a.stats_out->max_lw = M;
      a.stats_out->total = T;
      a.stats_out->sum_e = f1;
      a.stats_out->sum_e2 = f2;
    }
  }
  if (T == 0) return;  // every weight quantised to 0: nothing is written (the host raises)
  const bool any = M > neg_inf_f();
  if (tid == 0) {
    Comb c;
    c.u = draw_block(make_key(a.key), a.t, 0u, CUPPL_TAG_SMC_COMB).x;
    c.N = static_cast<unsigned int>(n);
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
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < kRsWin / 8; i += kRsThreads) reinterpret_cast<uint4*>(marks)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const Comb& cb = s_cb;
  const double n_over_t = cb.n_over_t;
  const unsigned long long jb_lo = n * blockIdx.x / gridDim.x;
  const unsigned long long jb_hi = n * (blockIdx.x + 1) / gridDim.x;
  if (jb_lo >= jb_hi) return;

  // the tile holding the ancestor of the first output (last tile with prefix <= target)
  if (warp == 0) {
    const unsigned long long tl = comb_target(static_cast<unsigned int>(jb_lo), cb);
    unsigned long long lo = 0, hi = a.n_tiles;
    while (hi - lo > 32) {
      const unsigned long long sp = hi - lo;
      const unsigned long long p = lo + sp * (lane + 1) / 33;
      const unsigned int bal = __ballot_sync(0xffffffffu, __ldg(a.tile_prefix + p) > tl);
      if (!bal) {
        lo = lo + sp * 32 / 33;
      } else {
        const int fl = __ffs(bal) - 1;
        hi = lo + sp * (fl + 1) / 33;
        if (fl > 0) lo = lo + sp * fl / 33;
      }
    }
    const unsigned long long p = lo + lane;
    const unsigned int bal = __ballot_sync(0xffffffffu, p < hi && __ldg(a.tile_prefix + p) <= tl);
    if (lane == 0) s_u64[0] = lo + (31 - __clz(bal));
  }
  __syncthreads();
  unsigned long long tile = s_u64[0];
  unsigned long long c_base = __ldg(a.tile_prefix + tile);
  unsigned long long j_cur = jb_lo;
  const bool tma_ok = a.tma;
  // double-buffered TMA staging: tile t + 1 is fetched while tile t is processed
  unsigned int ph[2] = {0u, 0u};
  bool pending[2] = {false, false};  // a bulk copy into buffer b is in flight (same in all threads)
  const unsigned int pay_bytes = STAGE_PAY ? static_cast<unsigned int>(kRsTile * P) : 0u;
  auto full_tile = [&](unsigned long long t) { return tma_ok && t < a.n_tiles && (t + 1) * kRsTile <= n; };
  auto issue = [&](int b, unsigned long long t) {  // thread 0
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of buffer b
    mbar_expect_tx(&mbar[b], kRsTile * 4u + pay_bytes);
    tma_load_1d(lws2[b], a.lw + t * kRsTile, kRsTile * 4u, &mbar[b]);
    if (STAGE_PAY) tma_load_1d(pay_s2 + static_cast<size_t>(b) * kRsTile * P, a.payload + t * kRsTile * P, pay_bytes,
                               &mbar[b]);
  };
  int bf = 0;
  if (full_tile(tile)) {
    if (tid == 0) issue(0, tile);
    pending[0] = true;
  }

  while (j_cur < jb_hi && tile < a.n_tiles) {
    const unsigned long long base = tile * kRsTile;
    const unsigned long long nv_tile = n - base < static_cast<unsigned long long>(kRsTile) ? n - base : kRsTile;
    float* lws = lws2[bf];
    uint8_t* pay_s = pay_s2 + static_cast<size_t>(bf) * kRsTile * P;
    // ---- the tile's log-weights (and payload) in shared memory
    if (pending[bf]) {
      mbar_wait(&mbar[bf], ph[bf]);
      ph[bf] ^= 1u;
      pending[bf] = false;
    } else {
      for (int i = tid; i < kRsTile; i += kRsThreads) lws[i] = i < static_cast<int>(nv_tile) ? a.lw[base + i] : neg_inf_f();
      if (STAGE_PAY)
        for (unsigned long long i = tid; i < nv_tile * P; i += kRsThreads) pay_s[i] = a.payload[base * P + i];
      __syncthreads();
    }
    if (full_tile(tile + 1)) {  // buffer 1 - bf was released by the previous tile's final barrier
      if (tid == 0) issue(1 - bf, tile + 1);
      pending[1 - bf] = true;
    }
    // ---- my sources [8 tid, +8): exact integer weights, block exclusive scan
    double wd[kRsSeg];
    unsigned long long tw = 0;
    {
      const float4 l0 = reinterpret_cast<const float4*>(lws)[2 * tid];  // two LDS.128
      const float4 l1 = reinterpret_cast<const float4*>(lws)[2 * tid + 1];
      const float lv[kRsSeg] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
#pragma unroll
      for (int k = 0; k < kRsSeg; k += 2) {
        const float2 ee = smc_e2(lv[k], lv[k + 1], M);
        const uint32_t w0 = any ? smc_w(ee.x) : 0u, w1 = any ? smc_w(ee.y) : 0u;
        tw += w0;
        tw += w1;
        wd[k] = static_cast<double>(w0);
        wd[k + 1] = static_cast<double>(w1);
      }
    }
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
    for (int q = 0; q < kRsThreads / 32; ++q) {
      if (q < warp) ex += wsum[q];
      btot += wsum[q];
    }
    const unsigned long long c0 = c_base + ex;
    const double est0 = __fma_rn(__ull2double_rn(c0), n_over_t, -cb.a_over_t);
    const unsigned int f0 = c0 == 0 ? 0u : comb_rank(est0, c0, cb);
    // F(C_k) of my 8 sources, once per tile: fp64 estimates, then the rare exact fix-ups in one
    // batch (no per-source branch)
    unsigned int fr[kRsSeg];
    {
      uint32_t need = 0;
      double cd = 0.0;
#pragma unroll
      for (int k = 0; k < kRsSeg; ++k) {
        cd += wd[k];
        bool ex;
        fr[k] = comb_rank_fast(__fma_rn(cd, n_over_t, est0), &ex);
        need |= static_cast<uint32_t>(ex) << k;
      }
      if (need) {
        double cd2 = 0.0;
#pragma unroll
        for (int k = 0; k < kRsSeg; ++k) {
          cd2 += wd[k];
          if ((need >> k) & 1u) fr[k] = comb_rank_exact2(__fma_rn(cd2, n_over_t, est0), c0, cd2, cb);
        }
      }
    }

    unsigned long long o0 = j_cur;
    while (true) {
      const unsigned long long wb = o0 & ~15ull;
      const unsigned long long we = wb + kRsWin;
      {
        const unsigned int wb32 = static_cast<unsigned int>(wb);
        unsigned int fp = f0;
#pragma unroll
        for (int k = 0; k < kRsSeg; ++k) {
          const unsigned int fn = fr[k];
          if (fp < fn && fn > wb32 && fp < wb32 + static_cast<unsigned int>(kRsWin))
            marks[(fp > wb32 ? fp : wb32) - wb32] = static_cast<uint16_t>(kRsSeg * tid + k + 1);
          fp = fn;
        }
        if (tid == kRsThreads - 1) s_jn = fp;
      }
      __syncthreads();
      const unsigned long long j_next = s_jn < jb_hi ? s_jn : jb_hi;
      if (o0 >= j_next) break;
      const unsigned long long o1 = we < j_next ? we : j_next;
      // chunk: positions wb + 16 tid + [0, 16)
      uint32_t mw[8];
      {
        uint4* mp = reinterpret_cast<uint4*>(marks) + 2 * tid;
        const uint4 a0 = mp[0], a1 = mp[1];
        mp[0] = make_uint4(0, 0, 0, 0);
        mp[1] = make_uint4(0, 0, 0, 0);
        mw[0] = a0.x; mw[1] = a0.y; mw[2] = a0.z; mw[3] = a0.w;
        mw[4] = a1.x; mw[5] = a1.y; mw[6] = a1.z; mw[7] = a1.w;
      }
      unsigned int cm = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) cm = __vmaxu2(cm, mw[i]);  // per-u16 max
      cm = max(cm & 0xFFFFu, cm >> 16);
      unsigned int pm = cm;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int t0 = __shfl_up_sync(0xffffffffu, pm, o);
        if (lane >= o) pm = max(pm, t0);
      }
      if (lane == 31) wmax[warp] = pm;
      __syncthreads();
      unsigned int run = 0;
      {
        const unsigned int e0 = __shfl_up_sync(0xffffffffu, pm, 1);
        if (lane > 0) run = e0;
      }
#pragma unroll
      for (int q = 0; q < kRsThreads / 32; ++q)
        if (q < warp) run = max(run, wmax[q]);
      uint32_t aw[8];
#pragma unroll
      for (int i = 0; i < kRsSeg * 2; ++i) {
        run = max(run, (mw[i >> 1] >> (16 * (i & 1))) & 0xFFFFu);
        if (i & 1)
          aw[i >> 1] |= run << 16;
        else
          aw[i >> 1] = run;
      }
      {
        uint4* ap = reinterpret_cast<uint4*>(ancs) + 2 * tid;
        ap[0] = make_uint4(aw[0], aw[1], aw[2], aw[3]);
        ap[1] = make_uint4(aw[4], aw[5], aw[6], aw[7]);
      }
      __syncthreads();
      // ---- outputs [max(o0, wb), o1): lane-consecutive stores
      const unsigned int q0 = static_cast<unsigned int>((o0 > wb ? o0 : wb) - wb);
      const unsigned int q1 = static_cast<unsigned int>(o1 - wb);
      if (a.anc_out)
        for (unsigned int q = q0 + tid; q < q1; q += kRsThreads) a.anc_out[wb + q] = base + ancs[q] - 1u;
      if (P) {
        if (a.word4) {
          const unsigned int PW = static_cast<unsigned int>(P >> 2);
          uint32_t* out = reinterpret_cast<uint32_t*>(a.payload_out) + wb * PW;
          const uint32_t* src = STAGE_PAY ? reinterpret_cast<const uint32_t*>(pay_s)
                                          : reinterpret_cast<const uint32_t*>(a.payload) + base * PW;
          if (PW == 1) {
            for (unsigned int q = q0 + tid; q < q1; q += kRsThreads) out[q] = src[ancs[q] - 1u];
          } else {
            const unsigned int nw = (q1 - q0) * PW;
            for (unsigned int w = tid; w < nw; w += kRsThreads) {
              const unsigned int q = q0 + w / PW, r = w - (w / PW) * PW;
              out[static_cast<unsigned long long>(q) * PW + r] = src[static_cast<unsigned long long>(ancs[q] - 1u) * PW + r];
            }
          }
        } else {
          const unsigned int PB = static_cast<unsigned int>(P);
          uint8_t* out = a.payload_out + wb * PB;
          const uint8_t* src = STAGE_PAY ? pay_s : a.payload + base * PB;
          const unsigned int nw = (q1 - q0) * PB;
          for (unsigned int w = tid; w < nw; w += kRsThreads) {
            const unsigned int q = q0 + w / PB, r = w - (w / PB) * PB;
            out[static_cast<unsigned long long>(q) * PB + r] = src[static_cast<unsigned long long>(ancs[q] - 1u) * PB + r];
          }
        }
      }
      o0 = we;
      if (o0 >= j_next) break;  // the end-of-tile barrier below orders the reuse
      __syncthreads();          // marks / ancs / wmax / s_jn reuse by the next window
    }
    j_cur = s_jn < jb_hi ? s_jn : jb_hi;
    c_base += btot;
    ++tile;
    bf ^= 1;
    __syncthreads();  // lws / pay_s / wsum / s_jn / ancs reuse
  }
  // a prefetch the CTA did not need must land before it exits
  if (pending[0]) mbar_wait(&mbar[0], ph[0]);
  if (pending[1]) mbar_wait(&mbar[1], ph[1]);
}

// ------------------------------------------------------------------ launch --------------
cudaError_t launch_resample(const RsArgs& a, int sm_count, cudaStream_t st) {
  rs_max_kernel<<<a.g1, kRsThreads, 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  rs_scan_kernel<<<static_cast<unsigned int>(a.n_scan_blocks), kRsThreads, 0, st>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const bool stage = a.P > 0 && a.P <= static_cast<unsigned long long>(kRsStageMaxP) && a.tma;
  const int smem = stage ? static_cast<int>(2 * kRsTile * a.P) : 0;
  int per_sm = 0;
  if (stage) {
    e = cudaFuncSetAttribute(rs_gather_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rs_gather_kernel<true>, kRsThreads, smem);
  } else {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rs_gather_kernel<false>, kRsThreads, 0);
  }
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  unsigned long long grid = static_cast<unsigned long long>(sm_count) * per_sm;
  const unsigned long long need = (a.n + kRsWin - 1) / kRsWin;
  if (grid > need) grid = need ? need : 1;
  if (stage)
    rs_gather_kernel<true><<<static_cast<unsigned int>(grid), kRsThreads, smem, st>>>(a);
  else
    rs_gather_kernel<false><<<static_cast<unsigned int>(grid), kRsThreads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cuppl
