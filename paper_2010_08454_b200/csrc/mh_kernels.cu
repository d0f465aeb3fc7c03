// mh_kernels.cu — K7: many independent lightweight Metropolis-Hastings chains on the Gaussian
// mixture model of SURVEY.md §8(d) C3.
//
// Replaces run_lmh for this model: the trace database is
// the K means and D labels; each step picks one site uniformly ("chosen uniformly randomly"),
// redraws it from its prior, RE-EXECUTES the model (the full log-likelihood over all D points,
// as the reference's re-execution does) and accepts with the single-site prior-proposal
// ratio log a = l' - l (the prior terms of the resampled site cancel with the
// proposal; |DB| is constant for this model). The oracle restatement is or_mh_gmm in
// oracle/cuppl_oracle.c (same Philox words; fp64).
//
// Decomposition: a CTA runs C <= 32 chains in lockstep. The data never move: thread t holds
// the y values of its 8-point groups g = t M + m (m < M) in REGISTERS, for every chain of the
// CTA. Per chain the labels are one byte per pair of points (even, odd), four pair bytes per
// u32 (one LDS.32 per group). A pair byte is the BYTE OFFSET 4e of the pair's entry e in the
// chain's split tables TA[e] = -mu_a, TB[e] = -mu_b, with e = a K + b for two data points,
// K^2 + a when the odd point is padding (D odd) and K^2 + K for two padding points (y = 0,
// residual 0). The tables sit at the start of shared memory, 512 B per chain, so a lookup is
// one PRMT (byte -> offset) and LDS [offset + chain immediate]; with K <= 5 a table has <= 31
// entries, one per bank: the warp's 32 random lookups never conflict. Per pair: PRMT, two
// LDS.32, FADD2 (y + t), FFMA2 (acc += r r). Shared memory moves 4 B per point per
// re-execution (the table entry; y is in registers), which bounds the kernel: one wavefront
// per 32 points. Per step:
//   A  lane c of warp 0 draws chain c's site / proposal / log u and applies the proposal;
//   B  every thread evaluates its points for all C chains; a 31-shuffle transpose reduction
//      leaves chain c's warp partial in lane c; warps' partials go to shared memory;
//   C  lane c folds the warp partials IN FP64 in fixed order, accepts or restores, records.
// Three barriers per step for all C chains. The chain's log-likelihood and the acceptance test
// are fp64 (the thread and warp partials are fp32 over <= 512 points).
// Philox counters: (chain, step, sub, TAG_MH) per step (sub > 0 only for Lemire redraws);
// initial trace: labels from (chain, i >> 2, 0, TAG_MH_INIT) word i & 3, means from
// (chain, b, 1, TAG_MH_INIT) as two Box-Muller pairs per block.
#include "cuppl_device.cuh"
#include "mh_kernels.cuh"

namespace cuppl {

namespace {

__device__ __forceinline__ uint4 mh_block(PhiloxKey k, unsigned int chain, unsigned int step,
                                          unsigned int sub, unsigned int tag) {
  return philox4x32_10(make_uint4(chain, step, sub, tag), k.k0, k.k1);
}

// Shared-memory layout of one CTA: [C][2][64] float split tables FIRST (byte offsets in the
// pair codes are relative to the start of shared memory), [C][G] u32 pair codes, [C][8] mu,
// [C][2K+2] double stats (written only by lane c), [n_warps][32] float warp partials.
struct MhLayout {
  size_t codes, tabs, mus, stats, parts, total;
};

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~static_cast<size_t>(15); }

constexpr int kMhTabBytes = 2 * kMhTab * 4;  // one chain's TA + TB

__host__ __device__ inline MhLayout mh_layout(int G, int C, int NT) {
  MhLayout L;
  size_t o = 0;
  L.tabs = o;
  o = align16(o + static_cast<size_t>(C) * kMhTabBytes);
  L.codes = o;
  o = align16(o + static_cast<size_t>(C) * G * 4);
  L.mus = o;
  o = align16(o + static_cast<size_t>(C) * 8 * 4);
  L.stats = o;
  o = align16(o + static_cast<size_t>(C) * (2 * kMhMaxK + 2) * 8);
  L.parts = o;
  o = align16(o + static_cast<size_t>(2 * (NT / 32)) * 16 * 4);
  L.total = o;
  return L;
}

// Pair entry e of labels (a, b); b == K marks a padding point (a == K: both padding).
__device__ __forceinline__ uint32_t pair_entry(uint32_t a, uint32_t b, uint32_t K) {
  return b < K ? a * K + b : (a < K ? K * K + a : K * K + K);
}
// Inverse: labels (a, b) of entry e (b == K for a padding odd point).
__device__ __forceinline__ void pair_labels(uint32_t e, uint32_t K, uint32_t* a, uint32_t* b) {
  if (e < K * K) {
    *a = e / K;
    *b = e - *a * K;
  } else {
    *a = e - K * K;
    *b = K;
  }
}

// Split pair tables of one chain: TA[e] = -mu_a, TB[e] = -mu_b (TB = TA + kMhTab).
__device__ __forceinline__ void rebuild_table(float* tab, const float* mu, int K) {
  const int T = K * K + K + 1;
  for (int e = 0; e < T; ++e) {
    uint32_t a, b;
    pair_labels(static_cast<uint32_t>(e), static_cast<uint32_t>(K), &a, &b);
    tab[e] = a < static_cast<uint32_t>(K) ? -mu[a] : 0.f;
    tab[kMhTab + e] = b < static_cast<uint32_t>(K) ? -mu[b] : 0.f;
  }
}

// Labels of points i0 .. i0 + 3 (i0 % 4 == 0): words of Philox(chain, i0 / 4, 0, TAG_MH_INIT),
// Lemire on K; a rejected word is redrawn from word 0 of blocks (chain, i, 2, ...), (.., 3, ..)
__device__ __forceinline__ void labels4(const MhArgs& a, PhiloxKey key, unsigned int chain, int i0,
                                        uint32_t lab[4]) {
  const uint4 b = mh_block(key, chain, static_cast<unsigned int>(i0) >> 2, 0u, CUPPL_TAG_MH_INIT);
  const uint32_t wv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const int i = i0 + h;
    lab[h] = static_cast<uint32_t>(a.K);  // padding
    if (i < a.D && !lemire(wv[h], static_cast<uint32_t>(a.K), &lab[h])) {
      for (unsigned int r = 2;; ++r)
        if (lemire(mh_block(key, chain, static_cast<unsigned int>(i), r, CUPPL_TAG_MH_INIT).x,
                   static_cast<uint32_t>(a.K), &lab[h]))
          break;
    }
  }
}

}  // namespace

// A chain's code words sit at a fixed stride of kMhMaxThreads * M words (>= G = NT * M): the
// chain offset of every code-word load is then a compile-time immediate.
size_t mh_smem_bytes(int G, int K, int chains_per_cta, int threads) {
  (void)K;
  const int M = (G + threads - 1) / threads;
  return mh_layout(kMhMaxThreads * M, chains_per_cta, threads).total;
}

// (21 warps: one SMSP holds 6, so <= 80 registers per thread.)
// Chain c's state lives with lane c of the CONTROL warp (the last warp of the CTA); the NT
// evaluation threads before it hold the data. The CTA's chains form two groups; per half-step
// the evaluation warps re-execute one group while the control warp folds, accepts and records
// the other group's previous re-execution and draws its next proposal — so the serial
// per-chain work overlaps the evaluation, with one barrier per half-step.
template <int M>
__global__ void __launch_bounds__(kMhMaxThreads + 32, 1) mh_gmm_kernel(const MhArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = a.threads;  // evaluation threads; thread NT .. NT + 31 is the control warp
  const bool control = tid >= NT;
  const int NW = NT / 32;
  const int K = a.K, G = a.G, C = a.chains_per_cta;
  constexpr int CS = kMhMaxThreads * M;  // code-word stride per chain (words)
  const MhLayout Ly = mh_layout(CS, C, NT);
  uint32_t* codes = reinterpret_cast<uint32_t*>(smem + Ly.codes);
  float* tabs = reinterpret_cast<float*>(smem + Ly.tabs);
  float* mus = reinterpret_cast<float*>(smem + Ly.mus);
  double* stats = reinterpret_cast<double*>(smem + Ly.stats);
  float* parts = reinterpret_cast<float*>(smem + Ly.parts);  // [2 groups][NW][16]
  const PhiloxKey key = make_key(a.key);
  const unsigned int local0 = blockIdx.x * C;  // first local chain of this CTA
  const int nc = min(C, static_cast<int>(a.n_chains) - static_cast<int>(local0));  // chains here
  const int c0 = (nc + 1) / 2;  // group 0: chains [0, c0); group 1: [c0, nc) (<= 16 each)
  const unsigned int n_sites = static_cast<unsigned int>(K + a.D);
  const uint32_t uK = static_cast<uint32_t>(K);

  // ---- my data (evaluation threads): groups g = tid M + m, points 8g .. 8g + 7 as 4 pairs
  f32x2 Y[M][4];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int g = control ? 0 : tid * M + m;  // a thread's groups are contiguous
    const float4 y0 = reinterpret_cast<const float4*>(a.y)[2 * g];
    const float4 y1 = reinterpret_cast<const float4*>(a.y)[2 * g + 1];
    Y[m][0] = pack2(y0.x, y0.y);
    Y[m][1] = pack2(y0.z, y0.w);
    Y[m][2] = pack2(y1.x, y1.y);
    Y[m][3] = pack2(y1.z, y1.w);
  }

  // ---- initial traces from the prior: labels (evaluation threads), means (control lane c)
  if (!control) {
    for (int c = 0; c < nc; ++c) {
      const unsigned int chain = a.chain_begin + local0 + c;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int g = tid * M + m;
        uint32_t l0[4], l1[4];
        labels4(a, key, chain, 8 * g, l0);
        labels4(a, key, chain, 8 * g + 4, l1);
        codes[c * CS + g] = (4u * pair_entry(l0[0], l0[1], uK)) | ((4u * pair_entry(l0[2], l0[3], uK)) << 8) |
                           ((4u * pair_entry(l1[0], l1[1], uK)) << 16) |
                           ((4u * pair_entry(l1[2], l1[3], uK)) << 24);
      }
    }
  }
  const bool owner = control && lane < nc;  // control lane c owns chain c
  const unsigned int chain = a.chain_begin + local0 + lane;
  const int grp = lane < c0 ? 0 : 1, lc = lane < c0 ? lane : lane - c0;  // my group, index in it
  float srt[kMhMaxK];
  unsigned int run = 0, rec = 0;
  double ll = 0.0;
  // the pending proposal of my chain (drawn one half-step ahead of its evaluation)
  bool mu_site = false;
  float old_mu = 0.f, logu = 0.f;
  uint32_t site = 0, old_word = 0;
  int gidx = 0;
  if (owner) {
    float* mu = mus + 8 * lane;
    for (int k = 0; k < 8; ++k) {
      float v = 0.f;
      if (k < K) {
        const uint4 b = mh_block(key, chain, static_cast<unsigned int>(k) >> 2, 1u, CUPPL_TAG_MH_INIT);
        const float2 z01 = box_muller(b.x, b.y), z23 = box_muller(b.z, b.w);
        const float zz[4] = {z01.x, z01.y, z23.x, z23.y};
        v = a.prior_sd * zz[k & 3];
      }
      mu[k] = v;
    }
    rebuild_table(tabs + lane * 2 * kMhTab, mu, K);
    double* st = stats + lane * (2 * kMhMaxK + 2);
    for (int k = 0; k < 2 * kMhMaxK + 2; ++k) st[k] = 0.0;
    for (int k = 0; k < K; ++k) {  // insertion sort (label switching: compare sorted means)
      const float v = mu[k];
      int q = k;
      while (q > 0 && srt[q - 1] > v) {
        srt[q] = srt[q - 1];
        --q;
      }
      srt[q] = v;
    }
  }
  __syncthreads();

  // re-execution of the log-likelihood of group q's chains (evaluation threads): lane l < 16
  // of warp w ends with the warp's partial of the group's chain l in parts[q][w][l]
  auto evaluate = [&](int q) {
    const int cb = q ? c0 : 0, ncq = q ? nc - c0 : c0;
    const uint32_t* cwq = codes + cb * CS + tid * M;  // this thread's M code words (contiguous)
    float v[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      v[c] = 0.f;
      if (c < ncq) {
        const uint32_t* cw = cwq + c * CS;
        const uint8_t* tab = smem + (cb + c) * kMhTabBytes;  // + byte offset: LDS [R + imm]
        f32x2 acc = pack2(0.f, 0.f);
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const uint32_t word = cw[m];
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const uint32_t off = __byte_perm(word, 0u, 0x4440u | static_cast<uint32_t>(b));
            const float ta = *reinterpret_cast<const float*>(tab + off);
            const float tb = *reinterpret_cast<const float*>(tab + kMhTab * 4 + off);
            const f32x2 r = add2(Y[m][b], pack2(ta, tb));
            acc = fma2(r, r, acc);
          }
        }
        const float2 s = unpack2(acc);
        v[c] = s.x + s.y;
      }
    }
    // lanes l and l + 16 fold, then a 15-shuffle transpose within 16 lanes: lane l < 16 holds
    // chain l's warp sum
#pragma unroll
    for (int c = 0; c < 16; ++c) v[c] += __shfl_xor_sync(0xffffffffu, v[c], 16);
#pragma unroll
    for (int s = 8; s >= 1; s >>= 1) {
      const bool upper = (lane & s) != 0;
#pragma unroll
      for (int i = 0; i < s; ++i) {
        const float send = upper ? v[i] : v[i + s];
        const float keep = upper ? v[i + s] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
      }
    }
    if (lane < 16) parts[(q * NW + warp) * 16 + lane] = v[0];
  };
  // control lane c: chain c's log-likelihood from its group's warp partials, in fp64, in a
  // fixed order
  auto fold = [&]() -> double {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += static_cast<double>(parts[(grp * NW + w) * 16 + lc]);
    return fma(a.neg_half_inv_var64, s, a.ll_const64);
  };
  // control lane c: draw step s's proposal and apply it to the chain's trace
  auto propose = [&](unsigned int s) {
    float* mu = mus + 8 * lane;
    const uint4 b = mh_block(key, chain, s, 0u, CUPPL_TAG_MH);
    if (!lemire(b.x, n_sites, &site)) {
      for (unsigned int r = 1;; ++r)
        if (lemire(mh_block(key, chain, s, r, CUPPL_TAG_MH).x, n_sites, &site)) break;
    }
    logu = kLn2 * fast_lg2(u01_open0(b.w));
    mu_site = site < uK;
    if (mu_site) {
      old_mu = mu[site];
      mu[site] = a.prior_sd * box_muller(b.y, b.z).x;
      rebuild_table(tabs + lane * 2 * kMhTab, mu, K);
    } else {
      uint32_t zprop;
      if (!lemire(b.y, uK, &zprop)) {
        for (unsigned int r = 1;; ++r)
          if (lemire(mh_block(key, chain, s, r, CUPPL_TAG_MH).y, uK, &zprop)) break;
      }
      const int i = static_cast<int>(site) - K;  // point index
      gidx = lane * CS + (i >> 3);
      const int sh = 8 * ((i & 7) >> 1);
      old_word = codes[gidx];
      uint32_t ca, cb;
      pair_labels(((old_word >> sh) & 0xFFu) >> 2, uK, &ca, &cb);
      const uint32_t e2 = (i & 1) ? pair_entry(ca, zprop, uK) : pair_entry(zprop, cb, uK);
      codes[gidx] = (old_word & ~(0xFFu << sh)) | ((4u * e2) << sh);
    }
  };
  // control lane c: accept / restore / record step s of chain c
  auto settle = [&](unsigned int s) {
    float* mu = mus + 8 * lane;
    double* st = stats + lane * (2 * kMhMaxK + 2);
    const double llp = fold();
    const bool accept = static_cast<double>(logu) < llp - ll;
    if (accept) {
      ll = llp;
      st[2 * kMhMaxK + 1] += 1.0;
      if (mu_site) {
        if (run) {  // the sorted means change: flush the run of identical records
          for (int k = 0; k < K; ++k) {
            st[k] += static_cast<double>(srt[k]) * run;
            st[kMhMaxK + k] += static_cast<double>(srt[k]) * srt[k] * run;
          }
          st[2 * kMhMaxK] += run;
          run = 0;
        }
        for (int k = 0; k < K; ++k) {
          const float v = mu[k];
          int q = k;
          while (q > 0 && srt[q - 1] > v) {
            srt[q] = srt[q - 1];
            --q;
          }
          srt[q] = v;
        }
      }
    } else if (mu_site) {
      mu[site] = old_mu;
      rebuild_table(tabs + lane * 2 * kMhTab, mu, K);
    } else {
      codes[gidx] = old_word;
    }
    if (s >= a.burn_in && (s - a.burn_in) % a.thin == 0) {
      ++run;
      if (a.trace_out && rec < a.n_rec)
        for (int k = 0; k < K; ++k)
          a.trace_out[(static_cast<size_t>(local0 + lane) * a.n_rec + rec) * K + k] = srt[k];
      ++rec;
    }
  };

  // ---- initial log-likelihoods (both groups), then the first proposals
  if (!control) {
    evaluate(0);
    evaluate(1);
  }
  __syncthreads();
  if (owner) {
    ll = fold();
    if (a.n_steps > 0) propose(0);
  }
  __syncthreads();

  // ---- half-step h: evaluate group h & 1 at step h >> 1 || settle + propose the other group
  const unsigned int H = 2u * a.n_steps;
  for (unsigned int h = 0; h < H; ++h) {
    const int q = static_cast<int>(h & 1u);
    if (!control) {
      evaluate(q);
    } else if (h > 0 && owner && grp != q) {
      const unsigned int s = (h - 1) >> 1;
      settle(s);
      if (s + 1 < a.n_steps) propose(s + 1);
    }
    __syncthreads();
  }
  if (H > 0 && owner && grp == 1) settle(a.n_steps - 1);  // the last half-step's group

  if (owner) {
    const unsigned int local = local0 + lane;
    const float* mu = mus + 8 * lane;
    double* st = stats + lane * (2 * kMhMaxK + 2);
    if (run) {
      for (int k = 0; k < K; ++k) {
        st[k] += static_cast<double>(srt[k]) * run;
        st[kMhMaxK + k] += static_cast<double>(srt[k]) * srt[k] * run;
      }
      st[2 * kMhMaxK] += run;
    }
    for (int k = 0; k < K; ++k) a.mu_out[static_cast<size_t>(local) * K + k] = mu[k];
    a.ll_out[local] = static_cast<float>(ll);
    double* out = a.stats_out + static_cast<size_t>(local) * (2 * K + 2);
    for (int k = 0; k < K; ++k) {
      out[k] = st[k];
      out[K + k] = st[kMhMaxK + k];
    }
    out[2 * K] = st[2 * kMhMaxK];
    out[2 * K + 1] = st[2 * kMhMaxK + 1];
  }
}

template <int M>
static cudaError_t launch_m(const MhArgs& a, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(mh_gmm_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const unsigned int grid = (a.n_chains + a.chains_per_cta - 1) / a.chains_per_cta;
  mh_gmm_kernel<M><<<grid, a.threads + 32, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_mh_gmm(const MhArgs& a, cudaStream_t st) {
  const size_t smem = mh_smem_bytes(a.G, a.K, a.chains_per_cta, a.threads);
  switch (a.groups_per_thread) {
    case 1: return launch_m<1>(a, smem, st);
    case 2: return launch_m<2>(a, smem, st);
    case 3: return launch_m<3>(a, smem, st);
    case 4: return launch_m<4>(a, smem, st);
    case 5: return launch_m<5>(a, smem, st);
    case 6: return launch_m<6>(a, smem, st);
    case 7: return launch_m<7>(a, smem, st);
    case 8: return launch_m<8>(a, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cuppl
