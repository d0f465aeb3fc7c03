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
// the y values of its 8-point groups g = t + NT m (m < M) in REGISTERS, for every chain of the
// CTA. Per chain the labels are one byte per pair of points, code = a W + b (W = K + 1, label
// K = padding with mu = 0), four pair codes per u32 (one LDS.32 per group), and split tables TA[code] = -mu_a,
// TB[code] = -mu_b (two conflict-light LDS.32 per pair). Per pair: one FADD2 (y + t) and one FFMA2
// (acc += r r). Shared-memory traffic is ~4.5 B per point per re-execution (the code byte and
// the table entry; y is in registers). Per step:
//   A  lane c of warp 0 draws chain c's site / proposal / log u and applies the proposal;
//   B  every thread evaluates its points for all C chains; a 31-shuffle transpose reduction
//      leaves chain c's warp partial in lane c; warps' partials go to shared memory;
//   C  lane c folds the warp partials in fixed order, accepts or restores, records.
// Three barriers per step for all C chains.
//
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

// Shared-memory layout of one CTA: [C][G] u32 pair codes, [C][2][64] float split tables, [C][8] mu,
// [C][2K+2] double stats (written only by lane c), [n_warps][32] float warp partials.
struct MhLayout {
  size_t codes, tabs, mus, stats, parts, total;
};

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~static_cast<size_t>(15); }

__host__ __device__ inline MhLayout mh_layout(int G, int W, int C, int NT) {
  MhLayout L;
  size_t o = 0;
  L.codes = o;
  o = align16(o + static_cast<size_t>(C) * G * 4);
  L.tabs = o;
  o = align16(o + static_cast<size_t>(C) * 2 * kMhTab * 4);
  L.mus = o;
  o = align16(o + static_cast<size_t>(C) * 8 * 4);
  L.stats = o;
  o = align16(o + static_cast<size_t>(C) * (2 * kMhMaxK + 2) * 8);
  L.parts = o;
  o = align16(o + static_cast<size_t>(NT / 32) * 32 * 4);
  L.total = o;
  return L;
}

// Split pair tables of one chain: TA[code] = -mu_a, TB[code] = -mu_b (TB = TA + kMhTab): a
// warp's 32 random codes < W^2 <= 64 hit at most two entries per bank.
__device__ __forceinline__ void rebuild_table(float* tab, const float* mu, int W, int K) {
  for (int e = 0; e < W * W; ++e) {
    const int a = e / W, b = e - a * W;
    tab[e] = a < K ? -mu[a] : 0.f;
    tab[kMhTab + e] = b < K ? -mu[b] : 0.f;
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

// Sum over lanes of v[c] lands in lane c (c < 32): recursive halving, 31 shuffles.
__device__ __forceinline__ float transpose_reduce(float (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = upper ? v[i] : v[i + s];
      const float keep = upper ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

}  // namespace

size_t mh_smem_bytes(int G, int K, int chains_per_cta, int threads) {
  return mh_layout(G, K + 1, chains_per_cta, threads).total;
}

template <int M>
__global__ void __launch_bounds__(kMhMaxThreads, 1) mh_gmm_kernel(const MhArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = blockDim.x;
  const int K = a.K, W = K + 1, G = a.G, C = a.chains_per_cta;
  const MhLayout Ly = mh_layout(G, W, C, NT);
  uint32_t* codes = reinterpret_cast<uint32_t*>(smem + Ly.codes);
  float* tabs = reinterpret_cast<float*>(smem + Ly.tabs);
  float* mus = reinterpret_cast<float*>(smem + Ly.mus);
  double* stats = reinterpret_cast<double*>(smem + Ly.stats);
  float* parts = reinterpret_cast<float*>(smem + Ly.parts);
  const PhiloxKey key = make_key(a.key);
  const unsigned int local0 = blockIdx.x * C;  // first local chain of this CTA
  const int nc = min(C, static_cast<int>(a.n_chains) - static_cast<int>(local0));  // chains here
  const unsigned int n_sites = static_cast<unsigned int>(K + a.D);

  // ---- my data: groups g = tid + NT m, points 8g .. 8g + 7 as 4 (even, odd) pairs
  f32x2 Y[M][4];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int g = tid + NT * m;
    const float4 y0 = reinterpret_cast<const float4*>(a.y)[2 * g];
    const float4 y1 = reinterpret_cast<const float4*>(a.y)[2 * g + 1];
    Y[m][0] = pack2(y0.x, y0.y);
    Y[m][1] = pack2(y0.z, y0.w);
    Y[m][2] = pack2(y1.x, y1.y);
    Y[m][3] = pack2(y1.z, y1.w);
  }

  // ---- initial traces from the prior: labels (all threads), means (lane c of warp 0)
  for (int c = 0; c < nc; ++c) {
    const unsigned int chain = a.chain_begin + local0 + c;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int g = tid + NT * m;
      uint32_t l0[4], l1[4];
      labels4(a, key, chain, 8 * g, l0);
      labels4(a, key, chain, 8 * g + 4, l1);
      codes[c * G + g] = (l0[0] * W + l0[1]) | ((l0[2] * W + l0[3]) << 8) | ((l1[0] * W + l1[1]) << 16) |
                         ((l1[2] * W + l1[3]) << 24);
    }
  }
  float srt[kMhMaxK];
  unsigned int run = 0, rec = 0;
  float ll = 0.f;
  if (warp == 0 && lane < nc) {
    const unsigned int chain = a.chain_begin + local0 + lane;
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
    rebuild_table(tabs + lane * 2 * kMhTab, mu, W, K);
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

  // one re-execution of the log-likelihood of every chain: lane c of every warp ends with its
  // warp's partial of chain c in parts[warp][c]
  auto evaluate = [&]() {
    float v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      v[c] = 0.f;
      if (c < nc) {
        const uint32_t* cw = codes + c * G;
        const float* tab = tabs + c * 2 * kMhTab;
        f32x2 acc = pack2(0.f, 0.f);
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const uint32_t word = cw[tid + NT * m];
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const uint32_t code = (word >> (8 * b)) & 0xFFu;
            const f32x2 r = add2(Y[m][b], pack2(tab[code], tab[kMhTab + code]));
            acc = fma2(r, r, acc);
          }
        }
        const float2 s = unpack2(acc);
        v[c] = s.x + s.y;
      }
    }
    parts[warp * 32 + lane] = transpose_reduce(v, lane);
  };
  // lane c of warp 0: the log-likelihood of chain c from the warp partials (fixed order)
  auto fold = [&]() -> float {
    float p[kMhMaxThreads / 32];  // independent loads first, then a fixed-order sum
#pragma unroll
    for (int w = 0; w < kMhMaxThreads / 32; ++w) p[w] = w < NT / 32 ? parts[w * 32 + lane] : 0.f;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kMhMaxThreads / 32; ++w) s += p[w];
    return fmaf(a.neg_half_inv_var, s, a.ll_const);
  };

  evaluate();
  __syncthreads();
  if (warp == 0 && lane < nc) ll = fold();
  __syncthreads();

  const bool owner = warp == 0 && lane < nc;
  const unsigned int chain = a.chain_begin + local0 + lane;
  for (unsigned int s = 0; s < a.n_steps; ++s) {
    // ---- A: proposal of chain `lane`
    bool mu_site = false;
    float old_mu = 0.f, logu = 0.f;
    uint32_t site = 0, old_word = 0;
    int gidx = 0;
    if (owner) {
      float* mu = mus + 8 * lane;
      const uint4 b = mh_block(key, chain, s, 0u, CUPPL_TAG_MH);
      if (!lemire(b.x, n_sites, &site)) {
        for (unsigned int r = 1;; ++r)
          if (lemire(mh_block(key, chain, s, r, CUPPL_TAG_MH).x, n_sites, &site)) break;
      }
      logu = kLn2 * fast_lg2(u01_open0(b.w));
      mu_site = site < static_cast<uint32_t>(K);
      if (mu_site) {
        old_mu = mu[site];
        mu[site] = a.prior_sd * box_muller(b.y, b.z).x;
        rebuild_table(tabs + lane * 2 * kMhTab, mu, W, K);
      } else {
        uint32_t zprop;
        if (!lemire(b.y, static_cast<uint32_t>(K), &zprop)) {
          for (unsigned int r = 1;; ++r)
            if (lemire(mh_block(key, chain, s, r, CUPPL_TAG_MH).y, static_cast<uint32_t>(K), &zprop)) break;
        }
        const int i = static_cast<int>(site) - K;  // point index
        gidx = lane * G + (i >> 3);
        const int sh = 8 * ((i & 7) >> 1);
        old_word = codes[gidx];
        const uint32_t code = (old_word >> sh) & 0xFFu;
        const uint32_t ca = code / W, cb = code - ca * W;
        const uint32_t nc2 = (i & 1) ? ca * W + zprop : zprop * W + cb;
        codes[gidx] = (old_word & ~(0xFFu << sh)) | (nc2 << sh);
      }
    }
    __syncthreads();
    // ---- B: re-execute every chain
    evaluate();
    __syncthreads();
    // ---- C: accept / restore / record
    if (owner) {
      float* mu = mus + 8 * lane;
      double* st = stats + lane * (2 * kMhMaxK + 2);
      const float llp = fold();
      const bool accept = logu < llp - ll;
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
        rebuild_table(tabs + lane * 2 * kMhTab, mu, W, K);
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
    }
    __syncthreads();
  }
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
    a.ll_out[local] = ll;
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
  mh_gmm_kernel<M><<<grid, a.threads, smem, st>>>(a);
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
