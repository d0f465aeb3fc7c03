// mh_kernels.cu — K7: many independent lightweight Metropolis-Hastings chains on the Gaussian
// mixture model of SURVEY.md §8(d) C3, one warp per chain.
//
// Replaces run_lmh for this model: the trace database is
// the K means and D labels; each step picks one site uniformly ("chosen uniformly randomly"),
// redraws it from its prior, RE-EXECUTES the model (the full log-likelihood over all D points,
// as the reference's re-execution does) and accepts with the single-site prior-proposal
// ratio log a = l' - l (the prior terms of the resampled site cancel with the
// proposal; |DB| is constant for this model). The oracle restatement is or_mh_gmm in
// oracle/cuppl_oracle.c (same Philox words; fp64).
//
// Layout: y (fp32, zero padded to 256 points) is staged once per CTA in shared memory and shared
// by its chains; each chain keeps one byte per pair of points, code = a W + b (W = K + 1, label
// K = padding with mu = 0), and two 64-entry tables TA[code] = -mu_a, TB[code] = -mu_b. Lane l
// handles float4 l + 32 j (points 4f..4f+3, pair codes read as one u16), so the y loads, the
// code loads and the table lookups are all bank-conflict free; each pair of points costs two
// LDS.32 + one FADD2 + one FFMA2. The kernel is bound by shared-memory bandwidth (about 8.5 B
// per point per re-execution).
//
// Philox counters: (chain, step, sub, TAG_MH) per step (sub > 0 only for Lemire redraws);
// initial trace: labels from (chain, i >> 2, 0, TAG_MH_INIT) word i & 3, means from
// (chain, b, 1, TAG_MH_INIT) as two Box-Muller pairs per block.
#include "cuppl_device.cuh"
#include "mh_kernels.cuh"

namespace cuppl {

namespace {

struct ChainSmem {
  uint8_t* z;     // [D_pad / 2] pair codes a W + b
  float* ta;      // [64] -mu_a of each code
  float* tb;      // [64] -mu_b of each code
  float* mu;      // [8]
  double* stats;  // [2 * kMhMaxK + 2]
};

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~static_cast<size_t>(15); }

__host__ __device__ inline size_t chain_bytes(int D_pad) {
  return align16(D_pad / 2) + 2 * 64 * sizeof(float) + 8 * sizeof(float) +
         (2 * kMhMaxK + 2) * sizeof(double);
}

__device__ __forceinline__ uint4 mh_block(PhiloxKey k, unsigned int chain, unsigned int step,
                                          unsigned int sub, unsigned int tag) {
  return philox4x32_10(make_uint4(chain, step, sub, tag), k.k0, k.k1);
}

__device__ __forceinline__ void rebuild_table(const ChainSmem& c, int lane, int W) {
  for (int e = lane; e < 64; e += 32) {
    const int a = e / W, b = e - a * W;
    c.ta[e] = a < 8 ? -c.mu[a] : 0.f;
    c.tb[e] = -c.mu[b];
  }
}

// Full re-execution: sum_i -0.5 ((y_i - mu_{z_i}) / sigma)^2 + const, fixed reduction order.
__device__ __forceinline__ float ll_pass(const float4* y4, const unsigned short* z2, const float* ta,
                                         const float* tb, int nf4, float nhiv, float ll_const,
                                         int lane) {
  f32x2 acc0 = pack2(0.f, 0.f), acc1 = pack2(0.f, 0.f);
#pragma unroll 4
  for (int f = lane; f < nf4; f += 32) {
    const unsigned int zz = z2[f];  // codes of pairs 2f, 2f + 1
    const float4 y = y4[f];
    const unsigned int c0 = zz & 0xFFu, c1 = zz >> 8;
    const f32x2 r0 = add2(pack2(y.x, y.y), pack2(ta[c0], tb[c0]));
    const f32x2 r1 = add2(pack2(y.z, y.w), pack2(ta[c1], tb[c1]));
    acc0 = fma2(r0, r0, acc0);
    acc1 = fma2(r1, r1, acc1);
  }
  const float2 s0 = unpack2(acc0), s1 = unpack2(acc1);
  float s = (s0.x + s0.y) + (s1.x + s1.y);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return fmaf(nhiv, s, ll_const);
}

}  // namespace

size_t mh_smem_bytes(int D_pad, int chains_per_cta) {
  return align16(static_cast<size_t>(D_pad) * sizeof(float)) +
         static_cast<size_t>(chains_per_cta) * chain_bytes(D_pad);
}

__global__ void __launch_bounds__(kMhMaxChainsPerCta * 32, 1) mh_gmm_kernel(const MhArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* ys = reinterpret_cast<float*>(smem);
  for (int i = threadIdx.x; i < a.D_pad / 4; i += blockDim.x)
    reinterpret_cast<float4*>(ys)[i] = reinterpret_cast<const float4*>(a.y)[i];
  __syncthreads();
  const unsigned int local = blockIdx.x * a.chains_per_cta + warp;
  if (local >= a.n_chains) return;
  const unsigned int chain = a.chain_begin + local;
  uint8_t* base = smem + align16(static_cast<size_t>(a.D_pad) * sizeof(float)) + warp * chain_bytes(a.D_pad);
  ChainSmem c;
  c.z = base;
  c.ta = reinterpret_cast<float*>(base + align16(a.D_pad / 2));
  c.tb = c.ta + 64;
  c.mu = c.tb + 64;
  c.stats = reinterpret_cast<double*>(c.mu + 8);
  const PhiloxKey key = make_key(a.key);
  const int K = a.K, D = a.D;
  const unsigned int n_sites = static_cast<unsigned int>(K + D);
  const int W = K + 1;  // label K = padding

  // ---- initial trace from the prior
  for (int p = lane; p < a.D_pad / 2; p += 32) {
    uint32_t code = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = 2 * p + h;
      uint32_t lab = static_cast<uint32_t>(K);  // padding
      if (i < D) {
        const uint4 b = mh_block(key, chain, static_cast<unsigned int>(i) >> 2, 0u, CUPPL_TAG_MH_INIT);
        const uint32_t wv[4] = {b.x, b.y, b.z, b.w};
        if (!lemire(wv[i & 3], static_cast<uint32_t>(K), &lab)) {
          for (unsigned int r = 2;; ++r)
            if (lemire(mh_block(key, chain, static_cast<unsigned int>(i), r, CUPPL_TAG_MH_INIT).x,
                       static_cast<uint32_t>(K), &lab))
              break;
        }
      }
      code = code * W + lab;
    }
    c.z[p] = static_cast<uint8_t>(code);
  }
  if (lane < 8) {
    float v = 0.f;
    if (lane < K) {
      const uint4 b = mh_block(key, chain, static_cast<unsigned int>(lane) >> 2, 1u, CUPPL_TAG_MH_INIT);
      const float2 z01 = box_muller(b.x, b.y), z23 = box_muller(b.z, b.w);
      const float zz[4] = {z01.x, z01.y, z23.x, z23.y};
      v = a.prior_sd * zz[lane & 3];
    }
    c.mu[lane] = v;
  }
  if (lane < 2 * kMhMaxK + 2) c.stats[lane] = 0.0;
  __syncwarp();
  rebuild_table(c, lane, W);
  __syncwarp();
  const float4* y4 = reinterpret_cast<const float4*>(ys);
  const unsigned short* z2 = reinterpret_cast<const unsigned short*>(c.z);
  const int nf4 = a.D_pad / 4;
  float ll = ll_pass(y4, z2, c.ta, c.tb, nf4, a.neg_half_inv_var, a.ll_const, lane);
  unsigned int rec = 0;
  // run-length statistics: the sorted means change only when a mean proposal is accepted
  float srt[kMhMaxK];
  unsigned int run = 0;  // recorded steps since the sorted means last changed
  auto sort_means = [&]() {
    for (int k = 0; k < K; ++k) {  // insertion sort (label switching: compare sorted means)
      const float v = c.mu[k];
      int q = k;
      while (q > 0 && srt[q - 1] > v) {
        srt[q] = srt[q - 1];
        --q;
      }
      srt[q] = v;
    }
  };
  auto flush_run = [&]() {
    if (run) {
      for (int k = 0; k < K; ++k) {
        c.stats[k] += static_cast<double>(srt[k]) * run;
        c.stats[kMhMaxK + k] += static_cast<double>(srt[k]) * srt[k] * run;
      }
      c.stats[2 * kMhMaxK] += run;
      run = 0;
    }
  };
  if (lane == 0) sort_means();

  for (unsigned int s = 0; s < a.n_steps; ++s) {
    // lane 0 draws the site, the proposal and the acceptance uniform; broadcast
    uint32_t site = 0, zprop = 0;
    float muprop = 0.f, logu = 0.f;
    if (lane == 0) {
      const uint4 b = mh_block(key, chain, s, 0u, CUPPL_TAG_MH);
      if (!lemire(b.x, n_sites, &site)) {
        for (unsigned int r = 1;; ++r)
          if (lemire(mh_block(key, chain, s, r, CUPPL_TAG_MH).x, n_sites, &site)) break;
      }
      if (site < static_cast<uint32_t>(K)) {
        muprop = a.prior_sd * box_muller(b.y, b.z).x;
      } else if (!lemire(b.y, static_cast<uint32_t>(K), &zprop)) {
        for (unsigned int r = 1;; ++r)
          if (lemire(mh_block(key, chain, s, r, CUPPL_TAG_MH).y, static_cast<uint32_t>(K), &zprop)) break;
      }
      logu = kLn2 * fast_lg2(u01_open0(b.w));
    }
    site = __shfl_sync(0xffffffffu, site, 0);
    const bool mu_site = site < static_cast<uint32_t>(K);
    float old_mu = 0.f;
    uint8_t old_byte = 0;
    int p = 0;
    if (mu_site) {
      if (lane == 0) {
        old_mu = c.mu[site];
        c.mu[site] = muprop;
      }
      __syncwarp();
      rebuild_table(c, lane, W);
    } else {
      const int i = static_cast<int>(site) - K;
      p = i >> 1;
      if (lane == 0) {
        old_byte = c.z[p];
        const int ca = old_byte / W, cbb = old_byte - ca * W;
        c.z[p] = (i & 1) ? static_cast<uint8_t>(ca * W + static_cast<int>(zprop))
                         : static_cast<uint8_t>(static_cast<int>(zprop) * W + cbb);
      }
    }
    __syncwarp();
    const float llp = ll_pass(y4, z2, c.ta, c.tb, nf4, a.neg_half_inv_var, a.ll_const, lane);
    logu = __shfl_sync(0xffffffffu, logu, 0);
    const bool accept = logu < llp - ll;
    if (accept) {
      ll = llp;
    } else {
      if (lane == 0) {
        if (mu_site) c.mu[site] = old_mu;
        else c.z[p] = old_byte;
      }
      __syncwarp();
      if (mu_site) rebuild_table(c, lane, W);
    }
    __syncwarp();
    if (lane == 0) {
      if (accept) {
        c.stats[2 * kMhMaxK + 1] += 1.0;
        if (mu_site) {
          flush_run();
          sort_means();
        }
      }
      if (s >= a.burn_in && (s - a.burn_in) % a.thin == 0) {
        ++run;
        if (a.trace_out && rec < a.n_rec)
          for (int k = 0; k < K; ++k) a.trace_out[(static_cast<size_t>(local) * a.n_rec + rec) * K + k] = srt[k];
      }
    }
    if (s >= a.burn_in && (s - a.burn_in) % a.thin == 0) ++rec;
  }
  if (lane == 0) flush_run();
  __syncwarp();
  if (lane < K) a.mu_out[static_cast<size_t>(local) * K + lane] = c.mu[lane];
  if (lane == 0) a.ll_out[local] = ll;
  if (lane < 2 * K) {
    const int src = lane < K ? lane : kMhMaxK + (lane - K);
    a.stats_out[static_cast<size_t>(local) * (2 * K + 2) + lane] = c.stats[src];
  }
  if (lane < 2)
    a.stats_out[static_cast<size_t>(local) * (2 * K + 2) + 2 * K + lane] = c.stats[2 * kMhMaxK + lane];
}

cudaError_t launch_mh_gmm(const MhArgs& a, cudaStream_t st) {
  const size_t smem = mh_smem_bytes(a.D_pad, a.chains_per_cta);
  cudaError_t e = cudaFuncSetAttribute(mh_gmm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const unsigned int grid = (a.n_chains + a.chains_per_cta - 1) / a.chains_per_cta;
  mh_gmm_kernel<<<grid, a.chains_per_cta * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cuppl
