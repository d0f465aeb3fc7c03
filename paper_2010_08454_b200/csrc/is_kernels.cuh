// is_kernels.cuh — launch parameters of the importance-sampling kernels (K1a/K1b + K2).
// Data vectors are passed BY VALUE in the kernel-parameter block (constant bank 0, up to
// 32 KB on sm_70+ with CUDA >= 12.1), so every thread reads x_i / y_i through the constant
// cache with a warp-uniform address and no shared-memory staging is needed.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/cuppl_gpu.h"

namespace cuppl {

constexpr int kIsThreads = 256;
constexpr int kLinregP = 8;  // particles per thread per chunk (4 FFMA2 pairs)
constexpr int kPolyP = 4;    // particles per thread per chunk (2 FFMA2 pairs)
constexpr int kPolyMinBlocks = 2;  // pair-packed accumulators need ~118 registers at P = 4
constexpr int kLinregCapSmall = 1024;
constexpr int kLinregCapLarge = 3968;
constexpr int kPolyCap = 64;

struct IsCommon {
  uint64_t pid_begin, pid_end;
  uint32_t k0, k1;
  uint32_t ks[20];  // Philox key schedule of (k0, k1) (philox_key_schedule)
  int n_points;
  int pad_;
  const float* injected;
  float* lw_out;
  float* coef_out;
  cuppl_is_record* block_recs;
  unsigned int* counter;
  cuppl_is_record* rec_out;
};

template <int CAP>
struct LinregParams : IsCommon {
  static constexpr int kCap = CAP;
  float neg_half_inv_var;  // -0.5 / sigma^2
  float lw_const;          // -D (ln sigma + 0.5 ln 2 pi)
  float one;               // 1.0f at run time (operand of the FFMA2 form of the add, V == 1)
  float pad1_;
  float2 xy[CAP > 0 ? CAP : 1];  // at kXyOffset (below)
  const float2* xy_g;  // CAP == 0: the (x_i, y_i) pairs in device memory (the workspace tail)
};

template <int CAP>
struct PolyParams : IsCommon {
  static constexpr int kCap = CAP;
  int32_t* deg_out;
  uint64_t pad2_;
  float2 xy[CAP > 0 ? CAP : 1];  // at kXyOffset (below)
  const float2* xy_g;  // CAP == 0: the (x_i, y_i) pairs in device memory (the workspace tail)
};

// Offset of the point array in both parameter blocks. Measured on B200 (xy offsets 168..256
// swept): the linreg loop runs 3% faster when the array starts 16 bytes past a 32-byte
// boundary of the constant bank (offsets 176 / 208 / 240: 89.1-89.5 ms per 1e9 particles; 184 /
// 192 / 224 / 256: 91.5-92.2 ms) and the poly kernel's LDCU.128 point loads want 16-byte
// alignment (176 / 192: 92.85 ms per 1.25e10 particles; 168 / 184 / 200: 93.5-93.7 ms). The
// kernel parameters start at a 32-byte-aligned bank address (c[0x0][0x380]).
constexpr size_t kXyOffset = 176;

// Point i of the data: the kernel-parameter block (constant bank) up to CAP points; larger
// data sets (CAP == 0) are read from device memory with warp-uniform __ldg (L1 broadcasts).
template <typename P>
__device__ __forceinline__ float2 xy_at(const P& prm, int i) {
  if constexpr (P::kCap > 0) {
    return prm.xy[i];
  } else {
    return __ldg(prm.xy_g + i);
  }
}
constexpr int kIsCapGlobal = 0;

template <int CAP>
cudaError_t launch_linreg(const LinregParams<CAP>& prm, bool injected, int sm_count,
                          int max_blocks, cudaStream_t stream, int variant);
// Inner-loop formulation of the linear-regression kernel: 0 = FADD2 + 2 FFMA2 per point and
// particle pair, 1 = 3 FFMA2, 2 = scalar with constant-bank operands. Default: kLinregVariant;
// the CUPPL_LINREG_VARIANT environment variable overrides it (tuning only).
constexpr int kLinregVariant = 0;
template <int CAP>
cudaError_t launch_poly(const PolyParams<CAP>& prm, bool injected, int sm_count, int max_blocks,
                        cudaStream_t stream, int variant);
// Poly benchmark-kernel tuning (CUPPL_POLY_VARIANT): 0 = P4/2 blocks, 1 = P4/3, 2 = P2/4, 3 = P2/3.
constexpr int kPolyVariant = 1;

}  // namespace cuppl
