// calib_kernels.cu — pipe-rate microbenchmarks that calibrate the compute rooflines.
//
// The importance-sampling kernels are FP32 / issue bound; the B200 has no
// vendor FP32-pipe figure in MEASURED_PEAKS.json, so bench.py measures the ceilings here on
// the same box and reports the kernels' fraction of them:
//   kind 0: FFMA2 (packed fp32 FMA, register operands)  -> fp32 FLOP/s ceiling
//   kind 1: FFMA (scalar, register operands)
//   kind 2: Philox4x32-10 blocks/s
//   kind 3: MUFU (ex2 + lg2 pairs)
#include "cuppl_device.cuh"
#include "capi_internal.cuh"

namespace cuppl {

constexpr int kCalibThreads = 256;

__global__ void __launch_bounds__(kCalibThreads) calib_ffma2(int iters, float seed, float* sink) {
  f32x2 a[8], b = pack2(seed * 1e-7f, seed * 2e-7f), c = pack2(1.0f - 1e-7f, 1.0f + 1e-7f);
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = pack2(threadIdx.x + j, j - 1.0f);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fma2(a[j], c, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 v = unpack2(a[j]);
    s += v.x + v.y;
  }
  if (s == 1.2345f) sink[threadIdx.x] = s;
}

__global__ void __launch_bounds__(kCalibThreads) calib_ffma(int iters, float seed, float* sink) {
  float a[8];
  const float b = seed * 1e-7f, c = 1.0f - 1e-7f * seed;
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], c, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1.2345f) sink[threadIdx.x] = s;
}

__global__ void __launch_bounds__(kCalibThreads) calib_philox(int iters, uint64_t key, float* sink) {
  const PhiloxKey k = make_key(key);
  uint32_t acc = 0;
  const uint64_t id = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    const uint4 w = draw_block(k, id, static_cast<uint32_t>(i), 1u);
    acc ^= w.x ^ w.y ^ w.z ^ w.w;
  }
  if (acc == 0x12345678u) sink[threadIdx.x] = 1.f;
}

__global__ void __launch_bounds__(kCalibThreads) calib_mufu(int iters, float seed, float* sink) {
  float a[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) a[j] = 1.0f + (threadIdx.x + j) * 1e-6f * seed;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int j = 0; j < 4; ++j) a[j] = fast_ex2(fast_lg2(a[j]));
    }
  }
  float s = a[0] + a[1] + a[2] + a[3];
  if (s == 1.2345f) sink[threadIdx.x] = s;
}


// Linear-regression inner-loop patterns (4 particle pairs per thread, 2 points per iter).
// variant 0: FADD2 + 2 FFMA2 per point; 1: 3 FFMA2 (the add as fma(NB, 1, Y)); 2: scalar
// FADD + 2 FFMA on 8 particles; 3: FADD2 chain only; 4: FADD chain only.
template <int V>
__global__ void __launch_bounds__(kCalibThreads) calib_pattern(int iters, float seed, float* sink) {
  f32x2 NA[4], NB[4], S[4];
  float na[8], nb[8], s[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    NA[q] = pack2(-seed * (q + 1) * 1e-3f, seed * 1e-3f);
    NB[q] = pack2(seed * 1e-4f * q, -seed * 1e-4f);
    S[q] = pack2(0.f, 0.f);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    na[q] = -seed * (q + 1) * 1e-3f;
    nb[q] = seed * 1e-4f * q;
    s[q] = 0.f;
  }
  const f32x2 ONE = pack2(seed, seed);  // runtime 1.0: keeps the add on the FFMA2 path
  float x = threadIdx.x * 1e-3f, y = 0.5f + threadIdx.x * 1e-4f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x += 1e-7f;  // keeps the broadcast operands loop-variant (as data would be)
      y -= 1e-7f;
      const f32x2 X = pack2(x, x), Y = pack2(y, y);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (V == 0) {
          const f32x2 r = fma2(NA[q], X, add2(Y, NB[q]));
          S[q] = fma2(r, r, S[q]);
        } else if (V == 1) {
          const f32x2 r = fma2(NA[q], X, fma2(NB[q], ONE, Y));
          S[q] = fma2(r, r, S[q]);
        } else if (V == 3) {
          S[q] = add2(S[q], add2(X, NB[q]));
        }
      }
      if (V == 2) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float r = fmaf(na[q], x, y + nb[q]);
          s[q] = fmaf(r, r, s[q]);
        }
      } else if (V == 4) {
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] += x + nb[q];
      }
    }
  }
  float t = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 v = unpack2(S[q]);
    t += v.x + v.y;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) t += s[q];
  if (t == 1.2345f) sink[threadIdx.x] = t;
}

}  // namespace cuppl

using namespace cuppl;

extern "C" CUPPL_API int cuppl_calibrate(int kind, int blocks, int iters, float* sink, void* stream) {
  if (blocks < 1 || iters < 1 || !sink) return set_error(CUPPL_E_ARGUMENT, "calibrate: bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (kind) {
    case 0: calib_ffma2<<<blocks, kCalibThreads, 0, st>>>(iters, 1.0f, sink); break;
    case 1: calib_ffma<<<blocks, kCalibThreads, 0, st>>>(iters, 1.0f, sink); break;
    case 2: calib_philox<<<blocks, kCalibThreads, 0, st>>>(iters, 0x9E0160293A33AAF7ull, sink); break;
    case 3: calib_mufu<<<blocks, kCalibThreads, 0, st>>>(iters, 1.0f, sink); break;
    case 4: calib_pattern<0><<<blocks, kCalibThreads, 0, st>>>(iters, 1.0f, sink); break;
    case 5: calib_pattern<1><<<blocks, kCalibThreads, 0, st>>>(iters, 1.0f, sink); break;
    case 6: calib_pattern<2><<<blocks, kCalibThreads, 0, st>>>(iters, 1.0f, sink); break;
    case 7: calib_pattern<3><<<blocks, kCalibThreads, 0, st>>>(iters, 1.0f, sink); break;
    case 8: calib_pattern<4><<<blocks, kCalibThreads, 0, st>>>(iters, 1.0f, sink); break;
    default: return set_error(CUPPL_E_ARGUMENT, "calibrate: unknown kind %d", kind);
  }
  return cuda_status(cudaGetLastError(), "calibrate");
}
