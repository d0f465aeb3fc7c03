// exp_repro vs exp_repro2 (packed) over a sweep of inputs: report mismatches
#include <cstdio>
#include "../../paper_2010_08454_b200/csrc/smc_common.cuh"
using namespace cuppl;
__global__ void k(unsigned int n, unsigned int* bad, float* ex) {
  for (unsigned int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float d0 = -87.0f * (i / (float)n);
    const float d1 = __uint_as_float(__float_as_uint(d0) ^ 1u);  // neighbour
    const float a = exp_repro(d0), b = exp_repro(d1);
    const float2 e = unpack2(exp_repro2(d0, d1));
    if (__float_as_uint(a) != __float_as_uint(e.x) || __float_as_uint(b) != __float_as_uint(e.y)) {
      const unsigned int j = atomicAdd(bad, 1u);
      if (j < 8) { ex[4 * j] = d0; ex[4 * j + 1] = a; ex[4 * j + 2] = e.x; ex[4 * j + 3] = d1; }
    }
  }
}
int main() {
  unsigned int* bad; float* ex;
  cudaMallocManaged(&bad, 4); cudaMallocManaged(&ex, 128);
  *bad = 0;
  k<<<1184, 256>>>(1u << 28, bad, ex);
  cudaDeviceSynchronize();
  printf("mismatches %u\n", *bad);
  for (unsigned j = 0; j < (*bad < 8 ? *bad : 8); ++j) printf("d=%.9g scalar=%.9g packed=%.9g (d1=%.9g)\n", ex[4*j], ex[4*j+1], ex[4*j+2], ex[4*j+3]);
  return 0;
}
