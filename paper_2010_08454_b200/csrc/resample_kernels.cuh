// resample_kernels.cuh — launch parameters of the generic systematic-resampling primitive
// (resample_kernels.cu, C ABI cuppl_resample in include/cuppl_gpu.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/cuppl_gpu.h"

namespace cuppl {

constexpr int kRsThreads = 256;
constexpr int kRsSeg = 8;                       // sources per thread per tile
constexpr int kRsTile = kRsThreads * kRsSeg;    // 2048 particles: RS2 tile == RS3 staged source tile
constexpr int kRsScanTiles = 4;                 // RS2 tiles per CTA (one look-back per 8192 particles)
constexpr int kRsWin = 16 * kRsThreads;         // RS3 output window: 16 consecutive outputs per thread
constexpr int kRsStageMaxP = 16;                // payloads up to 16 B/particle are TMA-staged (2 x 32 KB)
constexpr int kRsMaxG1 = 1024;                  // RS1 CTAs

struct RsArgs {
  unsigned long long n;        // particles (< 2^31)
  const float* lw;             // [n] log-weights
  const uint8_t* payload;      // [n][P] (NULL when P == 0)
  unsigned long long P;        // payload bytes per particle
  uint8_t* payload_out;        // [n][P]
  unsigned long long* anc_out; // [n] ancestor index or NULL
  unsigned long long key;      // Philox key (the comb offset u of step t)
  unsigned int t;
  int tma;                     // lw (and payload) 16-byte aligned: TMA staging of full tiles
  int word4;                   // P % 4 == 0 and payload buffers 4-byte aligned: 4-byte copies
  unsigned int g1;             // RS1 grid
  // workspace (cuppl_resample_workspace_bytes)
  float* blk_max;                   // [g1]
  unsigned int* counters;           // [4] zeroed per call: RS1 arrivals, RS2 dynamic CTA id
  float* M;                         // max lw
  unsigned long long* total;        // T
  unsigned long long* flags;        // [n_scan_blocks] look-back words, zeroed per call
  unsigned long long* tile_prefix;  // [n_tiles] exclusive weight prefix of each tile
  double* tile_s;                   // [n_scan_blocks][2] sum e, sum e^2
  cuppl_resample_stats* stats_out;  // device
  unsigned long long n_tiles, n_scan_blocks;
};

cudaError_t launch_resample(const RsArgs& a, int sm_count, cudaStream_t st);

}  // namespace cuppl
