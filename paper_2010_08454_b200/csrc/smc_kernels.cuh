// smc_kernels.cuh — launch parameters of the SMC kernels (K4 init, K5 scan, K6 resample).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/cuppl_gpu.h"

namespace cuppl {

constexpr int kSmcThreads = 256;
constexpr int kSegment = 16;                  // particles per thread in K5 / K6 (one uint4 of states)
constexpr int kTile = kSmcThreads * kSegment;  // 4096 particles per K5 tile == K6 source batch
constexpr int kBatch = kTile;
constexpr int kScanTiles = 8;                 // K5 tiles per CTA (one table build + look-back per 32K particles)
constexpr int kWindow = 2 * kSmcThreads * kSegment;  // K6 output window: two 16-output chunks per thread
constexpr int kSmemAliasMaxStates = 64;       // K6 stages the S x S alias tables in shared memory
constexpr int kMaxStates = 256;               // particle state stored as u8
constexpr int kMaxRanks = 64;

// Bootstrap-filter model (HMM), passed by value.
struct SmcModel {
  int S;         // number of states (<= 256)
  float inv_sd;  // 1 / sd of the Gaussian emission
  float c;       // -ln sd - 0.5 ln 2 pi
  int pad_;
  const unsigned long long* alias_trans;  // [S][S] alias tables of the rows of A (thr | alias << 40)
  const unsigned long long* alias_init;   // [S] alias table of pi0
  float mu[kMaxStates];               // emission means
};

// A population is only its states (u8): in a discrete-state HMM the log-weight of a particle
// is a function of its state, lw = log N(y_t; mu[x], sd), so every kernel rebuilds the S-entry
// per-step tables (emission, quantised weight) in shared memory instead of storing lw.
struct SmcInitArgs {
  unsigned long long n_local;  // particles on this rank
  unsigned long long j_begin;  // global index of local particle 0 (multiple of 8)
  unsigned long long key;
  const unsigned long long* key_dev;  // when non-NULL: the key, read at run time (graph replay)
  float y0;
  int pad_;
  uint8_t* x;
  int* m_key;  // ordered-int key of max lw_0 (atomicMax target)
};

struct SmcScanArgs {
  unsigned long long n_local;
  const uint8_t* x;
  float y;                       // observation of population t
  int S;
  const int* m_key;              // max of lw_t as an ordered int (global over ranks)
  unsigned long long* tile_prefix;  // [n_tiles] exclusive prefix of the tile sums (look-back)
  unsigned long long* flags;     // [n_tiles] look-back words (status << 62 | value), zero on entry
  unsigned int* counters;        // [2]: dynamic tile id (zero on entry; K6 resets it)
  double* tile_s;                // [n_scan_blocks][2] per-CTA sum e, sum e^2 (fixed 8-tile blocks)
  unsigned long long* hist;      // [S] integer filtering weights of x_t (NULL: skip), zero on entry
  unsigned long long* rank_rec;  // [4]: T_r written by the last tile (other words untouched)
};

struct SmcResampleArgs {
  unsigned long long n_local;
  unsigned long long n_total;
  unsigned long long key;
  const unsigned long long* key_dev;  // when non-NULL: the key, read at run time (graph replay)
  unsigned int t;  // population being resampled; the new one is t + 1
  int rank, world;
  float y_cur;     // observation of population t (source weights)
  float y_next;    // observation of population t + 1 (max of the new log-weights)
  int pad_;
  const uint8_t* x;
  const int* m_key;                        // max of lw_t (ordered int)
  const unsigned long long* tile_prefix;   // exclusive prefix of the tile sums
  const double* tile_s;                    // [n_scan_blocks][2] per-K5-CTA sum e, sum e^2 (folded by CTA 0)
  double* stats_out;                       // [2]: rank sum e, sum e^2 of population t
  unsigned int* counters;                  // K5 counters, reset here
  const unsigned long long* rank_recs;     // [world][4] gathered rank records of step t
  const unsigned long long* rank_begin;    // [world + 1] global index of each rank's first particle
  uint8_t* const* x_out;                   // [world] destination x (peer-mapped for q != rank)
  unsigned long long* const* anc_out;      // [world] debug ancestor (global index) or NULL
  int* m_key_next;                         // atomicMax of lw_{t+1} over the outputs written here
  unsigned long long* flags_to_clear;      // K5 look-back words, zeroed for the next scan
  unsigned long long n_tiles;
  unsigned long long n_scan_blocks;        // K5 CTAs = ceil(n_tiles / kScanTiles)
};

cudaError_t launch_smc_init(const SmcModel& m, const SmcInitArgs& a, int sm_count, cudaStream_t st);
cudaError_t launch_smc_scan(const SmcModel& m, const SmcScanArgs& a, int sm_count, cudaStream_t st);
cudaError_t launch_smc_log_weights(const SmcModel& m, float y, const uint8_t* x, unsigned long long n,
                                   float* lw, int sm_count, cudaStream_t st);
cudaError_t launch_smc_fold(const double* tile_s, unsigned long long n_tiles, double* stats_out,
                            unsigned int* counters, cudaStream_t st);
cudaError_t launch_smc_resample(const SmcModel& m, const SmcResampleArgs& a, int sm_count,
                                cudaStream_t st);

}  // namespace cuppl
