// capi_smc.cu — extern "C" entry points of the SMC engine (include/cuppl_gpu.h).
#include <cmath>
#include <cstring>

#include "capi_internal.cuh"
#include "cuppl_device.cuh"
#include "smc_kernels.cuh"

using namespace cuppl;

namespace {
struct SmcWs {
  unsigned long long* tile_prefix;
  unsigned long long* flags;
  unsigned int* counters;
  double* tile_s;
  size_t zero_bytes;  // flags + counters (prefix of the zeroed region)
};

size_t align256(size_t v) { return (v + 255) & ~static_cast<size_t>(255); }

size_t ws_layout(uint64_t n, SmcWs* w, void* base) {
  const uint64_t n_tiles = (n + kTile - 1) / kTile;
  char* p = static_cast<char*>(base);
  size_t off = 0;
  const size_t flags_off = off;
  off = align256(off + n_tiles * 8);
  const size_t counters_off = off;
  off = align256(off + 16);
  const size_t zero_end = off;
  const size_t tiles_off = off;
  off = align256(off + n_tiles * 16);
  const size_t prefix_off = off;
  off = align256(off + n_tiles * 8);
  if (w) {
    w->flags = reinterpret_cast<unsigned long long*>(p + flags_off);
    w->counters = reinterpret_cast<unsigned int*>(p + counters_off);
    w->tile_s = reinterpret_cast<double*>(p + tiles_off);
    w->tile_prefix = reinterpret_cast<unsigned long long*>(p + prefix_off);
    w->zero_bytes = zero_end;
  }
  return off;
}

int fill_model(const cuppl_smc_model* m, SmcModel* out) {
  if (!m) return set_error(CUPPL_E_ARGUMENT, "model is NULL");
  if (m->n_states < 1 || m->n_states > kMaxStates)
    return set_error(CUPPL_E_CAPACITY, "n_states=%d outside [1, %d]", m->n_states, kMaxStates);
  if (!(m->inv_sd > 0.f) || !std::isfinite(m->inv_sd))
    return set_error(CUPPL_E_INVALID_PARAM, "normal(mu, sd): sd must be > 0");
  if (!m->mu || !m->alias_trans || !m->alias_init)
    return set_error(CUPPL_E_ARGUMENT, "model tables are NULL");
  std::memset(out, 0, sizeof(*out));
  out->S = m->n_states;
  out->inv_sd = m->inv_sd;
  out->c = m->c;
  out->alias_trans = reinterpret_cast<const unsigned long long*>(m->alias_trans);
  out->alias_init = reinterpret_cast<const unsigned long long*>(m->alias_init);
  for (int s = 0; s < m->n_states; ++s) out->mu[s] = m->mu[s];
  return CUPPL_OK;
}

int check_ws(uint64_t n, void* ws, size_t bytes, SmcWs* w) {
  if (n == 0) return set_error(CUPPL_E_ARGUMENT, "n_local must be >= 1");
  if (n >= (1ull << 31)) return set_error(CUPPL_E_CAPACITY, "n_local must be < 2^31");
  const size_t need = ws_layout(n, w, ws);
  if (!ws || bytes < need) return set_error(CUPPL_E_CAPACITY, "workspace %zu < %zu bytes", bytes, need);
  return CUPPL_OK;
}
}  // namespace

extern "C" {

size_t cuppl_smc_workspace_bytes(uint64_t n_local) { return ws_layout(n_local, nullptr, nullptr); }

int cuppl_smc_init(const cuppl_smc_model* m, uint64_t n_local, uint64_t j_begin, uint64_t key,
                   float y0, uint8_t* x, int32_t* m_key, void* workspace, size_t workspace_bytes,
                   void* stream) {
  SmcModel sm;
  if (int s = fill_model(m, &sm)) return s;
  SmcWs w;
  if (int s = check_ws(n_local, workspace, workspace_bytes, &w)) return s;
  if (!x || !m_key) return set_error(CUPPL_E_ARGUMENT, "NULL buffer");
  if (j_begin % 16) return set_error(CUPPL_E_ARGUMENT, "j_begin must be a multiple of 16");
  int sms = 0;
  if (int s = device_sm_count(&sms)) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(workspace, 0, w.zero_bytes, st);
  if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync");
  SmcInitArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n_local = n_local;
  a.j_begin = j_begin;
  a.key = key;
  a.key_dev = reinterpret_cast<const unsigned long long*>(m->key_dev);
  a.y0 = y0;
  a.x = x;
  a.m_key = m_key;
  return cuda_status(launch_smc_init(sm, a, sms, st), "smc_init");
}

int cuppl_smc_scan(const cuppl_smc_model* m, uint64_t n_local, float y, const uint8_t* x,
                   const int32_t* m_key, uint64_t* hist, uint64_t* rank_rec, void* workspace,
                   size_t workspace_bytes, void* stream) {
  SmcModel sm;
  if (int s = fill_model(m, &sm)) return s;
  SmcWs w;
  if (int s = check_ws(n_local, workspace, workspace_bytes, &w)) return s;
  if (!x || !m_key || !rank_rec) return set_error(CUPPL_E_ARGUMENT, "NULL buffer");
  int sms = 0;
  if (int s = device_sm_count(&sms)) return s;
  SmcScanArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n_local = n_local;
  a.x = x;
  a.y = y;
  a.S = sm.S;
  a.m_key = m_key;
  a.tile_prefix = w.tile_prefix;
  a.flags = w.flags;
  a.counters = w.counters;
  a.tile_s = w.tile_s;
  a.hist = reinterpret_cast<unsigned long long*>(hist);
  a.rank_rec = reinterpret_cast<unsigned long long*>(rank_rec);
  return cuda_status(launch_smc_scan(sm, a, sms, static_cast<cudaStream_t>(stream)), "smc_scan");
}

int cuppl_smc_resample(const cuppl_smc_model* m, uint64_t n_local, uint64_t n_total, uint64_t key,
                       uint32_t t, int rank, int world, float y_cur, float y_next, const uint8_t* x,
                       const int32_t* m_key, const uint64_t* rank_recs, const uint64_t* rank_begin,
                       uint8_t* const* x_out, uint64_t* const* anc_out, int32_t* m_key_next,
                       double* stats_out, void* workspace, size_t workspace_bytes, void* stream) {
  SmcModel sm;
  if (int s = fill_model(m, &sm)) return s;
  SmcWs w;
  if (int s = check_ws(n_local, workspace, workspace_bytes, &w)) return s;
  if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
    return set_error(CUPPL_E_ARGUMENT, "rank %d / world %d", rank, world);
  // the comb arithmetic needs N < 2^31 (j*R0 + Ra ~ N^2 in signed 64 bits, T <= N*2^31 in the
  // 62-bit look-back flag words), as SmcRunner and check_ws already enforce
  if (n_total < n_local || n_total >= (1ull << 31)) return set_error(CUPPL_E_CAPACITY, "n_total >= 2^31");
  if (!x || !m_key || !rank_recs || !rank_begin || !x_out || !m_key_next || !stats_out)
    return set_error(CUPPL_E_ARGUMENT, "NULL buffer");
  int sms = 0;
  if (int s = device_sm_count(&sms)) return s;
  SmcResampleArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n_local = n_local;
  a.n_total = n_total;
  a.key = key;
  a.key_dev = reinterpret_cast<const unsigned long long*>(m->key_dev);
  a.t = t;
  a.rank = rank;
  a.world = world;
  a.y_cur = y_cur;
  a.y_next = y_next;
  a.x = x;
  a.m_key = m_key;
  a.tile_prefix = w.tile_prefix;
  a.tile_s = w.tile_s;
  a.stats_out = reinterpret_cast<double*>(stats_out);
  a.counters = w.counters;
  a.rank_recs = reinterpret_cast<const unsigned long long*>(rank_recs);
  a.rank_begin = reinterpret_cast<const unsigned long long*>(rank_begin);
  a.x_out = x_out;
  a.anc_out = reinterpret_cast<unsigned long long* const*>(anc_out);
  a.m_key_next = m_key_next;
  a.flags_to_clear = w.flags;
  a.n_tiles = (n_local + kTile - 1) / kTile;
  a.n_scan_blocks = (a.n_tiles + kScanTiles - 1) / kScanTiles;
  return cuda_status(launch_smc_resample(sm, a, sms, static_cast<cudaStream_t>(stream)),
                     "smc_resample");
}

int cuppl_smc_log_weights(const cuppl_smc_model* m, float y, const uint8_t* x, uint64_t n,
                          float* lw, void* stream) {
  SmcModel sm;
  if (int s = fill_model(m, &sm)) return s;
  if (n && (!x || !lw)) return set_error(CUPPL_E_ARGUMENT, "NULL buffer");
  int sms = 0;
  if (int s = device_sm_count(&sms)) return s;
  return cuda_status(launch_smc_log_weights(sm, y, x, n, lw, sms, static_cast<cudaStream_t>(stream)),
                     "smc_log_weights");
}

int cuppl_smc_fold(uint64_t n_local, double* stats_out, void* workspace, size_t workspace_bytes,
                   void* stream) {
  SmcWs w;
  if (int s = check_ws(n_local, workspace, workspace_bytes, &w)) return s;
  if (!stats_out) return set_error(CUPPL_E_ARGUMENT, "NULL buffer");
  const uint64_t n_tiles = (n_local + kTile - 1) / kTile;
  return cuda_status(launch_smc_fold(w.tile_s, (n_tiles + kScanTiles - 1) / kScanTiles, stats_out, w.counters,
                                     static_cast<cudaStream_t>(stream)),
                     "smc_fold");
}

}  // extern "C"
