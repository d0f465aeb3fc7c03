// capi.cu — extern "C" entry points of libcuppl_gpu.so (declared in include/cuppl_gpu.h).
// Argument validation, workspace carving, grid sizing and error mapping; no allocations and
// no host synchronisation.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <mutex>
#include <string>

#include "cuppl_device.cuh"
#include "dist_kernels.cuh"
#include "is_kernels.cuh"
#include "capi_internal.cuh"

namespace cuppl {

static thread_local std::string g_last_error;

int set_error(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return status;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return CUPPL_OK;
  return set_error(CUPPL_E_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

// Device properties are cached per device ordinal (read-only after first query).
int device_sm_count(int* sm) {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  if (dev < 0 || dev >= 64) return set_error(CUPPL_E_ARGUMENT, "device ordinal %d", dev);
  std::lock_guard<std::mutex> lock(mu);
  if (!cache[dev]) {
    int v = 0;
    e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
    cache[dev] = v;
  }
  *sm = cache[dev];
  return CUPPL_OK;
}

}  // namespace cuppl

using namespace cuppl;

namespace {
constexpr int kMaxBlocksPerSm = 32;

int linreg_variant() {
  static const int v = [] {
    const char* e = std::getenv("CUPPL_LINREG_VARIANT");
    return e ? std::atoi(e) : kLinregVariant;
  }();
  return v;
}

int poly_variant() {
  static const int v = [] {
    const char* e = std::getenv("CUPPL_POLY_VARIANT");
    return e ? std::atoi(e) : kPolyVariant;
  }();
  return v;
}

size_t is_ws_bytes(int sm) {
  return 256 + static_cast<size_t>(sm) * kMaxBlocksPerSm * sizeof(cuppl_is_record);
}
// ... plus the device copy of data sets too large for the kernel-parameter block
constexpr int kMaxDataPoints = 1 << 24;
size_t is_ws_bytes_data(int sm, int n_points) {
  return ((is_ws_bytes(sm) + 255) & ~static_cast<size_t>(255)) + static_cast<size_t>(n_points) * sizeof(float2);
}

int check_dist(const cuppl_dist* d, DistArgs* a) {
  if (!d) return set_error(CUPPL_E_ARGUMENT, "dist is NULL");
  std::memset(a, 0, sizeof(*a));
  a->tag = d->tag;
  a->p0 = static_cast<float>(d->p0);
  a->p1 = static_cast<float>(d->p1);
  a->p2 = static_cast<float>(d->p2);
  switch (d->tag) {
    case CUPPL_DIST_NORMAL:
      if (!(d->p1 > 0.0) || !std::isfinite(d->p0) || !std::isfinite(d->p1))
        return set_error(CUPPL_E_INVALID_PARAM, "normal(%g, %g): sd must be > 0", d->p0, d->p1);
      break;
    case CUPPL_DIST_BERNOULLI:
      if (!(d->p0 >= 0.0 && d->p0 <= 1.0))
        return set_error(CUPPL_E_INVALID_PARAM, "bernoulli(%g): p must be in [0, 1]", d->p0);
      break;
    case CUPPL_DIST_POISSON:
      // rate < 2^31: the count is an int32 (and the halving tree stays <= 27 levels deep)
      if (!(d->p0 >= 0.0 && d->p0 < 2147483648.0))
        return set_error(CUPPL_E_INVALID_PARAM, "poisson(%g): rate must be >= 0 and < 2^31", d->p0);
      break;
    case CUPPL_DIST_UNIFORM_DISCRETE: {
      const double lo = d->p0, hi = d->p1;
      if (lo != std::floor(lo) || hi != std::floor(hi) || !(hi > lo) || lo < -2147483648.0 ||
          hi > 2147483647.0)
        return set_error(CUPPL_E_INVALID_PARAM,
                         "uniform-discrete(%g, %g): needs integers a < b (support [a, b))", lo, hi);
      a->ia = static_cast<int>(lo);
      a->ib = static_cast<int>(hi);
      break;
    }
    case CUPPL_DIST_UNIFORM_CONTINUOUS:
      if (!(d->p1 > d->p0) || !std::isfinite(d->p0) || !std::isfinite(d->p1))
        return set_error(CUPPL_E_INVALID_PARAM, "uniform-continuous(%g, %g): needs a < b", d->p0, d->p1);
      break;
    case CUPPL_DIST_BETA:
      if (!(d->p0 > 0.0 && d->p1 > 0.0) || !std::isfinite(d->p0) || !std::isfinite(d->p1))
        return set_error(CUPPL_E_INVALID_PARAM, "beta(%g, %g): shapes must be > 0", d->p0, d->p1);
      break;
    case CUPPL_DIST_EXPONENTIAL:
      if (!(d->p0 > 0.0) || !std::isfinite(d->p0))
        return set_error(CUPPL_E_INVALID_PARAM, "exponential(%g): rate must be > 0", d->p0);
      break;
    case CUPPL_DIST_CATEGORICAL:
      if (d->n_table < 1 || (d->n_table > 1 && !d->table))
        return set_error(CUPPL_E_INVALID_PARAM, "categorical: needs K >= 1 and a threshold table");
      a->K = d->n_table;
      a->table = d->table;
      break;
    default:
      return set_error(CUPPL_E_UNSUPPORTED, "unsupported distribution tag %d", d->tag);
  }
  return CUPPL_OK;
}

template <typename P>
int fill_common(P& prm, const float* xs, const float* ys, int n_points, int cap,
                uint64_t pid_begin, uint64_t pid_end, uint64_t key, const float* injected,
                float* lw_out, float* coef_out, cuppl_is_record* rec_out, void* ws,
                size_t ws_bytes, int sm, cudaStream_t stream) {
  if (!xs || !ys) return set_error(CUPPL_E_ARGUMENT, "xs/ys are NULL");
  if (n_points < 1 || (cap > 0 && n_points > cap))
    return set_error(CUPPL_E_CAPACITY, "n_points=%d outside [1, %d]", n_points, cap);
  if (n_points > kMaxDataPoints)
    return set_error(CUPPL_E_CAPACITY, "n_points=%d > %d", n_points, kMaxDataPoints);
  if (pid_end < pid_begin) return set_error(CUPPL_E_ARGUMENT, "pid_end < pid_begin");
  if (!rec_out) return set_error(CUPPL_E_ARGUMENT, "rec_out is NULL");
  const size_t need = cap > 0 ? is_ws_bytes(sm) : is_ws_bytes_data(sm, n_points);
  if (!ws || ws_bytes < need)
    return set_error(CUPPL_E_CAPACITY, "workspace %zu < %zu bytes", ws_bytes, need);
  prm.pid_begin = pid_begin;
  prm.pid_end = pid_end;
  prm.k0 = static_cast<uint32_t>(key);
  prm.k1 = static_cast<uint32_t>(key >> 32);
  philox_key_schedule(key, prm.ks);
  prm.n_points = n_points;
  prm.pad_ = 0;
  prm.injected = injected;
  prm.lw_out = lw_out;
  prm.coef_out = coef_out;
  prm.counter = static_cast<unsigned int*>(ws);
  prm.block_recs = reinterpret_cast<cuppl_is_record*>(static_cast<char*>(ws) + 256);
  prm.rec_out = rec_out;
  prm.xy_g = nullptr;
  if (cap > 0) {
    for (int i = 0; i < n_points; ++i) prm.xy[i] = make_float2(xs[i], ys[i]);
    for (int i = n_points; i < cap; ++i) prm.xy[i] = make_float2(0.f, 0.f);
    return CUPPL_OK;
  }
  // large data: interleaved (x, y) pairs in the workspace tail (pageable H2D copy: the host
  // staging vector may be released as soon as cudaMemcpyAsync returns)
  prm.xy[0] = make_float2(0.f, 0.f);
  std::vector<float2> host(static_cast<size_t>(n_points));
  for (int i = 0; i < n_points; ++i) host[i] = make_float2(xs[i], ys[i]);
  float2* dev = reinterpret_cast<float2*>(static_cast<char*>(ws) + is_ws_bytes(sm));
  cudaError_t e = cudaMemcpyAsync(dev, host.data(), host.size() * sizeof(float2), cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return cuda_status(e, "cudaMemcpyAsync");
  prm.xy_g = dev;
  return CUPPL_OK;
}
}  // namespace

extern "C" {

int cuppl_abi_version(void) { return CUPPL_ABI_VERSION; }

const char* cuppl_last_error(void) { return g_last_error.c_str(); }

int cuppl_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  if (sm_count) {
    int s = device_sm_count(sm_count);
    if (s) return s;
  }
  if (cc_major) {
    e = cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
  }
  if (cc_minor) {
    e = cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
  }
  return CUPPL_OK;
}

int cuppl_philox_blocks(uint64_t key, uint64_t first_id, uint32_t block, uint32_t tag,
                        uint64_t count, uint32_t* out, void* stream) {
  if (count && !out) return set_error(CUPPL_E_ARGUMENT, "out is NULL");
  int sm = 0;
  if (int s = device_sm_count(&sm)) return s;
  return cuda_status(launch_philox_blocks(key, first_id, block, tag, count, out, sm,
                                          static_cast<cudaStream_t>(stream)),
                     "philox_blocks");
}

int cuppl_dist_sample(const cuppl_dist* d, uint64_t key, uint32_t tag, uint64_t first_id,
                      uint64_t count, void* out, void* stream) {
  DistArgs a;
  if (int s = check_dist(d, &a)) return s;
  if (count && !out) return set_error(CUPPL_E_ARGUMENT, "out is NULL");
  int sm = 0;
  if (int s = device_sm_count(&sm)) return s;
  return cuda_status(
      launch_dist_sample(a, key, tag, first_id, count, out, sm, static_cast<cudaStream_t>(stream)),
      "dist_sample");
}

int cuppl_dist_score(const cuppl_dist* d, const void* x, uint64_t count, float* score,
                     void* stream) {
  DistArgs a;
  if (int s = check_dist(d, &a)) return s;
  if (count && (!x || !score)) return set_error(CUPPL_E_ARGUMENT, "x/score is NULL");
  int sm = 0;
  if (int s = device_sm_count(&sm)) return s;
  return cuda_status(launch_dist_score(a, x, count, score, sm, static_cast<cudaStream_t>(stream)),
                     "dist_score");
}

size_t cuppl_is_workspace_bytes(void) {
  int sm = 0;
  if (device_sm_count(&sm)) sm = 256;  // no device: an upper bound
  return is_ws_bytes(sm);
}

size_t cuppl_is_workspace_bytes_n(int n_points) {
  int sm = 0;
  if (device_sm_count(&sm)) sm = 256;
  return n_points > kPolyCap ? is_ws_bytes_data(sm, n_points) : is_ws_bytes(sm);
}

int cuppl_is_linreg(const float* xs, const float* ys, int n_points, float sigma,
                    uint64_t pid_begin, uint64_t pid_end, uint64_t key, const float* injected,
                    float* lw_out, float* coef_out, cuppl_is_record* rec_out, void* workspace,
                    size_t workspace_bytes, void* stream) {
  if (!(sigma > 0.f) || !std::isfinite(sigma))
    return set_error(CUPPL_E_INVALID_PARAM, "normal(mu, %g): sd must be > 0", (double)sigma);
  int sm = 0;
  if (int s = device_sm_count(&sm)) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(workspace, 0, 256, st);
  if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync");
  const float nhiv = static_cast<float>(-0.5 / (static_cast<double>(sigma) * sigma));
  const float lwc = static_cast<float>(-n_points * (std::log(static_cast<double>(sigma)) +
                                                    0.91893853320467274178));
  if (n_points <= kLinregCapSmall) {
    LinregParams<kLinregCapSmall> prm;
    if (int s = fill_common(prm, xs, ys, n_points, kLinregCapSmall, pid_begin, pid_end, key,
                            injected, lw_out, coef_out, rec_out, workspace, workspace_bytes, sm, st))
      return s;
    prm.neg_half_inv_var = nhiv;
    prm.lw_const = lwc;
    prm.one = 1.0f;
    prm.pad1_ = 0.f;
    return cuda_status(
        launch_linreg(prm, injected != nullptr, sm, sm * kMaxBlocksPerSm, st, linreg_variant()),
        "is_linreg");
  }
  if (n_points > kLinregCapLarge) {  // data in device memory (workspace tail)
    LinregParams<kIsCapGlobal> prm;
    if (int s = fill_common(prm, xs, ys, n_points, kIsCapGlobal, pid_begin, pid_end, key, injected, lw_out,
                            coef_out, rec_out, workspace, workspace_bytes, sm, st))
      return s;
    prm.neg_half_inv_var = nhiv;
    prm.lw_const = lwc;
    prm.one = 1.0f;
    prm.pad1_ = 0.f;
    return cuda_status(
        launch_linreg(prm, injected != nullptr, sm, sm * kMaxBlocksPerSm, st, linreg_variant()),
        "is_linreg");
  }
  LinregParams<kLinregCapLarge> prm;
  if (int s = fill_common(prm, xs, ys, n_points, kLinregCapLarge, pid_begin, pid_end, key,
                          injected, lw_out, coef_out, rec_out, workspace, workspace_bytes, sm, st))
    return s;
  prm.neg_half_inv_var = nhiv;
  prm.lw_const = lwc;
  prm.one = 1.0f;
  prm.pad1_ = 0.f;
  return cuda_status(
      launch_linreg(prm, injected != nullptr, sm, sm * kMaxBlocksPerSm, st, linreg_variant()),
      "is_linreg");
}

int cuppl_is_poly(const float* xs, const float* ys, int n_points, uint64_t pid_begin,
                  uint64_t pid_end, uint64_t key, const float* injected, float* lw_out,
                  int32_t* deg_out, float* coef_out, cuppl_is_record* rec_out, void* workspace,
                  size_t workspace_bytes, void* stream) {
  int sm = 0;
  if (int s = device_sm_count(&sm)) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(workspace, 0, 256, st);
  if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync");
  if (n_points > kPolyCap) {  // data in device memory (workspace tail)
    PolyParams<kIsCapGlobal> prm;
    if (int s = fill_common(prm, xs, ys, n_points, kIsCapGlobal, pid_begin, pid_end, key, injected, lw_out,
                            coef_out, rec_out, workspace, workspace_bytes, sm, st))
      return s;
    prm.deg_out = deg_out;
    return cuda_status(launch_poly(prm, injected != nullptr, sm, sm * kMaxBlocksPerSm, st, poly_variant()),
                       "is_poly");
  }
  PolyParams<kPolyCap> prm;
  if (int s = fill_common(prm, xs, ys, n_points, kPolyCap, pid_begin, pid_end, key, injected,
                          lw_out, coef_out, rec_out, workspace, workspace_bytes, sm, st))
    return s;
  prm.deg_out = deg_out;
  return cuda_status(launch_poly(prm, injected != nullptr, sm, sm * kMaxBlocksPerSm, st, poly_variant()),
                     "is_poly");
}

int cuppl_is_record_merge(const cuppl_is_record* recs, int n, cuppl_is_record* out) {
  if (!out || (n > 0 && !recs)) return set_error(CUPPL_E_ARGUMENT, "NULL record pointer");
  cuppl_is_record acc;
  std::memset(&acc, 0, sizeof(acc));
  acc.max_lw = -INFINITY;
  acc.argmax_lw = -INFINITY;
  acc.argmax_pid = ~0ull;
  for (int i = 0; i < n; ++i) rec_merge(acc, recs[i]);
  *out = acc;
  return CUPPL_OK;
}

}  // extern "C"
