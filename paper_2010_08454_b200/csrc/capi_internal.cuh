// capi_internal.cuh — helpers shared by the C-ABI translation units.
#pragma once
#include <cstdarg>
#include <cuda_runtime.h>

namespace cuppl {
int set_error(int status, const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);
int device_sm_count(int* sm);
}  // namespace cuppl
