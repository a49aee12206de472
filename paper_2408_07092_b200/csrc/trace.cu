// trace.cu -- debug-only phase timestamps (compiled into libds_trace.so).
#ifdef DS_TRACE
#include <cuda_runtime_api.h>

#include "ds_common.cuh"

extern "C" int ds_debug_read_trace(void *host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, ds::g_trace, bytes);
}
extern "C" int ds_debug_clear_trace(void) {
  static unsigned long long zero[3][ds::kTraceCtas][ds::kTraceSlots];
  return (int)cudaMemcpyToSymbol(ds::g_trace, zero, sizeof(zero));
}
#endif
