// Shared helpers for the libblitz translation units: error reporting and
// small PTX utilities.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace bz {

// Driver API entry points are resolved at run time through
// cudaGetDriverEntryPoint, so libblitz.so links only the CUDA runtime and can
// be loaded (symbol checks) on a machine without a GPU driver.
#define BZ_DRIVER_FNS(X)                                                                       \
  X(cuGetErrorName) X(cuGetErrorString) X(cuDeviceGet) X(cuDeviceGetAttribute)                 \
  X(cuMemGetAllocationGranularity) X(cuMulticastGetGranularity) X(cuMemAddressReserve)         \
  X(cuMemAddressFree) X(cuMemMap) X(cuMemUnmap) X(cuMemSetAccess) X(cuMemCreate)               \
  X(cuMemRelease) X(cuMemExportToShareableHandle) X(cuMemImportFromShareableHandle)            \
  X(cuMulticastCreate) X(cuMulticastAddDevice) X(cuMulticastBindMem) X(cuMulticastUnbind)      \
  X(cuStreamWaitValue32) X(cuTensorMapEncodeTiled)

struct DriverApi {
#define BZ_DECL_FN(name) decltype(&::name) name = nullptr;
  BZ_DRIVER_FNS(BZ_DECL_FN)
#undef BZ_DECL_FN
};

// nullptr (and the error slot set) if the driver is unavailable
const DriverApi* driver_api();

// record a message in the thread-local last-error slot, return `code`
int bz_fail(int code, const char* msg);
int bz_fail_cuda(cudaError_t err, const char* what);
int bz_fail_cu(CUresult r, const char* what);
// cudaGetLastError() after a launch -> BZ_OK or BZ_ECUDA
int bz_check_launch(const char* what);

template <typename T>
__host__ __device__ __forceinline__ T tmin(T a, T b) {
  return a < b ? a : b;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

}  // namespace bz
