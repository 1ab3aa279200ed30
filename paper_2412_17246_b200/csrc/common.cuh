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
  X(cuStreamWaitValue32) X(cuTensorMapEncodeTiled) X(cuFuncGetModule) X(cuModuleGetFunctionCount)    \
  X(cuModuleEnumerateFunctions) X(cuFuncLoad)

struct DriverApi {
#define BZ_DECL_FN(name) decltype(&::name) name = nullptr;
  BZ_DRIVER_FNS(BZ_DECL_FN)
#undef BZ_DECL_FN
};

// nullptr (and the error slot set) if the driver is unavailable
const DriverApi* driver_api();

// one kernel of each translation unit (= one CUDA module), for bz_preload_kernels
const void* module_anchor_dataplane();
const void* module_anchor_decode();
const void* module_anchor_gemm();
const void* module_anchor_llama();
const void* module_anchor_attention();

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

// ---- programmatic dependent launch (PDL) ------------------------------------------------
// The compute kernels (GEMM, Llama glue, decode attention) are launched with
// programmatic stream serialization, so kernel N+1 is scheduled while kernel N
// is still running.  Each kernel lets its dependents launch at entry and calls
// pdl_wait() before it touches anything a predecessor wrote (griddepcontrol.wait
// returns once the preceding grid has completed and its writes are visible;
// without the launch attribute both instructions are no-ops).  What overlaps is
// launch latency and set-up (barrier init, TMEM allocation, descriptor
// prefetch) and, in the GEMM, the first weight tiles (see BZ_GEMM_B_STATIC).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// kernel classes for the BZ_PDL mask (unset: all; 0: none -- plain stream
// serialization for A/B checks)
enum PdlKind { PDL_GEMM = 1, PDL_GLUE = 2, PDL_ATTN = 4 };
bool pdl_enabled(int kind);

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(int kind, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled(kind) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace bz
