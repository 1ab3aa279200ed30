// Host runtime of libblitz: error slot, devices, VMM weight slabs shared across
// processes (POSIX fd + pidfd_getfd), NVLS multicast objects.
//
// This is the B200 replacement for the paper's pre-established P2P connection
// pool: one process per GPU exports its slab once; peers
// import and map it, so a scale-up never creates a communicator.  Fan-out
// groups bind their members' slabs into one multicast object so a single
// multimem.st stream is replicated by the NVSwitch.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/blitz.h"
#include "common.cuh"

#ifndef SYS_pidfd_open
#define SYS_pidfd_open 434
#endif
#ifndef SYS_pidfd_getfd
#define SYS_pidfd_getfd 438
#endif

namespace bz {

static thread_local std::string g_last_error;

static DriverApi g_drv;
static bool g_drv_ok = false;

const DriverApi* driver_api() {
  if (g_drv_ok) return &g_drv;
  cudaDriverEntryPointQueryResult q;
#define BZ_RESOLVE(name)                                                                       \
  if (cudaGetDriverEntryPoint(#name, reinterpret_cast<void**>(&g_drv.name), cudaEnableDefault, &q) != \
          cudaSuccess ||                                                                       \
      q != cudaDriverEntryPointSuccess || g_drv.name == nullptr) {                             \
    g_last_error = "driver entry point unavailable: " #name;                                  \
    return nullptr;                                                                            \
  }
  BZ_DRIVER_FNS(BZ_RESOLVE)
#undef BZ_RESOLVE
  g_drv_ok = true;
  return &g_drv;
}

#define DRV() (&g_drv)

int bz_fail(int code, const char* msg) {
  g_last_error = msg;
  return code;
}
int bz_fail_cuda(cudaError_t err, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(err) + " (" + cudaGetErrorString(err) + ")";
  return BZ_ECUDA;
}
int bz_fail_cu(CUresult r, const char* what) {
  const char* name = nullptr;
  const char* str = nullptr;
  if (driver_api()) {
    g_drv.cuGetErrorName(r, &name);
    g_drv.cuGetErrorString(r, &str);
  }
  g_last_error = std::string(what) + ": " + (name ? name : "?") + " (" + (str ? str : "?") + ")";
  return r == CUDA_ERROR_NOT_SUPPORTED ? BZ_EUNSUP : BZ_ECUDA;
}
bool pdl_enabled(int kind) {
  static const int mask = [] {
    const char* e = getenv("BZ_PDL");
    return e ? atoi(e) : (PDL_GEMM | PDL_GLUE | PDL_ATTN);
  }();
  return (mask & kind) != 0;
}

int bz_check_launch(const char* what) {
  cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? BZ_OK : bz_fail_cuda(err, what);
}

static int use_device(int dev) {
  cudaError_t e = cudaSetDevice(dev);
  if (e != cudaSuccess) return bz_fail_cuda(e, "cudaSetDevice");
  e = cudaFree(nullptr);  // make the primary context current for driver calls
  if (e != cudaSuccess) return bz_fail_cuda(e, "cudaFree(0)");
  return driver_api() ? BZ_OK : BZ_ECUDA;
}

#define CU_TRY(expr)                                   \
  do {                                                 \
    CUresult _r = (expr);                              \
    if (_r != CUDA_SUCCESS) return bz_fail_cu(_r, #expr); \
  } while (0)

static CUmemAllocationProp slab_prop(int dev) {
  CUmemAllocationProp p;
  memset(&p, 0, sizeof(p));
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = dev;
  p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

static int slab_granularity(int dev, uint64_t* gran) {
  CUmemAllocationProp p = slab_prop(dev);
  size_t g = 0;
  CU_TRY(DRV()->cuMemGetAllocationGranularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  int mc = 0;
  CUdevice d;
  CU_TRY(DRV()->cuDeviceGet(&d, dev));
  CU_TRY(DRV()->cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d));
  if (mc) {
    CUmulticastObjectProp mp;
    memset(&mp, 0, sizeof(mp));
    mp.numDevices = 1;
    mp.size = g;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t mg = 0;
    if (DRV()->cuMulticastGetGranularity(&mg, &mp, CU_MULTICAST_GRANULARITY_MINIMUM) == CUDA_SUCCESS && mg > g) g = mg;
  }
  *gran = g;
  return BZ_OK;
}

static int map_rw(CUmemGenericAllocationHandle h, uint64_t bytes, uint64_t align, int dev, uint64_t* out) {
  CUdeviceptr ptr = 0;
  CU_TRY(DRV()->cuMemAddressReserve(&ptr, bytes, align, 0, 0));
  CUresult r = DRV()->cuMemMap(ptr, bytes, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    DRV()->cuMemAddressFree(ptr, bytes);
    return bz_fail_cu(r, "cuMemMap");
  }
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = DRV()->cuMemSetAccess(ptr, bytes, &acc, 1);
  if (r != CUDA_SUCCESS) {
    DRV()->cuMemUnmap(ptr, bytes);
    DRV()->cuMemAddressFree(ptr, bytes);
    return bz_fail_cu(r, "cuMemSetAccess");
  }
  *out = ptr;
  return BZ_OK;
}

// Duplicate file descriptor `fd` of process `pid` into this process.
static int steal_fd(int pid, int fd, int* out) {
  if (pid == getpid()) {
    *out = dup(fd);
    if (*out < 0) return bz_fail(BZ_ESYS, "dup failed");
    return BZ_OK;
  }
  int pfd = static_cast<int>(syscall(SYS_pidfd_open, pid, 0));
  if (pfd < 0) return bz_fail(BZ_ESYS, (std::string("pidfd_open: ") + strerror(errno)).c_str());
  int local = static_cast<int>(syscall(SYS_pidfd_getfd, pfd, fd, 0));
  int saved = errno;
  close(pfd);
  if (local < 0) return bz_fail(BZ_ESYS, (std::string("pidfd_getfd: ") + strerror(saved)).c_str());
  *out = local;
  return BZ_OK;
}

}  // namespace bz

using namespace bz;

extern "C" const char* bz_last_error(void) { return g_last_error.c_str(); }
extern "C" int bz_version(void) { return 1; }

extern "C" int bz_device_count(int* n) {
  cudaError_t e = cudaGetDeviceCount(n);
  return e == cudaSuccess ? BZ_OK : bz_fail_cuda(e, "cudaGetDeviceCount");
}

extern "C" int bz_device_caps(int dev, int* multicast, int* posix_fd, int* fabric, int* sm_count) {
  if (int rc = use_device(dev)) return rc;
  CUdevice d;
  CU_TRY(DRV()->cuDeviceGet(&d, dev));
  CU_TRY(DRV()->cuDeviceGetAttribute(multicast, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d));
  CU_TRY(DRV()->cuDeviceGetAttribute(posix_fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, d));
  CU_TRY(DRV()->cuDeviceGetAttribute(fabric, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d));
  CU_TRY(DRV()->cuDeviceGetAttribute(sm_count, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, d));
  return BZ_OK;
}

extern "C" int bz_sm_count(int dev, int* n) {
  cudaError_t e = cudaDeviceGetAttribute(n, cudaDevAttrMultiProcessorCount, dev);
  return e == cudaSuccess ? BZ_OK : bz_fail_cuda(e, "sm count");
}

// Load every kernel of libblitz into `dev`'s context now.  Under CUDA lazy
// loading a kernel's first launch loads its module, which can wait for the
// device to drain -- a deadlock when that launch is what a spinning gate or
// tracker kernel (already resident) is waiting for.  The data plane launches
// such producer/consumer pairs concurrently, so every module is loaded up front.
extern "C" int bz_preload_kernels(int dev, int* nloaded) {
  int prev = 0;
  cudaGetDevice(&prev);
  int rc = use_device(dev);
  int total = 0;
  const void* anchors[] = {module_anchor_dataplane(), module_anchor_decode(), module_anchor_gemm(),
                           module_anchor_llama(), module_anchor_attention()};
  for (const void* a : anchors) {
    if (rc) break;
    cudaFunction_t f = nullptr;
    cudaError_t e = cudaGetFuncBySymbol(&f, a);
    if (e != cudaSuccess) {
      rc = bz_fail_cuda(e, "preload: cudaGetFuncBySymbol");
      break;
    }
    CUmodule m = nullptr;
    unsigned n = 0;
    CUresult r = DRV()->cuFuncGetModule(&m, reinterpret_cast<CUfunction>(f));
    if (r == CUDA_SUCCESS) r = DRV()->cuModuleGetFunctionCount(&n, m);
    std::vector<CUfunction> fns(n);
    if (r == CUDA_SUCCESS && n) r = DRV()->cuModuleEnumerateFunctions(fns.data(), n, m);
    for (unsigned i = 0; r == CUDA_SUCCESS && i < n; ++i) r = DRV()->cuFuncLoad(fns[i]);
    if (r != CUDA_SUCCESS) {
      rc = bz_fail_cu(r, "preload: module functions");
      break;
    }
    total += static_cast<int>(n);
  }
  cudaSetDevice(prev);
  if (nloaded) *nloaded = total;
  return rc;
}

extern "C" int bz_enable_peer_mesh(int dev) {
  if (int rc = use_device(dev)) return rc;
  int n = 0;
  cudaGetDeviceCount(&n);
  for (int p = 0; p < n; ++p) {
    if (p == dev) continue;
    int ok = 0;
    cudaDeviceCanAccessPeer(&ok, dev, p);
    if (!ok) continue;
    cudaError_t e = cudaDeviceEnablePeerAccess(p, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
      cudaGetLastError();
    } else if (e != cudaSuccess) {
      return bz_fail_cuda(e, "cudaDeviceEnablePeerAccess");
    }
  }
  return BZ_OK;
}

extern "C" int bz_slab_create(int dev, uint64_t bytes, bz_slab* out) {
  if (!out || bytes == 0) return bz_fail(BZ_EINVAL, "slab_create: bad args");
  if (int rc = use_device(dev)) return rc;
  uint64_t gran = 0;
  if (int rc = slab_granularity(dev, &gran)) return rc;
  const uint64_t size = (bytes + gran - 1) / gran * gran;
  CUmemAllocationProp p = slab_prop(dev);
  CUmemGenericAllocationHandle h;
  CU_TRY(DRV()->cuMemCreate(&h, size, &p, 0));
  uint64_t ptr = 0;
  if (int rc = map_rw(h, size, gran, dev, &ptr)) {
    DRV()->cuMemRelease(h);
    return rc;
  }
  out->ptr = ptr;
  out->bytes = size;
  out->handle = static_cast<uint64_t>(h);
  out->dev = dev;
  out->fd = -1;
  return BZ_OK;
}

extern "C" int bz_slab_export(bz_slab* slab) {
  if (!slab) return bz_fail(BZ_EINVAL, "slab_export: null");
  if (slab->fd >= 0) return BZ_OK;
  int fd = -1;
  CU_TRY(DRV()->cuMemExportToShareableHandle(&fd, static_cast<CUmemGenericAllocationHandle>(slab->handle),
                                      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  slab->fd = fd;
  return BZ_OK;
}

extern "C" int bz_slab_import(int local_dev, int owner_pid, int owner_fd, uint64_t bytes, bz_slab* out) {
  if (!out) return bz_fail(BZ_EINVAL, "slab_import: null");
  if (int rc = use_device(local_dev)) return rc;
  int fd = -1;
  if (int rc = steal_fd(owner_pid, owner_fd, &fd)) return rc;
  CUmemGenericAllocationHandle h;
  CUresult r = DRV()->cuMemImportFromShareableHandle(&h, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
                                              CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  close(fd);
  if (r != CUDA_SUCCESS) return bz_fail_cu(r, "cuMemImportFromShareableHandle");
  uint64_t gran = 0;
  if (int rc = slab_granularity(local_dev, &gran)) return rc;
  uint64_t ptr = 0;
  if (int rc = map_rw(h, bytes, gran, local_dev, &ptr)) {
    DRV()->cuMemRelease(h);
    return rc;
  }
  out->ptr = ptr;
  out->bytes = bytes;
  out->handle = static_cast<uint64_t>(h);
  out->dev = -1;
  out->fd = -1;
  return BZ_OK;
}

extern "C" int bz_slab_free(bz_slab* slab) {
  if (!slab || !slab->ptr) return BZ_OK;
  CU_TRY(DRV()->cuMemUnmap(slab->ptr, slab->bytes));
  CU_TRY(DRV()->cuMemAddressFree(slab->ptr, slab->bytes));
  CU_TRY(DRV()->cuMemRelease(static_cast<CUmemGenericAllocationHandle>(slab->handle)));
  if (slab->fd >= 0) close(slab->fd);
  slab->ptr = 0;
  slab->fd = -1;
  return BZ_OK;
}

// ---- multicast -------------------------------------------------------------------

extern "C" int bz_mc_granularity(int dev, int ndev, uint64_t* min_gran, uint64_t* rec_gran) {
  if (int rc = use_device(dev)) return rc;
  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof(mp));
  mp.numDevices = ndev;
  mp.size = 1ull << 21;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t a = 0, b = 0;
  CU_TRY(DRV()->cuMulticastGetGranularity(&a, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CU_TRY(DRV()->cuMulticastGetGranularity(&b, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  *min_gran = a;
  *rec_gran = b;
  return BZ_OK;
}

extern "C" int bz_mc_create(int ndev, uint64_t bytes, bz_mc* out) {
  if (!out || ndev < 1 || bytes == 0) return bz_fail(BZ_EINVAL, "mc_create: bad args");
  if (!driver_api()) return BZ_ECUDA;
  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof(mp));
  mp.numDevices = ndev;
  mp.size = bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle h;
  CU_TRY(DRV()->cuMulticastCreate(&h, &mp));
  int fd = -1;
  CUresult r = DRV()->cuMemExportToShareableHandle(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  if (r != CUDA_SUCCESS) {
    DRV()->cuMemRelease(h);
    return bz_fail_cu(r, "export multicast");
  }
  out->handle = static_cast<uint64_t>(h);
  out->mc_ptr = 0;
  out->bytes = bytes;
  out->fd = fd;
  return BZ_OK;
}

extern "C" int bz_mc_import(int owner_pid, int owner_fd, uint64_t bytes, bz_mc* out) {
  if (!out) return bz_fail(BZ_EINVAL, "mc_import: null");
  int fd = -1;
  if (int rc = steal_fd(owner_pid, owner_fd, &fd)) return rc;
  CUmemGenericAllocationHandle h;
  CUresult r = DRV()->cuMemImportFromShareableHandle(&h, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
                                              CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  close(fd);
  if (r != CUDA_SUCCESS) return bz_fail_cu(r, "import multicast");
  out->handle = static_cast<uint64_t>(h);
  out->mc_ptr = 0;
  out->bytes = bytes;
  out->fd = -1;
  return BZ_OK;
}

extern "C" int bz_mc_add_device(bz_mc* mc, int dev) {
  if (int rc = use_device(dev)) return rc;
  CUdevice d;
  CU_TRY(DRV()->cuDeviceGet(&d, dev));
  CU_TRY(DRV()->cuMulticastAddDevice(static_cast<CUmemGenericAllocationHandle>(mc->handle), d));
  return BZ_OK;
}

extern "C" int bz_mc_bind(bz_mc* mc, int dev, const bz_slab* slab, uint64_t slab_offset, uint64_t mc_offset,
                          uint64_t bytes) {
  if (!mc || !slab) return bz_fail(BZ_EINVAL, "mc_bind: null");
  if (int rc = use_device(dev)) return rc;
  CU_TRY(DRV()->cuMulticastBindMem(static_cast<CUmemGenericAllocationHandle>(mc->handle), mc_offset,
                            static_cast<CUmemGenericAllocationHandle>(slab->handle), slab_offset, bytes, 0));
  return BZ_OK;
}

extern "C" int bz_mc_map(bz_mc* mc, int dev) {
  if (!mc) return bz_fail(BZ_EINVAL, "mc_map: null");
  if (int rc = use_device(dev)) return rc;
  uint64_t mn = 0, rec = 0;
  if (int rc = bz_mc_granularity(dev, 1, &mn, &rec)) return rc;
  uint64_t ptr = 0;
  if (int rc = map_rw(static_cast<CUmemGenericAllocationHandle>(mc->handle), mc->bytes, mn, dev, &ptr)) return rc;
  mc->mc_ptr = ptr;
  return BZ_OK;
}

extern "C" int bz_mc_unbind(bz_mc* mc, int dev, uint64_t bound_bytes) {
  if (!mc || !mc->handle) return bz_fail(BZ_EINVAL, "mc_unbind: null");
  if (int rc = use_device(dev)) return rc;
  CUdevice d;
  CU_TRY(DRV()->cuDeviceGet(&d, dev));
  CU_TRY(DRV()->cuMulticastUnbind(static_cast<CUmemGenericAllocationHandle>(mc->handle), d, 0, bound_bytes));
  return BZ_OK;
}

extern "C" int bz_mc_free(bz_mc* mc, int dev, uint64_t bound_bytes) {
  if (!mc) return BZ_OK;
  if (mc->mc_ptr) {
    DRV()->cuMemUnmap(mc->mc_ptr, mc->bytes);
    DRV()->cuMemAddressFree(mc->mc_ptr, mc->bytes);
    mc->mc_ptr = 0;
  }
  if (bound_bytes) {
    CUdevice d;
    if (DRV()->cuDeviceGet(&d, dev) == CUDA_SUCCESS)
      DRV()->cuMulticastUnbind(static_cast<CUmemGenericAllocationHandle>(mc->handle), d, 0, bound_bytes);
  }
  if (mc->handle) DRV()->cuMemRelease(static_cast<CUmemGenericAllocationHandle>(mc->handle));
  mc->handle = 0;
  if (mc->fd >= 0) close(mc->fd);
  mc->fd = -1;
  return BZ_OK;
}
