// dsgd_multicast.cpp -- NVSwitch multicast objects for the NVLS all-reduce
// (see dsgd_multicast.h), with the CUDA driver API: cuMulticastCreate /
// cuMulticastAddDevice / cuMemCreate / cuMulticastBindMem / cuMemMap.  One
// process per GPU shares rank 0's object as a POSIX file descriptor fetched
// with pidfd_getfd (no helper process, no socket); an in-process group adds
// all its GPUs itself.
#include "dsgd_multicast.h"

#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <string>

#include "dsgd_internal.h"

#ifndef SYS_pidfd_open
#define SYS_pidfd_open 434
#endif
#ifndef SYS_pidfd_getfd
#define SYS_pidfd_getfd 438
#endif

namespace dsgd {

namespace {

// Driver entry points are resolved through the runtime (the library does not
// link libcuda, so it still loads on a machine without a driver, e.g. for the
// CPU-side ABI checks); a missing one reports CUDA_ERROR_NOT_FOUND.
template <typename F>
struct Drv;
template <typename R, typename... A>
struct Drv<R (*)(A...)> {
  R (*fn)(A...);
  R operator()(A... a) const { return fn ? fn(a...) : CUDA_ERROR_NOT_FOUND; }
};
template <typename F>
Drv<F> drv(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    fn = nullptr;
  return Drv<F>{reinterpret_cast<F>(fn)};
}
// DRV(cuFoo)(args...): cuFoo with the type cuda.h declares for it
#define DRV(fn) drv<decltype(&fn)>(#fn)

dsgd_status cu_fail(CUresult r, const char* what) {
  const char* s = nullptr;
  DRV(cuGetErrorString)(r, &s);
  const std::string why = s ? std::string(s) : "CUDA driver error " + std::to_string((int)r);
  return set_error(DSGD_ECUDA, std::string(what) + ": " + why);
}

#define CU_TRY(fn, ...)                              \
  do {                                               \
    CUresult r_ = DRV(fn)(__VA_ARGS__);              \
    if (r_ != CUDA_SUCCESS) return cu_fail(r_, #fn); \
  } while (0)

CUmemAllocationProp phys_prop(int device, bool shareable) {
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  // an exported / imported multicast object binds only shareable memory
  p.requestedHandleTypes = shareable ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
                                     : CU_MEM_HANDLE_TYPE_NONE;
  return p;
}

}  // namespace

bool mc_supported(int device) {
  if (cudaFree(nullptr) != cudaSuccess) return false;  // the runtime's context exists
  CUdevice d;
  if (DRV(cuDeviceGet)(&d, device) != CUDA_SUCCESS) return false;
  int v = 0;
  if (DRV(cuDeviceGetAttribute)(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d) != CUDA_SUCCESS)
    return false;
  return v != 0;
}

dsgd_status mc_create(McState* s, int device, uint32_t p, size_t need, bool shareable) {
  CUmulticastObjectProp prop = {};
  prop.numDevices = p;
  prop.handleTypes = shareable ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : 0;
  prop.size = need;
  size_t g_mc = 0, g_mem = 0;
  CU_TRY(cuMulticastGetGranularity, &g_mc, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  const CUmemAllocationProp mp = phys_prop(device, shareable);
  CU_TRY(cuMemGetAllocationGranularity, &g_mem, &mp, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  const size_t g = std::max(g_mc, g_mem);
  prop.size = (need + g - 1) / g * g;
  CU_TRY(cuMulticastCreate, &s->mc, &prop);
  s->size = prop.size;
  s->gran = g;
  return DSGD_OK;
}

dsgd_status mc_export_fd(McState* s, int* fd) {
  int out = -1;
  CU_TRY(cuMemExportToShareableHandle, &out, s->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  s->export_fd = out;
  *fd = out;
  return DSGD_OK;
}

dsgd_status mc_import_fd(McState* s, int pid, int fd, size_t size) {
  const long pfd = syscall(SYS_pidfd_open, pid, 0);
  if (pfd < 0) return set_error(DSGD_ECUDA, "pidfd_open of rank 0 failed");
  const long local = syscall(SYS_pidfd_getfd, (int)pfd, fd, 0);
  close((int)pfd);
  if (local < 0) return set_error(DSGD_ECUDA, "pidfd_getfd of the multicast handle failed");
  const CUresult r = DRV(cuMemImportFromShareableHandle)(
      &s->mc, reinterpret_cast<void*>(static_cast<uintptr_t>(local)),
      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  close((int)local);
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemImportFromShareableHandle");
  s->size = size;
  s->gran = size & (~size + 1);  // the largest power of two dividing the size
  if (s->gran > (size_t(1) << 30)) s->gran = size_t(1) << 30;
  return DSGD_OK;
}

void mc_share(McState* s, McState* owner) {
  if (!owner->refs) owner->refs = new std::atomic<int>(1);
  owner->refs->fetch_add(1);
  s->mc = owner->mc;
  s->size = owner->size;
  s->gran = owner->gran;
  s->refs = owner->refs;
}

dsgd_status mc_add_device(McState* s, int device) {
  CUdevice d;
  CU_TRY(cuDeviceGet, &d, device);
  CU_TRY(cuMulticastAddDevice, s->mc, d);
  s->added = true;
  return DSGD_OK;
}

dsgd_status mc_bind_map(McState* s, int device, bool shareable) {
  const CUmemAllocationProp mp = phys_prop(device, shareable);
  CU_TRY(cuMemCreate, &s->phys, s->size, &mp, 0);
  CU_TRY(cuMulticastBindMem, s->mc, 0, s->phys, 0, s->size, 0);
  s->bound = true;
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU_TRY(cuMemAddressReserve, &s->uc, s->size, s->gran, 0, 0);
  CU_TRY(cuMemMap, s->uc, s->size, 0, s->phys, 0);
  s->mapped_uc = true;
  CU_TRY(cuMemSetAccess, s->uc, s->size, &acc, 1);
  CU_TRY(cuMemAddressReserve, &s->mcva, s->size, s->gran, 0, 0);
  CU_TRY(cuMemMap, s->mcva, s->size, 0, s->mc, 0);
  s->mapped_mc = true;
  CU_TRY(cuMemSetAccess, s->mcva, s->size, &acc, 1);
  return DSGD_OK;
}

void mc_release(McState* s, int device) {
  if (s->mapped_mc) DRV(cuMemUnmap)(s->mcva, s->size);
  if (s->mcva) DRV(cuMemAddressFree)(s->mcva, s->size);
  if (s->mapped_uc) DRV(cuMemUnmap)(s->uc, s->size);
  if (s->uc) DRV(cuMemAddressFree)(s->uc, s->size);
  if (s->bound) {
    CUdevice d;
    if (DRV(cuDeviceGet)(&d, device) == CUDA_SUCCESS) DRV(cuMulticastUnbind)(s->mc, d, 0, s->size);
  }
  if (s->phys) DRV(cuMemRelease)(s->phys);
  if (s->refs) {
    // shared in-process object: only the last holder releases it (every
    // other holder has unbound its device by then)
    if (s->refs->fetch_sub(1) == 1) {
      if (s->mc) DRV(cuMemRelease)(s->mc);
      delete s->refs;
    }
  } else if (s->mc && s->owns_mc) {
    DRV(cuMemRelease)(s->mc);
  }
  if (s->export_fd >= 0) close(s->export_fd);
  *s = McState{};
}

}  // namespace dsgd
