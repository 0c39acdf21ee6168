// dsgd_multicast.h -- NVSwitch multicast (NVLS) buffers for the two-shot
// all-reduce, owned by the library (CUDA driver multicast objects): the
// exchange buffer x and the average buffer of every rank are one multicast
// object with per-GPU physical backing; the reduce kernel reads the sum of
// every GPU's x through the multicast address (multimem.ld_reduce) and
// writes the average to every GPU with one multimem.st.
#pragma once

#include <cuda.h>
#include <stddef.h>
#include <stdint.h>

#include <atomic>

#include "dsgd_b200.h"

namespace dsgd {

struct McState {
  CUmemGenericAllocationHandle mc = 0;    // the multicast object
  CUmemGenericAllocationHandle phys = 0;  // this GPU's backing
  CUdeviceptr uc = 0;                     // unicast mapping of the backing
  CUdeviceptr mcva = 0;                   // multicast mapping
  size_t size = 0;
  size_t gran = 0;                        // mapping alignment
  int export_fd = -1;                     // rank 0: the exported POSIX fd (until all imported)
  bool owns_mc = true;                    // releases `mc` (when `refs` is null)
  // in-process group: the contexts sharing one object count its holders; the
  // last one to release it (in any order) releases the object
  std::atomic<int>* refs = nullptr;
  bool added = false, bound = false, mapped_uc = false, mapped_mc = false;
};

// Device attribute CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED.
bool mc_supported(int device);
// Creates the object for p GPUs with >= `need` bytes per GPU (size rounded to
// the multicast and allocation granularities); shareable: exportable as a
// POSIX file descriptor (one process per GPU).
dsgd_status mc_create(McState* s, int device, uint32_t p, size_t need, bool shareable);
dsgd_status mc_export_fd(McState* s, int* fd);
// Imports rank 0's object through pidfd_getfd(pid, fd).
dsgd_status mc_import_fd(McState* s, int pid, int fd, size_t size);
// `s` joins `owner`'s object in the same process (shared holder count).
void mc_share(McState* s, McState* owner);
dsgd_status mc_add_device(McState* s, int device);
// Backing on `device`, bound to the object, mapped unicast and multicast.
// Blocks until every device of the team has been added.
dsgd_status mc_bind_map(McState* s, int device, bool shareable);
void mc_release(McState* s, int device);

}  // namespace dsgd
