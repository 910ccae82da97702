// mc_mcast.cu — NVLink multicast (NVLS) gather buffers for the fused push.
//
// A multicast object spans the gather buffers of every participating device: one
// `multimem.st` to the multicast address of a byte lands at that offset in every device's
// buffer, so the push of a rank's payload into its slot of every rank's gather buffer is one
// store per word instead of N (mc_encode_push_mc), and the flag word likewise.  This file
// owns the object: physical memory per device, bound to the object, mapped once per device
// (unicast: where the decode reads) and once for the multicast address (where the push
// writes).  The driver API is reached through cudaGetDriverEntryPoint, so the library does
// not link libcuda (it still loads on a machine without a driver).
//
// Replaces nothing in the reference (its allgather is a Python list, trainer.py:377-389).
// Scope: devices owned by one process (single-process multi-GPU, or one device and N
// simulated ranks); the object and memory are created with POSIX-fd handle types (as NCCL's
// NVLS buffers) so a later multi-process version can export them.  Status: on this pool's
// single-GPU boxes cuMulticastCreate returns CUDA_ERROR_INVALID_VALUE for every property set
// although CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED is 1 (scripts/probes/mcast_probe.py; torch's
// symmetric memory also falls back there), so this path compiles and its test skips — it
// has not run on hardware.
#include <cuda.h>

#include <cstring>

#include "mc_internal.cuh"

struct mc_mcast {
  int ndev = 0;
  int dev[mc::MC_MAX_PUSH] = {};
  size_t size = 0;
  CUmemGenericAllocationHandle mc = 0;
  CUmemGenericAllocationHandle mem[mc::MC_MAX_PUSH] = {};
  CUdeviceptr uc[mc::MC_MAX_PUSH] = {};
  CUdeviceptr mcva = 0;
};

namespace {

#define MC_DRV_FN(name) decltype(&name) p_##name = nullptr
struct Drv {
  MC_DRV_FN(cuDeviceGet);
  MC_DRV_FN(cuMulticastGetGranularity);
  MC_DRV_FN(cuMulticastCreate);
  MC_DRV_FN(cuMulticastAddDevice);
  MC_DRV_FN(cuMulticastBindMem);
  MC_DRV_FN(cuMulticastUnbind);
  MC_DRV_FN(cuMemGetAllocationGranularity);
  MC_DRV_FN(cuMemCreate);
  MC_DRV_FN(cuMemRelease);
  MC_DRV_FN(cuMemAddressReserve);
  MC_DRV_FN(cuMemAddressFree);
  MC_DRV_FN(cuMemMap);
  MC_DRV_FN(cuMemUnmap);
  MC_DRV_FN(cuMemSetAccess);
  MC_DRV_FN(cuDeviceGetAttribute);
  bool ok = false;
};
#undef MC_DRV_FN

const Drv& drv() {
  static const Drv d = [] {
    Drv x;
    bool ok = true;
    auto get = [&](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
          !*fn)
        ok = false;
    };
#define MC_GET(name) get(#name, reinterpret_cast<void**>(&x.p_##name))
    MC_GET(cuDeviceGet);
    MC_GET(cuMulticastGetGranularity);
    MC_GET(cuMulticastCreate);
    MC_GET(cuMulticastAddDevice);
    MC_GET(cuMulticastBindMem);
    MC_GET(cuMulticastUnbind);
    MC_GET(cuMemGetAllocationGranularity);
    MC_GET(cuMemCreate);
    MC_GET(cuMemRelease);
    MC_GET(cuMemAddressReserve);
    MC_GET(cuMemAddressFree);
    MC_GET(cuMemMap);
    MC_GET(cuMemUnmap);
    MC_GET(cuMemSetAccess);
    MC_GET(cuDeviceGetAttribute);
#undef MC_GET
    cudaGetLastError();
    x.ok = ok;
    return x;
  }();
  return d;
}

#define MC_CU(call)                                                                     \
  do {                                                                                  \
    const CUresult r_ = (call);                                                         \
    if (r_ != CUDA_SUCCESS) {                                                           \
      mc::set_error("%s failed: CUresult %d (%s:%d)", #call, (int)r_, __FILE__, __LINE__); \
      mc_mcast_destroy(h);                                                              \
      return MC_EPEER;                                                                  \
    }                                                                                   \
  } while (0)

}  // namespace

extern "C" {

void mc_mcast_destroy(mc_mcast* h) {
  if (!h) return;
  const Drv& d = drv();
  if (d.ok) {
    if (h->mcva) {
      d.p_cuMemUnmap(h->mcva, h->size);
      d.p_cuMemAddressFree(h->mcva, h->size);
    }
    for (int i = 0; i < h->ndev; ++i) {
      if (h->uc[i]) {
        d.p_cuMemUnmap(h->uc[i], h->size);
        d.p_cuMemAddressFree(h->uc[i], h->size);
      }
      if (h->mc && h->mem[i]) {
        CUdevice cd;
        if (d.p_cuDeviceGet(&cd, h->dev[i]) == CUDA_SUCCESS) d.p_cuMulticastUnbind(h->mc, cd, 0, h->size);
      }
      if (h->mem[i]) d.p_cuMemRelease(h->mem[i]);
    }
    if (h->mc) d.p_cuMemRelease(h->mc);
  }
  delete h;
}

int mc_mcast_create(const int32_t* devices, int32_t ndev, int64_t bytes, mc_mcast** out) {
  if (!devices || ndev < 1 || ndev > mc::MC_MAX_PUSH || bytes < 1 || !out) {
    mc::set_error("bad mc_mcast_create arguments");
    return MC_EINVAL;
  }
  *out = nullptr;
  const Drv& d = drv();
  if (!d.ok) { mc::set_error("driver entry points for multicast unavailable"); return MC_EPEER; }
  mc_mcast* h = new (std::nothrow) mc_mcast();
  if (!h) { mc::set_error("out of host memory"); return MC_EINVAL; }
  h->ndev = ndev;
  for (int i = 0; i < ndev; ++i) {
    h->dev[i] = devices[i];
    CUdevice cd;
    MC_CU(d.p_cuDeviceGet(&cd, devices[i]));
    int sup = 0;
    MC_CU(d.p_cuDeviceGetAttribute(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd));
    if (!sup) {
      mc::set_error("device %d does not support multicast objects", devices[i]);
      mc_mcast_destroy(h);
      return MC_EPEER;
    }
  }
  CUmulticastObjectProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.numDevices = (unsigned)ndev;
  prop.size = (size_t)bytes;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // as NCCL's NVLS buffers (exportable later)
  size_t gran = 0;
  MC_CU(d.p_cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = devices[0];
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t agran = 0;
  MC_CU(d.p_cuMemGetAllocationGranularity(&agran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t g = gran > agran ? gran : agran;
  h->size = ((size_t)bytes + g - 1) / g * g;
  prop.size = h->size;
  MC_CU(d.p_cuMulticastCreate(&h->mc, &prop));
  for (int i = 0; i < ndev; ++i) {  // every device joins before any memory is bound
    CUdevice cd;
    MC_CU(d.p_cuDeviceGet(&cd, devices[i]));
    MC_CU(d.p_cuMulticastAddDevice(h->mc, cd));
  }
  CUmemAccessDesc acc[mc::MC_MAX_PUSH];
  for (int i = 0; i < ndev; ++i) {
    ap.location.id = devices[i];
    MC_CU(d.p_cuMemCreate(&h->mem[i], h->size, &ap, 0));
    MC_CU(d.p_cuMulticastBindMem(h->mc, 0, h->mem[i], 0, h->size, 0));
    MC_CU(d.p_cuMemAddressReserve(&h->uc[i], h->size, g, 0, 0));
    MC_CU(d.p_cuMemMap(h->uc[i], h->size, 0, h->mem[i], 0));
    acc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[i].location.id = devices[i];
    acc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    MC_CU(d.p_cuMemSetAccess(h->uc[i], h->size, &acc[i], 1));
  }
  MC_CU(d.p_cuMemAddressReserve(&h->mcva, h->size, g, 0, 0));
  MC_CU(d.p_cuMemMap(h->mcva, h->size, 0, h->mc, 0));
  MC_CU(d.p_cuMemSetAccess(h->mcva, h->size, acc, (size_t)ndev));
  *out = h;
  return MC_OK;
}

int mc_mcast_ptrs(const mc_mcast* h, void** unicast, void** multicast, int64_t* bytes) {
  if (!h) { mc::set_error("null multicast object"); return MC_EINVAL; }
  if (unicast)
    for (int i = 0; i < h->ndev; ++i) unicast[i] = reinterpret_cast<void*>(h->uc[i]);
  if (multicast) *multicast = reinterpret_cast<void*>(h->mcva);
  if (bytes) *bytes = (int64_t)h->size;
  return MC_OK;
}

}  // extern "C"
