// NVLS (NVSwitch multicast) buffers for the position all-gather of the sharded leapfrog
// (DESIGN.md §6). One multicast object spans the ranks' GPUs; every
// rank binds a local allocation to it and maps both the unicast view (its own copy, read by
// the force kernel) and the multicast view: one `multimem.st` of a position into the
// multicast view lands in every rank's copy through the switch -- the all-gather is the
// update kernel's stores, one store per particle instead of one per peer.
//
// Driver API through cudaGetDriverEntryPointByVersion (no link-time libcuda dependency, so
// the library still loads on machines without a driver). Handles travel between processes
// as fabric handles (CU_MEM_HANDLE_TYPE_FABRIC: 64 bytes, no file-descriptor passing).
//
// Set-up order (multicast object rules): rank 0 creates the object, adds its device and
// exports the handle; every other rank imports it and adds its device; only after ALL ranks
// added their devices (a host barrier) does each rank bind its memory and map the views.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace b2 {
namespace {

struct Driver {
  CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                               unsigned long long) = nullptr;
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long) = nullptr;
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*,
                                          CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  bool ok = false;
};

template <class F>
bool entry(const char* name, F& fn) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPointByVersion(name, &p, 12010, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p) {
    cudaGetLastError();
    return false;
  }
  fn = reinterpret_cast<F>(p);
  return true;
}

const Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = entry("cuDeviceGet", d.DeviceGet) && entry("cuDeviceGetAttribute", d.DeviceGetAttribute) &&
           entry("cuMulticastCreate", d.MulticastCreate) &&
           entry("cuMulticastGetGranularity", d.MulticastGetGranularity) &&
           entry("cuMulticastAddDevice", d.MulticastAddDevice) && entry("cuMulticastBindMem", d.MulticastBindMem) &&
           entry("cuMulticastUnbind", d.MulticastUnbind) &&
           entry("cuMemExportToShareableHandle", d.MemExportToShareableHandle) &&
           entry("cuMemImportFromShareableHandle", d.MemImportFromShareableHandle) &&
           entry("cuMemCreate", d.MemCreate) && entry("cuMemRelease", d.MemRelease) &&
           entry("cuMemGetAllocationGranularity", d.MemGetAllocationGranularity) &&
           entry("cuMemAddressReserve", d.MemAddressReserve) && entry("cuMemAddressFree", d.MemAddressFree) &&
           entry("cuMemMap", d.MemMap) && entry("cuMemUnmap", d.MemUnmap) && entry("cuMemSetAccess", d.MemSetAccess);
  });
  return d;
}

// CUresult -> the library's status (positive, in the cudaError_t range callers already print
// through b2_error_string; the driver codes used here share their numbers with cudaError_t)
int status(CUresult r) { return r == CUDA_SUCCESS ? B2_OK : static_cast<int>(r); }

CUmulticastObjectProp mc_prop(size_t bytes, int ndev) {
  CUmulticastObjectProp p;
  std::memset(&p, 0, sizeof p);
  p.numDevices = static_cast<unsigned int>(ndev);
  p.size = bytes;
  p.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
  return p;
}

}  // namespace

// The mapped state of one rank's binding (what b2_mc_bind returns as an opaque handle).
struct McBinding {
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  CUdeviceptr uc = 0, mcva = 0;
  size_t bytes = 0;
  CUdevice dev = 0;
};

}  // namespace b2

using namespace b2;

extern "C" {

int b2_mc_supported(int device) {
  const Driver& d = driver();
  if (!d.ok) return 0;
  CUdevice dev;
  int mc = 0, fabric = 0;
  if (d.DeviceGet(&dev, device) != CUDA_SUCCESS) return 0;
  if (d.DeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS) return 0;
  if (d.DeviceGetAttribute(&fabric, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev) != CUDA_SUCCESS) return 0;
  if (!mc || !fabric) return 0;
  // the attributes say what the GPU can do, not whether this process reaches the fabric (a
  // container without the NVSwitch / IMEX devices): create and drop a minimal object, once
  static int reachable = -1;
  if (reachable < 0) {
    const CUmulticastObjectProp p = mc_prop(2u << 20, 1);
    size_t g = 0;
    CUmemGenericAllocationHandle h;
    CUmulticastObjectProp q = p;
    if (d.MulticastGetGranularity(&g, &p, CU_MULTICAST_GRANULARITY_MINIMUM) == CUDA_SUCCESS && g) q.size = g;
    reachable = d.MulticastCreate(&h, &q) == CUDA_SUCCESS;
    if (reachable) d.MemRelease(h);
  }
  return reachable;
}

size_t b2_mc_handle_bytes(void) { return sizeof(CUmemFabricHandle); }

int b2_mc_granular_bytes(size_t bytes, int ndev, size_t* out) {
  const Driver& d = driver();
  if (!d.ok) return B2_ENOTSUP;
  if (!out || ndev < 1 || bytes == 0) return B2_EINVAL;
  const CUmulticastObjectProp p = mc_prop(bytes, ndev);
  size_t g = 0;
  if (int rc = status(d.MulticastGetGranularity(&g, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED))) return rc;
  *out = (bytes + g - 1) / g * g;
  return B2_OK;
}

int b2_mc_create(size_t bytes, int ndev, int device, void* handle, void** binding) {
  const Driver& d = driver();
  if (!d.ok) return B2_ENOTSUP;
  if (!handle || !binding || ndev < 1 || bytes == 0) return B2_EINVAL;
  const CUmulticastObjectProp p = mc_prop(bytes, ndev);
  auto* b = new McBinding;
  int rc = status(d.MulticastCreate(&b->mc, &p));
  CUmemFabricHandle fh;
  if (!rc) rc = status(d.MemExportToShareableHandle(&fh, b->mc, CU_MEM_HANDLE_TYPE_FABRIC, 0));
  if (!rc) rc = status(d.DeviceGet(&b->dev, device));
  if (!rc) rc = status(d.MulticastAddDevice(b->mc, b->dev));
  if (rc) {
    if (b->mc) d.MemRelease(b->mc);
    delete b;
    return rc;
  }
  std::memcpy(handle, &fh, sizeof fh);
  *binding = b;  // the creator's reference keeps the object alive until b2_mc_release
  return B2_OK;
}

int b2_mc_add_device(const void* handle, int device, void** binding) {
  const Driver& d = driver();
  if (!d.ok) return B2_ENOTSUP;
  if (!handle || !binding) return B2_EINVAL;
  auto* b = new McBinding;
  CUmemFabricHandle fh;
  std::memcpy(&fh, handle, sizeof fh);
  int rc = status(d.MemImportFromShareableHandle(&b->mc, &fh, CU_MEM_HANDLE_TYPE_FABRIC));
  if (!rc) rc = status(d.DeviceGet(&b->dev, device));
  if (!rc) rc = status(d.MulticastAddDevice(b->mc, b->dev));
  if (rc) {
    if (b->mc) d.MemRelease(b->mc);
    delete b;
    return rc;
  }
  *binding = b;
  return B2_OK;
}

int b2_mc_bind(void* binding, size_t bytes, void** uc_ptr, void** mc_ptr) {
  const Driver& d = driver();
  if (!d.ok) return B2_ENOTSUP;
  auto* b = static_cast<McBinding*>(binding);
  if (!b || !uc_ptr || !mc_ptr || bytes == 0) return B2_EINVAL;
  CUmemAllocationProp ap;
  std::memset(&ap, 0, sizeof ap);
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = b->dev;
  int rc;
  if ((rc = status(d.MemCreate(&b->mem, bytes, &ap, 0)))) return rc;
  b->bytes = bytes;
  if ((rc = status(d.MulticastBindMem(b->mc, 0, b->mem, 0, bytes, 0)))) return rc;
  CUmemAccessDesc acc;
  std::memset(&acc, 0, sizeof acc);
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = b->dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if ((rc = status(d.MemAddressReserve(&b->uc, bytes, 0, 0, 0))) || (rc = status(d.MemMap(b->uc, bytes, 0, b->mem, 0))) ||
      (rc = status(d.MemSetAccess(b->uc, bytes, &acc, 1))))
    return rc;
  if ((rc = status(d.MemAddressReserve(&b->mcva, bytes, 0, 0, 0))) ||
      (rc = status(d.MemMap(b->mcva, bytes, 0, b->mc, 0))) || (rc = status(d.MemSetAccess(b->mcva, bytes, &acc, 1))))
    return rc;
  *uc_ptr = reinterpret_cast<void*>(b->uc);
  *mc_ptr = reinterpret_cast<void*>(b->mcva);
  return B2_OK;
}

int b2_mc_release(void* binding) {
  const Driver& d = driver();
  auto* b = static_cast<McBinding*>(binding);
  if (!b) return B2_OK;
  if (d.ok) {
    cudaDeviceSynchronize();
    if (b->mcva) {
      d.MemUnmap(b->mcva, b->bytes);
      d.MemAddressFree(b->mcva, b->bytes);
    }
    if (b->uc) {
      d.MemUnmap(b->uc, b->bytes);
      d.MemAddressFree(b->uc, b->bytes);
    }
    if (b->mem) {
      d.MulticastUnbind(b->mc, b->dev, 0, b->bytes);
      d.MemRelease(b->mem);
    }
    if (b->mc) d.MemRelease(b->mc);
  }
  delete b;
  return B2_OK;
}

}  // extern "C"
