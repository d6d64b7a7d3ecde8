// nvls.cpp — NVLink SHARP multicast windows for DTD's all-gathers (MOE_F_NVLS, comm.h).
//
// One region per rank holds the windows the all-gathers write (the X / O rings, dY, dS).
// It is a VMM allocation (cuMemCreate) exported as a POSIX file descriptor, so every rank
// maps every peer's region for the unicast exchange writes (the role cudaIpc* plays for the
// other windows), and each TP group (G_t ranks) shares one multicast object bound to its
// members' regions: a multimem.st through the group's multicast mapping lands at the same
// offset in every member's region, replicated by the NVSwitch. (pid, fd) pairs travel over
// the temporary NCCL world communicator of comm_create and each importer duplicates the
// descriptor with pidfd_getfd (fabric handles need an IMEX channel, which this box does not
// grant). Driver entry points are resolved at run time (no libcuda link).
#include "comm.h"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

#include <sys/prctl.h>
#include <sys/syscall.h>
#include <unistd.h>

namespace moe {
namespace {

struct Drv {
  PFN_cuDeviceGet_v2000 deviceGet = nullptr;
  PFN_cuDeviceGetAttribute_v2000 devAttr = nullptr;
  PFN_cuMemCreate_v10020 memCreate = nullptr;
  PFN_cuMemRelease_v10020 memRelease = nullptr;
  PFN_cuMemExportToShareableHandle_v10020 exportHandle = nullptr;
  PFN_cuMemImportFromShareableHandle_v10020 importHandle = nullptr;
  PFN_cuMemAddressReserve_v10020 addrReserve = nullptr;
  PFN_cuMemAddressFree_v10020 addrFree = nullptr;
  PFN_cuMemMap_v10020 map = nullptr;
  PFN_cuMemUnmap_v10020 unmap = nullptr;
  PFN_cuMemSetAccess_v10020 setAccess = nullptr;
  PFN_cuMemGetAllocationGranularity_v10020 allocGran = nullptr;
  PFN_cuMulticastCreate_v12010 mcCreate = nullptr;
  PFN_cuMulticastAddDevice_v12010 mcAddDevice = nullptr;
  PFN_cuMulticastBindMem_v12010 mcBindMem = nullptr;
  PFN_cuMulticastUnbind_v12010 mcUnbind = nullptr;
  PFN_cuMulticastGetGranularity_v12010 mcGran = nullptr;
  PFN_cuGetErrorString_v6000 errString = nullptr;
  bool ok = false;
};

Drv& drv() {
  static Drv d = [] {
    Drv x;
    bool ok = true;
    auto get = [&](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess || !*fn)
        ok = false;
    };
    get("cuDeviceGet", reinterpret_cast<void**>(&x.deviceGet));
    get("cuDeviceGetAttribute", reinterpret_cast<void**>(&x.devAttr));
    get("cuMemCreate", reinterpret_cast<void**>(&x.memCreate));
    get("cuMemRelease", reinterpret_cast<void**>(&x.memRelease));
    get("cuMemExportToShareableHandle", reinterpret_cast<void**>(&x.exportHandle));
    get("cuMemImportFromShareableHandle", reinterpret_cast<void**>(&x.importHandle));
    get("cuMemAddressReserve", reinterpret_cast<void**>(&x.addrReserve));
    get("cuMemAddressFree", reinterpret_cast<void**>(&x.addrFree));
    get("cuMemMap", reinterpret_cast<void**>(&x.map));
    get("cuMemUnmap", reinterpret_cast<void**>(&x.unmap));
    get("cuMemSetAccess", reinterpret_cast<void**>(&x.setAccess));
    get("cuMemGetAllocationGranularity", reinterpret_cast<void**>(&x.allocGran));
    get("cuMulticastCreate", reinterpret_cast<void**>(&x.mcCreate));
    get("cuMulticastAddDevice", reinterpret_cast<void**>(&x.mcAddDevice));
    get("cuMulticastBindMem", reinterpret_cast<void**>(&x.mcBindMem));
    get("cuMulticastUnbind", reinterpret_cast<void**>(&x.mcUnbind));
    get("cuMulticastGetGranularity", reinterpret_cast<void**>(&x.mcGran));
    get("cuGetErrorString", reinterpret_cast<void**>(&x.errString));
    x.ok = ok;
    return x;
  }();
  return d;
}

moe_status cu_fail(CUresult r, const char* what, std::string* why) {
  const char* s = nullptr;
  if (drv().errString) drv().errString(r, &s);
  *why = std::string(what) + ": " + (s ? s : "CUDA driver error");
  return r == CUDA_ERROR_NOT_SUPPORTED ? MOE_ERR_UNSUPPORTED : MOE_ERR_CUDA;
}

#define CU(expr)                                        \
  do {                                                  \
    CUresult _r = (expr);                               \
    if (_r != CUDA_SUCCESS) return cu_fail(_r, #expr, why); \
  } while (0)

// Maps `h` (size bytes) into a fresh VA range readable / writable by `dev`.
moe_status map_rw(CUmemGenericAllocationHandle h, size_t size, int dev, void** va, std::string* why) {
  Drv& D = drv();
  CUdeviceptr p = 0;
  CU(D.addrReserve(&p, size, 0, 0, 0));
  CUresult r = D.map(p, size, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    D.addrFree(p, size);
    return cu_fail(r, "cuMemMap", why);
  }
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = dev;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = D.setAccess(p, size, &ad, 1);
  if (r != CUDA_SUCCESS) {
    D.unmap(p, size);
    D.addrFree(p, size);
    return cu_fail(r, "cuMemSetAccess", why);
  }
  *va = reinterpret_cast<void*>(p);
  return MOE_OK;
}

moe_status nccl_sync(ncclComm_t comm, std::string* why) {
  int* d = nullptr;
  if (cudaMalloc(&d, sizeof(int)) != cudaSuccess) { *why = "cudaMalloc (sync word)"; return MOE_ERR_CUDA; }
  cudaStream_t st = nullptr;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  ncclResult_t r = ncclAllReduce(d, d, 1, ncclInt32, ncclSum, comm, st);
  cudaError_t e = r == ncclSuccess ? cudaStreamSynchronize(st) : cudaSuccess;
  cudaStreamDestroy(st);
  cudaFree(d);
  if (r != ncclSuccess) { *why = std::string("ncclAllReduce (sync): ") + ncclGetErrorString(r); return MOE_ERR_NCCL; }
  if (e != cudaSuccess) { *why = std::string("sync: ") + cudaGetErrorString(e); return MOE_ERR_CUDA; }
  return MOE_OK;
}

struct Handles {
  int32_t pid, phys_fd, mc_fd;
};

// A duplicate of descriptor `fd` of process `pid` in this process (-1 on failure).
int grab_fd(int pid, int fd) {
#if defined(SYS_pidfd_open) && defined(SYS_pidfd_getfd)
  const int pfd = (int)syscall(SYS_pidfd_open, pid, 0);
  if (pfd < 0) return -1;
  const int out = (int)syscall(SYS_pidfd_getfd, pfd, fd, 0);
  close(pfd);
  return out;
#else
  (void)pid; (void)fd;
  return -1;
#endif
}

}  // namespace

moe_status nvls_create(NvlsRegion* R, size_t bytes, int world, int rank, int Gt, ncclComm_t comm, std::string* why) {
  Drv& D = drv();
  if (!D.ok) { *why = "CUDA driver without the VMM / multicast entry points"; return MOE_ERR_UNSUPPORTED; }
  int dev_ord = 0;
  if (cudaGetDevice(&dev_ord) != cudaSuccess) { *why = "cudaGetDevice"; return MOE_ERR_CUDA; }
  CUdevice dev;
  CU(D.deviceGet(&dev, dev_ord));
  int mc_ok = 0;
  D.devAttr(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  if (!mc_ok) { *why = "this GPU does not support multicast objects (NVLink SHARP)"; return MOE_ERR_UNSUPPORTED; }

  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev_ord;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmulticastObjectProp mp = {};
  mp.numDevices = (unsigned)Gt;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g1 = 0, g2 = 0;
  CU(D.allocGran(&g1, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  mp.size = bytes;
  CU(D.mcGran(&g2, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  const size_t g = g1 > g2 ? g1 : g2;
  const size_t size = (bytes + g - 1) / g * g;
  mp.size = size;
  R->size = size;
  R->dev = dev_ord;
  CU(D.memCreate(&R->phys, size, &ap, 0));
  R->have_phys = true;
  const int t = rank % Gt, leader = rank - t;
  prctl(PR_SET_PTRACER, PR_SET_PTRACER_ANY, 0, 0, 0);  // let the peers duplicate our descriptors
  Handles mine;
  mine.pid = (int32_t)getpid();
  mine.phys_fd = mine.mc_fd = -1;
  int fd = -1;
  CU(D.exportHandle(&fd, R->phys, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  mine.phys_fd = fd;
  if (t == 0) {
    CU(D.mcCreate(&R->mc, &mp));
    R->have_mc = true;
    CU(D.exportHandle(&fd, R->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    mine.mc_fd = fd;
  }
  R->own_fds[0] = mine.phys_fd;
  R->own_fds[1] = mine.mc_fd;
  // every rank's handles, over the world communicator
  std::vector<Handles> all(world);
  {
    uint8_t* dbuf = nullptr;
    const size_t hb = sizeof(Handles);
    if (cudaMalloc(&dbuf, hb * world) != cudaSuccess) { *why = "cudaMalloc (handles)"; return MOE_ERR_CUDA; }
    cudaStream_t st = nullptr;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaError_t e = cudaMemcpy(dbuf + hb * rank, &mine, hb, cudaMemcpyHostToDevice);
    ncclResult_t r = e == cudaSuccess ? ncclAllGather(dbuf + hb * rank, dbuf, hb, ncclUint8, comm, st) : ncclSuccess;
    if (e == cudaSuccess && r == ncclSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess && r == ncclSuccess) e = cudaMemcpy(all.data(), dbuf, hb * world, cudaMemcpyDeviceToHost);
    cudaStreamDestroy(st);
    cudaFree(dbuf);
    if (r != ncclSuccess) { *why = std::string("ncclAllGather (handles): ") + ncclGetErrorString(r); return MOE_ERR_NCCL; }
    if (e != cudaSuccess) { *why = std::string("handle exchange: ") + cudaGetErrorString(e); return MOE_ERR_CUDA; }
  }
  // unicast mappings of every rank's region
  R->peer_uc.assign(world, nullptr);
  for (int q = 0; q < world; ++q) {
    CUmemGenericAllocationHandle h = R->phys;
    if (q != rank) {
      const int lfd = grab_fd(all[q].pid, all[q].phys_fd);
      if (lfd < 0) { *why = "pidfd_getfd of a peer's allocation handle failed"; return MOE_ERR_UNSUPPORTED; }
      const CUresult r = D.importHandle(&h, reinterpret_cast<void*>((intptr_t)lfd), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
      close(lfd);
      if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemImportFromShareableHandle (peer region)", why);
      R->imported.push_back(h);
    }
    moe_status s = map_rw(h, size, dev_ord, &R->peer_uc[q], why);
    if (s != MOE_OK) return s;
  }
  R->uc = R->peer_uc[rank];
  // the TP group's multicast object: every member adds its device, then binds its region
  if (t != 0) {
    const int lfd = grab_fd(all[leader].pid, all[leader].mc_fd);
    if (lfd < 0) { *why = "pidfd_getfd of the TP group's multicast handle failed"; return MOE_ERR_UNSUPPORTED; }
    const CUresult r = D.importHandle(&R->mc, reinterpret_cast<void*>((intptr_t)lfd), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(lfd);
    if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemImportFromShareableHandle (multicast)", why);
    R->have_mc = true;
  }
  CU(D.mcAddDevice(R->mc, dev));
  moe_status s = nccl_sync(comm, why);  // every import done: our exported descriptors can go
  if (s != MOE_OK) return s;
  for (int& f : R->own_fds)
    if (f >= 0) { close(f); f = -1; }
  CU(D.mcBindMem(R->mc, 0, R->phys, 0, size, 0));
  R->bound = true;
  s = nccl_sync(comm, why);
  if (s != MOE_OK) return s;
  s = map_rw(R->mc, size, dev_ord, &R->mcva, why);
  if (s != MOE_OK) return s;
  if (cudaMemset(R->uc, 0, size) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    *why = "cudaMemset (multicast region)";
    return MOE_ERR_CUDA;
  }
  return nccl_sync(comm, why);
}

void nvls_destroy(NvlsRegion* R) {
  Drv& D = drv();
  if (!D.ok) return;
  auto unmap = [&](void* va) {
    if (!va) return;
    const CUdeviceptr p = reinterpret_cast<CUdeviceptr>(va);
    D.unmap(p, R->size);
    D.addrFree(p, R->size);
  };
  unmap(R->mcva);
  for (void* p : R->peer_uc) unmap(p);
  if (R->bound) {
    CUdevice dev;
    if (D.deviceGet(&dev, R->dev) == CUDA_SUCCESS) D.mcUnbind(R->mc, dev, 0, R->size);
  }
  if (R->have_mc) D.memRelease(R->mc);
  for (CUmemGenericAllocationHandle h : R->imported) D.memRelease(h);
  if (R->have_phys) D.memRelease(R->phys);
  for (int f : R->own_fds)
    if (f >= 0) close(f);
  *R = NvlsRegion();
}

}  // namespace moe
