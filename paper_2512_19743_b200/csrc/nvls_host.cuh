// nvls_host.cuh -- host side of an NVLS team (k_nvls.cuh; declared in include/apml.h as
// apml_nvls_create / apml_nvls_destroy).  Included by apml_capi.cu only.
//
// Driver API through cudaGetDriverEntryPoint (no link-time dependency on libcuda):
//   rank 0: cuMulticastCreate (numDevices = world, POSIX file-descriptor handles), export the
//           handle as an fd and hand it to every other rank over an abstract Unix socket
//           (SCM_RIGHTS); the socket names carry a 64-bit rendezvous id that rank 0 broadcasts
//           with comm->allgather_bytes;
//   every rank: import (ranks > 0), cuMulticastAddDevice(its device), barrier, cuMemCreate a
//           buffer on its device, cuMulticastBindMem, map it twice -- unicast (own writes, flag
//           reads) and multicast (multimem red / ld_reduce) -- zero it, barrier.
#pragma once
#include <cuda.h>
#include <fcntl.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <cstdint>
#include <cstring>
#include <string>

struct apml_nvls {
  int rank = 0, world = 1;
  CUdevice dev = 0;
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  bool mc_ok = false, mem_ok = false, bound = false;
  CUdeviceptr uc = 0, mcva = 0;
  bool uc_mapped = false, mc_mapped = false;
  bool multicast = true;  // false: a one-device team in plain device memory (uc == mcva)
  size_t size = 0;
  uint32_t sig = 0;  // flag increments issued so far (the same count on every rank; modular)
  int use = 0;       // which partial-sum buffer the next reduction writes
  apml_comm comm{};
};

namespace {

struct NvlsDrv {
  CUresult (*deviceGet)(CUdevice*, int) = nullptr;
  CUresult (*deviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*mcGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                        unsigned long long) = nullptr;
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*exportHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) = nullptr;
  CUresult (*importHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*memGetGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*memSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  bool ok = false;
};

template <class F>
bool drv_fn(const char* name, F& f) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !p)
    return false;
  f = reinterpret_cast<F>(p);
  return true;
}

const NvlsDrv& nvls_drv() {
  static NvlsDrv d;
  static bool done = false;
  if (done) return d;
  done = true;
  d.ok = drv_fn("cuDeviceGet", d.deviceGet) && drv_fn("cuDeviceGetAttribute", d.deviceGetAttribute) &&
         drv_fn("cuMulticastGetGranularity", d.mcGetGranularity) && drv_fn("cuMulticastCreate", d.mcCreate) &&
         drv_fn("cuMulticastAddDevice", d.mcAddDevice) && drv_fn("cuMulticastBindMem", d.mcBindMem) &&
         drv_fn("cuMulticastUnbind", d.mcUnbind) && drv_fn("cuMemExportToShareableHandle", d.exportHandle) &&
         drv_fn("cuMemImportFromShareableHandle", d.importHandle) && drv_fn("cuMemCreate", d.memCreate) &&
         drv_fn("cuMemRelease", d.memRelease) && drv_fn("cuMemGetAllocationGranularity", d.memGetGranularity) &&
         drv_fn("cuMemAddressReserve", d.addrReserve) && drv_fn("cuMemAddressFree", d.addrFree) &&
         drv_fn("cuMemMap", d.memMap) && drv_fn("cuMemUnmap", d.memUnmap) &&
         drv_fn("cuMemSetAccess", d.memSetAccess);
  return d;
}

// ---- fd hand-over on one node: abstract Unix sockets, SCM_RIGHTS
std::string nvls_sock_name(uint64_t id, int rank) {
  char buf[64];
  snprintf(buf, sizeof buf, "apml-nvls-%016llx-%d", (unsigned long long)id, rank);
  return buf;
}
socklen_t nvls_addr(const std::string& name, sockaddr_un* a) {
  memset(a, 0, sizeof *a);
  a->sun_family = AF_UNIX;
  a->sun_path[0] = '\0';  // abstract namespace: nothing on the file system
  memcpy(a->sun_path + 1, name.data(), name.size());
  return (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + name.size());
}
bool nvls_send_fd(const std::string& name, int fd) {
  const int s = socket(AF_UNIX, SOCK_STREAM, 0);
  if (s < 0) return false;
  sockaddr_un a;
  const socklen_t al = nvls_addr(name, &a);
  bool ok = false;
  for (int tries = 0; tries < 2000 && !ok; ++tries) {  // the receiver listens before the barrier
    ok = connect(s, (sockaddr*)&a, al) == 0;
    if (!ok) usleep(1000);
  }
  if (ok) {
    char byte = 'x';
    iovec io{&byte, 1};
    char ctl[CMSG_SPACE(sizeof(int))];
    memset(ctl, 0, sizeof ctl);
    msghdr m{};
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    m.msg_control = ctl;
    m.msg_controllen = sizeof ctl;
    cmsghdr* c = CMSG_FIRSTHDR(&m);
    c->cmsg_level = SOL_SOCKET;
    c->cmsg_type = SCM_RIGHTS;
    c->cmsg_len = CMSG_LEN(sizeof(int));
    memcpy(CMSG_DATA(c), &fd, sizeof(int));
    ok = sendmsg(s, &m, 0) == 1;
  }
  close(s);
  return ok;
}
int nvls_recv_fd(int listener) {
  const int c = accept(listener, nullptr, nullptr);
  if (c < 0) return -1;
  char byte;
  iovec io{&byte, 1};
  char ctl[CMSG_SPACE(sizeof(int))];
  msghdr m{};
  m.msg_iov = &io;
  m.msg_iovlen = 1;
  m.msg_control = ctl;
  m.msg_controllen = sizeof ctl;
  int fd = -1;
  if (recvmsg(c, &m, 0) == 1) {
    cmsghdr* h = CMSG_FIRSTHDR(&m);
    if (h && h->cmsg_type == SCM_RIGHTS) memcpy(&fd, CMSG_DATA(h), sizeof(int));
  }
  close(c);
  return fd;
}

bool nvls_barrier(const apml_comm& c) {
  if (c.world == 1) return true;
  std::vector<char> r((size_t)c.world);
  const char x = 1;
  return c.allgather_bytes(&x, r.data(), 1, c.user) == 0;
}

void nvls_release(apml_nvls* t) {
  const NvlsDrv& d = nvls_drv();
  if (!t) return;
  if (!t->multicast) {
    if (t->uc) cudaFree(reinterpret_cast<void*>(t->uc));
    return;
  }
  if (!d.ok) return;
  if (t->mc_mapped) d.memUnmap(t->mcva, t->size);
  if (t->mcva) d.addrFree(t->mcva, t->size);
  if (t->uc_mapped) d.memUnmap(t->uc, t->size);
  if (t->uc) d.addrFree(t->uc, t->size);
  if (t->bound) d.mcUnbind(t->mc, t->dev, 0, t->size);
  if (t->mem_ok) d.memRelease(t->mem);
  if (t->mc_ok) d.memRelease(t->mc);
}

}  // namespace
