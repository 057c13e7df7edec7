// mcast.cpp -- NVLink multicast teams for the fused epilogue gather.
//
// The gather of C is a concatenation of the row blocks (S4.2.3 "concatenated";
// PAPER.md:291, S4.2.7): every GPU must end with every GPU's rows. With the unicast fused
// gather (p2p.cpp) the last K-chunk's epilogue stores each C tile into its own C_full and then
// once more per peer, so a GPU's NVLink egress is (g - 1) x its rows. Bound into one multicast
// team, the GPUs' C_full buffers share a multicast address: one multimem.st per 16 bytes
// leaves the GPU once and the NVSwitch writes it into every member's copy (this GPU's
// included), so the egress is 1 x its rows whatever g is.
//
// A team is made with the driver's VMM calls: a multicast object for g devices
// (cuMulticastCreate), every device added (cuMulticastAddDevice), then on each device a
// physical allocation (cuMemCreate) mapped at the address the caller uses as C_full and bound
// to the object (cuMulticastBindMem), and the object itself mapped at the multicast address
// the epilogue writes to. Two forms:
//   * single process over g distinct devices: giga_mc_alloc / giga_mc_free;
//   * one process per GPU (rank API): rank 0 creates the object and exports it as a POSIX file
//     descriptor, the others import it through pidfd_getfd (giga_rank_mc_create / _join /
//     _bind, orchestrated by the binding over torch.distributed).
// Drivers without multicast (no NVSwitch, no fabric manager / IMEX channel -- e.g. the 1-GPU
// pool this was built on, profiles/r02_nvls_probe.jsonl) refuse cuMulticastCreate: the calls
// return GIGA_ERR_UNSUPPORTED and callers keep ordinary C_full buffers (unicast gather).
#include "runtime.h"

#include <stdio.h>
#include <string.h>
#include <sys/syscall.h>
#include <type_traits>
#include <unistd.h>

namespace giga {

namespace {

struct McDrv {
  decltype(&cuDeviceGet) deviceGet = nullptr;
  decltype(&cuDeviceGetAttribute) attr = nullptr;
  decltype(&cuMulticastCreate) mcCreate = nullptr;
  decltype(&cuMulticastAddDevice) mcAdd = nullptr;
  decltype(&cuMulticastBindMem) mcBind = nullptr;
  decltype(&cuMulticastUnbind) mcUnbind = nullptr;
  decltype(&cuMulticastGetGranularity) mcGran = nullptr;
  decltype(&cuMemCreate) memCreate = nullptr;
  decltype(&cuMemRelease) memRelease = nullptr;
  decltype(&cuMemAddressReserve) vaReserve = nullptr;
  decltype(&cuMemAddressFree) vaFree = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) setAccess = nullptr;
  decltype(&cuMemGetAllocationGranularity) allocGran = nullptr;
  decltype(&cuMemExportToShareableHandle) exportH = nullptr;
  decltype(&cuMemImportFromShareableHandle) importH = nullptr;
  decltype(&cuGetErrorString) errStr = nullptr;
};

const McDrv *mc_drv() {
  static McDrv d;
  static std::once_flag once;
  static bool ok = false;
  std::call_once(once, [] {
    bool all = true;
    auto get = [&all](const char *name, auto &fn) {
      void *p = nullptr;
      cudaDriverEntryPointQueryResult q{};
      if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p)
        all = false;
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
    };
    get("cuDeviceGet", d.deviceGet);
    get("cuDeviceGetAttribute", d.attr);
    get("cuMulticastCreate", d.mcCreate);
    get("cuMulticastAddDevice", d.mcAdd);
    get("cuMulticastBindMem", d.mcBind);
    get("cuMulticastUnbind", d.mcUnbind);
    get("cuMulticastGetGranularity", d.mcGran);
    get("cuMemCreate", d.memCreate);
    get("cuMemRelease", d.memRelease);
    get("cuMemAddressReserve", d.vaReserve);
    get("cuMemAddressFree", d.vaFree);
    get("cuMemMap", d.map);
    get("cuMemUnmap", d.unmap);
    get("cuMemSetAccess", d.setAccess);
    get("cuMemGetAllocationGranularity", d.allocGran);
    get("cuMemExportToShareableHandle", d.exportH);
    get("cuMemImportFromShareableHandle", d.importH);
    get("cuGetErrorString", d.errStr);
    cudaGetLastError();
    ok = all;
  });
  return ok ? &d : nullptr;
}

int fail_cu(CUresult r, const char *what) {
  const McDrv *d = mc_drv();
  const char *s = nullptr;
  if (d) d->errStr(r, &s);
  return fail(r == CUDA_ERROR_OUT_OF_MEMORY ? GIGA_ERR_OOM : GIGA_ERR_CUDA, "%s: %s", what,
              s ? s : "?");
}

#define CU(x)                                      \
  do {                                             \
    CUresult r_ = (x);                             \
    if (r_ != CUDA_SUCCESS) return fail_cu(r_, #x); \
  } while (0)

// One GPU's side of a team: its physical memory mapped at va (what the caller uses as C_full)
// and the multicast object mapped at mcva.
struct McMember {
  int dev = -1;
  CUmemGenericAllocationHandle phys = 0;
  CUdeviceptr va = 0, mcva = 0;
};

struct McTeam {
  CUmemGenericAllocationHandle mc = 0;
  size_t size = 0;
  std::vector<McMember> m;  // single process: one per GPU (one mcva for all); rank: this rank
};

std::vector<McTeam> g_teams;  // single-process teams (giga_mc_alloc)
McTeam g_rank_team;           // rank mode: this process's team (giga_rank_mc_*)
int g_rank_fd = -1;           // rank 0: the exported descriptor (kept open until finalize)

// Sizes are rounded to the multicast granularity (and the allocation granularity).
int team_size(const McDrv *d, int ndev, int dev0, size_t bytes, size_t *out) {
  CUmulticastObjectProp mp{};
  mp.numDevices = unsigned(ndev);
  mp.size = bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
  size_t gmc = 0, gal = 0;
  CU(d->mcGran(&gmc, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev0;
  CU(d->allocGran(&gal, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  const size_t gr = std::max(gmc, gal);
  *out = (bytes + gr - 1) / gr * gr;
  return GIGA_OK;
}

int check_multicast_device(const McDrv *d, int dev) {
  CUdevice cd;
  CU(d->deviceGet(&cd, dev));
  int sup = 0;
  CU(d->attr(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd));
  if (!sup) return fail(GIGA_ERR_UNSUPPORTED, "device %d: no NVLink multicast support", dev);
  return GIGA_OK;
}

int create_object(const McDrv *d, int ndev, size_t size, CUmemAllocationHandleType ht,
                  CUmemGenericAllocationHandle *mc) {
  CUmulticastObjectProp mp{};
  mp.numDevices = unsigned(ndev);
  mp.size = size;
  mp.handleTypes = ht;
  const CUresult r = d->mcCreate(mc, &mp);
  if (r != CUDA_SUCCESS) {
    const char *s = nullptr;
    d->errStr(r, &s);
    return fail(GIGA_ERR_UNSUPPORTED,
                "cuMulticastCreate refused (%s): no NVSwitch multicast on this system -- keep "
                "ordinary C_full buffers (unicast gather)",
                s ? s : "?");
  }
  return GIGA_OK;
}

// Device memory for `dev`, mapped (read / write for dev) and bound to the team's object.
int bind_member(const McDrv *d, McTeam &t, McMember &mm) {
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = mm.dev;
  CU(d->memCreate(&mm.phys, t.size, &ap, 0));
  CU(d->vaReserve(&mm.va, t.size, 0, 0, 0));
  CU(d->map(mm.va, t.size, 0, mm.phys, 0));
  CUmemAccessDesc ad{};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = mm.dev;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU(d->setAccess(mm.va, t.size, &ad, 1));
  CU(d->mcBind(t.mc, 0, mm.phys, 0, t.size, 0));
  return GIGA_OK;
}

// The multicast object mapped at a fresh address, accessible from `devs`.
int map_object(const McDrv *d, McTeam &t, const std::vector<int> &devs, CUdeviceptr *mcva) {
  CU(d->vaReserve(mcva, t.size, 0, 0, 0));
  CU(d->map(*mcva, t.size, 0, t.mc, 0));
  std::vector<CUmemAccessDesc> ads(devs.size());
  for (size_t i = 0; i < devs.size(); ++i) {
    ads[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ads[i].location.id = devs[i];
    ads[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  CU(d->setAccess(*mcva, t.size, ads.data(), ads.size()));
  return GIGA_OK;
}

// Best-effort teardown of whatever part of a team exists (error paths and free).
void release_team(McTeam &t) {
  const McDrv *d = mc_drv();
  if (!d) return;
  for (auto &mm : t.m)
    if (mm.dev >= 0) cudaSetDevice(mm.dev), cudaDeviceSynchronize();
  CUdeviceptr mapped = 0;
  for (auto &mm : t.m) {
    if (mm.mcva && mm.mcva != mapped) {
      d->unmap(mm.mcva, t.size);
      d->vaFree(mm.mcva, t.size);
      mapped = mm.mcva;
    }
    if (t.mc && mm.phys) {
      CUdevice cd;
      if (d->deviceGet(&cd, mm.dev) == CUDA_SUCCESS) d->mcUnbind(t.mc, cd, 0, t.size);
    }
    if (mm.va) {
      d->unmap(mm.va, t.size);
      d->vaFree(mm.va, t.size);
    }
    if (mm.phys) d->memRelease(mm.phys);
  }
  if (t.mc) d->memRelease(t.mc);
  t = McTeam{};
  cudaGetLastError();
}

int alloc_team_locked(int ngpus, size_t bytes, float **C_full) {
  const McDrv *d = mc_drv();
  if (!d) return fail(GIGA_ERR_UNSUPPORTED, "driver multicast / VMM entry points unavailable");
  std::vector<int> devs;
  for (int i = 0; i < ngpus; ++i) {
    const int dev = g.devs[i].dev;
    for (int j : devs)
      if (j == dev)
        return fail(GIGA_ERR_INVALID_ARG,
                    "giga_mc_alloc: library GPUs %d share device %d (multicast needs distinct "
                    "devices)",
                    i, dev);
    devs.push_back(dev);
    TRY(check_multicast_device(d, dev));
  }
  McTeam t;
  TRY(team_size(d, ngpus, devs[0], bytes, &t.size));
  CK(cudaSetDevice(devs[0]));
  TRY(create_object(d, ngpus, t.size, CU_MEM_HANDLE_TYPE_NONE, &t.mc));
  int rc = GIGA_OK;
  for (int dev : devs) {  // every device joins before any memory is bound
    CUdevice cd;
    if (rc == GIGA_OK && d->deviceGet(&cd, dev) != CUDA_SUCCESS)
      rc = fail(GIGA_ERR_CUDA, "cuDeviceGet(%d)", dev);
    if (rc == GIGA_OK) {
      const CUresult r = d->mcAdd(t.mc, cd);
      if (r != CUDA_SUCCESS) rc = fail_cu(r, "cuMulticastAddDevice");
    }
  }
  for (int dev : devs) {
    if (rc != GIGA_OK) break;
    t.m.push_back(McMember{});
    t.m.back().dev = dev;
    cudaSetDevice(dev);
    rc = bind_member(d, t, t.m.back());
  }
  CUdeviceptr mcva = 0;
  if (rc == GIGA_OK) rc = map_object(d, t, devs, &mcva);
  if (rc != GIGA_OK) {
    if (mcva) t.m.push_back(McMember{-1, 0, 0, mcva});
    release_team(t);
    return rc;
  }
  for (auto &mm : t.m) mm.mcva = mcva;
  for (int i = 0; i < ngpus; ++i) {
    cudaSetDevice(devs[i]);
    CK(cudaMemset(reinterpret_cast<void *>(t.m[i].va), 0, t.size));
    C_full[i] = reinterpret_cast<float *>(t.m[i].va);
  }
  g_teams.push_back(std::move(t));
  return GIGA_OK;
}

}  // namespace

// The multicast address of the team whose members' C_full are exactly parts[i].C (library
// GPU i in order) and hold M x N floats, else nullptr (ordinary buffers: unicast gather).
float *mc_address(const std::vector<Part> &parts, int64_t M, int64_t N) {
  for (const McTeam &t : g_teams) {
    if (t.m.size() != parts.size() || size_t(M) * size_t(N) * 4 > t.size) continue;
    bool same = true;
    for (size_t i = 0; i < parts.size() && same; ++i)
      same = reinterpret_cast<CUdeviceptr>(parts[i].C) == t.m[i].va &&
             parts[i].d->dev == t.m[i].dev;
    if (same) return reinterpret_cast<float *>(t.m[0].mcva);
  }
  return nullptr;
}

// Rank mode: the multicast address when C_full is this rank's team buffer (M x N fits).
float *rank_mc_address(const float *C_full, int64_t M, int64_t N) {
  const McTeam &t = g_rank_team;
  if (t.m.empty() || !t.m[0].mcva || size_t(M) * size_t(N) * 4 > t.size) return nullptr;
  return reinterpret_cast<CUdeviceptr>(C_full) == t.m[0].va
             ? reinterpret_cast<float *>(t.m[0].mcva)
             : nullptr;
}

bool rank_mc_buffer(const float *p) {
  return !g_rank_team.m.empty() && reinterpret_cast<CUdeviceptr>(p) == g_rank_team.m[0].va;
}

void mc_release_all() {
  for (auto &t : g_teams) release_team(t);
  g_teams.clear();
  release_team(g_rank_team);
  if (g_rank_fd >= 0) close(g_rank_fd);
  g_rank_fd = -1;
}

// ---- rank mode: one process per GPU ------------------------------------------------------
// Blob (GIGA_MC_BLOB_BYTES): magic, the exporting process id, its descriptor, the size.
struct McBlob {
  uint64_t magic;
  int64_t pid;
  int64_t fd;
  uint64_t size;
};
constexpr uint64_t kMcMagic = 0x676967616d63ull;  // "gigamc"

int rank_mc_create_locked(size_t bytes, uint8_t *blob) {
  const McDrv *d = mc_drv();
  if (!d) return fail(GIGA_ERR_UNSUPPORTED, "driver multicast / VMM entry points unavailable");
  if (g.rank != 0) return fail(GIGA_ERR_INVALID_ARG, "giga_rank_mc_create: rank 0 only");
  if (!g_rank_team.m.empty() || g_rank_team.mc)
    return fail(GIGA_ERR_ALREADY_INITIALIZED, "giga_rank_mc_create: this rank has a team");
  const int dev = g.devs[0].dev;
  TRY(check_multicast_device(d, dev));
  McTeam &t = g_rank_team;
  TRY(team_size(d, g.world, dev, bytes, &t.size));
  CK(cudaSetDevice(dev));
  int rc = create_object(d, g.world, t.size, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, &t.mc);
  int fd = -1;
  if (rc == GIGA_OK) {
    const CUresult r = d->exportH(&fd, t.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (r != CUDA_SUCCESS) rc = fail_cu(r, "cuMemExportToShareableHandle");
  }
  if (rc != GIGA_OK) {
    release_team(t);
    return rc;
  }
  g_rank_fd = fd;
  McBlob b{kMcMagic, int64_t(getpid()), int64_t(fd), uint64_t(t.size)};
  memset(blob, 0, GIGA_MC_BLOB_BYTES);
  memcpy(blob, &b, sizeof b);
  return GIGA_OK;
}

int rank_mc_join_locked(const uint8_t *blob) {
  const McDrv *d = mc_drv();
  if (!d) return fail(GIGA_ERR_UNSUPPORTED, "driver multicast / VMM entry points unavailable");
  McBlob b;
  memcpy(&b, blob, sizeof b);
  if (b.magic != kMcMagic) return fail(GIGA_ERR_INVALID_ARG, "giga_rank_mc_join: bad blob");
  McTeam &t = g_rank_team;
  const int dev = g.devs[0].dev;
  CK(cudaSetDevice(dev));
  if (g.rank != 0) {
    if (t.mc) return fail(GIGA_ERR_ALREADY_INITIALIZED, "giga_rank_mc_join: joined already");
    TRY(check_multicast_device(d, dev));
    // the exporter's descriptor, duplicated into this process (Linux >= 5.6)
    const int pfd = int(syscall(SYS_pidfd_open, pid_t(b.pid), 0));
    if (pfd < 0) return fail(GIGA_ERR_UNSUPPORTED, "pidfd_open(%lld) failed", (long long)b.pid);
    const int fd = int(syscall(SYS_pidfd_getfd, pfd, int(b.fd), 0));
    close(pfd);
    if (fd < 0) return fail(GIGA_ERR_UNSUPPORTED, "pidfd_getfd failed (ptrace permission?)");
    const CUresult r = d->importH(&t.mc, reinterpret_cast<void *>(intptr_t(fd)),
                                  CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(fd);
    if (r != CUDA_SUCCESS) return fail_cu(r, "cuMemImportFromShareableHandle");
    t.size = size_t(b.size);
  }
  CUdevice cd;
  CU(d->deviceGet(&cd, dev));
  CU(d->mcAdd(t.mc, cd));
  return GIGA_OK;
}

int rank_mc_bind_locked(float **C_full) {
  const McDrv *d = mc_drv();
  McTeam &t = g_rank_team;
  if (!d || !t.mc || !t.m.empty())
    return fail(GIGA_ERR_NOT_INITIALIZED, "giga_rank_mc_bind: join the team first (once)");
  const int dev = g.devs[0].dev;
  CK(cudaSetDevice(dev));
  t.m.push_back(McMember{});
  t.m[0].dev = dev;
  int rc = bind_member(d, t, t.m[0]);
  if (rc == GIGA_OK) rc = map_object(d, t, {dev}, &t.m[0].mcva);
  if (rc == GIGA_OK) {
    const cudaError_t e = cudaMemset(reinterpret_cast<void *>(t.m[0].va), 0, t.size);
    if (e != cudaSuccess) rc = fail_cuda(e, "cudaMemset", __FILE__, __LINE__);
  }
  if (rc != GIGA_OK) {
    release_team(t);
    return rc;
  }
  *C_full = reinterpret_cast<float *>(t.m[0].va);
  return GIGA_OK;
}

}  // namespace giga

using namespace giga;

extern "C" {

int giga_mc_alloc(int ngpus, size_t bytes, float **C_full) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 1) return fail(GIGA_ERR_NOT_INITIALIZED, "giga_mc_alloc: call giga_init first");
  if (!C_full || bytes == 0 || ngpus < 1 || ngpus > int(g.devs.size()) || ngpus > kMaxCDst)
    return fail(GIGA_ERR_INVALID_ARG, "giga_mc_alloc: bad arguments");
  return alloc_team_locked(ngpus, bytes, C_full);
}

int giga_mc_free(float *C_full0) {
  std::lock_guard<std::mutex> lk(g.mu);
  for (size_t i = 0; i < g_teams.size(); ++i)
    if (!g_teams[i].m.empty() && g_teams[i].m[0].va == reinterpret_cast<CUdeviceptr>(C_full0)) {
      release_team(g_teams[i]);
      g_teams.erase(g_teams.begin() + long(i));
      return GIGA_OK;
    }
  return fail(GIGA_ERR_INVALID_ARG, "giga_mc_free: not a giga_mc_alloc buffer");
}

int giga_rank_mc_create(size_t bytes, uint8_t *blob) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 2) return fail(GIGA_ERR_NOT_INITIALIZED, "giga_rank_mc_create: rank mode only");
  if (!blob || bytes == 0) return fail(GIGA_ERR_INVALID_ARG, "giga_rank_mc_create: bad args");
  return rank_mc_create_locked(bytes, blob);
}

int giga_rank_mc_join(const uint8_t *blob) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 2) return fail(GIGA_ERR_NOT_INITIALIZED, "giga_rank_mc_join: rank mode only");
  if (!blob) return fail(GIGA_ERR_INVALID_ARG, "giga_rank_mc_join: NULL blob");
  return rank_mc_join_locked(blob);
}

int giga_rank_mc_bind(float **C_full) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 2) return fail(GIGA_ERR_NOT_INITIALIZED, "giga_rank_mc_bind: rank mode only");
  if (!C_full) return fail(GIGA_ERR_INVALID_ARG, "giga_rank_mc_bind: NULL");
  return rank_mc_bind_locked(C_full);
}

}  // extern "C"
