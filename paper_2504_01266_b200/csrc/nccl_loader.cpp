#include "nccl_loader.h"

#include <dlfcn.h>

#include <mutex>

namespace giga {

static NcclApi g_api;
static const char *g_why = nullptr;
static bool g_ok = false;
static std::once_flag g_once;

#ifndef GIGA_NCCL_PATH
#define GIGA_NCCL_PATH ""
#endif

template <class F>
static bool sym(void *h, const char *name, F &out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  return out != nullptr;
}

const NcclApi *nccl_api(const char **why) {
  std::call_once(g_once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h && GIGA_NCCL_PATH[0]) h = dlopen(GIGA_NCCL_PATH, RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      g_why = "cannot dlopen libnccl.so.2";
      return;
    }
    bool ok = sym(h, "ncclGetUniqueId", g_api.GetUniqueId) &&
              sym(h, "ncclCommInitRank", g_api.CommInitRank) &&
              sym(h, "ncclCommInitAll", g_api.CommInitAll) &&
              sym(h, "ncclCommInitRankConfig", g_api.CommInitRankConfig) &&
              sym(h, "ncclCommDestroy", g_api.CommDestroy) &&
              sym(h, "ncclCommGetAsyncError", g_api.CommGetAsyncError) &&
              sym(h, "ncclBroadcast", g_api.Broadcast) &&
              sym(h, "ncclAllGather", g_api.AllGather) &&
              sym(h, "ncclAllReduce", g_api.AllReduce) &&
              sym(h, "ncclGroupStart", g_api.GroupStart) &&
              sym(h, "ncclGroupEnd", g_api.GroupEnd) &&
              sym(h, "ncclGetErrorString", g_api.GetErrorString);
    if (!ok) {
      g_why = "libnccl.so.2 lacks a required symbol";
      return;
    }
    g_ok = true;
  });
  if (why) *why = g_why;
  return g_ok ? &g_api : nullptr;
}

}  // namespace giga
