// nccl_rt.cu -- run-time binding of NCCL (see nccl_rt.hpp).
#include <dlfcn.h>
#include <link.h>

#include <mutex>

#include "nccl_rt.hpp"

namespace l1b {

namespace {

void* open_nccl(std::string& path) {
  // 1) the copy already in the process (torch's bundled libnccl.so.2)
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  // 2) the system library
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (h) {
    link_map* lm = nullptr;
    if (dlinfo(h, RTLD_DI_LINKMAP, &lm) == 0 && lm && lm->l_name) path = lm->l_name;
  }
  return h;
}

template <class F>
void bind(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  if (!out) throw NcclError(std::string("libnccl: missing symbol ") + name);
}

}  // namespace

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = open_nccl(api.path);
    if (!h) {
      err = std::string("libnccl.so.2 not loadable: ") + (dlerror() ? dlerror() : "?");
      return;
    }
    try {
      bind(h, "ncclGetVersion", api.GetVersion);
      bind(h, "ncclGetUniqueId", api.GetUniqueId);
      bind(h, "ncclCommInitRank", api.CommInitRank);
      bind(h, "ncclCommDestroy", api.CommDestroy);
      bind(h, "ncclAllReduce", api.AllReduce);
      bind(h, "ncclSend", api.Send);
      bind(h, "ncclRecv", api.Recv);
      bind(h, "ncclGroupStart", api.GroupStart);
      bind(h, "ncclGroupEnd", api.GroupEnd);
      bind(h, "ncclGetErrorString", api.GetErrorString);
      bind(h, "ncclCommGetAsyncError", api.CommGetAsyncError);
      api.GetVersion(&api.version);
    } catch (const std::exception& e) {
      err = e.what();
    }
  });
  if (!err.empty()) throw NcclError(err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const NcclApi& n = nccl();
  throw NcclError(std::string(what) + ": " + n.GetErrorString(r));
}

void nccl_check_async(ncclComm_t comm) {
  if (!comm) return;
  const NcclApi& n = nccl();
  ncclResult_t async = ncclSuccess;
  nccl_check(n.CommGetAsyncError(comm, &async), "ncclCommGetAsyncError");
  if (async != ncclSuccess && async != ncclInProgress)
    throw NcclError(std::string("NCCL communicator failed: ") + n.GetErrorString(async));
}

}  // namespace l1b
