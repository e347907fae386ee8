// ndgx_nccl.cpp -- run-time NCCL loader (see ndgx_nccl.h).
#include "ndgx_nccl.h"

#include <dlfcn.h>

#include <type_traits>

#include <mutex>

namespace ndgx {

const Nccl* nccl(std::string* why) {
  static Nccl lib;
  static std::string error;
  static bool ok = false;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      error = std::string("cannot load libnccl.so.2: ") + (e ? e : "unknown error");
      return;
    }
    bool all = true;
    auto get = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) {
        all = false;
        error = std::string("libnccl.so.2 lacks ") + name;
      }
    };
    get(lib.GetUniqueId, "ncclGetUniqueId");
    get(lib.CommInitRank, "ncclCommInitRank");
    get(lib.CommDestroy, "ncclCommDestroy");
    get(lib.CommAbort, "ncclCommAbort");
    get(lib.GroupStart, "ncclGroupStart");
    get(lib.GroupEnd, "ncclGroupEnd");
    get(lib.Send, "ncclSend");
    get(lib.Recv, "ncclRecv");
    get(lib.AllReduce, "ncclAllReduce");
    get(lib.GetErrorString, "ncclGetErrorString");
    ok = all;
  });
  if (!ok) {
    if (why) *why = error;
    return nullptr;
  }
  return &lib;
}

}  // namespace ndgx
