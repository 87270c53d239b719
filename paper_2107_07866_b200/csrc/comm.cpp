// comm.cpp -- NCCL for the z-slab halo exchanges, loaded at run time.
//
// The library does not link NCCL: a single-GPU user never needs it, and in a
// PyTorch process the libnccl.so.2 torch already mapped is the one dlopen
// returns (same soname), so both share one NCCL.  Only the entry points the
// slab exchange uses are resolved.
#include "cbx_comm.h"

#include <dlfcn.h>

#include <mutex>
#include <string>

#include "cbx_host.h"

namespace cbx {

namespace {
NcclApi g_api;
std::once_flag g_once;
std::string g_err;

template <class F>
bool sym(void* h, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(h, name));
  if (!f) g_err = std::string("libnccl: missing symbol ") + name;
  return f != nullptr;
}

void load() {
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* n : names)
    if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) {
    const char* e = dlerror();
    g_err = std::string("cannot load libnccl.so.2: ") + (e ? e : "");
    return;
  }
  NcclApi a;
  if (sym(h, "ncclGetUniqueId", a.get_unique_id) && sym(h, "ncclCommInitRank", a.comm_init_rank) &&
      sym(h, "ncclCommDestroy", a.comm_destroy) && sym(h, "ncclSend", a.send) &&
      sym(h, "ncclRecv", a.recv) && sym(h, "ncclAllReduce", a.all_reduce) &&
      sym(h, "ncclGroupStart", a.group_start) && sym(h, "ncclGroupEnd", a.group_end) &&
      sym(h, "ncclGetErrorString", a.error_string)) {
    a.ok = true;
    g_api = a;
  }
}
}  // namespace

const NcclApi& nccl() {
  std::call_once(g_once, load);
  if (!g_api.ok) raise(CBX_RUNTIME, g_err.empty() ? "NCCL unavailable" : g_err);
  return g_api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    raise(CBX_RUNTIME, std::string(what) + ": " + (g_api.error_string ? g_api.error_string(r) : "NCCL error"));
}

}  // namespace cbx
