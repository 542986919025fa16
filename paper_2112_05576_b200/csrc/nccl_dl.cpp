// nccl_dl.cpp -- run-time loading of NCCL (see nccl_dl.h).
#include "nccl_dl.h"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "failure.h"

namespace eab {

namespace {

template <class F>
void bind(void* h, const char* name, F& fn, std::string& missing) {
    fn = reinterpret_cast<F>(dlsym(h, name));
    if (!fn) missing += std::string(missing.empty() ? "" : ", ") + name;
}

}  // namespace

const NcclApi& nccl() {
    static NcclApi api{};
    static std::string error;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* env = std::getenv("EAB_NCCL_LIB");
        // an NCCL already mapped into the process (torch's) wins: a second,
        // different libnccl.so.2 would shadow it by soname
        void* h = (env && *env) ? nullptr : dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
        std::string tried;
        for (const char* n : names) {
            if (h) break;
            if (!n || !*n) continue;
            h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
            const char* e = dlerror();
            tried += std::string(tried.empty() ? "" : "; ") + n + ": " + (e ? e : "?");
        }
        if (!h) {
            error = "NCCL is not loadable (" + tried + ")";
            return;
        }
        std::string missing;
        bind(h, "ncclGetUniqueId", api.GetUniqueId, missing);
        bind(h, "ncclCommInitRank", api.CommInitRank, missing);
        bind(h, "ncclCommDestroy", api.CommDestroy, missing);
        bind(h, "ncclCommAbort", api.CommAbort, missing);
        bind(h, "ncclCommGetAsyncError", api.CommGetAsyncError, missing);
        bind(h, "ncclAllGather", api.AllGather, missing);
        bind(h, "ncclBroadcast", api.Broadcast, missing);
        bind(h, "ncclGroupStart", api.GroupStart, missing);
        bind(h, "ncclGroupEnd", api.GroupEnd, missing);
        bind(h, "ncclGetVersion", api.GetVersion, missing);
        bind(h, "ncclGetErrorString", api.GetErrorString, missing);
        if (!missing.empty()) {
            error = "NCCL library lacks " + missing;
            api = NcclApi{};
        }
    });
    if (!error.empty()) fail(EA_ERR_NCCL, error);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    const NcclApi& a = nccl();
    fail(EA_ERR_NCCL, std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "?"));
}

}  // namespace eab
