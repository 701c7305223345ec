// alloc.cu -- device memory of the library behind one hook (fasq_set_allocator).
//
// north_star: "PyTorch is used only for device memory": every device buffer
// the library owns (layer storage, chain arenas and plans, KV caches, per-call
// split-K workspaces, pack scratch) is obtained through dev_alloc / released
// through dev_free, which call the caller's allocator when one is set (the
// Python binding can route them to torch's caching allocator,
// paper_2605_04084_b200.use_torch_allocator) and CUDA's stream-ordered
// allocator otherwise.  The one exception: a tensor-parallel chain arena
// (world > 1) is a plain cudaMalloc allocation, because cudaIpcGetMemHandle
// exports whole allocations (an allocator block inside a larger segment would
// open at the segment base on the peer).
//
// Every pointer remembers the allocator that produced it, so changing the
// hook never sends a pointer to the wrong free function.
#include <mutex>
#include <unordered_map>

#include "fasq_internal.cuh"

namespace fasq {
namespace {

struct Hook {
    fasq_alloc_fn alloc = nullptr;
    fasq_free_fn free = nullptr;
    void* ctx = nullptr;
};

std::mutex g_mu;
Hook g_hook;                                   // alloc == NULL: CUDA stream-ordered allocator
std::unordered_map<void*, Hook> g_owner;       // live pointers -> the hook that allocated them

}  // namespace

fasq_status dev_alloc(void** p, size_t bytes, cudaStream_t st) {
    *p = nullptr;
    if (bytes == 0) bytes = 16;
    Hook h;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        h = g_hook;
    }
    if (h.alloc) {
        void* q = h.alloc(h.ctx, bytes, (void*)st);
        if (!q) {
            set_error("caller allocator returned NULL for " + std::to_string(bytes) + " bytes");
            return FASQ_E_OOM;
        }
        if (reinterpret_cast<uintptr_t>(q) % 256) {
            h.free(h.ctx, q, (void*)st);
            set_error("caller allocator returned a pointer that is not 256-B aligned");
            return FASQ_E_ARG;
        }
        *p = q;
    } else {
        cudaError_t e = cudaMallocAsync(p, bytes, st);
        if (e != cudaSuccess) {
            cudaGetLastError();
            *p = nullptr;
            return FASQ_E_OOM;
        }
    }
    std::lock_guard<std::mutex> lk(g_mu);
    g_owner[*p] = h;
    return FASQ_OK;
}

void dev_free(void* p, cudaStream_t st) {
    if (!p) return;
    Hook h;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_owner.find(p);
        if (it == g_owner.end()) return;   // not ours (never happens for library pointers)
        h = it->second;
        g_owner.erase(it);
    }
    if (h.free) h.free(h.ctx, p, (void*)st);
    else cudaFreeAsync(p, st);
}

}  // namespace fasq

using namespace fasq;

extern "C" {

fasq_status fasq_set_allocator(fasq_alloc_fn alloc, fasq_free_fn free_fn, void* ctx) {
    if ((alloc == nullptr) != (free_fn == nullptr)) return FASQ_E_ARG;
    std::lock_guard<std::mutex> lk(g_mu);
    g_hook.alloc = alloc;
    g_hook.free = free_fn;
    g_hook.ctx = ctx;
    return FASQ_OK;
}

}  // extern "C"
