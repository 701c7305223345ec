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

// Per-(stream, purpose) workspace, zeroed when (re)allocated; kernels keep
// it in the state they need (GEMV: last contributors zero their words; EXPAND:
// the last CTA of a tile resets its tickets; LUT: partials are overwritten).
// Launches on one stream are ordered, so a workspace per stream keeps layers
// immutable without a per-launch allocation or memset.  Grown outside stream
// capture only: *out = NULL when `st` is capturing and the workspace is too
// small (callers fall back to a per-call workspace).
fasq_status stream_workspace(cudaStream_t st, int purpose, size_t bytes, void** out) {
    struct Ws { void* p = nullptr; size_t bytes = 0; };
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, Ws> ws_of[WS_KINDS];
    std::lock_guard<std::mutex> lk(mu);
    Ws& w = ws_of[purpose][st];
    *out = nullptr;
    if (w.bytes >= bytes) { *out = w.p; return FASQ_OK; }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs != cudaStreamCaptureStatusNone) return FASQ_OK;
    FASQ_CUDA_TRY(cudaStreamSynchronize(st));
    dev_free(w.p, st);
    w.p = nullptr;
    w.bytes = 0;
    const size_t nb = bytes > ((size_t)1 << 20) ? bytes : ((size_t)1 << 20);
    fasq_status s = dev_alloc(&w.p, nb, st);
    if (s != FASQ_OK) return s;
    FASQ_CUDA_TRY(cudaMemsetAsync(w.p, 0, nb, st));
    FASQ_CUDA_TRY(cudaStreamSynchronize(st));
    w.bytes = nb;
    *out = w.p;
    return FASQ_OK;
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
