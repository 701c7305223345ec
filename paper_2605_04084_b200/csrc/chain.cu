// chain.cu -- persistent decode-chain executor (sm_100a).
//
// A decode token runs the PQ linear layers of a model as a chain of grouped
// GEMVs (q/k/v, o, gate/up, down per block; every layer packed separately,
// P:219).  Launching one kernel per step pays, per step, a launch, the first
// stage's memory latency and a grid-wide completion before the next step may
// read its x.  This executor runs the whole chain in ONE persistent kernel
// (one CTA per SM, cooperative launch):
//
//  * the per-step work (row tile x K-range of groups, same tiling as gemv.cu)
//    is planned once on the host into a [steps][CTAs] table of work items;
//  * the producer warp of every CTA streams the codebook/index stages of ALL
//    its steps back to back through the SMEM ring -- weights do not depend on
//    x, so the ring keeps filling while the consumers wait for the previous
//    step (no pipeline drain at step boundaries);
//  * there is NO grid-wide barrier between steps: every output element is a
//    "counted accumulator" (gemv_core.cuh): an int64 red.add target that
//    carries the fixed-point sum (units 2^-32, exact and order-independent
//    -> deterministic) AND the number of K-split contributions; a consumer
//    polls exactly the words of its K range until each shows count == ks of
//    the producing layer, then rounds them to fp16 x (as FASQ_FLAG_X_ACC).
//    One L2 round trip after the data is final instead of a barrier round
//    trip plus a load round trip.
//
// Numerics are identical to chaining fasq_gemv_grouped calls with FASQ_ACC_I64
// outputs (same fixed-point units and rounding).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "fasq_internal.cuh"
#include "gemv_core.cuh"

struct fasq_chain {
    int n_steps = 0, B = 0, d = 0, nctas = 0;
    int world = 1, rank = 0;                         // row-sharded tensor parallelism (fasq_chain_create_tp)
    int rw = 0, nw = 0, st = 0, R = 0, gmax = 1, maxC = 1, mi = 1;
    size_t smem = 0;
    std::vector<std::vector<int64_t>> acc_off;       // per step, per layer: word offset in one arena buffer
    std::vector<std::vector<int64_t>> acc_Fout;      // per step, per layer: GLOBAL F_out (words per batch row)
    std::vector<std::vector<int>> acc_ks;            // per step, per layer: K-split count (contributions per word)
    std::vector<int> step_F_in;
    int ext_F_in = 0;
    // two arena buffers (ONE allocation, IPC-exportable): run n accumulates into
    // buffer parity(n) on every rank and zeroes its own buffer parity(n)^1 for
    // run n+1 -- no memset node, no host round trip between tokens
    unsigned long long* arenas = nullptr;
    int64_t arena_words = 0;                         // words per buffer
    unsigned* ctrl = nullptr;                        // device: [0] parity, [1] unused, [2] monotonic CTA entry counter
    unsigned long long** peers_dev = nullptr;        // device [world]: every rank's `arenas` (own rank = local)
    std::vector<void*> ipc_opened;                   // peer mappings opened by fasq_chain_set_peers
    bool peers_ready = true;
    void* items = nullptr;                           // device [n_steps][nctas] ChainItem
    void* phases = nullptr;                          // device [n_steps] ChainPhase
    unsigned long long* trace = nullptr;             // user buffer (fasq_chain_trace), not owned
};

namespace fasq {

namespace {

struct ChainItem {
    const uint8_t* idx;
    const uint8_t* cbimg;
    const void* cbmap;          // d <= 2: 3-D tensor map {32 words, n_groups, C} over cbimg (pair boxes)
    long long y_off;            // word offset of the layer's counted-accumulator output [B][F_out_g] in a buffer
    int F_out, F_out_g, row0_g; // local rows of this rank's shard, global F_out, global row of local row 0
    int F_out_pad, N_ss, C;
    int r0, rows_valid, g_begin, g_end;
};

struct ChainPhase {
    long long x_off;            // word offset of the counted-accumulator input (< 0: the external fp16 x)
    int F_in, x_ks;             // x_ks: contributions per input word (K-split of the producer)
};

struct ChainParams {
    const ChainItem* items;
    const ChainPhase* phases;
    const __half* x_ext;        // [B][F_in of the first step]
    unsigned long long* trace;  // optional [n_steps][nctas][4] globaltimer stamps (fasq_chain_trace)
    unsigned* ctrl;             // [0] parity, [2] CTA entry counter
    unsigned long long* const* peers;   // [world] arena bases (2 buffers each); peers[rank] = local
    long long arena_words;      // words per buffer
    int world, rank;
    int n_steps, nctas, B, gmax, cbb_max;
    int mi;                     // work items per (step, CTA): [n_steps][nctas][mi]
    int pf;                     // producer: L2-prefetch this many groups of the next step's item
    int backoff;                // ns slept between input polls (FASQ_CHAIN_BACKOFF, default 0)
    int dbg;                    // experiments only (FASQ_CHAIN_DBG): bit 0 = consumers skip the gather
                                // loop, bit 1 = producer skips the copies (compute on stale SMEM),
                                // bit 2 = producer skips the codebook copies only
};

// d <= 2 (4-B codebook entries) runs on codebook PAIR stages: a separate
// CS-deep ring of [C][2][32]-word slots, each filled by ONE 3-D TMA box that
// interleaves groups g and g+1 of the [group][C][32] image into 256-B k-rows
// (core::compute_group_pair: the gather address is one PRMT).  The index
// chunks keep their own ST-deep ring (one group per stage).
template <int D>
struct ChainPair {
    static constexpr bool value = D <= 2;
};
constexpr int kChainCS = kPairSlots;

template <int D, int NB, int NW, int ST>
__global__ void __launch_bounds__((NW + 1) * 32, 1) k_chain(ChainParams p) {
    constexpr int E = core::Entry<D>::value;
    constexpr bool PAIR = ChainPair<D>::value;
    // d <= 2: row-set mapping, 64 rows per warp at any B (gemv_core.cuh)
    constexpr int RW = PAIR ? 64 : core::RowsPerWarp<NB>::value;
    constexpr int R = RW * NW;
    constexpr int G = NB <= 2 ? 8 : NB == 4 ? 4 : 2;   // lanes per row set (<= 32 accumulators)
    constexpr bool XF = PAIR && NB == 8;               // x staged as fp32 (FFMA2 path, compute_group_set)
    constexpr int XG = XF ? 32 * NB * D * 4 : 32 * NB * E;
    constexpr int CS = kChainCS;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* s_cb = smem;                                       // PAIR: CS * 64 KiB, else ST * cbb_max
    uint8_t* s_idx = s_cb + (PAIR ? CS * kPairSlot : ST * p.cbb_max);   // ST * R * 32
    uint8_t* s_x = s_idx + ST * R * 32;                         // gmax * XG
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_x + p.gmax * XG);
    const uint32_t cb_u = dev::smem_u32(s_cb), idx_u = dev::smem_u32(s_idx), x_u = dev::smem_u32(s_x);
    const uint32_t full0 = dev::smem_u32(&bars[0]), empty0 = dev::smem_u32(&bars[ST]);
    const uint32_t cfull0 = dev::smem_u32(&bars[2 * ST]), cempty0 = dev::smem_u32(&bars[2 * ST + CS]);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < ST; ++s) {
            dev::mbar_init(full0 + 8 * s, 1);
            dev::mbar_init(empty0 + 8 * s, NW);
        }
        if (PAIR) {
#pragma unroll
            for (int s = 0; s < CS; ++s) {
                dev::mbar_init(cfull0 + 8 * s, 1);
                dev::mbar_init(cempty0 + 8 * s, NW);
            }
        }
        dev::fence_barrier_init();
    }
    __syncthreads();

    if (warp == NW) {
        // producer: every step's stages, back to back (no dependence on x)
        if (lane == 0) {
            int it = 0, cit = 0;
            for (int phj = 0; phj < p.n_steps * p.mi; ++phj) {
                const int ph = phj / p.mi;
                const ChainItem& w = p.items[((size_t)ph * p.nctas + blockIdx.x) * p.mi + phj % p.mi];
                if (w.rows_valid <= 0) continue;
                const uint32_t cbb = (uint32_t)w.C * 32u * E;
                const uint32_t chunk = (uint32_t)w.rows_valid * 32u;
                if (p.pf > 0 && ph + 1 < p.n_steps && phj % p.mi == 0) {
                    // warm L2 with the head of the next step's first item
                    const ChainItem& nw = p.items[((size_t)(ph + 1) * p.nctas + blockIdx.x) * p.mi];
                    if (nw.rows_valid > 0) {
                        const int ge = min(nw.g_end, nw.g_begin + p.pf);
                        for (int g = nw.g_begin; g < ge; ++g)
                            dev::bulk_prefetch_l2(nw.idx + ((size_t)g * nw.F_out_pad + nw.r0) * 32,
                                                  (uint32_t)nw.rows_valid * 32u);
                    }
                }
                for (int g = w.g_begin; g < w.g_end; ++g, ++it) {
                    if (PAIR && ((g - w.g_begin) & 1) == 0) {
                        // groups g, g+1 -> one pair slot (g+1 past the layer: zero fill)
                        const int cs = cit % CS;
                        if (cit >= CS) dev::mbar_wait(cempty0 + 8 * cs, ((cit / CS) + 1) & 1);
                        if (p.dbg & 6) {   // bit 2: codebook copies only skipped (stale SMEM codebooks)
                            dev::mbar_arrive(cfull0 + 8 * cs);
                        } else {
                            dev::mbar_arrive_expect_tx(cfull0 + 8 * cs, 2u * cbb);
                            dev::tma_load_3d(cb_u + (uint32_t)cs * kPairSlot, w.cbmap, 0, g, 0, cfull0 + 8 * cs);
                        }
                        ++cit;
                    }
                    const int slot = it % ST;
                    if (it >= ST) dev::mbar_wait(empty0 + 8 * slot, ((it / ST) + 1) & 1);
                    const uint32_t full = full0 + 8 * slot;
                    if (p.dbg & 2) { dev::mbar_arrive(full); continue; }
                    dev::mbar_arrive_expect_tx(full, PAIR ? chunk : chunk + cbb);
                    if (!PAIR)
                        dev::bulk_g2s(cb_u + (uint32_t)slot * (uint32_t)p.cbb_max, w.cbimg + (size_t)g * cbb, cbb,
                                      full);
                    dev::bulk_g2s(idx_u + (uint32_t)slot * R * 32u, w.idx + ((size_t)g * w.F_out_pad + w.r0) * 32,
                                  chunk, full);
                }
            }
        }
        __syncwarp();
        return;
    }

    // ---- run prologue: arena parity, zero the other buffer for the next run ----
    __shared__ unsigned s_par, s_target;
    if (threadIdx.x == 0) {
        unsigned par, old;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(par) : "l"(p.ctrl) : "memory");
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p.ctrl + 2) : "memory");
        s_par = par & 1u;
        s_target = (old / (unsigned)p.nctas + 1u) * (unsigned)p.nctas;
    }
    asm volatile("bar.sync 1, %0;" :: "n"(NW * 32) : "memory");
    const unsigned par = s_par;
    unsigned long long* const cur = p.peers[p.rank] + (long long)par * p.arena_words;   // this run's buffer
    {
        unsigned long long* nxt = p.peers[p.rank] + (long long)(par ^ 1u) * p.arena_words;
        const long long per = (p.arena_words + p.nctas - 1) / p.nctas;
        const long long zb = per * blockIdx.x, ze = min(p.arena_words, zb + per);
        for (long long i = zb + threadIdx.x; i < ze; i += NW * 32) nxt[i] = 0ull;
    }
    if (p.world > 1) {
        // peers write into our next buffer only after they consumed this run's
        // data; make the zeros visible system-wide and let every local CTA
        // finish zeroing before any of this rank's outputs leave the GPU
        __threadfence_system();
        asm volatile("bar.sync 1, %0;" :: "n"(NW * 32) : "memory");
        if (threadIdx.x == 0) {
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.ctrl + 2) : "memory");
            } while ((int)(v - s_target) < 0);
        }
        asm volatile("bar.sync 1, %0;" :: "n"(NW * 32) : "memory");
    }

    const int wrow0 = warp * RW;
    const auto co = core::chunk_offsets<RW>(wrow0, lane);
    const auto qm = core::set_map<G>(wrow0, lane);
    int slot = 0;            // ring position of the next stage (running across steps)
    uint32_t par_ring = 0;   // its mbarrier phase parity
    int cslot = 0;           // PAIR: codebook pair slot and parity
    uint32_t cpar = 0;
    // PAIR gather constant = PRMT operand b: byte 0 = h*128 + 4*sigma, byte 2 =
    // pair slot (64 KiB stride), so the address is PRMT(idx word, lbv) + the
    // ring base (uniform) -> LDS [R + UR] (gemv_core.cuh compute_group_set)
    for (int phj = 0; phj < p.n_steps * p.mi; ++phj) {
        const int ph = phj / p.mi, j = phj % p.mi;
        // the work item and phase are read-only for the kernel's lifetime
        const ChainItem w = p.items[((size_t)ph * p.nctas + blockIdx.x) * p.mi + j];
        const ChainPhase phs = p.phases[ph];
        // trace: t0 at the step's first item, t1/t2 of its first item, t3 after its last
        unsigned long long* tr = p.trace ? p.trace + ((size_t)ph * p.nctas + blockIdx.x) * 4 : nullptr;
        if (tr && threadIdx.x == 0 && j == 0) tr[0] = dev::globaltimer();
        if (w.rows_valid <= 0) continue;
        // every consumer warp is done with the previous step's s_x
        asm volatile("bar.sync 1, %0;" :: "n"(NW * 32) : "memory");
        const int ng = w.g_end - w.g_begin;
        if (phs.x_off >= 0)   // dataflow wait: poll this CTA's input words until final
            core::stage_x_counted<D, NB, NW, XF>(s_x, cur + phs.x_off, phs.x_ks, phs.F_in, p.B, w.N_ss, w.g_begin,
                                                 ng, p.world > 1, p.backoff);
        else
            core::stage_x<D, NB, NW, XF>(s_x, p.x_ext, 0, phs.F_in, p.B, w.N_ss, w.g_begin, ng);
        if (tr && threadIdx.x == 0 && j == 0) tr[1] = dev::globaltimer();
        asm volatile("bar.sync 1, %0;" :: "n"(NW * 32) : "memory");
        if (tr && threadIdx.x == 0 && j == 0) tr[2] = dev::globaltimer();
        const bool active = wrow0 < w.rows_valid;
        if constexpr (PAIR) {
            // pair stages: row-set mapping (gemv_core.cuh), 2G*NB accumulators
            // per lane, G-lane row reduction
            float acc[2 * G * NB];
#pragma unroll
            for (int q = 0; q < 2 * G * NB; ++q) acc[q] = 0.f;
            const bool run = active && !(p.dbg & 1);
            for (int i = 0; i < ng; i += 2) {
                dev::mbar_wait(cfull0 + 8 * cslot, cpar);
                const uint32_t lbs = (uint32_t)cslot << 16;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (h == 1 && i + 1 >= ng) break;
                    dev::mbar_wait(full0 + 8 * slot, par_ring);
                    if (run)
                        core::compute_group_set<D, NB, G>(acc, s_idx + slot * R * 32, qm, s_cb,
                                                          lbs + ((uint32_t)h << 7), s_x + (i + h) * XG);
                    __syncwarp();
                    if (lane == 0) dev::mbar_arrive(empty0 + 8 * slot);
                    if (++slot == ST) { slot = 0; par_ring ^= 1u; }
                }
                if (lane == 0) dev::mbar_arrive(cempty0 + 8 * cslot);
                if (++cslot == CS) { cslot = 0; cpar ^= 1u; }
            }
            core::reduce_set<NB, G>(acc, lane);
            if (active) {
                const long long off = (long long)par * p.arena_words + w.y_off + w.row0_g;
                for (int q = 0; q < p.world; ++q)
                    core::counted_store_set<NB, G>(acc, p.peers[q] + off, w.r0 + wrow0, lane, w.F_out, w.F_out_g,
                                                   p.B, p.world > 1);
            }
        } else {
        float acc[RW][NB];
#pragma unroll
        for (int q = 0; q < RW; ++q)
#pragma unroll
            for (int b = 0; b < NB; ++b) acc[q][b] = 0.f;
        {   // d = 4, 8: lane = subspace over 64/B rows per warp
            for (int i = 0; i < ng; ++i) {
                dev::mbar_wait(full0 + 8 * slot, par_ring);
                if (active && !(p.dbg & 1)) {
                    uint32_t xv[NB][E / 4];
                    core::load_x<D, NB>(xv, s_x + i * XG, lane);
                    core::compute_group<D, NB, RW>(acc, s_idx + slot * R * 32, co, s_cb + slot * p.cbb_max, xv,
                                                   lane);
                }
                __syncwarp();
                if (lane == 0) dev::mbar_arrive(empty0 + 8 * slot);
                if (++slot == ST) { slot = 0; par_ring ^= 1u; }
            }
        }
        core::RowTotals<NB, RW> tot;
        core::reduce_rows<NB, RW>(acc, tot, lane);
        if (active) {
            // this rank's rows go into EVERY rank's buffer (NVLink peer stores
            // when world > 1): the row-shard all-gather fused into the GEMV
            const long long off = (long long)par * p.arena_words + w.y_off + w.row0_g;
            for (int q = 0; q < p.world; ++q)
                core::counted_store<NB, RW>(tot, p.peers[q] + off, w.r0 + wrow0, w.F_out, w.F_out_g, p.B);
        }
        }
        if (tr && lane == 0 && warp == 0) tr[3] = dev::globaltimer();
    }
    // ---- run epilogue: flip the parity once every CTA has read it ----
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.ctrl + 2) : "memory");
        } while ((int)(v - s_target) < 0);
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p.ctrl), "r"(par ^ 1u) : "memory");
    }
}

constexpr size_t kChainSmem = kSmemMax;

struct ChainCfg {
    int rw, nw, st;
};

template <int D, int NB, int NW, int ST>
fasq_status launch_chain_t(const ChainParams& p, size_t smem, int grid, cudaStream_t st) {
    auto kern = k_chain<D, NB, NW, ST>;
    static size_t lim = 0;
    static std::once_flag once;
    std::call_once(once, [&] { lim = set_max_dyn_smem(kern); });
    if (lim < smem) {
        set_error("chain: dynamic SMEM plan (" + std::to_string(smem) + " B) exceeds the device limit (" +
                  std::to_string(lim) + " B)");
        return FASQ_E_UNSUPPORTED;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3((NW + 1) * 32, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident (consumers spin on producers' words)
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FASQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
    return FASQ_OK;
}

template <int D, int NB>
fasq_status chain_cfg(const fasq_chain* c, const ChainParams& p, cudaStream_t st) {
#define FASQ_CHAIN_CASE(NW_, ST_) \
    if (c->nw == NW_ && c->st == ST_) return launch_chain_t<D, NB, NW_, ST_>(p, c->smem, c->nctas, st);
    FASQ_CHAIN_CASE(16, 3)
    FASQ_CHAIN_CASE(16, 2)
    FASQ_CHAIN_CASE(16, 1)
    FASQ_CHAIN_CASE(8, 3)
    FASQ_CHAIN_CASE(8, 2)
    FASQ_CHAIN_CASE(8, 1)
#undef FASQ_CHAIN_CASE
    set_error("chain: no kernel instantiated for this tiling");
    return FASQ_E_UNSUPPORTED;
}

template <int D>
fasq_status chain_nb(const fasq_chain* c, const ChainParams& p, cudaStream_t st) {
    switch (c->B <= 1 ? 1 : c->B <= 2 ? 2 : c->B <= 4 ? 4 : 8) {
        case 1: return chain_cfg<D, 1>(c, p, st);
        case 2: return chain_cfg<D, 2>(c, p, st);
        case 4: return chain_cfg<D, 4>(c, p, st);
        case 8: return chain_cfg<D, 8>(c, p, st);
    }
    return FASQ_E_UNSUPPORTED;
}

// counted accumulator words of the LAST run -> value (units 2^-32) -> fp16 /
// fp32 / FASQ_ACC_I64.  The run flipped the parity at its end, so its buffer
// is parity ^ 1 (read on the device: graph replays need no host bookkeeping).
__global__ void k_counted_convert(const unsigned long long* __restrict__ arenas, long long arena_words,
                                  const unsigned* __restrict__ ctrl, long long off, int64_t n, int ks, void* out,
                                  int dtype) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned last = (ctrl[0] & 1u) ^ 1u;
    const unsigned long long wv = arenas[(long long)last * arena_words + off + i];
    const long long v = (long long)(wv & core::kCntMask) - (long long)ks * core::kCntBias;
    if (dtype == FASQ_ACC_I64) reinterpret_cast<long long*>(out)[i] = v;
    else if (dtype == FASQ_F32) reinterpret_cast<float*>(out)[i] = (float)((double)v * core::kAccInv);
    else reinterpret_cast<__half*>(out)[i] = __double2half((double)v * core::kAccInv);
}

int sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

void destroy_chain(fasq_chain* c) {
    if (!c) return;
    for (void* q : c->ipc_opened) cudaIpcCloseMemHandle(q);
    if (c->arenas) cudaFree(c->arenas);
    if (c->ctrl) cudaFree(c->ctrl);
    if (c->peers_dev) cudaFree(c->peers_dev);
    if (c->items) cudaFree(c->items);
    if (c->phases) cudaFree(c->phases);
    delete c;
}

fasq_status upload_peers(fasq_chain* c, const std::vector<unsigned long long*>& bases) {
    FASQ_CUDA_TRY(cudaMemcpy(c->peers_dev, bases.data(), bases.size() * sizeof(void*), cudaMemcpyHostToDevice));
    c->peers_ready = true;
    return FASQ_OK;
}

}  // namespace

}  // namespace fasq

using namespace fasq;

extern "C" {

fasq_status fasq_chain_create_tp(const fasq_chain_step* steps, int32_t n_steps, int32_t B, int32_t world,
                                 int32_t rank, int32_t max_ctas, void* stream, fasq_chain** out) {
    if (!out) return FASQ_E_ARG;
    *out = nullptr;
    if (!steps || n_steps < 1) return FASQ_E_ARG;
    if (world < 1 || world > 8 || rank < 0 || rank >= world || max_ctas < 0) return FASQ_E_ARG;
    if (B < 1 || B > 8) return FASQ_E_UNSUPPORTED;
    const int NB = B <= 1 ? 1 : B <= 2 ? 2 : B <= 4 ? 4 : 8;
    fasq_chain* c = new fasq_chain();
    c->n_steps = n_steps;
    c->B = B;
    c->world = world;
    c->rank = rank;
    c->nctas = sm_count();
    if (max_ctas > 0) c->nctas = std::min(c->nctas, (int)max_ctas);
    // same tiling family as the per-launch GEMV default (gemv.cu plan_gemv)
    c->nw = 16;
    c->rw = NB == 1 ? 64 : NB == 2 ? 32 : NB == 4 ? 16 : 8;   // core::RowsPerWarp (d = 4, 8)
    c->st = 3;
    if (const char* e = getenv("FASQ_CHAIN_CFG")) {   // experiments: "nw,st"
        int a = 0, b = 0;
        if (sscanf(e, "%d,%d", &a, &b) == 2) { c->nw = a; c->st = b; }
    }
    c->R = c->rw * c->nw;
    // validate + arena layout: every layer output is the FULL (all-rank) vector
    int64_t words = 16;   // [0..15]: reserved
    c->acc_off.resize(n_steps);
    c->acc_Fout.resize(n_steps);
    c->acc_ks.resize(n_steps);
    c->step_F_in.resize(n_steps);
    for (int s = 0; s < n_steps; ++s) {
        const fasq_chain_step& S = steps[s];
        if (!S.layers || S.n_layers < 1 || S.n_layers > 4) { destroy_chain(c); return FASQ_E_ARG; }
        const int64_t F_in = S.layers[0]->F_in;
        for (int l = 0; l < S.n_layers; ++l) {
            const fasq_layer* L = S.layers[l];
            if (!L) { destroy_chain(c); return FASQ_E_ARG; }
            if (L->F_in != F_in) { destroy_chain(c); return FASQ_E_SHAPE; }
            if (c->d == 0) c->d = L->d;
            if (L->d != c->d) { destroy_chain(c); return FASQ_E_UNSUPPORTED; }
            c->maxC = std::max(c->maxC, L->C);
            c->acc_off[s].push_back(words);
            c->acc_Fout[s].push_back(L->F_out * world);
            words += (int64_t)B * L->F_out * world;
        }
        c->step_F_in[s] = (int)F_in;
        if (S.input_step < 0) {
            if (c->ext_F_in == 0) c->ext_F_in = (int)F_in;
            if (c->ext_F_in != F_in) { destroy_chain(c); return FASQ_E_SHAPE; }
        } else {
            if (S.input_step >= s || S.input_layer < 0 || S.input_layer >= steps[S.input_step].n_layers) {
                destroy_chain(c);
                return FASQ_E_ARG;
            }
            if (steps[S.input_step].layers[S.input_layer]->F_out * world != F_in) {
                destroy_chain(c);
                return FASQ_E_SHAPE;
            }
        }
    }
    if (c->ext_F_in == 0) { destroy_chain(c); return FASQ_E_ARG; }   // the chain needs an external input
    if (c->d <= 2) c->rw = 64;   // pair stages: row-set mapping, 64 rows per warp at any B
    const int E = entry_bytes(c->d);
    const size_t cbb_max = (size_t)c->maxC * 32 * E;
    const bool pair = c->d <= 2;   // ChainPair: codebook pair ring next to the index ring
    auto cbring = [&](int st) { return pair ? (size_t)kChainCS * kPairSlot : (size_t)st * cbb_max; };
    // (x staging is added after the work plan, smem_of below)
    auto ring = [&](int st, int nw) { return cbring(st) + (size_t)st * c->rw * nw * 32; };
    while (c->st > 2 && ring(c->st, c->nw) > kChainSmem) --c->st;
    if (ring(c->st, c->nw) > kChainSmem && c->nw > 8) c->nw = 8;
    while (c->st > 1 && ring(c->st, c->nw) > kChainSmem) --c->st;
    c->R = c->rw * c->nw;
    c->arena_words = words;
    if (cudaMalloc(&c->arenas, (size_t)words * 2 * 8) != cudaSuccess ||
        cudaMalloc(&c->ctrl, 64) != cudaSuccess ||
        cudaMalloc(&c->peers_dev, 8 * sizeof(void*)) != cudaSuccess) {
        cudaGetLastError();
        destroy_chain(c);
        return FASQ_E_OOM;
    }
    // work plan: per step a list of items (row tile x K-range), dealt to the
    // CTAs round-robin; more items than CTAs (e.g. B = 8: 128-row tiles) ->
    // several items per CTA per step, [n_steps][nctas][mi]
    std::vector<std::vector<ChainItem>> per_step(n_steps);
    std::vector<ChainPhase> phases(n_steps);
    for (int s = 0; s < n_steps; ++s) {
        const fasq_chain_step& S = steps[s];
        const int nl = S.n_layers;
        double W = 0;
        for (int l = 0; l < nl; ++l) W += (double)S.layers[l]->F_out_pad * S.layers[l]->n_groups;
        std::vector<int> rt(nl), ks(nl);
        int total = 0;
        for (int l = 0; l < nl; ++l) {
            const fasq_layer* L = S.layers[l];
            rt[l] = (L->F_out_pad + c->R - 1) / c->R;
            const double share = c->nctas * ((double)L->F_out_pad * L->n_groups) / W;
            int k = std::max(1, (int)(share / rt[l]));
            k = std::min(k, L->n_groups);
            // use every CTA the share allows even when the K ranges then differ by
            // one group (e.g. down: 37 x 6-7 groups instead of 32 x 7): the
            // dataflow lets short items hand their outputs over early, and
            // measured 0.92-0.95 -> 0.90 ms/token; FASQ_CHAIN_EVEN=1 restores
            // equal-sized K ranges
            if (getenv("FASQ_CHAIN_EVEN") != nullptr) {
                const int gper = (L->n_groups + k - 1) / k;
                k = (L->n_groups + gper - 1) / gper;
            }
            ks[l] = k;
            total += rt[l] * k;
        }
        while (total > c->nctas) {
            int lm = -1;
            for (int l = 0; l < nl; ++l)
                if (ks[l] > 1 && (lm < 0 || ks[l] * rt[l] > ks[lm] * rt[lm])) lm = l;
            if (lm < 0) break;
            total -= rt[lm];
            ks[lm] -= 1;
        }
        for (int l = 0; l < nl; ++l) {
            if (ks[l] > 63) { destroy_chain(c); return FASQ_E_UNSUPPORTED; }   // counted-word count field
            c->acc_ks[s].push_back(ks[l]);
        }
        for (int l = 0; l < nl; ++l) {
            const fasq_layer* L = S.layers[l];
            for (int r = 0; r < rt[l]; ++r)
                for (int k = 0; k < ks[l]; ++k) {
                    ChainItem w{};
                    w.idx = L->idx;
                    w.cbimg = L->cbimg;
                    w.cbmap = L->cbmap;
                    w.y_off = c->acc_off[s][l];
                    w.F_out = (int)L->F_out;
                    w.F_out_g = (int)(L->F_out * world);
                    w.row0_g = (int)(L->F_out * rank);
                    w.F_out_pad = L->F_out_pad;
                    w.N_ss = L->N_ss;
                    w.C = L->C;
                    w.r0 = r * c->R;
                    w.rows_valid = std::min(c->R, L->F_out_pad - w.r0);
                    w.g_begin = (int)((int64_t)k * L->n_groups / ks[l]);
                    w.g_end = (int)((int64_t)(k + 1) * L->n_groups / ks[l]);
                    c->gmax = std::max(c->gmax, w.g_end - w.g_begin);
                    per_step[s].push_back(w);
                }
        }
        phases[s].F_in = c->step_F_in[s];
        phases[s].x_off = S.input_step < 0 ? -1 : c->acc_off[S.input_step][S.input_layer];
        phases[s].x_ks = S.input_step < 0 ? 0 : c->acc_ks[S.input_step][S.input_layer];
    }
    c->mi = 1;
    for (const auto& v : per_step) c->mi = std::max(c->mi, (int)((v.size() + c->nctas - 1) / c->nctas));
    std::vector<ChainItem> items((size_t)n_steps * c->nctas * c->mi);
    for (auto& w : items) w = ChainItem{};
    for (int s = 0; s < n_steps; ++s)
        for (size_t q = 0; q < per_step[s].size(); ++q)
            items[((size_t)s * c->nctas + q % c->nctas) * c->mi + q / c->nctas] = per_step[s][q];
    const size_t xg = (pair && NB == 8) ? (size_t)32 * NB * c->d * 4 : (size_t)32 * NB * E;   // k_chain XG
    auto smem_of = [&](int st) {
        return cbring(st) + (size_t)st * c->R * 32 + (size_t)c->gmax * xg + 16 * (st + kChainCS);
    };
    while (c->st > 1 && smem_of(c->st) > kChainSmem) --c->st;
    c->smem = smem_of(c->st);
    if (c->smem > kChainSmem) { destroy_chain(c); set_error("chain: SMEM plan too large"); return FASQ_E_UNSUPPORTED; }
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMalloc(&c->items, items.size() * sizeof(ChainItem)) != cudaSuccess ||
        cudaMalloc(&c->phases, phases.size() * sizeof(ChainPhase)) != cudaSuccess) {
        cudaGetLastError();
        destroy_chain(c);
        return FASQ_E_OOM;
    }
    cudaError_t e = cudaMemcpyAsync(c->items, items.data(), items.size() * sizeof(ChainItem), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(c->phases, phases.data(), phases.size() * sizeof(ChainPhase), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->arenas, 0, (size_t)words * 2 * 8, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->ctrl, 0, 64, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);   // host vectors go out of scope
    if (e != cudaSuccess) { fasq_status s = cuda_fail(e, "chain upload"); destroy_chain(c); return s; }
    std::vector<unsigned long long*> bases(world, nullptr);
    bases[rank] = c->arenas;
    fasq_status s = upload_peers(c, bases);
    if (s != FASQ_OK) { destroy_chain(c); return s; }
    c->peers_ready = world == 1;
    *out = c;
    return FASQ_OK;
}

fasq_status fasq_chain_create(const fasq_chain_step* steps, int32_t n_steps, int32_t B, void* stream,
                              fasq_chain** out) {
    return fasq_chain_create_tp(steps, n_steps, B, 1, 0, 0, stream, out);
}

fasq_status fasq_chain_ipc_handle(const fasq_chain* c, void* handle_out) {
    if (!c || !handle_out) return FASQ_E_ARG;
    cudaIpcMemHandle_t h;
    FASQ_CUDA_TRY(cudaIpcGetMemHandle(&h, c->arenas));
    std::memcpy(handle_out, &h, sizeof(h));
    return FASQ_OK;
}

fasq_status fasq_chain_set_peers(fasq_chain* c, const void* handles) {
    if (!c || !handles) return FASQ_E_ARG;
    std::vector<unsigned long long*> bases(c->world, nullptr);
    for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) { bases[r] = c->arenas; continue; }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const uint8_t*>(handles) + (size_t)r * sizeof(h), sizeof(h));
        void* q = nullptr;
        FASQ_CUDA_TRY(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(q);
        bases[r] = static_cast<unsigned long long*>(q);
    }
    return upload_peers(c, bases);
}

fasq_status fasq_chain_set_peer_chains(fasq_chain* c, const fasq_chain* const* chains) {
    if (!c || !chains) return FASQ_E_ARG;
    std::vector<unsigned long long*> bases(c->world, nullptr);
    for (int r = 0; r < c->world; ++r) {
        const fasq_chain* o = chains[r];
        if (!o || o->world != c->world || o->arena_words != c->arena_words || o->n_steps != c->n_steps)
            return FASQ_E_ARG;
        bases[r] = o->arenas;
    }
    if (bases[c->rank] != c->arenas) return FASQ_E_ARG;
    return upload_peers(c, bases);
}

fasq_status fasq_chain_run(fasq_chain* c, const void* x_dev, void* stream) {
    if (!c || !x_dev) return FASQ_E_ARG;
    if (!c->peers_ready) { set_error("chain: world > 1 needs fasq_chain_set_peers first"); return FASQ_E_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    ChainParams p{};
    p.items = static_cast<const ChainItem*>(c->items);
    p.phases = static_cast<const ChainPhase*>(c->phases);
    p.x_ext = static_cast<const __half*>(x_dev);
    p.trace = c->trace;
    p.ctrl = c->ctrl;
    p.peers = c->peers_dev;
    p.arena_words = c->arena_words;
    p.world = c->world;
    p.rank = c->rank;
    p.pf = 0;
    if (const char* e = getenv("FASQ_CHAIN_PF")) p.pf = atoi(e);
    p.dbg = 0;
    if (const char* e = getenv("FASQ_CHAIN_DBG")) p.dbg = atoi(e);
    p.backoff = 0;
    if (const char* e = getenv("FASQ_CHAIN_BACKOFF")) p.backoff = atoi(e);
    p.n_steps = c->n_steps;
    p.nctas = c->nctas;
    p.B = c->B;
    p.gmax = c->gmax;
    p.mi = c->mi;
    p.cbb_max = c->maxC * 32 * entry_bytes(c->d);
    fasq_status s;
    switch (c->d) {
        case 1: s = chain_nb<1>(c, p, st); break;
        case 2: s = chain_nb<2>(c, p, st); break;
        case 4: s = chain_nb<4>(c, p, st); break;
        case 8: s = chain_nb<8>(c, p, st); break;
        default: s = FASQ_E_UNSUPPORTED;
    }
    if (s == FASQ_OK) set_launch_count(1);
    return s;
}

fasq_status fasq_chain_output(const fasq_chain* c, int32_t step, int32_t layer, void* y_dev, fasq_dtype dtype,
                              void* stream) {
    if (!c || !y_dev || step < 0 || step >= c->n_steps) return FASQ_E_ARG;
    if (layer < 0 || layer >= (int)c->acc_off[step].size()) return FASQ_E_ARG;
    if (dtype != FASQ_F16 && dtype != FASQ_F32 && dtype != FASQ_ACC_I64) return FASQ_E_ARG;
    const int64_t n = (int64_t)c->B * c->acc_Fout[step][layer];
    if (n <= 0) return FASQ_OK;
    k_counted_convert<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        c->arenas, c->arena_words, c->ctrl, c->acc_off[step][layer], n, c->acc_ks[step][layer], y_dev, (int)dtype);
    FASQ_CUDA_TRY(cudaGetLastError());
    set_launch_count(1);
    return FASQ_OK;
}

fasq_status fasq_chain_trace(fasq_chain* c, void* trace_dev) {
    if (!c) return FASQ_E_ARG;
    c->trace = static_cast<unsigned long long*>(trace_dev);
    return FASQ_OK;
}

int32_t fasq_chain_ctas(const fasq_chain* c) { return c ? c->nctas : -1; }

void fasq_chain_free(fasq_chain* c) {
    if (!c) return;
    cudaDeviceSynchronize();
    destroy_chain(c);
}

}  // extern "C"
