// Microbenchmark: how fast can one CTA per SM stream HBM into SMEM with
// cp.async.bulk (TMA engine) at various request sizes, vs LDG.128?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_bulk tools/mb_bulk.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(c)); }
__device__ __forceinline__ void expect(uint32_t bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(b) : "memory"); }
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t ph) {
    uint32_t ok;
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
    return ok;
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// CTAs in groups of `share` read the SAME `region` bytes (L2-resident) in 32 KiB copies, `reps` times.
__global__ void k_bulk_share(const uint8_t* src, size_t region, int share, int reps, unsigned long long* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t bars[4];
    const uint8_t* base = src + (size_t)(blockIdx.x / share) * region;
    if (threadIdx.x == 0) { for (int s = 0; s < 4; ++s) mbar_init(smem_u32(&bars[s]), 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    const uint32_t stage = 32768;
    const int nst = (int)(region / stage) * reps;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) {
            int s = i % 4;
            if (i >= 4) { int j = i - 4; while (!try_wait(smem_u32(&bars[s]), (j / 4) & 1)) {} }
            expect(smem_u32(&bars[s]), stage);
            bulk(smem_u32(sm + s * stage), base + (size_t)(i % (region / stage)) * stage, stage, smem_u32(&bars[s]));
        }
        for (int j = nst - 4; j < nst; ++j) { if (j < 0) continue; while (!try_wait(smem_u32(&bars[j % 4]), (j / 4) & 1)) {} }
    }
    __syncthreads();
    if (threadIdx.x == 0) sink[blockIdx.x] = sm[5];
}

// Each CTA streams `per_cta` bytes in chunks of `chunk` bytes through a STAGES ring of `stage` bytes.
template <int STAGES>
__global__ void k_bulk(const uint8_t* src, size_t per_cta, uint32_t stage, uint32_t chunk, int issuers, unsigned long long* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t bars[STAGES];
    const uint8_t* base = src + blockIdx.x * per_cta;
    if (threadIdx.x == 0) { for (int s = 0; s < STAGES; ++s) mbar_init(smem_u32(&bars[s]), 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    const int nst = (int)(per_cta / stage);
    if (threadIdx.x < 32) {
        int lane = threadIdx.x;
        for (int i = 0; i < nst; ++i) {
            int s = i % STAGES;
            if (i >= STAGES) { while (!try_wait(smem_u32(&bars[s]), ((i / STAGES) + 1) & 1)) {} }
            // consumer in the same warp: wait for the previous fill of this slot ... simplified: single warp
            if (lane == 0) expect(smem_u32(&bars[s]), stage);
            __syncwarp();
            for (uint32_t c = lane; c < stage / chunk; c += issuers)
                if (lane < issuers) bulk(smem_u32(sm + s * stage + c * chunk), base + (size_t)i * stage + c * chunk, chunk, smem_u32(&bars[s]));
            // wait this stage immediately if ring full next time (the wait above handles reuse)
            // emulate consumption: wait full
            if (i >= STAGES - 1) {
                int j = i - (STAGES - 1);
                int sj = j % STAGES;
                while (!try_wait(smem_u32(&bars[sj]), (j / STAGES) & 1)) {}
            }
        }
        for (int j = nst - (STAGES - 1); j < nst; ++j) { if (j < 0) continue; int sj = j % STAGES; while (!try_wait(smem_u32(&bars[sj]), (j / STAGES) & 1)) {} }
    }
    __syncthreads();
    if (threadIdx.x == 0) sink[blockIdx.x] = sm[5];
}

__global__ void k_ldg(const uint4* src, size_t per_cta, unsigned long long* sink) {
    const uint4* base = src + blockIdx.x * (per_cta / 16);
    uint32_t acc = 0;
    const size_t n = per_cta / 16;
    for (size_t i = threadIdx.x; i < n; i += blockDim.x * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { size_t k = i + u * blockDim.x; v[u] = k < n ? __ldg(base + k) : make_uint4(0,0,0,0); }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x12345) sink[blockIdx.x] = acc;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t per_cta = 8u << 20;           // 8 MiB per CTA -> ~1.2 GB total
    uint8_t* src; cudaMalloc(&src, per_cta * sms);
    cudaMemset(src, 1, per_cta * sms);
    unsigned long long* sink; cudaMalloc(&sink, sms * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaFuncSetAttribute(k_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Cfg { uint32_t stage, chunk; int issuers; };
    Cfg cfgs[] = {{32768, 32768, 1}, {16384, 16384, 1}, {8192, 8192, 1}, {32768, 4096, 8}, {32768, 1024, 32}, {32768, 128, 32}, {32768, 128, 1}, {49152, 49152, 1}};
    for (auto c : cfgs) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_bulk<4><<<sms, 64, 4 * c.stage>>>(src, per_cta, c.stage, c.chunk, c.issuers, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("bulk stage=%u chunk=%u issuers=%d : %.1f GB/s  (%s)\n", c.stage, c.chunk, c.issuers, per_cta * sms / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    }
    for (int th : {256, 512, 1024}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_ldg<<<sms, th>>>((const uint4*)src, per_cta, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("ldg threads=%d : %.1f GB/s\n", th, per_cta * sms / ms / 1e6);
        }
    }
    // L2-resident re-read bandwidth: 64 MiB region read 8 times by all SMs via LDG
    {
        size_t l2b = 64u << 20; size_t pc = l2b / sms / 16 * 16;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            for (int it = 0; it < 8; ++it) k_ldg<<<sms, 1024>>>((const uint4*)src, pc, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep == 2) printf("ldg L2-resident (64MiB x8): %.1f GB/s\n", 8.0 * pc * sms / ms / 1e6);
        }
    }
    cudaFuncSetAttribute(k_bulk_share, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int share : {1, 2, 4, 8, 37, 148}) {
        size_t region = 256 * 1024;          // 256 KiB per sharing group (L2 resident)
        int reps = 64;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_bulk_share<<<sms, 32, 4 * 32768>>>(src, region, share, reps, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("bulk shared-region share=%d : delivered %.1f GB/s (%s)\n", share, (double)region * reps * sms / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
