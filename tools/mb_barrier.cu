// Grid-barrier latency microbenchmark (B200): one CTA per SM, `iters`
// back-to-back barriers, each optionally preceded by `nred` red.add.u64 per
// CTA (the chain's output stores).  Reports ns per barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_barrier tools/mb_barrier.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_bar(unsigned* counter, unsigned long long* sink, int iters, int nred, unsigned long long* out_t) {
    const int nct = gridDim.x;
    unsigned long long t0 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) {
        if (MODE >= 6) {
            // plain coalesced stores instead of reductions
            for (int r = threadIdx.x; r < nred; r += blockDim.x)
                asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(reinterpret_cast<unsigned*>(sink) + ((size_t)blockIdx.x * nred + r)), "r"(i) : "memory");
        } else {
            for (int r = threadIdx.x; r < nred; r += blockDim.x)
                asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" :: "l"(sink + ((size_t)blockIdx.x * nred + r)) : "memory");
        }
        if (MODE == 7) asm volatile("fence.acq_rel.gpu;" ::: "memory");   // every thread fences its own stores
        __syncthreads();
        if (MODE == 4) {
            // one flag per CTA (own 128-B line), every CTA polls all flags in parallel
            if (threadIdx.x == 0)
                asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(counter + 32 * blockIdx.x), "r"(i + 1) : "memory");
            if (threadIdx.x < nct) {
                unsigned v;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter + 32 * threadIdx.x) : "memory");
                } while ((int)(v - (unsigned)(i + 1)) < 0);
            }
        } else if (MODE == 5) {
            // 16 counters (own lines), CTA b adds to counter b % 16
            constexpr int NCNT = 16;
            if (threadIdx.x == 0)
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(counter + 32 * (blockIdx.x % NCNT)) : "memory");
            if (threadIdx.x < NCNT) {
                const unsigned per = (unsigned)(nct / NCNT + (threadIdx.x < nct % NCNT ? 1 : 0));
                const unsigned target = (unsigned)(i + 1) * per;
                unsigned v;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter + 32 * threadIdx.x) : "memory");
                } while ((int)(v - target) < 0);
            }
        }
        if (threadIdx.x == 0) {
            const unsigned target = (unsigned)(i + 1) * nct;
            if (MODE == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(counter) : "memory");
                unsigned v;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
                } while ((int)(v - target) < 0);
            } else if (MODE == 1) {
                __threadfence();
                atomicAdd(counter, 1u);
                unsigned v;
                do {
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
                } while ((int)(v - target) < 0);
                __threadfence();
            } else if (MODE == 2) {
                // atom returns the old value: the last arriver knows at once
                unsigned old;
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(counter) : "memory");
                if (old + 1 != target) {
                    unsigned v;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
                    } while ((int)(v - target) < 0);
                }
            } else if (MODE == 6) {
                unsigned old;
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(counter) : "memory");
                if (old + 1 != target) {
                    unsigned v;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
                    } while ((int)(v - target) < 0);
                }
            } else if (MODE == 7) {
                unsigned old;
                asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(counter) : "memory");
                if (old + 1 != target) {
                    unsigned v;
                    do {
                        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
                    } while ((int)(v - target) < 0);
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            } else if (MODE == 4 || MODE == 5) {
            } else {
                // per-die split: poll with nanosleep-free volatile loads
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(counter) : "memory");
                unsigned v;
                do {
                    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
                } while ((int)(v - target) < 0);
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
        }
        __syncthreads();
    }
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) out_t[blockIdx.x] = t1 - t0;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned* counter;
    unsigned long long *sink, *out_t;
    cudaMalloc(&counter, 256 * 128);
    cudaMalloc(&sink, (size_t)nsm * 4096 * 8);
    cudaMalloc(&out_t, nsm * 8);
    const int iters = 2000;
    for (int mode : {0, 2, 6, 7}) {
        for (int nred : {0, 256, 1024, 2048}) {
            float best = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
                cudaMemset(counter, 0, 256 * 128);
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                cudaEventRecord(a);
                switch (mode) {
                    case 0: k_bar<0><<<nsm, 512>>>(counter, sink, iters, nred, out_t); break;
                    case 1: k_bar<1><<<nsm, 512>>>(counter, sink, iters, nred, out_t); break;
                    case 2: k_bar<2><<<nsm, 512>>>(counter, sink, iters, nred, out_t); break;
                    case 3: k_bar<3><<<nsm, 512>>>(counter, sink, iters, nred, out_t); break;
                    case 4: k_bar<4><<<nsm, 512>>>(counter, sink, iters, nred, out_t); break;
                    case 5: k_bar<5><<<nsm, 512>>>(counter, sink, iters, nred, out_t); break;
                    case 6: k_bar<6><<<nsm, 512>>>(counter, sink, iters, nred, out_t); break;
                    default: k_bar<7><<<nsm, 512>>>(counter, sink, iters, nred, out_t); break;
                }
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("mode %d nred %4d: %.0f ns per barrier\n", mode, nred, best * 1e6f / iters);
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
