// mb_tma3d.cu -- checks that a 3-D TMA tensor map with a non-monotonic stride
// order (dim1 stride > dim2 stride) encodes and loads the codebook PAIR image
// [k][2 groups][32 words] from the [group][k][32] layout.
// nvcc -gencode arch=compute_100a,code=sm_100a -o mb_tma3d tools/mb_tma3d.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap map, uint32_t* out, int g, int C) {
    extern __shared__ __align__(1024) uint32_t sm[];
    __shared__ __align__(8) uint64_t bar;
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    uint32_t d = (uint32_t)__cvta_generic_to_shared(sm);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(2 * C * 128) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     :: "r"(d), "l"(&map), "r"(0), "r"(g), "r"(0), "r"(b) : "memory");
        uint32_t ok = 0;
        while (!ok) {
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(b) : "memory");
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * C * 32; i += blockDim.x) out[i] = sm[i];
}

int main() {
    const int G = 5, C = 256;
    std::vector<uint32_t> h((size_t)G * C * 32);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (uint32_t)i * 2654435761u;
    uint32_t *dimg, *dout;
    cudaMalloc(&dimg, h.size() * 4);
    cudaMalloc(&dout, 2 * C * 32 * 4);
    cudaMemcpy(dimg, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap map;
    cuuint64_t gdim[3] = {32, (cuuint64_t)G, (cuuint64_t)C};
    cuuint64_t gstr[2] = {(cuuint64_t)C * 128, 128};
    cuuint32_t box[3] = {32, 2, (cuuint32_t)C};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, dimg, gdim, gstr, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    if (r != CUDA_SUCCESS) return 1;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * C * 128);
    int bad = 0;
    for (int g = 0; g < G; ++g) {
        k<<<1, 256, 2 * C * 128>>>(map, dout, g, C);
        std::vector<uint32_t> o(2 * C * 32);
        cudaError_t e = cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
        for (int kk = 0; kk < C; ++kk)
            for (int hh = 0; hh < 2; ++hh)
                for (int w = 0; w < 32; ++w) {
                    uint32_t want = (g + hh < G) ? h[((size_t)(g + hh) * C + kk) * 32 + w] : 0u;
                    if (o[((size_t)kk * 2 + hh) * 32 + w] != want) ++bad;
                }
        printf("g=%d mismatches so far %d\n", g, bad);
    }
    printf(bad ? "FAIL\n" : "PASS\n");
    return bad != 0;
}
