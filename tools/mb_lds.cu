// Shared-memory load throughput on one SM: NW warps issue conflict-free
// LDS.32 / LDS.64 / LDS.128 (independent addresses) with K ALU ops each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_lds tools/mb_lds.cu
#include <cstdio>
#include <cstdint>
template <int W, int ALU>
__global__ void k(float* out, int iters) {
    __shared__ __align__(16) uint32_t s[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t a = (uint32_t)lane * (W / 4);
    uint32_t acc = 0;
    float f = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            uint32_t idx = (a + (uint32_t)j * 32u * (W / 4) + (acc & 0)) & (8191u & ~(uint32_t)(W / 4 - 1));
            if (W == 4) acc += s[idx];
            else if (W == 8) { uint2 v = *reinterpret_cast<uint2*>(&s[idx]); acc += v.x ^ v.y; }
            else { uint4 v = *reinterpret_cast<uint4*>(&s[idx]); acc += v.x ^ v.y ^ v.z ^ v.w; }
#pragma unroll
            for (int q = 0; q < ALU; ++q) f = fmaf(f, 1.0001f, (float)q);
        }
        a += 7 * 32 * (W / 4);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc + f;
}
template <int W, int ALU>
void run(float* out, int nw) {
    const int iters = 4096;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<W, ALU><<<148, nw * 32>>>(out, 16);
    cudaEventRecord(e0);
    k<W, ALU><<<148, nw * 32>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double clk = 1.92e9;
    double lds_per_sm = (double)nw * iters * 16;
    printf("LDS.%-3d alu %d nw %2d: %.3f warp-LDS/clk/SM  (%.1f B/clk)\n", W * 8, ALU, nw, lds_per_sm / (ms * 1e-3 * clk),
           lds_per_sm * 32 * W / (ms * 1e-3 * clk));
}
int main() {
    float* out; cudaMalloc(&out, 148 * 1024 * 4);
    for (int nw : {8, 16, 32}) { run<4, 0>(out, nw); run<4, 2>(out, nw); run<4, 4>(out, nw); }
    for (int nw : {16}) { run<8, 0>(out, nw); run<16, 0>(out, nw); }
    return 0;
}
