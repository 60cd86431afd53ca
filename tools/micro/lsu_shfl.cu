// Microbenchmark: shared-memory gather (LDS.32, lanes at distinct banks) vs
// SHFL.IDX throughput per SM, and a 50/50 mix.  nvcc -arch=sm_100a; run on 1 GPU.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters) {
    __shared__ float s[8][32];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s[i >> 5][i & 31] = i * 0.5f;
    __syncthreads();
    float acc = lane, v = lane * 0.25f;
    int idx = (lane * 7) & 31;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (MODE == 0) {  // 8 LDS
                acc += s[u][idx];
            } else if (MODE == 1) {  // 8 SHFL
                acc += __shfl_sync(0xffffffffu, v, idx + u);
            } else {  // 4 LDS + 4 SHFL
                if (u & 1) acc += s[u][idx];
                else acc += __shfl_sync(0xffffffffu, v, idx + u);
            }
        }
        idx = (idx + 5) & 31;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    float* d;
    cudaMalloc(&d, 148 * 16 * 1024 * 4);
    const int iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<148 * 4, 512>>>(d, iters);
            if (mode == 1) k<1><<<148 * 4, 512>>>(d, iters);
            if (mode == 2) k<2><<<148 * 4, 512>>>(d, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double warp_insts_per_sm = 4.0 * 16 * iters * 8;  // per SM: 4 blocks x 16 warps
            if (rep) printf("mode %d: %.3f ms, %.3f mem-insts/clk/SM (at 1.965 GHz)\n", mode, ms,
                            warp_insts_per_sm / (ms * 1e-3 * 1.965e9));
        }
    }
    return 0;
}
