// Microbenchmark: mma.sync.m16n8k8 tf32 throughput on sm_100a (legacy warp MMA path).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 + 1, b1 = a0 + 2;
    float c[4][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[u][0]), "+f"(c[u][1]), "+f"(c[u][2]), "+f"(c[u][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* d;
    cudaMalloc(&d, 148 * 8 * 256 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 8192;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        k<<<148 * 8, 256>>>(d, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double mmas = 148.0 * 8 * 8 * iters * 4;  // warps x iters x 4
        if (rep) printf("%.3f ms: %.2f mma/clk/SM, %.1f TFLOP/s tf32\n", ms, mmas / 148 / (ms * 1e-3 * 1.965e9),
                        mmas * 2048 / (ms * 1e-3) / 1e12);
    }
}
