#include <cstdio>
#include <cstdint>
__global__ void b1_peak(int *out, int iters) {
    uint32_t a0 = threadIdx.x * 0x9E3779B9u, a1 = a0 ^ 0x12345678u, a2 = a0 * 3u, a3 = a0 + 7u;
    uint32_t b0 = a0 ^ 0xdeadbeefu, b1 = a1 + 1u;
    int c[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
        }
    }
    int s = 0;
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int *d; cudaMalloc(&d, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    b1_peak<<<148 * 8, 256>>>(d, 10); cudaDeviceSynchronize();
    int iters = 2000;
    cudaEventRecord(e0);
    b1_peak<<<148 * 8, 256>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double mmas = 148.0 * 8 * 8 /*warps*/ * iters * 8;
    double bitops = mmas * 16 * 8 * 256;
    printf("b1 mma: %.3f ms, %.3e mma/s, %.1f T bit-AND/s (err %s)\n", ms, mmas / (ms * 1e-3), bitops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
