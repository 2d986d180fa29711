// legacy mma.sync (HMMA) bf16 throughput on B200 (dev probe)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) hmma(int iters, float *out) {
    unsigned a0 = 0x3f803f80u ^ threadIdx.x, a1 = a0, a2 = a0, a3 = a0, b0 = 0x3f803f80u, b1 = b0;
    float c[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[q][0]), "+f"(c[q][1]), "+f"(c[q][2]), "+f"(c[q][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
    if (s == 1234.5f) out[0] = s;
}
int main() {
    float *o;
    cudaMalloc(&o, 4);
    for (int wpb : {4, 8}) {
        const int iters = 20000;
        hmma<<<148 * 2, 32 * wpb>>>(10, o);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        hmma<<<148 * 2, 32 * wpb>>>(iters, o);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * 148 * 2 * wpb;
        printf("mma.sync bf16 m16n8k16, %d warps/CTA x 296 CTAs: %.3f ms  %.1f TFLOP/s\n", wpb, ms, flops / ms / 1e9);
    }
    return 0;
}
