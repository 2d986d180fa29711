// tcgen05.mma issue-path probe (dev tool): cycles per 128xNx16 bf16 MMA when the MMA chain is
// issued (a) by lane 0 inside a divergent `if (lane == 0)` (the compiler wraps every
// tcgen05.mma in an ELECT / BRA.U.ANY waterfall and moves operands through R2UR) or (b) by the
// whole warp in uniform control flow with `elect.sync` inside the asm (operands stay in
// uniform registers).  Descriptors are recomputed per MMA from a rotating smem offset, as in
// the production mainloops.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2403_13135_b200/csrc \
//        -o issue_probe issue_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"

__device__ __forceinline__ void umma_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_elect(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(tc::smem_u32(bar))
        : "memory");
}

template <int N, bool WARP, int M = 128>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *A = base;               // 4 slabs of 128 x 64 bf16, K-major SW128 (rotated through)
    uint8_t *B = base + 4 * 16384;   // N x 64
    __shared__ uint64_t done;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (4 * 128 + N) * 32; i += blockDim.x) reinterpret_cast<uint32_t *>(base)[i] = 0x3f803f80u;
    if (threadIdx.x == 0) {
        tc::mbar_init(&done, 1);
        tc::fence_barrier_init();
    }
    tc::fence_proxy_async_smem();
    if (warp == 0) tc::tmem_alloc<2 * N>(&tslot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tslot;
    constexpr uint32_t idesc = tc::idesc_bf16(M, N, false, false);
    const uint32_t a0 = tc::smem_u32(A), b0 = tc::smem_u32(B);
    if (warp == 1 && (WARP || lane == 0)) {
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t as = a0 + (it & 3) * 16384;  // a different slab per step
            const uint32_t d = tmem + (it & 1) * N;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t ad = tc::sw128_desc(as + 32 * k, 16, 1024), bd = tc::sw128_desc(b0 + 32 * k, 16, 1024);
                const uint32_t acc = (it > 1 || k) ? 1u : 0u;
                if (WARP) umma_elect(d, ad, bd, idesc, acc);
                else tc::umma_f16(d, ad, bd, idesc, acc);
            }
        }
        if (WARP) commit_elect(&done);
        else tc::umma_commit(&done);
        tc::mbar_wait(&done, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0 && lane == 0) *cycles = (unsigned long long)(t1 - t0);
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<2 * N>(tmem);
}

template <int N, bool WARP, int M = 128>
void run(int iters) {
    constexpr int smem = 1024 + 4 * 16384 + N * 128;
    auto k = probe<N, WARP, M>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long *dc;
    cudaMalloc(&dc, 8);
    k<<<148, 128, smem>>>(iters, dc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<148, 128, smem>>>(iters, dc);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    const double mmas = 4.0 * iters;
    const double tflops = 2.0 * M * N * 16 * mmas * 148 / (ms * 1e-3) / 1e12;
    printf("M=%3d N=%3d issue=%-11s %6.1f cycles/MMA  %7.1f TFLOP/s  %s\n", M, N, WARP ? "warp+elect" : "lane0", cyc / mmas, tflops,
           cudaGetErrorString(err));
    cudaFree(dc);
}

int main() {
    const int it = 20000;
    run<64, false>(it);
    run<64, true>(it);
    run<128, false>(it);
    run<128, true>(it);
    run<256, false>(it);
    run<256, true>(it);
    run<64, true, 64>(it);
    run<128, true, 64>(it);
    run<256, true, 64>(it);
    return 0;
}
