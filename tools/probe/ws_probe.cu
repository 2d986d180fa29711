// tcgen05.mma.ws probe (dev tool): can a 128x64x16 MMA pair that shares its B operand keep B in
// the collector buffer (.collector::b0::fill / ::lastuse) and beat the 48-cycle shared-memory
// floor of two plain N = 64 MMAs (each reads A 4 KB + B 2 KB)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2403_13135_b200/csrc -o ws_probe ws_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_common.cuh"

template <int MODE>  // 0: plain mma pairs, 1: mma.ws pairs without collector, 2: mma.ws with B fill/lastuse
__device__ __forceinline__ void mma2(uint32_t d0, uint32_t d1, uint64_t a0, uint64_t a1, uint64_t b, uint32_t idesc,
                                     uint32_t acc) {
    if (MODE == 0) {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %4, %6, p;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%1], %3, %4, %6, p;\n\t}" ::"r"(d0),
            "r"(d1), "l"(a0), "l"(a1), "l"(b), "r"(acc), "r"(idesc));
    } else if (MODE == 1) {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\t"
            "@e tcgen05.mma.ws.cta_group::1.kind::f16 [%0], %2, %4, %6, p;\n\t"
            "@e tcgen05.mma.ws.cta_group::1.kind::f16 [%1], %3, %4, %6, p;\n\t}" ::"r"(d0),
            "r"(d1), "l"(a0), "l"(a1), "l"(b), "r"(acc), "r"(idesc));
    } else {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\t"
            "@e tcgen05.mma.ws.cta_group::1.kind::f16.collector::b0::fill [%0], %2, %4, %6, p;\n\t"
            "@e tcgen05.mma.ws.cta_group::1.kind::f16.collector::b0::lastuse [%1], %3, %4, %6, p;\n\t}" ::"r"(d0),
            "r"(d1), "l"(a0), "l"(a1), "l"(b), "r"(acc), "r"(idesc));
    }
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *A = base;              // 4 slabs of 128 x 64 bf16
    uint8_t *B = base + 4 * 16384;  // 64 x 64
    __shared__ uint64_t done;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (4 * 128 + 64) * 32; i += blockDim.x) reinterpret_cast<uint32_t *>(base)[i] = 0x3f803f80u;
    if (threadIdx.x == 0) {
        tc::mbar_init(&done, 1);
        tc::fence_barrier_init();
    }
    tc::fence_proxy_async_smem();
    if (warp == 0) tc::tmem_alloc<256>(&tslot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tslot;
    constexpr uint32_t idesc = tc::idesc_bf16(128, 64, false, false);
    const uint32_t a0 = tc::smem_u32(A), b0 = tc::smem_u32(B);
    if (warp == 1) {
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t as = a0 + (it & 1) * 32768;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t ad0 = tc::sw128_desc(as + 32 * k, 16, 1024), ad1 = tc::sw128_desc(as + 16384 + 32 * k, 16, 1024);
                const uint64_t bd = tc::sw128_desc(b0 + 32 * k, 16, 1024);
                mma2<MODE>(tmem, tmem + 64, ad0, ad1, bd, idesc, (it > 0 || k) ? 1u : 0u);
            }
        }
        tc::mma_commit(&done);
        tc::mbar_wait(&done, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) *cycles = (unsigned long long)(t1 - t0);
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<256>(tmem);
}

template <int MODE>
void run(int iters) {
    constexpr int smem = 1024 + 4 * 16384 + 64 * 128;
    auto k = probe<MODE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long *dc;
    cudaMalloc(&dc, 8);
    k<<<148, 128, smem>>>(iters, dc);
    cudaError_t err = cudaDeviceSynchronize();
    k<<<148, 128, smem>>>(iters, dc);
    err = cudaDeviceSynchronize();
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %6.1f cycles per 128x64x16 MMA  %s\n", MODE,
           MODE == 0 ? "plain" : MODE == 1 ? "ws" : "ws + B collector fill/lastuse", cyc / (8.0 * iters),
           cudaGetErrorString(err));
    cudaFree(dc);
}

int main() {
    run<0>(20000);
    run<1>(20000);
    run<2>(20000);
    return 0;
}
