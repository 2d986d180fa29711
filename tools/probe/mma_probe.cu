// tcgen05 MMA throughput probe (dev tool): SS-mode bf16 MMA chains with operands resident in
// shared memory, cta_group::1 (M = 128) vs cta_group::2 (M = 256 / 128 over a CTA pair), for
// N = 64 / 128 / 256.  Answers: is an N = 64 tile capped by shared-memory operand bandwidth,
// and does a CTA pair lift the cap?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2403_13135_b200/csrc \
//        -o mma_probe mma_probe.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "tc_common.cuh"

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int CG, int M, int N, int NACC>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int MA = M / CG;   // A rows held by this CTA
    constexpr int NB = N / CG;   // B rows held by this CTA
    uint8_t *A = base;                   // MA x 64 bf16, K-major SW128
    uint8_t *B = base + MA * 128;        // NB x 64 bf16
    __shared__ uint64_t done;
    __shared__ uint32_t tslot;
    for (int i = threadIdx.x; i < (MA + NB) * 32; i += blockDim.x) reinterpret_cast<uint32_t *>(base)[i] = 0x3f803f80u;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        tc::mbar_init(&done, 1);
        tc::fence_barrier_init();
    }
    tc::fence_proxy_async_smem();
    constexpr int NC = N * NACC;
    constexpr int COLS = NC <= 32 ? 32 : (NC <= 64 ? 64 : (NC <= 128 ? 128 : (NC <= 256 ? 256 : 512)));
    if (warp == 0) {
        if (CG == 1) tc::tmem_alloc<COLS>(&tslot);
        else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tslot)), "n"(COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem = tslot;
    const bool leader = CG == 1 || cluster_rank() == 0;
    if (warp == 1 && leader && (threadIdx.x & 31) == 0) {
        constexpr uint32_t idesc = tc::idesc_bf16(M, N, false, false);
        const uint32_t a0 = tc::smem_u32(A), b0 = tc::smem_u32(B);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t ad = tc::sw128_desc(a0 + 32 * k, 16, 1024), bd = tc::sw128_desc(b0 + 32 * k, 16, 1024);
                const uint32_t acc = (it | k) ? 1u : 0u;
#pragma unroll
                for (int q = 0; q < NACC; ++q) {  // independent accumulators, interleaved
                    const uint32_t d = tmem + q * N;
                    if (CG == 1) tc::umma_f16(d, ad, bd, idesc, acc);
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                                     "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                }
            }
        }
        if (CG == 1) tc::umma_commit(&done);
        else
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                             tc::smem_u32(&done)), "h"((uint16_t)3) : "memory");
        tc::mbar_wait(&done, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
    } else if (warp == 1 && (threadIdx.x & 31) == 0) {
        tc::mbar_wait(&done, 0);  // the peer waits for the multicast commit
    }
    tc::tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();
    if (warp == 0) {
        if (CG == 1) tc::tmem_dealloc<COLS>(tmem);
        else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(COLS));
    }
}

template <int CG, int M, int N, int NACC = 1>
void run(int iters) {
    constexpr int smem = 1024 + (M / CG + N / CG) * 128;
    auto k = probe<CG, M, N, NACC>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long *dc;
    cudaMalloc(&dc, 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, iters, dc);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k, iters, dc);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    const double macs_per_cta = (double)(M / CG) * N * 64 * iters * NACC;  // this CTA's rows
    const double tflops = 2.0 * macs_per_cta * 148 / (ms * 1e-3) / 1e12;
    const double mac_per_cyc = macs_per_cta / (double)cyc;
    printf("cg=%d M=%3d N=%3d acc=%d smem/MMA/SM=%5d B: %8.3f ms  %7.1f TFLOP/s  %6.0f MAC/cyc/SM  %s\n", CG, M, N, NACC,
           (M / CG + N / CG) * 32, ms, tflops, mac_per_cyc, cudaGetErrorString(err));
    cudaFree(dc);
}

int main() {
    const int it = 20000;
    run<1, 128, 64>(it);
    run<1, 128, 128>(it);
    run<1, 128, 256>(it);
    run<2, 256, 64>(it);
    run<2, 256, 128>(it);
    run<2, 256, 256>(it);
    run<2, 128, 256>(it);
    run<2, 128, 128>(it);
    run<1, 128, 64, 2>(it);
    run<1, 128, 64, 4>(it);
    run<2, 256, 64, 2>(it);
    run<1, 128, 32, 4>(it);
    return 0;
}
