// reduce.cu -- the fixed-order finishers of reduce.cuh (deterministic gradient reductions).
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "reduce.cuh"

namespace ice {
namespace {

__device__ __forceinline__ bool visited(const RowSched &s, int b, int nt) {
    const int lo = nt * s.tm;
    const int hi = min(lo + s.tm, s.ntiles);
    const int t0 = lo + (((b - lo) % s.G) + s.G) % s.G;  // first tile >= lo that CTA b walks
    return t0 < hi;
}

// Block = 32 columns (lanes) x 32 row groups (warps).  Thread (g, lane) sums rows g, g + 32, ...
// of its column in order; the 32 group sums are then added in group order.  The partition
// depends only on (rows, cols), so the result is bit-identical run to run.
__global__ void __launch_bounds__(1024) colsum_kernel(const float *__restrict__ P, int rows, int ld, int cols,
                                                      ColSegs segs, RowSched sch) {
    __shared__ float red[32][33];
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int col = blockIdx.x * 32 + lane;
    float s = 0.f;
    if (col < cols) {
        const int nt = sch.bn ? col / sch.bn : 0;
#pragma unroll 4
        for (int r = g; r < rows; r += 32) {
            if (sch.bn && !visited(sch, r / sch.slots, nt)) continue;
            s += __ldcg(P + (size_t)r * ld + col);
        }
    }
    red[g][lane] = s;
    __syncthreads();
    if (g == 0 && col < cols) {
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < 32; ++k) t += red[k][lane];
        int c = col;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (c < segs.len[q]) {
                if (segs.dst[q]) segs.dst[q][c] += t;
                break;
            }
            c -= segs.len[q];
        }
    }
}

__global__ void splitsum_kernel4(const float4 *__restrict__ ws, int nsplit, size_t stride4, size_t n4,
                                 float4 *__restrict__ dst) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 a = __ldcg(ws + i);
        for (int z = 1; z < nsplit; ++z) {
            const float4 b = __ldcg(ws + z * stride4 + i);
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
        }
        float4 d = dst[i];
        d.x += a.x;
        d.y += a.y;
        d.z += a.z;
        d.w += a.w;
        dst[i] = d;
    }
}

__global__ void splitsum_kernel1(const float *__restrict__ ws, int nsplit, size_t stride, size_t n,
                                 float *__restrict__ dst) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float a = __ldcg(ws + i);
        for (int z = 1; z < nsplit; ++z) a += __ldcg(ws + z * stride + i);
        dst[i] += a;
    }
}

}  // namespace

static std::atomic<unsigned long long> g_launches{0};
void count_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

int colsum_finish(const float *P, int rows, int ld, int cols, const ColSegs &segs, const RowSched &sch,
                  cudaStream_t st) {
    if (rows <= 0 || cols <= 0) return 0;
    colsum_kernel<<<(cols + 31) / 32, 1024, 0, st>>>(P, rows, ld, cols, segs, sch);
    count_launch();
    return (int)cudaGetLastError();
}

int splitsum_finish(const float *ws, int nsplit, size_t stride, size_t n, float *dst, cudaStream_t st) {
    if (n == 0) return 0;
    const bool v4 = (stride % 4 == 0) && (n % 4 == 0) && ((reinterpret_cast<uintptr_t>(ws) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    const size_t work = v4 ? n / 4 : n;
    size_t blocks = (work + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (v4)
        splitsum_kernel4<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const float4 *>(ws), nsplit, stride / 4, n / 4,
                                                           reinterpret_cast<float4 *>(dst));
    else
        splitsum_kernel1<<<(unsigned)blocks, 256, 0, st>>>(ws, nsplit, stride, n, dst);
    count_launch();
    return (int)cudaGetLastError();
}

}  // namespace ice

// Kernels this library has launched in this process (every launch site counts itself): the
// evidence bench.py reports as gpu_launches.
extern "C" uint64_t ice_kernel_launches(void) { return ice::g_launches.load(std::memory_order_relaxed); }
