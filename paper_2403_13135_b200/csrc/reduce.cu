// reduce.cu -- the fixed-order finishers of reduce.cuh (deterministic gradient reductions).
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "reduce.cuh"

namespace ice {
namespace {

// Block = 32 columns (lanes) x 32 row groups (warps).  Thread (g, lane) sums rows k = g,
// g + 32, ... of its column in order; the 32 group sums are then added in group order.  The
// partition depends only on the shapes, so the result is bit-identical run to run.
__global__ void __launch_bounds__(1024) colsum_kernel(const float *__restrict__ P, int rows, int ld, int cols,
                                                      ColSegs segs, RowSched sch) {
    __shared__ float red[32][33];
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int col = blockIdx.x * 32 + lane;
    float s = 0.f;
    if (col < cols) {
        int count = rows, r0 = 0, G = rows;
        if (sch.bn) {  // the CTAs that visited this column's tile column, in cyclic order
            const int lo = (col / sch.bn) * sch.tm;
            const int hi = min(lo + sch.tm, sch.ntiles);
            G = sch.G;
            count = min(G, hi - lo);
            r0 = lo % G;
        }
        const float *p = P + col;
#pragma unroll 4
        for (int k = g; k < count; k += 32) {
            int r = r0 + k;
            if (r >= G) r -= G;
            s += __ldcg(p + (size_t)r * ld);
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

// few slices: one thread per float4, the slices' loads issued together, added in order
template <int MAXZ>
__global__ void splitsum_kernel4(const float4 *__restrict__ ws, int nsplit, size_t stride4, size_t n4,
                                 float4 *__restrict__ dst) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 v[MAXZ];
#pragma unroll
        for (int z = 0; z < MAXZ; ++z)
            if (z < nsplit) v[z] = __ldcg(ws + z * stride4 + i);
        float4 a = v[0];
#pragma unroll
        for (int z = 1; z < MAXZ; ++z)
            if (z < nsplit) {
                a.x += v[z].x;
                a.y += v[z].y;
                a.z += v[z].z;
                a.w += v[z].w;
            }
        float4 d = dst[i];
        d.x += a.x;
        d.y += a.y;
        d.z += a.z;
        d.w += a.w;
        dst[i] = d;
    }
}

// many slices (the halo weight gradients split pixels 50-150 ways): block = 32 float4 columns
// x 32 slice groups; thread (g, lane) adds slices g, g + 32, ... in order, then the group sums
// are added in group order
__global__ void __launch_bounds__(1024) splitsum_wide_kernel(const float4 *__restrict__ ws, int nsplit,
                                                             size_t stride4, size_t n4, float4 *__restrict__ dst) {
    __shared__ float4 red[32][33];
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    const size_t i = blockIdx.x * (size_t)32 + lane;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < n4) {
#pragma unroll 4
        for (int z = g; z < nsplit; z += 32) {
            const float4 b = __ldcg(ws + z * stride4 + i);
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
        }
    }
    red[g][lane] = a;
    __syncthreads();
    if (g == 0 && i < n4) {
        float4 t = red[0][lane];
        for (int k = 1; k < 32; ++k) {
            const float4 b = red[k][lane];
            t.x += b.x;
            t.y += b.y;
            t.z += b.z;
            t.w += b.w;
        }
        float4 d = dst[i];
        d.x += t.x;
        d.y += t.y;
        d.z += t.z;
        d.w += t.w;
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
    if (n == 0 || nsplit <= 0) return 0;
    const bool v4 = (stride % 4 == 0) && (n % 4 == 0) && ((reinterpret_cast<uintptr_t>(ws) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    auto grid = [](size_t work) {
        size_t b = (work + 255) / 256;
        return (unsigned)(b > 148 * 16 ? 148 * 16 : b);
    };
    const float4 *w4 = reinterpret_cast<const float4 *>(ws);
    float4 *d4 = reinterpret_cast<float4 *>(dst);
    if (!v4)
        splitsum_kernel1<<<grid(n), 256, 0, st>>>(ws, nsplit, stride, n, dst);
    else if (nsplit <= 4)
        splitsum_kernel4<4><<<grid(n / 4), 256, 0, st>>>(w4, nsplit, stride / 4, n / 4, d4);
    else if (nsplit <= 16)
        splitsum_kernel4<16><<<grid(n / 4), 256, 0, st>>>(w4, nsplit, stride / 4, n / 4, d4);
    else
        splitsum_wide_kernel<<<(unsigned)((n / 4 + 31) / 32), 1024, 0, st>>>(w4, nsplit, stride / 4, n / 4, d4);
    count_launch();
    return (int)cudaGetLastError();
}

}  // namespace ice

// Kernels this library has launched in this process (every launch site counts itself): the
// evidence bench.py reports as gpu_launches.
extern "C" uint64_t ice_kernel_launches(void) { return ice::g_launches.load(std::memory_order_relaxed); }
