// data_ops.cu -- the GPU-resident data path around the two hot paths:
// scene cutting / stitching (icetrain/data.py:55-80), the label colour codec
// (data.py:35-52), the inference head with fused argmax (infer.py:38-51) and the
// confusion matrix (icelabel/metrics.py:108-113).  All HBM-bound byte work: grid-stride
// loops sized in multiples of the SM count, 16-byte accesses where the layout allows.
#include <cuda_runtime.h>
#include <stdint.h>

#include "icelabel_b200.h"
#include "reduce.cuh"

namespace {

constexpr int NT = 256;

unsigned grid_for(long long work) {
    long long b = (work + NT - 1) / NT;
    const long long cap = 148LL * 32;
    return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}

__device__ __forceinline__ float bf(uint16_t v) { return __uint_as_float((uint32_t)v << 16); }

// tiles[t][i][j][c] = img[r*S + i][q*S + j][c] (t = r*cols + q), zero outside the image
__global__ void cut_kernel(const uint8_t *__restrict__ img, int h, int w, int c, int S, int cols, long long total,
                           uint8_t *__restrict__ tiles) {
    for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total; o += (long long)gridDim.x * blockDim.x) {
        const int ch = (int)(o % c);
        long long p = o / c;
        const int j = (int)(p % S);
        p /= S;
        const int i = (int)(p % S);
        const long long t = p / S;
        const int y = (int)(t / cols) * S + i, x = (int)(t % cols) * S + j;
        tiles[o] = (y < h && x < w) ? img[((long long)y * w + x) * c + ch] : 0;
    }
}

// out[y][x][c] = tiles[(y/S)*cols + x/S][y%S][x%S][c] for y < h, x < w (padding cropped)
__global__ void stitch_kernel(const uint8_t *__restrict__ tiles, int cols, int S, int c, int h, int w,
                              uint8_t *__restrict__ out) {
    const long long total = (long long)h * w * c;
    for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total; o += (long long)gridDim.x * blockDim.x) {
        const int ch = (int)(o % c);
        const long long p = o / c;
        const int y = (int)(p / w), x = (int)(p % w);
        const long long t = (long long)(y / S) * cols + x / S;
        out[o] = tiles[((t * S + y % S) * S + x % S) * c + ch];
    }
}

// class index -> RGB colour; first out-of-range index reported (encode_labels raises)
__global__ void encode_kernel(const uint8_t *__restrict__ mask, long long npx, const uint8_t *__restrict__ colors,
                              int ncls, uint8_t *__restrict__ rgb, unsigned long long *__restrict__ first_bad) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < npx; p += (long long)gridDim.x * blockDim.x) {
        const int k = mask[p];
        if (k >= ncls) {
            atomicMin(first_bad, (unsigned long long)p);
            continue;
        }
        rgb[3 * p] = colors[3 * k];
        rgb[3 * p + 1] = colors[3 * k + 1];
        rgb[3 * p + 2] = colors[3 * k + 2];
    }
}

// RGB colour -> class index (decode_labels); unknown colours -> 255 and the first one's index
__global__ void decode_kernel(const uint8_t *__restrict__ rgb, long long npx, const uint8_t *__restrict__ colors,
                              int ncls, uint8_t *__restrict__ mask, unsigned long long *__restrict__ first_bad) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < npx; p += (long long)gridDim.x * blockDim.x) {
        const uint8_t r = rgb[3 * p], g = rgb[3 * p + 1], b = rgb[3 * p + 2];
        int k = 255;
        for (int i = ncls - 1; i >= 0; --i)  // decode_labels assigns in class order: the last match wins
            if (r == colors[3 * i] && g == colors[3 * i + 1] && b == colors[3 * i + 2]) {
                k = i;
                break;
            }
        mask[p] = (uint8_t)k;
        if (k == 255) atomicMin(first_bad, (unsigned long long)p);
    }
}

// out 1x1 conv 64 -> 3 on the last activation + argmax (first maximum, as torch.argmax)
constexpr int HC = 64;
__global__ void __launch_bounds__(NT) head_argmax_kernel(const uint16_t *__restrict__ hact, long long npx,
                                                         const float *__restrict__ w_out,
                                                         const float *__restrict__ b_out, uint8_t *__restrict__ out) {
    __shared__ float sw[3 * HC];
    for (int i = threadIdx.x; i < 3 * HC; i += NT) sw[i] = w_out[i];
    __syncthreads();
    const float b0 = b_out[0], b1 = b_out[1], b2 = b_out[2];
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < npx; p += (long long)gridDim.x * blockDim.x) {
        const uint4 *src = reinterpret_cast<const uint4 *>(hact + p * HC);
        float l0 = b0, l1 = b1, l2 = b2;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint4 u = __ldg(src + q);
            const uint32_t wv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = q * 8 + 2 * e;
                const float h0 = bf((uint16_t)(wv[e] & 0xffffu)), h1 = bf((uint16_t)(wv[e] >> 16));
                l0 = fmaf(sw[j], h0, fmaf(sw[j + 1], h1, l0));
                l1 = fmaf(sw[HC + j], h0, fmaf(sw[HC + j + 1], h1, l1));
                l2 = fmaf(sw[2 * HC + j], h0, fmaf(sw[2 * HC + j + 1], h1, l2));
            }
        }
        out[p] = (l0 >= l1 && l0 >= l2) ? 0 : (l1 >= l2 ? 1 : 2);
    }
}

// counts[pred][ref] (metrics.py:108-113); pixels with a label >= k are counted in bad
__global__ void confusion_kernel(const uint8_t *__restrict__ pred, const uint8_t *__restrict__ ref, long long npx,
                                 int k, unsigned long long *__restrict__ counts, unsigned long long *__restrict__ bad) {
    __shared__ unsigned int h[17];
    for (int i = threadIdx.x; i < 17; i += NT) h[i] = 0;
    __syncthreads();
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < npx; p += (long long)gridDim.x * blockDim.x) {
        const int a = pred[p], b = ref[p];
        const int bin = (a < k && b < k) ? a * k + b : 16;
        const unsigned act = __activemask();
        const unsigned peers = __match_any_sync(act, bin);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[bin], __popc(peers));
    }
    __syncthreads();
    if (threadIdx.x < k * k && h[threadIdx.x]) atomicAdd(&counts[threadIdx.x], (unsigned long long)h[threadIdx.x]);
    if (threadIdx.x == 16 && h[16]) atomicAdd(bad, (unsigned long long)h[16]);
}

}  // namespace

extern "C" int ice_cut_tiles(const uint8_t *img, int32_t h, int32_t w, int32_t c, int32_t size, uint8_t *tiles,
                             void *stream) {
    if (!img || !tiles || h < 1 || w < 1 || c < 1 || size < 1) return ICE_EINVAL;
    const int rows = (h + size - 1) / size, cols = (w + size - 1) / size;
    const long long total = (long long)rows * cols * size * size * c;
    cut_kernel<<<grid_for(total), NT, 0, (cudaStream_t)stream>>>(img, h, w, c, size, cols, total, tiles);
    ice::count_launch();
    return (int)cudaGetLastError();
}

extern "C" int ice_stitch_tiles(const uint8_t *tiles, int32_t cols, int32_t size, int32_t c, int32_t h, int32_t w,
                                uint8_t *out, void *stream) {
    if (!tiles || !out || h < 1 || w < 1 || c < 1 || size < 1) return ICE_EINVAL;
    if (cols <= 0) cols = (w + size - 1) / size;
    if ((long long)cols * size < w) return ICE_EINVAL;
    stitch_kernel<<<grid_for((long long)h * w * c), NT, 0, (cudaStream_t)stream>>>(tiles, cols, size, c, h, w, out);
    ice::count_launch();
    return (int)cudaGetLastError();
}

extern "C" int ice_encode_labels(const uint8_t *mask, int64_t npx, const uint8_t *colors, int32_t ncls, uint8_t *rgb,
                                 uint64_t *first_bad, void *stream) {
    if (npx < 0 || ncls < 1 || ncls > 255 || (npx > 0 && (!mask || !colors || !rgb || !first_bad))) return ICE_EINVAL;
    if (npx == 0) return ICE_OK;
    encode_kernel<<<grid_for(npx), NT, 0, (cudaStream_t)stream>>>(mask, npx, colors, ncls, rgb,
                                                                  reinterpret_cast<unsigned long long *>(first_bad));
    ice::count_launch();
    return (int)cudaGetLastError();
}

extern "C" int ice_decode_labels(const uint8_t *rgb, int64_t npx, const uint8_t *colors, int32_t ncls, uint8_t *mask,
                                 uint64_t *first_bad, void *stream) {
    if (npx < 0 || ncls < 1 || ncls > 255 || (npx > 0 && (!mask || !colors || !rgb || !first_bad))) return ICE_EINVAL;
    if (npx == 0) return ICE_OK;
    decode_kernel<<<grid_for(npx), NT, 0, (cudaStream_t)stream>>>(rgb, npx, colors, ncls, mask,
                                                                  reinterpret_cast<unsigned long long *>(first_bad));
    ice::count_launch();
    return (int)cudaGetLastError();
}

extern "C" int ice_head_argmax(const uint16_t *h, int64_t npx, const float *w_out, const float *b_out, uint8_t *mask,
                               void *stream) {
    if (npx < 0 || (npx > 0 && (!h || !w_out || !b_out || !mask))) return ICE_EINVAL;
    if (npx == 0) return ICE_OK;
    head_argmax_kernel<<<grid_for(npx), NT, 0, (cudaStream_t)stream>>>(h, npx, w_out, b_out, mask);
    ice::count_launch();
    return (int)cudaGetLastError();
}

extern "C" int ice_confusion(const uint8_t *pred, const uint8_t *ref, int64_t npx, int32_t k, uint64_t *counts,
                             uint64_t *bad, void *stream) {
    if (npx < 0 || k < 1 || k > 4 || (npx > 0 && (!pred || !ref || !counts || !bad))) return ICE_EINVAL;
    if (npx == 0) return ICE_OK;
    confusion_kernel<<<grid_for(npx), NT, 0, (cudaStream_t)stream>>>(
        pred, ref, npx, k, reinterpret_cast<unsigned long long *>(counts), reinterpret_cast<unsigned long long *>(bad));
    ice::count_launch();
    return (int)cudaGetLastError();
}
