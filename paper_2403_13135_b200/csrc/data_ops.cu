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

// parse_labels(snap=True) (segmentation.py:140-157): nearest colormap colour in squared RGB
// distance, ties to the earlier class (argmin keeps the first minimum)
__global__ void snap_kernel(const uint8_t *__restrict__ rgb, long long npx, const uint8_t *__restrict__ colors,
                            int ncls, uint8_t *__restrict__ mask) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < npx; p += (long long)gridDim.x * blockDim.x) {
        const int r = rgb[3 * p], g = rgb[3 * p + 1], b = rgb[3 * p + 2];
        int best = 0, bd = 0x7fffffff;
        for (int i = 0; i < ncls; ++i) {
            const int dr = r - colors[3 * i], dg = g - colors[3 * i + 1], db = b - colors[3 * i + 2];
            const int d = dr * dr + dg * dg + db * db;
            if (d < bd) {
                bd = d;
                best = i;
            }
        }
        mask[p] = (uint8_t)best;
    }
}

// ---- SSIM (icelabel/metrics.py:145-172): single-scale, 11 x 11 Gaussian window (sigma 1.5),
// "valid" positions, per channel mean of num / den, float64 like the reference.  Block =
// SSIM_TX x SSIM_TY valid output positions of one channel: the (TX + 10) x (TY + 10) input
// patches of both images are staged in shared memory, each thread forms the five windowed
// moments of its position with the 121 weights (host-computed in float64, as numpy does), and
// the block's sum of num/den goes to part[blockIdx] (fixed-order finish: deterministic).
constexpr int SSIM_K = 11, SSIM_TX = 32, SSIM_TY = 8;
__constant__ double c_ssim_w[SSIM_K * SSIM_K];

__global__ void __launch_bounds__(SSIM_TX * SSIM_TY) ssim_kernel(const uint8_t *__restrict__ a,
                                                                 const uint8_t *__restrict__ b, int h, int w,
                                                                 double c1, double c2, double *__restrict__ part) {
    __shared__ double sa[SSIM_TY + SSIM_K - 1][SSIM_TX + SSIM_K - 1];
    __shared__ double sb[SSIM_TY + SSIM_K - 1][SSIM_TX + SSIM_K - 1];
    __shared__ double red[SSIM_TX * SSIM_TY / 32];
    const int ch = blockIdx.z;
    const int x0 = blockIdx.x * SSIM_TX, y0 = blockIdx.y * SSIM_TY;
    const int vw = w - SSIM_K + 1, vh = h - SSIM_K + 1;  // valid output extent
    for (int i = threadIdx.x; i < (SSIM_TY + SSIM_K - 1) * (SSIM_TX + SSIM_K - 1); i += blockDim.x) {
        const int yy = i / (SSIM_TX + SSIM_K - 1), xx = i % (SSIM_TX + SSIM_K - 1);
        const int gy = min(y0 + yy, h - 1), gx = min(x0 + xx, w - 1);
        const size_t o = ((size_t)gy * w + gx) * 3 + ch;
        sa[yy][xx] = (double)a[o];
        sb[yy][xx] = (double)b[o];
    }
    __syncthreads();
    const int tx = threadIdx.x % SSIM_TX, ty = threadIdx.x / SSIM_TX;
    double v = 0.0;
    if (x0 + tx < vw && y0 + ty < vh) {
        double mx = 0, my = 0, xx2 = 0, yy2 = 0, xy = 0;
        for (int i = 0; i < SSIM_K; ++i)
#pragma unroll
            for (int j = 0; j < SSIM_K; ++j) {
                const double k = c_ssim_w[i * SSIM_K + j];
                const double p = sa[ty + i][tx + j], q = sb[ty + i][tx + j];
                mx += k * p;
                my += k * q;
                xx2 += k * (p * p);
                yy2 += k * (q * q);
                xy += k * (p * q);
            }
        const double vx = xx2 - mx * mx, vy = yy2 - my * my, cov = xy - mx * my;
        const double num = (2 * mx * my + c1) * (2 * cov + c2);
        const double den = (mx * mx + my * my + c1) * (vx + vy + c2);
        v = num / den;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < SSIM_TX * SSIM_TY / 32; ++k) t += red[k];
        part[((size_t)ch * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
}

// per channel: sum of the block partials in block order
__global__ void ssim_finish(const double *__restrict__ part, int blocks_per_ch, double *__restrict__ sums) {
    __shared__ double red[256];
    const int ch = blockIdx.x;
    double t = 0.0;
    for (int i = threadIdx.x; i < blocks_per_ch; i += 256) t += part[(size_t)ch * blocks_per_ch + i];
    red[threadIdx.x] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int k = 0; k < 256; ++k) s += red[k];
        sums[ch] = s;
    }
}

}  // namespace

extern "C" int ice_snap_labels(const uint8_t *rgb, int64_t npx, const uint8_t *colors, int32_t ncls, uint8_t *mask,
                               void *stream) {
    if (npx < 0 || ncls < 1 || ncls > 255 || (npx > 0 && (!mask || !colors || !rgb))) return ICE_EINVAL;
    if (npx == 0) return ICE_OK;
    snap_kernel<<<grid_for(npx), NT, 0, (cudaStream_t)stream>>>(rgb, npx, colors, ncls, mask);
    ice::count_launch();
    return (int)cudaGetLastError();
}

extern "C" int ice_ssim(const uint8_t *a, const uint8_t *b, int32_t h, int32_t w, const double *window, double c1,
                        double c2, double *sums, void *scratch, uint64_t *scratch_bytes, void *stream) {
    if (!a || !b || !window || !sums || h < SSIM_K || w < SSIM_K) return ICE_EINVAL;
    ice::Arena ar(scratch, scratch_bytes);
    const dim3 grid((w - SSIM_K + 1 + SSIM_TX - 1) / SSIM_TX, (h - SSIM_K + 1 + SSIM_TY - 1) / SSIM_TY, 3);
    const int per_ch = (int)(grid.x * grid.y);
    double *part = ar.take<double>((size_t)3 * per_ch * 8);
    const int q = ar.settle(scratch_bytes);
    if (q) return q > 0 ? ICE_OK : ICE_ESCRATCH;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyToSymbolAsync(c_ssim_w, window, sizeof(double) * SSIM_K * SSIM_K, 0,
                                            cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return (int)e;
    ssim_kernel<<<grid, SSIM_TX * SSIM_TY, 0, st>>>(a, b, h, w, c1, c2, part);
    ice::count_launch();
    ssim_finish<<<3, 256, 0, st>>>(part, per_ch, sums);
    ice::count_launch();
    return (int)cudaGetLastError();
}

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
