// unet_ops.cu -- the bandwidth-bound U-Net kernels around the tcgen05 convolutions:
// input stem (u8 -> bf16 im2col), 2x2 max-pool forward / fused backward, fused
// 1x1-head + softmax cross-entropy forward/backward, bias gradients, Dropout2d scales,
// weight-layout prep, and the fused multi-tensor Adam step.
//
// All NHWC bf16; every kernel is a single streaming pass (HBM roofline), vectorised to
// 16-byte accesses where the channel count allows.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "icelabel_b200.h"
#include "reduce.cuh"

namespace {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ float bf(uint16_t u) { return __uint_as_float((uint32_t)u << 16); }
__device__ __forceinline__ uint16_t to_bf(float f) {
    bf16 h = __float2bfloat16_rn(f);
    return *reinterpret_cast<uint16_t *>(&h);
}

inline unsigned grid_for(long long work, int per_block) {
    long long b = (work + per_block - 1) / per_block;
    if (b > 148LL * 32) b = 148LL * 32;
    if (b < 1) b = 1;
    return (unsigned)b;
}

// ---- stem: train.py:63 (u8 / 255) + im2col of the 3x3x3 first conv, K padded to 64 ----
// out[p][(r*3+s)*3 + c] = img[p + (r-1, s-1)][c] / 255 (zero outside), out[p][27..63] = 0
// 8-bit values: the bf16 of v / 255 comes from a 256-entry table built once per block (the
// same expression, so bit-identical); each warp stages its 32 pixels' 128-B rows in shared
// memory and writes them as 8 fully coalesced 512-B stores (per-lane 128-B rows would touch 32
// lines per store instruction).
__global__ void __launch_bounds__(256) stem_im2col_kernel(const uint8_t *__restrict__ img, int n, int h, int w,
                                                          uint16_t *__restrict__ out) {
    __shared__ uint16_t lut[256];
    __shared__ __align__(16) uint4 stage[8][32 * 8 + 8];  // per warp: 32 px x 128 B (+ pad)
    lut[threadIdx.x] = to_bf((float)threadIdx.x / 255.0f);
    __syncthreads();
    const long long npx = (long long)n * h * w;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint4 *st = stage[wid];
    for (long long base = (long long)blockIdx.x * blockDim.x; base < npx; base += (long long)gridDim.x * blockDim.x) {
        const long long p = base + threadIdx.x;
        if (p < npx) {
            const long long row = p / w;
            const int x = (int)(p - row * w);
            const int y = (int)(row % h);
            const long long img0 = p - (long long)y * w - x;  // first pixel of this image
            uint16_t v[32];
#pragma unroll
            for (int i = 27; i < 32; ++i) v[i] = 0;
#pragma unroll
            for (int t = 0; t < 9; ++t) {
                const int yy = y + t / 3 - 1, xx = x + t % 3 - 1;
                const bool in = yy >= 0 && yy < h && xx >= 0 && xx < w;
                const uint8_t *px = img + 3 * (img0 + (long long)yy * w + xx);
#pragma unroll
                for (int c = 0; c < 3; ++c) v[t * 3 + c] = in ? lut[px[c]] : (uint16_t)0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // 16-B chunk q of the row, chunks 4-7 are the zero pad
                uint4 u;
                u.x = v[q * 8 + 0] | ((uint32_t)v[q * 8 + 1] << 16);
                u.y = v[q * 8 + 2] | ((uint32_t)v[q * 8 + 3] << 16);
                u.z = v[q * 8 + 4] | ((uint32_t)v[q * 8 + 5] << 16);
                u.w = v[q * 8 + 6] | ((uint32_t)v[q * 8 + 7] << 16);
                st[lane * 8 + ((q + lane) & 7)] = u;  // rotate chunks: conflict-free 16-B stores
                st[lane * 8 + ((q + 4 + lane) & 7)] = make_uint4(0, 0, 0, 0);
            }
        }
        __syncwarp();
        const long long p0 = base + (wid << 5);
        uint4 *dst = reinterpret_cast<uint4 *>(out) + p0 * 8;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int idx = k * 32 + lane, px = idx >> 3, ch = idx & 7;
            if (p0 + px < npx) dst[idx] = st[px * 8 + ((ch + px) & 7)];
        }
        __syncwarp();
    }
}

// same stem from an fp32 NHWC image already scaled to [0, 1] (UNet.forward on float input)
__global__ void stem_im2col_f32_kernel(const float *__restrict__ img, int n, int h, int w, uint16_t *__restrict__ out) {
    const long long npx = (long long)n * h * w;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < npx; p += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(p % w);
        const int y = (int)((p / w) % h);
        const long long img0 = p - (long long)y * w - x;
        uint16_t v[64];
#pragma unroll
        for (int i = 27; i < 64; ++i) v[i] = 0;
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const int yy = y + t / 3 - 1, xx = x + t % 3 - 1;
            const bool in = yy >= 0 && yy < h && xx >= 0 && xx < w;
            const float *px = img + 3 * (img0 + (long long)yy * w + xx);
#pragma unroll
            for (int c = 0; c < 3; ++c) v[t * 3 + c] = in ? to_bf(px[c]) : (uint16_t)0;
        }
        uint4 *dst = reinterpret_cast<uint4 *>(out + p * 64);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            uint4 u;
            u.x = v[q * 8 + 0] | ((uint32_t)v[q * 8 + 1] << 16);
            u.y = v[q * 8 + 2] | ((uint32_t)v[q * 8 + 3] << 16);
            u.z = v[q * 8 + 4] | ((uint32_t)v[q * 8 + 5] << 16);
            u.w = v[q * 8 + 6] | ((uint32_t)v[q * 8 + 7] << 16);
            dst[q] = u;
        }
    }
}

// fp32 [rows][k] -> bf16 [rows][kp], zero padded (stem weights 64 x 27 -> 64 x 64)
__global__ void pad_weights_kernel(const float *__restrict__ src, int rows, int k, uint16_t *__restrict__ dst, int kp) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows * kp; i += gridDim.x * blockDim.x) {
        const int r = i / kp, c = i % kp;
        dst[i] = c < k ? to_bf(src[r * k + c]) : (uint16_t)0;
    }
}

// 2x2 weights [cout][2][2][c] -> 9 combined sub-pixel slabs [cout][9][c] (see conv_tc.cu)
__global__ void halve_prep_kernel(const float *__restrict__ w, int cout, int c, uint16_t *__restrict__ wc) {
    const long long total = (long long)cout * c;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long o = i / c, ci = i % c;
        const float *b = w + o * 4 * c + ci;
        const float w00 = b[0], w01 = b[c], w10 = b[2 * c], w11 = b[3 * c];
        uint16_t *d = wc + o * 9 * c + ci;
        d[0 * c] = to_bf(w00 + w01 + w10 + w11);
        d[1 * c] = to_bf(w00 + w10);
        d[2 * c] = to_bf(w01 + w11);
        d[3 * c] = to_bf(w00 + w01);
        d[4 * c] = to_bf(w10 + w11);
        d[5 * c] = to_bf(w00);
        d[6 * c] = to_bf(w01);
        d[7 * c] = to_bf(w10);
        d[8 * c] = to_bf(w11);
    }
}

// ---- max-pool 2x2 / 2 (model.py:102,125 nn.MaxPool2d(2)) ----------------------------
// 8 channels per thread (16-byte vectors)
__global__ void maxpool_fwd_kernel(const uint16_t *__restrict__ x, int n, int h, int w, int c, uint16_t *__restrict__ y) {
    // 32-bit index math (the host guarantees 4 x total < 2^31): 64-bit division made the
    // level-0 passes instruction-bound
    const int ho = h / 2, wo = w / 2, cv = c / 8;
    const int total = n * ho * wo * cv;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int cg = i % cv;
        const int p = i / cv;
        const int xo = p % wo, q = p / wo;
        const int yo = q % ho, img = q / ho;
        const uint4 *src = reinterpret_cast<const uint4 *>(x);
        const int r0 = ((img * h + 2 * yo) * w + 2 * xo) * cv + cg;
        uint4 a = src[r0], b = src[r0 + cv], cc = src[r0 + w * cv], d = src[r0 + w * cv + cv];
        const uint16_t *pa = reinterpret_cast<const uint16_t *>(&a), *pb = reinterpret_cast<const uint16_t *>(&b);
        const uint16_t *pc = reinterpret_cast<const uint16_t *>(&cc), *pd = reinterpret_cast<const uint16_t *>(&d);
        uint4 o;
        uint16_t *po = reinterpret_cast<uint16_t *>(&o);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            // first maximum in window order wins (torch CPU max_pool2d uses a strict '>')
            uint16_t best = pa[e];
            float bv = bf(best);
            if (bf(pb[e]) > bv) { best = pb[e]; bv = bf(best); }
            if (bf(pc[e]) > bv) { best = pc[e]; bv = bf(best); }
            if (bf(pd[e]) > bv) { best = pd[e]; }
            po[e] = best;
        }
        reinterpret_cast<uint4 *>(y)[i] = o;
    }
}

// dz = (add + maxpool_backward(dpool)) * drop[n][c] * [x > 0]: the fused backward of
// "ReLU -> Dropout2d -> {skip, MaxPool2d}" for a down block's output x (model.py:115-118).
// The grid-stride is a multiple of c/8, so each thread always owns the same 8 channels and
// keeps their bias-gradient partial sums (sum of dz) in registers; each block stores its
// channel sums as row blockIdx.x of bpart[blocks][c] (colsum_finish adds the rows in order).
__global__ void maxpool_bwd_kernel(const uint16_t *__restrict__ x, const uint16_t *__restrict__ dpool,
                                   const uint16_t *__restrict__ add, const float *__restrict__ drop, int n, int h, int w,
                                   int c, uint16_t *__restrict__ dz, float *__restrict__ bpart) {
    // 32-bit index math (the host guarantees 4 x total < 2^31); cv is a power of two and the
    // grid-stride a multiple of it, so the thread's channel group is fixed
    const int ho = h / 2, wo = w / 2, cv = c / 8, lcv = __ffs(cv) - 1;
    const int total = n * ho * wo * cv;
    float bsum[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int stride = gridDim.x * blockDim.x;  // multiple of cv (host)
    const int cg = (blockIdx.x * blockDim.x + threadIdx.x) & (cv - 1);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int p = i >> lcv;
        const int xo = p % wo, q = p / wo;
        const int yo = q % ho, img = q / ho;
        const int r0 = ((img * h + 2 * yo) * w + 2 * xo) * cv + cg;
        const int idx[4] = {r0, r0 + cv, r0 + w * cv, r0 + w * cv + cv};
        uint4 xv[4], av[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            xv[k] = reinterpret_cast<const uint4 *>(x)[idx[k]];
            av[k] = add ? reinterpret_cast<const uint4 *>(add)[idx[k]] : make_uint4(0, 0, 0, 0);
        }
        const uint4 g = reinterpret_cast<const uint4 *>(dpool)[i];
        const uint16_t *pg = reinterpret_cast<const uint16_t *>(&g);
        uint4 out[4];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            float v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = bf(reinterpret_cast<const uint16_t *>(&xv[k])[e]);
            int arg = 0;
            float bv = v[0];
#pragma unroll
            for (int k = 1; k < 4; ++k)
                if (v[k] > bv) { bv = v[k]; arg = k; }
            const float s = drop ? drop[img * c + cg * 8 + e] : 1.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float d = bf(reinterpret_cast<const uint16_t *>(&av[k])[e]) + (k == arg ? bf(pg[e]) : 0.f);
                d = v[k] > 0.f ? d * s : 0.f;
                bsum[e] += d;
                reinterpret_cast<uint16_t *>(&out[k])[e] = to_bf(d);
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) reinterpret_cast<uint4 *>(dz)[idx[k]] = out[k];
    }
    if (bpart) {  // block reduction per channel (thread t owns channel group t % cv)
        __shared__ float red[256 * 8];
#pragma unroll
        for (int e = 0; e < 8; ++e) red[threadIdx.x * 8 + e] = bsum[e];
        __syncthreads();
        for (int ch = threadIdx.x; ch < c; ch += blockDim.x) {
            const int cg = ch >> 3, e = ch & 7;
            float acc = 0.f;
            for (int t = cg; t < (int)blockDim.x; t += cv) acc += red[t * 8 + e];
            bpart[(size_t)blockIdx.x * c + ch] = acc;
        }
    }
}

// ---- head: out 1x1 conv 64 -> 3 (model.py:109,130) + CrossEntropyLoss (train.py:89,96) --
// One thread per pixel (64 bf16 channels = 8 x 16 B loads).  Forward: 3 logits, log-softmax
// loss, argmax hit.  Backward: dlogits = (p - onehot) * scale; dz = (dlogits W) * drop *
// [h > 0] (the ReLU/Dropout2d of up.{d-1}'s output); dW[k][c] = sum_p dlogits_k h_c via a
// per-warp smem stage (lane l owns channels 2l, 2l+1 of all 32 staged pixels), db and
// loss/hit counts via warp reductions; at the end the block's sums (warps added in order) are
// stored as row blockIdx.x of part[blocks][HEAD_LD] = [dW 192 | db 3 | dz bias 64 | loss, hits]
// and colsum_finish adds the rows in order (no atomics: bit-reproducible).  h is read and dz
// written with coalesced 16 B accesses through the same per-warp stage.
constexpr int HEAD_NT = 256;
constexpr int HC = 64;
constexpr int HEAD_COLS = 3 * HC + 3 + HC + 2, HEAD_LD = 264;

__global__ void __launch_bounds__(HEAD_NT, 4) head_ce_kernel(
    const uint16_t *__restrict__ hact, long long npx, int hw, const uint8_t *__restrict__ labels,
    const float *__restrict__ w_out, const float *__restrict__ b_out, const float *__restrict__ drop, float grad_scale,
    uint16_t *__restrict__ dz, bool train, bool zsum,
    float *__restrict__ logits_out, float *__restrict__ part) {
    __shared__ float sw[3 * HC];
    __shared__ float sdrop[HC];
    // per-warp staging of 32 pixels x 128 B (row pitch 144 B: conflict-free 16 B row reads)
    __shared__ __align__(16) uint8_t stage[HEAD_NT / 32][32 * 144];
    __shared__ float sdl[HEAD_NT / 32][32][4];  // per warp: dlogits of its 32 pixels
    for (int i = threadIdx.x; i < 3 * HC; i += HEAD_NT) sw[i] = w_out[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint8_t *wst = stage[threadIdx.x >> 5];
    long long cur_img = -1;
    float accw[6] = {0, 0, 0, 0, 0, 0};
    float accz0 = 0.f, accz1 = 0.f;  // bias gradient of the conv that produced h: sum of dz
    float accb0 = 0.f, accb1 = 0.f, accb2 = 0.f, loss_sum = 0.f, correct = 0.f;
    const float b0 = b_out[0], b1 = b_out[1], b2 = b_out[2];
    const long long stride = (long long)gridDim.x * HEAD_NT;
    for (long long base = (long long)blockIdx.x * HEAD_NT; base < npx; base += stride) {
        const long long p = base + threadIdx.x;
        const bool valid = p < npx;
        if (train && drop && hw % HEAD_NT == 0 && base / hw != cur_img) {  // block-uniform
            cur_img = base / hw;
            __syncthreads();
            if (threadIdx.x < HC) sdrop[threadIdx.x] = drop[cur_img * HC + threadIdx.x];
            __syncthreads();
        }
        // coalesced load of the warp's 32 pixels (4 KB) into smem, then each lane reads its row
        const long long p0 = base + (threadIdx.x & ~31);
        {
            const uint4 *src = reinterpret_cast<const uint4 *>(hact + p0 * HC);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = q * 32 + lane, px = idx >> 3, ch = idx & 7;
                uint4 u = p0 + px < npx ? src[idx] : make_uint4(0, 0, 0, 0);
                *reinterpret_cast<uint4 *>(wst + px * 144 + ch * 16) = u;
            }
            __syncwarp();
        }
        // the lane's activation row is read from the stage twice (logits here, the ReLU mask
        // of dz below) instead of being held in 64 registers: 4 blocks per SM instead of 2
        float l0 = b0, l1 = b1, l2 = b2;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            uint4 u = *reinterpret_cast<const uint4 *>(wst + lane * 144 + q * 16);
            const uint16_t *e = reinterpret_cast<const uint16_t *>(&u);
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const int j = q * 8 + jj;
                const float hj = bf(e[jj]);
                l0 = fmaf(sw[j], hj, l0);
                l1 = fmaf(sw[HC + j], hj, l1);
                l2 = fmaf(sw[2 * HC + j], hj, l2);
            }
        }
        float d0 = 0.f, d1 = 0.f, d2 = 0.f;
        if (valid) {
            const int y = labels[p];
            const float mx = fmaxf(l0, fmaxf(l1, l2));
            const float e0 = __expf(l0 - mx), e1 = __expf(l1 - mx), e2 = __expf(l2 - mx);
            const float se = e0 + e1 + e2;
            const float ly = y == 0 ? l0 : (y == 1 ? l1 : l2);
            loss_sum += mx + __logf(se) - ly;
            const int am = (l0 >= l1 && l0 >= l2) ? 0 : (l1 >= l2 ? 1 : 2);
            correct += am == y;
            if (logits_out) {
                logits_out[3 * p] = l0;
                logits_out[3 * p + 1] = l1;
                logits_out[3 * p + 2] = l2;
            }
            if (train) {
                const float inv = 1.f / se;
                d0 = (e0 * inv - (y == 0)) * grad_scale;
                d1 = (e1 * inv - (y == 1)) * grad_scale;
                d2 = (e2 * inv - (y == 2)) * grad_scale;
            }
        }
        if (!train) {
            __syncwarp();
            continue;
        }
        // dW[k][c] over this warp's 32 pixels: lane l owns channels 2l, 2l+1 (6 entries); the
        // pixels' h stay staged in smem, their dlogits go through a small per-warp table
        {
            float *dl = sdl[threadIdx.x >> 5][lane];
            dl[0] = d0;
            dl[1] = d1;
            dl[2] = d2;
            __syncwarp();
#pragma unroll 4
            for (int q = 0; q < 32; ++q) {
                const uint32_t hv = *reinterpret_cast<const uint32_t *>(wst + q * 144 + lane * 4);
                const float h0 = bf((uint16_t)(hv & 0xffffu)), h1 = bf((uint16_t)(hv >> 16));
                const float4 dq = *reinterpret_cast<const float4 *>(sdl[threadIdx.x >> 5][q]);
                accw[0] = fmaf(dq.x, h0, accw[0]);
                accw[1] = fmaf(dq.x, h1, accw[1]);
                accw[2] = fmaf(dq.y, h0, accw[2]);
                accw[3] = fmaf(dq.y, h1, accw[3]);
                accw[4] = fmaf(dq.z, h0, accw[4]);
                accw[5] = fmaf(dq.z, h1, accw[5]);
            }
            __syncwarp();
        }
        if (dz) {
            const long long img = p / hw;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint4 hu = *reinterpret_cast<const uint4 *>(wst + lane * 144 + q * 16);
                const uint16_t *he = reinterpret_cast<const uint16_t *>(&hu);
                uint32_t pk[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    float g[2];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int j = q * 8 + e * 2 + u;
                        float v = d0 * sw[j] + d1 * sw[HC + j] + d2 * sw[2 * HC + j];
                        if (drop) v *= hw % HEAD_NT == 0 ? sdrop[j] : __ldg(drop + img * HC + j);
                        g[u] = bf(he[e * 2 + u]) > 0.f ? v : 0.f;
                    }
                    pk[e] = (uint32_t)to_bf(g[0]) | ((uint32_t)to_bf(g[1]) << 16);
                }
                *reinterpret_cast<uint4 *>(wst + lane * 144 + q * 16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
            __syncwarp();
            if (zsum) {  // lane l sums channels 2l, 2l+1 of the 32 staged dz rows
#pragma unroll 4
                for (int q = 0; q < 32; ++q) {
                    const uint32_t zv = *reinterpret_cast<const uint32_t *>(wst + q * 144 + lane * 4);
                    accz0 += bf((uint16_t)(zv & 0xffffu));
                    accz1 += bf((uint16_t)(zv >> 16));
                }
            }
            uint4 *dst = reinterpret_cast<uint4 *>(dz + p0 * HC);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = q * 32 + lane, px = idx >> 3, ch = idx & 7;
                if (p0 + px < npx) dst[idx] = *reinterpret_cast<const uint4 *>(wst + px * 144 + ch * 16);
            }
            __syncwarp();
        }
        accb0 += d0;
        accb1 += d1;
        accb2 += d2;
    }
    for (int o = 16; o; o >>= 1) {
        loss_sum += __shfl_xor_sync(0xffffffffu, loss_sum, o);
        correct += __shfl_xor_sync(0xffffffffu, correct, o);
        accb0 += __shfl_xor_sync(0xffffffffu, accb0, o);
        accb1 += __shfl_xor_sync(0xffffffffu, accb1, o);
        accb2 += __shfl_xor_sync(0xffffffffu, accb2, o);
    }
    // per warp: its row of the block's sums (in the staging buffer, free once all warps are done)
    __syncthreads();
    float(*wsum)[HEAD_LD] = reinterpret_cast<float(*)[HEAD_LD]>(&stage[0][0]);
    static_assert(sizeof(stage) >= sizeof(float) * (HEAD_NT / 32) * HEAD_LD, "head partial rows");
    float *row = wsum[threadIdx.x >> 5];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        row[k * HC + 2 * lane] = accw[2 * k];
        row[k * HC + 2 * lane + 1] = accw[2 * k + 1];
    }
    row[3 * HC + 3 + 2 * lane] = accz0;
    row[3 * HC + 3 + 2 * lane + 1] = accz1;
    if (lane == 0) {
        row[3 * HC] = accb0;
        row[3 * HC + 1] = accb1;
        row[3 * HC + 2] = accb2;
        row[4 * HC + 3] = loss_sum;
        row[4 * HC + 4] = correct;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < HEAD_COLS; i += HEAD_NT) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < HEAD_NT / 32; ++k) s += wsum[k][i];
        part[(size_t)blockIdx.x * HEAD_LD + i] = s;
    }
}

// ---- bias gradient: db[c] += sum over rows of dz[row][c] --------------------------------
// (block sums stored as row blockIdx.x of part[blocks][c], added in order by colsum_finish)
__global__ void bias_grad_kernel(const uint16_t *__restrict__ dz, long long rows, int c, float *__restrict__ part) {
    extern __shared__ float red[];
    const int groups = c / 8;               // 16-byte vectors per row
    const int rows_per_iter = blockDim.x / groups;
    const int g = threadIdx.x % groups, r0 = threadIdx.x / groups;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (r0 < rows_per_iter) {
        for (long long r = (long long)blockIdx.x * rows_per_iter + r0; r < rows; r += (long long)gridDim.x * rows_per_iter) {
            uint4 u = reinterpret_cast<const uint4 *>(dz + r * c)[g];
            const uint16_t *e = reinterpret_cast<const uint16_t *>(&u);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += bf(e[j]);
        }
    }
    for (int j = 0; j < 8; ++j) red[threadIdx.x * 8 + j] = r0 < rows_per_iter ? acc[j] : 0.f;
    __syncthreads();
    for (int i = threadIdx.x; i < c; i += blockDim.x) {
        const int gg = i / 8, j = i % 8;
        float s = 0.f;
        for (int rr = 0; rr < rows_per_iter; ++rr) s += red[(rr * groups + gg) * 8 + j];
        part[(size_t)blockIdx.x * c + i] = s;
    }
}

// ---- Dropout2d (model.py:74-75): per (sample, channel) keep with prob 1 - p, scale 1/(1-p)
__device__ __forceinline__ uint32_t mix32(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return (uint32_t)x;
}
__global__ void dropout_scale_kernel(int count, float p, unsigned long long seed, const long long *__restrict__ step,
                                     float *__restrict__ out) {
    if (step) seed += 0x632BE59BD9B4E019ULL * (unsigned long long)(*step);  // device step counter (graph replays)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const float u = (mix32(seed * 0x9E3779B97F4A7C15ULL + (unsigned long long)i) >> 8) * (1.0f / 16777216.0f);
        out[i] = u >= p ? 1.0f / (1.0f - p) : 0.0f;
    }
}

// ---- fused Adam (torch.optim.Adam defaults, train.py:149): one pass over p, g, m, v;
// writes the bf16 working copy and zeroes the gradient for the next step ---------------
__global__ void adam_kernel(float *__restrict__ p, float *__restrict__ g, float *__restrict__ m, float *__restrict__ v,
                            long long n, float lr_corr, float omb1, float b2, float omb2, float eps, float bc2_sqrt,
                            uint16_t *__restrict__ out_bf16, const long long *__restrict__ step_dev, double lr,
                            double b1d, double b2d, bool zero_g) {
    if (step_dev) {  // bias corrections from the device step counter (CUDA-graph replays):
        __shared__ float corr[2];  // one thread per block evaluates the fp64 pows
        if (threadIdx.x == 0) {
            const double t = (double)*step_dev;
            corr[0] = (float)(lr / (1.0 - pow(b1d, t)));
            corr[1] = (float)sqrt(1.0 - pow(b2d, t));
        }
        __syncthreads();
        lr_corr = corr[0];
        bc2_sqrt = corr[1];
    }
    const long long n4 = n / 4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        float4 pp = reinterpret_cast<float4 *>(p)[i];
        float4 gg = reinterpret_cast<float4 *>(g)[i];
        float4 mm = reinterpret_cast<float4 *>(m)[i];
        float4 vv = reinterpret_cast<float4 *>(v)[i];
        float *pe = &pp.x, *ge = &gg.x, *me = &mm.x, *ve = &vv.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            me[e] = me[e] + omb1 * (ge[e] - me[e]);
            ve[e] = ve[e] * b2 + omb2 * ge[e] * ge[e];
            const float denom = sqrtf(ve[e]) / bc2_sqrt + eps;
            pe[e] = pe[e] - lr_corr * (me[e] / denom);
        }
        reinterpret_cast<float4 *>(p)[i] = pp;
        reinterpret_cast<float4 *>(m)[i] = mm;
        reinterpret_cast<float4 *>(v)[i] = vv;
        if (zero_g) reinterpret_cast<float4 *>(g)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (out_bf16) {
            uint2 o;
            o.x = (uint32_t)to_bf(pp.x) | ((uint32_t)to_bf(pp.y) << 16);
            o.y = (uint32_t)to_bf(pp.z) | ((uint32_t)to_bf(pp.w) << 16);
            reinterpret_cast<uint2 *>(out_bf16)[i] = o;
        }
    }
    // tail
    for (long long i = n4 * 4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float ge = g[i];
        const float me = m[i] + omb1 * (ge - m[i]);
        const float ve = v[i] * b2 + omb2 * ge * ge;
        const float pe = p[i] - lr_corr * (me / (sqrtf(ve) / bc2_sqrt + eps));
        m[i] = me;
        v[i] = ve;
        p[i] = pe;
        if (zero_g) g[i] = 0.f;
        if (out_bf16) out_bf16[i] = to_bf(pe);
    }
}

__global__ void cast_bf16_kernel(const float *__restrict__ src, long long n, uint16_t *__restrict__ dst) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = to_bf(src[i]);
}

__global__ void fill_f32_kernel(float *__restrict__ dst, long long n, float v) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = v;
}

}  // namespace

#define LAUNCH_CHECK() return (int)cudaGetLastError()

extern "C" int ice_stem_im2col(const uint8_t *img, int32_t n, int32_t h, int32_t w, uint16_t *out, void *stream) {
    if (!img || !out || n < 1 || h < 1 || w < 1) return ICE_EINVAL;
    stem_im2col_kernel<<<grid_for((long long)n * h * w, 256), 256, 0, (cudaStream_t)stream>>>(img, n, h, w, out);
    ice::count_launch();
    LAUNCH_CHECK();
}

extern "C" int ice_stem_im2col_f32(const float *img, int32_t n, int32_t h, int32_t w, uint16_t *out, void *stream) {
    if (!img || !out || n < 1 || h < 1 || w < 1) return ICE_EINVAL;
    stem_im2col_f32_kernel<<<grid_for((long long)n * h * w, 256), 256, 0, (cudaStream_t)stream>>>(img, n, h, w, out);
    ice::count_launch();
    LAUNCH_CHECK();
}

extern "C" int ice_pad_weights(const float *src, int32_t rows, int32_t k, uint16_t *dst, int32_t kp, void *stream) {
    if (!src || !dst || rows < 1 || k < 1 || kp < k) return ICE_EINVAL;
    pad_weights_kernel<<<grid_for((long long)rows * kp, 256), 256, 0, (cudaStream_t)stream>>>(src, rows, k, dst, kp);
    ice::count_launch();
    LAUNCH_CHECK();
}

extern "C" int ice_halve_prep(const float *w, int32_t cout, int32_t c, uint16_t *wc, void *stream) {
    if (!w || !wc || cout < 1 || c < 1) return ICE_EINVAL;
    halve_prep_kernel<<<grid_for((long long)cout * c, 256), 256, 0, (cudaStream_t)stream>>>(w, cout, c, wc);
    ice::count_launch();
    LAUNCH_CHECK();
}

extern "C" int ice_maxpool_fwd(const uint16_t *x, int32_t n, int32_t h, int32_t w, int32_t c, uint16_t *y,
                               void *stream) {
    if (!x || !y || n < 1 || h < 2 || w < 2 || (h | w) & 1 || c % 8) return ICE_EINVAL;
    if ((long long)n * h * w * (c / 8) >= (1LL << 31)) return ICE_ETOOBIG;
    maxpool_fwd_kernel<<<grid_for((long long)n * (h / 2) * (w / 2) * (c / 8), 256), 256, 0, (cudaStream_t)stream>>>(
        x, n, h, w, c, y);
    ice::count_launch();
    LAUNCH_CHECK();
}

#define ICE_SETTLE(ar)                                 \
    do {                                               \
        const int q_ = (ar).settle(scratch_bytes);     \
        if (q_) return q_ > 0 ? ICE_OK : ICE_ESCRATCH; \
    } while (0)

extern "C" int ice_maxpool_bwd(const uint16_t *x, const uint16_t *dpool, const uint16_t *add, const float *drop,
                               int32_t n, int32_t h, int32_t w, int32_t c, uint16_t *dz, float *dbias, void *scratch,
                               uint64_t *scratch_bytes, void *stream) {
    if (!x || !dpool || !dz || n < 1 || h < 2 || w < 2 || (h | w) & 1 || c % 8) return ICE_EINVAL;
    ice::Arena ar(scratch, scratch_bytes);
    const long long total = (long long)n * (h / 2) * (w / 2) * (c / 8);
    const int cv = c / 8, threads = 256;
    // grid * threads must be a multiple of cv (fixed channels per thread for the bias sums)
    if (cv > threads || threads % cv) return ICE_EINVAL;  // c <= 2048, power-of-two channel groups
    if ((long long)n * h * w * cv >= (1LL << 31)) return ICE_ETOOBIG;
    long long blocks = (total + threads - 1) / threads;
    // one wave of resident blocks (72 registers: 3 per SM, not 4 -- a 4th would run as a tail)
    static int resident = 0;
    if (!resident && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, maxpool_bwd_kernel, threads, 0) !=
                          cudaSuccess || resident < 1))
        resident = 2;
    int sms = 148;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    if (blocks > (long long)sms * resident) blocks = (long long)sms * resident;
    float *part = dbias ? ar.take<float>((size_t)blocks * c * 4) : nullptr;
    ICE_SETTLE(ar);
    cudaStream_t st = (cudaStream_t)stream;
    maxpool_bwd_kernel<<<(unsigned)blocks, threads, 0, st>>>(x, dpool, add, drop, n, h, w, c, dz, part);
    ice::count_launch();
    const int rc = (int)cudaGetLastError();
    if (rc || !dbias) return rc;
    const int ow = ice::grad_overwrite() ? 1 : 0;
    return ice::colsum_finish(part, (int)blocks, c, c, ice::ColSegs{{dbias, nullptr, nullptr, nullptr}, {c, 0, 0, 0}, {ow, 0, 0, 0}},
                              ice::RowSched{1, 1, 1, 1, 0}, st);
}

extern "C" int ice_head_ce(const uint16_t *h, int64_t npx, int32_t hw, const uint8_t *labels, const float *w_out,
                           const float *b_out, const float *drop, float grad_scale, uint16_t *dz, float *dw, float *db,
                           float *stats, float *logits, float *dzbias, void *scratch, uint64_t *scratch_bytes,
                           void *stream) {
    if (!h || !labels || !w_out || !b_out || npx < 0 || hw < 1 || ((dw == nullptr) != (db == nullptr))) return ICE_EINVAL;
    ice::Arena ar(scratch, scratch_bytes);
    unsigned blocks = grid_for(npx, HEAD_NT);
    if (blocks > 148 * 4) blocks = 148 * 4;
    const bool train = dw != nullptr, zsum = train && dz && dzbias;
    const bool need = train || stats;
    float *part = need ? ar.take<float>((size_t)blocks * HEAD_LD * 4) : nullptr;
    ICE_SETTLE(ar);
    if (npx == 0) return ICE_OK;
    cudaStream_t st = (cudaStream_t)stream;
    head_ce_kernel<<<blocks, HEAD_NT, 0, st>>>(h, npx, hw, labels, w_out, b_out, drop, grad_scale, dz, train, zsum,
                                               logits, part);
    ice::count_launch();
    const int rc = (int)cudaGetLastError();
    if (rc || !need) return rc;
    const int ow = ice::grad_overwrite() ? 1 : 0;  // gradients only: the loss statistics accumulate
    const ice::ColSegs segs{{dw, db, zsum ? dzbias : nullptr, stats}, {3 * HC, 3, HC, 2}, {ow, ow, ow, 0}};
    return ice::colsum_finish(part, (int)blocks, HEAD_LD, HEAD_COLS, segs, ice::RowSched{1, 1, 1, 1, 0}, st);
}

extern "C" int ice_bias_grad(const uint16_t *dz, int64_t rows, int32_t c, float *db, void *scratch,
                             uint64_t *scratch_bytes, void *stream) {
    if (!dz || !db || rows < 0 || c < 8 || c % 8 || c / 8 > 256) return ICE_EINVAL;
    ice::Arena ar(scratch, scratch_bytes);
    const int threads = 256;
    const int rows_per_iter = threads / (c / 8);
    unsigned blocks = grid_for(rows, rows_per_iter * 64);
    if (blocks > 148 * 4) blocks = 148 * 4;
    float *part = ar.take<float>((size_t)blocks * c * 4);
    ICE_SETTLE(ar);
    if (rows == 0) return ICE_OK;
    cudaStream_t st = (cudaStream_t)stream;
    bias_grad_kernel<<<blocks, threads, threads * 8 * sizeof(float), st>>>(dz, rows, c, part);
    ice::count_launch();
    const int rc = (int)cudaGetLastError();
    if (rc) return rc;
    const int ow = ice::grad_overwrite() ? 1 : 0;
    return ice::colsum_finish(part, (int)blocks, c, c, ice::ColSegs{{db, nullptr, nullptr, nullptr}, {c, 0, 0, 0}, {ow, 0, 0, 0}},
                              ice::RowSched{1, 1, 1, 1, 0}, st);
}

extern "C" int ice_dropout_scale(int32_t count, float p, uint64_t seed, const int64_t *step_dev, float *out,
                                 void *stream) {
    if (!out || count < 0 || p < 0.f || p >= 1.f) return ICE_EINVAL;
    if (count == 0) return ICE_OK;
    dropout_scale_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(
        count, p, seed, reinterpret_cast<const long long *>(step_dev), out);
    ice::count_launch();
    LAUNCH_CHECK();
}

extern "C" int ice_adam(float *p, float *g, float *m, float *v, int64_t n, int64_t step, const int64_t *step_dev,
                        double lr, double beta1, double beta2, double eps, int32_t zero_grad, uint16_t *out_bf16,
                        void *stream) {
    if (!p || !g || !m || !v || n < 0 || (step < 1 && !step_dev)) return ICE_EINVAL;
    if (n == 0) return ICE_OK;
    // torch.optim.Adam (_single_tensor_adam): exp_avg.lerp_(g, 1 - b1); exp_avg_sq.mul_(b2)
    // .addcmul_(g, g, value=1 - b2); step_size = lr / (1 - b1^t), denom = sqrt(v)/sqrt(1 - b2^t)
    // + eps.  The scalars are formed in double from the caller's (Python) values, then used as
    // fp32 like torch's fp32 kernels do (1 - 0.999 in double is 0.001; in fp32 from 0.999f it
    // would be 0.00099999 -- a 1.3e-5 relative bias in the second moment).
    const double t = step < 1 ? 1.0 : (double)step;
    const double bc1 = 1.0 - pow(beta1, t);
    const double bc2 = 1.0 - pow(beta2, t);
    adam_kernel<<<grid_for(n / 4 + 1, 256), 256, 0, (cudaStream_t)stream>>>(
        p, g, m, v, n, (float)(lr / bc1), (float)(1.0 - beta1), (float)beta2, (float)(1.0 - beta2), (float)eps,
        (float)sqrt(bc2), out_bf16, reinterpret_cast<const long long *>(step_dev), lr, beta1, beta2, zero_grad != 0);
    ice::count_launch();
    LAUNCH_CHECK();
}

__global__ void counter_add_kernel(long long *c, long long d) { *c += d; }

extern "C" int ice_counter_add(int64_t *counter, int64_t delta, void *stream) {
    if (!counter) return ICE_EINVAL;
    counter_add_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(reinterpret_cast<long long *>(counter), delta);
    ice::count_launch();
    LAUNCH_CHECK();
}

extern "C" int ice_cast_bf16(const float *src, int64_t n, uint16_t *dst, void *stream) {
    if (!src || !dst || n < 0) return ICE_EINVAL;
    if (n == 0) return ICE_OK;
    cast_bf16_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(src, n, dst);
    ice::count_launch();
    LAUNCH_CHECK();
}

extern "C" int ice_fill_f32(float *dst, int64_t n, float value, void *stream) {
    if (!dst || n < 0) return ICE_EINVAL;
    if (n == 0) return ICE_OK;
    fill_f32_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(dst, n, value);
    ice::count_launch();
    LAUNCH_CHECK();
}
