// stem.cu -- the U-Net's first convolution (down.0.block.0: 3 -> 64 channels, 3 x 3,
// model.py:64-76 with the input scaling of train.py:63, x = u8 / 255) straight from the u8
// NHWC images, forward and weight gradient, without an im2col buffer.
//
// With K = 27 (3 x 3 taps x 3 channels) the stem is HBM-bound, not MMA-bound: the forward
// writes 128 B of bf16 activations per pixel and the weight gradient reads 128 B of dZ per
// pixel, against 2 x 27 x 64 MACs.  The im2col path it replaces wrote a 128-B bf16 column per
// pixel, read it back in the forward GEMM and again in the weight gradient (3 x 268 MB at
// batch 32, 256^2).  Here the 27-tap columns are gathered from the 3-byte pixels (L1/L2
// resident: 6.3 MB per batch) straight into mma.sync fragments (m16n8k16, bf16 in, fp32
// accumulate; K padded to 32 with zeros), so each pass moves only its unavoidable bytes.
// The legacy tensor path (HMMA, ~550 TFLOP/s measured on B200) does the 8.6 GFLOP of a batch
// in ~16 us, well under the ~41 us of HBM traffic.
//
// Numerics: the bf16 of v / 255 comes from the same table as ice_stem_im2col (bit-identical
// inputs); products accumulate in fp32.  The forward epilogue is the conv epilogue's: bias add
// in fp32, ReLU, RN bf16 rounding, and the packed ReLU mask computed from the stored bf16.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "icelabel_b200.h"
#include "reduce.cuh"

namespace {

constexpr int SNT = 256;       // threads per CTA (8 warps)

__device__ __forceinline__ uint16_t bf_bits(float f) {
    __nv_bfloat16 b = __float2bfloat16_rn(f);
    return *reinterpret_cast<uint16_t *>(&b);
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ uint32_t pos_bits2(uint32_t w) {  // bf16 pair -> (lo > 0) | (hi > 0) << 1
    const uint32_t lo = w & 0xffffu, hi = w >> 16;
    return (uint32_t)((lo & 0x7fffu) != 0 && !(lo & 0x8000u)) | ((uint32_t)((hi & 0x7fffu) != 0 && !(hi & 0x8000u)) << 1);
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// ---- the stem's im2col row of one pixel, built by one lane --------------------------------
// Column k = tap * 3 + c (tap = (dy + 1) * 3 + dx + 1) of pixel p = bf16(img[p + (dy, dx)][c] /
// 255), zero outside the image and for k >= 27 (the ice_stem_im2col order).  The lane writes
// its 32 columns (64 B) as one row of a per-warp [32 px][CT_PITCH] bf16 tile in shared memory.
constexpr int CT_PITCH = 40;  // bf16 per tile row (80 B: conflict-free ldmatrix row sets)

struct Geo {
    int n, h, w, lw, lh;  // lw / lh: log2 of w / h, or -1 when not a power of two
    int npx;
};
__device__ __forceinline__ void decode(const Geo &G, int p, int &y, int &x) {
    int row;
    if (G.lw >= 0) {
        row = p >> G.lw;
        x = p & (G.w - 1);
    } else {
        row = p / G.w;
        x = p - row * G.w;
    }
    y = G.lh >= 0 ? (row & (G.h - 1)) : row % G.h;
}
__device__ __forceinline__ void build_col_row(const uint8_t *__restrict__ img, const uint16_t *lut, const Geo &G,
                                              int p, uint16_t *dst) {
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0;
    if (p < G.npx) {
        int y, x;
        decode(G, p, y, x);
        const uint8_t *px = img + 3 * (size_t)p;
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy) {
            const bool vy = (unsigned)(y + dy) < (unsigned)G.h;
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx) {
                const bool ok = vy && (unsigned)(x + dx) < (unsigned)G.w;
                const uint8_t *q = px + (dy * G.w + dx) * 3;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int k = ((dy + 1) * 3 + dx + 1) * 3 + c;
                    const uint32_t b = ok ? (uint32_t)lut[__ldg(q + c)] : 0u;
                    v[k >> 1] |= b << (16 * (k & 1));
                }
            }
        }
    }
    uint4 *d = reinterpret_cast<uint4 *>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q) d[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void *row_addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"((uint32_t)__cvta_generic_to_shared(row_addr)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void *row_addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"((uint32_t)__cvta_generic_to_shared(row_addr)));
}

// ---- forward: y = ReLU(conv(x) + b) (bf16 NHWC, 64 channels) + packed ReLU mask ----------
// Per warp step: 32 consecutive pixels.  Lane j builds pixel p0 + j's im2col row in the warp's
// column tile; A fragments (M = pixels, K = columns) come by ldmatrix; B (the weights, 8 n8
// tiles x 2 k16 steps) stays in registers.  The accumulators go through the same tile memory
// (as a [32 px][64 ch] bf16 row stage) so the 128-B output rows leave as coalesced 512-B
// stores, and each lane derives its pixel's two ReLU-mask words from its staged row.
constexpr int YW = 36;  // staged output row pitch in 32-bit words

__global__ void __launch_bounds__(SNT, 2) stem_fprop_kernel(const uint8_t *__restrict__ img, Geo G,
                                                            const uint16_t *__restrict__ wt, const float *__restrict__ bias,
                                                            uint16_t *__restrict__ y, uint32_t *__restrict__ rbits) {
    __shared__ uint16_t lut[256];
    __shared__ float sbias[64];
    __shared__ __align__(16) uint32_t stage[SNT / 32][32 * YW];  // col tile (32 x 40 bf16) / output stage
    lut[threadIdx.x] = bf_bits((float)threadIdx.x / 255.0f);
    if (threadIdx.x < 64) sbias[threadIdx.x] = bias ? bias[threadIdx.x] : 0.f;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
    // B fragments: b0 = W[co][16 ks + 2t .. +1], b1 = W[co][16 ks + 2t + 8 .. +9], co = 8 nt + g
    uint32_t bw[8][2][2];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            const uint32_t *r = reinterpret_cast<const uint32_t *>(wt + (8 * nt + g) * 64 + 16 * ks + 2 * t);
            bw[nt][ks][0] = __ldg(r);
            bw[nt][ks][1] = __ldg(r + 4);
        }
    __syncthreads();
    uint32_t *st = stage[wid];
    uint16_t *tile = reinterpret_cast<uint16_t *>(st);
    const int groups = (G.npx + 31) / 32;
    for (int gi = blockIdx.x * (SNT / 32) + wid; gi < groups; gi += gridDim.x * (SNT / 32)) {
        const int p0 = gi * 32;
        __syncwarp();
        build_col_row(img, lut, G, p0 + lane, tile + lane * CT_PITCH);
        __syncwarp();
        float acc[2][8][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = acc[mt][nt][2] = acc[mt][nt][3] = 0.f;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                uint32_t a[4];  // rows 16 mt + (lane & 15), columns 16 ks + 8 (lane >> 4)
                ldsm_x4(a, tile + (16 * mt + (lane & 15)) * CT_PITCH + 16 * ks + 8 * (lane >> 4));
#pragma unroll
                for (int nt = 0; nt < 8; ++nt) mma16816(acc[mt][nt], a, bw[nt][ks][0], bw[nt][ks][1]);
            }
        }
        // epilogue: bias, ReLU, bf16 -> stage row r = pixel p0 + r, word 4 nt + t = channels 8 nt + 2t, +1
        __syncwarp();
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                const float b0 = sbias[8 * nt + 2 * t], b1 = sbias[8 * nt + 2 * t + 1];
                st[(16 * mt + g) * YW + 4 * nt + t] =
                    pack2(fmaxf(acc[mt][nt][0] + b0, 0.f), fmaxf(acc[mt][nt][1] + b1, 0.f));
                st[(16 * mt + g + 8) * YW + 4 * nt + t] =
                    pack2(fmaxf(acc[mt][nt][2] + b0, 0.f), fmaxf(acc[mt][nt][3] + b1, 0.f));
            }
        __syncwarp();
        // ReLU mask words of this lane's pixel: bit j of word c = channel 32 c + j > 0
        const int pl = p0 + lane;
        if (rbits && pl < G.npx) {
            uint32_t m0 = 0, m1 = 0;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                m0 |= pos_bits2(st[lane * YW + e]) << (2 * e);
                m1 |= pos_bits2(st[lane * YW + 16 + e]) << (2 * e);
            }
            rbits[pl] = m0;
            rbits[(size_t)G.npx + pl] = m1;
        }
        // 32 rows x 128 B, 4 rows per warp-wide 512-B store
        uint4 *dst = reinterpret_cast<uint4 *>(y) + (size_t)p0 * 8;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int idx = k * 32 + lane, r = idx >> 3, ch = idx & 7;
            if (p0 + r < G.npx) __stcs(dst + idx, *reinterpret_cast<const uint4 *>(st + r * YW + 4 * ch));
        }
    }
}

// ---- weight gradient: dW[co][k] += sum_p dZ[p][co] x col[p][k] ---------------------------
// MMA view: M = co (4 m16 tiles), N = k (4 n8 tiles, k < 32), K = pixels.  Per warp step of 32
// pixels: dZ rows -> a [32 px][64 co] shared tile (16-B coalesced streaming loads), the column
// tile built lane-per-pixel as in the forward; A = dZ^T and B = col come by ldmatrix.trans.
// Warps take contiguous pixel ranges; the CTA adds its warps' partials in warp order and
// stores ONE 64 x 64 slice (columns >= 32 zero); the fixed-order slice sum
// (splitsum_finish, deferrable) adds the slices in CTA order into dw: no atomics.
constexpr int DZP = 72;  // dZ tile row pitch in bf16 (144 B)
constexpr int WG_SMEM = (SNT / 32) * 32 * (DZP + CT_PITCH) * 2;

__global__ void __launch_bounds__(SNT, 2) stem_wgrad_kernel(const uint8_t *__restrict__ img, Geo G,
                                                            const uint16_t *__restrict__ dz, float *__restrict__ part,
                                                            int px_per_warp) {
    __shared__ uint16_t lut[256];
    extern __shared__ __align__(16) uint8_t wsm[];  // WG_SMEM bytes: dZ tiles | column tiles (| CTA sums after)
    uint16_t(*sdz)[32 * DZP] = reinterpret_cast<uint16_t(*)[32 * DZP]>(wsm);
    uint16_t(*scol)[32 * CT_PITCH] = reinterpret_cast<uint16_t(*)[32 * CT_PITCH]>(wsm + (SNT / 32) * 32 * DZP * 2);
    float(*cta)[33] = reinterpret_cast<float(*)[33]>(wsm);
    lut[threadIdx.x] = bf_bits((float)threadIdx.x / 255.0f);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
    __syncthreads();
    const int wg = blockIdx.x * (SNT / 32) + wid;
    const int lo = wg * px_per_warp, hi = min(G.npx, lo + px_per_warp);
    float acc[4][4][4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = acc[mt][nt][2] = acc[mt][nt][3] = 0.f;
    uint16_t *sd = sdz[wid], *sc = scol[wid];
    for (int p0 = lo; p0 < hi; p0 += 32) {
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // dZ rows p0 .. p0 + 31, zero past hi
            const int idx = k * 32 + lane, r = idx >> 3, ch = idx & 7;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (p0 + r < hi) v = __ldcs(reinterpret_cast<const uint4 *>(dz) + (size_t)(p0 + r) * 8 + ch);
            *reinterpret_cast<uint4 *>(sd + r * DZP + 8 * ch) = v;
        }
        build_col_row(img, lut, G, p0 + lane < hi ? p0 + lane : G.npx, sc + lane * CT_PITCH);
        __syncwarp();
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {  // pixels 16 ks .. 16 ks + 15
            const int prow = 16 * ks + (lane & 7) + 8 * ((lane >> 4) & 1);
            uint32_t b[2][4];  // n tiles (2q, 2q + 1): lanes 0-15 -> n0, 16-31 -> n0 + 8 ... (see below)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                // matrices: [px 0-7][kc 16q..], [px 8-15][kc 16q..], [px 0-7][kc 16q+8..], [px 8-15][kc 16q+8..]
                const int r = 16 * ks + (lane & 7) + 8 * ((lane >> 3) & 1);
                ldsm_x4_t(b[q], sc + r * CT_PITCH + 16 * q + 8 * (lane >> 4));
            }
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                // A = dZ^T: matrices [px 0-7][co 16mt..], [px 0-7][co 16mt+8..], [px 8-15][co 16mt..], [px 8-15][co 16mt+8..]
                uint32_t a[4];
                ldsm_x4_t(a, sd + prow * DZP + 16 * mt + 8 * ((lane >> 3) & 1));
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    mma16816(acc[mt][2 * q], a, b[q][0], b[q][1]);
                    mma16816(acc[mt][2 * q + 1], a, b[q][2], b[q][3]);
                }
            }
        }
    }
    // CTA partial: the warps' accumulators added in warp order in shared memory (over the dZ
    // tiles, free now), then ONE 64 x 64 slice per CTA (columns 32..63 zero).  acc[mt][nt][e]:
    // co = 16 mt + g (+8 for e >= 2), k = 8 nt + 2t + (e & 1).
    __syncthreads();
    for (int wq = 0; wq < SNT / 32; ++wq) {
        if (wid == wq) {
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float *d = &cta[16 * mt + g + 8 * (e >> 1)][8 * nt + 2 * t + (e & 1)];
                        *d = (wq == 0 ? 0.f : *d) + acc[mt][nt][e];
                    }
        }
        __syncthreads();
    }
    float *slice = part + (size_t)blockIdx.x * 4096;  // [64 co][64 k]
    for (int i = threadIdx.x; i < 4096; i += SNT) slice[i] = (i & 63) < 32 ? cta[i >> 6][i & 63] : 0.f;
}

int ilog2_or(int v) {
    if (v <= 0 || (v & (v - 1))) return -1;
    int l = 0;
    while ((1 << l) < v) ++l;
    return l;
}
Geo make_geo(int n, int h, int w) {
    Geo G;
    G.n = n;
    G.h = h;
    G.w = w;
    G.lw = ilog2_or(w);
    G.lh = ilog2_or(h);
    G.npx = n * h * w;
    return G;
}

}  // namespace

extern "C" int ice_stem_fprop(const uint8_t *img, int32_t n, int32_t h, int32_t w, const uint16_t *wt,
                              const float *bias, uint16_t *y, uint32_t *relu_bits, void *stream) {
    if (n < 0 || h < 1 || w < 1) return ICE_EINVAL;
    const long long npx = (long long)n * h * w;
    if (npx == 0) return ICE_OK;
    if (npx > 0x7fffffffLL / 3) return ICE_ETOOBIG;
    if (!img || !wt || !y || ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(wt)) & 15)) return ICE_EINVAL;
    long long blocks = (npx / 32 + SNT / 32 - 1) / (SNT / 32);
    if (blocks > 148 * 2) blocks = 148 * 2;
    if (blocks < 1) blocks = 1;
    stem_fprop_kernel<<<(unsigned)blocks, SNT, 0, (cudaStream_t)stream>>>(img, make_geo(n, h, w), wt, bias, y, relu_bits);
    ice::count_launch();
    return (int)cudaGetLastError();
}

extern "C" int ice_stem_wgrad(const uint8_t *img, int32_t n, int32_t h, int32_t w, const uint16_t *dz, float *dw,
                              void *scratch, uint64_t *scratch_bytes, void *stream) {
    if (n < 0 || h < 1 || w < 1) return ICE_EINVAL;
    const long long npx = (long long)n * h * w;
    if (npx > 0x7fffffffLL / 3) return ICE_ETOOBIG;
    int ctas = 148 * 2;
    const long long warps_total = (long long)ctas * (SNT / 32);
    long long ppw = (npx + warps_total - 1) / warps_total;
    ppw = (ppw + 31) / 32 * 32;
    if (ppw < 32) ppw = 32;
    const long long warps_needed = (npx + ppw - 1) / ppw;
    ctas = (int)((warps_needed + SNT / 32 - 1) / (SNT / 32));
    if (ctas < 1) ctas = 1;
    ice::Arena ar(scratch, scratch_bytes);
    float *part = ar.take<float>((size_t)ctas * 4096 * 4);
    const int rc0 = ar.settle(scratch_bytes);
    if (rc0 == 1) return ICE_OK;
    if (rc0) return rc0;
    if (npx == 0) return ICE_OK;
    if (!img || !dz || !dw || (reinterpret_cast<uintptr_t>(dz) & 15)) return ICE_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    static bool attr = false;
    if (!attr) {
        const cudaError_t e = cudaFuncSetAttribute(stem_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, WG_SMEM);
        if (e != cudaSuccess) return (int)e;
        attr = true;
    }
    stem_wgrad_kernel<<<(unsigned)ctas, SNT, WG_SMEM, st>>>(img, make_geo(n, h, w), dz, part, (int)ppw);
    ice::count_launch();
    const int rc = (int)cudaGetLastError();
    if (rc) return rc;
    return ice::splitsum_finish(part, ctas, 4096, 4096, dw, st, ice::grad_overwrite());
}
