// conv_tc.cu -- NHWC bf16 implicit-GEMM convolutions on 5th-gen tensor cores (tcgen05).
//
// One warp-specialised kernel template serves fprop, dgrad and wgrad of the U-Net's
// convolutions (icetrain/model.py:64-88):
//   warp 0      TMA producer: per K-block, tap-shifted boxes of the NHWC activation
//               (4-D tensor map (C, W, H, N); out-of-image rows/cols arrive zero-filled,
//               which IS the conv's zero padding) and the weight slab;
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (128 x BN x 16 per op);
//   warps 2..5  epilogue: tcgen05.ld of the fp32 accumulator, fused bias / ReLU /
//               Dropout2d / ReLU-backward / gradient-sum, bf16 NHWC store (or fp32
//               red.add for weight gradients).
// The concatenation cat([skip, x], 1) of model.py:129 is never materialised: channel
// blocks below c1 come from the skip tensor's map, the rest from the other map.
//
// GEMM views (m = output row in TMEM lanes, n = TMEM column, k = reduction):
//   fprop  D[pixel][cout]     = sum_{tap,cin}  X[pixel+tap][cin]  * W[cout][tap][cin]   A,B K-major
//   dgrad  D[pixel][cin]      = sum_{tap,cout} dY[pixel-tap][cout]* W[cout][tap][cin]   A K-major, B MN-major
//   wgrad  D[cout][(tap,cin)] = sum_{pixel}    dY[pixel][cout]    * X[pixel+tap][cin]   A,B MN-major
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "icelabel_b200.h"
#include "reduce.cuh"
#include "tc_common.cuh"

namespace {

using bf16 = __nv_bfloat16;
constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = one 128-byte swizzle row
constexpr int A_BYTES = BM * BK * 2;
constexpr int EPI_WARPS = 8;
constexpr int STAGE_BYTES = 32 * 64;  // one warp's 32 px x 32 ch bf16 output box (staged TMA stores)
// single-buffered: with the staged ReLU reference (double-buffered, 32 KB) a second output
// buffer would overflow the 227 KB of shared memory; a box's store reads smem in well under
// the time the warp spends on the next tile's TMEM load and math
constexpr int STAGE_BUFS = 1;  // two warps per TMEM lane quarter, each draining half the columns
constexpr int NTHREADS = 64 + 32 * EPI_WARPS;
constexpr int BIAS_SLOTS = 8;  // shared-memory rows of the fused bias-gradient column sums

// a box of Wt x Ht x Nt pixels, and how many boxes tile (W, H, N).  Every entry point
// requires power-of-two H and W (shape_ok), so Wt, Ht, Nt, tw, th are powers of two and the
// index math is shifts and masks (the epilogue runs it per tile; integer division by a
// runtime value costs ~25 instructions and dominated the short-K epilogues).
__device__ __forceinline__ int lg2(int v) { return __ffs(v) - 1; }
struct PixTile {
    int Wt, Ht, Nt, tw, th, tn;
    __device__ __forceinline__ void origin(int t, int &n0, int &h0, int &w0) const {
        const int wi = t & (tw - 1);
        t >>= lg2(tw);
        const int hi = t & (th - 1);
        const int ni = t >> lg2(th);
        w0 = wi * Wt;
        h0 = hi * Ht;
        n0 = ni * Nt;
    }
    __device__ __forceinline__ void pixel(int row, int n0, int h0, int w0, int &n, int &h, int &w) const {
        w = w0 + (row & (Wt - 1));
        const int r = row >> lg2(Wt);
        h = h0 + (r & (Ht - 1));
        n = n0 + (r >> lg2(Ht));
    }
};

struct Taps {
    int n;
    int8_t dy[9], dx[9], plane[9], wt[9];  // pixel shift, source plane (5-D maps), weight tap
};

// 8 consecutive floats (or `fill` when p is null); 16 B vector loads when p is aligned
__device__ __forceinline__ void ld8(const float *p, float fill, float (&o)[8]) {
    if (!p) {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = fill;
    } else if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(p)), b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
        o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = __ldg(p + i);
    }
}

// 2 bits per packed bf16 pair: element > 0 (the ReLU mask backward needs, exact on bf16)
__device__ __forceinline__ uint32_t pos_bits2(uint32_t w) {
    const uint32_t lo = w & 0xffffu, hi = w >> 16;
    return (uint32_t)((lo & 0x7fffu) != 0 && !(lo & 0x8000u)) | ((uint32_t)((hi & 0x7fffu) != 0 && !(hi & 0x8000u)) << 1);
}

// Column sums of a warp's 32 rows x 32 columns (one row per lane): after 31 shuffles lane j
// holds the sum of column j over the 32 rows.
__device__ __forceinline__ float warp_col_sum32(float (&v)[32], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const bool hi = lane & o;
            const float send = hi ? v[i] : v[i + o];
            const float keep = hi ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

// ------------------------------------------------------------------------------------
struct FpropProb {
    static constexpr bool A_MN = false, B_MN = false;
    static constexpr int EPI_STAGE = STAGE_BYTES;
    static constexpr bool BIAS_ROWS = true;
    static constexpr bool STAGE_REF = false;
    static constexpr int ref_tma = 0;
    __device__ void load_ref(uint8_t *, uint64_t *, int, int) const {}
    CUtensorMap xa, xb, wm;
    PixTile pt;
    Taps taps[4];  // per blockIdx.z (the 4 sub-pixel classes of the halving conv; else 1)
    int N, H, W, c1, c2, cout;
    int omul;      // 1: output pixel = input pixel; 2: output (2h + cy, 2w + cx), z = 2 cy + cx
    int merged;    // halving conv with the 4 sub-pixel classes side by side in N (class = col / cout)
    const float *bias;
    const float *drop;  // [N][cout] or null
    int relu;
    bf16 *y;
    uint32_t *rbits;    // optional ReLU mask of y: [cout / 32][N*H*W] words, bit j = column 32 k + j > 0
    CUtensorMap ym;     // y as (cout, W, H, N), box 32 ch x 32 px, SWIZZLE_64B (staged stores)
    int y_tma;

    __device__ void kb_range(int z, int &kb0, int &nkb) const {
        kb0 = 0;
        nkb = taps[z].n * ((c1 + c2) / BK);
    }
    __device__ void prefetch() const {
        tc::tma_prefetch_desc(&xa);
        if (c2) tc::tma_prefetch_desc(&xb);
        tc::tma_prefetch_desc(&wm);
    }
    template <int BN>
    __device__ void load(int kb, uint8_t *sa, uint8_t *sb, uint64_t *bar, int mt, int nt, int z) const {
        const Taps &tp = taps[z];
        const int cch = (c1 + c2) / BK;
        const int t = kb / cch, c = (kb % cch) * BK;
        int n0, h0, w0;
        pt.origin(mt, n0, h0, w0);
        if (c < c1) tc::tma_load_4d(sa, &xa, bar, c, w0 + tp.dx[t], h0 + tp.dy[t], n0);
        else tc::tma_load_4d(sa, &xb, bar, c - c1, w0 + tp.dx[t], h0 + tp.dy[t], n0);
        tc::tma_load_3d(sb, &wm, bar, c, tp.wt[t], nt * BN);
    }
    // 256-row tile mt = pixel tiles 2 mt and 2 mt + 1 over one 256-column weight block
    template <int BN>
    __device__ void load_m2(int kb, uint8_t *sa, uint8_t *sb, uint64_t *bar, int mt, int nt, int z) const {
        load<BN>(kb, sa, sb, bar, 2 * mt, nt, z);
        const Taps &tp = taps[z];
        const int cch = (c1 + c2) / BK;
        const int t = kb / cch, c = (kb % cch) * BK;
        int n0, h0, w0;
        pt.origin(2 * mt + 1, n0, h0, w0);
        if (c < c1) tc::tma_load_4d(sa + A_BYTES, &xa, bar, c, w0 + tp.dx[t], h0 + tp.dy[t], n0);
        else tc::tma_load_4d(sa + A_BYTES, &xb, bar, c - c1, w0 + tp.dx[t], h0 + tp.dy[t], n0);
    }
    // ---- row-halo path (3x3, W % 128 == 0): one 3 x 130-pixel slab per 64-channel chunk
    __device__ int halo_chunks() const { return (c1 + c2) / BK; }
    __device__ void load_halo(int chunk, uint8_t *dst, uint64_t *bar, int mt) const {
        int n0, h0, w0;
        pt.origin(mt, n0, h0, w0);
        const int c = chunk * BK;
        if (c < c1) tc::tma_load_4d(dst, &xa, bar, c, w0 - 1, h0 - 1, n0);
        else tc::tma_load_4d(dst, &xb, bar, c - c1, w0 - 1, h0 - 1, n0);
    }
    template <int BN>
    __device__ void load_tap_b(int tap, int chunk, uint8_t *dst, uint64_t *bar, int nt) const {
        tc::tma_load_3d(dst, &wm, bar, chunk * BK, tap, nt * BN);
    }
    __device__ int view_row(int tap) const { return (taps[0].dy[tap] + 1) * 130 + taps[0].dx[tap] + 1; }

    // Epilogue operands of the NEXT tile, loaded before the accumulator wait: lane j holds
    // bias[col0 + j] and (when all 32 rows of the warp are one image) drop[n][col0 + j] of
    // the first two 32-column chunks; the epilogue broadcasts them with shuffles.
    struct Pre {
        float b[2], d[2];
        int uni;
    };
    template <int BN>
    __device__ void pre_load(Pre &pr, int row, int mt, int nt, int, int cc0, int cc1) const {
        int n0, h0, w0, n, h, w;
        pt.origin(mt, n0, h0, w0);
        pt.pixel(row, n0, h0, w0, n, h, w);
        const int lane = threadIdx.x & 31;
        const int n_first = __shfl_sync(0xffffffffu, n, 0);
        pr.uni = __all_sync(0xffffffffu, n == n_first) && n_first < N;
#pragma unroll
        for (int ci = 0; ci < 2; ++ci) {
            const int col = nt * BN + (cc0 + ci) * 32 + lane;
            const bool have = cc0 + ci < cc1;
            pr.b[ci] = (have && bias) ? __ldg(bias + (merged ? col & (cout - 1) : col)) : 0.f;
            pr.d[ci] = (have && drop && pr.uni) ? __ldg(drop + (size_t)n_first * cout + col) : 1.f;
        }
    }
    template <int BN>
    __device__ void stash_bias(int, int, float *, int, float *) const {}
    template <int BN>
    __device__ void commit_bias(int, float *) const {}
    template <int BN>
    __device__ void epilogue(uint32_t tmem, int row, int mt, int nt, int z, int cc0, int cc1, float *,
                             const Pre &pr, uint8_t *stage = nullptr, const uint8_t * = nullptr) const {
        int n0, h0, w0, n, h, w;
        pt.origin(mt, n0, h0, w0);
        pt.pixel(row, n0, h0, w0, n, h, w);
        const bool valid = n < N;
        const int OH = H * omul, OW = W * omul;
        const int hb = h, wb = w;
        if (omul == 2 && !merged) {
            h = 2 * hb + (z >> 1);
            w = 2 * wb + (z & 1);
        }
#pragma unroll 1
        for (int cc = cc0; cc < cc1; ++cc) {
            float v[32];
            tc::tmem_ld32(tmem + cc * 32, v);
            int col0 = nt * BN + cc * 32;
            if (merged) {  // this 32-column chunk belongs to sub-pixel class col0 / cout
                const int cls = col0 >> lg2(cout);  // merged: cout is 64 or 128
                col0 -= cls * cout;
                h = 2 * hb + (cls >> 1);
                w = 2 * wb + (cls & 1);
            }
            const int ci = cc - cc0;
            if (ci < 2) {  // warp-uniform: prefetched operands, broadcast through shared memory
                const float bsrc = ci == 0 ? pr.b[0] : pr.b[1];
                const float dsrc = ci == 0 ? pr.d[0] : pr.d[1];
                __shared__ __align__(16) float sbd[EPI_WARPS][64];  // per epilogue warp: bias | drop
                float *mine = sbd[((threadIdx.x >> 5) - 2) & (EPI_WARPS - 1)];
                const int ln = threadIdx.x & 31;
                __syncwarp();
                mine[ln] = bsrc;
                mine[32 + ln] = dsrc;
                __syncwarp();
                float dl[32];
                if (drop && !pr.uni && valid) {  // rows of several images (tiny levels)
                    const float *dr = drop + (size_t)n * cout + col0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        float t8[8];
                        ld8(dr + q * 8, 1.f, t8);
#pragma unroll
                        for (int e = 0; e < 8; ++e) dl[q * 8 + e] = t8[e];
                    }
                }
#pragma unroll
                for (int j4 = 0; j4 < 8; ++j4) {
                    const float4 b4 = *reinterpret_cast<const float4 *>(mine + 4 * j4);
                    const float4 d4 = *reinterpret_cast<const float4 *>(mine + 32 + 4 * j4);
                    const float bb[4] = {b4.x, b4.y, b4.z, b4.w}, dd[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int j = 4 * j4 + e;
                        float a = v[j] + bb[e];
                        if (relu) a = fmaxf(a, 0.f);
                        v[j] = a * ((drop && !pr.uni) ? dl[j] : dd[e]);
                    }
                }
                uint32_t pk[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) pk[e] = tc::pack_bf16(v[2 * e], v[2 * e + 1]);
                if (rbits && valid) {
                    uint32_t b = 0;
#pragma unroll
                    for (int e = 0; e < 16; ++e) b |= pos_bits2(pk[e]) << (2 * e);
                    rbits[(size_t)(col0 >> 5) * ((size_t)N * OH * OW) + ((size_t)n * OH + h) * OW + w] = b;
                }
                if (stage && y_tma) {  // warp-uniform: rows of one image row, all valid (halo tiles)
                    const int lane = threadIdx.x & 31;
                    if (lane == 0) tc::bulk_wait_read<STAGE_BUFS - 1>();  // the buffer's last store has read smem
                    __syncwarp();
                    tc::stage_row64(stage, lane, pk);
                    tc::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tc::tma_store_4d(&ym, stage, col0, w, h, n);  // lane 0's pixel starts the box
                        tc::bulk_commit();
                    }
                    continue;
                }
                if (!valid) continue;
                uint4 *dst = reinterpret_cast<uint4 *>(y + ((size_t)((size_t)n * OH + h) * OW + w) * cout + col0);
#pragma unroll
                for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                continue;
            }
            const bool staged = stage && y_tma;  // warp-uniform
            if (!valid && !staged) continue;
            const float *dr = (drop && valid) ? drop + (size_t)n * cout + col0 : nullptr;
            uint32_t rb = 0, pk[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float bq[8], dq[8];
                ld8(bias ? bias + col0 + q * 8 : nullptr, 0.f, bq);
                ld8(dr ? dr + q * 8 : nullptr, 1.f, dq);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    float a = v[q * 8 + 2 * e] + bq[2 * e], b = v[q * 8 + 2 * e + 1] + bq[2 * e + 1];
                    if (relu) {
                        a = fmaxf(a, 0.f);
                        b = fmaxf(b, 0.f);
                    }
                    pk[4 * q + e] = tc::pack_bf16(a * dq[2 * e], b * dq[2 * e + 1]);
                    rb |= pos_bits2(pk[4 * q + e]) << (8 * q + 2 * e);
                }
            }
            if (rbits && valid) rbits[(size_t)(col0 >> 5) * ((size_t)N * OH * OW) + ((size_t)n * OH + h) * OW + w] = rb;
            if (staged) {
                const int lane = threadIdx.x & 31;
                if (lane == 0) tc::bulk_wait_read<0>();
                __syncwarp();
                tc::stage_row64(stage, lane, pk);
                tc::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tc::tma_store_4d(&ym, stage, col0, w, h, n);  // lane 0's pixel starts the box
                    tc::bulk_commit();
                }
                continue;
            }
            uint4 *dst = reinterpret_cast<uint4 *>(y + ((size_t)((size_t)n * OH + h) * OW + w) * cout + col0);
#pragma unroll
            for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
    }
};

// ------------------------------------------------------------------------------------
struct DgradProb {
    static constexpr bool A_MN = false, B_MN = true;
    static constexpr int EPI_STAGE = STAGE_BYTES;
    static constexpr bool BIAS_ROWS = true;
    static constexpr bool STAGE_REF = true;
    CUtensorMap dym, wm;  // dY (box 64 x pixel tile), weights (box 64 cin x 1 x 64 cout)
    CUtensorMap refm;     // ReLU reference of dx1, box 64 ch x 128 px (halo BN = 64 tiles)
    int ref_tma;          // the halo producer TMA-stages ref1 tiles into shared memory
    PixTile pt;
    Taps taps;
    int N, H, W, c1, c2, cout;
    int planes_in;    // dY given as 4 sub-pixel planes [4][N][H][W][cout] (5-D map, plane per tap)
    int planes_out2;  // dx2 written as sub-pixel planes [4][N][H/2][W/2][c2]
    bf16 *out1, *out2;
    const bf16 *ref1, *ref2, *add1, *add2;
    const uint32_t *rbits1;  // optional ReLU mask of dx1 as bits ([c1 / 32][N*H*W]); replaces ref1
    const float *drop1, *drop2;
    float *db1, *db2;  // fused bias gradients of the layers whose pre-activation grads these are
    float *bpart;      // their per-CTA partial column sums (scratch), bslots rows per CTA
    int bslots;
    CUtensorMap o1m;   // dx1 as (c1, W, H, N), box 32 ch x 32 px, SWIZZLE_64B (staged stores)
    int o1_tma;
    CUtensorMap o2m;   // dx2 planes as (c2, W/2, H/2, N, 4), box 32 ch x 16 px (row tiles, staged stores)
    int o2_tma;

    __device__ void kb_range(int, int &kb0, int &nkb) const {
        kb0 = 0;
        nkb = taps.n * (cout / BK);
    }
    __device__ void prefetch() const {
        tc::tma_prefetch_desc(&dym);
        tc::tma_prefetch_desc(&wm);
    }
    template <int BN>
    __device__ void load(int kb, uint8_t *sa, uint8_t *sb, uint64_t *bar, int mt, int nt, int) const {
        const int cch = cout / BK;
        const int t = kb / cch, c = (kb % cch) * BK;
        int n0, h0, w0;
        pt.origin(mt, n0, h0, w0);
        if (planes_in) tc::tma_load_5d(sa, &dym, bar, c, w0 - taps.dx[t], h0 - taps.dy[t], n0, taps.plane[t]);
        else tc::tma_load_4d(sa, &dym, bar, c, w0 - taps.dx[t], h0 - taps.dy[t], n0);
#pragma unroll
        for (int j = 0; j < BN / 64; ++j) tc::tma_load_3d(sb + j * 8192, &wm, bar, nt * BN + j * 64, taps.wt[t], c);
    }
    template <int BN>
    __device__ void load_m2(int kb, uint8_t *sa, uint8_t *sb, uint64_t *bar, int mt, int nt, int z) const {
        load<BN>(kb, sa, sb, bar, 2 * mt, nt, z);
        const int cch = cout / BK;
        const int t = kb / cch, c = (kb % cch) * BK;
        int n0, h0, w0;
        pt.origin(2 * mt + 1, n0, h0, w0);
        if (planes_in) tc::tma_load_5d(sa + A_BYTES, &dym, bar, c, w0 - taps.dx[t], h0 - taps.dy[t], n0, taps.plane[t]);
        else tc::tma_load_4d(sa + A_BYTES, &dym, bar, c, w0 - taps.dx[t], h0 - taps.dy[t], n0);
    }
    // ---- row-halo path: slab of dY around the tile; tap t reads dY[p - shift_t]
    __device__ int halo_chunks() const { return cout / BK; }
    // the tile's ReLU-reference rows (64 channels x 128 pixels, SWIZZLE_128B) for the epilogue
    __device__ void load_ref(uint8_t *dst, uint64_t *bar, int mt, int nt) const {
        int n0, h0, w0;
        pt.origin(mt, n0, h0, w0);
        tc::tma_load_4d(dst, &refm, bar, nt * 64, w0, h0, n0);
    }
    __device__ void load_halo(int chunk, uint8_t *dst, uint64_t *bar, int mt) const {
        int n0, h0, w0;
        pt.origin(mt, n0, h0, w0);
        tc::tma_load_4d(dst, &dym, bar, chunk * BK, w0 - 1, h0 - 1, n0);
    }
    template <int BN>
    __device__ void load_tap_b(int tap, int chunk, uint8_t *dst, uint64_t *bar, int nt) const {
#pragma unroll
        for (int j = 0; j < BN / 64; ++j) tc::tma_load_3d(dst + j * 8192, &wm, bar, nt * BN + j * 64, tap, chunk * BK);
    }
    __device__ int view_row(int tap) const { return (1 - taps.dy[tap]) * 130 + 1 - taps.dx[tap]; }

    // lane j of each epilogue warp keeps, per owned 32-column chunk, the running sum of
    // column j over all rows it has stored for the current column tile
    // ... and at the end of its run over a column tile stashes them in shared memory (row
    // `slot` of sb[bslots][BN]: the TMEM lane quarter, x the M half for 256-row tiles); the
    // commit then adds the slots in slot order and stores the CTA's column sums as row
    // blockIdx.x of bpart[G][c1 + c2] (no atomics); colsum_finish adds the rows of the CTAs
    // that visited the column tile, in CTA order (reduce.cuh).  Every epilogue warp reaches
    // each stash/commit at the same tile, so the commit's named barrier (id 1, the 256
    // epilogue threads) is uniform.
    template <int BN>
    __device__ void stash_bias(int cc0, int cc1, float *bacc, int slot, float *sb) const {
        const int lane = threadIdx.x & 31;
        constexpr int NCH = BN / 32, PER = (NCH + 1) / 2;
#pragma unroll
        for (int ci = 0; ci < PER; ++ci) {
            const int cc = cc0 + ci;
            if (cc < cc1) sb[slot * BN + cc * 32 + lane] = bacc[ci];
            bacc[ci] = 0.f;
        }
    }
    template <int BN>
    __device__ void commit_bias(int nt, float *sb) const {
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
        if (bpart) {
            float *row = bpart + (size_t)blockIdx.x * (c1 + c2) + nt * BN;
            for (int j = threadIdx.x - 64; j < BN; j += 32 * EPI_WARPS) {
                float s = 0.f;
                for (int k = 0; k < bslots; ++k) s += sb[k * BN + j];
                row[j] = s;
            }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
    }
    // (register prefetch of the next tile's ReLU-reference rows measured slower: the
    // extra in-flight loads contend with the epilogue's stores).  The packed ReLU-mask words
    // (4 B per row and 32 channels) are prefetched for the next tile ahead of its accumulator
    // wait, so the epilogue does not stall on their global-load latency.
    struct Pre {
        uint32_t b[4];
    };
    template <int BN>
    __device__ void pre_load(Pre &pr, int row, int mt, int nt, int, int cc0, int cc1) const {
#pragma unroll
        for (int ci = 0; ci < 4; ++ci) pr.b[ci] = 0xffffffffu;
        if (!rbits1) return;
        int n0, h0, w0, n, h, w;
        pt.origin(mt, n0, h0, w0);
        pt.pixel(row, n0, h0, w0, n, h, w);
        if (n >= N) return;
        const size_t pix = ((size_t)n * H + h) * W + w;
        constexpr int NCH = BN / 32, PER = (NCH + 1) / 2;
#pragma unroll
        for (int ci = 0; ci < PER && ci < 4; ++ci) {
            const int cc = cc0 + ci, col = nt * BN + cc * 32;
            if (cc < cc1 && col < c1) pr.b[ci] = __ldg(rbits1 + (size_t)(col >> 5) * ((size_t)N * H * W) + pix);
        }
    }
    template <int BN>
    __device__ void epilogue(uint32_t tmem, int row, int mt, int nt, int, int cc0, int cc1, float *bacc,
                             const Pre &pr, uint8_t *stage = nullptr, const uint8_t *ref_smem = nullptr) const {
        int n0, h0, w0, n, h, w;
        pt.origin(mt, n0, h0, w0);
        pt.pixel(row, n0, h0, w0, n, h, w);
        const bool valid = n < N;
        const size_t pix = ((size_t)n * H + h) * W + w;
        const size_t pix_planes =
            ((((size_t)((h & 1) * 2 + (w & 1)) * N + n) * (H >> 1) + (h >> 1)) * (W >> 1)) + (w >> 1);
        const int lane = threadIdx.x & 31;
        constexpr int NCH = BN / 32, PER = (NCH + 1) / 2;
        // not unrolled: the body holds every output variant (add / mask / drop / staged dx1 /
        // staged planes / direct), and one copy per chunk overflowed the instruction cache
        // (ncu: 25% of the epilogue's stall samples were no_inst); bacc and the prefetched mask
        // words are indexed through selects, so they stay in registers
#pragma unroll 1
        for (int ci = 0; ci < PER; ++ci) {
            const int cc = cc0 + ci;
            if (cc >= cc1) break;
            float v[32];
            tc::tmem_ld32(tmem + cc * 32, v);
            int col = nt * BN + cc * 32;
            bf16 *out;
            const bf16 *ref, *add;
            const float *drop;
            float *db;
            int cs;
            if (col < c1) {
                out = out1; ref = ref1; add = add1; drop = drop1; cs = c1; db = db1;
            } else {
                col -= c1;
                out = out2; ref = ref2; add = add2; drop = drop2; cs = c2; db = db2;
            }
            if (!out) continue;  // warp-uniform
            const size_t off = ((out == out2 && planes_out2) ? pix_planes : pix) * cs + col;
            if (valid) {
                if (add) {
                    const uint4 *ap = reinterpret_cast<const uint4 *>(add + off);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint4 u = ap[q];
                        const bf16 *b = reinterpret_cast<const bf16 *>(&u);
#pragma unroll
                        for (int e = 0; e < 8; ++e) v[q * 8 + e] += __bfloat162float(b[e]);
                    }
                }
                if (rbits1 && out == out1) {  // the forward's packed ReLU mask: 4 B instead of 64 B per row
                    const uint32_t b = ci == 0 ? pr.b[0] : ci == 1 ? pr.b[1] : ci == 2 ? pr.b[2] : pr.b[3];  // (pre_load)
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (!((b >> e) & 1u)) v[e] = 0.f;
                } else if (ref) {
                    const uint4 *rp = reinterpret_cast<const uint4 *>(ref + off);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        // staged tile (64 ch x 128 px, 128-B swizzle: 16-B chunk j of row r at j ^ (r & 7))
                        uint4 u = (ref_smem && ref == ref1)
                                      ? *reinterpret_cast<const uint4 *>(ref_smem + row * 128 + (((cc * 4 + q) ^ (row & 7)) << 4))
                                      : rp[q];
                        const bf16 *b = reinterpret_cast<const bf16 *>(&u);
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            if (!(__bfloat162float(b[e]) > 0.f)) v[q * 8 + e] = 0.f;
                    }
                }
                if (drop) {
                    const float4 *dp = reinterpret_cast<const float4 *>(drop + (size_t)n * cs + col);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float4 d = __ldg(dp + q);
                        v[4 * q] *= d.x;
                        v[4 * q + 1] *= d.y;
                        v[4 * q + 2] *= d.z;
                        v[4 * q + 3] *= d.w;
                    }
                }
                if (stage && o1_tma && out == out1) {  // warp-uniform (halo tiles: all rows valid)
                    uint32_t pk[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) pk[e] = tc::pack_bf16(v[2 * e], v[2 * e + 1]);
                    if (lane == 0) tc::bulk_wait_read<STAGE_BUFS - 1>();  // the buffer's last store has read smem
                    __syncwarp();
                    tc::stage_row64(stage, lane, pk);
                    tc::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tc::tma_store_4d(&o1m, stage, col, w, h, n);  // lane 0's pixel starts the box
                        tc::bulk_commit();
                    }
                } else if (stage && o2_tma && out == out2) {
                    // sub-pixel planes: the warp's 32 pixels of one row split by column parity into
                    // two 16-pixel runs of planes 2 (h & 1) and 2 (h & 1) + 1 -- staged as rows
                    // 0-15 (even lanes) and 16-31 (odd lanes), written by two TMA stores
                    uint32_t pk[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) pk[e] = tc::pack_bf16(v[2 * e], v[2 * e + 1]);
                    if (lane == 0) tc::bulk_wait_read<STAGE_BUFS - 1>();
                    __syncwarp();
                    tc::stage_row64_at(stage, (lane & 1) * 16 + (lane >> 1), pk);
                    tc::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {  // lane 0's pixel (w even) starts both runs
                        const int cls = 2 * (h & 1);
                        tc::tma_store_5d(&o2m, stage, col, w >> 1, h >> 1, n, cls);
                        tc::tma_store_5d(&o2m, stage + 16 * 64, col, w >> 1, h >> 1, n, cls + 1);
                        tc::bulk_commit();
                    }
                } else {
                    uint4 *dst = reinterpret_cast<uint4 *>(out + off);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        dst[q] = make_uint4(tc::pack_bf16(v[q * 8 + 0], v[q * 8 + 1]), tc::pack_bf16(v[q * 8 + 2], v[q * 8 + 3]),
                                            tc::pack_bf16(v[q * 8 + 4], v[q * 8 + 5]), tc::pack_bf16(v[q * 8 + 6], v[q * 8 + 7]));
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = 0.f;
            }
            if (db) {  // warp-uniform: bias gradient = column sums of the (fp32) gradient

                const float cs = warp_col_sum32(v, lane);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (k == ci) bacc[k] += cs;
            }
        }
    }
};

// ------------------------------------------------------------------------------------
struct WgradProb {
    static constexpr bool A_MN = true, B_MN = true;
    // 256-row tiles: a 4 KB fp32 staging block per epilogue warp (transposed stores), no bias rows
    static constexpr int EPI_STAGE = 4096;
    static constexpr bool BIAS_ROWS = false;
    CUtensorMap dym, xa, xb;  // boxes of 64 channels x 64 pixels
    PixTile pk;               // the 64-pixel K-block geometry
    Taps taps;
    int N, H, W, c1, c2, cout;
    int total_kb, kb_per_split;
    int halve;  // 2x2 halving conv: dY = 4 sub-pixel planes (5-D map), K runs over (class, pixel block)
    int trans;  // narrow cout (< 128): D = [(tap, cin)][cout], A = shifted x, B = dY (no wasted M rows)
    int nbx, nby;  // non-halve: maps are 5-D (64, W, H, N, C/64) and one TMA box carries nb 64-ch blocks
    float *dw;  // [cout][taps][c1+c2]
    float *ws;  // partials of splits 1.. [splits - 1][cout][taps][c1+c2] (scratch) when splits > 1
    size_t wsize;
    int ow;     // gradient overwrite mode: split 0 stores instead of adding (ice_grad_overwrite)

    __device__ void kb_range(int z, int &kb0, int &nkb) const {
        kb0 = z * kb_per_split;
        nkb = min(total_kb - kb0, kb_per_split);
    }
    __device__ void prefetch() const {
        tc::tma_prefetch_desc(&dym);
        tc::tma_prefetch_desc(&xa);
        if (c2) tc::tma_prefetch_desc(&xb);
    }
    // one 64-channel x 64-pixel box of x for the 64-wide (tap, cin) block starting at col
    __device__ __forceinline__ void load_x(uint8_t *dst, uint64_t *bar, int col, int cls, int n0, int h0,
                                           int w0) const {
        const int ct = c1 + c2;
        int t = col / ct, c = col - t * ct;
        if (t >= taps.n) t = 0, c = 0;  // padding rows of the last M tile: any valid box, never stored
        int sy = taps.dy[t], sx = taps.dx[t];
        if (halve) {  // output (2p + cy, 2q + cx) reads up[2p + cy + a][2q + cx + b] = x[p + (cy + a) / 2][...]
            sy = ((cls >> 1) + (t >> 1)) >> 1;
            sx = ((cls & 1) + (t & 1)) >> 1;
        }
        if (nbx == 1) {
            if (c < c1) tc::tma_load_4d(dst, &xa, bar, c, w0 + sx, h0 + sy, n0);
            else tc::tma_load_4d(dst, &xb, bar, c - c1, w0 + sx, h0 + sy, n0);
        } else {
            if (c < c1) tc::tma_load_5d(dst, &xa, bar, 0, w0 + sx, h0 + sy, n0, c >> 6);
            else tc::tma_load_5d(dst, &xb, bar, 0, w0 + sx, h0 + sy, n0, (c - c1) >> 6);
        }
    }
    __device__ __forceinline__ void load_dy(uint8_t *dst, uint64_t *bar, int c0, int cls, int n0, int h0,
                                            int w0) const {
        const int img = halve ? cls * N + n0 : n0;  // sub-pixel planes [4][N] flatten to 4N images
        if (nby == 1) tc::tma_load_4d(dst, &dym, bar, c0, w0, h0, img);
        else tc::tma_load_5d(dst, &dym, bar, 0, w0, h0, img, c0 >> 6);
    }
    template <int BN>
    __device__ void load(int kb, uint8_t *sa, uint8_t *sb, uint64_t *bar, int mt, int nt, int) const {
        load_rows<BN, 2>(kb, sa, sb, bar, mt * BM, nt);
    }
    template <int BN>
    __device__ void load_m2(int kb, uint8_t *sa, uint8_t *sb, uint64_t *bar, int mt, int nt, int) const {
        load_rows<BN, 4>(kb, sa, sb, bar, mt * 2 * BM, nt);
    }
    // MB 64-row blocks of the M operand starting at row m0 (MB = 4: the 256-row tiles of conv_gemm_m2)
    template <int BN, int MB>
    __device__ void load_rows(int kb, uint8_t *sa, uint8_t *sb, uint64_t *bar, int m0, int nt) const {
        int n0, h0, w0, cls = 0;
        if (halve) {
            const int nblk = pk.tw * pk.th * pk.tn;
            cls = kb / nblk;
            kb -= cls * nblk;
        }
        pk.origin(kb, n0, h0, w0);
        // one TMA box carries nb consecutive 64-channel blocks ([block][pixel][64 ch] in smem)
        const int bx = nbx, by = nby;
        if (!trans) {
            for (int j = 0; j < MB; j += by) load_dy(sa + j * 8192, bar, m0 + j * 64, cls, n0, h0, w0);
            for (int j = 0; j < BN / 64; j += bx) load_x(sb + j * 8192, bar, nt * BN + j * 64, cls, n0, h0, w0);
        } else {
            for (int j = 0; j < MB; j += bx) load_x(sa + j * 8192, bar, m0 + j * 64, cls, n0, h0, w0);
            for (int j = 0; j < BN / 64; j += by) load_dy(sb + j * 8192, bar, nt * BN + j * 64, cls, n0, h0, w0);
        }
    }
    struct Pre {};
    template <int BN>
    __device__ void pre_load(Pre &, int, int, int, int, int, int) const {}
    template <int BN>
    __device__ void stash_bias(int, int, float *, int, float *) const {}
    template <int BN>
    __device__ void commit_bias(int, float *) const {}
    template <int BN>
    // split 0: dw += tile with fire-and-forget reductions (RED) -- the launch's only
    // contribution to these elements, so the result does not depend on timing; split z > 0
    // stores its partial tile into slice z - 1 of ws and splitsum_finish then adds the slices in
    // split order: dw = (dw + p0) + ((p1 + p2) + ...), a fixed association -> bit-reproducible
    __device__ void epilogue(uint32_t tmem, int row, int mt, int nt, int z, int cc0, int cc1, float *, const Pre &,
                             uint8_t *stage = nullptr, const uint8_t * = nullptr) const {
        const int m = mt * BM + row;
        const int ld = taps.n * (c1 + c2);
        const bool part = z > 0;
        float *base = part ? ws + (size_t)(z - 1) * wsize : dw;
#pragma unroll 1
        for (int cc = cc0; cc < cc1; ++cc) {
            float v[32];
            tc::tmem_ld32(tmem + cc * 32, v);
            if (!trans && stage) {
                // 256-row tiles drain with the mainloop stopped (TMEM holds one tile): a lane's
                // 128-B row segment as 8 x 16-B stores touches 32 lines per warp instruction;
                // through the warp's 4 KB staging block each instruction covers 4 full rows
                // (lane l: row 4 i + l / 8, 16-B chunk l % 8), 8x fewer L2 requests
                const int lane = threadIdx.x & 31;
                __syncwarp();
#pragma unroll
                for (int q = 0; q < 8; ++q)  // chunk q of row `lane` at q ^ (lane & 7): conflict-free
                    *reinterpret_cast<float4 *>(stage + lane * 128 + ((q ^ (lane & 7)) << 4)) =
                        make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                __syncwarp();
                const int m0 = m - lane, q = lane & 7;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int r = 4 * i + (lane >> 3);
                    const float4 u = *reinterpret_cast<const float4 *>(stage + r * 128 + ((q ^ (r & 7)) << 4));
                    if (m0 + r >= cout) continue;
                    float *dst = base + (size_t)(m0 + r) * ld + nt * BN + cc * 32 + 4 * q;
                    if (part || ow) __stcg(reinterpret_cast<float4 *>(dst), u);
                    else tc::red_add_v4(dst, u.x, u.y, u.z, u.w);
                }
            } else if (!trans) {
                if (m >= cout) continue;
                float *dst = base + (size_t)m * ld + nt * BN + cc * 32;
                if (part || ow) {  // a slice, or the first gradient of the step (overwrite mode)
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        __stcg(reinterpret_cast<float4 *>(dst) + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
                } else {
#pragma unroll
                    for (int q = 0; q < 8; ++q) tc::red_add_v4(dst + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                }
            } else {
                if (m >= ld) continue;
                const int o0 = nt * BN + cc * 32;  // output channels; lanes hold consecutive (tap, cin)
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (o0 + j >= cout) continue;
                    float *dst = base + (size_t)(o0 + j) * ld + m;
                    if (part || ow) __stcg(dst, v[j]);
                    else atomicAdd(dst, v[j]);  // RED, fire-and-forget; one contribution per element
                }
            }
        }
    }
};

// ------------------------------------------------------------------------------------
// ------------------------------------------------------------------------------------
// Split-K wrapper for fprop / dgrad problems whose (M, N) tile grid is smaller than one wave
// of SMs (the 8 x 8 and 16 x 16 U-Net levels at batch 32: 16-64 M tiles).  Split z covers
// K-blocks [z kps, (z+1) kps); the epilogue stores the fp32 partial tile into slice z of a
// row-major [split][pixel][column] scratch buffer, and a finishing kernel (split_finish_*)
// adds the slices in split order (deterministic) and applies the problem's own epilogue
// (bias / ReLU / Dropout2d, or gradient-sum / ReLU-backward / split / planes / bias gradient).
template <class P>
struct SplitK {
    static constexpr bool A_MN = P::A_MN, B_MN = P::B_MN;
    static constexpr int EPI_STAGE = STAGE_BYTES;
    static constexpr bool BIAS_ROWS = true;
    P p;
    float *ws;
    size_t zstride;  // floats per split slice (pixels x ld)
    int ld, kps, total_kb;
    __device__ void kb_range(int z, int &kb0, int &nkb) const {
        kb0 = z * kps;
        nkb = min(kps, total_kb - kb0);
    }
    __device__ void prefetch() const { p.prefetch(); }
    template <int BN>
    __device__ void load(int kb, uint8_t *sa, uint8_t *sb, uint64_t *bar, int mt, int nt, int) const {
        p.template load<BN>(kb, sa, sb, bar, mt, nt, 0);
    }
    struct Pre {};
    template <int BN>
    __device__ void pre_load(Pre &, int, int, int, int, int, int) const {}
    template <int BN>
    __device__ void stash_bias(int, int, float *, int, float *) const {}
    template <int BN>
    __device__ void commit_bias(int, float *) const {}
    template <int BN>
    __device__ void epilogue(uint32_t tmem, int row, int mt, int nt, int z, int cc0, int cc1, float *, const Pre &,
                             uint8_t * = nullptr, const uint8_t * = nullptr) const {
        int n0, h0, w0, n, h, w;
        p.pt.origin(mt, n0, h0, w0);
        p.pt.pixel(row, n0, h0, w0, n, h, w);
        const bool valid = n < p.N;
        float *dst = ws + (size_t)z * zstride + (((size_t)n * p.H + h) * p.W + w) * ld + nt * BN;
#pragma unroll 1
        for (int cc = cc0; cc < cc1; ++cc) {
            float v[32];
            tc::tmem_ld32(tmem + cc * 32, v);
            if (!valid) continue;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                __stcg(reinterpret_cast<float4 *>(dst + cc * 32) + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
        }
    }
};

// sum of the nsplit partial slices of 8 consecutive floats, in split order
__device__ __forceinline__ void split_sum8(const float *ws, int nsplit, size_t zstride, size_t off, float (&v)[8]) {
    const float4 *s0 = reinterpret_cast<const float4 *>(ws + off);
    float4 a = __ldcg(s0), b = __ldcg(s0 + 1);
    for (int z = 1; z < nsplit; ++z) {
        const float4 *sz = reinterpret_cast<const float4 *>(ws + z * zstride + off);
        const float4 c = __ldcg(sz), d = __ldcg(sz + 1);
        a.x += c.x; a.y += c.y; a.z += c.z; a.w += c.w;
        b.x += d.x; b.y += d.y; b.z += d.z; b.w += d.w;
    }
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// y = act(sum_z ws[z] + bias) * drop, bf16.  One thread per 8 columns of one pixel.
__global__ void split_finish_fprop(const float *__restrict__ ws, int nsplit, long long npx, int hw, int cout,
                                   const float *__restrict__ bias, const float *__restrict__ drop, int relu,
                                   bf16 *__restrict__ y) {
    const int groups = cout / 8;
    const long long total = npx * groups;
    const size_t zstride = (size_t)npx * cout;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long px = i / groups;
        const int col = (int)(i - px * groups) * 8;
        float v[8], bq[8], dq[8];
        split_sum8(ws, nsplit, zstride, (size_t)px * cout + col, v);
        ld8(bias ? bias + col : nullptr, 0.f, bq);
        ld8(drop ? drop + (px / hw) * cout + col : nullptr, 1.f, dq);
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float x0 = v[2 * e] + bq[2 * e], x1 = v[2 * e + 1] + bq[2 * e + 1];
            if (relu) {
                x0 = fmaxf(x0, 0.f);
                x1 = fmaxf(x1, 0.f);
            }
            pk[e] = tc::pack_bf16(x0 * dq[2 * e], x1 * dq[2 * e + 1]);
        }
        *reinterpret_cast<uint4 *>(y + px * cout + col) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
}

// dgrad finish: the DgradProb epilogue on the split-ordered sums.  Block = 256 columns (32
// column groups of 8, one per lane) x FIN_STRIP pixels (8 warps, interleaved rows); the bias
// gradient column sums reduce through shared memory into row `strip` of p.bpart ([strips][ct]),
// which colsum_finish adds in strip order.
constexpr int FIN_STRIP = 64;
__global__ void __launch_bounds__(256) split_finish_dgrad(const float *__restrict__ ws, int nsplit, int npx, int N,
                                                          int H, int W, DgradProb p) {
    __shared__ float red[8][32][9];
    const int ct = p.c1 + p.c2, cblocks = ct / 256;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int cb = blockIdx.x % cblocks, strip = blockIdx.x / cblocks;
    const int cg = cb * 32 + lane;
    int col = cg * 8;
    bf16 *out;
    const bf16 *ref, *add;
    const float *drop;
    float *db;
    int cs;
    bool second = false;
    if (col < p.c1) {
        out = p.out1; ref = p.ref1; add = p.add1; drop = p.drop1; cs = p.c1; db = p.db1;
    } else {
        col -= p.c1;
        out = p.out2; ref = p.ref2; add = p.add2; drop = p.drop2; cs = p.c2; db = p.db2;
        second = true;
    }
    float dsum[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int px0 = strip * FIN_STRIP, px1 = min(npx, px0 + FIN_STRIP);
    for (int px = px0 + wid; px < px1; px += 8) {
        if (!out) continue;
        float v[8];
        split_sum8(ws, nsplit, (size_t)npx * ct, (size_t)px * ct + cg * 8, v);
        const int n = px / (H * W), hw = px - n * H * W, h = hw / W, w = hw - h * W;
        size_t pix = (size_t)px;
        if (second && p.planes_out2)
            pix = ((((size_t)((h & 1) * 2 + (w & 1)) * N + n) * (H >> 1) + (h >> 1)) * (W >> 1)) + (w >> 1);
        const size_t off = pix * cs + col;
        if (add) {
            const uint4 u = *reinterpret_cast<const uint4 *>(add + off);
            const bf16 *b8 = reinterpret_cast<const bf16 *>(&u);
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] += __bfloat162float(b8[e]);
        }
        if (!second && p.rbits1) {
            const uint32_t b = p.rbits1[(size_t)(col >> 5) * (size_t)npx + px] >> (col & 31);
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (!((b >> e) & 1u)) v[e] = 0.f;
        } else if (ref) {
            const uint4 u = *reinterpret_cast<const uint4 *>(ref + off);
            const bf16 *b8 = reinterpret_cast<const bf16 *>(&u);
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (!(__bfloat162float(b8[e]) > 0.f)) v[e] = 0.f;
        }
        if (drop) {
            float dq[8];
            ld8(drop + (size_t)n * cs + col, 1.f, dq);
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] *= dq[e];
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) dsum[e] += v[e];
        *reinterpret_cast<uint4 *>(out + off) =
            make_uint4(tc::pack_bf16(v[0], v[1]), tc::pack_bf16(v[2], v[3]), tc::pack_bf16(v[4], v[5]), tc::pack_bf16(v[6], v[7]));
    }
    if (!db || !out) return;  // block-uniform (one column region per block)
#pragma unroll
    for (int e = 0; e < 8; ++e) red[wid][lane][e] = dsum[e];
    __syncthreads();
    // 256 threads: thread -> (column group, element) = (tid >> 3, tid & 7)
    const int g = threadIdx.x >> 3, e = threadIdx.x & 7;
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][g][e];
    p.bpart[(size_t)strip * ct + (cb * 32 + g) * 8 + e] = t;
}

template <int BN, int STAGES>
constexpr int smem_bytes() {
    return 1024 + STAGES * (A_BYTES + BN * BK * 2) + EPI_WARPS * STAGE_BYTES + (2 * STAGES + 4) * 8 + 16 +
           BIAS_SLOTS * BN * 4;
}

// exact t / d for 0 <= t < 2^24 from a float reciprocal and one correction step
__device__ __forceinline__ int fdiv(int t, int d, float inv) {
    int q = __float2int_rz((float)t * inv);
    int r = t - q * d;
    if (r < 0) --q;
    else if (r >= d) ++q;
    return q;
}
struct TileGrid {  // persistent schedule: tile t -> (m fastest, then n, then split z)
    int tm, tn, tz;
    float itm, itn;  // 1 / tm, 1 / tn (tile_grid)
    __device__ __forceinline__ int count() const { return tm * tn * tz; }
    __device__ __forceinline__ void coords(int t, int &mt, int &nt, int &z) const {
        int q = fdiv(t, tm, itm);
        mt = t - q * tm;
        z = fdiv(q, tn, itn);
        nt = q - z * tn;
    }
};
TileGrid tile_grid(dim3 tiles) {
    return TileGrid{(int)tiles.x, (int)tiles.y, (int)tiles.z, 1.f / (float)tiles.x, 1.f / (float)tiles.y};
}

// Persistent, warp-specialised tcgen05 GEMM.  One CTA per SM walks the tile list; the
// TMA producer streams K-blocks through a STAGES-deep smem ring across tile boundaries,
// the MMA thread accumulates each tile into one of two TMEM accumulators (2 x BN fp32
// columns), and the 4 epilogue warps drain the other accumulator concurrently, so TMA,
// tensor cores and the epilogue all overlap.
template <int BN, int STAGES, class P>
__global__ void __launch_bounds__(NTHREADS, 1) conv_gemm(const __grid_constant__ P p, const TileGrid g) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int B_BYTES = BN * BK * 2;
    uint8_t *sa = base;
    uint8_t *sb = base + STAGES * A_BYTES;
    uint8_t *sst = sb + STAGES * B_BYTES;  // [EPI_WARPS][STAGE_BYTES] staged output boxes
    uint64_t *full = reinterpret_cast<uint64_t *>(sst + EPI_WARPS * STAGE_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;  // [2]
    uint64_t *tempty = tfull + 2;      // [2]
    uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 2);
    float *sbias = reinterpret_cast<float *>(tslot + 4);  // [BIAS_SLOTS][BN] (DgradProb)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = g.count();

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], EPI_WARPS);  // one arrive per epilogue warp
        }
        tc::fence_barrier_init();
    }
    if (warp == 0 && lane == 0) p.prefetch();
    if (warp == 1) tc::tmem_alloc<2 * BN>(tslot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int mt, nt, z, kb0, nkb;
                g.coords(t, mt, nt, z);
                p.kb_range(z, kb0, nkb);
                for (int i = 0; i < nkb; ++i, ++it) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    tc::mbar_wait(&empty[s], ph ^ 1);
                    tc::mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
                    p.template load<BN>(kb0 + i, sa + s * A_BYTES, sb + s * B_BYTES, &full[s], mt, nt, z);
                }
            }
        }
    } else if (warp == 1) {
        if (tc::issuer(lane)) {
            constexpr uint32_t idesc = tc::idesc_bf16(BM, BN, P::A_MN, P::B_MN);
            int it = 0, local = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
                int mt, nt, z, kb0, nkb;
                g.coords(t, mt, nt, z);
                p.kb_range(z, kb0, nkb);
                const int acc = local & 1;
                const uint32_t aph = (local >> 1) & 1;
                tc::mbar_wait(&tempty[acc], aph ^ 1);  // epilogue has drained this accumulator
                tc::tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int i = 0; i < nkb; ++i, ++it) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    tc::mbar_wait(&full[s], ph);
                    tc::tc_fence_after();
                    // descriptors built once per stage; per-k steps are plain adds of the
                    // encoded (addr >> 4) start field (smem offsets stay below 2^18, no carry)
                    const uint64_t ad0 = tc::sw128_desc(tc::smem_u32(sa + s * A_BYTES), P::A_MN ? 8192 : 16, 1024);
                    const uint64_t bd0 = tc::sw128_desc(tc::smem_u32(sb + s * B_BYTES), P::B_MN ? 8192 : 16, 1024);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        tc::mma(d, ad0 + (P::A_MN ? 128 : 2) * k, bd0 + (P::B_MN ? 128 : 2) * k, idesc,
                                     (i | k) != 0 ? 1u : 0u);
                    tc::mma_commit(&empty[s]);
                }
                tc::mma_commit(&tfull[acc]);
            }
        }
        __syncwarp();
    } else {
        const int sub = warp & 3, half = (warp - 2) >> 2;
        constexpr int NCH = BN / 32, PER = (NCH + 1) / 2;
        const int cc0 = half * PER, cc1 = min(NCH, (half + 1) * PER);
        float bacc[4] = {0.f, 0.f, 0.f, 0.f};  // fused bias-gradient partial sums (DgradProb)
        int cur_nt = -1;
        int local = 0;
        typename P::Pre pre;
        if (blockIdx.x < (unsigned)ntiles) {
            int mt, nt, z;
            g.coords(blockIdx.x, mt, nt, z);
            p.template pre_load<BN>(pre, sub * 32 + lane, mt, nt, z, cc0, cc1);
        }
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
            int mt, nt, z;
            g.coords(t, mt, nt, z);
            if (nt != cur_nt) {
                if (cur_nt >= 0) {
                    p.template stash_bias<BN>(cc0, cc1, bacc, sub, sbias);
                    p.template commit_bias<BN>(cur_nt, sbias);
                }
                cur_nt = nt;
            }
            const typename P::Pre cur = pre;
            if (t + (int)gridDim.x < ntiles) {  // next tile's epilogue operands, ahead of the wait
                int mt2, nt2, z2;
                g.coords(t + gridDim.x, mt2, nt2, z2);
                p.template pre_load<BN>(pre, sub * 32 + lane, mt2, nt2, z2, cc0, cc1);
            }
            const int acc = local & 1;
            tc::mbar_wait(&tfull[acc], (local >> 1) & 1);
            tc::tc_fence_after();
            p.template epilogue<BN>(tmem + acc * BN + ((uint32_t)(sub * 32) << 16), sub * 32 + lane, mt, nt, z, cc0,
                                    cc1, bacc, cur, P::EPI_STAGE == STAGE_BYTES ? sst + (warp - 2) * STAGE_BYTES : nullptr);
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
        }
        if (cur_nt >= 0) {
            p.template stash_bias<BN>(cc0, cc1, bacc, sub, sbias);
            p.template commit_bias<BN>(cur_nt, sbias);
        }
        if (lane == 0) tc::bulk_wait<0>();  // staged stores complete before the CTA ends
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc<2 * BN>(tmem);
}

// 256 x 256 tiles: two 128-row M halves share every B block, so a K-block moves 64 KB
// through L2 for 2 x 128 x 256 x 64 MACs instead of 96 KB for two 128 x 256 tiles.  The
// 128-row wgrad is L2-throughput bound (a TMA-only replay of it streams 12 TB/s, the LTS
// cap; its MMA-only replay runs at 1.84 PFLOP/s).  Both halves fill TMEM (2 x 256 columns),
// so the epilogue drains between tiles instead of overlapping the next one: used where a
// CTA owns few, long tiles.  Each epilogue warp drains its 32 TMEM lanes of one M half in
// two 128-column passes (the problems' epilogues take 4 chunks per call).  BN = 128 (layers
// with 128 output columns): 256 x 128 tiles move 48 KB per K-block for 256 x 128 x 64 MACs
// (a 128 x 128 tile: 32 KB for half of that) and two accumulator pairs fit TMEM, so the
// epilogue overlaps the next tile as in conv_gemm.
#ifdef ICE_CONV_PROF
// MMA-thread cycle accounting of conv_gemm_m2 (debug build): [0] waiting for the epilogue
// (tmem empty), [1] waiting for TMA (full), [2] issuing, [3] tiles, [4] K-blocks
__device__ unsigned long long g_conv_prof[8];
#endif
template <int BN, int STAGES, class P>
constexpr int m2_smem_bytes() {
    return 1024 + STAGES * (2 * A_BYTES + BN * BK * 2) + EPI_WARPS * P::EPI_STAGE + (2 * STAGES + 4) * 8 + 16 +
           (P::BIAS_ROWS ? BIAS_SLOTS * BN * 4 : 0);
}

template <int BN, int STAGES, class P>
__global__ void __launch_bounds__(NTHREADS, 1) conv_gemm_m2(const __grid_constant__ P p, const TileGrid g) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int AB = 2 * A_BYTES, B_BYTES = BN * BK * 2;
    constexpr int NACC = 4 * BN <= 512 ? 2 : 1;  // BN = 128: two accumulator pairs, epilogue overlapped
    uint8_t *sa = base;
    uint8_t *sb = base + STAGES * AB;
    uint8_t *sst = sb + STAGES * B_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(sst + EPI_WARPS * P::EPI_STAGE);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;  // [2]
    uint64_t *tempty = tfull + 2;      // [2]
    uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 2);
    float *sbias = reinterpret_cast<float *>(tslot + 4);  // [BIAS_SLOTS][BN] (DgradProb)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = g.count();
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], EPI_WARPS);
        }
        tc::fence_barrier_init();
    }
    if (warp == 0 && lane == 0) p.prefetch();
    if (warp == 1) tc::tmem_alloc<512>(tslot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int mt, nt, z, kb0, nkb;
                g.coords(t, mt, nt, z);
                p.kb_range(z, kb0, nkb);
                for (int i = 0; i < nkb; ++i, ++it) {
                    const int s = it % STAGES;
                    tc::mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
                    tc::mbar_expect_tx(&full[s], AB + B_BYTES);
                    p.template load_m2<BN>(kb0 + i, sa + s * AB, sb + s * B_BYTES, &full[s], mt, nt, z);
                }
            }
        }
    } else if (warp == 1) {
        if (tc::issuer(lane)) {
            constexpr uint32_t idesc = tc::idesc_bf16(BM, BN, P::A_MN, P::B_MN);
            int it = 0, local = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
                int mt, nt, z, kb0, nkb;
                g.coords(t, mt, nt, z);
                p.kb_range(z, kb0, nkb);
                const int acc = local % NACC;
#ifdef ICE_CONV_PROF
                long long q0 = clock64();
#endif
                tc::mbar_wait(&tempty[acc], ((local / NACC) & 1) ^ 1);
                tc::tc_fence_after();
#ifdef ICE_CONV_PROF
                long long q1 = clock64();
                if (lane == 0) {
                    atomicAdd(&g_conv_prof[0], (unsigned long long)(q1 - q0));
                    atomicAdd(&g_conv_prof[3], 1ull);
                }
#endif
                const uint32_t d = tmem + acc * 2 * BN;
                for (int i = 0; i < nkb; ++i, ++it) {
                    const int s = it % STAGES;
#ifdef ICE_CONV_PROF
                    const long long w0 = clock64();
#endif
                    tc::mbar_wait(&full[s], (it / STAGES) & 1);
                    tc::tc_fence_after();
#ifdef ICE_CONV_PROF
                    const long long w1 = clock64();
                    if (lane == 0) {
                        atomicAdd(&g_conv_prof[1], (unsigned long long)(w1 - w0));
                        atomicAdd(&g_conv_prof[4], 1ull);
                    }
#endif
                    const uint64_t a0 = tc::sw128_desc(tc::smem_u32(sa + s * AB), P::A_MN ? 8192 : 16, 1024);
                    const uint64_t a1 = tc::sw128_desc(tc::smem_u32(sa + s * AB + A_BYTES), P::A_MN ? 8192 : 16, 1024);
                    const uint64_t b0 = tc::sw128_desc(tc::smem_u32(sb + s * B_BYTES), P::B_MN ? 8192 : 16, 1024);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const uint64_t bk = b0 + (P::B_MN ? 128 : 2) * k;
                        tc::mma(d, a0 + (P::A_MN ? 128 : 2) * k, bk, idesc, (i | k) != 0 ? 1u : 0u);
                        tc::mma(d + BN, a1 + (P::A_MN ? 128 : 2) * k, bk, idesc, (i | k) != 0 ? 1u : 0u);
                    }
                    tc::mma_commit(&empty[s]);
                }
                tc::mma_commit(&tfull[acc]);
            }
        }
        __syncwarp();
    } else {
        const int sub = warp & 3, half = (warp - 2) >> 2;  // TMEM lane quarter, M half
        const int row = sub * 32 + lane;
        constexpr int NCH = BN / 32, PER = (NCH + 1) / 2;  // two passes of PER chunks
        uint8_t *stage = sst + (warp - 2) * P::EPI_STAGE;
        float bacc0[4] = {0.f, 0.f, 0.f, 0.f}, bacc1[4] = {0.f, 0.f, 0.f, 0.f};
        int cur_nt = -1, local = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
            int mt, nt, z;
            g.coords(t, mt, nt, z);
            if (nt != cur_nt) {
                if (cur_nt >= 0) {
                    p.template stash_bias<BN>(0, PER, bacc0, half * 4 + sub, sbias);
                    p.template stash_bias<BN>(PER, NCH, bacc1, half * 4 + sub, sbias);
                    p.template commit_bias<BN>(cur_nt, sbias);
                }
                cur_nt = nt;
            }
            typename P::Pre pre0, pre1;  // operands issued before the wait (hidden by the mainloop)
            p.template pre_load<BN>(pre0, row, 2 * mt + half, nt, z, 0, PER);
            p.template pre_load<BN>(pre1, row, 2 * mt + half, nt, z, PER, NCH);
            const int acc = local % NACC;
            tc::mbar_wait(&tfull[acc], (local / NACC) & 1);
            tc::tc_fence_after();
            const uint32_t tm = tmem + acc * 2 * BN + half * BN + ((uint32_t)(sub * 32) << 16);
            p.template epilogue<BN>(tm, row, 2 * mt + half, nt, z, 0, PER, bacc0, pre0, stage);
            p.template epilogue<BN>(tm, row, 2 * mt + half, nt, z, PER, NCH, bacc1, pre1, stage);
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
        }
        if (cur_nt >= 0) {
            p.template stash_bias<BN>(0, PER, bacc0, half * 4 + sub, sbias);
            p.template stash_bias<BN>(PER, NCH, bacc1, half * 4 + sub, sbias);
            p.template commit_bias<BN>(cur_nt, sbias);
        }
        if (lane == 0) tc::bulk_wait<0>();  // staged stores complete before the CTA ends
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

// Row-halo variant for 3x3 convs on wide images (W % 128 == 0; U-Net levels 0-1, where
// the channel count is 64-128 and a per-tap TMA box per K-block would make the tile
// latency/L2-bound).  An M tile is 128 consecutive pixels of one image row; per 64-channel
// chunk the producer loads ONE 3 x 130-pixel halo slab (49,920 B, zero-filled outside the
// image) and the 9 taps read their A operands as 128-row windows of that slab starting at
// row (dy+1)*130 + (dx+1) -- the SW128 swizzle is address-based, so an unaligned window
// start needs no descriptor base offset (probed on B200).  Weights stream through their own
// BSTAGES-deep ring, one (tap, chunk) slab per stage.
constexpr int HALO_ROWS = 3 * 130;
constexpr int HALO_TX = HALO_ROWS * 128;        // bytes a halo load delivers
constexpr int HALO_BYTES = (HALO_TX + 1023) / 1024 * 1024;

constexpr int TAPS_PER_SLOT = 3;
// PAIR tiles: two 128-pixel tiles of consecutive rows (same columns) share every weight stage.
// Their halo is ONE 4 x 130-pixel slab (rows h0-1 .. h0+2; sub-tile s reads windows s rows
// lower), so per 256 pixels the weights are streamed once instead of twice and the halo is
// 4 rows instead of 6: for the 128-wide streamed-weight tiles the shared-memory traffic per
// MAC (operand reads + TMA writes + staged stores) drops ~16%, and that traffic is what bounds
// them.  Weights then stream one tap per stage (the two halo buffers take 130 KB).
constexpr int HALO4_TX = 4 * 130 * 128;
// first 128-pixel tile (row tile index of PixTile: w fastest, then h, then n) of pair tile u:
// rows 2k and 2k + 1 of an image are tiles t0 and t0 + tw
__device__ __forceinline__ int pair_first(int u, const PixTile &pt) {
    return ((u >> lg2(pt.tw)) << (lg2(pt.tw) + 1)) | (u & (pt.tw - 1));
}
constexpr int HALO4_BYTES = (HALO4_TX + 1023) / 1024 * 1024;
constexpr int REF_BYTES = 128 * 128;  // staged ReLU-reference tile: 128 px x 64 ch bf16  // one kernel row per weight stage: 12 MMAs per barrier wait

template <int BN, int BSTAGES, bool RES, bool PAIR = false>
constexpr int halo_smem_bytes(bool refs = false) {
    return 1024 + 2 * (PAIR ? HALO4_BYTES : HALO_BYTES) + (RES ? 9 : BSTAGES * (PAIR ? 1 : TAPS_PER_SLOT)) * BN * BK * 2 +
           (((BN == 64 && (RES || PAIR)) || BN == 128) ? EPI_WARPS * STAGE_BUFS * STAGE_BYTES : 0) +
           ((BN == 64 && RES && refs) ? 2 * REF_BYTES : 0) +
           (2 * 2 + 2 * BSTAGES + 6 + 4) * 8 + 16 + BIAS_SLOTS * BN * 4;
}

// RES (resident weights): single-chunk problems (64 input channels) keep all 9 weight taps
// of the current column tile in smem; they are reloaded only when the persistent CTA moves
// to another column tile, so the MMA thread waits once per tile (36 MMAs per wait).
template <int BN, int BSTAGES, bool RES, class P, bool DUAL, bool PAIR = false>
__global__ void __launch_bounds__(NTHREADS + (DUAL ? 32 : 0), 1) halo_gemm(const __grid_constant__ P p, const TileGrid g) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    static_assert(!PAIR || (!RES && !DUAL), "pair tiles stream their weights");
    constexpr int NSUB = PAIR ? 2 : 1;                 // 128-pixel sub-tiles per tile
    constexpr int TPS = PAIR ? 1 : TAPS_PER_SLOT;      // weight taps per stage
    constexpr int HB = PAIR ? HALO4_BYTES : HALO_BYTES, HTX = PAIR ? HALO4_TX : HALO_TX;
    constexpr int B_TAP = BN * BK * 2;
    constexpr int B_BYTES = RES ? 9 * B_TAP : TPS * B_TAP;
    constexpr int NBS = RES ? 1 : BSTAGES;
    // BN = 64 resident-weight tiles stage each warp's 32 x 32 output box in shared memory and
    // write it with a TMA store (per-lane 64-B row stores were the epilogue's bottleneck)
    constexpr bool STAGE = (BN == 64 && (RES || PAIR)) || BN == 128;
    uint8_t *sa = base;            // [2][HB]
    uint8_t *sb = base + 2 * HB;   // [NBS][B_BYTES]
    uint8_t *sst = sb + NBS * B_BYTES;     // [EPI_WARPS][STAGE_BUFS][STAGE_BYTES] when STAGE
    // ... and TMA-stage the tile's ReLU reference (dgrad) for the epilogue
    constexpr bool REFS = BN == 64 && RES && P::STAGE_REF;
    uint8_t *sref = sst + (STAGE ? EPI_WARPS * STAGE_BUFS * STAGE_BYTES : 0);  // [2][REF_BYTES] when REFS
    uint64_t *afull = reinterpret_cast<uint64_t *>(sref + (REFS ? 2 * REF_BYTES : 0));
    uint64_t *aempty = afull + 2;
    uint64_t *bfull = aempty + 2;
    uint64_t *bempty = bfull + BSTAGES;
    uint64_t *tfull = bempty + BSTAGES;
    uint64_t *tempty = tfull + 2;
    uint64_t *rfull = tempty + 2;   // [2]
    uint64_t *rempty = rfull + 2;   // [2]
    uint32_t *tslot = reinterpret_cast<uint32_t *>(rempty + 2);
    float *sbias = reinterpret_cast<float *>(tslot + 4);  // [BIAS_SLOTS][BN] (DgradProb)
    const bool stage_ref = REFS && p.ref_tma;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = g.count();
    const int nch = p.halo_chunks();

    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&afull[s], 1);
            tc::mbar_init(&aempty[s], 1);
            tc::mbar_init(&tfull[s], 1);
            tc::mbar_init(&tempty[s], EPI_WARPS);
            tc::mbar_init(&rfull[s], 1);
            tc::mbar_init(&rempty[s], EPI_WARPS);
        }
        for (int s = 0; s < BSTAGES; ++s) {
            tc::mbar_init(&bfull[s], 1);
            tc::mbar_init(&bempty[s], 1);
        }
        tc::fence_barrier_init();
    }
    if (warp == 0 && lane == 0) p.prefetch();
    if (warp == 1) tc::tmem_alloc<2 * BN * NSUB>(tslot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            int ait = 0, bit = 0, cur_nt = -1, run = -1, lt = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
                int mt, nt, z;
                g.coords(t, mt, nt, z);
                if (REFS && stage_ref) {  // the epilogue's ReLU reference for this tile
                    const int rs = lt & 1;
                    tc::mbar_wait(&rempty[rs], ((lt >> 1) & 1) ^ 1);
                    tc::mbar_expect_tx(&rfull[rs], REF_BYTES);
                    p.load_ref(sref + rs * REF_BYTES, &rfull[rs], mt, nt);
                }
                if (RES && nt != cur_nt) {  // (re)load the column tile's 9 weight taps
                    if (run >= 0) tc::mbar_wait(&bempty[0], run & 1);
                    ++run;
                    cur_nt = nt;
                    tc::mbar_expect_tx(&bfull[0], B_BYTES);
                    for (int tap = 0; tap < 9; ++tap) p.template load_tap_b<BN>(tap, 0, sb + tap * B_TAP, &bfull[0], nt);
                }
                for (int ch = 0; ch < nch; ++ch, ++ait) {
                    const int as = ait & 1;
                    tc::mbar_wait(&aempty[as], ((ait >> 1) & 1) ^ 1);
#ifdef ICE_EXP_NOTMA
                    tc::mbar_arrive(&afull[as]);
#else
                    tc::mbar_expect_tx(&afull[as], HTX);
                    p.load_halo(ch, sa + as * HB, &afull[as], PAIR ? pair_first(mt, p.pt) : mt);
#endif
                    if (RES) continue;
                    for (int r = 0; r < 9 / TPS; ++r, ++bit) {
                        const int bs = bit % BSTAGES;
                        tc::mbar_wait(&bempty[bs], ((bit / BSTAGES) & 1) ^ 1);
                        tc::mbar_expect_tx(&bfull[bs], B_BYTES);
                        for (int q = 0; q < TPS; ++q)
                            p.template load_tap_b<BN>(r * TPS + q, ch, sb + bs * B_BYTES + q * B_TAP,
                                                      &bfull[bs], nt);
                    }
                }
            }
        }
    } else if (DUAL && (warp == 1 || warp == 2 + EPI_WARPS)) {
        // Two MMA issuers (single column tile, resident weights): the tensor pipe accepts an
        // MMA only when the previous one is nearly done, so an issuer's per-tile barrier waits
        // and bookkeeping would idle it; issuer i owns the CTA's tiles j = i mod 2 together
        // with A slot i and accumulator i, and the other issuer's MMAs fill its gaps.
        if (tc::issuer(lane)) {
            constexpr uint32_t idesc = tc::idesc_bf16(BM, BN, false, P::B_MN);
            const int iss = warp == 1 ? 0 : 1;
            uint32_t voff[9];
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) voff[tap] = p.view_row(tap) * 8;
            const uint64_t adesc = tc::sw128_desc(tc::smem_u32(sa + iss * HB), 16, 1024);
            const uint64_t bdesc = tc::sw128_desc(tc::smem_u32(sb), P::B_MN ? 8192 : 16, 1024);
            const uint32_t d = tmem + iss * BN;
            tc::mbar_wait(&bfull[0], 0);
            int j = iss;
            for (int t = blockIdx.x + iss * gridDim.x; t < ntiles; t += 2 * gridDim.x, j += 2) {
                const uint32_t ph = (j >> 1) & 1;
                tc::mbar_wait(&tempty[iss], ph ^ 1);
                tc::mbar_wait(&afull[iss], ph);
                tc::tc_fence_after();
#pragma unroll
                for (int tap = 0; tap < 9; ++tap) {
                    const uint64_t ad = adesc + voff[tap];
                    const uint64_t bd = bdesc + tap * (B_TAP >> 4);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        tc::mma(d, ad + 2 * k, bd + (P::B_MN ? 128 : 2) * k, idesc, (tap | k) != 0 ? 1u : 0u);
                }
                tc::mma_commit(&aempty[iss]);
                tc::mma_commit(&tfull[iss]);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (tc::issuer(lane)) {
            constexpr uint32_t idesc = tc::idesc_bf16(BM, BN, false, P::B_MN);
            // per-tap window offsets in descriptor units (128 B halo rows), hoisted out of the
            // tile loop: a constant-bank load chain per tap would stall every tap's first MMA
            uint32_t voff[9];
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) voff[tap] = p.view_row(tap) * 8;
            int ait = 0, bit = 0, local = 0, cur_nt = -1, run = -1;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
                int mt, nt, z;
                g.coords(t, mt, nt, z);
                if (RES && nt != cur_nt) {
                    ++run;
                    cur_nt = nt;
                    tc::mbar_wait(&bfull[0], run & 1);
                }
                const int acc = local & 1;
                tc::mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
                tc::tc_fence_after();
                const uint32_t d = tmem + acc * BN * NSUB;
                for (int ch = 0; ch < nch; ++ch, ++ait) {
                    const int as = ait & 1;
                    tc::mbar_wait(&afull[as], (ait >> 1) & 1);
                    tc::tc_fence_after();
                    const uint64_t adesc = tc::sw128_desc(tc::smem_u32(sa + as * HB), 16, 1024);
#pragma unroll
                    for (int r = 0; r < 9 / TPS; ++r) {
                        int bs = 0;
                        uint32_t bslot;
                        if (RES) {
                            bslot = tc::smem_u32(sb + r * TPS * B_TAP);
                        } else {
                            bs = bit % BSTAGES;
                            tc::mbar_wait(&bfull[bs], (bit / BSTAGES) & 1);
                            tc::tc_fence_after();
                            bslot = tc::smem_u32(sb + bs * B_BYTES);
                        }
                        const uint64_t bdesc = tc::sw128_desc(bslot, P::B_MN ? 8192 : 16, 1024);
#pragma unroll
                        for (int q = 0; q < TPS; ++q) {
                            const int tap = r * TPS + q;
                            const uint64_t bd = bdesc + q * (B_TAP >> 4);
#pragma unroll
                            for (int sub = 0; sub < NSUB; ++sub) {  // sub-tile sub: windows sub rows lower
                                const uint64_t ad = adesc + voff[tap] + sub * 130 * 8;
#pragma unroll
                                for (int k = 0; k < BK / 16; ++k)
                                    tc::mma(d + sub * BN, ad + 2 * k, bd + (P::B_MN ? 128 : 2) * k, idesc,
                                            (ch | tap | k) != 0 ? 1u : 0u);
                            }
                        }
                        if (!RES) {
                            tc::mma_commit(&bempty[bs]);
                            ++bit;
                        }
                    }
                    tc::mma_commit(&aempty[as]);
                }
                tc::mma_commit(&tfull[acc]);
                if (RES) {  // last tile of this column run: release the resident weights
                    int nmt, nnt = -1, nz;
                    if (t + (int)gridDim.x < ntiles) g.coords(t + gridDim.x, nmt, nnt, nz);
                    if (nnt != nt) tc::mma_commit(&bempty[0]);
                }
            }
        }
        __syncwarp();
    } else if (warp < 2 + EPI_WARPS) {
        const int sub = warp & 3, half = (warp - 2) >> 2;
        constexpr int NCH = BN / 32, PER = (NCH + 1) / 2;
        const int cc0 = half * PER, cc1 = min(NCH, (half + 1) * PER);
        float bacc[4] = {0.f, 0.f, 0.f, 0.f};  // fused bias-gradient partial sums (DgradProb)
        int cur_nt = -1;
        int local = 0;
        typename P::Pre pre;
        if (blockIdx.x < (unsigned)ntiles) {
            int mt, nt, z;
            g.coords(blockIdx.x, mt, nt, z);
            p.template pre_load<BN>(pre, sub * 32 + lane, PAIR ? pair_first(mt, p.pt) : mt, nt, z, cc0, cc1);
        }
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
            int mt, nt, z;
            g.coords(t, mt, nt, z);
            if (nt != cur_nt) {
                if (cur_nt >= 0) {
                    p.template stash_bias<BN>(cc0, cc1, bacc, sub, sbias);
                    p.template commit_bias<BN>(cur_nt, sbias);
                }
                cur_nt = nt;
            }
            const int acc = local & 1;
            const int m0 = PAIR ? pair_first(mt, p.pt) : mt;
#pragma unroll 1
            for (int s2 = 0; s2 < NSUB; ++s2) {  // (one copy of the epilogue: instruction cache)
                const typename P::Pre cur = pre;
                // the next sub-tile's epilogue operands, ahead of the accumulator wait
                if (s2 + 1 < NSUB) {
                    p.template pre_load<BN>(pre, sub * 32 + lane, m0 + p.pt.tw, nt, z, cc0, cc1);
                } else if (t + (int)gridDim.x < ntiles) {
                    int mt2, nt2, z2;
                    g.coords(t + gridDim.x, mt2, nt2, z2);
                    p.template pre_load<BN>(pre, sub * 32 + lane, PAIR ? pair_first(mt2, p.pt) : mt2, nt2, z2, cc0, cc1);
                }
                if (s2 == 0) {
                    tc::mbar_wait(&tfull[acc], (local >> 1) & 1);
                    tc::tc_fence_after();
                    if (REFS && stage_ref) tc::mbar_wait(&rfull[acc], (local >> 1) & 1);
                }
#ifndef ICE_EXP_NOEPI
                p.template epilogue<BN>(tmem + (acc * NSUB + s2) * BN + ((uint32_t)(sub * 32) << 16), sub * 32 + lane,
                                        m0 + s2 * p.pt.tw, nt, z, cc0, cc1, bacc, cur,
                                        STAGE ? sst + ((warp - 2) * STAGE_BUFS + acc % STAGE_BUFS) * STAGE_BYTES : nullptr,
                                        (REFS && stage_ref) ? sref + acc * REF_BYTES : nullptr);
#endif
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                tc::mbar_arrive(&tempty[acc]);
                if (REFS && stage_ref) tc::mbar_arrive(&rempty[acc]);
            }
        }
        if (cur_nt >= 0) {
            p.template stash_bias<BN>(cc0, cc1, bacc, sub, sbias);
            p.template commit_bias<BN>(cur_nt, sbias);
        }
        if (STAGE && lane == 0) tc::bulk_wait<0>();  // staged stores complete before the CTA ends
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc<2 * BN * NSUB>(tmem);
}

// Row-halo weight gradient for 3x3 convs with narrow outputs (cout 64/128) on wide images
// (W % 64 == 0, U-Net levels 0-1).  Transposed GEMM D[(tap, cin)][cout] = sum_p x[p+s_t] dY[p]:
// a K-block is a 64-pixel row segment; per K-block the producer loads, for every 64-channel
// chunk of x, ONE 3 x 66-pixel halo slab (zero-filled outside the image) plus the dY segment.
// An M tile is a pair of (tap, chunk) windows of those slabs (MN-major, K = pixel rows): the
// two 64-row blocks sit at arbitrary row offsets, expressed through the descriptor's LBO
// (unaligned windows / LBO are legal, the swizzle is address-based -- probed on B200).  A CTA
// owns a group of G M tiles (G x cout <= 512 TMEM columns) for a split of the pixels, so each
// K-block feeds G x 4 MMAs from one barrier wait.
struct HWgrad {
    CUtensorMap xm[4];  // per 64-channel chunk: halo box (64, 66, 3, 1) on its source
    CUtensorMap dym;    // dY: (64 ch x 64 px x cout/64 blocks)
    int N, H, W, ct, cout, nchx;
    int total_kb, kb_per_split, groups, G, total_mt;
    float *dw;  // [cout][9][ct]
    float *ws;  // partials of splits 1.. [splits - 1][cout][9][ct] (scratch)
    size_t wsize;
    int ow;     // gradient overwrite mode: split 0 stores instead of adding
};

// HALVE variant (2x2 halving conv, model.py:79-88): dW[(a,b), c] accumulates, for each of
// the 4 sub-pixel classes (cy, cx), x[p + ((cy+a)/2, (cx+b)/2)] (x) dY_cls[p]; the halo is
// 2 rows x 65 pixels and the dY segment comes as 4 class planes.
// KR: output rows per K-block.  The 3x3 variant takes two output rows (128 pixels) per K-block
// from one 4-row halo slab: every x row is fetched twice instead of three times, and each
// barrier wait feeds twice the MMAs (the 1-row form was L2-bound: 58 KB per K-block of 64
// pixels at cin 128, ~17 TB/s of L2 reads at the MMA rate).
template <bool HALVE>
struct HWGeom {
    static constexpr int KR = HALVE ? 1 : 2;
    static constexpr int ROWS = HALVE ? 2 : 4, COLS = HALVE ? 65 : 66;
    static constexpr int TX = ROWS * COLS * 128;
    static constexpr int BYTES = (TX + 1023) / 1024 * 1024;
    static constexpr int TAPS = HALVE ? 4 : 9;
    static constexpr int CLASSES = HALVE ? 4 : 1;
};

template <int COUT, int NCH, int STAGES, bool HALVE>
constexpr int hw_stage_bytes() {
    return NCH * HWGeom<HALVE>::BYTES + HWGeom<HALVE>::CLASSES * (COUT / 64) * 8192 * HWGeom<HALVE>::KR;
}
template <int COUT, int NCH, int STAGES, bool HALVE>
constexpr int hw_smem_bytes() {
    return 1024 + STAGES * hw_stage_bytes<COUT, NCH, STAGES, HALVE>() + (2 * STAGES + 2) * 8 + 16;
}

// halo row of the window for weight tap `tap` (and sub-pixel class `cls` for HALVE)
template <bool HALVE>
__device__ __forceinline__ int hw_view_row(int tap, int cls) {
    if (HALVE) return (((cls >> 1) + (tap >> 1)) >> 1) * 65 + (((cls & 1) + (tap & 1)) >> 1);
    return (tap / 3) * 66 + tap % 3;
}

template <int COUT, int NCH, int STAGES, bool HALVE>
__global__ void __launch_bounds__(NTHREADS, 1) hwgrad_kernel(const __grid_constant__ HWgrad p) {
    using G = HWGeom<HALVE>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int STAGE = hw_stage_bytes<COUT, NCH, STAGES, HALVE>();
    constexpr int DY_BYTES = (COUT / 64) * 8192 * G::KR;  // [cout block][KR rows][64 px][64 ch]
    constexpr int TX = NCH * G::TX + G::CLASSES * DY_BYTES;
    constexpr int NBLK = G::TAPS * NCH;  // M blocks: (tap, chunk), tap-major
    constexpr int TCOLS = 512;
    uint64_t *full = reinterpret_cast<uint64_t *>(base + STAGES * STAGE);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 1;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int units = p.groups * ((p.total_kb + p.kb_per_split - 1) / p.kb_per_split);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(tfull, 1);
        tc::mbar_init(tempty, EPI_WARPS);
        tc::fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        for (int c = 0; c < NCH; ++c) tc::tma_prefetch_desc(&p.xm[c]);
        tc::tma_prefetch_desc(&p.dym);
    }
    if (warp == 1) tc::tmem_alloc<TCOLS>(tslot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tslot;
    const int segs = p.W / 64;

    if (warp == 0) {
        if (lane == 0) {
            int it = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const int split = u / p.groups;
                const int kb0 = split * p.kb_per_split, kb1 = min(p.total_kb, kb0 + p.kb_per_split);
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % STAGES;
                    tc::mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
                    tc::mbar_expect_tx(&full[s], TX);
                    const int seg = kb & (segs - 1), row = kb >> lg2(segs);  // W, H powers of two
                    const int hk = p.H / G::KR;  // K-block rows per image
                    const int h = (row & (hk - 1)) * G::KR, n = row >> lg2(hk), w0 = seg * 64;
                    uint8_t *st = base + s * STAGE;
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
                        tc::tma_load_4d(st + c * G::BYTES, &p.xm[c], &full[s], 0, w0 - (HALVE ? 0 : 1),
                                        h - (HALVE ? 0 : 1), n);
#pragma unroll
                    for (int cls = 0; cls < G::CLASSES; ++cls) {
                        const int img = HALVE ? cls * p.N + n : n;  // class planes flatten to 4N images
                        uint8_t *dst = st + NCH * G::BYTES + cls * DY_BYTES;
                        if (COUT == 64) tc::tma_load_4d(dst, &p.dym, &full[s], 0, w0, h, img);
                        else tc::tma_load_5d(dst, &p.dym, &full[s], 0, w0, h, img, 0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (tc::issuer(lane)) {
            constexpr uint32_t idesc = tc::idesc_bf16(BM, COUT, true, true);
            int it = 0, local = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x, ++local) {
                const int grp = u % p.groups, split = u / p.groups;
                const int kb0 = split * p.kb_per_split, kb1 = min(p.total_kb, kb0 + p.kb_per_split);
                const int mt0 = grp * p.G, mt1 = min(p.total_mt, mt0 + p.G);
                tc::mbar_wait(tempty, (local & 1) ^ 1);
                tc::tc_fence_after();
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % STAGES;
                    tc::mbar_wait(&full[s], (it / STAGES) & 1);
                    tc::tc_fence_after();
                    const uint32_t st = tc::smem_u32(base + s * STAGE);
#pragma unroll
                    for (int cls = 0; cls < G::CLASSES; ++cls) {
                        const uint32_t bbase = st + NCH * G::BYTES + cls * DY_BYTES;
                        for (int mt = mt0; mt < mt1; ++mt) {
                            // blocks 2 mt, 2 mt + 1 of the (tap, chunk) list; a missing one repeats the first
                            const int b0 = 2 * mt, b1 = min(2 * mt + 1, NBLK - 1);
                            const uint32_t a0 = st + (b0 % NCH) * G::BYTES + hw_view_row<HALVE>(b0 / NCH, cls) * 128;
                            const uint32_t a1 = st + (b1 % NCH) * G::BYTES + hw_view_row<HALVE>(b1 / NCH, cls) * 128;
                            // LBO must not be negative: swap the blocks and remember it in the epilogue
                            const bool sw = a1 < a0;
                            const uint32_t lo = sw ? a1 : a0, dl = sw ? a0 - a1 : a1 - a0;
                            const uint32_t d = tmem + (mt - mt0) * COUT;
#pragma unroll
                            for (int orow = 0; orow < G::KR; ++orow) {  // output row orow: halo rows + orow
                                const uint64_t ad = tc::sw128_desc(lo + orow * G::COLS * 128, dl, 1024);
                                const uint64_t bd = tc::sw128_desc(bbase + orow * 8192, 8192 * G::KR, 1024);
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    tc::mma(d, ad + 128 * k, bd + 128 * k, idesc,
                                                 (kb > kb0 || cls > 0 || orow > 0 || k > 0) ? 1u : 0u);
                            }
                        }
                    }
                    tc::mma_commit(&empty[s]);
                }
                tc::mma_commit(tfull);
            }
        }
        __syncwarp();
    } else {
        const int sub = warp & 3, half = (warp - 2) >> 2;
        const int r = sub * 32 + lane;  // TMEM lane = row of the M tile
        constexpr int NCC = COUT / 32, PER = (NCC + 1) / 2;
        const int ld = G::TAPS * p.ct;
        int local = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++local) {
            const int grp = u % p.groups, split = u / p.groups;
            const int mt0 = grp * p.G, mt1 = min(p.total_mt, mt0 + p.G);
            const bool part = split > 0;
            float *base = part ? p.ws + (size_t)(split - 1) * p.wsize : p.dw;
            tc::mbar_wait(tfull, local & 1);
            tc::tc_fence_after();
            for (int mt = mt0; mt < mt1; ++mt) {
                // row r of the tile is block (2 mt + r/64) unless the issuer swapped the pair
                const int b0 = 2 * mt, b1 = min(2 * mt + 1, NBLK - 1);
                // the swap decision depends on the view rows; it is class-independent for the
                // pairs used here (same tap, different chunk, or taps in increasing halo order)
                const int v0 = (b0 % NCH) * G::BYTES + hw_view_row<HALVE>(b0 / NCH, 0) * 128;
                const int v1 = (b1 % NCH) * G::BYTES + hw_view_row<HALVE>(b1 / NCH, 0) * 128;
                const bool sw = v1 < v0;
                const int second = (r >> 6) ^ (sw ? 1 : 0);
                const int b = 2 * mt + second;
                const bool valid = b < NBLK && !(second == 1 && b1 == b0);
                const int tap = b / NCH, c = (b % NCH) * 64 + (r & 63);
                // split 0: dw += (its only writer in the launch); split s > 0: store slice s - 1
                // of ws (lanes hold consecutive channels: 128-B coalesced stores), added in
                // split order by splitsum_finish
                float *dst = base + (size_t)tap * p.ct + c;
#pragma unroll
                for (int cc = half * PER; cc < min(NCC, (half + 1) * PER); ++cc) {
                    float v[32];
                    tc::tmem_ld32(tmem + (mt - mt0) * COUT + cc * 32 + ((uint32_t)(sub * 32) << 16), v);
                    if (!valid) continue;
                    if (part || p.ow) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) __stcg(dst + (size_t)(cc * 32 + j) * ld, v[j]);
                    } else {  // RED (fire-and-forget): the launch's one contribution per element
#pragma unroll
                        for (int j = 0; j < 32; ++j) atomicAdd(dst + (size_t)(cc * 32 + j) * ld, v[j]);
                    }
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tempty);
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc<TCOLS>(tmem);
}

// ------------------------------------------------------------------------------------
// host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// NHWC activation viewed as 4-D (C, W, H, N); box = 64 channels x a pixel box
bool map_act(CUtensorMap *m, const void *ptr, int N, int H, int W, int C, const PixTile &pt) {
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)pt.Wt, (cuuint32_t)pt.Ht, (cuuint32_t)pt.Nt};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(ptr), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// NHWC activation as 5-D (64, W, H, N, C/64): box = 64 ch x pixel box x nb channel blocks, so
// one TMA instruction lands nb MN-major 64-channel blocks back to back ([block][px][64] in smem)
bool map_act_blocked(CUtensorMap *m, const void *ptr, int N, int H, int W, int C, const PixTile &pt, int nb) {
    cuuint64_t dims[5] = {64, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N, (cuuint64_t)(C / 64)};
    cuuint64_t strides[4] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2, 128};
    cuuint32_t box[5] = {64, (cuuint32_t)pt.Wt, (cuuint32_t)pt.Ht, (cuuint32_t)pt.Nt, (cuuint32_t)nb};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(ptr), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool map_act_nb(CUtensorMap *m, const void *ptr, int N, int H, int W, int C, const PixTile &pt, int nb) {
    return nb == 1 ? map_act(m, ptr, N, H, W, C, pt) : map_act_blocked(m, ptr, N, H, W, C, pt, nb);
}

// NHWC activation with the row-halo box (64 channels x 130 pixels x 3 rows x 1 image)
// output box of one epilogue warp for a generic pixel tile: its 32 rows are bw x bh x bn pixels
bool map_out_tile(CUtensorMap *m, const void *ptr, int N, int H, int W, int C, const PixTile &pt) {
    const int bw = pt.Wt < 32 ? pt.Wt : 32, bh = (32 / bw) < pt.Ht ? 32 / bw : pt.Ht, bn = 32 / (bw * bh);
    if (bw * bh * bn != 32 || bn > pt.Nt) return false;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {32, (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bn};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(ptr), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool map_out32(CUtensorMap *m, const void *ptr, int N, int H, int W, int C) {
    // NHWC bf16 output, box 32 channels x 32 pixels of one row, SWIZZLE_64B (staged TMA stores)
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {32, 32, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(ptr), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool map_halo(CUtensorMap *m, const void *ptr, int N, int H, int W, int C, int rows = 3) {
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {64, 130, (cuuint32_t)rows, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(ptr), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4 sub-pixel planes [4][N][H][W][C] viewed as 5-D (C, W, H, N, 4); box = 64 x pixel box x 1
bool map_planes(CUtensorMap *m, const void *ptr, int N, int H, int W, int C, const PixTile &pt) {
    cuuint64_t dims[5] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N, 4};
    cuuint64_t strides[4] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2,
                             (cuuint64_t)N * H * W * C * 2};
    cuuint32_t box[5] = {64, (cuuint32_t)pt.Wt, (cuuint32_t)pt.Ht, (cuuint32_t)pt.Nt, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(ptr), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// KRSC weights viewed as 3-D (Cin, taps, Cout); box = 64 cin x 1 tap x rows
bool map_wgt(CUtensorMap *m, const void *ptr, int cout, int taps, int cin, int rows) {
    cuuint64_t dims[3] = {(cuuint64_t)cin, (cuuint64_t)taps, (cuuint64_t)cout};
    cuuint64_t strides[2] = {(cuuint64_t)cin * 2, (cuuint64_t)taps * cin * 2};
    cuuint32_t box[3] = {64, 1, (cuuint32_t)rows};
    cuuint32_t es[3] = {1, 1, 1};
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(ptr), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

PixTile pix_tile(int N, int H, int W, int npx) {
    PixTile t;
    t.Wt = W < npx ? W : npx;
    int rest = npx / t.Wt;
    t.Ht = H < rest ? H : rest;
    t.Nt = rest / t.Ht;
    t.tw = W / t.Wt;
    t.th = H / t.Ht;
    t.tn = (N + t.Nt - 1) / t.Nt;
    return t;
}

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    }
    return n;
}

bool pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

Taps make_taps(int ksize) {
    Taps t;
    memset(&t, 0, sizeof t);
    if (ksize == 1) {
        t.n = 1;
    } else {
        t.n = 9;
        for (int i = 0; i < 9; ++i) {
            t.dy[i] = (int8_t)(i / 3 - 1);
            t.dx[i] = (int8_t)(i % 3 - 1);
            t.wt[i] = (int8_t)i;
        }
    }
    return t;
}

// Halving conv (model.py:79-88, 105, 128): y = conv2x2(pad(upsample2x(x), (0,1,0,1))).
// Output pixel (2p + cy, 2q + cx) only sees x[p + {0,1}][q + {0,1}]; per sub-pixel class
// the 2x2 taps collapse onto 1, 2, 2 and 4 distinct inputs with summed weights (9 combined
// weight slabs, see ice_halve_prep in unet_ops.cu).  The zero pad row/column is exactly
// the TMA out-of-bounds fill of x[p+1] / x[q+1] at the last row / column.
//   combined slab: 0:(0,0)c0  1:(0,0)c1 2:(0,1)c1  3:(0,0)c2 4:(1,0)c2  5..8:(0,0),(0,1),(1,0),(1,1)c3
const int8_t HALVE_CLS[9] = {0, 1, 1, 2, 2, 3, 3, 3, 3};
const int8_t HALVE_DY[9] = {0, 0, 0, 0, 1, 0, 0, 1, 1};
const int8_t HALVE_DX[9] = {0, 0, 1, 0, 0, 0, 1, 0, 1};

// A/B switches of the tiling heuristics (test / tuning hooks), read when the library is first
// used and again on ice_conv_reload_knobs(); the defaults are the measured-best choices.
struct Knobs {
    bool no_dual, no_stage, no_splitk, no_wgrad_trans256, no_ref_tma, no_halo_wgrad, no_halve_merge, no_pair;
    int conv_m2, wg_m2;  // -1 = automatic, 0 / 1 forced
};
Knobs read_knobs() {
    auto flag = [](const char *n) { return getenv(n) != nullptr; };
    auto tri = [](const char *n) {
        const char *e = getenv(n);
        return e ? (atoi(e) != 0 ? 1 : 0) : -1;
    };
    Knobs r;
    r.no_dual = flag("ICE_NO_DUAL");
    r.no_stage = flag("ICE_NO_STAGE");
    r.no_splitk = flag("ICE_NO_SPLITK");
    r.no_wgrad_trans256 = flag("ICE_NO_WGRAD_TRANS256");
    r.no_ref_tma = flag("ICE_NO_REF_TMA");
    r.no_halo_wgrad = flag("ICE_NO_HALO_WGRAD");
    r.no_halve_merge = flag("ICE_NO_HALVE_MERGE");
    r.no_pair = flag("ICE_NO_PAIR");
    r.conv_m2 = tri("ICE_CONV_M2");
    r.wg_m2 = tri("ICE_WG_M2");
    return r;
}
Knobs g_knobs = read_knobs();
const Knobs &knobs() { return g_knobs; }

// (settle the scratch arena: answer a size query or reject a too-small buffer before any launch)
#define ICE_SETTLE(ar)                                           \
    do {                                                         \
        const int q_ = (ar).settle(scratch_bytes);               \
        if (q_) return q_ > 0 ? ICE_OK : ICE_ESCRATCH;           \
    } while (0)

int persist_grid(long long total) { return (int)(total < num_sms() ? total : num_sms()); }

// The persistent schedule a launch used (for the bias-gradient finisher's row validity).
ice::RowSched sched(dim3 tiles, int bn, int slots) {
    const long long total = (long long)tiles.x * tiles.y * tiles.z;
    return ice::RowSched{persist_grid(total), slots, (int)tiles.x, (int)total, bn};
}

template <int BN, int BSTAGES, bool RES, class P, bool DUAL = false, bool PAIR = false>
int launch_halo(const P &p, dim3 tiles, cudaStream_t st) {
    constexpr int smem = halo_smem_bytes<BN, BSTAGES, RES, PAIR>(P::STAGE_REF);
    static_assert(smem <= 232448, "halo kernel smem");
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(halo_gemm<BN, BSTAGES, RES, P, DUAL, PAIR>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return (int)e;
        attr = true;
    }
    const TileGrid g = tile_grid(tiles);
    const long long total = (long long)tiles.x * tiles.y * tiles.z;
    halo_gemm<BN, BSTAGES, RES, P, DUAL, PAIR><<<persist_grid(total), NTHREADS + (DUAL ? 32 : 0), smem, st>>>(p, g);
    ice::count_launch();
    return (int)cudaGetLastError();
}

// halo-path tile width: N = 64 tiles are shared-memory-bandwidth bound (4 KB of A + 2 KB
// of B per 32-cycle MMA), so use 128-wide tiles whenever there are 128 columns; a single
// 64-column problem keeps its 9 weight taps resident instead.
int halo_bn(int nch, int ncols) { return ncols % 128 == 0 ? 128 : 64; }

struct HaloPlan {
    int kind;  // 0: BN 64, resident weights (dual issuers when ncols == 64); 1: BN 128; 2: BN 64 streamed
    int bn;
    bool pair;  // streamed-weight kinds on row pairs (pair tiles: 2 x 128 pixels, one 4-row halo slab)
    dim3 tiles;
    int halo_rows() const { return pair ? 4 : 3; }
};
// Row pairs are taken where they measured faster (tools/pair_ab.sh): every streamed-weight
// fprop (+5% at 64 columns, +13-15% at 128) and the 128-wide dgrads with K >= 128 (+7-9%);
// the K = 64 dgrads are bound by their epilogue and lose ~1% with the coarser accumulators.
HaloPlan halo_plan(int nch, int ncols, unsigned mtiles, int h, bool dgrad) {
    HaloPlan hp;
    hp.bn = halo_bn(nch, ncols);
    hp.kind = (hp.bn == 64 && nch == 1) ? 0 : (hp.bn == 128 ? 1 : 2);
    hp.pair = (dgrad ? hp.kind == 1 && nch >= 2 : hp.kind != 0) && h % 2 == 0 && !knobs().no_pair;
    hp.tiles = dim3(hp.pair ? mtiles / 2 : mtiles, ncols / hp.bn, 1);
    return hp;
}

template <class P>
int run_halo(const P &p, const HaloPlan &h, int ncols, cudaStream_t st) {
    if (h.kind == 0) {
        if (ncols == 64 && !knobs().no_dual) return launch_halo<64, 1, true, P, true>(p, h.tiles, st);
        return launch_halo<64, 1, true>(p, h.tiles, st);
    }
    if (h.kind == 1 && h.pair) return launch_halo<128, 4, false, P, false, true>(p, h.tiles, st);
    if (h.kind == 1) return launch_halo<128, 2, false>(p, h.tiles, st);
    if (h.pair) return launch_halo<64, 6, false, P, false, true>(p, h.tiles, st);
    return launch_halo<64, 5, false>(p, h.tiles, st);
}

bool use_halo(int ksize, int w) { return ksize == 3 && w >= 128 && w % 128 == 0; }

template <int BN, int STAGES, class P>
int launch(const P &p, dim3 tiles, cudaStream_t st) {
    constexpr int smem = smem_bytes<BN, STAGES>();
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(conv_gemm<BN, STAGES, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return (int)e;
        attr = true;
    }
    const TileGrid g = tile_grid(tiles);
    conv_gemm<BN, STAGES, P><<<persist_grid((long long)tiles.x * tiles.y * tiles.z), NTHREADS, smem, st>>>(p, g);
    ice::count_launch();
    return (int)cudaGetLastError();
}

template <int BN, int STAGES, class P>
int launch_m2(const P &p, dim3 tiles, cudaStream_t st) {
    constexpr int smem = m2_smem_bytes<BN, STAGES, P>();
    static_assert(smem <= 232448, "conv_gemm_m2 smem");
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(conv_gemm_m2<BN, STAGES, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return (int)e;
        attr = true;
    }
    const TileGrid g = tile_grid(tiles);
    conv_gemm_m2<BN, STAGES, P><<<persist_grid((long long)tiles.x * tiles.y * tiles.z), NTHREADS, smem, st>>>(p, g);
    ice::count_launch();
    return (int)cudaGetLastError();
}

// one-column-tile-width dispatch of the 128-row kernel
template <class P>
int launch_bn(const P &p, int bn, dim3 tiles, cudaStream_t st) {
    if (bn == 256) return launch<256, 4>(p, tiles, st);
    if (bn == 128) return launch<128, 6>(p, tiles, st);
    return launch<64, 8>(p, tiles, st);
}
template <class P>
int launch_bn_m2(const P &p, int bn, dim3 tiles, cudaStream_t st) {
    return bn == 256 ? launch_m2<256, 3>(p, tiles, st) : launch_m2<128, 4>(p, tiles, st);
}

int pick_bn(int ntot, long long m_tiles) {
    // largest tile that still gives >= one wave of CTAs; 64 as the floor
    const int cands[3] = {256, 128, 64};
    for (int i = 0; i < 3; ++i) {
        int bn = cands[i];
        if (ntot % bn) continue;
        if (m_tiles * (ntot / bn) >= 148 || bn == 64) return bn;
    }
    return 64;
}

bool shape_ok(int N, int H, int W) { return N > 0 && pow2(H) && pow2(W); }

// fprop / dgrad tiling for the non-halo path.  N = 256 tiles run at ~95% of the MMA peak,
// N = 128 tiles at ~60% (their A + B operand stream per FLOP is 1.5x larger and becomes
// L2-bound), so 256-wide tiles are kept even when they give fewer tiles than SMs; below
// 80% of a wave the K range is split (fp32 partial slices + split_finish_*).
void pick_tiling(int ntot, long long m_tiles, int &bn, int &splits, int total_kb) {
    splits = 1;
    if (ntot % 256) {
        bn = pick_bn(ntot, m_tiles);
        return;
    }
    bn = 256;
    const long long tiles = m_tiles * (ntot / 256);
    const long long sms = num_sms();
    if (tiles * 5 >= sms * 4) return;
    for (int sp = 2; sp <= 4; ++sp) {
        if (total_kb / sp < 8) break;
        splits = sp;
        const long long units = tiles * sp;
        const double eff = (double)units / (double)(((units + sms - 1) / sms) * sms);
        if (eff >= 0.85) break;
    }
}

// K-blocks per split and the number of non-empty splits it gives
void split_shape(int total_kb, int splits, int &kps, int &z) {
    kps = (total_kb + splits - 1) / splits;
    z = (total_kb + kps - 1) / kps;
}

template <class P>
int launch_split(const P &p, long long mtiles, int ncols, int total_kb, int kps, int z, float *ws, cudaStream_t st) {
    SplitK<P> q;
    q.p = p;
    q.ws = ws;
    q.ld = ncols;
    q.kps = kps;
    q.total_kb = total_kb;
    q.zstride = (size_t)p.N * p.H * p.W * ncols;
    return launch<256, 4>(q, dim3((unsigned)mtiles, ncols / 256, (unsigned)z), st);
}

// Weight-gradient tiling.  cout >= 128: D = [cout][(tap, cin)] (M = cout); narrower layers
// transpose the GEMM (M = (tap, cin), N = cout) so no TMEM lane holds a padding row.
void wgrad_tiles(int ncols, int cout, int &trans, int &mtiles, int &ntiles, int &bn) {
    trans = cout < BM;
    // 256-wide tiles only exist along the dimension divisible by 256: for (tap, cin) widths like
    // 9 x 128 = 1152 with cout % 256 == 0, the transposed GEMM gets N = cout in 256-wide tiles
    if (!trans && ncols % 256 && cout % 256 == 0 && !knobs().no_wgrad_trans256) {
        trans = 1;
        mtiles = (ncols + BM - 1) / BM;
        bn = 256;
        ntiles = cout / bn;
        return;
    }
    if (!trans) {
        mtiles = (cout + BM - 1) / BM;
        bn = ncols % 256 == 0 ? 256 : (ncols % 128 == 0 ? 128 : 64);
        ntiles = ncols / bn;
    } else {
        mtiles = (ncols + BM - 1) / BM;
        bn = 64;  // cout is a multiple of 64 below 128
        ntiles = cout / bn;
    }
}

// 256-row fprop / dgrad tiles (conv_gemm_m2) for unsplit 256-wide tilings (ICE_CONV_M2=0/1
// overrides).  Measured per shape in the train step: they gain 8-20% on long K (>= 72
// K-blocks) when halving the tile count does not worsen the last wave, and lose up to 40%
// otherwise (short K exposes the drain; 64x64 levels drop from 99% to 87% wave fill).
bool conv_m2(long long mtiles, int ncols, int bn, int splits, int total_kb) {
    if ((bn != 256 && bn != 128) || splits != 1 || mtiles % 2) return false;
    if (knobs().conv_m2 >= 0) return knobs().conv_m2 != 0;
    const long long sms = num_sms(), t1 = mtiles * (ncols / bn), t2 = t1 / 2;
    if (t2 * 5 < sms * 4) return false;
    if (bn == 128) return true;  // double-buffered accumulators: no exposed drain
    if (total_kb < 72) return false;
    const double e1 = (double)t1 / (double)(((t1 + sms - 1) / sms) * sms);
    const double e2 = (double)t2 / (double)(((t2 + sms - 1) / sms) * sms);
    return e2 >= e1 - 0.01;
}

// 256-row weight-gradient tiles (conv_gemm_m2) when the M extent pairs up
bool wgrad_m2(int mtiles, int bn, int total_kb) {
    if (bn != 256 || mtiles % 2) return false;
    (void)total_kb;  // measured faster at every wgrad shape of the model, 32 K-blocks included
    return knobs().wg_m2 != 0;
}

// K-blocks per split.  The persistent grid runs ceil(units / SMs) rounds of equal-size
// units (units = tiles * splits), so pick the split count whose last round is fullest
// (>= 4 K-blocks per split, at most max_units units); fewer splits win ties.  Every split
// beyond the first writes a partial slice of the weight gradient (fixed-order reduction,
// reduce.cuh), so the GEMM path caps the units at one round: its layers' weights are MBs and
// 80-split slices cost GBs of traffic; the halo path's weights are 0.15-0.6 MB.
int split_k(int total_kb, long long tiles, long long max_units = 8LL * 148) {
    const long long sms = num_sms();
    int best = 1;
    double best_eff = -1.0;
    for (int s = 1; s <= total_kb; ++s) {
        const int kps = (total_kb + s - 1) / s;
        if ((total_kb + kps - 1) / kps != s) continue;  // not an exact split count
        if (kps < 4 && s > 1) break;
        const long long units = tiles * s;
        const long long rounds = (units + sms - 1) / sms;
        double eff = (double)units / (double)(rounds * sms);
        eff *= (double)total_kb / ((double)kps * s);  // short last split
        if (units > max_units && s > 1) break;
        if (eff > best_eff + 1e-3) {
            best_eff = eff;
            best = s;
        }
        if (units > 8 * sms) break;
    }
    return (total_kb + best - 1) / best;
}

bool map_halo_box(CUtensorMap *m, const void *ptr, int N, int H, int W, int C, int c0, int cols, int rows) {
    // halo box (64 ch, cols px, rows rows, 1 image) starting at channel c0 of a C-channel NHWC tensor
    const char *base = reinterpret_cast<const char *>(ptr) + (size_t)c0 * 2;
    cuuint64_t dims[4] = {64, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)cols, (cuuint32_t)rows, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<char *>(base), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int COUT, int NCH, int STAGES, bool HALVE>
int launch_hwgrad(const HWgrad &p, int grid, cudaStream_t st) {
    constexpr int smem = hw_smem_bytes<COUT, NCH, STAGES, HALVE>();
    static_assert(smem <= 232448, "hwgrad smem");
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(hwgrad_kernel<COUT, NCH, STAGES, HALVE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return (int)e;
        attr = true;
    }
    hwgrad_kernel<COUT, NCH, STAGES, HALVE><<<grid, NTHREADS, smem, st>>>(p);
    ice::count_launch();
    return (int)cudaGetLastError();
}

// halo weight-gradient path: 3x3 (or the 2x2 halving conv with HALVE), W % 64 == 0,
// cout in {64, 128}, cin / 64 in {1, 2}.  Returns 1 when not applicable (nothing taken from
// the arena, nothing launched).
int try_hwgrad(const uint16_t *x1, int c1, const uint16_t *x2, int c2, const uint16_t *dy, int cout, int n, int h,
               int w, float *dw, ice::Arena &ar, uint64_t *scratch_bytes, cudaStream_t st, bool halve = false) {
    const int nch = (c1 + c2) / 64;
    if (w % 64 || w < 64 || (cout != 64 && cout != 128) || (nch != 1 && nch != 2)) return 1;
    if (halve && cout != 64) return 1;
    HWgrad p;
    memset(&p, 0, sizeof p);
    p.N = n; p.H = h; p.W = w; p.ct = c1 + c2; p.cout = cout; p.nchx = nch; p.dw = dw;
    p.ow = ice::grad_overwrite() ? 1 : 0;
    const int kr = halve ? 1 : 2;  // output rows per K-block (HWGeom::KR)
    if (h % kr) return 1;
    p.total_kb = n * (h / kr) * (w / 64);
    for (int c = 0; c < nch; ++c) {
        const int cc = c * 64;
        const int cols = halve ? 65 : 66, rows = halve ? 2 : 4;
        const bool ok = cc < c1 ? map_halo_box(&p.xm[c], x1, n, h, w, c1, cc, cols, rows)
                                : map_halo_box(&p.xm[c], x2, n, h, w, c2, cc - c1, cols, rows);
        if (!ok) return ICE_EINVAL;
    }
    PixTile seg{64, kr, 1, w / 64, h / kr, (halve ? 4 : 1) * n};
    if (!map_act_nb(&p.dym, dy, (halve ? 4 : 1) * n, h, w, cout, seg, cout / 64)) return ICE_EINVAL;
    // work split: M tile groups (G x cout <= 512 TMEM columns) x pixel splits
    p.total_mt = ((halve ? 4 : 9) * nch + 1) / 2;
    const int gmax = 512 / cout;
    p.groups = (p.total_mt + gmax - 1) / gmax;
    p.G = (p.total_mt + p.groups - 1) / p.groups;
    p.kb_per_split = split_k(p.total_kb, p.groups);
    const int splits = (p.total_kb + p.kb_per_split - 1) / p.kb_per_split;
    const long long units = (long long)p.groups * splits;
    p.wsize = (size_t)cout * (halve ? 4 : 9) * p.ct;
    if (splits > 1) p.ws = ar.take<float>((size_t)(splits - 1) * p.wsize * 4);
    ICE_SETTLE(ar);
    const int grid = persist_grid(units);
    int rc;
    if (halve) rc = nch == 1 ? launch_hwgrad<64, 1, 3, true>(p, grid, st) : launch_hwgrad<64, 2, 3, true>(p, grid, st);
    else if (cout == 64 && nch == 1) rc = launch_hwgrad<64, 1, 4, false>(p, grid, st);
    else if (cout == 64) rc = launch_hwgrad<64, 2, 2, false>(p, grid, st);
    else if (nch == 1) rc = launch_hwgrad<128, 1, 3, false>(p, grid, st);
    else rc = launch_hwgrad<128, 2, 2, false>(p, grid, st);
    if (rc || splits == 1) return rc;
    return ice::splitsum_finish(p.ws, splits - 1, p.wsize, p.wsize, dw, st);
}

// The non-halo weight gradient (WgradProb on conv_gemm / conv_gemm_m2), split over pixels
// when the tile grid is below a wave: partial slices in scratch + splitsum_finish.
int run_wgrad(WgradProb &p, int ncols, int mtiles, int ntiles, int bn, bool m2, ice::Arena &ar,
              uint64_t *scratch_bytes, cudaStream_t st) {
    const int splits = (p.total_kb + p.kb_per_split - 1) / p.kb_per_split;
    p.wsize = (size_t)p.cout * ncols;
    p.ws = splits > 1 ? ar.take<float>((size_t)(splits - 1) * p.wsize * 4) : nullptr;
    ICE_SETTLE(ar);
    dim3 grid((unsigned)mtiles, (unsigned)ntiles, (unsigned)splits);
    const int rc = m2 ? launch_m2<256, 3>(p, grid, st) : launch_bn(p, bn, grid, st);
    if (rc || splits == 1) return rc;
    return ice::splitsum_finish(p.ws, splits - 1, p.wsize, p.wsize, p.dw, st);
}

// channel blocks per TMA box: as many consecutive 64-blocks as the tile reads from one
// (tap, source) run; the M operand supplies 2 blocks (4 for 256-row tiles), B BN/64
void wgrad_boxes(WgradProb &p, bool m2, int bn) {
    const int mb = m2 ? 4 : 2;
    const int want_x = p.trans ? mb : bn / 64, want_y = p.trans ? bn / 64 : mb;
    int nbx = want_x;
    while (nbx > 1 && ((p.c1 % (64 * nbx)) || (p.c2 % (64 * nbx)))) nbx >>= 1;
    int nby = want_y;
    while (nby > 1 && (p.cout % (64 * nby))) nby >>= 1;
    p.nbx = nbx;
    p.nby = nby;
}

// dgrad bias gradients: one row of per-CTA column sums per CTA, taken from the arena
// (s.slots = the shared-memory slots the CTA adds first: 4 lane quarters, x2 M halves in m2)
void take_bias_rows(DgradProb &p, const ice::RowSched &s, ice::Arena &ar) {
    if (!p.db1 && !p.db2) return;
    p.bslots = s.slots;
    p.bpart = ar.take<float>((size_t)s.G * (p.c1 + p.c2) * 4);
}
int finish_bias(const DgradProb &p, const ice::RowSched &s, cudaStream_t st) {
    if (!p.db1 && !p.db2) return 0;
    const int ow = ice::grad_overwrite() ? 1 : 0;
    const ice::ColSegs segs{{p.db1, p.db2, nullptr, nullptr}, {p.c1, p.c2, 0, 0}, {ow, ow, 0, 0}};
    return ice::colsum_finish(p.bpart, s.G, p.c1 + p.c2, p.c1 + p.c2, segs, s, st);
}
}  // namespace

extern "C" int ice_conv_reload_knobs(void) {
    g_knobs = read_knobs();
    return ICE_OK;
}

// merged halving-conv weights wm[(cls * cout + co)][t][ci] (t = 2 dy + dx) from the 9 combined
// slabs wc[co][slab][ci] (ice_halve_prep); taps a class does not use are zero
__global__ void halve_merge_kernel(const uint16_t *__restrict__ wc, int cout, int c, uint16_t *__restrict__ wm,
                                   unsigned long long tab) {
    const long long total = 16LL * cout * c;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int ci = (int)(i % c);
        const long long r = i / c;
        const int t = (int)(r % 4), row = (int)(r / 4), cls = row / cout, co = row % cout;
        const int slab = (int)((tab >> (4 * (cls * 4 + t))) & 15);
        wm[i] = slab == 15 ? (uint16_t)0 : wc[((size_t)co * 9 + slab) * c + ci];
    }
}

// builds the merged weights into buf (scratch, 16 * cout * c bf16)
int halve_merged_weights(const uint16_t *wc, int cout, int c, uint16_t *buf, cudaStream_t st) {
    // class -> tap -> slab (15 = unused), from HALVE_CLS / HALVE_DY / HALVE_DX
    unsigned long long tab = ~0ull;
    for (int i = 0; i < 9; ++i) {
        const int cls = HALVE_CLS[i], t = 2 * HALVE_DY[i] + HALVE_DX[i];
        tab &= ~(15ull << (4 * (cls * 4 + t)));
        tab |= (unsigned long long)i << (4 * (cls * 4 + t));
    }
    const long long total = 16LL * cout * c;
    const unsigned grid = (unsigned)((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
    halve_merge_kernel<<<grid, 256, 0, st>>>(wc, cout, c, buf, tab);
    ice::count_launch();
    return (int)cudaGetLastError();
}

extern "C" int ice_conv_fprop(const uint16_t *x1, int32_t c1, const uint16_t *x2, int32_t c2, int32_t n, int32_t h,
                              int32_t w, int32_t ksize, const uint16_t *wgt, const float *bias, int32_t cout,
                              int32_t relu, const float *drop_scale, uint16_t *y, uint32_t *relu_bits, void *scratch,
                              uint64_t *scratch_bytes, void *stream) {
    if (!encode_fn()) return ICE_ENODRIVER;
    if (!x1 || !wgt || !y || c1 <= 0 || c1 % 64 || c2 < 0 || c2 % 64 || (c2 && !x2) || cout <= 0 || cout % 64 ||
        (ksize != 1 && ksize != 3) || !shape_ok(n, h, w))
        return ICE_EINVAL;
    ice::Arena ar(scratch, scratch_bytes);
    FpropProb p;
    memset(&p, 0, sizeof p);
    p.pt = pix_tile(n, h, w, BM);
    p.taps[0] = make_taps(ksize);
    p.omul = 1;
    p.N = n; p.H = h; p.W = w; p.c1 = c1; p.c2 = c2; p.cout = cout;
    p.bias = bias; p.drop = drop_scale; p.relu = relu; p.y = reinterpret_cast<bf16 *>(y);
    p.rbits = relu_bits;
    cudaStream_t st = (cudaStream_t)stream;
    const long long mtiles = (long long)p.pt.tw * p.pt.th * p.pt.tn;
    if (use_halo(ksize, w)) {
        const int nch = (c1 + c2) / 64;
        const HaloPlan hp = halo_plan(nch, cout, (unsigned)mtiles, h, false);
        if (!map_halo(&p.xa, x1, n, h, w, c1, hp.halo_rows())) return ICE_EINVAL;
        if (c2 && !map_halo(&p.xb, x2, n, h, w, c2, hp.halo_rows())) return ICE_EINVAL;
        if (!map_wgt(&p.wm, wgt, cout, 9, c1 + c2, hp.bn)) return ICE_EINVAL;
        if (((nch == 1 && cout == 64) || hp.bn == 128 || hp.pair) && !knobs().no_stage) {  // staged TMA stores
            if (!map_out32(&p.ym, y, n, h, w, cout)) return ICE_EINVAL;
            p.y_tma = 1;
        }
        ICE_SETTLE(ar);
        return run_halo(p, hp, cout, st);
    }
    int bn, splits;
    const int total_kb = p.taps[0].n * ((c1 + c2) / BK);
    pick_tiling(cout, mtiles, bn, splits, total_kb);
    if (knobs().no_splitk || relu_bits) splits = 1;  // the split finisher writes no mask bits
    if (!knobs().no_stage && map_out_tile(&p.ym, y, n, h, w, cout, p.pt)) p.y_tma = 1;  // staged stores
    if (!map_act(&p.xa, x1, n, h, w, c1, p.pt)) return ICE_EINVAL;
    if (c2 && !map_act(&p.xb, x2, n, h, w, c2, p.pt)) return ICE_EINVAL;
    if (!map_wgt(&p.wm, wgt, cout, p.taps[0].n, c1 + c2, bn)) return ICE_EINVAL;
    if (splits > 1) {
        const long long npx = (long long)n * h * w;
        int kps, z;
        split_shape(total_kb, splits, kps, z);
        float *ws = ar.take<float>((size_t)z * npx * cout * 4);
        ICE_SETTLE(ar);
        int rc = launch_split(p, mtiles, cout, total_kb, kps, z, ws, st);
        if (rc) return rc;
        const long long work = npx * (cout / 8), nblk = (work + 255) / 256;
        const unsigned fgrid = (unsigned)(nblk < 148 * 16 ? nblk : 148 * 16);
        split_finish_fprop<<<fgrid, 256, 0, st>>>(ws, z, npx, h * w, cout, bias, drop_scale, relu, p.y);
        ice::count_launch();
        return (int)cudaGetLastError();
    }
    ICE_SETTLE(ar);
    if (conv_m2(mtiles, cout, bn, splits, total_kb))
        return launch_bn_m2(p, bn, dim3((unsigned)(mtiles / 2), cout / bn, 1), st);
    return launch_bn(p, bn, dim3((unsigned)mtiles, cout / bn, 1), st);
}

extern "C" int ice_conv_dgrad(const uint16_t *dy, int32_t cout, int32_t n, int32_t h, int32_t w, int32_t ksize,
                              const uint16_t *wgt, int32_t c1, int32_t c2, uint16_t *dx1, const uint16_t *relu_ref1,
                              const float *drop_scale1, const uint16_t *add1, uint16_t *dx2,
                              const uint16_t *relu_ref2, const float *drop_scale2, const uint16_t *add2,
                              int32_t dx2_planes, float *dbias1, float *dbias2, const uint32_t *relu_bits1,
                              void *scratch, uint64_t *scratch_bytes, void *stream) {
    if (!encode_fn()) return ICE_ENODRIVER;
    if (!dy || !wgt || c1 <= 0 || c1 % 64 || c2 < 0 || c2 % 64 || cout <= 0 || cout % 64 ||
        (ksize != 1 && ksize != 3) || !shape_ok(n, h, w))
        return ICE_EINVAL;
    ice::Arena ar(scratch, scratch_bytes);
    DgradProb p;
    memset(&p, 0, sizeof p);
    p.pt = pix_tile(n, h, w, BM);
    p.taps = make_taps(ksize);
    p.N = n; p.H = h; p.W = w; p.c1 = c1; p.c2 = c2; p.cout = cout;
    p.out1 = reinterpret_cast<bf16 *>(dx1); p.out2 = reinterpret_cast<bf16 *>(dx2);
    p.ref1 = reinterpret_cast<const bf16 *>(relu_ref1); p.ref2 = reinterpret_cast<const bf16 *>(relu_ref2);
    p.add1 = reinterpret_cast<const bf16 *>(add1); p.add2 = reinterpret_cast<const bf16 *>(add2);
    p.drop1 = drop_scale1; p.drop2 = drop_scale2;
    p.db1 = dx1 ? dbias1 : nullptr; p.db2 = dx2 ? dbias2 : nullptr;
    p.rbits1 = relu_bits1;
    p.planes_out2 = dx2_planes;
    if (dx2_planes && ((h | w) & 1)) return ICE_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const int ct = c1 + c2;
    const long long mtiles = (long long)p.pt.tw * p.pt.th * p.pt.tn;
    if (use_halo(ksize, w)) {  // the epilogue picks dx1/dx2 (and the plane layout) per 32-column chunk
        const HaloPlan hp = halo_plan(cout / 64, ct, (unsigned)mtiles, h, true);
        if (!map_halo(&p.dym, dy, n, h, w, cout, hp.halo_rows())) return ICE_EINVAL;
        if (!map_wgt(&p.wm, wgt, cout, 9, ct, 64)) return ICE_EINVAL;
        const bool res64 = cout == 64 && ct == 64 && c2 == 0;  // resident-weight BN = 64 tiles
        if ((res64 || hp.bn == 128) && dx1 && !knobs().no_stage) {  // staged TMA stores
            if (!map_out32(&p.o1m, dx1, n, h, w, c1)) return ICE_EINVAL;
            p.o1_tma = 1;
        }
        if (hp.bn == 128 && dx2 && dx2_planes && !knobs().no_stage) {  // staged plane stores
            cuuint64_t dims[5] = {(cuuint64_t)c2, (cuuint64_t)(w / 2), (cuuint64_t)(h / 2), (cuuint64_t)n, 4};
            cuuint64_t strides[4] = {(cuuint64_t)c2 * 2, (cuuint64_t)(w / 2) * c2 * 2, (cuuint64_t)(h / 2) * (w / 2) * c2 * 2,
                                     (cuuint64_t)n * (h / 2) * (w / 2) * c2 * 2};
            cuuint32_t box[5] = {32, 16, 1, 1, 1};
            cuuint32_t es[5] = {1, 1, 1, 1, 1};
            if (encode_fn()(&p.o2m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, dx2, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return ICE_EINVAL;
            p.o2_tma = 1;
        }
        if (res64 && dx1 && !knobs().no_stage && relu_ref1 && !relu_bits1 && !knobs().no_ref_tma) {
            // ReLU reference staged by the producer
            cuuint64_t dims[4] = {(cuuint64_t)c1, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
            cuuint64_t strides[3] = {(cuuint64_t)c1 * 2, (cuuint64_t)w * c1 * 2, (cuuint64_t)h * w * c1 * 2};
            cuuint32_t box[4] = {64, 128, 1, 1};
            cuuint32_t es[4] = {1, 1, 1, 1};
            if (encode_fn()(&p.refm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t *>(relu_ref1), dims,
                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return ICE_EINVAL;
            p.ref_tma = 1;
        }
        const ice::RowSched s = sched(hp.tiles, hp.bn, 4);
        take_bias_rows(p, s, ar);
        ICE_SETTLE(ar);
        const int rc = run_halo(p, hp, ct, st);
        return rc ? rc : finish_bias(p, s, st);
    }
    int bn, splits;
    const int total_kb = p.taps.n * (cout / BK);
    pick_tiling(ct, mtiles, bn, splits, total_kb);
    if (knobs().no_splitk) splits = 1;
    // a column tile must not straddle the dx1 / dx2 split
    while (bn > 64 && (c1 % bn)) {
        bn >>= 1;
        splits = 1;
    }
    if (!map_act(&p.dym, dy, n, h, w, cout, p.pt)) return ICE_EINVAL;
    if (!map_wgt(&p.wm, wgt, cout, p.taps.n, ct, 64)) return ICE_EINVAL;
    // staged dx1 stores: the warp's rows must all be valid (no partial image tile)
    if (dx1 && n % p.pt.Nt == 0 && !knobs().no_stage && map_out_tile(&p.o1m, dx1, n, h, w, c1, p.pt))
        p.o1_tma = 1;
    if (splits > 1) {
        const long long npx = (long long)n * h * w;
        int kps, z;
        split_shape(total_kb, splits, kps, z);
        float *ws = ar.take<float>((size_t)z * npx * ct * 4);
        const int strips = (int)((npx + FIN_STRIP - 1) / FIN_STRIP);
        if (p.db1 || p.db2) p.bpart = ar.take<float>((size_t)strips * ct * 4);
        ICE_SETTLE(ar);
        int rc = launch_split(p, mtiles, ct, total_kb, kps, z, ws, st);
        if (rc) return rc;
        split_finish_dgrad<<<(ct / 256) * strips, 256, 0, st>>>(ws, z, (int)npx, n, h, w, p);
        ice::count_launch();
        rc = (int)cudaGetLastError();
        if (rc || (!p.db1 && !p.db2)) return rc;
        const int ow = ice::grad_overwrite() ? 1 : 0;
        const ice::ColSegs segs{{p.db1, p.db2, nullptr, nullptr}, {c1, c2, 0, 0}, {ow, ow, 0, 0}};
        return ice::colsum_finish(p.bpart, strips, ct, ct, segs, ice::RowSched{1, 1, 1, 1, 0}, st);
    }
    const bool m2 = conv_m2(mtiles, ct, bn, splits, total_kb);
    const dim3 tiles = m2 ? dim3((unsigned)(mtiles / 2), ct / bn, 1) : dim3((unsigned)mtiles, ct / bn, 1);
    const ice::RowSched s = sched(tiles, bn, m2 ? 8 : 4);
    take_bias_rows(p, s, ar);
    ICE_SETTLE(ar);
    const int rc = m2 ? launch_bn_m2(p, bn, tiles, st) : launch_bn(p, bn, tiles, st);
    return rc ? rc : finish_bias(p, s, st);
}

extern "C" int ice_conv_wgrad(const uint16_t *x1, int32_t c1, const uint16_t *x2, int32_t c2, const uint16_t *dy,
                              int32_t cout, int32_t n, int32_t h, int32_t w, int32_t ksize, float *dw, void *scratch,
                              uint64_t *scratch_bytes, void *stream) {
    if (!encode_fn()) return ICE_ENODRIVER;
    if (!x1 || !dy || !dw || c1 <= 0 || c1 % 64 || c2 < 0 || c2 % 64 || (c2 && !x2) || cout <= 0 || cout % 64 ||
        (ksize != 1 && ksize != 3) || !shape_ok(n, h, w))
        return ICE_EINVAL;
    ice::Arena ar(scratch, scratch_bytes);
    cudaStream_t st = (cudaStream_t)stream;
    if (ksize == 3 && !knobs().no_halo_wgrad) {
        const int rc = try_hwgrad(x1, c1, x2, c2, dy, cout, n, h, w, dw, ar, scratch_bytes, st);
        if (rc <= 0) return rc;  // 1 = not applicable
    }
    WgradProb p;
    memset(&p, 0, sizeof p);
    p.pk = pix_tile(n, h, w, BK);
    p.taps = make_taps(ksize);
    p.N = n; p.H = h; p.W = w; p.c1 = c1; p.c2 = c2; p.cout = cout;
    p.dw = dw;
    p.ow = ice::grad_overwrite() ? 1 : 0;
    const int ncols = p.taps.n * (c1 + c2);
    int mtiles, ntiles, bn;
    wgrad_tiles(ncols, cout, p.trans, mtiles, ntiles, bn);
    p.total_kb = p.pk.tw * p.pk.th * p.pk.tn;
    const bool m2 = wgrad_m2(mtiles, bn, p.total_kb);
    if (m2) mtiles /= 2;
    p.kb_per_split = split_k(p.total_kb, (long long)mtiles * ntiles, num_sms());
    wgrad_boxes(p, m2, bn);
    if (!map_act_nb(&p.dym, dy, n, h, w, cout, p.pk, p.nby)) return ICE_EINVAL;
    if (!map_act_nb(&p.xa, x1, n, h, w, c1, p.pk, p.nbx)) return ICE_EINVAL;
    if (c2 && !map_act_nb(&p.xb, x2, n, h, w, c2, p.pk, p.nbx)) return ICE_EINVAL;
    return run_wgrad(p, ncols, mtiles, ntiles, bn, m2, ar, scratch_bytes, st);
}

extern "C" int ice_halve_fprop(const uint16_t *x, int32_t c, int32_t n, int32_t h, int32_t w, const uint16_t *wc,
                               const float *bias, int32_t cout, uint16_t *y, void *scratch, uint64_t *scratch_bytes,
                               void *stream) {
    if (!encode_fn()) return ICE_ENODRIVER;
    if (!x || !wc || !y || c <= 0 || c % 64 || cout <= 0 || cout % 64 || !shape_ok(n, h, w)) return ICE_EINVAL;
    ice::Arena ar(scratch, scratch_bytes);
    FpropProb p;
    memset(&p, 0, sizeof p);
    p.pt = pix_tile(n, h, w, BM);
    for (int i = 0; i < 9; ++i) {
        Taps &t = p.taps[HALVE_CLS[i]];
        t.dy[t.n] = HALVE_DY[i];
        t.dx[t.n] = HALVE_DX[i];
        t.wt[t.n] = (int8_t)i;
        t.n++;
    }
    p.omul = 2;
    p.N = n; p.H = h; p.W = w; p.c1 = c; p.c2 = 0; p.cout = cout;
    p.bias = bias; p.relu = 0; p.y = reinterpret_cast<bf16 *>(y);
    const long long mtiles = (long long)p.pt.tw * p.pt.th * p.pt.tn;
    cudaStream_t st = (cudaStream_t)stream;
    // staged stores: a warp's 32 input pixels of one row land on every other output pixel of
    // row 2h + cy -- a 64-pixel box traversed with element stride 2
    auto map_y = [&]() {
        const int OH = 2 * h, OW = 2 * w;
        cuuint64_t dims[4] = {(cuuint64_t)cout, (cuuint64_t)OW, (cuuint64_t)OH, (cuuint64_t)n};
        cuuint64_t strides[3] = {(cuuint64_t)cout * 2, (cuuint64_t)OW * cout * 2, (cuuint64_t)OH * OW * cout * 2};
        cuuint32_t box[4] = {32, 64, 1, 1};
        cuuint32_t es[4] = {1, 2, 1, 1};
        if (!knobs().no_stage &&
            encode_fn()(&p.ym, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, y, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
            p.y_tma = 1;
    };
    // wide levels: the 4 sub-pixel classes side by side in N (4 x cout columns, 4 taps each, the
    // class's unused taps zero): 16/9 of the MACs, but one 256-wide tile per 128 pixels instead of
    // four short-K 64-wide ones (halve.4: 2 + 4 + 4 + 8 K-blocks on 64 columns)
    if ((4 * cout) % 256 == 0 && cout <= 128 && w >= 64 && p.pt.Wt >= 32 && !knobs().no_halve_merge) {
        uint16_t *wm = ar.take<uint16_t>(16ull * cout * c * 2);
        p.merged = 1;
        p.taps[0].n = 4;
        for (int t = 0; t < 4; ++t) {
            p.taps[0].dy[t] = (int8_t)(t >> 1);
            p.taps[0].dx[t] = (int8_t)(t & 1);
            p.taps[0].wt[t] = (int8_t)t;
        }
        map_y();
        if (!map_act(&p.xa, x, n, h, w, c, p.pt)) return ICE_EINVAL;
        ICE_SETTLE(ar);
        if (!map_wgt(&p.wm, wm, 4 * cout, 4, c, 256)) return ICE_EINVAL;
        const int rc = halve_merged_weights(wc, cout, c, wm, st);
        if (rc) return rc;
        return launch<256, 4>(p, dim3((unsigned)mtiles, 4 * cout / 256, 1), st);
    }
    const int bn = pick_bn(cout, mtiles * 4);
    if (p.pt.Wt >= 32) map_y();
    if (!map_act(&p.xa, x, n, h, w, c, p.pt)) return ICE_EINVAL;
    if (!map_wgt(&p.wm, wc, cout, 9, c, bn)) return ICE_EINVAL;
    ICE_SETTLE(ar);
    return launch_bn(p, bn, dim3((unsigned)mtiles, cout / bn, 4), st);
}

extern "C" int ice_halve_dgrad(const uint16_t *dy_planes, int32_t cout, int32_t n, int32_t h, int32_t w,
                               const uint16_t *wc, int32_t c, uint16_t *dx, const uint16_t *relu_ref,
                               const uint32_t *relu_bits, const float *drop_scale, float *dbias, void *scratch,
                               uint64_t *scratch_bytes, void *stream) {
    if (!encode_fn()) return ICE_ENODRIVER;
    if (!dy_planes || !wc || !dx || c <= 0 || c % 64 || cout <= 0 || cout % 64 || !shape_ok(n, h, w))
        return ICE_EINVAL;
    ice::Arena ar(scratch, scratch_bytes);
    DgradProb p;
    memset(&p, 0, sizeof p);
    p.pt = pix_tile(n, h, w, BM);
    p.taps.n = 9;
    for (int i = 0; i < 9; ++i) {
        p.taps.dy[i] = HALVE_DY[i];
        p.taps.dx[i] = HALVE_DX[i];
        p.taps.plane[i] = HALVE_CLS[i];
        p.taps.wt[i] = (int8_t)i;
    }
    p.planes_in = 1;
    p.N = n; p.H = h; p.W = w; p.c1 = c; p.c2 = 0; p.cout = cout;
    p.out1 = reinterpret_cast<bf16 *>(dx);
    p.ref1 = reinterpret_cast<const bf16 *>(relu_ref);
    p.rbits1 = relu_bits;  // packed ReLU mask (4 B per 32 channels) instead of the bf16 reference
    p.drop1 = drop_scale;
    p.db1 = dbias;
    const long long mtiles = (long long)p.pt.tw * p.pt.th * p.pt.tn;
    const int bn = pick_bn(c, mtiles);
    if (!map_planes(&p.dym, dy_planes, n, h, w, cout, p.pt)) return ICE_EINVAL;
    if (!map_wgt(&p.wm, wc, cout, 9, c, 64)) return ICE_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const bool m2 = conv_m2(mtiles, c, bn, 1, 9 * (cout / BK));
    const dim3 tiles = m2 ? dim3((unsigned)(mtiles / 2), c / bn, 1) : dim3((unsigned)mtiles, c / bn, 1);
    const ice::RowSched s = sched(tiles, bn, m2 ? 8 : 4);
    take_bias_rows(p, s, ar);
    ICE_SETTLE(ar);
    const int rc = m2 ? launch_bn_m2(p, bn, tiles, st) : launch_bn(p, bn, tiles, st);
    return rc ? rc : finish_bias(p, s, st);
}

extern "C" int ice_halve_wgrad(const uint16_t *x, int32_t c, const uint16_t *dy_planes, int32_t cout, int32_t n,
                               int32_t h, int32_t w, float *dw, void *scratch, uint64_t *scratch_bytes, void *stream) {
    if (!encode_fn()) return ICE_ENODRIVER;
    if (!x || !dy_planes || !dw || c <= 0 || c % 64 || cout <= 0 || cout % 64 || !shape_ok(n, h, w))
        return ICE_EINVAL;
    ice::Arena ar(scratch, scratch_bytes);
    cudaStream_t st = (cudaStream_t)stream;
    if (!knobs().no_halo_wgrad) {
        const int rc = try_hwgrad(x, c, nullptr, 0, dy_planes, cout, n, h, w, dw, ar, scratch_bytes, st, true);
        if (rc <= 0) return rc;  // 1 = not applicable
    }
    WgradProb p;
    memset(&p, 0, sizeof p);
    p.pk = pix_tile(n, h, w, BK);
    p.taps.n = 4;  // (a, b) of the 2x2 kernel; shifts derive from (class, tap) in load()
    p.halve = 1;
    p.N = n; p.H = h; p.W = w; p.c1 = c; p.c2 = 0; p.cout = cout;
    p.dw = dw;
    p.ow = ice::grad_overwrite() ? 1 : 0;
    const int ncols = 4 * c;
    int mtiles, ntiles, bn;
    wgrad_tiles(ncols, cout, p.trans, mtiles, ntiles, bn);
    p.total_kb = 4 * p.pk.tw * p.pk.th * p.pk.tn;
    const bool m2 = wgrad_m2(mtiles, bn, p.total_kb);
    if (m2) mtiles /= 2;
    p.kb_per_split = split_k(p.total_kb, (long long)mtiles * ntiles, num_sms());
    wgrad_boxes(p, m2, bn);
    if (!map_act_nb(&p.dym, dy_planes, 4 * n, h, w, cout, p.pk, p.nby)) return ICE_EINVAL;
    if (!map_act_nb(&p.xa, x, n, h, w, c, p.pk, p.nbx)) return ICE_EINVAL;
    return run_wgrad(p, ncols, mtiles, ntiles, bn, m2, ar, scratch_bytes, st);
}

#ifdef ICE_CONV_PROF
extern "C" int ice_conv_prof_read(unsigned long long *out8, int reset) {
    cudaMemcpyFromSymbol(out8, g_conv_prof, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_conv_prof, z, sizeof z);
    }
    return 0;
}
#endif
