// autolabel.cu -- K1 (fused thin-cloud/shadow filter + HSV segmentation) and K1s
// (segment only) for sm_100a.
//
// One CTA owns one tile for the whole pipeline of engine.process_tile
// (/root/reference/pkg/src/icelabel/engine.py:145-160): every tile-global quantity the
// reference computes (min/max of the difference image, the Otsu histogram, the channel
// medians, the mask population) is a CTA reduction, and all working planes stay in
// shared memory (three 256 x 260 u8 planes ~ 195 KB).  HBM sees the RGB tile once (a
// second read for the output pass hits L2) and the filtered tile + label once.
//
// The expensive part is the 21 x 21 median of estimate_background
// (cloudfilter.py:82-84).  It is computed exactly by threshold decomposition:
//     median(p) = s_0 + sum_{i} [count_{x <= s_i}(window(p)) <= rank] * (s_{i+1} - s_i)
// over the sorted distinct values s_i present in the (dilated) plane.  Each threshold
// costs one separable box count (row pass + column pass, O(1) per pixel), so flat sea-ice
// tiles with a handful of grey levels cost a handful of passes.  Border handling is
// replicate (clamped indices), identical to cv2.medianBlur / BORDER_REPLICATE as pinned
// by the reference oracles (pkg/tests/oracles.py:39-56).
#include <cuda_runtime.h>
#include <stdint.h>

#include "icelabel_b200.h"
#include "reduce.cuh"

#ifdef ICE_AL_PROF
__device__ unsigned long long g_al_prof[16];
#define PROF_MARK(k)                                                          \
    do {                                                                      \
        __syncthreads();                                                      \
        if (threadIdx.x == 0) {                                               \
            long long now = clock64();                                        \
            atomicAdd(&g_al_prof[k], (unsigned long long)(now - prof_t0));    \
            prof_t0 = now;                                                    \
        }                                                                     \
    } while (0)
#else
#define PROF_MARK(k) \
    do {             \
    } while (0)
#endif

namespace {

constexpr int NT = 512;        // threads per CTA
constexpr int MAXD = 256;      // max tile extent handled on chip
constexpr int PITCH = 260;     // plane row pitch: 65 words -> row-parallel access is bank-conflict free
constexpr int PLANE = MAXD * PITCH;

struct Params {
    IceFilterCfg cfg;
    IceScheme scheme;
    int v_only;  // every range passes all hues and saturations: classify on V alone
};

struct Smem {
    uint8_t p[3][PLANE];            // working planes
    uint32_t maskbits[MAXD * MAXD / 32];
    uint32_t hist[256];
    uint32_t present[8];            // 256-bit value-presence set
    int red_i[NT / 32];
    int red_j[NT / 32];
    int bcast[8];
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// ---- block reductions ------------------------------------------------------------
__device__ int block_sum(int v, Smem &s) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s.red_i[threadIdx.x >> 5] = v;
    __syncthreads();
    int t = 0;
    for (int i = 0; i < NT / 32; ++i) t += s.red_i[i];
    return t;
}

__device__ void block_minmax(int &lo, int &hi, Smem &s) {
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        s.red_i[threadIdx.x >> 5] = lo;
        s.red_j[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    lo = 255;
    hi = 0;
    for (int i = 0; i < NT / 32; ++i) {
        lo = min(lo, s.red_i[i]);
        hi = max(hi, s.red_j[i]);
    }
}

// warp-aggregated histogram increment (flat tiles send every lane to one bin)
__device__ __forceinline__ void hist_add(uint32_t *hist, int v, bool active) {
    unsigned act = __ballot_sync(0xffffffffu, active);
    if (!active) return;
    unsigned peers = __match_any_sync(act, v);
    if ((threadIdx.x & 31) == (__ffs(peers) - 1)) atomicAdd(&hist[v], __popc(peers));
}

// ---- windowed primitives on planes -----------------------------------------------
// kernels.py:49-54 dilate: separable max, replicate border. src -> tmp (rows) -> dst (cols)
__device__ void dilate_plane(const uint8_t *src, uint8_t *tmp, uint8_t *dst, int h, int w, int k) {
    int r = k >> 1;
    for (int i = threadIdx.x; i < h * w; i += NT) {
        int y = i / w, x = i - y * w;
        const uint8_t *row = src + y * PITCH;
        int m = 0;
        for (int j = -r; j <= r; ++j) m = max(m, (int)row[clampi(x + j, 0, w - 1)]);
        tmp[y * PITCH + x] = (uint8_t)m;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < h * w; i += NT) {
        int y = i / w, x = i - y * w;
        int m = 0;
        for (int j = -r; j <= r; ++j) m = max(m, (int)tmp[clampi(y + j, 0, h - 1) * PITCH + x]);
        dst[y * PITCH + x] = (uint8_t)m;
    }
    __syncthreads();
}

__device__ void presence(const uint8_t *src, int h, int w, Smem &s) {
    if (threadIdx.x < 8) s.present[threadIdx.x] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < h * w; i += NT) {
        int y = i / w, x = i - y * w;
        int v = src[y * PITCH + x];
        atomicOr(&s.present[v >> 5], 1u << (v & 31));
    }
    __syncthreads();
}

// next present value strictly above t, or -1
__device__ __forceinline__ int next_present(const uint32_t *present, int t) {
    for (int v = t + 1; v < 256;) {
        uint32_t word = present[v >> 5] >> (v & 31);
        if (word) return v + __ffs(word) - 1;
        v = (v | 31) + 1;
    }
    return -1;
}

// kernels.py:42-46 median_blur with k x k window, rank k*k/2, replicate border.
// Exact threshold decomposition.  src: plane D, tmp: H counts, dst: M.
__device__ void median_plane(const uint8_t *src, uint8_t *tmp, uint8_t *dst, int h, int w, int k,
                             Smem &s) {
    const int r = k >> 1;
    const int rank = (k * k) >> 1;
    presence(src, h, w, s);
    int lo = next_present(s.present, -1);
    for (int i = threadIdx.x; i < h * w; i += NT) {
        int y = i / w, x = i - y * w;
        dst[y * PITCH + x] = (uint8_t)lo;
    }
    __syncthreads();
    for (int t = lo, nx = next_present(s.present, lo); nx >= 0; t = nx, nx = next_present(s.present, nx)) {
        const int gap = nx - t;
        // row pass: tmp(y,x) = #{j in [x-r, x+r] : src(y, clamp j) <= t}
        for (int task = threadIdx.x; task < 2 * h; task += NT) {
            int y = task >> 1;
            int half = task & 1;
            int x0 = half ? (w >> 1) : 0, x1 = half ? w : (w >> 1);
            const uint8_t *row = src + y * PITCH;
            uint8_t *out = tmp + y * PITCH;
            int cnt = 0;
            for (int j = x0 - r; j <= x0 + r; ++j) cnt += row[clampi(j, 0, w - 1)] <= t;
            for (int x = x0; x < x1; ++x) {
                out[x] = (uint8_t)cnt;
                cnt += (int)(row[min(x + r + 1, w - 1)] <= t) - (int)(row[max(x - r, 0)] <= t);
            }
        }
        __syncthreads();
        // column pass: window count; pixels whose count <= rank have median > t
        for (int task = threadIdx.x; task < 2 * w; task += NT) {
            int x = task % w;
            int half = task / w;
            int hh = (h + 1) >> 1;
            int y0 = half ? hh : 0, y1 = half ? h : hh;
            int cnt = 0;
            for (int j = y0 - r; j <= y0 + r; ++j) cnt += tmp[clampi(j, 0, h - 1) * PITCH + x];
            for (int y = y0; y < y1; ++y) {
                if (cnt <= rank) dst[y * PITCH + x] += (uint8_t)gap;
                cnt += (int)tmp[min(y + r + 1, h - 1) * PITCH + x] - (int)tmp[max(y - r, 0) * PITCH + x];
            }
        }
        __syncthreads();
    }
}

// per-pixel exact k x k median by bitwise radix select (used for noise_median_k != 3)
__device__ int median_at(const uint8_t *src, int h, int w, int y, int x, int k) {
    const int r = k >> 1, rank = (k * k) >> 1;
    int ans = 0;
    for (int b = 7; b >= 0; --b) {
        int cand = ans | ((1 << b) - 1);  // is the median <= cand ?
        int cnt = 0;
        for (int dy = -r; dy <= r; ++dy) {
            const uint8_t *row = src + clampi(y + dy, 0, h - 1) * PITCH;
            for (int dx = -r; dx <= r; ++dx) cnt += row[clampi(x + dx, 0, w - 1)] <= cand;
        }
        if (cnt <= rank) ans |= 1 << b;
    }
    return ans;
}

#define SORT2(a, b) { int _t = min(a, b); b = max(a, b); a = _t; }
__device__ __forceinline__ int median3x3_at(const uint8_t *src, int h, int w, int y, int x) {
    const uint8_t *r0 = src + clampi(y - 1, 0, h - 1) * PITCH;
    const uint8_t *r1 = src + y * PITCH;
    const uint8_t *r2 = src + clampi(y + 1, 0, h - 1) * PITCH;
    int xl = clampi(x - 1, 0, w - 1), xr = clampi(x + 1, 0, w - 1);
    int p0 = r0[xl], p1 = r0[x], p2 = r0[xr], p3 = r1[xl], p4 = r1[x], p5 = r1[xr];
    int p6 = r2[xl], p7 = r2[x], p8 = r2[xr];
    // 19-exchange median-of-9 network
    SORT2(p1, p2); SORT2(p4, p5); SORT2(p7, p8); SORT2(p0, p1); SORT2(p3, p4); SORT2(p6, p7);
    SORT2(p1, p2); SORT2(p4, p5); SORT2(p7, p8); SORT2(p0, p3); SORT2(p5, p8); SORT2(p4, p7);
    SORT2(p3, p6); SORT2(p1, p4); SORT2(p2, p5); SORT2(p4, p7); SORT2(p4, p2); SORT2(p6, p4);
    SORT2(p4, p2);
    return p4;
}

// ---- HSV + scheme (raster.py:187-216, segmentation.py:118-128), integer-exact form ----
// S = round(255 C / V) = (510 C + V) div 2V ; H = round(hue / 2) = (num + C) div 2C with
// num >= 0 per branch (np.select order V==R, V==G, else).  Equal to the float64 reference
// on all 2^24 RGB triples (tests/test_hsv_integer.py, tests/test_autolabel_gpu.py).
__device__ __forceinline__ void hsv_of(int R, int G, int B, int &H, int &S, int &V) {
    V = max(R, max(G, B));
    int mn = min(R, min(G, B));
    int C = V - mn;
    S = V == 0 ? 0 : (510 * C + V) / (2 * V);
    H = 0;
    if (C > 0) {
        int num;
        if (V == R) num = 60 * (G - B) + (G < B ? 360 * C : 0);
        else if (V == G) num = 60 * (B - R) + 120 * C;
        else num = 60 * (R - G) + 240 * C;
        H = (num + C) / (2 * C);
        if (H == 180) H = 0;
    }
}

// NEED_H / NEED_S = false when every range of the scheme passes all hues / saturations
// (the shipped ross-sea-summer preset): then only V = max(r, g, b) decides the class, and
// the two integer divisions of the HSV conversion are skipped -- exact, since H <= 179 and
// S <= 255 always lie inside full-range boxes.
// Scheme ranges unpacked into registers (indexing the by-value IceScheme parameter through a
// reference spills it to local memory and reloads it per pixel).
struct SchemeR {
    int lo[3][3], hi[3][3], cls[3];
    __device__ __forceinline__ explicit SchemeR(const IceScheme &sc) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                lo[k][c] = sc.lo[k][c];
                hi[k][c] = sc.hi[k][c];
            }
            cls[k] = sc.cls[k];
        }
    }
};

template <bool NEED_H = true, bool NEED_S = true>
__device__ __forceinline__ int classify(int R, int G, int B, const SchemeR &sc) {
    int H = 0, S = 0, V;
    if (NEED_H || NEED_S) {
        hsv_of(R, G, B, H, S, V);
    } else {
        V = max(R, max(G, B));
    }
    int out = 255;
#pragma unroll
    for (int k = 2; k >= 0; --k) {  // first matching range wins
        bool in = V >= sc.lo[k][2] && V <= sc.hi[k][2];
        if (NEED_H) in = in && H >= sc.lo[k][0] && H <= sc.hi[k][0];
        if (NEED_S) in = in && S >= sc.lo[k][1] && S <= sc.hi[k][1];
        out = in ? sc.cls[k] : out;
    }
    return out;
}

__global__ void hsv_kernel(const uint8_t *__restrict__ rgb, int64_t npx, uint8_t *__restrict__ hsv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npx; i += (int64_t)gridDim.x * blockDim.x) {
        int H, S, V;
        hsv_of(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2], H, S, V);
        hsv[3 * i] = (uint8_t)H;
        hsv[3 * i + 1] = (uint8_t)S;
        hsv[3 * i + 2] = (uint8_t)V;
    }
}

// ---- Otsu (kernels.py:77-110) with unsigned 128-bit exact compare ----------------------
__device__ int otsu_from_hist(const uint32_t *hist) {
    // warp 0 only; lane l owns bins [8l, 8l+8)
    int lane = threadIdx.x & 31;
    unsigned long long n_loc = 0, s_loc = 0;
    for (int j = 0; j < 8; ++j) {
        n_loc += hist[8 * lane + j];
        s_loc += (unsigned long long)(8 * lane + j) * hist[8 * lane + j];
    }
    unsigned long long n_pre = n_loc, s_pre = s_loc;  // inclusive scan
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long a = __shfl_up_sync(0xffffffffu, n_pre, o);
        unsigned long long b = __shfl_up_sync(0xffffffffu, s_pre, o);
        if (lane >= o) { n_pre += a; s_pre += b; }
    }
    unsigned long long n_tot = __shfl_sync(0xffffffffu, n_pre, 31);
    unsigned long long s_tot = __shfl_sync(0xffffffffu, s_pre, 31);
    long long n0 = (long long)(n_pre - n_loc), s0 = (long long)(s_pre - s_loc);
    int best_t = -1;
    unsigned __int128 best_num = 0;
    unsigned long long best_den = 1;
    for (int j = 0; j < 8; ++j) {
        int t = 8 * lane + j;
        n0 += hist[t];
        s0 += (long long)t * hist[t];
        long long n1 = (long long)n_tot - n0;
        if (n0 == 0 || n1 == 0) continue;
        long long s1 = (long long)s_tot - s0;
        __int128 diff = (__int128)s0 * n1 - (__int128)s1 * n0;
        unsigned __int128 a = (unsigned __int128)(diff < 0 ? -diff : diff);
        unsigned __int128 num = a * a;
        unsigned long long den = (unsigned long long)(n0 * n1);
        if (best_t < 0 || num * best_den > best_num * den) {
            best_t = t; best_num = num; best_den = den;
        }
    }
    // warp argmax: larger ratio wins; equal ratio -> smaller t; lanes without candidates lose
    for (int o = 16; o; o >>= 1) {
        int ot = __shfl_xor_sync(0xffffffffu, best_t, o);
        unsigned long long on_lo = __shfl_xor_sync(0xffffffffu, (unsigned long long)best_num, o);
        unsigned long long on_hi = __shfl_xor_sync(0xffffffffu, (unsigned long long)(best_num >> 64), o);
        unsigned long long od = __shfl_xor_sync(0xffffffffu, best_den, o);
        unsigned __int128 onum = ((unsigned __int128)on_hi << 64) | on_lo;
        bool take;
        if (ot < 0) take = false;
        else if (best_t < 0) take = true;
        else {
            unsigned __int128 lhs = onum * best_den, rhs = best_num * od;
            take = lhs > rhs || (lhs == rhs && ot < best_t);
        }
        if (take) { best_t = ot; best_num = onum; best_den = od; }
    }
    // reference: the first strict improvement over (0, 1) wins; ratio 0 never beats it
    if (best_t < 0 || best_num == 0) best_t = 0;
    return best_t;
}

// median over all pixels of a channel (np.median, then round_half_up) from a histogram
__device__ int center_from_hist(const uint32_t *hist, int npx) {
    int lo_rank = (npx - 1) >> 1, hi_rank = npx >> 1;
    int a = -1, b = -1, acc = 0;
    for (int v = 0; v < 256; ++v) {
        acc += hist[v];
        if (a < 0 && acc > lo_rank) a = v;
        if (b < 0 && acc > hi_rank) { b = v; break; }
    }
    return (a + b + 1) >> 1;
}

__device__ void load_channel(const uint8_t *tile, int ch, uint8_t *dst, int h, int w) {
    // ch = 3 -> V = max(r,g,b) (cloudfilter.py:89)
    for (int i = threadIdx.x; i < h * w; i += NT) {
        int y = i / w, x = i - y * w;
        const uint8_t *px = tile + 3 * i;
        int v = ch == 3 ? max(px[0], max(px[1], px[2])) : px[ch];
        dst[y * PITCH + x] = (uint8_t)v;
    }
    __syncthreads();
}

__device__ void histogram_plane(const uint8_t *src, int h, int w, Smem &s) {
    for (int i = threadIdx.x; i < 256; i += NT) s.hist[i] = 0;
    __syncthreads();
    int total = h * w;
    for (int base = 0; base < total; base += NT) {
        int i = base + threadIdx.x;
        bool act = i < total;
        int v = 0;
        if (act) {
            int y = i / w, x = i - y * w;
            v = src[y * PITCH + x];
        }
        hist_add(s.hist, v, act);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(NT, 1)
autolabel_kernel(const uint8_t *__restrict__ rgb, int h, int w, Params prm,
                 uint8_t *__restrict__ filtered, uint8_t *__restrict__ label,
                 uint8_t *__restrict__ maskout, uint32_t *__restrict__ affected,
                 uint32_t *__restrict__ counts, int32_t *__restrict__ unmatched) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Smem &s = *reinterpret_cast<Smem *>(smem_raw);
    const IceFilterCfg &cfg = prm.cfg;
    const int npx = h * w;
    const size_t tile_id = blockIdx.x;
    const uint8_t *tile = rgb + tile_id * (size_t)npx * 3;
    uint8_t *ftile = filtered + tile_id * (size_t)npx * 3;
    uint8_t *P0 = s.p[0], *P1 = s.p[1], *P2 = s.p[2];

#ifdef ICE_AL_PROF
    long long prof_t0 = clock64();
#endif
    // 1. V plane, dilate, background = median(dilate(V))   (cloudfilter.py:82-84, 89)
    load_channel(tile, 3, P0, h, w);
    PROF_MARK(0);
    dilate_plane(P0, P2, P1, h, w, cfg.bg_dilate_k);        // D in P1
    PROF_MARK(1);
    median_plane(P1, P2, P0, h, w, cfg.bg_median_k, s);     // bg in P0
    PROF_MARK(2);
    // 2. V again, smooth = median_noise(V); d = |smooth - bg|, [truncate]  (:90-93)
    load_channel(tile, 3, P1, h, w);
    int lo = 255, hi = 0;
    for (int i = threadIdx.x; i < npx; i += NT) {
        int y = i / w, x = i - y * w;
        int sm = cfg.noise_median_k == 3 ? median3x3_at(P1, h, w, y, x)
                                         : median_at(P1, h, w, y, x, cfg.noise_median_k);
        int d = abs(sm - (int)P0[y * PITCH + x]);
        if (cfg.diff_truncate) d = min(d, cfg.truncate_t);
        P2[y * PITCH + x] = (uint8_t)d;
        lo = min(lo, d);
        hi = max(hi, d);
    }
    block_minmax(lo, hi, s);
    PROF_MARK(3);
    // 3. minmax normalize (kernels.py:66-74, exact integer form), Otsu, binary (:94-96)
    for (int i = threadIdx.x; i < 256; i += NT) s.hist[i] = 0;
    __syncthreads();
    const int range = hi - lo;
    for (int base = 0; base < npx; base += NT) {
        int i = base + threadIdx.x;
        bool act = i < npx;
        int dn = 0;
        if (act) {
            int y = i / w, x = i - y * w;
            int d = P2[y * PITCH + x];
            dn = range == 0 ? 0 : (510 * (d - lo) + range) / (2 * range);
            P2[y * PITCH + x] = (uint8_t)dn;
        }
        hist_add(s.hist, dn, act);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        int t = cfg.mask_mode_fixed ? cfg.fixed_t : otsu_from_hist(s.hist);
        if (threadIdx.x == 0) s.bcast[0] = t;
    }
    __syncthreads();
    const int thr = s.bcast[0];
    int cnt = 0;
    int unequal = 0;
    for (int base = 0; base < npx; base += NT) {
        int i = base + threadIdx.x;
        bool m = false;
        if (i < npx) {
            int y = i / w, x = i - y * w;
            m = P2[y * PITCH + x] > thr;
            const uint8_t *px = tile + 3 * i;
            unequal |= (px[0] != px[1]) | (px[1] != px[2]);
        }
        unsigned bits = __ballot_sync(0xffffffffu, m);
        if ((threadIdx.x & 31) == 0 && base + (threadIdx.x & ~31) < npx)
            s.maskbits[(base + threadIdx.x) >> 5] = bits;
        cnt += m;
    }
    const int masked = block_sum(cnt, s);
    const int any_unequal = block_sum(unequal, s);
    PROF_MARK(4);
    // 4. repair (cloudfilter.py:108-116)
    int center[3] = {0, 0, 0};
    if (masked > 0) {
        if (!any_unequal) {
            // R == G == B everywhere: every channel equals V, so bg_c == bg_V (kept in P0)
            histogram_plane(P1, h, w, s);  // P1 still holds V
            int c = center_from_hist(s.hist, npx);
            center[0] = center[1] = center[2] = c;
        } else {
            for (int ch = 0; ch < 3; ++ch) {
                load_channel(tile, ch, P1, h, w);
                histogram_plane(P1, h, w, s);
                int c = center_from_hist(s.hist, npx);
                dilate_plane(P1, P0, P2, h, w, cfg.bg_dilate_k);  // D_c in P2
                median_plane(P2, P1, P0, h, w, cfg.bg_median_k, s);  // bg_c in P0
                for (int i = threadIdx.x; i < npx; i += NT) {
                    if (s.maskbits[i >> 5] >> (i & 31) & 1) {
                        int y = i / w, x = i - y * w;
                        int f = (int)tile[3 * i + ch] - (int)P0[y * PITCH + x] + c;
                        ftile[3 * i + ch] = (uint8_t)clampi(f, 0, 255);
                    }
                }
                __syncthreads();
            }
        }
    }
    PROF_MARK(5);
    // 5. output pass: filtered tile, HSV segmentation, counts, first unmatched
    int c0 = 0, c1 = 0, c2 = 0, first = 0x7fffffff;
    uint8_t *ltile = label + tile_id * (size_t)npx;
    uint8_t *mtile = maskout ? maskout + tile_id * (size_t)npx : nullptr;
    const SchemeR scr(prm.scheme);
    for (int i = threadIdx.x; i < npx; i += NT) {
        int R = tile[3 * i], G = tile[3 * i + 1], B = tile[3 * i + 2];
        const bool mk = masked > 0 && (s.maskbits[i >> 5] >> (i & 31) & 1);
        if (mtile) mtile[i] = mk ? 255 : 0;
        if (mk) {
            if (!any_unequal) {
                int y = i / w, x = i - y * w;
                int bg = P0[y * PITCH + x];
                R = clampi(R - bg + center[0], 0, 255);
                G = clampi(G - bg + center[1], 0, 255);
                B = clampi(B - bg + center[2], 0, 255);
            } else {
                R = ftile[3 * i];
                G = ftile[3 * i + 1];
                B = ftile[3 * i + 2];
            }
        }
        ftile[3 * i] = (uint8_t)R;
        ftile[3 * i + 1] = (uint8_t)G;
        ftile[3 * i + 2] = (uint8_t)B;
        const int cls = prm.v_only ? classify<false, false>(R, G, B, scr) : classify(R, G, B, scr);
        ltile[i] = (uint8_t)cls;
        c0 += cls == 0;
        c1 += cls == 1;
        c2 += cls == 2;
        if (cls == 255) first = min(first, i);
    }
    PROF_MARK(6);
    c0 = block_sum(c0, s);
    c1 = block_sum(c1, s);
    c2 = block_sum(c2, s);
    for (int o = 16; o; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s.red_i[threadIdx.x >> 5] = first;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < NT / 32; ++i) first = min(first, s.red_i[i]);
        affected[tile_id] = (uint32_t)masked;
        counts[3 * tile_id] = c0;
        counts[3 * tile_id + 1] = c1;
        counts[3 * tile_id + 2] = c2;
        unmatched[tile_id] = first == 0x7fffffff ? -1 : first;
    }
}

// =====================================================================================
// Region path: tiles and whole scenes larger than one CTA's 256 x 256 planes
// (cloudfilter.apply_filter on a scene, cli.py:112-125; 512^2 tiles of BASELINE configs[4]).
// The image is cut into cores of at most (256 - 2 * halo)^2 pixels, halo = dilate radius +
// background-median radius (>= noise-median radius).  Each CTA loads its core plus the halo
// clipped to the image, so:
//   * at an image border the region border IS the image border: the clamped indices of
//     dilate_plane / median_plane replicate exactly as cv2's BORDER_REPLICATE does;
//   * at an interior region border, dilated values within dilate-radius of the edge are
//     wrong, but the background median of a core pixel only reads dilated values within
//     median-radius of the core, i.e. >= dilate-radius inside the region.
// The image-global quantities become three launches:
//   1. region_d_kernel      d = |median_noise(V) - median(dilate(V))| [truncated] of the core
//                           -> u8 d plane in scratch; integer histograms of d and of each
//                           channel added into per-image counters (integer atomics: exact,
//                           order-free);
//   2. region_stats_kernel  per image: min/max of d, the exact stretch, Otsu (192-bit exact
//                           compare: scenes beyond ~2^19 pixels overflow 128-bit products),
//                           masked-pixel count, the three channel medians;
//   3. region_out_kernel    mask of the core; per-channel backgrounds only when the core holds
//                           masked pixels; repair, HSV segmentation, per-class counts and the
//                           first unmatched pixel (integer atomics).
//   + region_finish_kernel  per-image outputs.
struct RegionGeom {
    int h, w;          // image extent
    int ny, nx;        // regions per column / row
    int cs_y, cs_x;    // core extent (the last row / column of cores may be shorter)
    int halo;
};

struct RegionBox {
    int cy0, cx0, ch, cw;  // core, image coordinates
    int ry0, rx0, rh, rw;  // core + halo clipped to the image
};

struct RegionStats {       // per image, in caller scratch
    uint32_t hist_d[256];
    uint32_t hist_c[3][256];
    int lo, range, thr, masked;
    int center[3];
    uint32_t counts[3];
    int first;
    int pad[3];
};
static_assert(sizeof(RegionStats) == 4152, "documented in icelabel_b200.h");

__device__ __forceinline__ RegionBox region_box(const RegionGeom &g, int r) {
    RegionBox b;
    const int by = r / g.nx, bx = r - by * g.nx;
    b.cy0 = by * g.cs_y;
    b.ch = min(g.cs_y, g.h - b.cy0);
    b.cx0 = bx * g.cs_x;
    b.cw = min(g.cs_x, g.w - b.cx0);
    b.ry0 = max(b.cy0 - g.halo, 0);
    b.rh = min(b.cy0 + b.ch + g.halo, g.h) - b.ry0;
    b.rx0 = max(b.cx0 - g.halo, 0);
    b.rw = min(b.cx0 + b.cw + g.halo, g.w) - b.rx0;
    return b;
}

// channel ch (3 = V = max(r, g, b), cloudfilter.py:89) of the region -> plane
__device__ void load_region(const uint8_t *img, int w_img, int ch, const RegionBox &b, uint8_t *dst) {
    for (int i = threadIdx.x; i < b.rh * b.rw; i += NT) {
        const int y = i / b.rw, x = i - y * b.rw;
        const uint8_t *px = img + 3 * ((size_t)(b.ry0 + y) * w_img + b.rx0 + x);
        dst[y * PITCH + x] = (uint8_t)(ch == 3 ? max(px[0], max(px[1], px[2])) : px[ch]);
    }
    __syncthreads();
}

__device__ __forceinline__ void flush_hist(const uint32_t *sh, uint32_t *gh) {
    for (int i = threadIdx.x; i < 256; i += NT)
        if (sh[i]) atomicAdd(&gh[i], sh[i]);
}

__global__ void __launch_bounds__(NT, 1)
region_d_kernel(const uint8_t *__restrict__ rgb, RegionGeom g, IceFilterCfg cfg, int regions,
                uint8_t *__restrict__ dplanes, RegionStats *__restrict__ st) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Smem &s = *reinterpret_cast<Smem *>(smem_raw);
    const int img = blockIdx.x / regions;
    const RegionBox b = region_box(g, blockIdx.x - img * regions);
    const size_t npx = (size_t)g.h * g.w;
    const uint8_t *im = rgb + img * npx * 3;
    uint8_t *dp = dplanes + img * npx;
    RegionStats &S = st[img];
    uint8_t *P0 = s.p[0], *P1 = s.p[1], *P2 = s.p[2];
    // background of V over the region (cloudfilter.py:82-84, 89)
    load_region(im, g.w, 3, b, P0);
    dilate_plane(P0, P2, P1, b.rh, b.rw, cfg.bg_dilate_k);
    median_plane(P1, P2, P0, b.rh, b.rw, cfg.bg_median_k, s);
    load_region(im, g.w, 3, b, P1);
    for (int i = threadIdx.x; i < 256; i += NT) s.hist[i] = 0;
    uint32_t *hc = reinterpret_cast<uint32_t *>(P2);  // 3 channel histograms (P2 is free now)
    for (int i = threadIdx.x; i < 3 * 256; i += NT) hc[i] = 0;
    __syncthreads();
    const int oy = b.cy0 - b.ry0, ox = b.cx0 - b.rx0, cn = b.ch * b.cw;
    for (int base = 0; base < cn; base += NT) {
        const int i = base + threadIdx.x;
        const bool act = i < cn;
        int d = 0, r = 0, gr = 0, bl = 0;
        if (act) {
            const int y = i / b.cw, x = i - y * b.cw, ly = oy + y, lx = ox + x;
            const int sm = cfg.noise_median_k == 3 ? median3x3_at(P1, b.rh, b.rw, ly, lx)
                                                   : median_at(P1, b.rh, b.rw, ly, lx, cfg.noise_median_k);
            d = abs(sm - (int)P0[ly * PITCH + lx]);
            if (cfg.diff_truncate) d = min(d, cfg.truncate_t);
            const size_t gi = (size_t)(b.cy0 + y) * g.w + b.cx0 + x;
            dp[gi] = (uint8_t)d;
            const uint8_t *px = im + 3 * gi;
            r = px[0];
            gr = px[1];
            bl = px[2];
        }
        hist_add(s.hist, d, act);
        hist_add(hc, r, act);
        hist_add(hc + 256, gr, act);
        hist_add(hc + 512, bl, act);
    }
    __syncthreads();
    flush_hist(s.hist, S.hist_d);
    for (int c = 0; c < 3; ++c) flush_hist(hc + 256 * c, S.hist_c[c]);
}

// a1^2 * d2 > a2^2 * d1 exactly (320-bit products; kernels.py:104-106 compares Python ints)
__device__ bool sq_ratio_greater(unsigned __int128 a1, uint64_t d1, unsigned __int128 a2, uint64_t d2) {
    uint64_t x1[2] = {(uint64_t)a1, (uint64_t)(a1 >> 64)}, x2[2] = {(uint64_t)a2, (uint64_t)(a2 >> 64)};
    uint64_t q1[4] = {0, 0, 0, 0}, q2[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        unsigned __int128 c1 = 0, c2 = 0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            c1 += (unsigned __int128)x1[i] * x1[j] + q1[i + j];
            q1[i + j] = (uint64_t)c1;
            c1 >>= 64;
            c2 += (unsigned __int128)x2[i] * x2[j] + q2[i + j];
            q2[i + j] = (uint64_t)c2;
            c2 >>= 64;
        }
        q1[i + 2] = (uint64_t)c1;
        q2[i + 2] = (uint64_t)c2;
    }
    uint64_t l[5], r[5];
    unsigned __int128 cl = 0, cr = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        cl += (unsigned __int128)q1[i] * d2;
        l[i] = (uint64_t)cl;
        cl >>= 64;
        cr += (unsigned __int128)q2[i] * d1;
        r[i] = (uint64_t)cr;
        cr >>= 64;
    }
    l[4] = (uint64_t)cl;
    r[4] = (uint64_t)cr;
#pragma unroll
    for (int i = 4; i >= 0; --i)
        if (l[i] != r[i]) return l[i] > r[i];
    return false;
}

// Otsu (kernels.py:77-110) for any pixel count < 2^32: warp 0, lane l owns bins [8l, 8l+8)
__device__ int otsu_wide(const uint32_t *hist) {
    const int lane = threadIdx.x & 31;
    unsigned long long n_loc = 0, s_loc = 0;
    for (int j = 0; j < 8; ++j) {
        n_loc += hist[8 * lane + j];
        s_loc += (unsigned long long)(8 * lane + j) * hist[8 * lane + j];
    }
    unsigned long long n_pre = n_loc, s_pre = s_loc;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long a = __shfl_up_sync(0xffffffffu, n_pre, o);
        const unsigned long long c = __shfl_up_sync(0xffffffffu, s_pre, o);
        if (lane >= o) { n_pre += a; s_pre += c; }
    }
    const unsigned long long n_tot = __shfl_sync(0xffffffffu, n_pre, 31);
    const unsigned long long s_tot = __shfl_sync(0xffffffffu, s_pre, 31);
    unsigned long long n0 = n_pre - n_loc, s0 = s_pre - s_loc;
    int best_t = -1;
    unsigned __int128 best_a = 0;
    unsigned long long best_den = 1;
    for (int j = 0; j < 8; ++j) {
        const int t = 8 * lane + j;
        n0 += hist[t];
        s0 += (unsigned long long)t * hist[t];
        const unsigned long long n1 = n_tot - n0;
        if (n0 == 0 || n1 == 0) continue;
        const unsigned long long s1 = s_tot - s0;
        const unsigned __int128 p = (unsigned __int128)s0 * n1, q = (unsigned __int128)s1 * n0;
        const unsigned __int128 a = p > q ? p - q : q - p;
        const unsigned long long den = n0 * n1;
        if (best_t < 0 || sq_ratio_greater(a, den, best_a, best_den)) {
            best_t = t; best_a = a; best_den = den;
        }
    }
    for (int o = 16; o; o >>= 1) {
        const int ot = __shfl_xor_sync(0xffffffffu, best_t, o);
        const unsigned long long alo = __shfl_xor_sync(0xffffffffu, (unsigned long long)best_a, o);
        const unsigned long long ahi = __shfl_xor_sync(0xffffffffu, (unsigned long long)(best_a >> 64), o);
        const unsigned long long od = __shfl_xor_sync(0xffffffffu, best_den, o);
        const unsigned __int128 oa = ((unsigned __int128)ahi << 64) | alo;
        bool take;
        if (ot < 0) take = false;
        else if (best_t < 0) take = true;
        else take = sq_ratio_greater(oa, od, best_a, best_den) ||
                    (!sq_ratio_greater(best_a, best_den, oa, od) && ot < best_t);
        if (take) { best_t = ot; best_a = oa; best_den = od; }
    }
    if (best_t < 0 || best_a == 0) best_t = 0;  // ratio 0 never beats the initial (0, 1)
    return best_t;
}

__device__ __forceinline__ int stretch(int d, int lo, int range) {  // kernels.py:66-74, exact
    return range == 0 ? 0 : (510 * (d - lo) + range) / (2 * range);
}

__global__ void __launch_bounds__(256)
region_stats_kernel(RegionStats *__restrict__ st, int npx, IceFilterCfg cfg) {
    __shared__ uint32_t hn[256];
    __shared__ int slo, shi, sthr;
    __shared__ uint32_t smasked;
    RegionStats &S = st[blockIdx.x];
    const int t = threadIdx.x;
    if (t == 0) { slo = 255; shi = 0; smasked = 0; }
    hn[t] = 0;
    __syncthreads();
    const uint32_t c = S.hist_d[t];
    if (c) { atomicMin(&slo, t); atomicMax(&shi, t); }
    __syncthreads();
    const int lo = slo, range = shi - slo;
    const int dn = stretch(t, lo, range);
    if (c) atomicAdd(&hn[dn], c);
    __syncthreads();
    if (t < 32) {
        const int thr = cfg.mask_mode_fixed ? cfg.fixed_t : otsu_wide(hn);
        if (t == 0) sthr = thr;
    }
    __syncthreads();
    if (c && dn > sthr) atomicAdd(&smasked, c);
    if (t < 3) S.center[t] = center_from_hist(S.hist_c[t], npx);
    __syncthreads();
    if (t == 0) {
        S.lo = lo; S.range = range; S.thr = sthr; S.masked = (int)smasked;
        S.counts[0] = S.counts[1] = S.counts[2] = 0;
        S.first = 0x7fffffff;
    }
}

__global__ void __launch_bounds__(NT, 1)
region_out_kernel(const uint8_t *__restrict__ rgb, RegionGeom g, Params prm, int regions,
                  const uint8_t *__restrict__ dplanes, RegionStats *__restrict__ st,
                  uint8_t *__restrict__ filtered, uint8_t *__restrict__ label, uint8_t *__restrict__ maskout) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Smem &s = *reinterpret_cast<Smem *>(smem_raw);
    const IceFilterCfg &cfg = prm.cfg;
    const int img = blockIdx.x / regions;
    const RegionBox b = region_box(g, blockIdx.x - img * regions);
    const size_t npx = (size_t)g.h * g.w;
    const uint8_t *im = rgb + img * npx * 3;
    const uint8_t *dp = dplanes + img * npx;
    uint8_t *fim = filtered + img * npx * 3;
    RegionStats &S = st[img];
    const int lo = S.lo, range = S.range, thr = S.thr;
    uint8_t *P0 = s.p[0], *P1 = s.p[1], *P2 = s.p[2];
    const int oy = b.cy0 - b.ry0, ox = b.cx0 - b.rx0, cn = b.ch * b.cw;
    // 1. the core's mask (cloudfilter.py:94-96 on the image-global stretch and threshold)
    int cnt = 0;
    for (int base = 0; base < cn; base += NT) {
        const int i = base + threadIdx.x;
        bool m = false;
        if (i < cn) {
            const int y = i / b.cw, x = i - y * b.cw;
            m = stretch(dp[(size_t)(b.cy0 + y) * g.w + b.cx0 + x], lo, range) > thr;
        }
        const unsigned bits = __ballot_sync(0xffffffffu, m);
        if ((threadIdx.x & 31) == 0 && base + (threadIdx.x & ~31) < cn) s.maskbits[(base + threadIdx.x) >> 5] = bits;
        cnt += m;
    }
    const bool repair = block_sum(cnt, s) > 0;
    // 2. per-channel backgrounds of the region, only where the core has masked pixels
    bool gray = true;
    if (repair) {
        int unequal = 0;
        for (int i = threadIdx.x; i < b.rh * b.rw; i += NT) {
            const int y = i / b.rw, x = i - y * b.rw;
            const uint8_t *px = im + 3 * ((size_t)(b.ry0 + y) * g.w + b.rx0 + x);
            unequal |= (px[0] != px[1]) | (px[1] != px[2]);
        }
        gray = block_sum(unequal, s) == 0;
        if (gray) {  // R == G == B over the region: every channel's background is V's (in P0)
            load_region(im, g.w, 3, b, P1);
            dilate_plane(P1, P0, P2, b.rh, b.rw, cfg.bg_dilate_k);
            median_plane(P2, P1, P0, b.rh, b.rw, cfg.bg_median_k, s);
        } else {
            for (int ch = 0; ch < 3; ++ch) {
                load_region(im, g.w, ch, b, P1);
                dilate_plane(P1, P0, P2, b.rh, b.rw, cfg.bg_dilate_k);
                median_plane(P2, P1, P0, b.rh, b.rw, cfg.bg_median_k, s);
                const int cc = S.center[ch];
                for (int i = threadIdx.x; i < cn; i += NT) {
                    if (s.maskbits[i >> 5] >> (i & 31) & 1) {
                        const int y = i / b.cw, x = i - y * b.cw;
                        const size_t gi = (size_t)(b.cy0 + y) * g.w + b.cx0 + x;
                        fim[3 * gi + ch] = (uint8_t)clampi((int)im[3 * gi + ch] - (int)P0[(oy + y) * PITCH + ox + x] + cc, 0, 255);
                    }
                }
                __syncthreads();
            }
        }
    }
    // 3. output: filtered core, mask, HSV segmentation, counts, first unmatched
    int c0 = 0, c1 = 0, c2 = 0, first = 0x7fffffff;
    uint8_t *lim = label + img * npx;
    uint8_t *mim = maskout ? maskout + img * npx : nullptr;
    const SchemeR scr(prm.scheme);
    for (int i = threadIdx.x; i < cn; i += NT) {
        const int y = i / b.cw, x = i - y * b.cw;
        const size_t gi = (size_t)(b.cy0 + y) * g.w + b.cx0 + x;
        int R = im[3 * gi], G = im[3 * gi + 1], B = im[3 * gi + 2];
        const bool mk = repair && (s.maskbits[i >> 5] >> (i & 31) & 1);
        if (mim) mim[gi] = mk ? 255 : 0;
        if (mk) {
            if (gray) {
                const int bg = P0[(oy + y) * PITCH + ox + x];
                R = clampi(R - bg + S.center[0], 0, 255);
                G = clampi(G - bg + S.center[1], 0, 255);
                B = clampi(B - bg + S.center[2], 0, 255);
            } else {
                R = fim[3 * gi];
                G = fim[3 * gi + 1];
                B = fim[3 * gi + 2];
            }
        }
        fim[3 * gi] = (uint8_t)R;
        fim[3 * gi + 1] = (uint8_t)G;
        fim[3 * gi + 2] = (uint8_t)B;
        const int cls = prm.v_only ? classify<false, false>(R, G, B, scr) : classify(R, G, B, scr);
        lim[gi] = (uint8_t)cls;
        c0 += cls == 0;
        c1 += cls == 1;
        c2 += cls == 2;
        if (cls == 255) first = min(first, (int)gi);
    }
    c0 = block_sum(c0, s);
    c1 = block_sum(c1, s);
    c2 = block_sum(c2, s);
    for (int o = 16; o; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s.red_i[threadIdx.x >> 5] = first;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < NT / 32; ++i) first = min(first, s.red_i[i]);
        if (c0) atomicAdd(&S.counts[0], (uint32_t)c0);
        if (c1) atomicAdd(&S.counts[1], (uint32_t)c1);
        if (c2) atomicAdd(&S.counts[2], (uint32_t)c2);
        if (first != 0x7fffffff) atomicMin(&S.first, first);
    }
}

__global__ void region_finish_kernel(const RegionStats *__restrict__ st, int n, uint32_t *__restrict__ affected,
                                     uint32_t *__restrict__ counts, int32_t *__restrict__ unmatched) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const RegionStats &S = st[i];
    affected[i] = (uint32_t)S.masked;
    counts[3 * i] = S.counts[0];
    counts[3 * i + 1] = S.counts[1];
    counts[3 * i + 2] = S.counts[2];
    unmatched[i] = S.first == 0x7fffffff ? -1 : S.first;
}

// K1s: segment only.  One CTA per tile, any size.
constexpr int SEG_NT = 256;
__global__ void __launch_bounds__(SEG_NT)
segment_kernel(const uint8_t *__restrict__ rgb, int npx, IceScheme sc_in, uint8_t *__restrict__ label,
               uint32_t *__restrict__ counts, int32_t *__restrict__ unmatched) {
    const SchemeR sc(sc_in);
    __shared__ int red[4][SEG_NT / 32];
    const size_t tile_id = blockIdx.x;
    const uint8_t *tile = rgb + tile_id * (size_t)npx * 3;
    uint8_t *ltile = label + tile_id * (size_t)npx;
    int c0 = 0, c1 = 0, c2 = 0, first = 0x7fffffff;
    for (int i = threadIdx.x; i < npx; i += SEG_NT) {
        int cls = classify(tile[3 * i], tile[3 * i + 1], tile[3 * i + 2], sc);
        ltile[i] = (uint8_t)cls;
        c0 += cls == 0;
        c1 += cls == 1;
        c2 += cls == 2;
        if (cls == 255) first = min(first, i);
    }
    for (int o = 16; o; o >>= 1) {
        c0 += __shfl_xor_sync(0xffffffffu, c0, o);
        c1 += __shfl_xor_sync(0xffffffffu, c1, o);
        c2 += __shfl_xor_sync(0xffffffffu, c2, o);
        first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    }
    if ((threadIdx.x & 31) == 0) {
        int wi = threadIdx.x >> 5;
        red[0][wi] = c0; red[1][wi] = c1; red[2][wi] = c2; red[3][wi] = first;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < SEG_NT / 32; ++i) {
            c0 += red[0][i]; c1 += red[1][i]; c2 += red[2][i]; first = min(first, red[3][i]);
        }
        counts[3 * tile_id] = c0;
        counts[3 * tile_id + 1] = c1;
        counts[3 * tile_id + 2] = c2;
        unmatched[tile_id] = first == 0x7fffffff ? -1 : first;
    }
}

// K1s vectorised: 16 pixels per thread per step (3 x 16 B RGB loads, one 16 B label store);
// requires npx % 16 == 0 (tile bases are then 16 B aligned).  HBM-bound: 4 B/px.
constexpr int SEG_VNT = 128, SEG_U = 4;
template <bool NH, bool NS>
__global__ void __launch_bounds__(SEG_VNT)
segment_vec_kernel(const uint8_t *__restrict__ rgb, int npx, IceScheme sc_in, uint8_t *__restrict__ label,
                   uint32_t *__restrict__ counts, int32_t *__restrict__ unmatched) {
    const SchemeR sc(sc_in);
    __shared__ uint32_t vlut[256];  // V -> class | count increment (V-only schemes)
    if (!NH && !NS) {
        for (int v = threadIdx.x; v < 256; v += SEG_VNT) {
            int cls = 255;
#pragma unroll
            for (int k = 2; k >= 0; --k)
                if (v >= sc.lo[k][2] && v <= sc.hi[k][2]) cls = sc.cls[k];
            const int slot = cls == 255 ? 3 : cls;
            vlut[v] = (uint32_t)cls | (slot <= 3 ? 1u << (12 + 5 * slot) : 0u);
        }
        __syncthreads();
    }
    __shared__ int red[4][SEG_VNT / 32];
    const size_t tile_id = blockIdx.x;
    const uint4 *tile = reinterpret_cast<const uint4 *>(rgb + tile_id * (size_t)npx * 3);
    uint4 *ltile = reinterpret_cast<uint4 *>(label + tile_id * (size_t)npx);
    int c0 = 0, c1 = 0, c2 = 0, first = 0x7fffffff;
    // Each warp moves SEG_U x 32 groups (SEG_U x 1,536 B) per step with fully coalesced 512 B
    // loads (all issued before any is consumed), bounced through shared memory so that lane l
    // then owns group l of each 32-group slice (pixels 16 l .. 16 l + 15).
    __shared__ uint4 stage[SEG_VNT / 32][SEG_U * 96];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int ngroups = npx / 16;
    uint4 *st = stage[wid];
    for (int gb = wid * 32 * SEG_U; gb < ngroups; gb += SEG_VNT * SEG_U) {
        const int valid = min(32 * SEG_U, ngroups - gb);
        uint4 r[3 * SEG_U];
#pragma unroll
        for (int j = 0; j < 3 * SEG_U; ++j) {
            const int idx = j * 32 + lane;
            if (idx < 3 * valid) r[j] = __ldg(tile + 3 * (size_t)gb + idx);
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 3 * SEG_U; ++j) st[j * 32 + lane] = r[j];
        __syncwarp();
#pragma unroll
        for (int u = 0; u < SEG_U; ++u) {
            const int gl = u * 32 + lane;
            if (gl < valid) {
                const uint4 a = st[3 * gl], b = st[3 * gl + 1], c = st[3 * gl + 2];
                const uint32_t wv[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
                uint32_t lw[4] = {0, 0, 0, 0};
                const int g = gb + gl;
                if (!NH && !NS) {
                    // V-only scheme: one shared-memory lookup per pixel yields the class byte and a
                    // packed count increment; the 16 increments of a group sum without overflow.
                    uint32_t sum = 0;
                    uint32_t e[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        // one PRMT per channel byte (zero-extended), one 3-way max
                        const uint32_t R = __byte_perm(wv[(3 * k) >> 2], 0, 0x4440 | ((3 * k) & 3));
                        const uint32_t G = __byte_perm(wv[(3 * k + 1) >> 2], 0, 0x4440 | ((3 * k + 1) & 3));
                        const uint32_t B = __byte_perm(wv[(3 * k + 2) >> 2], 0, 0x4440 | ((3 * k + 2) & 3));
                        e[k] = vlut[max(R, max(G, B))];
                        sum += e[k];
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        lw[q] = __byte_perm(__byte_perm(e[4 * q], e[4 * q + 1], 0x0040),
                                            __byte_perm(e[4 * q + 2], e[4 * q + 3], 0x0040), 0x5410);
                    c0 += (sum >> 12) & 31;
                    c1 += (sum >> 17) & 31;
                    c2 += (sum >> 22) & 31;
                    if (sum >> 27) {
#pragma unroll
                        for (int k = 15; k >= 0; --k)
                            if ((e[k] & 255) == 255) first = min(first, 16 * g + k);
                    }
                } else {
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int R = (wv[(3 * k) >> 2] >> (8 * ((3 * k) & 3))) & 255;
                    const int G = (wv[(3 * k + 1) >> 2] >> (8 * ((3 * k + 1) & 3))) & 255;
                    const int B = (wv[(3 * k + 2) >> 2] >> (8 * ((3 * k + 2) & 3))) & 255;
                    const int cls = classify<NH, NS>(R, G, B, sc);
                    lw[k >> 2] |= (uint32_t)cls << (8 * (k & 3));
                    c0 += cls == 0;
                    c1 += cls == 1;
                    c2 += cls == 2;
                    if (cls == 255) first = min(first, 16 * g + k);
                }
                }
                ltile[g] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        c0 += __shfl_xor_sync(0xffffffffu, c0, o);
        c1 += __shfl_xor_sync(0xffffffffu, c1, o);
        c2 += __shfl_xor_sync(0xffffffffu, c2, o);
        first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    }
    if ((threadIdx.x & 31) == 0) {
        int wi = threadIdx.x >> 5;
        red[0][wi] = c0; red[1][wi] = c1; red[2][wi] = c2; red[3][wi] = first;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < SEG_VNT / 32; ++i) {
            c0 += red[0][i]; c1 += red[1][i]; c2 += red[2][i]; first = min(first, red[3][i]);
        }
        counts[3 * tile_id] = c0;
        counts[3 * tile_id + 1] = c1;
        counts[3 * tile_id + 2] = c2;
        unmatched[tile_id] = first == 0x7fffffff ? -1 : first;
    }
}

// =====================================================================================
// K1 fast path: 256 x 256 tiles with the default windows (dilate 7, background median 21,
// noise median 3).  Same pipeline and the same exact arithmetic as autolabel_kernel, but
// every plane is processed 4 pixels per 32-bit word (SWAR):
//   * the 21 x 21 median's threshold passes count "D > t" with a carry trick (5 ops / 4 px),
//     sum 21-wide row windows by log-doubling of byte lanes (counts <= 21 fit a byte), and
//     sum 21-tall column windows by sliding 16-bit lanes (<= 441), so one pass costs ~9
//     integer ops per pixel instead of ~80 byte-granular shared-memory operations;
//   * the per-pixel median accumulator lives in registers for the whole pass loop, and the
//     loop stops as soon as no pixel's median exceeds the current threshold;
//   * 7 x 7 dilation by log-doubling maxima, the 3 x 3 noise median from column-sorted
//     triples (max of mins / median of medians / min of maxes);
//   * the RGB tile is read with 16-byte loads, filtered tile + label written with 16-byte
//     stores.
// Plane layout: 256 rows x 65 words (64 + 1 pad: row- and column-parallel sweeps are both
// bank-conflict free).  Thread maps: "row" = (row = tid & 255, half = tid >> 8, 32 words);
// "col" = (word column = tid & 63, band = tid >> 6, 32 rows); "group" = 16 px per step.
namespace fastk {

constexpr int NTF = 512;
constexpr int WP = 65;
constexpr int PW = 256 * WP;
constexpr int MK = 21, MR = 10, MRANK = (MK * MK) / 2, MGE = MK * MK - MRANK;  // median > t <=> #(x > t) >= MGE

struct SmemF {
    uint32_t p[3][PW];
    uint32_t maskbits[2048];
    uint32_t hist[256];
    uint32_t hist2[256];
    uint32_t vlut[256];
    uint8_t flags[256];
    uint8_t vals[256];
    uint8_t rank[256];      // value -> 0x80 | index in vals (median21 rank mode)
    int red[NTF / 32][4];
    int bc[8];
    int act[16];            // median21 block activity, [band][half]
    int kmin[16], kmax[16]; // median21 coarse buckets per block
    unsigned int done_bits; // median21: blocks whose current bucket is final
    unsigned int need_bits; // blocks holding masked pixels (the channel repair needs bg_c only there)
    uint32_t hist_v[256];   // histogram of V (channel median of the gray repair)
};

__device__ __forceinline__ uint32_t fsr(uint32_t lo, uint32_t hi, int n) { return __funnelshift_r(lo, hi, n); }
__device__ __forceinline__ uint32_t fsl(uint32_t lo, uint32_t hi, int n) { return __funnelshift_l(lo, hi, n); }
__device__ __forceinline__ uint32_t even16(uint32_t w) { return __byte_perm(w, 0, 0x4240); }  // bytes 0, 2
__device__ __forceinline__ uint32_t odd16(uint32_t w) { return __byte_perm(w, 0, 0x4341); }   // bytes 1, 3
__device__ __forceinline__ uint32_t rep0(uint32_t w) { return __byte_perm(w, 0, 0x0000); }
__device__ __forceinline__ uint32_t rep3(uint32_t w) { return __byte_perm(w, 0, 0x3333); }
__device__ __forceinline__ uint32_t vmax(uint32_t a, uint32_t b) { return __vmaxu4(a, b); }
__device__ __forceinline__ uint32_t vmin(uint32_t a, uint32_t b) { return __vminu4(a, b); }
// V = max(r, g, b) per byte; gray words (r == g == b, the sea-ice corpus) skip the emulated
// byte-wise maxima
__device__ __forceinline__ uint32_t vmax3(uint32_t r, uint32_t g, uint32_t b) {
    return ((r ^ g) | (g ^ b)) ? __vmaxu4(r, __vmaxu4(g, b)) : r;
}
// per byte: 1 if x > t, else 0; c4 = (255 - t) * 0x01010101, c7f = c4 & 0x7f7f7f7f
// (x + (255 - t) carries out of the byte  <=>  x > t; carry = majority(x7, c7, carry-in7))
__device__ __forceinline__ uint32_t gt4(uint32_t x, uint32_t c4, uint32_t c7f) {
    const uint32_t p = (x & 0x7f7f7f7fu) + c7f;
    const uint32_t m = (x & c4) | ((x | c4) & p);
    return (m >> 7) & 0x01010101u;
}
// word k of a plane row, replicate border (cv2 BORDER_REPLICATE / clamped indices)
__device__ __forceinline__ uint32_t ldw(const uint32_t *row, int k) {
    return k < 0 ? rep0(row[0]) : (k > 63 ? rep3(row[63]) : row[k]);
}
// ---- 7 x 7 dilation (kernels.py:49-54): src -> tmp (row max) -> dst (column max) ----------
// Also records the presence of every value of dst in s.flags.
__device__ void dilate7(const uint32_t *src, uint32_t *tmp, uint32_t *dst, SmemF &s) {
    {
        const int row = threadIdx.x & 255, m0 = (threadIdx.x >> 8) * 32;
        const uint32_t *sr = src + row * WP;
        uint32_t *dr = tmp + row * WP;
        uint32_t x[36], m2[35], m4[34], m7[33];
#pragma unroll
        for (int j = 0; j < 36; ++j) x[j] = ldw(sr, m0 - 1 + j);
#pragma unroll
        for (int j = 0; j < 35; ++j) m2[j] = vmax(x[j], fsr(x[j], x[j + 1], 8));
#pragma unroll
        for (int j = 0; j < 34; ++j) m4[j] = vmax(m2[j], fsr(m2[j], m2[j + 1], 16));
#pragma unroll
        for (int j = 0; j < 33; ++j) m7[j] = vmax(m4[j], fsr(m4[j], m4[j + 1], 24));
#pragma unroll
        for (int j = 0; j < 32; ++j) dr[m0 + j] = fsr(m7[j], m7[j + 1], 8);
    }
    __syncthreads();
    {
        const int c = threadIdx.x & 63, y0 = (threadIdx.x >> 6) * 32;
        uint32_t last = 0xffffffffu;
        bool have = false;
#pragma unroll 1
        for (int yc = y0; yc < y0 + 32; yc += 8) {
            uint32_t r[14], a[13], b[11];
#pragma unroll
            for (int j = 0; j < 14; ++j) r[j] = tmp[clampi(yc - 3 + j, 0, 255) * WP + c];
#pragma unroll
            for (int j = 0; j < 13; ++j) a[j] = vmax(r[j], r[j + 1]);
#pragma unroll
            for (int j = 0; j < 11; ++j) b[j] = vmax(a[j], a[j + 2]);
#pragma unroll
            for (int y = 0; y < 8; ++y) {
                const uint32_t o = vmax(b[y], b[y + 3]);  // rows yc + y - 3 .. yc + y + 3
                dst[(yc + y) * WP + c] = o;
                if (!have || o != last) {
                    s.flags[o & 255] = 1;
                    s.flags[(o >> 8) & 255] = 1;
                    s.flags[(o >> 16) & 255] = 1;
                    s.flags[o >> 24] = 1;
                    last = o;
                    have = true;
                }
            }
        }
    }
}

// sorted list of the values flagged in s.flags -> s.vals[0..nd); returns nd (all threads)
__device__ int collect_values(SmemF &s) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (wid < 8) {
        const unsigned b = __ballot_sync(0xffffffffu, s.flags[32 * wid + lane] != 0);
        if (lane == 0) s.red[wid][0] = __popc(b);
    }
    __syncthreads();
    if (wid < 8) {
        int base = 0;
        for (int i = 0; i < wid; ++i) base += s.red[i][0];
        const int v = 32 * wid + lane;
        const unsigned b = __ballot_sync(0xffffffffu, s.flags[v] != 0);
        const int r = base + __popc(b & ((1u << lane) - 1));
        if (s.flags[v]) {
            s.vals[r] = (uint8_t)v;
            s.rank[v] = (uint8_t)(0x80 | r);
        }
    }
    __syncthreads();
    int nd = 0;
    for (int i = 0; i < 8; ++i) nd += s.red[i][0];
    return nd;
}

// ---- row pass of one threshold: dst(y, x) = #{j in [x-10, x+10] : src(y, clamp j) > t} ----
// 16 output words per call.  local j <-> word k = m0 - 3 + j.  s2: 2-px sums, s4: 4-px sums
// (<= 4 per byte), t_k = s4_k + .. + s4_{k+4} + i_{k+5}: the 21 px from 4k + byte.
// EDGE: 0 interior, 1 left tile edge (m0 == 0), 2 right tile edge (m0 == 48).
// RANK: the plane holds 0x80 | rank(value) (nd <= 128) and "x > t_i" is one subtraction:
// bit 7 of (0x80 + r - (i + 1)) per byte (no borrow since r, i + 1 <= 128); k = (i+1)*0x01010101.
// Otherwise the plane holds values and gt4 (c = (255 - t) * 0x01010101) is used.
template <int EDGE, bool RANK>
__device__ __forceinline__ void row_chunk(const uint32_t *sr, uint32_t *dr, int m0, uint32_t k) {
    uint32_t I[23], S2[22], S4[21], S8[19], T[17];
#pragma unroll
    for (int j = 0; j < 23; ++j) {
        uint32_t w;
        if (EDGE == 1 && j < 3) w = rep0(sr[0]);
        else if (EDGE == 2 && j >= 19) w = rep3(sr[63]);
        else w = sr[m0 - 3 + j];
        I[j] = RANK ? ((w - k) >> 7) & 0x01010101u : gt4(w, k, k & 0x7f7f7f7fu);
    }
#pragma unroll
    for (int j = 0; j < 22; ++j) S2[j] = I[j] + fsr(I[j], I[j + 1], 8);
#pragma unroll
    for (int j = 0; j < 21; ++j) S4[j] = S2[j] + fsr(S2[j], S2[j + 1], 16);
#pragma unroll
    for (int j = 0; j < 19; ++j) S8[j] = S4[j] + S4[j + 1];
#pragma unroll
    for (int j = 0; j < 17; ++j) T[j] = S8[j] + S8[j + 2] + S4[j + 4] + I[j + 5];
    // pixel 4m + i has its window start at 4(m - 3) + i + 2
#pragma unroll
    for (int j = 0; j < 16; ++j) dr[m0 + j] = fsr(T[j], T[j + 1], 16);
}

template <bool RANK>
__device__ __forceinline__ void row_counts(const uint32_t *src, uint32_t *dst, uint32_t k) {
    const int row = threadIdx.x & 255, half = threadIdx.x >> 8;
    const uint32_t *sr = src + row * WP;
    uint32_t *dr = dst + row * WP;
    if (half == 0) {
        row_chunk<1, RANK>(sr, dr, 0, k);
        row_chunk<0, RANK>(sr, dr, 16, k);
    } else {
        row_chunk<0, RANK>(sr, dr, 32, k);
        row_chunk<2, RANK>(sr, dr, 48, k);
    }
}

// ---- column pass: window count >= MGE (median > t) adds gap to the pixel's median --------
// Sliding 16-bit lane sums (even / odd pixels of the word), biased by K so that bit 15 of a
// lane is the comparison.  EDGE: 0 interior band, 1 top band, 2 bottom band (clamped rows).
// MODE 0: acc += bits * arg (value-mode median, arg = value gap); MODE 1: acc += bits (rank
// units); MODE 2: acc += bits where acc <= i (arg = (i | 0x80) per byte: the fine pass of
// rank i counts only for pixels whose coarse bucket holds i).
template <int EDGE, int MODE>
__device__ __forceinline__ uint32_t col_band(const uint32_t *cnt, uint32_t *acc, uint32_t gap, int c, int y0) {
    constexpr uint32_t M = 0x00ff00ffu;
    constexpr uint32_t K = (0x8000u - MGE) * 0x00010001u;
    uint32_t ae = K, ao = K, any = 0;
#pragma unroll
    for (int j = -MR; j <= MR; ++j) {
        const uint32_t w = cnt[(EDGE ? clampi(y0 + j, 0, 255) : y0 + j) * WP + c];
        ae += w & M;
        ao += (w >> 8) & M;
    }
    const uint32_t *pn = cnt + (y0 + MR + 1) * WP + c;
    const uint32_t *po = cnt + (y0 - MR) * WP + c;
    uint32_t *pa = acc + y0 * WP + c;
#pragma unroll 8
    for (int y = 0; y < 32; ++y) {
        uint32_t bits = ((ae >> 15) & 0x00010001u) | ((ao >> 7) & 0x01000100u);
        if (MODE == 0) {
            pa[y * WP] += bits * gap;
        } else if (MODE == 1) {
            pa[y * WP] += bits;
        } else {
            const uint32_t a = pa[y * WP];
            bits &= ((gap - a) >> 7) & 0x01010101u;  // 0x80 + i - acc: bit 7 <=> acc <= i (both < 128)
            pa[y * WP] = a + bits;
        }
        any |= bits;
        uint32_t n, o;
        if (EDGE == 0) {
            n = pn[y * WP];
            o = po[y * WP];
        } else {
            n = cnt[min(y0 + y + MR + 1, 255) * WP + c];
            o = cnt[max(y0 + y - MR, 0) * WP + c];
        }
        // per byte 128 + n - o in [107, 149]: no borrow; the 128 bias is removed per lane
        const uint32_t df = (n | 0x80808080u) - o;
        ae += even16(df) - 0x00800080u;
        ao += odd16(df) - 0x00800080u;
    }
    return any;
}

// value-mode column pass with the band's 32 median words in registers (one-level loop)
template <int EDGE>
__device__ __forceinline__ uint32_t col_band_reg(const uint32_t *cnt, uint32_t (&ra)[32], uint32_t gap, int c, int y0) {
    constexpr uint32_t M = 0x00ff00ffu;
    constexpr uint32_t K = (0x8000u - MGE) * 0x00010001u;
    uint32_t ae = K, ao = K, any = 0;
#pragma unroll
    for (int j = -MR; j <= MR; ++j) {
        const uint32_t w = cnt[(EDGE ? clampi(y0 + j, 0, 255) : y0 + j) * WP + c];
        ae += w & M;
        ao += (w >> 8) & M;
    }
    const uint32_t *pn = cnt + (y0 + MR + 1) * WP + c;
    const uint32_t *po = cnt + (y0 - MR) * WP + c;
#pragma unroll
    for (int y = 0; y < 32; ++y) {
        const uint32_t bits = ((ae >> 15) & 0x00010001u) | ((ao >> 7) & 0x01000100u);
        ra[y] += bits * gap;
        any |= bits;
        if (y == 31) break;
        uint32_t n, o;
        if (EDGE == 0) {
            n = pn[y * WP];
            o = po[y * WP];
        } else {
            n = cnt[min(y0 + y + MR + 1, 255) * WP + c];
            o = cnt[max(y0 + y - MR, 0) * WP + c];
        }
        const uint32_t df = (n | 0x80808080u) - o;
        ae += even16(df) - 0x00800080u;
        ao += odd16(df) - 0x00800080u;
    }
    return any;
}

template <int MODE>
__device__ __forceinline__ uint32_t col_pass(const uint32_t *tmp, uint32_t *acc, uint32_t arg, int c, int band) {
    return band == 0 ? col_band<1, MODE>(tmp, acc, arg, c, 0)
                     : (band == 7 ? col_band<2, MODE>(tmp, acc, arg, c, 224) : col_band<0, MODE>(tmp, acc, arg, c, band * 32));
}

// 21 x 21 median of src (kernels.py:42-46) into the plane acc ("col" map).  The value set
// must already be flagged in s.flags (dilate7 does that).  tmp is scratch; src is clobbered.
//
// Rank mode (<= 128 distinct values; src rewritten as 0x80 | rank): the median's rank R(p) =
// #{i : median > s_i} accumulates in acc, coarse-to-fine:
//   1. coarse passes at ranks CG*k + CG-1 give the bucket K(p) = floor(R / CG) of every pixel; a
//      (32-row x 128-px) block whose pixels all stopped is skipped from then on (counts are
//      monotone in the threshold), and the loop ends when no block is active;
//   2. acc becomes CG*K; each block then runs only the fine ranks of the buckets its pixels
//      occupy ([Kmin, Kmax] of the block), adding a pass's bit only where acc <= i (pixels of
//      higher buckets have bit 1 there and are already counted by CG*K);
//   3. median = s_R through a byte LUT.
// A row-pass warp runs only when one of the blocks it feeds (+-10 rows) runs the pass.
// Value mode (> 128 distinct values): one pass per distinct value, acc += gap.
#ifndef ICE_AL_CG
#define ICE_AL_CG 8
#endif
constexpr int CG = ICE_AL_CG;  // coarse group (ranks per bucket)
#ifndef ICE_AL_COARSE_V
#define ICE_AL_COARSE_V false
#endif
#ifndef ICE_AL_COARSE_C
#define ICE_AL_COARSE_C true
#endif

// `need`: 16-bit block mask; blocks outside it start inactive and are never computed (their
// acc words are left unspecified) -- the channel repair reads bg_c only at masked pixels.
__device__ void median21(uint32_t *src, uint32_t *tmp, uint32_t *acc, SmemF &s, bool coarse,
                         uint32_t need = 0xffffu) {
    const int nd = collect_values(s);
#ifdef ICE_AL_PROF
    if (threadIdx.x == 0) atomicAdd(&g_al_prof[8], (unsigned long long)nd);
#endif
    const int c = threadIdx.x & 63, band = threadIdx.x >> 6, lane = threadIdx.x & 31;
    const int rwarp = (threadIdx.x & 255) >> 5, rhalf = threadIdx.x >> 8;  // row map: rows 32 rwarp..
    const int blk = 2 * band + (c >> 5);
    const bool rank_mode = nd <= 128;
    const bool two_level = rank_mode && coarse;
    const uint32_t v0 = two_level ? 0u : s.vals[0] * 0x01010101u;
    for (int y = band * 32; y < band * 32 + 32; ++y) acc[y * WP + c] = v0;
    if (threadIdx.x < 16) s.act[threadIdx.x] = (need >> threadIdx.x) & 1;
    // 16-bit block mask (bit 2*band + half) -> does this row-pass warp feed an active block?
    const uint32_t feed = (1u << (2 * rwarp + rhalf)) | (rwarp > 0 ? 1u << (2 * (rwarp - 1) + rhalf) : 0u) |
                          (rwarp < 7 ? 1u << (2 * (rwarp + 1) + rhalf) : 0u);
    auto act_mask = [&]() {
        uint32_t m = 0;
#pragma unroll
        for (int b2 = 0; b2 < 16; ++b2) m |= (s.act[b2] ? 1u : 0u) << b2;
        return m;
    };
    if (rank_mode) {  // src plane -> 0x80 | rank (in place; values come back through s.vals)
        for (int i = threadIdx.x; i < 256 * 64; i += NTF) {
            uint32_t *w = src + (i >> 6) * WP + (i & 63);
            const uint32_t v = *w;
            *w = s.rank[v & 255] | (uint32_t)s.rank[(v >> 8) & 255] << 8 | (uint32_t)s.rank[(v >> 16) & 255] << 16 |
                 (uint32_t)s.rank[v >> 24] << 24;
        }
    }
    if (!two_level) {  // one pass per distinct value, acc += value gap, block skipping
        uint32_t ra[32];  // this thread's 32 median words ("col" map), in registers
#pragma unroll
        for (int y = 0; y < 32; ++y) ra[y] = v0;
        uint32_t any = 1;
        for (int i = 0; i + 1 < nd; ++i) {
            const uint32_t t = s.vals[i], gap = (uint32_t)s.vals[i + 1] - t;
            if (!__syncthreads_or(any)) break;  // no pixel moved in the previous pass: all final
            if (s.act[2 * rwarp + rhalf] | (rwarp > 0 ? s.act[2 * (rwarp - 1) + rhalf] : 0) |
                (rwarp < 7 ? s.act[2 * (rwarp + 1) + rhalf] : 0)) {
                if (rank_mode) row_counts<true>(src, tmp, (uint32_t)(i + 1) * 0x01010101u);
                else row_counts<false>(src, tmp, (255u - t) * 0x01010101u);
            }
            __syncthreads();
            any = 0;
            if (s.act[blk]) {
                any = band == 0 ? col_band_reg<1>(tmp, ra, gap, c, 0)
                                : (band == 7 ? col_band_reg<2>(tmp, ra, gap, c, 224)
                                             : col_band_reg<0>(tmp, ra, gap, c, band * 32));
                const bool wa = __any_sync(0xffffffffu, any != 0);
                if (lane == 0) s.act[blk] = wa;
            }
        }
#pragma unroll
        for (int y = 0; y < 32; ++y) acc[(band * 32 + y) * WP + c] = ra[y];
        __syncthreads();
        if (threadIdx.x < 256) s.flags[threadIdx.x] = 0;
        return;
    }
    const int cg = CG;
    // 1. coarse passes
    uint32_t any = 1;
    for (int i = cg - 1; i + 1 < nd; i += cg) {
        if (!__syncthreads_or(any)) break;
        if (act_mask() & feed) row_counts<true>(src, tmp, (uint32_t)(i + 1) * 0x01010101u);
        __syncthreads();
#ifdef ICE_AL_PROF
        if (threadIdx.x == 0) {
            int na = 0;
            for (int k = 0; k < 16; ++k) na += s.act[k];
            atomicAdd(&g_al_prof[9], 1ull);
            atomicAdd(&g_al_prof[10], (unsigned long long)na);
        }
#endif
        any = 0;
        if (s.act[blk]) {
            any = col_pass<1>(tmp, acc, 1u, c, band);
            const bool wa = __any_sync(0xffffffffu, any != 0);
            if (lane == 0) s.act[blk] = wa;
        }
    }
    __syncthreads();
    // 2. buckets: per-block [Kmin, Kmax], acc = CG*K
    {
        uint32_t mn = 0xffffffffu, mx = 0;
        for (int y = band * 32; y < band * 32 + 32; ++y) {
            const uint32_t a = acc[y * WP + c];
            mn = vmin(mn, a);
            mx = vmax(mx, a);
            acc[y * WP + c] = a * (uint32_t)CG;  // per byte CG*K <= nd - 1 < 128: no carry
        }
        int kmn = min(min(mn & 255, (mn >> 8) & 255), min((mn >> 16) & 255, mn >> 24));
        int kmx = max(max(mx & 255, (mx >> 8) & 255), max((mx >> 16) & 255, mx >> 24));
        for (int o = 16; o; o >>= 1) {
            kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, o));
            kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, o));
        }
        if (lane == 0) {
            s.kmin[blk] = kmn;
            s.kmax[blk] = kmx;
        }
    }
    __syncthreads();
    uint32_t span = 0, top = 0;  // blocks whose bucket range holds k / whose top bucket is k
    for (int i = 0; i + 1 < nd; ++i) {
        if (i % cg == cg - 1) continue;  // coarse rank: counted
        const int k = i / cg;
        if (i % cg == 0) {  // new bucket: static masks, clear the done set (rare: <= nd / CG times)
            span = 0;
            top = 0;
#pragma unroll
            for (int b2 = 0; b2 < 16; ++b2) {
                span |= (s.kmin[b2] <= k && k <= s.kmax[b2] && (need >> b2 & 1) ? 1u : 0u) << b2;
                top |= (s.kmax[b2] == k ? 1u : 0u) << b2;
            }
            __syncthreads();
            if (threadIdx.x == 0) s.done_bits = 0;
            __syncthreads();
        }
        const uint32_t need = span & ~s.done_bits;
        if (!need) continue;  // block-uniform
        if (need & feed) row_counts<true>(src, tmp, (uint32_t)(i + 1) * 0x01010101u);
        __syncthreads();
#ifdef ICE_AL_PROF
        if (threadIdx.x == 0) {
            atomicAdd(&g_al_prof[9], 1ull);
            atomicAdd(&g_al_prof[10], (unsigned long long)__popc(need));
        }
#endif
        if ((need >> blk) & 1) {
            // the block's top bucket holds no higher-bucket pixels: no mask needed
            const uint32_t moved = ((top >> blk) & 1) ? col_pass<1>(tmp, acc, 1u, c, band)
                                                      : col_pass<2>(tmp, acc, (uint32_t)(i | 0x80) * 0x01010101u, c, band);
            // bucket k of this block is final once no pixel of it still moves
            if (!__any_sync(0xffffffffu, moved != 0) && lane == 0) atomicOr(&s.done_bits, 1u << blk);
        }
        __syncthreads();
    }
    // 3. rank -> value
    for (int y = band * 32; y < band * 32 + 32; ++y) {
        const uint32_t r = acc[y * WP + c];
        acc[y * WP + c] = s.vals[r & 255] | (uint32_t)s.vals[(r >> 8) & 255] << 8 |
                          (uint32_t)s.vals[(r >> 16) & 255] << 16 | (uint32_t)s.vals[r >> 24] << 24;
    }
    __syncthreads();
    if (threadIdx.x < 256) s.flags[threadIdx.x] = 0;  // ready for the next median
}

// ---- 3 x 3 median (noise_median_k = 3) of src into dst, "col" map ----------------------
// In 16-bit lanes (native VIMNMX.U16x2): E = even pixels (bytes 0, 2), O = odd (bytes 1, 3).
// Even pixel 4c+2i has neighbours O_{c-1}/O_c (funnel) and O_c; odd pixel 4c+2i+1 has E_c
// and E_c/E_{c+1}.  Column-sorted triples give median9 = med3(max of mins, med of mids,
// min of maxes).
__device__ __forceinline__ uint32_t mn2(uint32_t a, uint32_t b) { return __vminu2(a, b); }
__device__ __forceinline__ uint32_t mx2(uint32_t a, uint32_t b) { return __vmaxu2(a, b); }
__device__ __forceinline__ void sort3_2(uint32_t a, uint32_t b, uint32_t c, uint32_t &lo, uint32_t &md,
                                        uint32_t &hi) {
    const uint32_t l1 = mn2(a, b), h1 = mx2(a, b);
    lo = mn2(l1, c);
    const uint32_t m2 = mx2(l1, c);
    md = mn2(h1, m2);
    hi = mx2(h1, m2);
}
__device__ __forceinline__ uint32_t med3_2(uint32_t a, uint32_t b, uint32_t c) {
    return mx2(mn2(a, b), mn2(mx2(a, b), c));
}

__device__ void median3_plane(const uint32_t *src, uint32_t *dst) {
    const int c = threadIdx.x & 63, y0 = (threadIdx.x >> 6) * 32;
    // per row: Ol = odd half of the left word, E/O of the own word, Er = even half of the right
    auto ld = [&](int y, uint32_t &ol, uint32_t &e, uint32_t &o, uint32_t &er) {
        const uint32_t *row = src + clampi(y, 0, 255) * WP;
        const uint32_t m = row[c];
        const uint32_t l = c > 0 ? row[c - 1] : rep0(m);
        const uint32_t r = c < 63 ? row[c + 1] : rep3(m);
        ol = odd16(l);
        e = even16(m);
        o = odd16(m);
        er = even16(r);
    };
    uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
    ld(y0 - 1, a0, a1, a2, a3);
    ld(y0, b0, b1, b2, b3);
#pragma unroll 2
    for (int y = y0; y < y0 + 32; ++y) {
        uint32_t c0, c1, c2, c3;
        ld(y + 1, c0, c1, c2, c3);
        uint32_t olL, olM, olH, eL, eM, eH, oL, oM, oH, erL, erM, erH;
        sort3_2(a0, b0, c0, olL, olM, olH);
        sort3_2(a1, b1, c1, eL, eM, eH);
        sort3_2(a2, b2, c2, oL, oM, oH);
        sort3_2(a3, b3, c3, erL, erM, erH);
        // even pixels: left = fsl(Ol, O, 16), centre = E, right = O
        const uint32_t ev = med3_2(mx2(mx2(fsl(olL, oL, 16), eL), oL), med3_2(fsl(olM, oM, 16), eM, oM),
                                   mn2(mn2(fsl(olH, oH, 16), eH), oH));
        // odd pixels: left = E, centre = O, right = fsr(E, Er, 16)
        const uint32_t od = med3_2(mx2(mx2(eL, oL), fsr(eL, erL, 16)), med3_2(eM, oM, fsr(eM, erM, 16)),
                                   mn2(mn2(eH, oH), fsr(eH, erH, 16)));
        dst[y * WP + c] = ev | (od << 8);
        a0 = b0; a1 = b1; a2 = b2; a3 = b3;
        b0 = c0; b1 = c1; b2 = c2; b3 = c3;
    }
}

// ---- sub-histograms: 64 copies (one per 8 lanes), stride 257 words (bank-spread) ------------
constexpr int SH = 64, SHS = 257;  // 64 x 257 words = 65,792 B <= one plane
__device__ __forceinline__ void subhist_zero(uint32_t *sh) {
    for (int i = threadIdx.x; i < SH * SHS; i += NTF) sh[i] = 0;
}
__device__ __forceinline__ void subhist_add4(uint32_t *sh, uint32_t w) {
    uint32_t *h = sh + (threadIdx.x >> 3) * SHS;
    atomicAdd(h + (w & 255), 1u);
    atomicAdd(h + ((w >> 8) & 255), 1u);
    atomicAdd(h + ((w >> 16) & 255), 1u);
    atomicAdd(h + (w >> 24), 1u);
}
__device__ __forceinline__ void subhist_reduce(const uint32_t *sh, uint32_t *hist) {
    // 512 threads: bin = tid & 255, half the copies each
    const int v = threadIdx.x & 255, h0 = (threadIdx.x >> 8) * (SH / 2);
    uint32_t t = 0;
#pragma unroll 8
    for (int k = 0; k < SH / 2; ++k) t += sh[(h0 + k) * SHS + v];
    if (threadIdx.x >= 256) hist[v] = t;
    __syncthreads();
    if (threadIdx.x < 256) hist[v] += t;
}

// RGB (16 px in 3 uint4) -> 4 words of R, G, B (pixels 4q .. 4q+3)
__device__ __forceinline__ void unpack16(const uint4 &a, const uint4 &b, const uint4 &c, uint32_t (&R)[4],
                                         uint32_t (&G)[4], uint32_t (&B)[4]) {
    const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t x0 = w[3 * q], x1 = w[3 * q + 1], x2 = w[3 * q + 2];
        R[q] = __byte_perm(__byte_perm(x0, x1, 0x0630), x2, 0x5210);
        G[q] = __byte_perm(__byte_perm(x0, x1, 0x0741), x2, 0x6210);
        B[q] = __byte_perm(__byte_perm(x0, x1, 0x0052), x2, 0x7410);
    }
}
__device__ __forceinline__ void pack16(const uint32_t (&R)[4], const uint32_t (&G)[4], const uint32_t (&B)[4],
                                       uint4 &a, uint4 &b, uint4 &c) {
    uint32_t w[12];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        // bytes 12q.. : R0 G0 B0 R1 | G1 B1 R2 G2 | B2 R3 G3 B3
        const uint32_t rg = __byte_perm(R[q], G[q], 0x5140);  // R0 G0 R1 G1
        const uint32_t rg2 = __byte_perm(R[q], G[q], 0x7362);  // R2 G2 R3 G3
        w[3 * q] = __byte_perm(rg, B[q], 0x2410);             // R0 G0 B0 R1
        w[3 * q + 1] = __byte_perm(__byte_perm(rg, B[q], 0x0053), rg2, 0x5410);  // G1 B1 R2 G2
        w[3 * q + 2] = __byte_perm(B[q], rg2, 0x3762);                          // B2 R3 G3 B3
    }
    a = make_uint4(w[0], w[1], w[2], w[3]);
    b = make_uint4(w[4], w[5], w[6], w[7]);
    c = make_uint4(w[8], w[9], w[10], w[11]);
}

// V = max(r, g, b) (cloudfilter.py:89) or one channel of the tile into a plane ("group" map);
// returns whether any pixel has unequal channels
// rstride: bytes between the rows of the 256 x 256 window (768: a contiguous tile; 3 w: a
// window of a w-wide image, 16-B aligned rows)
__device__ int load_plane(const uint8_t *tile, int ch, uint32_t *dst, uint32_t *sh = nullptr, int rstride = 768) {
    int uneq = 0;
    for (int g = threadIdx.x; g < 4096; g += NTF) {
        const uint4 *t4 = reinterpret_cast<const uint4 *>(tile + (size_t)(g >> 4) * rstride) + 3 * (g & 15);
        const uint4 a = __ldg(t4), b = __ldg(t4 + 1), c = __ldg(t4 + 2);
        uint32_t R[4], G[4], B[4];
        unpack16(a, b, c, R, G, B);
        uint32_t *d = dst + (g >> 4) * WP + 4 * (g & 15);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            d[q] = ch == 3 ? vmax3(R[q], G[q], B[q]) : (ch == 0 ? R[q] : (ch == 1 ? G[q] : B[q]));
            if (sh) subhist_add4(sh, d[q]);
            uneq |= (R[q] ^ G[q]) | (G[q] ^ B[q]);
        }
    }
    return uneq != 0;
}

__device__ __forceinline__ int block_sum_f(int v, SmemF &s) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s.red[threadIdx.x >> 5][0] = v;
    __syncthreads();
    int t = 0;
    for (int i = 0; i < NTF / 32; ++i) t += s.red[i][0];
    return t;
}

__device__ __forceinline__ void prefetch_tile_l2(const uint8_t *tile) {
    // 196,608 B = 12 x 16 KB bulk L2 prefetches
    if (threadIdx.x < 12)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(tile + threadIdx.x * 16384), "r"(16384)
                     : "memory");
}

__device__ __forceinline__ void process_tile256(const uint8_t *__restrict__ rgb, const Params &prm,
                                                uint8_t *__restrict__ filtered, uint8_t *__restrict__ label,
                                                uint8_t *__restrict__ maskout, uint32_t *__restrict__ affected,
                                                uint32_t *__restrict__ counts, int32_t *__restrict__ unmatched,
                                                SmemF &s, const size_t tile_id) {
    const IceFilterCfg &cfg = prm.cfg;
    constexpr int NPX = 65536;
    const uint8_t *tile = rgb + tile_id * (size_t)NPX * 3;
    uint8_t *ftile = filtered + tile_id * (size_t)NPX * 3;
    uint32_t *P0 = s.p[0], *P1 = s.p[1], *P2 = s.p[2];
    const int cc = threadIdx.x & 63, y0 = (threadIdx.x >> 6) * 32;  // "col" map
#ifdef ICE_AL_PROF
    long long prof_t0 = clock64();
#endif
    if (threadIdx.x < 256) {
        s.flags[threadIdx.x] = 0;
        s.hist[threadIdx.x] = 0;
        s.hist2[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) s.need_bits = 0;
    subhist_zero(P2);
    __syncthreads();
    // 1. V plane (cloudfilter.py:89) + its histogram, D = dilate7(V) (cloudfilter.py:84)
    const int any_unequal = __syncthreads_or(load_plane(tile, 3, P0, P2));
    subhist_reduce(P2, s.hist_v);
    PROF_MARK(0);
    dilate7(P0, P1, P2, s);  // D in P2 (its column pass starts after a barrier: P2 reads done)
    PROF_MARK(1);
    // 2. bg = median21(D) (estimate_background, cloudfilter.py:82-84) into P1
    median21(P2, P0, P1, s, ICE_AL_COARSE_V);
    PROF_MARK(2);
    // 3. smooth = median3(V) (:90), d = |smooth - bg| [truncated] (:91-93) into P2, histogram
    load_plane(tile, 3, P0);  // V again (L2-resident re-read)
    __syncthreads();
    median3_plane(P0, P2);
    __syncthreads();
    subhist_zero(P0);
    __syncthreads();
    const uint32_t tt4 = (uint32_t)cfg.truncate_t * 0x01010101u;
#pragma unroll 4
    for (int y = 0; y < 32; ++y) {
        const int o = (y0 + y) * WP + cc;
        uint32_t d = __vabsdiffu4(P2[o], P1[o]);
        if (cfg.diff_truncate) d = vmin(d, tt4);
        P2[o] = d;
        subhist_add4(P0, d);
    }
    __syncthreads();
    subhist_reduce(P0, s.hist);
    __syncthreads();
    if (threadIdx.x < 32) {  // lo / hi of d from the histogram
        const int lane = threadIdx.x;
        uint32_t nz = 0;
        for (int j = 0; j < 8; ++j) nz |= (s.hist[8 * lane + j] != 0) << j;
        const unsigned have = __ballot_sync(0xffffffffu, nz != 0);
        const int wlo = __ffs(have) - 1, whi = 31 - __clz(have);
        const uint32_t nlo = __shfl_sync(0xffffffffu, nz, wlo), nhi = __shfl_sync(0xffffffffu, nz, whi);
        if (lane == 0) {
            s.bc[2] = 8 * wlo + __ffs(nlo) - 1;
            s.bc[3] = 8 * whi + 31 - __clz(nhi);
        }
    }
    __syncthreads();
    const int lo = s.bc[2], hi = s.bc[3];
    const int range = hi - lo;
    PROF_MARK(3);
    // 4. minmax normalize (kernels.py:66-74, exact integer form) applied to the histogram
    //    bins, Otsu / fixed threshold (:77-116) -> mask = normalized > thr = d > dthr
    if (threadIdx.x < 256) {
        const int v = threadIdx.x;
        const uint32_t h = s.hist[v];
        if (h) atomicAdd(&s.hist2[range == 0 ? 0 : (510 * (v - lo) + range) / (2 * range)], h);
    }
    if (threadIdx.x == 0) s.bc[1] = -1;
    __syncthreads();
    if (threadIdx.x < 32) {
        const int t = cfg.mask_mode_fixed ? cfg.fixed_t : otsu_from_hist(s.hist2);
        if (threadIdx.x == 0) s.bc[0] = t;
    }
    __syncthreads();
    const int thr = s.bc[0];
    if (threadIdx.x < 256) {
        const int v = threadIdx.x;
        if (v >= lo && v <= hi) {
            const int dn = range == 0 ? 0 : (510 * (v - lo) + range) / (2 * range);
            if (dn <= thr) atomicMax(&s.bc[1], v);
        }
    }
    __syncthreads();
    const int dthr = s.bc[1] < lo ? lo - 1 : s.bc[1];  // masked <=> d > dthr
    int mcnt = (threadIdx.x < 256 && (int)threadIdx.x > dthr) ? (int)s.hist[threadIdx.x] : 0;
    const int masked = block_sum_f(mcnt, s);
    const bool all_masked = dthr < 0;
    const uint32_t mc4 = (uint32_t)(255 - max(dthr, 0)) * 0x01010101u;
    PROF_MARK(4);
    // 5. repair (cloudfilter.py:108-116)
    int center = 0;
    if (masked > 0) {
        if (!any_unequal) {
            // R == G == B everywhere: every channel equals V, bg_c == bg(V) (kept in P1)
            center = center_from_hist(s.hist_v, NPX);
        } else {
            // mask bits, then per channel: bg_c = median21(dilate7(c)), masked pixels repaired
            for (int w = threadIdx.x; w < 2048; w += NTF) {
                uint32_t bits = 0;
                const int y = w >> 3, x0 = (w & 7) * 32;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t dw = P2[y * WP + (x0 >> 2) + q];
                    const uint32_t g = all_masked ? 0x01010101u : gt4(dw, mc4, mc4 & 0x7f7f7f7fu);
                    bits |= ((g & 1) | ((g >> 7) & 2) | ((g >> 14) & 4) | ((g >> 21) & 8)) << (4 * q);
                }
                s.maskbits[w] = bits;
                if (bits) atomicOr(&s.need_bits, 1u << (2 * (y >> 5) + ((w & 7) >> 2)));
            }
            __syncthreads();
            const uint32_t need = s.need_bits;
            for (int ch = 0; ch < 3; ++ch) {
                subhist_zero(P2);
                __syncthreads();
                load_plane(tile, ch, P0, P2);  // + its histogram in 64 bank-spread copies (P2)
                __syncthreads();
                subhist_reduce(P2, s.hist);
                __syncthreads();
                const int c_ch = center_from_hist(s.hist, NPX);
                dilate7(P0, P1, P2, s);
                median21(P2, P0, P1, s, ICE_AL_COARSE_C, need);  // bg_c in P1 (blocks in need)
                load_plane(tile, ch, P0);  // the channel again (L2-resident re-read)
                __syncthreads();
#pragma unroll 2
                for (int y = 0; y < 32; ++y) {
                    const int yy = y0 + y;
                    const uint32_t mb = (s.maskbits[yy * 8 + (cc >> 3)] >> (4 * (cc & 7))) & 15;
                    if (mb) {
                        const uint32_t chw = P0[yy * WP + cc], bgw = P1[yy * WP + cc];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            if (mb >> k & 1) {
                                const int i = yy * 256 + 4 * cc + k;
                                const int f = (int)((chw >> (8 * k)) & 255) - (int)((bgw >> (8 * k)) & 255) + c_ch;
                                ftile[3 * i + ch] = (uint8_t)clampi(f, 0, 255);
                            }
                        }
                    }
                }
                __syncthreads();
            }
        }
    }
    PROF_MARK(5);
    // 6. output pass: filtered tile, mask, HSV segmentation, counts, first unmatched
    int c0 = 0, c1 = 0, c2 = 0, first = 0x7fffffff;
    uint8_t *ltile = label + tile_id * (size_t)NPX;
    uint8_t *mtile = maskout ? maskout + tile_id * (size_t)NPX : nullptr;
    const SchemeR scr(prm.scheme);
    const uint4 *t4 = reinterpret_cast<const uint4 *>(tile);
    uint4 *f4 = reinterpret_cast<uint4 *>(ftile);
    for (int g = threadIdx.x; g < 4096; g += NTF) {
        const uint4 a = __ldg(t4 + 3 * g), b = __ldg(t4 + 3 * g + 1), c = __ldg(t4 + 3 * g + 2);
        uint32_t R[4], G[4], B[4];
        unpack16(a, b, c, R, G, B);
        const int prow = (g >> 4) * WP + 4 * (g & 15);
        uint32_t mk[4];
        if (masked == 0) {
            mk[0] = mk[1] = mk[2] = mk[3] = 0;
        } else if (any_unequal) {  // P2 was reused by the per-channel repair: mask bits
            const uint32_t bits16 = s.maskbits[g >> 1] >> (16 * (g & 1));
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t n = bits16 >> (4 * q);
                mk[q] = (n & 1) | ((n & 2) << 7) | ((n & 4) << 14) | ((n & 8) << 21);
            }
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) mk[q] = all_masked ? 0x01010101u : gt4(P2[prow + q], mc4, mc4 & 0x7f7f7f7fu);
        }
        if ((mk[0] | mk[1] | mk[2] | mk[3]) != 0) {
            if (!any_unequal) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t bgw = P1[prow + q];
                    uint32_t f = 0;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int x = (R[q] >> (8 * k)) & 255;
                        const int v = clampi(x - (int)((bgw >> (8 * k)) & 255) + center, 0, 255);
                        f |= (uint32_t)((mk[q] >> (8 * k) & 1) ? v : x) << (8 * k);
                    }
                    R[q] = G[q] = B[q] = f;
                }
            } else {
                // repaired channel bytes were written to ftile by step 5 (same CTA, after a barrier)
                const uint4 *fsrc = reinterpret_cast<const uint4 *>(ftile);
                uint32_t FR[4], FG[4], FB[4];
                unpack16(fsrc[3 * g], fsrc[3 * g + 1], fsrc[3 * g + 2], FR, FG, FB);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t sel = mk[q] * 255u;  // 0xff per masked byte
                    R[q] = (FR[q] & sel) | (R[q] & ~sel);
                    G[q] = (FG[q] & sel) | (G[q] & ~sel);
                    B[q] = (FB[q] & sel) | (B[q] & ~sel);
                }
            }
        }
        uint4 fa, fb, fc;
        pack16(R, G, B, fa, fb, fc);
        f4[3 * g] = fa;
        f4[3 * g + 1] = fb;
        f4[3 * g + 2] = fc;
        if (mtile)
            reinterpret_cast<uint4 *>(mtile)[g] = make_uint4(mk[0] * 255u, mk[1] * 255u, mk[2] * 255u, mk[3] * 255u);
        uint32_t lw[4];
        if (prm.v_only) {
            uint32_t sum = 0, e[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t v = vmax3(R[q], G[q], B[q]);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    e[4 * q + k] = s.vlut[(v >> (8 * k)) & 255];
                    sum += e[4 * q + k];
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                lw[q] = __byte_perm(__byte_perm(e[4 * q], e[4 * q + 1], 0x0040),
                                    __byte_perm(e[4 * q + 2], e[4 * q + 3], 0x0040), 0x5410);
            c0 += (sum >> 12) & 31;
            c1 += (sum >> 17) & 31;
            c2 += (sum >> 22) & 31;
            if (sum >> 27) {
#pragma unroll
                for (int k = 15; k >= 0; --k)
                    if ((e[k] & 255) == 255) first = min(first, 16 * g + k);
            }
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                lw[q] = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int cls = classify((R[q] >> (8 * k)) & 255, (G[q] >> (8 * k)) & 255,
                                             (B[q] >> (8 * k)) & 255, scr);
                    lw[q] |= (uint32_t)cls << (8 * k);
                    c0 += cls == 0;
                    c1 += cls == 1;
                    c2 += cls == 2;
                    if (cls == 255) first = min(first, 16 * g + 4 * q + k);
                }
            }
        }
        reinterpret_cast<uint4 *>(ltile)[g] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
    PROF_MARK(6);
    for (int o = 16; o; o >>= 1) {
        c0 += __shfl_xor_sync(0xffffffffu, c0, o);
        c1 += __shfl_xor_sync(0xffffffffu, c1, o);
        c2 += __shfl_xor_sync(0xffffffffu, c2, o);
        first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        const int wi = threadIdx.x >> 5;
        s.red[wi][0] = c0; s.red[wi][1] = c1; s.red[wi][2] = c2; s.red[wi][3] = first;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < NTF / 32; ++i) {
            c0 += s.red[i][0]; c1 += s.red[i][1]; c2 += s.red[i][2]; first = min(first, s.red[i][3]);
        }
        affected[tile_id] = (uint32_t)masked;
        counts[3 * tile_id] = c0;
        counts[3 * tile_id + 1] = c1;
        counts[3 * tile_id + 2] = c2;
        unmatched[tile_id] = first == 0x7fffffff ? -1 : first;
    }
    __syncthreads();  // shared state is reused by the next tile
}

// One CTA per tile (the hardware scheduler balances hazy / clean tiles); each CTA prefetches
// into L2 the RGB of the tile one "wave" ahead (blockIdx.x + ahead), which runs about one
// tile-time later on some SM, so its loads hit L2.
__global__ void __launch_bounds__(NTF, 1)
autolabel256_kernel(const uint8_t *__restrict__ rgb, int n, int ahead, Params prm, uint8_t *__restrict__ filtered,
                    uint8_t *__restrict__ label, uint8_t *__restrict__ maskout, uint32_t *__restrict__ affected,
                    uint32_t *__restrict__ counts, int32_t *__restrict__ unmatched) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    SmemF &s = *reinterpret_cast<SmemF *>(smem_raw);
    if (threadIdx.x < 256 && prm.v_only) {
        int cls = 255;
        const int v = threadIdx.x;
        for (int k = 2; k >= 0; --k)
            if (v >= prm.scheme.lo[k][2] && v <= prm.scheme.hi[k][2]) cls = prm.scheme.cls[k];
        const int slot = cls == 255 ? 3 : cls;
        s.vlut[v] = (uint32_t)cls | (1u << (12 + 5 * slot));
    }
    const int t = blockIdx.x;
    if (t < ahead) prefetch_tile_l2(rgb + (size_t)t * 65536 * 3);
    if (t + ahead < n) prefetch_tile_l2(rgb + (size_t)(t + ahead) * 65536 * 3);
    process_tile256(rgb, prm, filtered, label, maskout, affected, counts, unmatched, s, (size_t)t);
}


// =====================================================================================
// SWAR region path: the 256 x 256 SWAR pipeline on 256 x 256 WINDOWS of a larger image
// (whole scenes, 512^2 tiles) with the default windows.  h, w >= 256, w % 16 == 0.  The image
// is cut into cores (<= 230 rows, <= 224 columns, column starts at multiples of 16); each
// core's window is the 256 x 256 block that holds the core plus its 13-pixel halo, shifted
// inside the image at the borders (so window borders that are image borders replicate, as
// cv2 does, and interior window borders lie >= 13 pixels from the core).  Window rows are
// 16-B aligned (column origin a multiple of 16), so the SWAR loads / stores apply unchanged.
// Pass 1 (region256_d_kernel) writes the core's d and background-of-V bytes to scratch
// planes and adds the core's d / channel histograms to the image's counters; the
// image-global statistics come from region_stats_kernel; pass 2 (region256_out_kernel)
// masks the core, recomputes channel backgrounds only when the window is not gray and the
// core holds masked pixels (blocks without masked pixels skipped), and writes filtered /
// mask / label for the core.
struct R256 {
    int h, w, ny, nx, cs_y, cs_x;
};
struct R256Box {
    int cy0, ch, cx0, cw, ry0, rx0;
};
__device__ __forceinline__ R256Box r256_box(const R256 &g, int r) {
    R256Box b;
    const int by = r / g.nx, bx = r - by * g.nx;
    b.cy0 = by * g.cs_y;
    b.ch = min(g.cs_y, g.h - b.cy0);
    b.cx0 = bx * g.cs_x;
    b.cw = min(g.cs_x, g.w - b.cx0);
    b.ry0 = min(max(b.cy0 - MR - 3, 0), g.h - 256);
    b.rx0 = min(max(b.cx0 - 16, 0), g.w - 256);
    return b;
}

__global__ void __launch_bounds__(NTF, 1)
region256_d_kernel(const uint8_t *__restrict__ rgb, R256 g, IceFilterCfg cfg, int regions,
                   uint8_t *__restrict__ dplanes, uint8_t *__restrict__ bgplanes, RegionStats *__restrict__ st) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    SmemF &s = *reinterpret_cast<SmemF *>(smem_raw);
    const int img = blockIdx.x / regions;
    const R256Box b = r256_box(g, blockIdx.x - img * regions);
    const size_t npx = (size_t)g.h * g.w;
    const uint8_t *im = rgb + img * npx * 3;
    const uint8_t *win = im + ((size_t)b.ry0 * g.w + b.rx0) * 3;
    const int rs = 3 * g.w;
    RegionStats &S = st[img];
    uint32_t *P0 = s.p[0], *P1 = s.p[1], *P2 = s.p[2];
    const int cc = threadIdx.x & 63, y0 = (threadIdx.x >> 6) * 32;  // "col" map
    if (threadIdx.x < 256) s.flags[threadIdx.x] = 0;
    __syncthreads();
    load_plane(win, 3, P0, nullptr, rs);  // V (cloudfilter.py:89)
    __syncthreads();
    dilate7(P0, P1, P2, s);  // D in P2
    median21(P2, P0, P1, s, ICE_AL_COARSE_V);  // background of V in P1
    load_plane(win, 3, P0, nullptr, rs);
    __syncthreads();
    median3_plane(P0, P2);  // smooth in P2
    __syncthreads();
    subhist_zero(P0);
    __syncthreads();
    // the core's d (and bg) words -> scratch planes; d histogram over the core
    const int oy = b.cy0 - b.ry0, ox4 = (b.cx0 - b.rx0) >> 2, cw4 = b.cw >> 2;
    const uint32_t tt4 = (uint32_t)cfg.truncate_t * 0x01010101u;
    uint32_t *dpl = reinterpret_cast<uint32_t *>(dplanes + img * npx);
    uint32_t *bpl = reinterpret_cast<uint32_t *>(bgplanes + img * npx);
    const bool col_in = cc >= ox4 && cc < ox4 + cw4;
#pragma unroll 4
    for (int y = 0; y < 32; ++y) {
        const int r = y0 + y;
        if (!col_in || r < oy || r >= oy + b.ch) continue;
        const int o = r * WP + cc;
        uint32_t d = __vabsdiffu4(P2[o], P1[o]);
        if (cfg.diff_truncate) d = vmin(d, tt4);
        const size_t gw = (((size_t)(b.ry0 + r) * g.w + b.rx0) >> 2) + cc;
        dpl[gw] = d;
        bpl[gw] = P1[o];
        subhist_add4(P0, d);
    }
    __syncthreads();
    subhist_reduce(P0, s.hist);
    __syncthreads();
    if (threadIdx.x < 256 && s.hist[threadIdx.x]) atomicAdd(&S.hist_d[threadIdx.x], s.hist[threadIdx.x]);
    __syncthreads();
    // channel histograms of the core (for the channel medians of the repair)
    subhist_zero(P0);
    subhist_zero(P1);
    subhist_zero(P2);
    __syncthreads();
    const int cg = b.cw >> 4, ng = b.ch * cg;
    for (int q = threadIdx.x; q < ng; q += NTF) {
        const int r = q / cg, k = q - r * cg;
        const uint4 *t4 = reinterpret_cast<const uint4 *>(im + ((size_t)(b.cy0 + r) * g.w + b.cx0 + 16 * k) * 3);
        uint32_t R[4], G[4], B[4];
        unpack16(__ldg(t4), __ldg(t4 + 1), __ldg(t4 + 2), R, G, B);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            subhist_add4(P0, R[e]);
            subhist_add4(P1, G[e]);
            subhist_add4(P2, B[e]);
        }
    }
    __syncthreads();
#pragma unroll 1
    for (int c = 0; c < 3; ++c) {
        subhist_reduce(s.p[c], s.hist);
        __syncthreads();
        if (threadIdx.x < 256 && s.hist[threadIdx.x]) atomicAdd(&S.hist_c[c][threadIdx.x], s.hist[threadIdx.x]);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(NTF, 1)
region256_out_kernel(const uint8_t *__restrict__ rgb, R256 g, Params prm, int regions,
                     const uint8_t *__restrict__ dplanes, const uint8_t *__restrict__ bgplanes,
                     RegionStats *__restrict__ st, uint8_t *__restrict__ filtered, uint8_t *__restrict__ label,
                     uint8_t *__restrict__ maskout) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    SmemF &s = *reinterpret_cast<SmemF *>(smem_raw);
    if (threadIdx.x < 256 && prm.v_only) {
        int cls = 255;
        const int v = threadIdx.x;
        for (int k = 2; k >= 0; --k)
            if (v >= prm.scheme.lo[k][2] && v <= prm.scheme.hi[k][2]) cls = prm.scheme.cls[k];
        const int slot = cls == 255 ? 3 : cls;
        s.vlut[v] = (uint32_t)cls | (1u << (12 + 5 * slot));
    }
    const int img = blockIdx.x / regions;
    const R256Box b = r256_box(g, blockIdx.x - img * regions);
    const size_t npx = (size_t)g.h * g.w;
    const uint8_t *im = rgb + img * npx * 3;
    const uint8_t *win = im + ((size_t)b.ry0 * g.w + b.rx0) * 3;
    const int rs = 3 * g.w;
    uint8_t *fim = filtered + img * npx * 3;
    const uint32_t *dpl = reinterpret_cast<const uint32_t *>(dplanes + img * npx);
    const uint32_t *bpl = reinterpret_cast<const uint32_t *>(bgplanes + img * npx);
    RegionStats &S = st[img];
    uint32_t *P0 = s.p[0], *P1 = s.p[1], *P2 = s.p[2];
    const int cc = threadIdx.x & 63, y0 = (threadIdx.x >> 6) * 32;
    const int oy = b.cy0 - b.ry0, ox = b.cx0 - b.rx0;
    // masked <=> d > dthr, dthr = the largest d whose stretch is <= thr (kernels.py:66-74, 94-96)
    if (threadIdx.x == 0) {
        int dthr = S.lo - 1;
        for (int v = S.lo; v <= S.lo + S.range; ++v)
            if (stretch(v, S.lo, S.range) <= S.thr) dthr = v;
        s.bc[0] = dthr;
        s.need_bits = 0;
        for (int k = 0; k < 256; ++k) s.flags[k] = 0;
    }
    __syncthreads();
    const int dthr = s.bc[0];
    const bool all_masked = dthr < 0;
    const uint32_t mc4 = (uint32_t)(255 - max(dthr, 0)) * 0x01010101u;
    // mask bits of the window (non-core pixels are never masked here)
    int any = 0;
    for (int w = threadIdx.x; w < 2048; w += NTF) {
        uint32_t bits = 0;
        const int y = w >> 3, x0 = (w & 7) * 32;
        if (S.masked > 0 && y >= oy && y < oy + b.ch) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int x = x0 + 4 * q;
                if (x < ox || x >= ox + b.cw) continue;
                const uint32_t dw = dpl[(((size_t)(b.ry0 + y) * g.w + b.rx0 + x) >> 2)];
                const uint32_t gq = all_masked ? 0x01010101u : gt4(dw, mc4, mc4 & 0x7f7f7f7fu);
                bits |= ((gq & 1) | ((gq >> 7) & 2) | ((gq >> 14) & 4) | ((gq >> 21) & 8)) << (4 * q);
            }
        }
        s.maskbits[w] = bits;
        if (bits) atomicOr(&s.need_bits, 1u << (2 * (y >> 5) + ((w & 7) >> 2)));
        any |= bits != 0;
    }
    const bool repair = __syncthreads_or(any) != 0;
    bool gray = true;
    if (repair) {
        // R == G == B over the window: every channel's background is V's (pass 1's bg plane)
        gray = !__syncthreads_or(load_plane(win, 0, P0, nullptr, rs));
        if (!gray) {
            const uint32_t need = s.need_bits;
            for (int ch = 0; ch < 3; ++ch) {
                load_plane(win, ch, P0, nullptr, rs);
                __syncthreads();
                dilate7(P0, P1, P2, s);
                median21(P2, P0, P1, s, ICE_AL_COARSE_C, need);  // bg_c in P1 (blocks in need)
                load_plane(win, ch, P0, nullptr, rs);
                __syncthreads();
                const int c_ch = S.center[ch];
#pragma unroll 2
                for (int y = 0; y < 32; ++y) {
                    const int yy = y0 + y;
                    const uint32_t mb = (s.maskbits[yy * 8 + (cc >> 3)] >> (4 * (cc & 7))) & 15;
                    if (mb) {
                        const uint32_t chw = P0[yy * WP + cc], bgw = P1[yy * WP + cc];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            if (mb >> k & 1) {
                                const size_t gi = (size_t)(b.ry0 + yy) * g.w + b.rx0 + 4 * cc + k;
                                const int f = (int)((chw >> (8 * k)) & 255) - (int)((bgw >> (8 * k)) & 255) + c_ch;
                                fim[3 * gi + ch] = (uint8_t)clampi(f, 0, 255);
                            }
                        }
                    }
                }
                __syncthreads();
            }
        }
    }
    // output: the core in 16-pixel groups
    int c0 = 0, c1 = 0, c2 = 0, first = 0x7fffffff;
    const SchemeR scr(prm.scheme);
    const int cgw = b.cw >> 4, ng = b.ch * cgw;
    const int cen = S.center[0];
    for (int q = threadIdx.x; q < ng; q += NTF) {
        const int r = q / cgw, k = q - r * cgw;
        const size_t gi = (size_t)(b.cy0 + r) * g.w + b.cx0 + 16 * k;  // first pixel of the group
        const uint4 *t4 = reinterpret_cast<const uint4 *>(im + gi * 3);
        uint32_t R[4], G[4], B[4];
        unpack16(__ldg(t4), __ldg(t4 + 1), __ldg(t4 + 2), R, G, B);
        const int wy = oy + r, wx = ox + 16 * k;
        const uint32_t bits16 = (s.maskbits[wy * 8 + (wx >> 5)] >> (wx & 31)) & 0xffffu;
        uint32_t mk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t n = bits16 >> (4 * e);
            mk[e] = (n & 1) | ((n & 2) << 7) | ((n & 4) << 14) | ((n & 8) << 21);
        }
        if (bits16) {
            if (gray) {
                const uint4 bgv = *reinterpret_cast<const uint4 *>(bpl + (gi >> 2));
                const uint32_t bw[4] = {bgv.x, bgv.y, bgv.z, bgv.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    uint32_t f = 0;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const int x = (R[e] >> (8 * kk)) & 255;
                        const int v = clampi(x - (int)((bw[e] >> (8 * kk)) & 255) + cen, 0, 255);
                        f |= (uint32_t)((mk[e] >> (8 * kk) & 1) ? v : x) << (8 * kk);
                    }
                    R[e] = G[e] = B[e] = f;
                }
            } else {
                const uint4 *f4 = reinterpret_cast<const uint4 *>(fim + gi * 3);
                uint32_t FR[4], FG[4], FB[4];
                unpack16(f4[0], f4[1], f4[2], FR, FG, FB);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t sel = mk[e] * 255u;
                    R[e] = (FR[e] & sel) | (R[e] & ~sel);
                    G[e] = (FG[e] & sel) | (G[e] & ~sel);
                    B[e] = (FB[e] & sel) | (B[e] & ~sel);
                }
            }
        }
        uint4 fa, fb, fc;
        pack16(R, G, B, fa, fb, fc);
        uint4 *fo = reinterpret_cast<uint4 *>(fim + gi * 3);
        fo[0] = fa;
        fo[1] = fb;
        fo[2] = fc;
        if (maskout)
            *reinterpret_cast<uint4 *>(maskout + img * npx + gi) =
                make_uint4(mk[0] * 255u, mk[1] * 255u, mk[2] * 255u, mk[3] * 255u);
        uint32_t lw[4];
        if (prm.v_only) {
            uint32_t sum = 0, e16[16];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t v = vmax3(R[e], G[e], B[e]);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    e16[4 * e + kk] = s.vlut[(v >> (8 * kk)) & 255];
                    sum += e16[4 * e + kk];
                }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e)
                lw[e] = __byte_perm(__byte_perm(e16[4 * e], e16[4 * e + 1], 0x0040),
                                    __byte_perm(e16[4 * e + 2], e16[4 * e + 3], 0x0040), 0x5410);
            c0 += (sum >> 12) & 31;
            c1 += (sum >> 17) & 31;
            c2 += (sum >> 22) & 31;
            if (sum >> 27) {
#pragma unroll
                for (int kk = 15; kk >= 0; --kk)
                    if ((e16[kk] & 255) == 255) first = min(first, (int)gi + kk);
            }
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                lw[e] = 0;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const int cls = classify((R[e] >> (8 * kk)) & 255, (G[e] >> (8 * kk)) & 255,
                                             (B[e] >> (8 * kk)) & 255, scr);
                    lw[e] |= (uint32_t)cls << (8 * kk);
                    c0 += cls == 0;
                    c1 += cls == 1;
                    c2 += cls == 2;
                    if (cls == 255) first = min(first, (int)gi + 4 * e + kk);
                }
            }
        }
        *reinterpret_cast<uint4 *>(label + img * npx + gi) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
    for (int o = 16; o; o >>= 1) {
        c0 += __shfl_xor_sync(0xffffffffu, c0, o);
        c1 += __shfl_xor_sync(0xffffffffu, c1, o);
        c2 += __shfl_xor_sync(0xffffffffu, c2, o);
        first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        const int wi = threadIdx.x >> 5;
        s.red[wi][0] = c0; s.red[wi][1] = c1; s.red[wi][2] = c2; s.red[wi][3] = first;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < NTF / 32; ++i) {
            c0 += s.red[i][0]; c1 += s.red[i][1]; c2 += s.red[i][2]; first = min(first, s.red[i][3]);
        }
        if (c0) atomicAdd(&S.counts[0], (uint32_t)c0);
        if (c1) atomicAdd(&S.counts[1], (uint32_t)c1);
        if (c2) atomicAdd(&S.counts[2], (uint32_t)c2);
        if (first != 0x7fffffff) atomicMin(&S.first, first);
    }
}
}  // namespace fastk

bool full_hue(const IceScheme &sc) {
    for (int k = 0; k < 3; ++k)
        if (sc.lo[k][0] != 0 || sc.hi[k][0] < 179) return false;
    return true;
}
bool full_sat(const IceScheme &sc) {
    for (int k = 0; k < 3; ++k)
        if (sc.lo[k][1] != 0 || sc.hi[k][1] != 255) return false;
    return true;
}

bool window_ok(int k, int h, int w) { return k >= 3 && (k & 1) && k <= (h < w ? h : w); }

int g_autolabel_path = 0;  // 0 = auto, 1 = generic kernel only, 2 = fast kernel only (tests)

}  // namespace

extern "C" int ice_autolabel(const uint8_t *rgb, int64_t n, int32_t h, int32_t w,
                             const IceFilterCfg *cfg, const IceScheme *scheme,
                             uint8_t *filtered, uint8_t *label, uint8_t *mask,
                             uint32_t *affected, uint32_t *counts, int32_t *unmatched,
                             void *stream) {
    if (!cfg || !scheme || n < 0 || h < 1 || w < 1) return ICE_EINVAL;
    if (n == 0) return ICE_OK;
    if (!rgb || !filtered || !label || !affected || !counts || !unmatched) return ICE_EINVAL;
    if (h > MAXD || w > MAXD) return ICE_ETOOBIG;
    if (!window_ok(cfg->noise_median_k, h, w) || !window_ok(cfg->bg_dilate_k, h, w) ||
        !window_ok(cfg->bg_median_k, h, w))
        return ICE_EWINDOW;
    if (n > 0x7fffffff) return ICE_EINVAL;
    Params prm;
    prm.cfg = *cfg;
    prm.scheme = *scheme;
    prm.v_only = full_hue(*scheme) && full_sat(*scheme);
    const bool aligned = ((reinterpret_cast<uintptr_t>(rgb) | reinterpret_cast<uintptr_t>(filtered) |
                           reinterpret_cast<uintptr_t>(label) | reinterpret_cast<uintptr_t>(mask)) & 15) == 0;
    const bool fast = g_autolabel_path != 1 && h == 256 && w == 256 && aligned && cfg->bg_dilate_k == 7 &&
                      cfg->bg_median_k == fastk::MK && cfg->noise_median_k == 3;
    if (g_autolabel_path == 2 && !fast) return ICE_EINVAL;
    if (fast) {
        static bool attr_fast = false;
        if (!attr_fast) {
            cudaError_t e = cudaFuncSetAttribute(fastk::autolabel256_kernel,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(fastk::SmemF));
            if (e != cudaSuccess) return (int)e;
            attr_fast = true;
        }
        static int n_sm = 0;
        if (!n_sm) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
            if (n_sm <= 0) n_sm = 148;
        }
        fastk::autolabel256_kernel<<<(unsigned)n, fastk::NTF, sizeof(fastk::SmemF), (cudaStream_t)stream>>>(
            rgb, (int)n, n_sm, prm, filtered, label, mask, affected, counts, unmatched);
        ice::count_launch();
        return (int)cudaGetLastError();
    }
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(autolabel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(Smem));
        if (e != cudaSuccess) return (int)e;
        attr_set = true;
    }
    autolabel_kernel<<<(unsigned)n, NT, sizeof(Smem), (cudaStream_t)stream>>>(
        rgb, h, w, prm, filtered, label, mask, affected, counts, unmatched);
    ice::count_launch();
    return (int)cudaGetLastError();
}

extern "C" int ice_autolabel_set_path(int32_t mode) {
    if (mode < 0 || mode > 3) return ICE_EINVAL;
    g_autolabel_path = mode;
    return ICE_OK;
}

extern "C" int ice_autolabel_scene(const uint8_t *rgb, int64_t n, int32_t h, int32_t w,
                                   const IceFilterCfg *cfg, const IceScheme *scheme,
                                   uint8_t *filtered, uint8_t *label, uint8_t *mask,
                                   uint32_t *affected, uint32_t *counts, int32_t *unmatched,
                                   void *scratch, uint64_t *scratch_bytes, void *stream) {
    if (!cfg || !scheme || n < 0 || h < 1 || w < 1) return ICE_EINVAL;
    const bool region = h > MAXD || w > MAXD || g_autolabel_path == 3;
    if (!region) {  // one CTA per tile: no scratch
        if (!scratch && scratch_bytes) {
            *scratch_bytes = 0;
            return ICE_OK;
        }
        return ice_autolabel(rgb, n, h, w, cfg, scheme, filtered, label, mask, affected, counts, unmatched, stream);
    }
    if ((int64_t)h * w > 0x7fffffff || n > 0x7fffffff) return ICE_ETOOBIG;
    if (!window_ok(cfg->noise_median_k, h, w) || !window_ok(cfg->bg_dilate_k, h, w) ||
        !window_ok(cfg->bg_median_k, h, w))
        return ICE_EWINDOW;
    // SWAR windows (default windows, 16-B aligned rows) unless a test hook forces the generic path
    const bool swar = g_autolabel_path != 1 && g_autolabel_path != 3 && h >= 256 && w >= 256 && w % 16 == 0 &&
                      cfg->bg_dilate_k == 7 && cfg->bg_median_k == fastk::MK && cfg->noise_median_k == 3 &&
                      ((reinterpret_cast<uintptr_t>(rgb) | reinterpret_cast<uintptr_t>(filtered) |
                        reinterpret_cast<uintptr_t>(label) | reinterpret_cast<uintptr_t>(mask)) & 15) == 0;
    if (swar) {
        fastk::R256 g;
        g.h = h;
        g.w = w;
        g.ny = (h + 229) / 230;
        g.cs_y = (h + g.ny - 1) / g.ny;
        g.nx = (w + 223) / 224;
        g.cs_x = ((w + g.nx - 1) / g.nx + 15) / 16 * 16;
        g.nx = (w + g.cs_x - 1) / g.cs_x;
        const int regions = g.ny * g.nx;
        const uint64_t stats_bytes = ((uint64_t)n * sizeof(RegionStats) + 255) & ~(uint64_t)255;
        const uint64_t plane_bytes = ((uint64_t)n * h * w + 255) & ~(uint64_t)255;
        const uint64_t need = stats_bytes + 2 * plane_bytes;
        if (!scratch) {
            if (!scratch_bytes) return ICE_ESCRATCH;
            *scratch_bytes = need;
            return ICE_OK;
        }
        if (!scratch_bytes || *scratch_bytes < need) return ICE_ESCRATCH;
        if (n == 0) return ICE_OK;
        if (!rgb || !filtered || !label || !affected || !counts || !unmatched) return ICE_EINVAL;
        if ((int64_t)n * regions > 0x7fffffff) return ICE_ETOOBIG;
        Params prm;
        prm.cfg = *cfg;
        prm.scheme = *scheme;
        prm.v_only = full_hue(*scheme) && full_sat(*scheme);
        static bool attr_swar = false;
        if (!attr_swar) {
            cudaError_t e = cudaFuncSetAttribute(fastk::region256_d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)sizeof(fastk::SmemF));
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(fastk::region256_out_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(fastk::SmemF));
            if (e != cudaSuccess) return (int)e;
            attr_swar = true;
        }
        cudaStream_t st = (cudaStream_t)stream;
        RegionStats *stats = reinterpret_cast<RegionStats *>(scratch);
        uint8_t *dplanes = reinterpret_cast<uint8_t *>(scratch) + stats_bytes;
        uint8_t *bgplanes = dplanes + plane_bytes;
        cudaError_t e = cudaMemsetAsync(stats, 0, (size_t)n * sizeof(RegionStats), st);
        if (e != cudaSuccess) return (int)e;
        const unsigned grid = (unsigned)(n * regions);
        fastk::region256_d_kernel<<<grid, fastk::NTF, sizeof(fastk::SmemF), st>>>(rgb, g, *cfg, regions, dplanes,
                                                                                  bgplanes, stats);
        region_stats_kernel<<<(unsigned)n, 256, 0, st>>>(stats, h * w, *cfg);
        fastk::region256_out_kernel<<<grid, fastk::NTF, sizeof(fastk::SmemF), st>>>(
            rgb, g, prm, regions, dplanes, bgplanes, stats, filtered, label, mask);
        region_finish_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(stats, (int)n, affected, counts, unmatched);
        for (int k = 0; k < 4; ++k) ice::count_launch();
        return (int)cudaGetLastError();
    }
    const int halo = max(cfg->bg_dilate_k / 2 + cfg->bg_median_k / 2, cfg->noise_median_k / 2);
    int cmax = MAXD - 2 * halo;
    if (g_autolabel_path == 3) cmax = min(cmax, 40);  // test hook: many small regions
    if (cmax < 16) return ICE_ETOOBIG;
    RegionGeom g;
    g.h = h;
    g.w = w;
    g.halo = halo;
    g.ny = (h + cmax - 1) / cmax;
    g.nx = (w + cmax - 1) / cmax;
    g.cs_y = (h + g.ny - 1) / g.ny;
    g.cs_x = (w + g.nx - 1) / g.nx;
    const int regions = g.ny * g.nx;
    const uint64_t stats_bytes = ((uint64_t)n * sizeof(RegionStats) + 255) & ~(uint64_t)255;
    const uint64_t need = stats_bytes + (((uint64_t)n * h * w + 255) & ~(uint64_t)255);
    if (!scratch) {
        if (!scratch_bytes) return ICE_ESCRATCH;
        *scratch_bytes = need;
        return ICE_OK;
    }
    if (!scratch_bytes || *scratch_bytes < need) return ICE_ESCRATCH;
    if (n == 0) return ICE_OK;
    if (!rgb || !filtered || !label || !affected || !counts || !unmatched) return ICE_EINVAL;
    if ((int64_t)n * regions > 0x7fffffff) return ICE_ETOOBIG;
    Params prm;
    prm.cfg = *cfg;
    prm.scheme = *scheme;
    prm.v_only = full_hue(*scheme) && full_sat(*scheme);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(region_d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(region_out_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
        if (e != cudaSuccess) return (int)e;
        attr_set = true;
    }
    cudaStream_t st = (cudaStream_t)stream;
    RegionStats *stats = reinterpret_cast<RegionStats *>(scratch);
    uint8_t *dplanes = reinterpret_cast<uint8_t *>(scratch) + stats_bytes;
    cudaError_t e = cudaMemsetAsync(stats, 0, (size_t)n * sizeof(RegionStats), st);
    if (e != cudaSuccess) return (int)e;
    const unsigned grid = (unsigned)(n * regions);
    region_d_kernel<<<grid, NT, sizeof(Smem), st>>>(rgb, g, *cfg, regions, dplanes, stats);
    region_stats_kernel<<<(unsigned)n, 256, 0, st>>>(stats, h * w, *cfg);
    region_out_kernel<<<grid, NT, sizeof(Smem), st>>>(rgb, g, prm, regions, dplanes, stats, filtered, label, mask);
    region_finish_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(stats, (int)n, affected, counts, unmatched);
    for (int k = 0; k < 4; ++k) ice::count_launch();
    return (int)cudaGetLastError();
}

extern "C" int ice_segment(const uint8_t *rgb, int64_t n, int32_t h, int32_t w,
                           const IceScheme *scheme, uint8_t *label, uint32_t *counts,
                           int32_t *unmatched, void *stream) {
    if (!scheme || n < 0 || h < 1 || w < 1) return ICE_EINVAL;
    if (n == 0) return ICE_OK;
    if (!rgb || !label || !counts || !unmatched || n > 0x7fffffff) return ICE_EINVAL;
    if ((int64_t)h * w > 0x7fffffff / 3) return ICE_ETOOBIG;
    const int npx = h * w;
    cudaStream_t st = (cudaStream_t)stream;
    if (npx % 16 == 0 && (reinterpret_cast<uintptr_t>(rgb) & 15) == 0 && (reinterpret_cast<uintptr_t>(label) & 15) == 0) {
        const bool nh = !full_hue(*scheme), ns = !full_sat(*scheme);
        if (!nh && !ns) segment_vec_kernel<false, false><<<(unsigned)n, SEG_VNT, 0, st>>>(rgb, npx, *scheme, label, counts, unmatched);
        else if (nh && ns) segment_vec_kernel<true, true><<<(unsigned)n, SEG_VNT, 0, st>>>(rgb, npx, *scheme, label, counts, unmatched);
        else if (nh) segment_vec_kernel<true, false><<<(unsigned)n, SEG_VNT, 0, st>>>(rgb, npx, *scheme, label, counts, unmatched);
        else segment_vec_kernel<false, true><<<(unsigned)n, SEG_VNT, 0, st>>>(rgb, npx, *scheme, label, counts, unmatched);
        ice::count_launch();
    } else {
        segment_kernel<<<(unsigned)n, SEG_NT, 0, st>>>(rgb, npx, *scheme, label, counts, unmatched);
        ice::count_launch();
    }
    return (int)cudaGetLastError();
}

extern "C" int ice_rgb_to_hsv(const uint8_t *rgb, int64_t npx, uint8_t *hsv, void *stream) {
    if (npx < 0 || (npx > 0 && (!rgb || !hsv))) return ICE_EINVAL;
    if (npx == 0) return ICE_OK;
    int64_t blocks = (npx + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    hsv_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(rgb, npx, hsv);
    ice::count_launch();
    return (int)cudaGetLastError();
}

#ifdef ICE_AL_PROF
extern "C" int ice_al_prof_read(unsigned long long *out16, int reset) {
    cudaMemcpyFromSymbol(out16, g_al_prof, sizeof(unsigned long long) * 16);
    if (reset) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_al_prof, z, sizeof z);
    }
    return 0;
}
#endif
