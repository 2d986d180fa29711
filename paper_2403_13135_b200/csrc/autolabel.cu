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
__device__ int otsu_from_hist(const uint32_t *hist, Smem &s) {
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
        int t = cfg.mask_mode_fixed ? cfg.fixed_t : otsu_from_hist(s.hist, s);
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
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(autolabel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(Smem));
        if (e != cudaSuccess) return (int)e;
        attr_set = true;
    }
    autolabel_kernel<<<(unsigned)n, NT, sizeof(Smem), (cudaStream_t)stream>>>(
        rgb, h, w, prm, filtered, label, mask, affected, counts, unmatched);
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
    } else {
        segment_kernel<<<(unsigned)n, SEG_NT, 0, st>>>(rgb, npx, *scheme, label, counts, unmatched);
    }
    return (int)cudaGetLastError();
}

extern "C" int ice_rgb_to_hsv(const uint8_t *rgb, int64_t npx, uint8_t *hsv, void *stream) {
    if (npx < 0 || (npx > 0 && (!rgb || !hsv))) return ICE_EINVAL;
    if (npx == 0) return ICE_OK;
    int64_t blocks = (npx + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    hsv_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(rgb, npx, hsv);
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
