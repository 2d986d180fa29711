/*
 * oracle/autolabel_ref.c -- CPU restatement of the reference auto-labeler.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the
 * checker or the timed CPU arm.  The product path (paper_2403_13135_b200) never
 * links or calls it.
 *
 * Each function restates one reference function; citations are relative to
 * /root/reference/pkg/src/icelabel/.  The restatement is deliberately naive
 * (per-pixel windows, float64 where the reference uses float64) so that it is
 * obviously the reference's arithmetic.  It is pinned against sha256 digests of
 * the reference's own outputs in tests/golden/autolabel_golden.json.
 *
 * Build: oracle/Makefile -> oracle/liboracle_autolabel.so
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_ERR_WINDOW_NOISE 1   /* kernels.py:38-39 via detect_mask median_blur  */
#define OR_ERR_WINDOW_DILATE 2  /* kernels.py:38-39 via estimate_background dilate */
#define OR_ERR_WINDOW_MEDIAN 3  /* kernels.py:38-39 via estimate_background median */
#define OR_ERR_UNMATCHED 4      /* segmentation.py:123-127 */

typedef struct {
    int bg_dilate_k, bg_median_k, noise_median_k;
    int mask_mode_fixed; /* 0 = otsu, 1 = fixed (cloudfilter.py:34-35) */
    int fixed_t;
    int diff_truncate;
    int truncate_t;
} or_filter_cfg;

typedef struct {
    /* precedence order (sorted by class id, segmentation.py:62) */
    uint8_t lo[3][3]; /* [range][h,s,v] */
    uint8_t hi[3][3];
    uint8_t cls[3];
} or_scheme;

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* kernels.py:42-46 (cv2.medianBlur == oracles.median_oracle): rank k*k/2 of the
 * k x k window, edges replicated.  Counting sort per pixel. */
void or_median_blur(const uint8_t *src, int h, int w, int k, uint8_t *dst) {
    int r = k / 2, rank = (k * k) / 2;
    unsigned cnt[256];
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            memset(cnt, 0, sizeof cnt);
            for (int dy = -r; dy <= r; ++dy) {
                const uint8_t *row = src + (size_t)clampi(y + dy, 0, h - 1) * w;
                for (int dx = -r; dx <= r; ++dx) cnt[row[clampi(x + dx, 0, w - 1)]]++;
            }
            int acc = 0, v = 0;
            for (; v < 256; ++v) {
                acc += cnt[v];
                if (acc > rank) break;
            }
            dst[(size_t)y * w + x] = (uint8_t)v;
        }
}

/* kernels.py:49-54 (cv2.dilate, BORDER_REPLICATE == oracles.dilate_oracle) */
void or_dilate(const uint8_t *src, int h, int w, int k, uint8_t *dst) {
    int r = k / 2;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            int m = 0;
            for (int dy = -r; dy <= r; ++dy)
                for (int dx = -r; dx <= r; ++dx) {
                    int v = src[(size_t)clampi(y + dy, 0, h - 1) * w + clampi(x + dx, 0, w - 1)];
                    if (v > m) m = v;
                }
            dst[(size_t)y * w + x] = (uint8_t)m;
        }
}

/* kernels.py:66-74: float64 stretch, floor(x + 0.5); constant -> zeros */
void or_minmax_normalize(const uint8_t *src, size_t n, uint8_t *dst) {
    int lo = 255, hi = 0;
    for (size_t i = 0; i < n; ++i) {
        if (src[i] < lo) lo = src[i];
        if (src[i] > hi) hi = src[i];
    }
    if (hi == lo) {
        memset(dst, 0, n);
        return;
    }
    for (size_t i = 0; i < n; ++i) {
        double scaled = 255.0 * ((double)src[i] - (double)lo) / (double)(hi - lo);
        dst[i] = (uint8_t)floor(scaled + 0.5);
    }
}

/* kernels.py:77-110: exact integer between-class variance argmax, smallest t on ties */
/* z[0..nx+ny) = x * y, little-endian 64-bit limbs (schoolbook) */
static void mul_limbs(const uint64_t *x, int nx, const uint64_t *y, int ny, uint64_t *z) {
    for (int i = 0; i < nx + ny; ++i) z[i] = 0;
    for (int i = 0; i < nx; ++i) {
        unsigned __int128 carry = 0;
        for (int j = 0; j < ny; ++j) {
            unsigned __int128 t = (unsigned __int128)x[i] * y[j] + z[i + j] + carry;
            z[i + j] = (uint64_t)t;
            carry = t >> 64;
        }
        z[i + ny] = (uint64_t)carry;
    }
}

/* a1^2 * d2 > a2^2 * d1, exactly: the reference compares Python big ints
 * (num * best_den > best_num * den, kernels.py:104-106); for scenes beyond ~2^19 pixels
 * these products exceed 128 bits (a <= 255 * n0 * n1 < 2^128, d = n0 * n1 < 2^64). */
static int sq_ratio_greater(unsigned __int128 a1, uint64_t d1, unsigned __int128 a2, uint64_t d2) {
    uint64_t x1[2] = {(uint64_t)a1, (uint64_t)(a1 >> 64)}, x2[2] = {(uint64_t)a2, (uint64_t)(a2 >> 64)};
    uint64_t sq1[4], sq2[4], l[5], r[5];
    mul_limbs(x1, 2, x1, 2, sq1);
    mul_limbs(x2, 2, x2, 2, sq2);
    mul_limbs(sq1, 4, &d2, 1, l);
    mul_limbs(sq2, 4, &d1, 1, r);
    for (int i = 4; i >= 0; --i)
        if (l[i] != r[i]) return l[i] > r[i];
    return 0;
}

int or_otsu_threshold(const uint8_t *src, size_t n) {
    int64_t counts[256] = {0};
    for (size_t i = 0; i < n; ++i) counts[src[i]]++;
    __int128 n_total = 0, s_total = 0;
    for (int t = 0; t < 256; ++t) {
        n_total += counts[t];
        s_total += (__int128)t * counts[t];
    }
    int best_t = 0;
    unsigned __int128 best_a = 0; /* best_num = best_a^2 */
    uint64_t best_den = 1;
    __int128 n0 = 0, s0 = 0;
    for (int t = 0; t < 256; ++t) {
        n0 += counts[t];
        s0 += (__int128)t * counts[t];
        __int128 n1 = n_total - n0;
        if (n0 == 0 || n1 == 0) continue;
        __int128 s1 = s_total - s0;
        __int128 diff = s0 * n1 - s1 * n0;
        unsigned __int128 a = (unsigned __int128)(diff < 0 ? -diff : diff);
        uint64_t den = (uint64_t)(n0 * n1);
        if (sq_ratio_greater(a, den, best_a, best_den)) {
            best_a = a;
            best_den = den;
            best_t = t;
        }
    }
    return best_t;
}

/* raster.py:187-216: float64 HSV, half-up rounding, hue 180 -> 0 */
void or_rgb_to_hsv(const uint8_t *rgb, size_t n, uint8_t *hsv) {
    for (size_t i = 0; i < n; ++i) {
        double r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
        double v = r > g ? r : g;
        if (b > v) v = b;
        double mn = r < g ? r : g;
        if (b < mn) mn = b;
        double c = v - mn;
        double s = 0.0;
        if (v > 0) s = floor(255.0 * c / v + 0.5);
        double h = 0.0;
        if (c > 0) {
            double hdeg;
            if (v == r) {
                hdeg = fmod(60.0 * (g - b) / c, 360.0); /* np.mod: sign of divisor */
                if (hdeg < 0) hdeg += 360.0;
            } else if (v == g) {
                hdeg = 60.0 * (b - r) / c + 120.0;
            } else {
                hdeg = 60.0 * (r - g) / c + 240.0;
            }
            double half = floor(hdeg / 2.0 + 0.5);
            if (half == 180.0) half = 0.0;
            h = half;
        }
        hsv[3 * i] = (uint8_t)h;
        hsv[3 * i + 1] = (uint8_t)s;
        hsv[3 * i + 2] = (uint8_t)v;
    }
}

/* segmentation.py:118-128: first range (precedence order) containing the pixel.
 * Returns the row-major index of the first unmatched pixel, or -1. */
long or_segment(const uint8_t *rgb, size_t n, const or_scheme *sc, uint8_t *label) {
    uint8_t *hsv = (uint8_t *)malloc(3 * n);
    or_rgb_to_hsv(rgb, n, hsv);
    long first = -1;
    for (size_t i = 0; i < n; ++i) {
        int out = 255;
        for (int k = 0; k < 3 && out == 255; ++k) {
            int ok = 1;
            for (int ch = 0; ch < 3; ++ch)
                if (hsv[3 * i + ch] < sc->lo[k][ch] || hsv[3 * i + ch] > sc->hi[k][ch]) ok = 0;
            if (ok) out = sc->cls[k];
        }
        label[i] = (uint8_t)out;
        if (out == 255 && first < 0) first = (long)i;
    }
    free(hsv);
    return first;
}

/* cloudfilter.py:82-84 */
static void background(const uint8_t *c, int h, int w, const or_filter_cfg *cfg, uint8_t *bg) {
    uint8_t *tmp = (uint8_t *)malloc((size_t)h * w);
    or_dilate(c, h, w, cfg->bg_dilate_k, tmp);
    or_median_blur(tmp, h, w, cfg->bg_median_k, bg);
    free(tmp);
}

/* np.median over all pixels then round_half_up (cloudfilter.py:113) */
static int channel_center(const uint8_t *c, size_t n) {
    size_t cnt[256] = {0};
    for (size_t i = 0; i < n; ++i) cnt[c[i]]++;
    size_t lo_rank = (n - 1) / 2, hi_rank = n / 2;
    int a = -1, b = -1;
    size_t acc = 0;
    for (int v = 0; v < 256; ++v) {
        acc += cnt[v];
        if (a < 0 && acc > lo_rank) a = v;
        if (b < 0 && acc > hi_rank) b = v;
    }
    double med = ((double)a + (double)b) / 2.0;
    return (int)floor(med + 0.5);
}

static int check_window(int k, int h, int w) { return k <= (h < w ? h : w); }

/* cloudfilter.py:87-96 + 99-117; writes filtered (HxWx3), mask (HxW {0,255}).
 * Returns OR_OK or an OR_ERR_WINDOW_* code; *affected = masked pixel count. */
int or_apply_filter(const uint8_t *rgb, int h, int w, const or_filter_cfg *cfg,
                    uint8_t *filtered, uint8_t *mask, long *affected) {
    if (!check_window(cfg->noise_median_k, h, w)) return OR_ERR_WINDOW_NOISE;
    if (!check_window(cfg->bg_dilate_k, h, w)) return OR_ERR_WINDOW_DILATE;
    if (!check_window(cfg->bg_median_k, h, w)) return OR_ERR_WINDOW_MEDIAN;
    size_t n = (size_t)h * w;
    uint8_t *gray = (uint8_t *)malloc(n), *smooth = (uint8_t *)malloc(n);
    uint8_t *bg = (uint8_t *)malloc(n), *d = (uint8_t *)malloc(n), *dn = (uint8_t *)malloc(n);
    for (size_t i = 0; i < n; ++i) {
        uint8_t r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
        uint8_t v = r > g ? r : g;
        gray[i] = b > v ? b : v;
    }
    or_median_blur(gray, h, w, cfg->noise_median_k, smooth);
    background(gray, h, w, cfg, bg);
    for (size_t i = 0; i < n; ++i) {
        int diff = abs((int)smooth[i] - (int)bg[i]);
        if (cfg->diff_truncate && diff > cfg->truncate_t) diff = cfg->truncate_t;
        d[i] = (uint8_t)diff;
    }
    or_minmax_normalize(d, n, dn);
    int t = cfg->mask_mode_fixed ? cfg->fixed_t : or_otsu_threshold(dn, n);
    long count = 0;
    for (size_t i = 0; i < n; ++i) {
        mask[i] = dn[i] > t ? 255 : 0;
        count += mask[i] == 255;
    }
    memcpy(filtered, rgb, 3 * n);
    if (count > 0) {
        uint8_t *c = (uint8_t *)malloc(n), *bgc = (uint8_t *)malloc(n);
        for (int ch = 0; ch < 3; ++ch) {
            for (size_t i = 0; i < n; ++i) c[i] = rgb[3 * i + ch];
            background(c, h, w, cfg, bgc);
            int center = channel_center(c, n);
            for (size_t i = 0; i < n; ++i)
                if (mask[i] == 255) {
                    int f = (int)c[i] - (int)bgc[i] + center;
                    filtered[3 * i + ch] = (uint8_t)clampi(f, 0, 255);
                }
        }
        free(c);
        free(bgc);
    }
    *affected = count;
    free(gray);
    free(smooth);
    free(bg);
    free(d);
    free(dn);
    return OR_OK;
}

/* engine.py:145-160: apply_filter then segment(filtered).  label may hold 255 at
 * unmatched pixels; *unmatched = first row-major unmatched index or -1. */
int or_process_tile(const uint8_t *rgb, int h, int w, const or_filter_cfg *cfg,
                    const or_scheme *sc, uint8_t *filtered, uint8_t *label,
                    long *affected, long *unmatched) {
    uint8_t *mask = (uint8_t *)malloc((size_t)h * w);
    int rc = or_apply_filter(rgb, h, w, cfg, filtered, mask, affected);
    free(mask);
    if (rc != OR_OK) return rc;
    *unmatched = or_segment(filtered, (size_t)h * w, sc, label);
    return *unmatched >= 0 ? OR_ERR_UNMATCHED : OR_OK;
}
