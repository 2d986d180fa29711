/*
 * icelabel_b200.h -- C ABI of the B200-native sea-ice labeling / U-Net training path.
 *
 * One shared library (paper_2403_13135_b200/_C/libicelabel_b200.so, sm_100a only).
 * Conventions for every entry point:
 *   - all array arguments are DEVICE pointers owned by the caller; the library never
 *     allocates caller-visible memory;
 *   - work is enqueued asynchronously on `stream` (a cudaStream_t, NULL = legacy);
 *   - return 0 on success, a negative ICE_E* code for an argument error detected on
 *     the host before any launch, or a positive CUDA error code.
 *
 * The reference (arxiv 2403.13135, /root/reference/pkg) is pure Python; it has no FFI.
 * Each entry point below names the Python function whose semantics it replaces; the
 * Python bindings in paper_2403_13135_b200/_native.py keep those signatures.
 */
#ifndef ICELABEL_B200_H
#define ICELABEL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ICE_OK 0
#define ICE_EINVAL (-1)     /* bad size / pointer / configuration                     */
#define ICE_EWINDOW (-2)    /* window k exceeds tile extent (kernels.py:38-39)         */
#define ICE_ETOOBIG (-3)    /* tile larger than the on-chip plane (256 x 256)         */
#define ICE_ENODRIVER (-4)  /* cuTensorMapEncodeTiled entry point unavailable          */

/* FilterConfig (icelabel/cloudfilter.py:23-66) as a POD. */
typedef struct {
    int32_t bg_dilate_k;     /* odd >= 3, default 7   */
    int32_t bg_median_k;     /* odd >= 3, default 21  */
    int32_t noise_median_k;  /* odd >= 3, default 3   */
    int32_t mask_mode_fixed; /* 0 = "otsu", 1 = "fixed" */
    int32_t fixed_t;         /* 0..255, default 128   */
    int32_t diff_truncate;   /* 0/1                   */
    int32_t truncate_t;      /* 0..255, default 16    */
} IceFilterCfg;

/* SegmentationScheme (icelabel/segmentation.py:50-89): three inclusive (h,s,v) boxes in
 * precedence order (sorted by class id), hue bounds already clamped to 179. */
typedef struct {
    uint8_t lo[3][3];
    uint8_t hi[3][3];
    uint8_t cls[3];
    uint8_t pad[5];
} IceScheme;

/* Fused auto-label kernel (K1): replaces engine.process_tile (engine.py:145-160) =
 * cloudfilter.apply_filter (cloudfilter.py:99-117) + segmentation.segment
 * (segmentation.py:118-128) over a batch of n tiles, plus per-class counts (new).
 *   rgb       u8 [n][h][w][3]            input tiles (h, w <= 256)
 *   filtered  u8 [n][h][w][3]            repaired tiles (FilterOutput.filtered)
 *   label     u8 [n][h][w]               class ids; 255 where the scheme matched nothing
 *   mask      u8 [n][h][w] or NULL       cloud/shadow mask {0,255} (FilterOutput.cloud_shadow_mask)
 *   affected  u32 [n]                    masked-pixel count (affected_fraction * h * w)
 *   counts    u32 [n][3]                 per-class pixel counts of `label`
 *   unmatched i32 [n]                    first row-major unmatched pixel, or -1
 * Returns ICE_EWINDOW when a window exceeds min(h, w) (checked in the reference order
 * noise_median_k, bg_dilate_k, bg_median_k). */
int ice_autolabel(const uint8_t *rgb, int64_t n, int32_t h, int32_t w,
                  const IceFilterCfg *cfg, const IceScheme *scheme,
                  uint8_t *filtered, uint8_t *label, uint8_t *mask,
                  uint32_t *affected, uint32_t *counts, int32_t *unmatched,
                  void *stream);

/* Segment-only kernel (K1s): replaces segmentation.segment (segmentation.py:118-128)
 * as called by `icelabel label` (cli.py:131-146).  Any h, w. */
int ice_segment(const uint8_t *rgb, int64_t n, int32_t h, int32_t w,
                const IceScheme *scheme, uint8_t *label, uint32_t *counts,
                int32_t *unmatched, void *stream);

/* 8-bit HSV conversion: replaces raster.convert_raster (raster.py:187-216); integer-exact
 * restatement of the float64 reference.  rgb/hsv u8 [npx][3]. */
int ice_rgb_to_hsv(const uint8_t *rgb, int64_t npx, uint8_t *hsv, void *stream);

/* ---------------------------------------------------------------------------------
 * U-Net training ops (icetrain/model.py:64-130, train.py:85-120).  Activations are
 * NHWC bf16 (uint16_t bit patterns), conv weights KRSC bf16 ([cout][kh][kw][cin]),
 * master weights / grads / Adam state fp32.
 * --------------------------------------------------------------------------------- */

/* Implicit-GEMM convolution on tcgen05 (model.py:68-69 Conv2d(k=3, padding=1), and the
 * 1x1 / im2col-stem case with ksize = 1).  NHWC bf16 activations, KRSC bf16 weights
 * [cout][ksize][ksize][c1 + c2].  The input is the channel concatenation [x1 | x2]
 * (model.py:129 torch.cat([skip, x], 1)); x2 may be NULL with c2 = 0.  All channel
 * counts must be multiples of 64, h and w powers of two.
 *   y = act(conv(x, w) + bias) * drop_scale[n][cout]; act = ReLU if relu != 0;
 *   bias, drop_scale may be NULL. */
int ice_conv_fprop(const uint16_t *x1, int32_t c1, const uint16_t *x2, int32_t c2,
                   int32_t n, int32_t h, int32_t w, int32_t ksize, const uint16_t *wgt,
                   const float *bias, int32_t cout, int32_t relu, const float *drop_scale,
                   uint16_t *y, void *stream);

/* Data gradient of ice_conv_fprop w.r.t. its input (autograd of model.py:68-69, 129).
 * dx is written split into dx1 (first c1 channels) and dx2 (last c2; may be NULL), each
 *   dx_i = (conv_transpose(dy, w)_i + add_i) * drop_scale_i[n][c] * [relu_ref_i > 0]
 * i.e. the fused backward of "ReLU -> Dropout2d" for the tensor that fed the conv, plus an
 * optional second gradient contribution (the skip path).  Optional pointers may be NULL. */
int ice_conv_dgrad(const uint16_t *dy, int32_t cout, int32_t n, int32_t h, int32_t w,
                   int32_t ksize, const uint16_t *wgt, int32_t c1, int32_t c2,
                   uint16_t *dx1, const uint16_t *relu_ref1, const float *drop_scale1,
                   const uint16_t *add1, uint16_t *dx2, const uint16_t *relu_ref2,
                   const float *drop_scale2, const uint16_t *add2, void *stream);

/* Weight gradient: dw[cout][ksize][ksize][c1 + c2] (fp32) += sum over pixels of
 * dy[p][cout] * x[p + tap][c].  dw must be zeroed by the caller before the first call. */
int ice_conv_wgrad(const uint16_t *x1, int32_t c1, const uint16_t *x2, int32_t c2,
                   const uint16_t *dy, int32_t cout, int32_t n, int32_t h, int32_t w,
                   int32_t ksize, float *dw, void *stream);

#ifdef __cplusplus
}
#endif
#endif
