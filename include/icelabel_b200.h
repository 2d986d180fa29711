/*
 * icelabel_b200.h -- C ABI of the B200-native sea-ice labeling / U-Net training path.
 *
 * One shared library (paper_2403_13135_b200/_C/libicelabel_b200.so, sm_100a only).
 * Conventions for every entry point:
 *   - all array arguments are DEVICE pointers owned by the caller; the library never
 *     allocates device memory (temporary space comes from caller-owned scratch, below);
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
#define ICE_ETOOBIG (-3)    /* extent beyond what the entry point handles             */
#define ICE_ENODRIVER (-4)  /* cuTensorMapEncodeTiled entry point unavailable          */
#define ICE_ESCRATCH (-5)   /* caller scratch smaller than the call needs              */

/* Scratch.  Entry points with a (void *scratch, uint64_t *scratch_bytes) pair take their
 * temporary device space from the caller (split-K partial slices, per-CTA / per-block partial
 * sums of bias and head gradients, the merged halving-conv weights):
 *   - scratch == NULL, scratch_bytes != NULL: size query -- *scratch_bytes = bytes this call
 *     needs; nothing is launched, ICE_OK is returned (CUB-style two-phase call);
 *   - scratch != NULL: *scratch_bytes is its capacity; a call that needs more returns
 *     ICE_ESCRATCH before any launch;
 *   - both NULL: only calls that need no scratch succeed.
 * Calls sharing one scratch buffer must be ordered (same stream).
 * Determinism: no fp32 value on the training path is accumulated with atomics.  Partial sums
 * are stored into scratch and added by finishing kernels in a fixed order, so equal inputs
 * give bit-identical gradients, losses and weights run to run (the reference's same-seed
 * reproducibility, pkg/trainer/tests/test_train.py:71-75). */

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

/* Deferred finishing.  ice_finish_defer(1): from now on the fixed-order finishers of the
 * gradient reductions (split-K weight-gradient slice sums, bias-gradient column sums of
 * ice_conv_dgrad / ice_halve_dgrad / ice_maxpool_bwd / ice_bias_grad) are recorded instead of
 * launched; ice_finish_flush(stream) runs every recorded finisher in ONE kernel launch (same
 * partition and summation order as the immediate path: bit-identical results), ordered after
 * the work already on `stream`.  While deferring, the caller must keep each call's scratch
 * untouched until the flush (give every call its own scratch slice).  ice_finish_defer(0)
 * stops recording and drops anything not yet flushed.  Process-wide; not thread-safe. */
int ice_finish_defer(int32_t on);
int ice_finish_flush(void *stream);

/* Gradient overwrite mode.  ice_grad_overwrite(1): until ice_grad_overwrite(0), every gradient
 * producer (ice_conv_wgrad, ice_halve_wgrad, ice_stem_wgrad, and the bias / head gradients of
 * ice_conv_dgrad, ice_halve_dgrad, ice_maxpool_bwd, ice_head_ce, ice_bias_grad) STORES its
 * contribution (dw = contribution) instead of adding it; each gradient element has exactly one
 * producer per backward, so a backward in this mode writes every gradient without the buffer
 * having been zeroed.  The optimizer step can then skip zeroing (ice_adam zero_grad = 0), and
 * split-K weight gradients need not read the old value.  Process-wide; not thread-safe. */
int ice_grad_overwrite(int32_t on);

/* Re-read the convolution tiling switches (ICE_CONV_M2, ICE_WG_M2, ICE_NO_SPLITK, ... -- tuning
 * and test hooks; the defaults are the measured-best tilings) from the environment.  They are
 * read once when the library loads; a test that sets them calls this before and after. */
int ice_conv_reload_knobs(void);

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

/* ice_autolabel for any extent: whole scenes (cloudfilter.apply_filter as cli.py:112-125
 * calls it) and tiles larger than 256 x 256 (BASELINE configs[4]'s 512^2 tiles).  Extents
 * <= 256 go to ice_autolabel (no scratch).  Larger ones run the multi-CTA region path:
 * cores of <= (256 - 2 * halo)^2 pixels with their halo (halo = bg_dilate_k / 2 +
 * bg_median_k / 2), image-global statistics (d histogram -> stretch -> Otsu, channel
 * medians) in per-image scratch counters; 4 kernels + one memset.  With the default windows,
 * h, w >= 256 and w % 16 == 0 the cores run the SWAR pipeline on 256 x 256 windows of the
 * image (scratch: n * (4152 + 2 h w) bytes, rounded up); otherwise the generic byte pipeline
 * (n * (4152 + h w)).  Bit-exact like ice_autolabel.
 * ICE_ETOOBIG: h * w >= 2^31, or windows so large that a core would be < 16 pixels. */
int ice_autolabel_scene(const uint8_t *rgb, int64_t n, int32_t h, int32_t w,
                        const IceFilterCfg *cfg, const IceScheme *scheme,
                        uint8_t *filtered, uint8_t *label, uint8_t *mask,
                        uint32_t *affected, uint32_t *counts, int32_t *unmatched,
                        void *scratch, uint64_t *scratch_bytes, void *stream);

/* Kernel selection for ice_autolabel (test hook, process-wide): 0 = automatic (the SWAR
 * 256 x 256 kernel for 256 x 256 tiles with the default windows 7/21/3, the generic
 * kernel otherwise), 1 = generic kernel only, 2 = SWAR kernel only (ICE_EINVAL when the
 * call does not qualify), 3 = ice_autolabel_scene takes the region path at every extent
 * with cores of <= 40 x 40 pixels (exercises the halo logic on small inputs).  All paths
 * are exact; the hook lets tests compare them. */
int ice_autolabel_set_path(int32_t mode);

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
 *   bias, drop_scale may be NULL.  relu_bits (may be NULL) receives the mask y > 0 packed as
 *   uint32 words [cout / 32][n * h * w] (bit j of word k = channel 32 k + j), the 16x smaller
 *   ReLU reference ice_conv_dgrad's relu_bits1 consumes. */
int ice_conv_fprop(const uint16_t *x1, int32_t c1, const uint16_t *x2, int32_t c2,
                   int32_t n, int32_t h, int32_t w, int32_t ksize, const uint16_t *wgt,
                   const float *bias, int32_t cout, int32_t relu, const float *drop_scale,
                   uint16_t *y, uint32_t *relu_bits, void *scratch, uint64_t *scratch_bytes,
                   void *stream);

/* Data gradient of ice_conv_fprop w.r.t. its input (autograd of model.py:68-69, 129).
 * dx is written split into dx1 (first c1 channels) and dx2 (last c2; may be NULL), each
 *   dx_i = (conv_transpose(dy, w)_i + add_i) * drop_scale_i[n][c] * [relu_ref_i > 0]
 * i.e. the fused backward of "ReLU -> Dropout2d" for the tensor that fed the conv, plus an
 * optional second gradient contribution (the skip path).  Optional pointers may be NULL.
 * dx2_planes != 0 writes dx2 as four sub-pixel planes [4][n][h/2][w/2][c2] (plane
 * 2*(y&1)+(x&1)), the layout ice_halve_dgrad / ice_halve_wgrad consume.
 * dbias{1,2} (fp32 [c1] / [c2], may be NULL): += column sums of dx{1,2} -- the bias gradient
 * of the layer whose pre-activation gradient dx_i is, fused into the epilogue.
 * relu_bits1 (may be NULL): the ReLU mask of dx1 as ice_conv_fprop's packed relu_bits, used
 * instead of relu_ref1. */
int ice_conv_dgrad(const uint16_t *dy, int32_t cout, int32_t n, int32_t h, int32_t w,
                   int32_t ksize, const uint16_t *wgt, int32_t c1, int32_t c2,
                   uint16_t *dx1, const uint16_t *relu_ref1, const float *drop_scale1,
                   const uint16_t *add1, uint16_t *dx2, const uint16_t *relu_ref2,
                   const float *drop_scale2, const uint16_t *add2, int32_t dx2_planes,
                   float *dbias1, float *dbias2, const uint32_t *relu_bits1,
                   void *scratch, uint64_t *scratch_bytes, void *stream);

/* Weight gradient: dw[cout][ksize][ksize][c1 + c2] (fp32) += sum over pixels of
 * dy[p][cout] * x[p + tap][c].  dw must be zeroed by the caller before the first call.
 * When the pixel range is split across CTAs, each split's partial goes to scratch and the
 * splits are added in split order. */
int ice_conv_wgrad(const uint16_t *x1, int32_t c1, const uint16_t *x2, int32_t c2,
                   const uint16_t *dy, int32_t cout, int32_t n, int32_t h, int32_t w,
                   int32_t ksize, float *dw, void *scratch, uint64_t *scratch_bytes,
                   void *stream);

/* Halving conv forward (model.py:79-88,105,128): y[n][2h][2w][cout] =
 * conv2x2(pad(upsample_nearest_2x(x), (0,1,0,1))) + bias, as four sub-pixel GEMMs over
 * the low-res x[n][h][w][c] with the 9 combined weight slabs wc[cout][9][c] (bf16) that
 * ice_halve_prep builds from the 2x2 weights. */
int ice_halve_fprop(const uint16_t *x, int32_t c, int32_t n, int32_t h, int32_t w,
                    const uint16_t *wc, const float *bias, int32_t cout, uint16_t *y,
                    void *scratch, uint64_t *scratch_bytes, void *stream);

/* Halving conv data gradient: dx[n][h][w][c] = (sum over sub-pixel classes and taps of
 * dy_planes[cls][n][h - dy][w - dx][cout] * wc^T) * drop_scale[n][c] * [relu_ref > 0];
 * dbias (may be NULL) += column sums of dx (fused bias gradient). */
int ice_halve_dgrad(const uint16_t *dy_planes, int32_t cout, int32_t n, int32_t h, int32_t w,
                    const uint16_t *wc, int32_t c, uint16_t *dx, const uint16_t *relu_ref,
                    const uint32_t *relu_bits, const float *drop_scale, float *dbias, void *scratch,
                    uint64_t *scratch_bytes, void *stream);

/* Halving conv weight gradient: dw[cout][2][2][c] (fp32, caller-zeroed) +=
 * sum over classes/pixels of dy_planes[cls][p] (x) x[p + ((cy + a) / 2, (cx + b) / 2)]. */
int ice_halve_wgrad(const uint16_t *x, int32_t c, const uint16_t *dy_planes, int32_t cout,
                    int32_t n, int32_t h, int32_t w, float *dw, void *scratch,
                    uint64_t *scratch_bytes, void *stream);

/* ---- bandwidth-bound U-Net kernels (unet_ops.cu) ---------------------------------- */

/* Input stem: train.py:63 (u8 NHWC / 255) fused with the im2col of the first 3x3 conv
 * (model.py:68, Cin = 3): out[p][(r*3+s)*3+c] = img[p+(r-1,s-1)][c] / 255, zero outside
 * and in columns 27..63.  img u8 [n][h][w][3], out bf16 [n][h][w][64]. */
int ice_stem_im2col(const uint8_t *img, int32_t n, int32_t h, int32_t w, uint16_t *out,
                    void *stream);

/* Fused stem forward, replacing ice_stem_im2col + the K = 64 GEMM on the training path: the
 * first conv (3 -> 64, 3 x 3, model.py:64-76 on x = u8 / 255, train.py:63) straight from the
 * u8 images, no im2col buffer.  wt bf16 [64][64] = W[co][(r*3+s)*3+c] (columns 27..63 zero,
 * the ice_stem_im2col column order), bias fp32 [64]; y = ReLU(conv + bias) bf16 [n][h][w][64];
 * relu_bits (optional) u32 [2][n*h*w]: bit j of word c = channel 32 c + j of y > 0. */
int ice_stem_fprop(const uint8_t *img, int32_t n, int32_t h, int32_t w, const uint16_t *wt,
                   const float *bias, uint16_t *y, uint32_t *relu_bits, void *stream);

/* Fused stem weight gradient: dw[co][k] += sum_p dz[p][co] * x_col[p][k] with the im2col
 * columns gathered from the u8 images (k < 27; columns 27..63 get nothing).  dz bf16
 * [n][h][w][64], dw fp32 [64][64].  Per-CTA partial slices in scratch, added in CTA order
 * (deterministic; deferrable, see ice_finish_defer). */
int ice_stem_wgrad(const uint8_t *img, int32_t n, int32_t h, int32_t w, const uint16_t *dz, float *dw,
                   void *scratch, uint64_t *scratch_bytes, void *stream);

/* Same stem from an fp32 NHWC image already in [0, 1] (UNet.forward on float input). */
int ice_stem_im2col_f32(const float *img, int32_t n, int32_t h, int32_t w, uint16_t *out,
                        void *stream);

/* fp32 [rows][k] -> bf16 [rows][kp] zero-padded (stem weights 64 x 27 -> 64 x 64). */
int ice_pad_weights(const float *src, int32_t rows, int32_t k, uint16_t *dst, int32_t kp,
                    void *stream);

/* 2x2 halving-conv weights fp32 [cout][2][2][c] -> 9 combined bf16 slabs [cout][9][c]. */
int ice_halve_prep(const float *w, int32_t cout, int32_t c, uint16_t *wc, void *stream);

/* nn.MaxPool2d(2) forward (model.py:102,125), NHWC bf16, c % 8 == 0. */
int ice_maxpool_fwd(const uint16_t *x, int32_t n, int32_t h, int32_t w, int32_t c,
                    uint16_t *y, void *stream);

/* Fused backward of ReLU -> Dropout2d -> {skip, MaxPool2d} for a down block output x:
 * dz = (add + maxpool_backward(dpool)) * drop[n][c] * [x > 0]; add/drop may be NULL.
 * Ties route to the first maximum in window order, like torch's CPU max_pool2d.
 * dbias (fp32 [c], may be NULL) += sum of dz over pixels (fused bias gradient). */
int ice_maxpool_bwd(const uint16_t *x, const uint16_t *dpool, const uint16_t *add,
                    const float *drop, int32_t n, int32_t h, int32_t w, int32_t c,
                    uint16_t *dz, float *dbias, void *scratch, uint64_t *scratch_bytes,
                    void *stream);

/* Head (model.py:109,130 out = Conv2d(64, 3, 1)) + nn.CrossEntropyLoss (train.py:89,96).
 * h bf16 [npx][64] (hw pixels per image), labels u8 [npx], w_out fp32 [3][64], b_out [3].
 * Accumulates stats[0] += sum of per-pixel losses, stats[1] += argmax hits (if stats).
 * Training (dw, db non-NULL): dlogits = (softmax - onehot) * grad_scale; dw += dlogits^T h,
 * db += sum dlogits, and dz (if non-NULL) = (dlogits W) * drop[n][c] * [h > 0].
 * logits (optional) fp32 [npx][3]; dzbias (optional) fp32 [64] += sum of dz (the bias
 * gradient of the conv that produced h). */
int ice_head_ce(const uint16_t *h, int64_t npx, int32_t hw, const uint8_t *labels,
                const float *w_out, const float *b_out, const float *drop, float grad_scale,
                uint16_t *dz, float *dw, float *db, float *stats, float *logits, float *dzbias,
                void *scratch, uint64_t *scratch_bytes, void *stream);

/* Bias gradient: db[c] += sum_rows dz[row][c] (dz bf16 [rows][c], c % 8 == 0, c <= 2048). */
int ice_bias_grad(const uint16_t *dz, int64_t rows, int32_t c, float *db, void *scratch,
                  uint64_t *scratch_bytes, void *stream);

/* Dropout2d multipliers (model.py:74-75): out[i] = (u_i >= p) / (1 - p), u from a
 * counter-based hash of (seed + f(*step_dev), i); step_dev (may be NULL) is the device step
 * counter, so CUDA-graph replays draw fresh masks. */
int ice_dropout_scale(int32_t count, float p, uint64_t seed, const int64_t *step_dev, float *out,
                      void *stream);

/* torch.optim.Adam step (defaults of train.py:149: no weight decay, no amsgrad) over flat
 * fp32 buffers, fused with the bf16 working-copy write and (zero_grad != 0) zeroing of g --
 * skipped when the next backward runs in gradient overwrite mode.  Hyper-parameters are
 * doubles (torch forms 1 - beta and the bias corrections from Python floats).  The step t is
 * `step`, or *step_dev when step_dev is non-NULL (bias corrections computed on the device). */
int ice_adam(float *p, float *g, float *m, float *v, int64_t n, int64_t step,
             const int64_t *step_dev, double lr, double beta1, double beta2, double eps,
             int32_t zero_grad, uint16_t *out_bf16, void *stream);

/* *counter += delta on the device (the step counter advanced inside CUDA graphs). */
int ice_counter_add(int64_t *counter, int64_t delta, void *stream);

/* fp32 -> bf16 cast; fill. */
int ice_cast_bf16(const float *src, int64_t n, uint16_t *dst, void *stream);
int ice_fill_f32(float *dst, int64_t n, float value, void *stream);

/* ---------------------------------------------------------------------------------
 * Data path around the hot paths: u8 byte work, HBM-bound.
 * --------------------------------------------------------------------------------- */

/* cut_tiles (icetrain/data.py:55-66): img u8 [h][w][c] -> tiles u8 [rows*cols][size][size][c],
 * rows = ceil(h/size), cols = ceil(w/size), tile t = (t / cols, t % cols), zero padded. */
int ice_cut_tiles(const uint8_t *img, int32_t h, int32_t w, int32_t c, int32_t size, uint8_t *tiles,
                  void *stream);

/* stitch_tiles (data.py:69-80): inverse of ice_cut_tiles for a grid `cols` tiles wide
 * (cols <= 0: ceil(w/size)), padding cropped to h x w. */
int ice_stitch_tiles(const uint8_t *tiles, int32_t cols, int32_t size, int32_t c, int32_t h, int32_t w,
                     uint8_t *out, void *stream);

/* encode_labels (data.py:47-52): class index u8 [npx] -> RGB u8 [npx][3] from colors u8
 * [ncls][3].  *first_bad (caller-initialised to UINT64_MAX) = min index of a class >= ncls. */
int ice_encode_labels(const uint8_t *mask, int64_t npx, const uint8_t *colors, int32_t ncls, uint8_t *rgb,
                      uint64_t *first_bad, void *stream);

/* decode_labels (data.py:35-44): RGB u8 [npx][3] -> class index u8 [npx] (last matching
 * colour wins, 255 for unknown); *first_bad = min index of an unknown colour. */
int ice_decode_labels(const uint8_t *rgb, int64_t npx, const uint8_t *colors, int32_t ncls, uint8_t *mask,
                      uint64_t *first_bad, void *stream);

/* Inference head (infer.py:47 model.probabilities(x).argmax(1); softmax is monotone, so the
 * argmax of the out 1x1 conv logits): h bf16 [npx][64], w_out fp32 [3][64], b_out [3] ->
 * mask u8 [npx], first maximum on ties (torch.argmax). */
int ice_head_argmax(const uint16_t *h, int64_t npx, const float *w_out, const float *b_out, uint8_t *mask,
                    void *stream);

/* parse_labels(snap=True) (icelabel/segmentation.py:140-157): RGB u8 [npx][3] -> class index of
 * the nearest colour of colors u8 [ncls][3] in squared RGB distance (ties: earlier class). */
int ice_snap_labels(const uint8_t *rgb, int64_t npx, const uint8_t *colors, int32_t ncls, uint8_t *mask,
                    void *stream);

/* ssim (icelabel/metrics.py:153-172): a, b u8 [h][w][3]; window = the 11 x 11 normalised Gaussian
 * (float64, DEVICE memory); sums[c] (float64, device) = sum over the valid positions of channel c
 * of num / den in float64 (the caller divides by (h - 10) * (w - 10) and averages the channels).
 * Block sums are added in a fixed order (deterministic).  Needs scratch (see above). */
int ice_ssim(const uint8_t *a, const uint8_t *b, int32_t h, int32_t w, const double *window, double c1,
             double c2, double *sums, void *scratch, uint64_t *scratch_bytes, void *stream);

/* confusion (icelabel/metrics.py:108-113): counts u64 [k][k] += #(pred == a, ref == b),
 * k <= 4; pixels with a label >= k are added to *bad instead. */
int ice_confusion(const uint8_t *pred, const uint8_t *ref, int64_t npx, int32_t k, uint64_t *counts, uint64_t *bad,
                  void *stream);

/* Number of kernels this library has launched in the process so far (host-side count kept
 * at every launch site, finishing kernels included). */
uint64_t ice_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif
