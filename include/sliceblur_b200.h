/*
 * sliceblur_b200.h - C ABI of the B200 (sm_100a) running-sum Gaussian filter.
 *
 * This is the drop-in boundary for the reference package `sliceblur`
 * (/root/reference/pkg/src/sliceblur/).  The reference is pure Python/numpy
 * and has no FFI of its own; each entry point below replaces one function of
 * its filtering module, and the host package `paper_1107_4958_b200` binds them
 * with ctypes (see INTEGRATION.md for the binding a sliceblur maintainer would
 * add).
 *
 *   sb_check_kernel          <- filtering.py:39-45   _check_kernel
 *   sb_separable_filter_2d   <- filtering.py:76-104  separable_filter_2d
 *   sb_separable_filter_2d_window  (row-strip variant for the multi-GPU partition)
 *                               (+ batched / interleaved-channel layouts that
 *                               the reference reaches by looping in Python)
 *   sb_slice_filter_1d       <- filtering.py:67-73   slice_filter_1d
 *   sb_prefix_sum_f64        <- filtering.py:31-36   prefix_sum
 *   sb_filter_rows           <- filtering.py:48-64   _filter_rows (row pass only)
 *
 * Conventions
 *   - All image/signal pointers are DEVICE pointers owned by the caller; the
 *     library never allocates or frees memory and keeps no global mutable
 *     state besides a thread-local error string (sb_last_error).
 *   - Strides are in ELEMENTS.  `channels` > 1 means interleaved channels
 *     (pixel stride = channels); every channel is filtered independently.
 *   - Work is enqueued on `stream` (a cudaStream_t passed as void*; NULL =
 *     legacy default stream) and is stream-ordered: the call returns before
 *     the GPU finishes.
 *   - `radii` (int64, strictly increasing, >= 0) and `weights` (float64) are
 *     exactly the SliceKernel arrays of the reference (approx.py:82-129).
 *   - Arithmetic: exact int32 fixed-point running sums.  For
 *     uint8/uint16 input the first pass is exact; float input is quantised
 *     with a quantum derived from `value_bound` (an upper bound on |pixel|;
 *     pass <= 0 to declare "unknown", which the host wrapper resolves with a
 *     device max before calling).  For uint16 input a value_bound in
 *     (0, 65535) only refines the row-value quantum (the samples stay exact).
 *     Pixels violating the bound are reported through `status_dev` (bit
 *     SB_STATUS_RANGE) - never silently.
 *   - Return value: SB_OK or an error code; the message is in sb_last_error().
 */
#ifndef SLICEBLUR_B200_H
#define SLICEBLUR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Largest k (number of slices) the library accepts.  The templated sweep
 * kernels take k <= 8 (the paper's kernels have k = 3..5); larger k runs the
 * generic two-pass kernels, which also cover every radius < extent. */
#define SB_MAX_K 1024

/* Path policy (sb_set_path_policy): AUTO picks the fastest path that applies;
 * the others force a path for A/B timing and for the bit-identity tests. */
enum {
  SB_PATH_AUTO = 0,
  SB_PATH_GENERIC = 1,      /* generic two-pass kernels (row prefix, column prefix) for every call */
  SB_PATH_UNFUSED = 2,      /* row pass to an int32 plane, then a column kernel (no fused sweep)     */
  SB_PATH_U8_THREE_CTA = 3, /* uint8 fused sweep: three CTAs per SM, one band per consumer turn     */
  SB_PATH_U8_ONE_BAND = 4,  /* uint8 fused sweep: two CTAs per SM, one band per consumer turn       */
  SB_PATH_FUSED_WIDE = 5,   /* float32 one-channel, radii past the fused sweep: one launch, the row
                               values never in HBM (DRAM 1.05x algorithmic; slower than the default
                               two-launch path at these radii); else as AUTO          */
  SB_PATH_U8_ROWTILE = 6,   /* uint8 one-channel, small radii: the row-tile sweep (row pass on
                               thread-per-row warps with the row prefix in TMEM); else as AUTO      */
  SB_PATH_U8_PAIRED = 7,    /* uint8 fused sweep: two consumer warps per TMEM lane quadrant that
                               alternate bands (eight consumer warps per CTA); else as AUTO         */
  SB_PATH_U8_TWO_BAND = 8   /* uint8 fused sweep: four consumer warps, two bands per turn           */
};

/* return codes */
enum {
  SB_OK = 0,
  SB_ERR_INVALID_ARGUMENT = 1, /* -> ValueError (filtering.py:34-35, 70-71, 85-86)          */
  SB_ERR_KERNEL_TOO_LARGE = 2, /* -> KernelTooLargeError (filtering.py:27-28, 40-43)          */
  SB_ERR_NOT_UNIT_DC = 3,      /* -> ValueError "kernel must have unit DC gain" (44-45)       */
  SB_ERR_CUDA = 4,             /* launch / runtime failure                                    */
  SB_ERR_WORKSPACE = 5         /* workspace pointer NULL or smaller than sb_*_workspace_bytes */
};

/* source element types */
enum { SB_DTYPE_U8 = 0, SB_DTYPE_U16 = 1, SB_DTYPE_F32 = 2, SB_DTYPE_F64 = 3 };

/* bits written (atomicOr) into *status_dev by the kernels */
#define SB_STATUS_RANGE 1 /* a pixel exceeded value_bound (or was NaN/Inf)                     */
#define SB_STATUS_HALF 2  /* float sources: some |pixel| >= value_bound / 2.  A caller that     \
                             guessed the bound (e.g. from its previous image) keeps the result \
                             when RANGE is clear and HALF is set: the quantum is then within   \
                             one bit of the one the measured maximum gives.                    */

/* ABI version, bumped on any signature change. */
int sb_version(void);

/* Thread-local path policy (SB_PATH_*) for the calls made afterwards on this
 * thread; returns the previous policy, or -1 for an unknown value.  The
 * workspace queries honour it too. */
int sb_set_path_policy(int policy);

/* Thread-local description of the last error returned on this thread. */
const char* sb_last_error(void);

/* filtering.py:39-45: SB_ERR_KERNEL_TOO_LARGE if radii[k-1] >= extent,
 * SB_ERR_NOT_UNIT_DC if |sum w_i (2 p_i + 1) - 1| > 1e-6, else SB_OK. */
int sb_check_kernel(const int64_t* radii, const double* weights, int k, int64_t extent);

/* Bytes of device workspace sb_separable_filter_2d needs for this source
 * type and shape: 0 when the single fused kernel applies; otherwise the
 * intermediate plane of the two-kernel path (int32, or int64 past
 * 2 p_max + 1 > 2048; its row pitch is the width rounded up to four elements)
 * plus the generic kernels' scratch rows when they run.  Always ask: which path
 * runs depends on type, width, channels and radii (and the path policy). */
size_t sb_separable_filter_2d_workspace_bytes(int src_dtype, int64_t batch, int64_t height, int64_t width,
                                              int channels, const int64_t* radii, int k);

/* filtering.py:76-104 separable_filter_2d over a batch of images:
 *   dst[b, y, x, c] = cols(rows(src[b, :, :, c]))[y, x]
 * src: `batch` images of `height` x `width` pixels with `channels`
 * interleaved channels, element type `src_dtype`; dst: float32, same
 * layout rules.  src_image_stride / dst_image_stride may be 0 when batch == 1.
 * Validates like the reference: height/width >= 1, kernel fits both extents
 * (KernelTooLarge), unit DC gain. */
int sb_separable_filter_2d(const void* src, int src_dtype, int64_t batch, int64_t height, int64_t width,
                           int channels, int64_t src_image_stride, int64_t src_row_stride, float* dst,
                           int64_t dst_image_stride, int64_t dst_row_stride, const int64_t* radii,
                           const double* weights, int k, double value_bound, void* workspace,
                           size_t workspace_bytes, int* status_dev, void* stream);

/* Strip variant of sb_separable_filter_2d (the multi-GPU row-strip partition):
 * `src` holds `height` rows per image - a strip plus the halo rows received
 * from its neighbours - and only output rows [row_begin, row_end) are
 * written, to dst rows 0 .. row_end-row_begin-1.  Rows outside [0, height)
 * replicate the first/last row, so a strip at the global top/bottom passes
 * no halo there and gets the reference's boundary; interior strip edges see
 * real neighbour rows (a halo of radii[k-1] rows suffices). */
int sb_separable_filter_2d_window(const void* src, int src_dtype, int64_t batch, int64_t height, int64_t width,
                                  int channels, int64_t src_image_stride, int64_t src_row_stride,
                                  int64_t row_begin, int64_t row_end, float* dst, int64_t dst_image_stride,
                                  int64_t dst_row_stride, const int64_t* radii, const double* weights, int k,
                                  double value_bound, void* workspace, size_t workspace_bytes, int* status_dev,
                                  void* stream);

/* filtering.py:48-64 _filter_rows: the row pass alone, every row of a
 * (rows x width) array (row stride in elements), float32 output.  Needs
 * sb_filter_rows_workspace_bytes(...) bytes of workspace (0 unless the row is
 * too long for the shared-memory prefix of the generic kernel). */
size_t sb_filter_rows_workspace_bytes(int src_dtype, int64_t rows, int64_t width, const int64_t* radii, int k);
int sb_filter_rows(const void* src, int src_dtype, int64_t rows, int64_t width, int64_t src_row_stride,
                   float* dst, int64_t dst_row_stride, const int64_t* radii, const double* weights, int k,
                   double value_bound, void* workspace, size_t workspace_bytes, int* status_dev, void* stream);

/* filtering.py:67-73 slice_filter_1d on one signal of length n (workspace as
 * sb_filter_rows with rows = 1, width = n). */
int sb_slice_filter_1d(const void* src, int src_dtype, int64_t n, float* dst, const int64_t* radii,
                       const double* weights, int k, double value_bound, void* workspace, size_t workspace_bytes,
                       int* status_dev, void* stream);

/* filtering.py:31-36 prefix_sum: inclusive float64 scan of n >= 1 values.
 * Needs sb_prefix_sum_workspace_bytes(n) bytes of device workspace. */
size_t sb_prefix_sum_workspace_bytes(int64_t n);
int sb_prefix_sum_f64(const double* src, double* dst, int64_t n, void* workspace, size_t workspace_bytes,
                      void* stream);

/* max |x| over n elements of a device array (float32/float64/u8/u16),
 * written as a double to *out_dev; used by the host wrapper to derive
 * value_bound when the caller does not supply one. */
int sb_max_abs(const void* src, int src_dtype, int64_t n, double* out_dev, void* stream);

/* Accuracy harness - replaces oracle.exact_gaussian_2d and the sum behind
 * oracle.mse / oracle.psnr (reference oracle.py:58-102).  Not the hot path.
 * sb_exact_gaussian_2d: dense separable correlation with the ntaps (odd) fp64
 * taps in taps_dev (gaussian_taps(sigma): truncation radius ceil(pi*sigma),
 * sum 1), replicate boundary, rows then columns, fp64 (height, width) output in
 * dst; bit-identical to the reference's numpy arithmetic.  Needs
 * sb_exact_gaussian_workspace_bytes(height, width) bytes of workspace.
 * sb_sum_sq_diff: *out_dev += sum (a[i] - b[i])^2 in fp64 over n elements
 * (a, b: SB_DTYPE_F32 or SB_DTYPE_F64 device arrays). */
size_t sb_exact_gaussian_workspace_bytes(int64_t height, int64_t width);
int sb_exact_gaussian_2d(const void* src, int src_dtype, int64_t height, int64_t width, int64_t src_row_stride,
                         const double* taps_dev, int ntaps, double* dst, void* workspace, size_t workspace_bytes,
                         void* stream);
int sb_sum_sq_diff(const void* a, int a_dtype, const void* b, int b_dtype, int64_t n, double* out_dev, void* stream);

/* Sampled evaluation - replaces filtering.filter_at (filtering.py:107-148).
 * out[n] = pixel (pt_y[n], cols[pt_col[n]]) of sb_separable_filter_2d of the
 * (height, width) single-channel image `src` (bit-identical to it): the row
 * pass runs only at the ncols touched columns `cols`, the column pass only at
 * the npts points.  cols, pt_col, pt_y (int32) and out (npts floats) are device
 * arrays; the caller guarantees 0 <= cols < width, 0 <= pt_col < ncols and
 * 0 <= pt_y < height (the reference raises ValueError for points outside the
 * image before any arithmetic).  Needs sb_filter_at_workspace_bytes(height,
 * ncols) bytes of device workspace; value_bound and status_dev as in
 * sb_separable_filter_2d. */
size_t sb_filter_at_workspace_bytes(int64_t height, int64_t ncols);
int sb_filter_at(const void* src, int src_dtype, int64_t height, int64_t width, int64_t src_row_stride,
                 const int32_t* cols, int64_t ncols, const int32_t* pt_col, const int32_t* pt_y, int64_t npts,
                 float* out, const int64_t* radii, const double* weights, int k, double value_bound, void* workspace,
                 size_t workspace_bytes, int* status_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SLICEBLUR_B200_H */
