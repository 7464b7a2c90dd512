// filter_at.cu - sampled evaluation of the separable filter (reference
// filtering.py:107-148, `filter_at`): the row pass only at the touched columns,
// then the column pass only at the requested points.
//
// The arithmetic is the one of the image sweeps (same fixed-point quanta from
// make_taps, same exact int32 box sums, same fp32 operation order), so every
// value is bit-identical to the same pixel of sb_separable_filter_2d - the
// property the reference states for its own filter_at.
#include "sweep_kernels.cuh"

namespace sb {

// R[col][y]: the row value at (y, cols[col]) rounded to the mid quantum.  The k nested
// boxes grow outward from the pixel (replicate boundary): box i adds the taps
// p_{i-1} < |d| <= p_i to box i-1, and is weighted as soon as it is complete, so the
// fp32 sum runs in slice order like every other kernel's.
template <typename Tin>
__global__ void __launch_bounds__(128) filter_at_rows_kernel(const Tin* __restrict__ src, long long row_stride, int H,
                                                             int W, const int* __restrict__ cols, int* __restrict__ R,
                                                             const __grid_constant__ TapsG t, int* status) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  const int ci = blockIdx.y;
  if (y >= H) return;
  const int x = cols[ci];
  const Tin* row = src + (long long)y * row_stride;
  RangeAcc bad;
  long long box = 0;  // int64: exact for the int32 quanta and for the wide (int64) ones alike
  int covered = -1;
  float acc = 0.0f;
  for (int i = 0; i < t.k; ++i) {
    for (int d = covered + 1; d <= t.p[i]; ++d) {
      box += to_fixed<Tin>(row[min(x + d, W - 1)], t, bad);
      if (d > 0) box += to_fixed<Tin>(row[max(x - d, 0)], t, bad);
    }
    covered = t.p[i];
    acc = fmaf(t.w_row[i], __ll2float_rn(box), acc);
  }
  R[(long long)ci * H + y] = __float_as_int(__fadd_rn(acc, kMagic)) - kMagicBits;  // _rn: never contracted into the last product
  report_status(status, bad, t);
}

// out[n]: the column pass of column pt_col[n] at row pt_y[n] (exact wrapping int32
// box sums of R, weighted in fp32 in slice order as the sweeps do)
__global__ void __launch_bounds__(128) filter_at_points_kernel(const int* __restrict__ R, int H,
                                                               const int* __restrict__ pt_col,
                                                               const int* __restrict__ pt_y, long long npts,
                                                               float* __restrict__ out,
                                                               const __grid_constant__ TapsG t) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= npts) return;
  const int* rc = R + (long long)pt_col[n] * H;
  const int y = pt_y[n];
  long long box = 0;
  int covered = -1;
  float acc = 0.0f;
  for (int i = 0; i < t.k; ++i) {
    for (int d = covered + 1; d <= t.p[i]; ++d) {
      box += rc[min(y + d, H - 1)];
      if (d > 0) box += rc[max(y - d, 0)];
    }
    covered = t.p[i];
    acc = fmaf(t.w_col[i], __ll2float_rn(box), acc);
  }
  out[n] = acc;
}

int launch_filter_at(const void* src, int src_dtype, long long row_stride, int H, int W, const int* cols, int ncols,
                     const int* pt_col, const int* pt_y, long long npts, float* out, int* R, const TapsG& t,
                     int* status, cudaStream_t st) {
  const dim3 g1((H + 127) / 128, ncols);
  switch (src_dtype) {
    case SB_DTYPE_U8:
      filter_at_rows_kernel<uint8_t><<<g1, 128, 0, st>>>((const uint8_t*)src, row_stride, H, W, cols, R, t, status);
      break;
    case SB_DTYPE_U16:
      filter_at_rows_kernel<uint16_t><<<g1, 128, 0, st>>>((const uint16_t*)src, row_stride, H, W, cols, R, t, status);
      break;
    case SB_DTYPE_F32:
      filter_at_rows_kernel<float><<<g1, 128, 0, st>>>((const float*)src, row_stride, H, W, cols, R, t, status);
      break;
    default:
      filter_at_rows_kernel<double><<<g1, 128, 0, st>>>((const double*)src, row_stride, H, W, cols, R, t, status);
      break;
  }
  filter_at_points_kernel<<<(unsigned)((npts + 127) / 128), 128, 0, st>>>(R, H, pt_col, pt_y, npts, out, t);
  return (int)cudaGetLastError();
}

}  // namespace sb
