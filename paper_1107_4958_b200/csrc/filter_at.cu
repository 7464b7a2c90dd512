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

// R[col][y]: the row value at (y, cols[col]) rounded to the mid quantum; the k box
// sums come from one walk over the 2*pmax+1 taps (replicate boundary, nested boxes).
template <typename Tin>
__global__ void __launch_bounds__(128) filter_at_rows_kernel(const Tin* __restrict__ src, long long row_stride, int H,
                                                             int W, const int* __restrict__ cols, int* __restrict__ R,
                                                             Taps t, int* status) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  const int ci = blockIdx.y;
  if (y >= H) return;
  const int x = cols[ci];
  const Tin* row = src + (long long)y * row_stride;
  int box[SB_MAX_K];
#pragma unroll
  for (int i = 0; i < SB_MAX_K; ++i) box[i] = 0;
  bool bad = false;
  for (int d = -t.pmax; d <= t.pmax; ++d) {
    const int v = to_fixed<Tin>(row[min(max(x + d, 0), W - 1)], t, bad);
    const int ad = d < 0 ? -d : d;
#pragma unroll
    for (int i = 0; i < SB_MAX_K; ++i)
      if (i < t.k && ad <= t.p[i]) box[i] += v;
  }
  float acc = 0.0f;
#pragma unroll
  for (int i = 0; i < SB_MAX_K; ++i)
    if (i < t.k) acc = fmaf(t.w_row[i], i2f_fast((uint32_t)box[i]), acc);
  R[(long long)ci * H + y] = __float_as_int(acc + kMagic) - kMagicBits;
  if (bad && status) atomicOr(status, SB_STATUS_RANGE);
}

// out[n]: the column pass of column pt_col[n] at row pt_y[n] (exact wrapping int32
// box sums of R, weighted in fp32 in box order as the sweeps do)
__global__ void __launch_bounds__(128) filter_at_points_kernel(const int* __restrict__ R, int H,
                                                               const int* __restrict__ pt_col,
                                                               const int* __restrict__ pt_y, long long npts,
                                                               float* __restrict__ out, Taps t) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= npts) return;
  const int* rc = R + (long long)pt_col[n] * H;
  const int y = pt_y[n];
  uint32_t box[SB_MAX_K];
#pragma unroll
  for (int i = 0; i < SB_MAX_K; ++i) box[i] = 0;
  for (int d = -t.pmax; d <= t.pmax; ++d) {
    const uint32_t v = (uint32_t)rc[min(max(y + d, 0), H - 1)];
    const int ad = d < 0 ? -d : d;
#pragma unroll
    for (int i = 0; i < SB_MAX_K; ++i)
      if (i < t.k && ad <= t.p[i]) box[i] += v;
  }
  float acc = 0.0f;
#pragma unroll
  for (int i = 0; i < SB_MAX_K; ++i)
    if (i < t.k) acc = fmaf(t.w_col[i], i2f_fast(box[i]), acc);
  out[n] = acc;
}

int launch_filter_at(const void* src, int src_dtype, long long row_stride, int H, int W, const int* cols, int ncols,
                     const int* pt_col, const int* pt_y, long long npts, float* out, int* R, const Taps& t, int* status,
                     cudaStream_t st) {
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
