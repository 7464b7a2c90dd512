// quality.cu - the accuracy harness of the reference (oracle.py:58-102) on the
// GPU: the dense, truncated, separable Gaussian with replicate boundary
// (`exact_gaussian_2d`) and the squared-difference sum behind `mse` / `psnr`.
// Not the hot path: it exists so the quality of the running-sum approximation
// can be measured at BASELINE sizes in milliseconds instead of minutes.
//
// The dense passes follow the reference's numpy order exactly - for each
// output, out += taps[j] * f(x + j - r) for j = 0, 1, ..., 2r with a separate
// fp64 multiply and add (no FMA contraction), rows first, then columns - so the
// result is bit-identical to exact_gaussian_2d.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "sliceblur_b200.h"

namespace sb {
namespace {

constexpr int GQ = 8;  // outputs per thread along the tap direction

template <typename Tin>
__device__ __forceinline__ double as_f64(Tin v) {
  return (double)v;
}

// rows: thread -> GQ consecutive x of row y; every loaded pixel feeds up to GQ outputs
template <typename Tin>
__global__ void __launch_bounds__(128) gauss_rows_kernel(const Tin* __restrict__ src, long long row_stride, int H,
                                                         int W, const double* __restrict__ taps, int r,
                                                         double* __restrict__ mid) {
  const int y = blockIdx.y;
  const int x0 = (blockIdx.x * blockDim.x + threadIdx.x) * GQ;
  if (y >= H || x0 >= W) return;
  const Tin* row = src + (long long)y * row_stride;
  double o[GQ];
#pragma unroll
  for (int i = 0; i < GQ; ++i) o[i] = 0.0;
  const int nt = 2 * r + 1;
  for (int m = 0; m < nt + GQ - 1; ++m) {
    const double v = as_f64(row[min(max(x0 + m - r, 0), W - 1)]);
#pragma unroll
    for (int i = 0; i < GQ; ++i) {
      const int j = m - i;
      if (j >= 0 && j < nt) o[i] = __dadd_rn(o[i], __dmul_rn(taps[j], v));
    }
  }
  double* out = mid + (long long)y * W;
#pragma unroll
  for (int i = 0; i < GQ; ++i)
    if (x0 + i < W) out[x0 + i] = o[i];
}

// columns: thread -> column x (coalesced) and GQ consecutive rows
__global__ void __launch_bounds__(128) gauss_cols_kernel(const double* __restrict__ mid, int H, int W,
                                                         const double* __restrict__ taps, int r,
                                                         double* __restrict__ dst, long long dst_row) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y0 = blockIdx.y * GQ;
  if (x >= W || y0 >= H) return;
  double o[GQ];
#pragma unroll
  for (int i = 0; i < GQ; ++i) o[i] = 0.0;
  const int nt = 2 * r + 1;
  for (int m = 0; m < nt + GQ - 1; ++m) {
    const double v = mid[(long long)min(max(y0 + m - r, 0), H - 1) * W + x];
#pragma unroll
    for (int i = 0; i < GQ; ++i) {
      const int j = m - i;
      if (j >= 0 && j < nt) o[i] = __dadd_rn(o[i], __dmul_rn(taps[j], v));
    }
  }
#pragma unroll
  for (int i = 0; i < GQ; ++i)
    if (y0 + i < H) dst[(long long)(y0 + i) * dst_row + x] = o[i];
}

template <typename Ta, typename Tb>
__global__ void __launch_bounds__(256) sum_sq_diff_kernel(const Ta* __restrict__ a, const Tb* __restrict__ b,
                                                          long long n, double* out) {
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double d = (double)a[i] - (double)b[i];
    s += d * d;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  __shared__ double part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
    atomicAdd(out, t);
  }
}

template <typename Ta>
int launch_ssd(const Ta* a, const void* b, int b_dtype, long long n, double* out, cudaStream_t st) {
  const int grid = (int)std::min<long long>((n + 255) / 256, 148 * 8);
  if (b_dtype == SB_DTYPE_F32)
    sum_sq_diff_kernel<Ta, float><<<grid, 256, 0, st>>>(a, (const float*)b, n, out);
  else
    sum_sq_diff_kernel<Ta, double><<<grid, 256, 0, st>>>(a, (const double*)b, n, out);
  return (int)cudaGetLastError();
}

}  // namespace
}  // namespace sb

extern "C" {

size_t sb_exact_gaussian_workspace_bytes(int64_t height, int64_t width) {
  if (height < 1 || width < 1) return 0;
  return (size_t)height * (size_t)width * sizeof(double);
}

int sb_exact_gaussian_2d(const void* src, int src_dtype, int64_t height, int64_t width, int64_t src_row_stride,
                         const double* taps_dev, int ntaps, double* dst, void* workspace, size_t workspace_bytes,
                         void* stream) {
  if (!src || !taps_dev || !dst || height < 1 || width < 1 || height > 0x7fffffffLL || width > 0x7fffffffLL ||
      src_row_stride < width || ntaps < 1 || (ntaps & 1) == 0)
    return SB_ERR_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < sb_exact_gaussian_workspace_bytes(height, width)) return SB_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  const int H = (int)height, W = (int)width, r = ntaps / 2;
  double* mid = (double*)workspace;
  const dim3 g1((unsigned)((W + 128 * sb::GQ - 1) / (128 * sb::GQ)), (unsigned)H);
  switch (src_dtype) {
    case SB_DTYPE_U8:
      sb::gauss_rows_kernel<uint8_t><<<g1, 128, 0, st>>>((const uint8_t*)src, src_row_stride, H, W, taps_dev, r, mid);
      break;
    case SB_DTYPE_U16:
      sb::gauss_rows_kernel<uint16_t><<<g1, 128, 0, st>>>((const uint16_t*)src, src_row_stride, H, W, taps_dev, r, mid);
      break;
    case SB_DTYPE_F32:
      sb::gauss_rows_kernel<float><<<g1, 128, 0, st>>>((const float*)src, src_row_stride, H, W, taps_dev, r, mid);
      break;
    case SB_DTYPE_F64:
      sb::gauss_rows_kernel<double><<<g1, 128, 0, st>>>((const double*)src, src_row_stride, H, W, taps_dev, r, mid);
      break;
    default: return SB_ERR_INVALID_ARGUMENT;
  }
  const dim3 g2((unsigned)((W + 127) / 128), (unsigned)((H + sb::GQ - 1) / sb::GQ));
  sb::gauss_cols_kernel<<<g2, 128, 0, st>>>(mid, H, W, taps_dev, r, dst, W);
  return cudaGetLastError() == cudaSuccess ? SB_OK : SB_ERR_CUDA;
}

int sb_sum_sq_diff(const void* a, int a_dtype, const void* b, int b_dtype, int64_t n, double* out_dev, void* stream) {
  if (!a || !b || !out_dev || n < 1) return SB_ERR_INVALID_ARGUMENT;
  if ((a_dtype != SB_DTYPE_F32 && a_dtype != SB_DTYPE_F64) || (b_dtype != SB_DTYPE_F32 && b_dtype != SB_DTYPE_F64))
    return SB_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  const int e = a_dtype == SB_DTYPE_F32 ? sb::launch_ssd((const float*)a, b, b_dtype, n, out_dev, st)
                                        : sb::launch_ssd((const double*)a, b, b_dtype, n, out_dev, st);
  return e == 0 ? SB_OK : SB_ERR_CUDA;
}

}  // extern "C"
