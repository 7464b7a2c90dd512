// aux_kernels.cu - the non-2D siblings of the hot path.
//
//   sb_prefix_sum_f64 <- filtering.py:31-36 prefix_sum (inclusive float64 cumsum)
//   sb_max_abs        -> value_bound for the fixed-point quantum (host wrapper)
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "sliceblur_b200.h"

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kTile = kScanThreads * kScanItems;


__device__ __forceinline__ double warp_inclusive_scan(double x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Block-wide inclusive scan of one value per thread; returns the inclusive value.
__device__ double block_inclusive_scan(double x, double* warp_totals) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  x = warp_inclusive_scan(x);
  if (lane == 31) warp_totals[warp] = x;
  __syncthreads();
  if (warp == 0) {
    double w = (lane < (int)(blockDim.x >> 5)) ? warp_totals[lane] : 0.0;
    w = warp_inclusive_scan(w);
    if (lane < (int)(blockDim.x >> 5)) warp_totals[lane] = w;
  }
  __syncthreads();
  if (warp > 0) x += warp_totals[warp - 1];
  __syncthreads();
  return x;
}

__global__ void tile_sums(const double* __restrict__ src, long long n, double* __restrict__ sums) {
  __shared__ double wt[32];
  const long long base = (long long)blockIdx.x * kTile + (long long)threadIdx.x * kScanItems;
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) s += src[base + i];
  double inc = block_inclusive_scan(s, wt);
  if (threadIdx.x == blockDim.x - 1) sums[blockIdx.x] = inc;
}

// Exclusive scan of the tile sums, one block walking the array sequentially.
__global__ void scan_tile_sums(double* sums, long long ntiles) {
  __shared__ double wt[32];
  double carry = 0.0;
  for (long long base = 0; base < ntiles; base += blockDim.x) {
    long long i = base + threadIdx.x;
    double v = (i < ntiles) ? sums[i] : 0.0;
    double inc = block_inclusive_scan(v, wt);
    if (i < ntiles) sums[i] = carry + inc - v;
    __shared__ double last;
    if (threadIdx.x == blockDim.x - 1) last = inc;
    __syncthreads();
    carry += last;
    __syncthreads();
  }
}

__global__ void tile_scan(const double* __restrict__ src, double* __restrict__ dst, long long n,
                          const double* __restrict__ offsets) {
  __shared__ double wt[32];
  const long long base = (long long)blockIdx.x * kTile + (long long)threadIdx.x * kScanItems;
  double v[kScanItems];
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? src[base + i] : 0.0;
    s += v[i];
  }
  double inc = block_inclusive_scan(s, wt);
  double run = offsets[blockIdx.x] + (inc - s);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    run += v[i];
    if (base + i < n) dst[base + i] = run;
  }
}

template <typename T>
__global__ void max_abs_kernel(const T* __restrict__ src, long long n, unsigned long long* out) {
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double a = fabs((double)src[i]);
    m = (a > m || a != a) ? a : m;  // keep NaN
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double y = __shfl_down_sync(0xffffffffu, m, o);
    m = (y > m || y != y) ? y : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

}  // namespace

extern "C" {

size_t sb_prefix_sum_workspace_bytes(int64_t n) {
  if (n < 1) return 0;
  return (size_t)((n + kTile - 1) / kTile) * sizeof(double);
}

int sb_prefix_sum_f64(const double* src, double* dst, int64_t n, void* workspace, size_t workspace_bytes,
                      void* stream) {
  if (!src || !dst || n < 1) return 1;  // SB_ERR_INVALID_ARGUMENT
  const long long ntiles = (n + kTile - 1) / kTile;
  if (!workspace || workspace_bytes < sb_prefix_sum_workspace_bytes(n)) return SB_ERR_WORKSPACE;
  if (ntiles > 0x7fffffffLL) return SB_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  double* sums = (double*)workspace;
  tile_sums<<<(unsigned)ntiles, kScanThreads, 0, st>>>(src, n, sums);
  scan_tile_sums<<<1, 1024, 0, st>>>(sums, ntiles);
  tile_scan<<<(unsigned)ntiles, kScanThreads, 0, st>>>(src, dst, n, sums);
  return cudaGetLastError() == cudaSuccess ? SB_OK : SB_ERR_CUDA;
}

int sb_max_abs(const void* src, int src_dtype, int64_t n, double* out_dev, void* stream) {
  if (!src || !out_dev || n < 1) return SB_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* out = (unsigned long long*)out_dev;
  if (cudaMemsetAsync(out, 0, sizeof(double), st) != cudaSuccess) return SB_ERR_CUDA;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long want = (n + 255) / 256;
  unsigned blocks = (unsigned)(want < (long long)sms * 8 ? want : (long long)sms * 8);
  switch (src_dtype) {
    case SB_DTYPE_U8: max_abs_kernel<uint8_t><<<blocks, 256, 0, st>>>((const uint8_t*)src, n, out); break;
    case SB_DTYPE_U16: max_abs_kernel<uint16_t><<<blocks, 256, 0, st>>>((const uint16_t*)src, n, out); break;
    case SB_DTYPE_F32: max_abs_kernel<float><<<blocks, 256, 0, st>>>((const float*)src, n, out); break;
    case SB_DTYPE_F64: max_abs_kernel<double><<<blocks, 256, 0, st>>>((const double*)src, n, out); break;
    default: return SB_ERR_INVALID_ARGUMENT;
  }
  return cudaGetLastError() == cudaSuccess ? SB_OK : SB_ERR_CUDA;
}

}  // extern "C"
