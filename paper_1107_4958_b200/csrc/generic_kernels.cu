// generic_kernels.cu - the two-pass filter for every kernel the reference accepts.
//
// The reference filters any image whose extents exceed the largest slice radius
// (filtering.py:39-45) with any number of slices (approx.py:82-102).  The sweep
// kernels (sweep_kernels.cuh) keep their halos and rings on chip, which bounds the
// radius and k (k <= FAST_K); these kernels have no such bound:
//
//   rows_generic_kernel   one CTA per row: the row's exact int32 prefix I (input
//                         quantum, wrapping) in shared memory (or, for rows longer
//                         than kGenericSmemBytes, in a per-CTA global scratch row),
//                         then out[x] = sum_i w_i (hi_i - lo_i) with the reference's
//                         boundary terms (filtering.py:57-62):
//                           hi = I[min(x+p, n-1)] + max(x+p-n+1, 0) * f[n-1]
//                           lo = x-p-1 < 0 ? (x-p) * f[0] : I[x-p-1]
//                         rounded to the mid quantum (int32 plane) or, for the row
//                         pass alone, written as float;
//   col_prefix_kernel     the running column prefix C of the int32 plane, in place;
//   cols_generic_kernel   out[y] = sum_i w_col_i (C-box of rows y-p_i .. y+p_i), the
//                         same boundary terms along the column.
//
// Every box sum is the same exact integer the sweep kernels form, and the weighted
// sums run in the same fp32 order (fmaf in slice order from 0), so the results are
// bit-identical to the sweep kernels' (tests/test_gpu_parity.py forces both paths).
//
// A = int (the sweep kernels' int32 quanta) or long long ("wide"): for 2*pmax+1 >
// kWideSpan the int32 box-sum limit would coarsen the quantum past the 1e-3 bar, so the
// host picks quanta for int64 sums (make_taps) and the plane holds int64 values.
#include <algorithm>

#include "sweep_kernels.cuh"

namespace sb {

constexpr int GT = 256;    // threads of the generic row / column kernels
constexpr int GITEMS = 8;  // elements per thread and scan step

// Box sum of slice radius p at position x of a length-n sequence with inclusive prefix
// I (exact modulo 2^32; the true value fits int32 by the quantum choice), first / last
// elements f0 / fl.  Unsigned arithmetic: the boundary products may wrap.
template <typename U, typename IdxFn>
__device__ __forceinline__ U box_sum(IdxFn I, int x, int p, int n, U f0, U fl) {
  SB_ASSERT(x >= 0 && x < n && p >= 0 && p < n);
  const long long xh = (long long)x + p;
  const U hi = xh < n ? (U)I((int)xh) : (U)I(n - 1) + (U)(xh - n + 1) * fl;
  const long long xl = (long long)x - p - 1;
  const U lo = xl >= 0 ? (U)I((int)xl) : (U)(long long)(x - p) * f0;
  return hi - lo;
}

template <typename A>
struct Acc;
template <>
struct Acc<int> {
  using U = uint32_t;
  static __device__ __forceinline__ float to_f32(U v) { return i2f_fast(v); }
};
template <>
struct Acc<long long> {
  using U = unsigned long long;
  static __device__ __forceinline__ float to_f32(U v) { return __ll2float_rn((long long)v); }
};

template <typename A>
__device__ __forceinline__ A warp_incl_scan_a(A x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const A y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

template <typename Tin, bool TO_MID, typename A>
__global__ void __launch_bounds__(GT) rows_generic_kernel(const Tin* __restrict__ src, A* __restrict__ mid_out,
                                                          float* __restrict__ dst, Geometry g,
                                                          const __grid_constant__ TapsG t,
                                                          A* __restrict__ scratch, int use_smem, int* status) {
  using U = typename Acc<A>::U;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ A wsum[GT / 32];
  A* S = use_smem ? (A*)smem_raw : scratch + (long long)blockIdx.x * g.W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long nrows = (long long)g.nimg * g.H * g.in_px;  // (image, row, channel)
  RangeAcc bad;
  for (long long r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int ch = (int)(r % g.in_px);
    const long long ir = r / g.in_px;
    const int img = (int)(ir / g.H), y = (int)(ir - (long long)img * g.H);
    const Tin* row = src + (long long)img * g.in_img + (long long)y * g.in_row + ch;
    // 1) inclusive prefix of the fixed-point row, GT*GITEMS elements per step
    A carry = 0;
    for (int base = 0; base < g.W; base += GT * GITEMS) {
      const int x0 = base + threadIdx.x * GITEMS;
      A v[GITEMS];
      A tot = 0;
#pragma unroll
      for (int m = 0; m < GITEMS; ++m) {
        const int x = x0 + m;
        if (x < g.W) tot += to_fixed<Tin>(row[(long long)x * g.in_px], t, bad);
        v[m] = tot;
      }
      const A inc = warp_incl_scan_a(tot);
      if (lane == 31) wsum[warp] = inc;
      __syncthreads();
      if (warp == 0) {
        A w = lane < GT / 32 ? wsum[lane] : 0;
        w = warp_incl_scan_a(w);
        if (lane < GT / 32) wsum[lane] = w;
      }
      __syncthreads();
      const A excl = carry + inc - tot + (warp > 0 ? wsum[warp - 1] : 0);
#pragma unroll
      for (int m = 0; m < GITEMS; ++m)
        if (x0 + m < g.W) S[x0 + m] = v[m] + excl;
      carry += wsum[GT / 32 - 1];
      __syncthreads();  // S complete for this step, wsum free for the next
    }
    // 2) the weighted box sums of every column of the row
    const U f0 = (U)S[0];
    const U fl = g.W > 1 ? (U)S[g.W - 1] - (U)S[g.W - 2] : f0;
    auto I = [&](int i) { return S[i]; };
    for (int x = threadIdx.x; x < g.W; x += GT) {
      float acc = 0.0f;
      for (int i = 0; i < t.k; ++i)
        acc = fmaf(TO_MID ? t.w_row[i] : t.w_out1[i], Acc<A>::to_f32(box_sum<U>(I, x, t.p[i], g.W, f0, fl)), acc);
      if constexpr (TO_MID) {
        mid_out[ch * g.mid_ch + (long long)img * g.mid_img + (long long)y * g.mid_row + x] =
            (A)(__float_as_int(__fadd_rn(acc, kMagic)) - kMagicBits);  // _rn: never contracted (k = 1)
      } else {
        dst[(long long)img * g.out_img + (long long)y * g.out_row + (long long)x * g.out_px + ch] = acc;
      }
    }
    __syncthreads();  // S is rewritten by the next row
  }
  report_status(status, bad, t);
}

// Running column prefix of the int32 plane [channel][image][H][W], in place (wrapping).
template <typename A>
__global__ void __launch_bounds__(128) col_prefix_kernel(A* __restrict__ mid, Geometry g) {
  using U = typename Acc<A>::U;
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long ncols = (long long)g.W * g.nimg * g.in_px;
  if (q >= ncols) return;
  const int x = (int)(q % g.W);
  const long long rest = q / g.W;
  const int img = (int)(rest % g.nimg), ch = (int)(rest / g.nimg);
  A* p = mid + ch * g.mid_ch + (long long)img * g.mid_img + x;
  const long long rs = g.mid_row;
  U run = 0;
  int y = 0;
  for (; y + 8 <= g.H; y += 8) {
    U v[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) v[m] = (U)p[(long long)(y + m) * rs];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      run += v[m];
      p[(long long)(y + m) * rs] = (A)run;
    }
  }
  for (; y < g.H; ++y) {
    run += (U)p[(long long)y * rs];
    p[(long long)y * rs] = (A)run;
  }
}

// Output rows [oy0, oy1) of every image and channel from the column prefix plane.
template <typename A>
__global__ void __launch_bounds__(GT) cols_generic_kernel(const A* __restrict__ C, float* __restrict__ dst,
                                                          Geometry g, const __grid_constant__ TapsG t) {
  using U = typename Acc<A>::U;
  const int wh = g.oy1 - g.oy0;
  const long long total = (long long)g.W * wh * g.nimg * g.in_px;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(e % g.W);
    long long rest = e / g.W;
    const int yo = (int)(rest % wh);
    rest /= wh;
    const int img = (int)(rest % g.nimg), ch = (int)(rest / g.nimg);
    const A* col = C + ch * g.mid_ch + (long long)img * g.mid_img + x;
    const long long rs = g.mid_row;
    auto I = [&](int v) { return __ldg(col + (long long)v * rs); };
    const U f0 = (U)I(0);
    const U fl = g.H > 1 ? (U)I(g.H - 1) - (U)I(g.H - 2) : f0;
    const int y = g.oy0 + yo;
    float acc = 0.0f;
    for (int i = 0; i < t.k; ++i)
      acc = fmaf(t.w_col[i], Acc<A>::to_f32(box_sum<U>(I, y, t.p[i], g.H, f0, fl)), acc);
    dst[(long long)img * g.out_img + (long long)yo * g.out_row + (long long)x * g.out_px + ch] = acc;
  }
}

size_t generic_rows_scratch_bytes(int W, bool wide) {
  const size_t es = wide ? sizeof(long long) : sizeof(int);
  return (size_t)W * es <= kGenericSmemBytes ? 0 : (size_t)kGenericScratchRows * (size_t)W * es;
}

template <typename Tin, typename A>
static int launch_rows_generic_t(const Tin* src, A* mid_out, float* dst, const Geometry& g, const TapsG& t,
                                 A* scratch, int* status, int sms, cudaStream_t st) {
  const size_t row_bytes = (size_t)g.W * sizeof(A);
  const bool use_smem = row_bytes <= kGenericSmemBytes;
  const size_t smem = use_smem ? row_bytes : 0;
  const long long nrows = (long long)g.nimg * g.H * g.in_px;
  const int per_sm = use_smem ? (int)std::max<size_t>(1, std::min<size_t>(8, (220 * 1024) / (smem + 1024))) : 2;
  long long grid = std::min<long long>(nrows, (long long)sms * per_sm);
  if (!use_smem) grid = std::min<long long>(grid, kGenericScratchRows);
  if (mid_out) {
    auto fn = rows_generic_kernel<Tin, true, A>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fn<<<(unsigned)grid, GT, smem, st>>>(src, mid_out, dst, g, t, scratch, use_smem ? 1 : 0, status);
  } else {
    auto fn = rows_generic_kernel<Tin, false, A>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fn<<<(unsigned)grid, GT, smem, st>>>(src, mid_out, dst, g, t, scratch, use_smem ? 1 : 0, status);
  }
  return (int)cudaGetLastError();
}

template <typename A>
static int rows_generic_dispatch(const void* src, int src_dtype, A* mid_out, float* dst, const Geometry& g,
                                 const TapsG& t, A* scratch, int* status, int sms, cudaStream_t st) {
  switch (src_dtype) {
    case SB_DTYPE_U8:
      return launch_rows_generic_t((const uint8_t*)src, mid_out, dst, g, t, scratch, status, sms, st);
    case SB_DTYPE_U16:
      return launch_rows_generic_t((const uint16_t*)src, mid_out, dst, g, t, scratch, status, sms, st);
    case SB_DTYPE_F32:
      return launch_rows_generic_t((const float*)src, mid_out, dst, g, t, scratch, status, sms, st);
    default:
      return launch_rows_generic_t((const double*)src, mid_out, dst, g, t, scratch, status, sms, st);
  }
}

int launch_rows_generic(const void* src, int src_dtype, void* mid_out, float* dst, const Geometry& g,
                        const TapsG& t, void* scratch, bool wide, int* status, int sms, cudaStream_t st) {
  if (wide)
    return rows_generic_dispatch<long long>(src, src_dtype, (long long*)mid_out, dst, g, t, (long long*)scratch,
                                            status, sms, st);
  return rows_generic_dispatch<int>(src, src_dtype, (int*)mid_out, dst, g, t, (int*)scratch, status, sms, st);
}

template <typename A>
static int launch_cols_generic_t(A* mid, float* dst, const Geometry& g, const TapsG& t, int sms, cudaStream_t st) {
  const long long ncols = (long long)g.W * g.nimg * g.in_px;
  col_prefix_kernel<A><<<(unsigned)((ncols + 127) / 128), 128, 0, st>>>(mid, g);
  const long long total = (long long)g.W * (g.oy1 - g.oy0) * g.nimg * g.in_px;
  const long long grid = std::max<long long>(1, std::min<long long>((total + GT - 1) / GT, (long long)sms * 16));
  cols_generic_kernel<A><<<(unsigned)grid, GT, 0, st>>>(mid, dst, g, t);
  return (int)cudaGetLastError();
}

int launch_cols_generic(void* mid, float* dst, const Geometry& g, const TapsG& t, bool wide, int sms,
                        cudaStream_t st) {
  if (wide) return launch_cols_generic_t<long long>((long long*)mid, dst, g, t, sms, st);
  return launch_cols_generic_t<int>((int*)mid, dst, g, t, sms, st);
}

}  // namespace sb
