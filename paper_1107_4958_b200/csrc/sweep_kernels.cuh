// sweep_kernels.cuh - sm_100a kernels of the running-sum Gaussian filter.
//
// Reference arithmetic (filtering.py:48-64, `_filter_rows`):
//     out[x] = sum_i w_i * (I(x + p_i) - I(x - p_i - 1))
// with I the inclusive prefix sum and replicate (clamp) boundaries realised on
// I (filtering.py:10-13), i.e. out[x] = sum_i w_i * sum_{|t|<=p_i} f(clamp(x+t)).
// separable_filter_2d (filtering.py:76-104) runs it over rows, then columns.
//
// B200 formulation (see DESIGN.md for the derivation and error bound):
//   * every value that enters a running sum is an int32 fixed-point number, so
//     box sums are EXACT (two's-complement wraparound makes prefix
//     differences exact even when the prefix itself overflows);
//   * pass 1 (rows): a CTA owns a strip of Ws columns and walks down a range of
//     rows.  For each band of HB rows it stages the input segment
//     [x0-pmax-1, x0+Ws+pmax) with replicate-clamped columns into shared
//     memory as fixed point, prefix-scans each staged row in place (warp
//     shuffles), and thread c forms
//         R = sum_i w_i * (P[c+pmax+1+p_i] - P[c+pmax-p_i])
//     rounded to the mid quantum (fp32 magic-number rounding, no F2I);
//   * pass 2 (columns), fused: R lands in a shared-memory ring (rows on the
//     slow axis, double-mapped so every HB-row window is contiguous) and thread
//     c keeps k exact int32 running box sums, B_i += R[y+p_i] - R[y-p_i-1];
//     the pixel is sum_i (w_i 2^-s_mid) * float(B_i).
//   * large radii (ring does not fit) use two launches: RowsToMid writes the
//     int32 R plane to a workspace, ColsFromMid runs the same column sweep
//     reading lagged rows straight from L2/HBM.
//
// Vertical replicate boundary: R of a virtual row v outside [0,H) is the R of
// row clamp(v) (the column pass of the reference clamps the row-filtered
// image), so the sweep simply stages clamped input rows.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "sliceblur_b200.h"

namespace sb {

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: x + kMagic rounds x to an integer (|x| < 2^22)
constexpr int kMagicBits = 0x4B400000;  // bit pattern of kMagic; bits(kMagic + n) = kMagicBits + n

struct Geometry {
  long long in_img, in_row;   // source strides (elements)
  int in_px;                  // source pixel stride (= channels)
  long long out_img, out_row; // destination strides (elements)
  int out_px;
  long long mid_img, mid_row; // int32 workspace strides (two-pass only)
  int H, W, nimg;
};

struct Taps {
  int k, pmax;
  int p[SB_MAX_K];
  float w_row[SB_MAX_K];  // w_i * 2^(s_mid - s_in): pass 1 output in mid quanta
  float w_col[SB_MAX_K];  // w_i * 2^-s_mid: pass 2 output in pixel units
  float w_out1[SB_MAX_K]; // w_i * 2^-s_in: pass 1 output in pixel units (row-only mode)
  float in_scale;         // 2^s_in (float sources)
  float in_limit;         // |x| * in_scale must be < in_limit (2^22)
};

struct Tiling {
  int Ws;                 // strip width = threads per CTA
  int L;                  // staged row length (Ws + 2 pmax + 1, padded to a multiple of 4)
  int D;                  // ring depth in rows (HB + 2 pmax + 1)
  int nstrips;            // ceil(W / Ws)
  long long rows_per_item;  // rows of the (batch x H) tall image swept per CTA
};

enum class Mode : int { Fused = 0, RowsToMid = 1, RowsToOut = 2, ColsFromMid = 3 };

// ---------------------------------------------------------------- loads
template <typename T>
__device__ __forceinline__ int to_fixed(T v, const Taps& t, int* status);

template <>
__device__ __forceinline__ int to_fixed<uint8_t>(uint8_t v, const Taps&, int*) { return (int)v; }
template <>
__device__ __forceinline__ int to_fixed<uint16_t>(uint16_t v, const Taps&, int*) { return (int)v; }
template <>
__device__ __forceinline__ int to_fixed<float>(float v, const Taps& t, int* status) {
  float s = v * t.in_scale;
  // NaN fails the comparison too, so non-finite input is reported.
  if (!(fabsf(s) < t.in_limit)) {
    if (status) atomicOr(status, SB_STATUS_RANGE);
    s = 0.0f;
  }
  return __float_as_int(s + kMagic) - kMagicBits;  // round-to-nearest-even of v * 2^s_in
}
template <>
__device__ __forceinline__ int to_fixed<double>(double v, const Taps& t, int* status) {
  double s = v * (double)t.in_scale;
  if (!(fabs(s) < (double)t.in_limit)) {
    if (status) atomicOr(status, SB_STATUS_RANGE);
    s = 0.0;
  }
  return __double2int_rn(s);
}

// ---------------------------------------------------------------- pass 1 pieces
// Stage rows v0..v0+n-1 (image-local, clamped) of strip x0 into stage[r][j],
// j <-> column x0 - pmax - 1 + j (clamped to [0, W)).
template <typename Tin>
__device__ __forceinline__ void stage_rows(const Tin* __restrict__ src_img, const Geometry& g, const Taps& t,
                                           const Tiling& tl, int* stage, int x0, int v0, int n, int* status) {
  const int span = tl.Ws + 2 * t.pmax + 1;
  const int xbase = x0 - t.pmax - 1;
  for (int r = 0; r < n; ++r) {
    int v = min(max(v0 + r, 0), g.H - 1);
    const Tin* row = src_img + (long long)v * g.in_row;
    int* dstrow = stage + r * tl.L;
    for (int j = threadIdx.x; j < span; j += blockDim.x) {
      int x = min(max(xbase + j, 0), g.W - 1);
      dstrow[j] = to_fixed<Tin>(row[(long long)x * g.in_px], t, status);
    }
  }
}

// In-place inclusive prefix scan of each staged row (int32, wraparound).
__device__ __forceinline__ void scan_rows(int* stage, const Tiling& tl, int span, int n) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  for (int r = warp; r < n; r += nwarps) {
    int* row = stage + r * tl.L;
    int carry = 0;
    for (int base = 0; base < span; base += 32) {
      int j = base + lane;
      int x = (j < span) ? row[j] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      x += carry;
      if (j < span) row[j] = x;
      carry = __shfl_sync(0xffffffffu, x, 31);
    }
  }
}

// R of staged row r for column c, in fixed-point quanta as magic-float bits,
// or (ROW_OUT) in pixel units.
template <int K, bool ROW_OUT>
__device__ __forceinline__ float row_value(const int* prow, int c, const Taps& t) {
  float acc = 0.0f;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    int d = prow[c + t.pmax + 1 + t.p[i]] - prow[c + t.pmax - t.p[i]];  // exact box sum
    acc = fmaf(ROW_OUT ? t.w_out1[i] : t.w_row[i], (float)d, acc);
  }
  return ROW_OUT ? acc : acc + kMagic;  // magic add = round to the mid quantum
}

// ---------------------------------------------------------------- the sweep kernel
// Grid: x = nstrips * items, y = channel.  Block: Ws threads.
template <typename Tin, int K, Mode M>
__global__ void __launch_bounds__(256) sweep_kernel(const Tin* __restrict__ src, const int* __restrict__ mid_in,
                                                    int* __restrict__ mid_out, float* __restrict__ dst, Geometry g,
                                                    Taps t, Tiling tl, int* status) {
  extern __shared__ __align__(16) int smem[];
  constexpr int HB = 16;
  const int strip = blockIdx.x % tl.nstrips;
  const long long item = blockIdx.x / tl.nstrips;
  const int ch = blockIdx.y;
  const int x0 = strip * tl.Ws;
  const int c = threadIdx.x;
  const bool active = (x0 + c) < g.W;
  const long long total = (long long)g.nimg * g.H;
  const long long T0 = item * tl.rows_per_item;
  const long long T1 = min(T0 + tl.rows_per_item, total);
  const int span = tl.Ws + 2 * t.pmax + 1;

  int* stage = smem;                        // HB x L (pass 1 modes)
  int* ring = smem + (M == Mode::ColsFromMid ? 0 : HB * tl.L);  // 2D x Ws (column modes)
  const int D = tl.D;

  for (long long T = T0; T < T1;) {
    const int img = (int)(T / g.H);
    const int a = (int)(T - (long long)img * g.H);
    const int b = (int)min((long long)g.H, T1 - (long long)img * g.H);
    T = (long long)img * g.H + b;
    const Tin* src_img = src ? src + (long long)img * g.in_img + ch : nullptr;

    if constexpr (M == Mode::RowsToMid || M == Mode::RowsToOut) {
      for (int v0 = a; v0 < b; v0 += HB) {
        const int n = min(HB, b - v0);
        stage_rows<Tin>(src_img, g, t, tl, stage, x0, v0, n, status);
        __syncthreads();
        scan_rows(stage, tl, span, n);
        __syncthreads();
        if (active) {
          for (int r = 0; r < n; ++r) {
            float val = row_value<K, M == Mode::RowsToOut>(stage + r * tl.L, c, t);
            if constexpr (M == Mode::RowsToMid) {
              mid_out[(long long)img * g.mid_img + (long long)(v0 + r) * g.mid_row + x0 + c] =
                  __float_as_int(val) - kMagicBits;
            } else {
              dst[(long long)img * g.out_img + (long long)(v0 + r) * g.out_row + (long long)(x0 + c) * g.out_px +
                  ch] = val;
            }
          }
        }
        __syncthreads();
      }
    } else {
      // Column sweep over output rows [a, b) of image img.
      // Virtual row v is stored in ring slots s and s + D, s = (v - vbase) mod D.
      const int vbase = a - 1 - t.pmax;
      int produced = 0;  // rows [vbase, vbase + produced) are in the ring
      auto produce = [&](int n) {
        const int v0 = vbase + produced;
        if constexpr (M == Mode::Fused) {
          stage_rows<Tin>(src_img, g, t, tl, stage, x0, v0, n, status);
          __syncthreads();
          scan_rows(stage, tl, span, n);
          __syncthreads();
          if (active) {
            for (int r = 0; r < n; ++r) {
              int bits = __float_as_int(row_value<K, false>(stage + r * tl.L, c, t)) - kMagicBits;
              int s = (produced + r) % D;
              ring[s * tl.Ws + c] = bits;
              ring[(s + D) * tl.Ws + c] = bits;
            }
          }
          __syncthreads();
        } else {  // ColsFromMid
          if (active) {
            const int* mimg = mid_in + (long long)img * g.mid_img + x0 + c;
            for (int r = 0; r < n; ++r) {
              int v = min(max(v0 + r, 0), g.H - 1);
              int bits = mimg[(long long)v * g.mid_row];
              int s = (produced + r) % D;
              ring[s * tl.Ws + c] = bits;
              ring[(s + D) * tl.Ws + c] = bits;
            }
          }
          __syncthreads();
        }
        produced += n;
      };

      // warm-up: rows [a-1-pmax, a-1+pmax]
      for (int left = 2 * t.pmax + 1; left > 0;) {
        int n = min(HB, left);
        produce(n);
        left -= n;
      }
      int box[K];
      {
        // B_i(a-1) = sum_{|u|<=p_i} R(a-1+u); row a-1+u sits at ring offset pmax+u from vbase.
#pragma unroll
        for (int i = 0; i < K; ++i) box[i] = 0;
        if (active) {
          for (int u = -t.pmax; u <= t.pmax; ++u) {
            int val = ring[((t.pmax + u) % D) * tl.Ws + c];
            int au = u < 0 ? -u : u;
#pragma unroll
            for (int i = 0; i < K; ++i)
              if (au <= t.p[i]) box[i] += val;
          }
        }
      }
      float* dcol = dst + (long long)img * g.out_img + (long long)(x0 + c) * g.out_px + ch;
      for (int y0 = a; y0 < b; y0 += HB) {
        const int n = min(HB, b - y0);
        produce(n);  // rows up to y0 + n - 1 + pmax
        if (active) {
          // ring offsets (from vbase) of the lead/trail rows of output row y0:
          // lead_i = y0 + p_i - vbase, trail_i = y0 - p_i - 1 - vbase.
          int lead_s[K], trail_s[K];
#pragma unroll
          for (int i = 0; i < K; ++i) {
            lead_s[i] = (y0 + t.p[i] - vbase) % D;
            trail_s[i] = (y0 - t.p[i] - 1 - vbase) % D;
          }
          for (int r = 0; r < n; ++r) {
            float acc = 0.0f;
#pragma unroll
            for (int i = 0; i < K; ++i) {
              // double mapping: slot s + r < 2D is always a valid copy
              box[i] += ring[(lead_s[i] + r) * tl.Ws + c] - ring[(trail_s[i] + r) * tl.Ws + c];
              acc = fmaf(t.w_col[i], (float)box[i], acc);
            }
            dcol[(long long)(y0 + r) * g.out_row] = acc;
          }
        }
        __syncthreads();
      }
    }
  }
}

}  // namespace sb
