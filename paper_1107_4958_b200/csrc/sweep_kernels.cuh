// sweep_kernels.cuh - sm_100a kernels of the running-sum Gaussian filter.
//
// Reference arithmetic (filtering.py:48-64, `_filter_rows`):
//     out[x] = sum_i w_i * (I(x + p_i) - I(x - p_i - 1))
// with I the inclusive prefix sum and replicate (clamp) boundaries realised on
// I (filtering.py:10-13), i.e. out[x] = sum_i w_i * sum_{|t|<=p_i} f(clamp(x+t)).
// separable_filter_2d (filtering.py:76-104) runs it over rows, then columns.
//
// B200 formulation (DESIGN.md has the derivation and the error bound):
//   * every value entering a running sum is an int32 fixed-point number, so
//     box sums are EXACT (two's-complement wraparound keeps prefix differences
//     exact even when a prefix overflows);
//   * a CTA (128 threads) owns a strip of WS=128 columns of the (batch x H)
//     "tall" image and walks down a contiguous range of its rows;
//   * pass 1 (rows), per band of HB=16 rows: the input segment
//     [xb, xb+L) (xb = x0-pmax-1 rounded down to 16 px) is staged with
//     cp.async into a double buffer one band ahead; edge strips replicate the
//     border columns in place; each staged row is prefix-scanned by a warp
//     (16-px chunks per lane, shuffle scan of chunk totals).  For uint8 input
//     with small radii two rows share one 32-bit word (15-bit modular prefix
//     fields, guard bits 15/31), halving the lagged shared-memory reads;
//     thread c then forms R = sum_i w_i (P[c+p_i] - P[c-p_i-1]) rounded to the
//     mid quantum (fp32 magic-number rounding, no F2I);
//   * pass 2 (columns), fused: R goes to a shared-memory ring of D rows whose
//     first HB rows are mirrored after the end, so every HB-row window of any
//     lag is contiguous (immediate offsets, no wrap arithmetic); thread c keeps
//     k exact int32 box sums, B_i += R[y+p_i] - R[y-p_i-1], and writes
//     sum_i (w_i 2^-s_mid) float(B_i);
//   * large radii (ring does not fit): RowsToMid writes the int32 R plane,
//     ColsFromMid runs the column sweep reading lagged rows from L2/HBM.
//
// Vertical replicate boundary: R of a virtual row v outside [0,H) is R of row
// clamp(v) (the reference's column pass clamps the row-filtered image), so
// the sweep stages clamped input rows.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "sliceblur_b200.h"

namespace sb {

constexpr int HB = 16;          // rows per band
constexpr int WS = 128;         // strip width = threads per CTA
constexpr int NWARPS = WS / 32;
constexpr int CH = 16;          // px per scan chunk (one lane)
constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23: x + kMagic rounds x to an integer (|x| < 2^22)
constexpr int kMagicBits = 0x4B400000;  // bits(kMagic + n) = kMagicBits + n
constexpr uint32_t kGuard = 0x80008000u;
constexpr uint32_t kField = 0x7FFF7FFFu;

struct Geometry {
  long long in_img, in_row;    // source strides (elements)
  int in_px;                   // source pixel stride (= channels)
  int es;                      // source element size (bytes)
  long long out_img, out_row;  // destination strides (elements)
  int out_px;
  long long mid_img, mid_row;  // int32 workspace strides (two-pass only)
  long long mid_ch;            // int32 workspace channel-plane stride
  int H, W, nimg;
  int aligned16;               // rows are 16-byte aligned: cp.async 16 B staging
};

struct Taps {
  int k, pmax;
  int p[SB_MAX_K];
  float w_row[SB_MAX_K];   // w_i * 2^(s_mid - s_in): pass 1 output in mid quanta
  float w_col[SB_MAX_K];   // w_i * 2^-s_mid: pass 2 output in pixel units
  float w_out1[SB_MAX_K];  // w_i * 2^-s_in: pass 1 output in pixel units (row-only mode)
  float in_scale;          // 2^s_in (float sources)
  float in_limit;          // |x| * in_scale must be < in_limit (2^22)
};

struct Tiling {
  int L;                // staged / prefix row length in px (multiple of 16)
  int xoff;             // x0 - xb (same for every strip)
  int stage_row_bytes;  // bytes per staged row (multiple of 16)
  int lanes_per_row;    // power of two >= L / CH, <= 32
  int D;                // ring rows (the ring holds D + HB rows incl. the mirror)
  int nstrips;          // ceil(W / WS)
  long long rows_per_item;
  int packed;           // uint8 two-rows-per-word prefix
};

enum class Mode : int { Fused = 0, RowsToMid = 1, RowsToOut = 2, ColsFromMid = 3 };

// ---------------------------------------------------------------- small helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void st_stream(float* p, float v) {
  asm volatile("st.global.cs.f32 [%0], %1;\n" ::"l"(p), "f"(v));
}

template <typename T>
struct SrcTraits;
template <>
struct SrcTraits<uint8_t> {
  static constexpr bool kFloat = false;
};
template <>
struct SrcTraits<uint16_t> {
  static constexpr bool kFloat = false;
};
template <>
struct SrcTraits<float> {
  static constexpr bool kFloat = true;
};
template <>
struct SrcTraits<double> {
  static constexpr bool kFloat = true;
};

// fixed-point value of one source element; `bad` collects range violations
template <typename T>
__device__ __forceinline__ int to_fixed(T v, const Taps& t, bool& bad) {
  if constexpr (SrcTraits<T>::kFloat) {
    float s = (float)v * t.in_scale;
    bool ok = fabsf(s) < t.in_limit;  // false for NaN too
    bad |= !ok;
    s = ok ? s : 0.0f;
    return __float_as_int(s + kMagic) - kMagicBits;  // round-to-nearest-even of v * 2^s_in
  } else {
    return (int)v;
  }
}

// ---------------------------------------------------------------- pass 1: staging
// Issue the copies of virtual rows v0..v0+n-1 (clamped to the image) of the
// strip segment [xb, xb+L) into `buf` (row r at buf + r*stage_row_bytes).
template <typename Tin>
__device__ __forceinline__ void issue_stage(unsigned char* buf, const Tin* __restrict__ src_img, const Geometry& g,
                                            const Tiling& tl, int xb, int v0, int n) {
  const int rowbytes_img = g.W * g.in_px * g.es;
  const int lo = max(xb, 0) * g.in_px * g.es;
  const int hi = min(xb + tl.L, g.W) * g.in_px * g.es;
  const int base = xb * g.in_px * g.es;  // byte of column xb (may be negative)
  if (g.aligned16) {
    const int lo16 = lo;                 // multiple of 16 (xb is a multiple of 16 px)
    const int hi16 = hi & ~15;
    const int nchunk = (hi16 - lo16) >> 4;
    for (int idx = threadIdx.x; idx < n * nchunk; idx += WS) {
      const int r = idx / nchunk, q = idx - r * nchunk;
      const int v = min(max(v0 + r, 0), g.H - 1);
      const unsigned char* grow = (const unsigned char*)(src_img + (long long)v * g.in_row);
      cp_async16(buf + r * tl.stage_row_bytes + (lo16 + 16 * q - base), grow + lo16 + 16 * q);
    }
    cp_async_commit();
    if (hi16 < hi) {  // unaligned tail of the last strip (row bytes not a multiple of 16)
      const int tail = hi - hi16;
      for (int idx = threadIdx.x; idx < n * tail; idx += WS) {
        const int r = idx / tail, q = idx - r * tail;
        const int v = min(max(v0 + r, 0), g.H - 1);
        const unsigned char* grow = (const unsigned char*)(src_img + (long long)v * g.in_row);
        buf[r * tl.stage_row_bytes + (hi16 + q - base)] = grow[hi16 + q];
      }
    }
    (void)rowbytes_img;
  } else {
    // generic path: element copies (any stride / alignment)
    const int nel = (hi - lo) / g.es;
    for (int idx = threadIdx.x; idx < n * nel; idx += WS) {
      const int r = idx / nel, q = idx - r * nel;
      const int v = min(max(v0 + r, 0), g.H - 1);
      const Tin* grow = src_img + (long long)v * g.in_row;
      const int eoff = lo / g.es + q;
      *(Tin*)(buf + r * tl.stage_row_bytes + eoff * g.es - base) = grow[eoff];
    }
  }
}

// Replicate the border column into staged positions outside [0, W).
__device__ __forceinline__ void fixup_edges(unsigned char* buf, const Geometry& g, const Tiling& tl, int xb, int n) {
  const int pxb = g.in_px * g.es;
  const int left = max(0, -xb);                  // positions [0, left) <- column 0
  const int right0 = max(0, g.W - xb);           // positions [right0, L) <- column W-1
  const int nright = max(0, tl.L - right0);
  const int per_row = (left + nright) * pxb;
  for (int idx = threadIdx.x; idx < n * per_row; idx += WS) {
    const int r = idx / per_row;
    int q = idx - r * per_row;
    const int pos = q / pxb, byte = q - pos * pxb;
    unsigned char* row = buf + r * tl.stage_row_bytes;
    if (pos < left) {
      row[pos * pxb + byte] = row[left * pxb + byte];
    } else {
      const int dst = right0 + (pos - left);
      row[dst * pxb + byte] = row[(right0 - 1) * pxb + byte];
    }
  }
}

// ---------------------------------------------------------------- pass 1: prefix scans
// Inclusive modular int32 prefix of `n` staged rows, channel `ch`, into P[r][j].
template <typename Tin>
__device__ __forceinline__ void scan_rows(const unsigned char* buf, int* __restrict__ P, const Geometry& g,
                                          const Taps& t, const Tiling& tl, int ch, int n, int* status) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lpr = tl.lanes_per_row;
  const int rows_per_warp = 32 / lpr;
  const int sub = lane / lpr, sl = lane - sub * lpr;
  const int nchunk = tl.L / CH;
  bool bad = false;
  for (int r0 = warp * rows_per_warp; r0 < n; r0 += NWARPS * rows_per_warp) {
    const int r = r0 + sub;
    int running = 0;  // prefix of the chunk groups already done (rows longer than lpr chunks)
    for (int cg = 0; cg < nchunk; cg += lpr) {
      const int chunk = cg + sl;
      const bool live = (r < n) && (chunk < nchunk);
      int v[CH];
      int tot = 0;
      if (live) {
        const unsigned char* row = buf + r * tl.stage_row_bytes;
        if (g.in_px == 1 && sizeof(Tin) * CH % 16 == 0) {
          const uint4* p4 = (const uint4*)(row + chunk * CH * sizeof(Tin));
          Tin e[CH];
#pragma unroll
          for (int m = 0; m < (int)(sizeof(Tin) * CH / 16); ++m) *(uint4*)((unsigned char*)e + 16 * m) = p4[m];
#pragma unroll
          for (int m = 0; m < CH; ++m) {
            tot += to_fixed<Tin>(e[m], t, bad);
            v[m] = tot;
          }
        } else {
          const Tin* e = (const Tin*)row;
#pragma unroll
          for (int m = 0; m < CH; ++m) {
            tot += to_fixed<Tin>(e[(chunk * CH + m) * g.in_px + ch], t, bad);
            v[m] = tot;
          }
        }
      }
      // inclusive scan of chunk totals across the lpr lanes of this row
      int inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        if (o >= lpr) break;
        int y = __shfl_up_sync(0xffffffffu, inc, o, lpr);
        if (sl >= o) inc += y;
      }
      const int carry = running + inc - tot;
      if (live) {
        int4* dst = (int4*)(P + r * tl.L + chunk * CH);
#pragma unroll
        for (int m = 0; m < CH / 4; ++m)
          dst[m] = make_int4(v[4 * m] + carry, v[4 * m + 1] + carry, v[4 * m + 2] + carry, v[4 * m + 3] + carry);
      }
      running += __shfl_sync(0xffffffffu, inc, lpr - 1, lpr);
    }
  }
  if (bad && status) atomicOr(status, SB_STATUS_RANGE);
}

// uint8, one channel: rows q and q+8 of the band share P word q (15-bit fields).
__device__ __forceinline__ void scan_rows_packed(const unsigned char* buf, uint32_t* __restrict__ P,
                                                 const Tiling& tl) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lpr = tl.lanes_per_row;
  const int pairs_per_warp = 32 / lpr;
  const int sub = lane / lpr, sl = lane - sub * lpr;
  const int nchunk = tl.L / CH;
  for (int q0 = warp * pairs_per_warp; q0 < HB / 2; q0 += NWARPS * pairs_per_warp) {
    const int q = q0 + sub;
    const bool live = (q < HB / 2) && (sl < nchunk);
    uint32_t v[CH];
    uint32_t tot = 0;
    if (live) {
      const uint4 a = *(const uint4*)(buf + q * tl.stage_row_bytes + sl * CH);
      const uint4 b = *(const uint4*)(buf + (q + HB / 2) * tl.stage_row_bytes + sl * CH);
      const uint32_t aw[4] = {a.x, a.y, a.z, a.w};
      const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int m = 0; m < CH; ++m) {
        const uint32_t lo = __byte_perm(aw[m >> 2], 0u, 0x4440u | (m & 3));
        const uint32_t hi = __byte_perm(bw[m >> 2], 0u, 0x4044u | ((m & 3) << 8));
        tot = tot + lo + hi;  // < 16*255 per field: no carry between fields
        v[m] = tot;
      }
    }
    uint32_t inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      if (o >= lpr) break;
      uint32_t y = __shfl_up_sync(0xffffffffu, inc, o, lpr);
      if (sl >= o) inc = (inc + y) & kField;
    }
    const uint32_t carry = (inc + kGuard - tot) & kField;  // fieldwise (inc - tot) mod 2^15, no borrow
    if (live) {
      uint4* dst = (uint4*)(P + q * tl.L + sl * CH);
#pragma unroll
      for (int m = 0; m < CH / 4; ++m)
        dst[m] = make_uint4((v[4 * m] + carry) & kField, (v[4 * m + 1] + carry) & kField,
                            (v[4 * m + 2] + carry) & kField, (v[4 * m + 3] + carry) & kField);
    }
  }
}

// ---------------------------------------------------------------- pass 1: row values
// Row-filtered value of staged row r at strip column c (unpacked prefix), in
// mid quanta (magic-rounded) or, ROW_OUT, in pixel units.
template <int K, bool ROW_OUT>
__device__ __forceinline__ float row_value(const int* prow, int c, const Taps& t, const Tiling& tl) {
  float acc = 0.0f;
  const int base = c + tl.xoff;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int d = prow[base + t.p[i]] - prow[base - t.p[i] - 1];  // exact box sum
    acc = fmaf(ROW_OUT ? t.w_out1[i] : t.w_row[i], (float)d, acc);
  }
  return ROW_OUT ? acc : acc + kMagic;
}

// Rows q and q+8 of a packed band at column c, magic-rounded.
template <int K>
__device__ __forceinline__ void row_value_packed(const uint32_t* prow, int c, const Taps& t, const Tiling& tl,
                                                 float& lo_v, float& hi_v) {
  float a = 0.0f, b = 0.0f;
  const int base = c + tl.xoff;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const uint32_t d = prow[base + t.p[i]] + kGuard - prow[base - t.p[i] - 1];
    a = fmaf(t.w_row[i], (float)(d & 0x7FFFu), a);
    b = fmaf(t.w_row[i], (float)((d >> 16) & 0x7FFFu), b);
  }
  lo_v = a + kMagic;
  hi_v = b + kMagic;
}

// ---------------------------------------------------------------- the sweep kernel
// Grid: x = nstrips * items, y = channel.  Block: WS threads.
template <typename Tin, int K, Mode M>
__global__ void __launch_bounds__(WS) sweep_kernel(const Tin* __restrict__ src, const int* __restrict__ mid_in,
                                                   int* __restrict__ mid_out, float* __restrict__ dst, Geometry g,
                                                   Taps t, Tiling tl, int* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int strip = blockIdx.x % tl.nstrips;
  const long long item = blockIdx.x / tl.nstrips;
  const int ch = blockIdx.y;
  const int x0 = strip * WS;
  const int xb = x0 - tl.xoff;
  const int c = threadIdx.x;
  const bool active = (x0 + c) < g.W;
  const long long total = (long long)g.nimg * g.H;
  const long long T0 = item * tl.rows_per_item;
  const long long T1 = min(T0 + tl.rows_per_item, total);
  const bool edge = (xb < 0) || (xb + tl.L > g.W);
  const bool packed = (sizeof(Tin) == 1) && tl.packed;

  // shared-memory carve-up
  unsigned char* stage = smem;                                               // 2 x HB rows
  int* P = (int*)(smem + 2 * HB * tl.stage_row_bytes);                       // HB x L (or HB/2 x L packed)
  int* ring = (int*)(smem + (M == Mode::ColsFromMid ? 0 : 2 * HB * tl.stage_row_bytes + HB * tl.L * 4));
  const int D = tl.D;

  for (long long T = T0; T < T1;) {
    const int img = (int)(T / g.H);
    const int a = (int)(T - (long long)img * g.H);
    const int b = (int)min((long long)g.H, T1 - (long long)img * g.H);
    T = (long long)img * g.H + b;
    const Tin* src_img = src ? src + (long long)img * g.in_img : nullptr;

    if constexpr (M == Mode::ColsFromMid) {
      // Column sweep straight from the int32 R plane (large radii).
      if (!active) continue;
      const int* mcol = mid_in + ch * g.mid_ch + (long long)img * g.mid_img + x0 + c;
      auto R = [&](int v) { return mcol[(long long)min(max(v, 0), g.H - 1) * g.mid_row]; };
      int box[K];
#pragma unroll
      for (int i = 0; i < K; ++i) box[i] = 0;
      for (int u = -t.pmax; u <= t.pmax; ++u) {
        const int val = R(a - 1 + u);
        const int au = u < 0 ? -u : u;
#pragma unroll
        for (int i = 0; i < K; ++i)
          if (au <= t.p[i]) box[i] += val;
      }
      float* dcol = dst + (long long)img * g.out_img + (long long)(x0 + c) * g.out_px + ch;
      for (int y = a; y < b; ++y) {
        float acc = 0.0f;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          box[i] += R(y + t.p[i]) - R(y - t.p[i] - 1);
          acc = fmaf(t.w_col[i], (float)box[i], acc);
        }
        st_stream(dcol + (long long)y * g.out_row, acc);
      }
      continue;
    }

    // ---- pass-1 producer shared by all other modes
    // virtual rows to produce: [vstart, vstart + count)
    const int vstart = (M == Mode::Fused) ? a - 1 - t.pmax : a;
    const int count = (M == Mode::Fused) ? (b - a) + 2 * t.pmax + 1 : (b - a);
    const int nbands = (count + HB - 1) / HB;
    issue_stage<Tin>(stage, src_img, g, tl, xb, vstart, min(HB, count));

    int box[K];
    int lead_s[K], trail_s[K];
    int out_next = a;  // next output row (Fused)
#pragma unroll
    for (int i = 0; i < K; ++i) box[i] = 0;

    for (int pb = 0; pb < nbands; ++pb) {
      const int n = min(HB, count - pb * HB);
      unsigned char* cur = stage + (pb & 1) * HB * tl.stage_row_bytes;
      cp_async_wait_all();
      __syncthreads();  // staged band visible; everyone done with P and the other buffer
      if (pb + 1 < nbands)
        issue_stage<Tin>(stage + ((pb + 1) & 1) * HB * tl.stage_row_bytes, src_img, g, tl, xb,
                         vstart + (pb + 1) * HB, min(HB, count - (pb + 1) * HB));
      if (edge) {
        fixup_edges(cur, g, tl, xb, n);
        __syncthreads();
      }
      if (packed)
        scan_rows_packed(cur, (uint32_t*)P, tl);
      else
        scan_rows<Tin>(cur, P, g, t, tl, ch, n, status);
      __syncthreads();

      if constexpr (M == Mode::RowsToMid || M == Mode::RowsToOut) {
        if (active) {
          for (int r = 0; r < n; ++r) {
            const int v = vstart + pb * HB + r;
            if constexpr (M == Mode::RowsToMid) {
              float val = row_value<K, false>(P + r * tl.L, c, t, tl);
              mid_out[ch * g.mid_ch + (long long)img * g.mid_img + (long long)v * g.mid_row + x0 + c] =
                  __float_as_int(val) - kMagicBits;
            } else {
              float val = row_value<K, true>(P + r * tl.L, c, t, tl);
              dst[(long long)img * g.out_img + (long long)v * g.out_row + (long long)(x0 + c) * g.out_px + ch] = val;
            }
          }
        }
      } else {  // Fused
        // row values of this band -> ring (slot = offset mod D, mirrored below HB)
        const int off0 = pb * HB;
        if (active) {
          if (packed) {
#pragma unroll 2
            for (int q = 0; q < HB / 2; ++q) {
              float lo_v, hi_v;
              row_value_packed<K>((const uint32_t*)P + q * tl.L, c, t, tl, lo_v, hi_v);
              const int r2[2] = {q, q + HB / 2};
              const int bits[2] = {__float_as_int(lo_v) - kMagicBits, __float_as_int(hi_v) - kMagicBits};
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                if (r2[h] < n) {
                  const int s = (off0 + r2[h]) % D;
                  ring[s * WS + c] = bits[h];
                  if (s < HB) ring[(s + D) * WS + c] = bits[h];
                }
              }
            }
          } else {
            for (int r = 0; r < n; ++r) {
              const int bits = __float_as_int(row_value<K, false>(P + r * tl.L, c, t, tl)) - kMagicBits;
              const int s = (off0 + r) % D;
              ring[s * WS + c] = bits;
              if (s < HB) ring[(s + D) * WS + c] = bits;
            }
          }
        }
        const int produced = off0 + n;
        // box sums at row a-1 once rows a-1-pmax .. a-1+pmax (offsets 0..2pmax) exist
        if (active && produced >= 2 * t.pmax + 1 && produced - n < 2 * t.pmax + 1) {
          for (int u = 0; u <= 2 * t.pmax; ++u) {
            const int val = ring[(u % D) * WS + c];
            const int au = u > t.pmax ? u - t.pmax : t.pmax - u;
#pragma unroll
            for (int i = 0; i < K; ++i)
              if (au <= t.p[i]) box[i] += val;
          }
        }
        // emit every output band whose lead rows are in the ring
        while (out_next < b) {
          const int nb = min(HB, b - out_next);
          const int need = (out_next - a) + nb + 2 * t.pmax + 1;  // offsets required
          if (produced < need && produced < count) break;
          if (active) {
            const int ob = out_next - a;  // offset of output row out_next relative to a
#pragma unroll
            for (int i = 0; i < K; ++i) {
              lead_s[i] = (ob + t.pmax + 1 + t.p[i]) % D;   // row out_next + p_i
              trail_s[i] = (ob + t.pmax - t.p[i]) % D;      // row out_next - p_i - 1
            }
            float* dcol = dst + (long long)img * g.out_img + (long long)out_next * g.out_row +
                          (long long)(x0 + c) * g.out_px + ch;
            if (nb == HB) {
#pragma unroll
              for (int r = 0; r < HB; ++r) {
                float acc = 0.0f;
#pragma unroll
                for (int i = 0; i < K; ++i) {
                  box[i] += ring[(lead_s[i] + r) * WS + c] - ring[(trail_s[i] + r) * WS + c];
                  acc = fmaf(t.w_col[i], (float)box[i], acc);
                }
                st_stream(dcol + (long long)r * g.out_row, acc);
              }
            } else {
              for (int r = 0; r < nb; ++r) {
                float acc = 0.0f;
#pragma unroll
                for (int i = 0; i < K; ++i) {
                  box[i] += ring[(lead_s[i] + r) * WS + c] - ring[(trail_s[i] + r) * WS + c];
                  acc = fmaf(t.w_col[i], (float)box[i], acc);
                }
                st_stream(dcol + (long long)r * g.out_row, acc);
              }
            }
          }
          out_next += nb;
        }
      }
    }
    __syncthreads();  // P / stage reuse by the next segment
  }
}

}  // namespace sb
