// sweep_kernels.cuh - sm_100a kernels of the running-sum Gaussian filter (shared header).
//
// Reference arithmetic (filtering.py:48-64, `_filter_rows`):
//     out[x] = sum_i w_i * (I(x + p_i) - I(x - p_i - 1))
// with I the inclusive prefix sum and replicate (clamp) boundaries realised on
// I (filtering.py:10-13), i.e. out[x] = sum_i w_i * sum_{|t|<=p_i} f(clamp(x+t)).
// separable_filter_2d (filtering.py:76-104) runs it over rows, then columns.
//
// B200 formulation (DESIGN.md "Arithmetic" has the derivation and the error bound):
//   * every value entering a running sum is an int32 fixed-point number, so box sums are
//     EXACT (two's-complement wraparound keeps prefix differences exact);
//   * the column pass keeps the running column PREFIX C of the rounded row values in a ring
//     in tensor memory (thread / column c <-> TMEM lane c, ring row <-> TMEM column, first
//     band mirrored after the end so every window is contiguous) and every output box sum is
//     C(y+p) - C(y-p-1): two tcgen05.ld windows, no running state;
//   * full output bands leave by TMA tensor stores.
//
// Kernels in this header (instantiated per source type in sweep_<dtype>.cu):
//   fused_kernel        one launch: producer warps stage (cp.async) and prefix-scan 16-row
//                       bands of a 128-column strip into shared memory, consumer warps form the
//                       row values, the TMEM column ring and the outputs (uint8: biased-fp32
//                       prefixes, IDP4A scans, FADD2/FFMA2 on row pairs, two bands per turn)
//                       (opt-in variants: three CTAs per SM, one band per turn, paired consumer
//                       warps - two warps per TMEM lane quadrant alternating bands)
//   stream_rows_kernel  two-launch row pass (float32): full-width 16-row bands streamed in
//                       128-column chunks (four staged chunks in flight per producer warp) with
//                       the row prefix carried in a ring -> int32 plane
//   stream_rows_mc_kernel  the same for 2..4 interleaved channels: bands of virtual (row,
//                       channel) rows, the band's image rows staged once by bulk copies
//   cols2_kernel        two-launch column pass: TMA loads of plane bands, loader warps append
//                       the column prefix to the TMEM ring, two output groups read windows;
//                       trails older than the ring come from shared-memory band copies;
//                       ring-only tilings use the split loader (two loader warps per quadrant)
//   cols_kernel         running-sum column pass (fallback when no tensor map fits)
//   rows_kernel         tiled row pass (other source types, row pass alone)
// and, in their own translation units: sweep_wide.cu (fusedw_kernel, one-launch float32 for
// large radii), sweep_rowtile.cu (rowtile_kernel, uint8 row pass on thread-per-row warps
// with the row prefix in TMEM), generic_kernels.cu (any radius / k, int64 when needed).
//
// Vertical replicate boundary: R of a virtual row v outside [0,H) is R of row clamp(v) (the
// reference's column pass clamps the row-filtered image), so the sweeps stage clamped rows.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#include "sliceblur_b200.h"

namespace sb {

constexpr int HB = 16;          // rows per band
constexpr int WS = 128;         // strip width = threads per CTA
constexpr int NWARPS = WS / 32;
constexpr int CH = 16;          // px per scan chunk (one lane)
constexpr int LS = 516;         // fused prefix row stride in words (compile-time offsets; 2064 B = 16 mod 128)
// float32 sources pick the smallest of these strides >= L (all 16 mod 128 bytes, so the
// 8-row phases of the prefix stores stay conflict-free): small radii then fit two CTAs' or
// one CTA's shared memory with the f32 staging (C1, C2)
constexpr int LS_SMALL = 196, LS_MID = 324;
constexpr int LMAX = 512;       // longest staged / prefix row of the fused sweep
constexpr int LSP2 = 194;       // uint8 float2-prefix row stride (L <= 192): 1552 B = 16 (mod 128), conflict-free
constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23: x + kMagic rounds x to an integer (|x| < 2^22)
constexpr int kMagicBits = 0x4B400000;  // bits(kMagic + n) = kMagicBits + n

struct Geometry {
  long long in_img, in_row;    // source strides (elements)
  int in_px;                   // source pixel stride (= channels)
  int es;                      // source element size (bytes)
  long long out_img, out_row;  // destination strides (elements)
  int out_px;
  long long mid_img, mid_row;  // int32 workspace strides (two-pass only)
  long long mid_ch;            // int32 workspace channel-plane stride
  int H, W, nimg;
  int oy0, oy1;                // output row window of every image (column sweeps write rows oy0..oy1-1)
  int aligned16;               // rows are 16-byte aligned: cp.async 16 B staging
  int out_bulk;                // one channel, 16-byte aligned rows: full output bands leave by TMA tensor stores
};

constexpr int FAST_K = 8;  // the templated sweep kernels take k <= FAST_K slices

struct Taps {
  int k, pmax;
  int p[FAST_K];
  float w_row[FAST_K];   // w_i * 2^(s_mid - s_in): pass 1 output in mid quanta
  float w_col[FAST_K];   // w_i * 2^-s_mid: pass 2 output in pixel units
  float w_out1[FAST_K];  // w_i * 2^-s_in: pass 1 output in pixel units (row-only mode)
  float in_scale;        // 2^s_in (float sources)
  float in_limit;        // float sources: |x| * in_scale <= in_limit (the caller's bound, scaled; < 2^22)
                         // uint16: x <= in_limit
  float seen_limit;      // float sources: |x| * in_scale >= seen_limit (half the bound) sets SB_STATUS_HALF
};

// The same quanta for any k <= SB_MAX_K (generic two-pass kernels, filter_at): passed by
// value (16 KB of kernel parameters, within the 32 KB sm_70+/CUDA 12.1 limit).
struct TapsG {
  int k, pmax;
  float in_scale, in_limit, seen_limit;
  int p[SB_MAX_K];
  float w_row[SB_MAX_K];
  float w_col[SB_MAX_K];
  float w_out1[SB_MAX_K];
};

struct Tiling {
  int L;                // staged / prefix row length in px (multiple of 16)
  int ls;               // prefix row stride in words (LS for the fused mode, >= L)
  int xoff;             // x0 - xb (same for every strip)
  int stage_row_bytes;  // bytes per staged row (multiple of 16)
  int lanes_per_row;    // power of two >= L / CH, <= 32
  int D;                // ring rows, a multiple of HB (the ring holds D + HB rows incl. the mirror)
  int nstrips;          // ceil(W / WS)
  long long rows_per_item;
  int packed;           // uint8 two-rows-per-word prefix
  int tmem_cols;        // tensor-memory columns allocated for the ring (power of two, >= D + HB)
  int sw;               // strip width in columns (WS for sweeps, wider for the row pass alone)
  int npb;              // fused: prefix buffers per producer warp (1 or 2)
  int obuf_off;         // fused: byte offset of the output staging bands in shared memory
  int pf;               // cols: plane bands prefetched ahead (2, 3, 4, 6 or 8)
  int ndeep;            // cols: largest boxes whose trails are re-read from the plane (0..SB_NDEEP)
  int ds;               // cols2: ring-band copies kept in shared memory (0 = none)
  int deepmask;         // cols2: bit i = box i's trail window is read from the copies
  int lag;              // cols2: ring band v is written once output band v - lag is done
  int copy_e;           // cols2: band v - D/HB + copy_e is copied out of the ring while band v is written
  int split;            // fused: 3 = three-CTA-per-SM variant (fused_kernel<uint8_t, K, 3>)
  int nsb;              // fused: staged bands per producer warp (1 or 2; the output box is buffered alike)
  int s0;               // row-tile: first scanned staged column (multiple of 4)
  int ta;               // row-tile: TMEM columns of the row-prefix region (the ring follows)
};

enum class Mode : int { Fused = 0, RowsToMid = 1, RowsToOut = 2, ColsFromMid = 3, ColsPrefix = 4 };

// ---------------------------------------------------------------- checked build
// SB_CHECKED (tools/build_checked.py): device-side bounds traps at the shared-memory / TMEM
// indexing points, and a pseudo-random sleep (0-1 us, from %globaltimer) at every hand-off
// (mbarrier arrive / wait, named barrier, bulk-store wait) so each run interleaves the
// producer, consumer and TMA traffic differently; tools/checked_run.py then requires
// bit-identical results across runs and agreement with the oracle.  compute-sanitizer is
// closed on this pool, so this is the race / bounds check.
#ifdef SB_CHECKED
__device__ __forceinline__ void sb_perturb() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  uint32_t h = (uint32_t)t * 2654435761u ^ (threadIdx.x * 40503u) ^ (blockIdx.x * 2246822519u);
  h ^= h >> 15;
  h *= 2246822519u;
  h ^= h >> 13;
  if ((h & 3) == 0) __nanosleep((h >> 8) & 1023);
}
#define SB_ASSERT(c)                                                                                      \
  do {                                                                                                    \
    if (!(c)) {                                                                                           \
      printf("SB_ASSERT %s failed at %s:%d block %d thread %d\n", #c, __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x);                                                                           \
      __trap();                                                                                           \
    }                                                                                                     \
  } while (0)
#else
__device__ __forceinline__ void sb_perturb() {}
#define SB_ASSERT(c) \
  do {               \
  } while (0)
#endif

// ---------------------------------------------------------------- small helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
// R-plane loads: keep the line in L2 (its row is re-read as a deep trail 2*pmax+1 rows later)
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ int ld_keep(const int* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_stream(float* p, float v) {
  asm volatile("st.global.cs.f32 [%0], %1;\n" ::"l"(p), "f"(v));
}
// ---- TMA tensor stores from shared memory (async proxy)
// 32-bit word store at (global address base) + 4 * idx: one IMAD.WIDE per address
__device__ __forceinline__ void st_global_idx(size_t base, int idx, int v) {
  asm volatile("{\n\t.reg .u64 a;\n\tmad.wide.s32 a, %1, 4, %0;\n\tst.global.b32 [a], %2;\n\t}" ::"l"(base), "r"(idx),
               "r"(v)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* ssrc, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"(smem_u32(ssrc)), "r"(x), "r"(y), "r"(z)
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* sdst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(sdst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// bulk copy global -> shared (bytes and both addresses multiples of 16), completion on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
  sb_perturb();
}

// ---- tensor memory (tcgen05): the fused column ring.  Thread c of the CTA owns
// TMEM lane c (warp w reaches lanes 32w..32w+31); ring slot s is TMEM column s.
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}

// ---- mbarriers (producer/consumer hand-off inside a CTA)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  sb_perturb();
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p "
      "bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
  sb_perturb();
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait with exponential back-off sleep: for warps that usually run ahead (producers),
// so their polling does not take issue slots from the warps they wait for.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  unsigned ns = 32;
  while (!mbar_test(bar, parity)) {
    __nanosleep(ns);
    ns = ns < 1024 ? 2 * ns : ns;
  }
  sb_perturb();
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  sb_perturb();
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// int32 -> fp32 through the full-rate I2FP.F32.S32 path: the inline cvt hides the
// operand's range, so the compiler cannot pick the slow I2F.U16 form for 16-bit values.
__device__ __forceinline__ float i2f_fast(uint32_t x) {
  float f;
  asm("cvt.rn.f32.s32 %0, %1;" : "=f"(f) : "r"(x));
  return f;
}

// Rounding of packed row values to the mid quantum (x + 1.5*2^23) as its own rounding step on
// every path.  ptxas 12.9 contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 despite the explicit
// rounding modifiers, so a one-slice kernel (a single FMUL2 before the add) would round once
// where the scalar paths round twice: for K = 1 the add is done on the halves (add.rn.f32 is
// honoured); for K >= 2 the preceding op is already an FFMA2 and nothing can be contracted.
template <int K>
__device__ __forceinline__ float2 round_mid2(float2 a) {
  if constexpr (K == 1)
    return make_float2(__fadd_rn(a.x, 12582912.0f), __fadd_rn(a.y, 12582912.0f));
  else
    return __fadd2_rn(a, make_float2(12582912.0f, 12582912.0f));
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

// Range of the source elements a thread converted: the NaN-propagating max |x| of float
// sources (one FMNMX per element), turned into status bits once per thread by
// report_status; uint16 sources set SB_STATUS_RANGE directly.
struct RangeAcc {
  float m = 0.0f;
  uint32_t st = 0;
};

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}

// fixed-point value of one source element: round(x * 2^s_in) by the magic-number FFMA
// (x * 2^s_in is exact, so this is the rounding of the exact product); an element past the
// caller's bound (or NaN / Inf) gives an unspecified value and is reported, never hidden
template <typename T, typename TT>
__device__ __forceinline__ int to_fixed(T v, const TT& t, RangeAcc& r) {
  if constexpr (SrcTraits<T>::kFloat) {
    const float f = (float)v;
    r.m = fmax_nan(r.m, fabsf(f));
    return __float_as_int(fmaf(f, t.in_scale, kMagic)) - kMagicBits;
  } else {
    if constexpr (sizeof(T) == 2) r.st |= (float)v > t.in_limit ? (uint32_t)SB_STATUS_RANGE : 0u;
    return (int)v;
  }
}

// OR a thread's status bits into the caller's word: SB_STATUS_RANGE (an element above the
// caller's bound, or not finite), SB_STATUS_HALF (one at least half the bound); one atomic
// per bit the word lacks (the HALF bit is seen by most threads of a typical image)
template <typename TT>
__device__ __forceinline__ void report_status(int* status, const RangeAcc& r, const TT& t) {
  if (!status) return;
  const float s = r.m * t.in_scale;  // exact (power of two); NaN stays NaN
  uint32_t st = r.st;
  st |= s <= t.in_limit ? 0u : (uint32_t)SB_STATUS_RANGE;
  st |= s >= t.seen_limit ? (uint32_t)SB_STATUS_HALF : 0u;
  if (!st) return;
  const uint32_t have = (uint32_t)*(volatile int*)status;
  if (st & ~have) atomicOr(status, (int)st);
}

// ---------------------------------------------------------------- pass 1: staging
// Issue the copies of virtual rows v0..v0+n-1 (clamped to the image) of the
// strip segment [xb, xb+L) into `buf` (row r at buf + r*stage_row_bytes).
// floor(a / d) for 0 <= a < 2^16 and 1 <= d < 2^15, with magic = 2^32 / d + 1 precomputed
__device__ __forceinline__ int fast_div(int a, uint32_t magic) { return (int)__umulhi((uint32_t)a, magic); }

// Staging by 4-byte asynchronous copies: rows that are 4-byte but not 16-byte multiples (a
// 1000-pixel-wide uint8 image).  64 x 1000^2 uint8: 0.43 ms with element copies, 0.165 ms with these.
__device__ __forceinline__ void issue_stage_words(unsigned char* buf, const unsigned char* src_img, long long row_bytes,
                                               int H, int srb, int base, int v0, int n, int lo, int nchunk,
                                               uint32_t chunk_magic, int hi4, int hi, int tid, int nthr) {
  for (int idx = tid; idx < n * nchunk; idx += nthr) {
    const int r = fast_div(idx, chunk_magic), q = idx - r * nchunk;
    const int v = min(max(v0 + r, 0), H - 1);
    const unsigned char* grow = src_img + (long long)v * row_bytes;
    cp_async4(buf + r * srb + (lo + 4 * q - base), grow + lo + 4 * q);
  }
  cp_async_commit();
  if (hi4 < hi) {  // tail bytes past the last whole word
    const int tail = hi - hi4;
    for (int r = 0; r < n; ++r) {
      const int v = min(max(v0 + r, 0), H - 1);
      const unsigned char* grow = src_img + (long long)v * row_bytes;
      for (int q = tid; q < tail; q += nthr) buf[r * srb + (hi4 + q - base)] = grow[hi4 + q];
    }
  }
}

template <typename Tin, bool A4 = false>
__device__ __forceinline__ void issue_stage(unsigned char* buf, const Tin* __restrict__ src_img, const Geometry& g,
                                            const Tiling& tl, int xb, int v0, int n, int lo, int nchunk,
                                            uint32_t chunk_magic, int hi16, int hi, int tid = threadIdx.x,
                                            int nthr = WS, int gran = -1) {
  const int base = xb * g.in_px * g.es;  // byte of column xb (may be negative)
  // gran: bytes per asynchronous copy (16, or 4 for rows that are only 4-byte multiples - a
  // 1000-pixel-wide uint8 image), 0 = element copies; nchunk / hi16 are in units of gran
  if (A4 && gran == 4) {
    // A4 kernels only: the 16-byte kernels (every BASELINE config) keep the code they had
    issue_stage_words(buf, (const unsigned char*)src_img, (long long)g.in_row * g.es, g.H, tl.stage_row_bytes, base, v0,
                      n, lo, nchunk, chunk_magic, hi16, hi, tid, nthr);
  } else if (A4 ? gran == 16 : g.aligned16) {
    for (int idx = tid; idx < n * nchunk; idx += nthr) {
      const int r = fast_div(idx, chunk_magic), q = idx - r * nchunk;
      const int v = min(max(v0 + r, 0), g.H - 1);
      const unsigned char* grow = (const unsigned char*)(src_img + (long long)v * g.in_row);
      SB_ASSERT(lo + 16 * q - base >= 0 && lo + 16 * q - base + 16 <= tl.stage_row_bytes && r < HB);
      cp_async16(buf + r * tl.stage_row_bytes + (lo + 16 * q - base), grow + lo + 16 * q);
    }
    cp_async_commit();
    if (hi16 < hi) {  // unaligned tail of the last strip (row bytes not a multiple of 16)
      const int tail = hi - hi16;
      for (int r = 0; r < n; ++r) {
        const int v = min(max(v0 + r, 0), g.H - 1);
        const unsigned char* grow = (const unsigned char*)(src_img + (long long)v * g.in_row);
        for (int q = tid; q < tail; q += nthr) buf[r * tl.stage_row_bytes + (hi16 + q - base)] = grow[hi16 + q];
      }
    }
  } else {
    // generic path: element copies (any stride / alignment)
    const int e0 = lo / g.es, e1 = hi / g.es;
    for (int r = 0; r < n; ++r) {
      const int v = min(max(v0 + r, 0), g.H - 1);
      const Tin* grow = src_img + (long long)v * g.in_row;
      for (int e = e0 + tid; e < e1; e += nthr) *(Tin*)(buf + r * tl.stage_row_bytes + e * g.es - base) = grow[e];
    }
  }
}

// Replicate the border column into staged positions outside [0, W).
__device__ __forceinline__ void fixup_edges(unsigned char* buf, const Geometry& g, const Tiling& tl, int xb, int n,
                                            int tid = threadIdx.x, int nthr = WS) {
  const int pxb = g.in_px * g.es;
  const int left = max(0, -xb);         // positions [0, left) <- column 0
  const int right0 = max(0, g.W - xb);  // positions [right0, L) <- column W-1
  const int lb = left * pxb;
  const int rb = max(0, tl.L - right0) * pxb;
  if (pxb == 1) {
    for (int r = 0; r < n; ++r) {
      unsigned char* row = buf + r * tl.stage_row_bytes;
      for (int q = tid; q < lb; q += nthr) row[q] = row[lb];
      for (int q = tid; q < rb; q += nthr) row[right0 + q] = row[right0 - 1];
    }
    return;
  }
  for (int r = 0; r < n; ++r) {
    unsigned char* row = buf + r * tl.stage_row_bytes;
    for (int q = tid; q < lb; q += nthr) row[q] = row[lb + (q % pxb)];
    for (int q = tid; q < rb; q += nthr) row[right0 * pxb + q] = row[(right0 - 1) * pxb + (q % pxb)];
  }
}

// ---------------------------------------------------------------- pass 1: prefix scans
// Inclusive modular int32 prefix of `n` staged rows, channel `ch`, into P[r][j].
template <typename Tin>
__device__ __forceinline__ void scan_rows(const unsigned char* buf, int* __restrict__ P, const Geometry& g,
                                          const Taps& t, const Tiling& tl, int ch, int n, int* status,
                                          int warp = threadIdx.x >> 5, int nwarps = NWARPS) {
  const int lane = threadIdx.x & 31;
  const int lpr = tl.lanes_per_row;
  const int rows_per_warp = 32 / lpr;
  const int sub = lane / lpr, sl = lane - sub * lpr;
  const int nchunk = tl.L / CH;
  RangeAcc bad;
  for (int r0 = warp * rows_per_warp; r0 < n; r0 += nwarps * rows_per_warp) {
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
        int4* dst = (int4*)(P + r * tl.ls + chunk * CH);
#pragma unroll
        for (int m = 0; m < CH / 4; ++m)
          dst[m] = make_int4(v[4 * m] + carry, v[4 * m + 1] + carry, v[4 * m + 2] + carry, v[4 * m + 3] + carry);
      }
      running += __shfl_sync(0xffffffffu, inc, lpr - 1, lpr);
    }
  }
  report_status(status, bad, t);
}

// The same scan for one warp over a whole band, bank-conflict free: lane (rr, cq)
// = (lane & 7, lane >> 3) takes chunk cg + cq of row r0 + rr, so each 8-lane
// phase of the 128-bit staging loads and prefix stores touches 8 rows of one
// chunk, which sit in 8 distinct bank groups (row strides are an odd multiple of
// 16 bytes); the row prefix of the chunk groups already done is carried in the
// row's 4 lanes.
template <typename Tin, int PLS = LS>
__device__ __forceinline__ void scan_band8(const unsigned char* buf, int* __restrict__ P, const Geometry& g,
                                           const Taps& t, const Tiling& tl, int ch, int n, int* status) {
  const int lane = threadIdx.x & 31;
  const int rr = lane & 7, cq = lane >> 3;
  const int nchunk = tl.L / CH;
  RangeAcc bad;
  for (int r0 = 0; r0 < n; r0 += 8) {
    const int r = r0 + rr;
    int running = 0;
    for (int cg = 0; cg < nchunk; cg += 4) {
      const int chunk = cg + cq;
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
      int inc = tot;
      int y = __shfl_up_sync(0xffffffffu, inc, 8);
      if (cq >= 1) inc += y;
      y = __shfl_up_sync(0xffffffffu, inc, 16);
      if (cq >= 2) inc += y;
      const int carry = running + inc - tot;
      if (live) {
        int4* dst = (int4*)(P + r * PLS + chunk * CH);
#pragma unroll
        for (int m = 0; m < CH / 4; ++m)
          dst[m] = make_int4(v[4 * m] + carry, v[4 * m + 1] + carry, v[4 * m + 2] + carry, v[4 * m + 3] + carry);
      }
      running += __shfl_sync(0xffffffffu, inc, rr + 24);
    }
  }
  report_status(status, bad, t);
}

// uint8, one channel, float prefixes: rows q and q+8 of the band share float2 q of
// P (x = row q, y = row q+8), stored as the fp32 numbers 2^23 + prefix.  For
// 0 <= v < 2^23 the bit pattern of 2^23 + v is 0x4B000000 + v, so the scan is
// integer: one IDP4A per pixel turns a word of four bytes into a prefix
// (dp4a(word, 0x00010101, base) = base + b0 + b1 + b2), and a box sum is one
// exact fp32 subtraction (FADD2 on a row pair) of two such values.
// Lane = seg * 8 + q scans columns [seg*4*NW, (seg+1)*4*NW) of rows q and q+8;
// the four segment offsets come from a two-step shuffle scan of packed 16-bit
// totals (<= 192*255 < 2^16).  Staging rows are an odd multiple of 16 bytes
// apart and P rows 1552 bytes, so each 8-lane phase of the 128-bit loads and
// stores touches 8 distinct bank groups.
template <int NW>
__device__ __forceinline__ void scan_rows_b2(const unsigned char* buf, float2* __restrict__ P, int srb) {
  const int lane = threadIdx.x & 31;
  const int q = lane & 7, seg = lane >> 3;
  const unsigned char* ra = buf + q * srb + seg * (4 * NW);
  const unsigned char* rb = ra + (HB / 2) * srb;
  uint32_t wa[NW], wb[NW];
#pragma unroll
  for (int j = 0; j < NW / 4; ++j) {
    const uint4 x = *(const uint4*)(ra + 16 * j);
    const uint4 y = *(const uint4*)(rb + 16 * j);
    wa[4 * j] = x.x, wa[4 * j + 1] = x.y, wa[4 * j + 2] = x.z, wa[4 * j + 3] = x.w;
    wb[4 * j] = y.x, wb[4 * j + 1] = y.y, wb[4 * j + 2] = y.z, wb[4 * j + 3] = y.w;
  }
  uint32_t ta = 0, tb = 0;
#pragma unroll
  for (int j = 0; j < NW; ++j) {
    ta = __dp4a(wa[j], 0x01010101u, ta);
    tb = __dp4a(wb[j], 0x01010101u, tb);
  }
  const uint32_t t = ta | (tb << 16);
  uint32_t inc = t;
  uint32_t y = __shfl_up_sync(0xffffffffu, inc, 8);
  if (seg >= 1) inc += y;
  y = __shfl_up_sync(0xffffffffu, inc, 16);
  if (seg >= 2) inc += y;
  const uint32_t ex = inc - t;
  uint32_t ba = 0x4B000000u + (ex & 0xFFFFu), bb = 0x4B000000u + (ex >> 16);
  float2* dst = P + q * LSP2 + seg * (4 * NW);
#pragma unroll
  for (int j = 0; j < NW; ++j) {
    const uint32_t a0 = __dp4a(wa[j], 0x00000001u, ba), b0 = __dp4a(wb[j], 0x00000001u, bb);
    const uint32_t a1 = __dp4a(wa[j], 0x00000101u, ba), b1 = __dp4a(wb[j], 0x00000101u, bb);
    const uint32_t a2 = __dp4a(wa[j], 0x00010101u, ba), b2 = __dp4a(wb[j], 0x00010101u, bb);
    ba = __dp4a(wa[j], 0x01010101u, ba);
    bb = __dp4a(wb[j], 0x01010101u, bb);
    float4* d4 = (float4*)(dst + 4 * j);
    d4[0] = make_float4(__uint_as_float(a0), __uint_as_float(b0), __uint_as_float(a1), __uint_as_float(b1));
    d4[1] = make_float4(__uint_as_float(a2), __uint_as_float(b2), __uint_as_float(ba), __uint_as_float(bb));
  }
}

__device__ __forceinline__ void scan_rows_b2_dispatch(const unsigned char* buf, float2* __restrict__ P,
                                                      const Tiling& tl) {
  switch (tl.L >> 6) {  // packed tilings have L a multiple of 64, at most 192
    case 1: scan_rows_b2<4>(buf, P, tl.stage_row_bytes); break;
    case 2: scan_rows_b2<8>(buf, P, tl.stage_row_bytes); break;
    default: scan_rows_b2<12>(buf, P, tl.stage_row_bytes); break;
  }
}

// ---------------------------------------------------------------- pass 1: row values
// Row-filtered values of the HB staged rows at strip column c, accumulated box by
// box so every shared-memory load is (lag pointer) + (row * L): the lag pointers
// are per-thread constants and the row offsets are uniform.
template <int K, int STRIDE>
__device__ __forceinline__ void band_rows(const int* __restrict__ P, int c, const float* __restrict__ w,
                                          const Taps& t, const Tiling& tl, float (&acc)[HB]) {
  const int ls = STRIDE ? STRIDE : tl.ls;  // compile-time stride -> immediate load offsets
#pragma unroll
  for (int r = 0; r < HB; ++r) acc[r] = 0.0f;
  const int base = c + tl.xoff;
  SB_ASSERT(base - t.p[K - 1] - 1 >= 0 && base + t.p[K - 1] < tl.L && tl.L <= ls);
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int* pl = P + base + t.p[i];
    const int* pt = P + base - t.p[i] - 1;
    const float wi = w[i];
#pragma unroll
    for (int r = 0; r < HB; ++r) acc[r] = fmaf(wi, (float)(pl[r * ls] - pt[r * ls]), acc[r]);  // exact box sum
  }
}

// Float-prefix uint8 variant: float2 q holds rows q (x) and q+8 (y); the box sum is
// an exact packed subtraction and the weighted sum one packed FFMA2 per box.
template <int K>
__device__ __forceinline__ void band_rows_f2(const float2* __restrict__ P, int c, const Taps& t, const Tiling& tl,
                                             float2 (&acc)[HB / 2]) {
  const int base = c + tl.xoff;
  SB_ASSERT(base - t.p[K - 1] - 1 >= 0 && base + t.p[K - 1] < tl.L && tl.L <= LSP2);
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const float2* pl = P + base + t.p[i];
    const float2* pt = P + base - t.p[i] - 1;
    const float2 w2 = make_float2(t.w_row[i], t.w_row[i]);
#pragma unroll
    for (int q = 0; q < HB / 2; ++q) {
      const float2 l = pl[q * LSP2], r = pt[q * LSP2];
      const float2 d = __fadd2_rn(l, make_float2(-r.x, -r.y));  // exact box sums of rows q, q+8
      acc[q] = i == 0 ? __fmul2_rn(w2, d) : __ffma2_rn(w2, d, acc[q]);
    }
  }
}

// Column pass over one output band from the TMEM ring, which holds the running
// column PREFIX C of the rounded row values (exact int32, wraps): the box sum of
// slice i at row y is C(y+p_i) - C(y-p_i-1), a difference of two 16-row windows
// (contiguous thanks to the mirrored first band), with no running state.
#ifndef SB_COL_GROUP
#define SB_COL_GROUP 2
#endif
template <int K>
__device__ __forceinline__ void column_band_tmem(uint32_t tlane, const int (&lead_s)[K], const int (&trail_s)[K],
                                                 const Taps& t, float (&out)[HB]) {
  float2 o2[HB / 2];
  // boxes in pairs: four window loads in flight per tcgen05.wait (latency, not bandwidth, bounds this)
#pragma unroll
  for (int i0 = 0; i0 < K; i0 += SB_COL_GROUP) {
    uint32_t lv[SB_COL_GROUP][HB], tv[SB_COL_GROUP][HB];
#pragma unroll
    for (int d = 0; d < SB_COL_GROUP; ++d)
      if (i0 + d < K) {
        tmem_ld16(tlane + (uint32_t)lead_s[i0 + d], lv[d]);
        tmem_ld16(tlane + (uint32_t)trail_s[i0 + d], tv[d]);
      }
    tmem_wait_ld();
#pragma unroll
    for (int d = 0; d < SB_COL_GROUP; ++d) {
      const int i = i0 + d;
      if (i >= K) break;
      const float2 w2 = make_float2(t.w_col[i], t.w_col[i]);
#pragma unroll
      for (int r = 0; r < HB / 2; ++r) {
        // exact box sums of rows 2r, 2r+1, weighted with one packed FFMA2
        const float2 dd = make_float2(i2f_fast(lv[d][2 * r] - tv[d][2 * r]), i2f_fast(lv[d][2 * r + 1] - tv[d][2 * r + 1]));
        o2[r] = i == 0 ? __fmul2_rn(w2, dd) : __ffma2_rn(w2, dd, o2[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < HB / 2; ++r) {
    out[2 * r] = o2[r].x;
    out[2 * r + 1] = o2[r].y;
  }
}

// ---------------------------------------------------------------- row pass alone
// RowsToMid (two-launch path for large radii: int32 R plane, magic-rounded to
// the mid quantum) and RowsToOut (slice_filter_1d / _filter_rows: float rows).
// A CTA owns a strip of tl.sw columns (a multiple of WS; wide strips keep the
// 2*pmax+1 halo small) and walks down a contiguous range of rows in bands of
// HB, staging with cp.async one band ahead.  Multi-channel (interleaved)
// sources gather only this CTA's channel (4-byte cp.async), so shared memory
// holds one channel.
template <typename Tin, int K, Mode M>
__global__ void __launch_bounds__(WS) rows_kernel(const Tin* __restrict__ src, int* __restrict__ mid_out,
                                                  float* __restrict__ dst, Geometry g, Taps t, Tiling tl,
                                                  int* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int strip = blockIdx.x % tl.nstrips;
  const long long item = blockIdx.x / tl.nstrips;
  const int ch = blockIdx.y;
  const int x0 = strip * tl.sw;
  const int xb = x0 - tl.xoff;
  const long long total = (long long)g.nimg * g.H;
  const long long T0 = item * tl.rows_per_item;
  const long long T1 = min(T0 + tl.rows_per_item, total);
  const bool edge = (xb < 0) || (xb + tl.L > g.W);
  // staged source layout: gather = one channel, contiguous; otherwise the raw interleaved bytes
  const bool gather = g.in_px > 1;
  Geometry gs = g;  // geometry of the staged buffer as the scan sees it
  if (gather) {
    gs.in_px = 1;
    gs.W = g.W;
  }
  const int st_lo = max(xb, 0) * g.in_px * g.es;
  const int st_hi = min(xb + tl.L, g.W) * g.in_px * g.es;
  const int st_hi16 = g.aligned16 ? (st_hi & ~15) : st_hi;
  const int st_nchunk = max(0, (st_hi16 - st_lo) >> 4);
  const uint32_t st_magic = 0xFFFFFFFFu / (uint32_t)max(1, st_nchunk) + 1u;
  unsigned char* stage = smem;
  int* P = (int*)(smem + 2 * HB * tl.stage_row_bytes);

  auto stage_band = [&](unsigned char* buf, const Tin* src_img, int v0, int n) {
    if (!gather) {
      issue_stage<Tin>(buf, src_img, g, tl, xb, v0, n, st_lo, st_nchunk, st_magic, st_hi16, st_hi);
      return;
    }
    const int e0 = max(xb, 0), e1 = min(xb + tl.L, g.W);
    const int cnt = e1 - e0;
    for (int r = 0; r < n; ++r) {
      const int v = min(max(v0 + r, 0), g.H - 1);
      const Tin* grow = src_img + (long long)v * g.in_row + ch;
      Tin* srow = (Tin*)(buf + r * tl.stage_row_bytes) + (e0 - xb);
      for (int e = threadIdx.x; e < cnt; e += WS) {
        if constexpr (sizeof(Tin) == 4) {
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(srow + e)),
                       "l"(grow + (long long)(e0 + e) * g.in_px));
        } else {
          srow[e] = grow[(long long)(e0 + e) * g.in_px];
        }
      }
    }
    cp_async_commit();
  };

  for (long long T = T0; T < T1;) {
    const int img = (int)(T / g.H);
    const int a = (int)(T - (long long)img * g.H);
    const int b = (int)min((long long)g.H, T1 - (long long)img * g.H);
    T = (long long)img * g.H + b;
    const Tin* src_img = src + (long long)img * g.in_img;
    const int count = b - a;
    const int nbands = (count + HB - 1) / HB;
    stage_band(stage, src_img, a, min(HB, count));
    for (int pb = 0; pb < nbands; ++pb) {
      const int n = min(HB, count - pb * HB);
      unsigned char* cur = stage + (pb & 1) * HB * tl.stage_row_bytes;
      cp_async_wait_all();
      __syncthreads();  // staged band visible; everyone done with P and the other buffer
      if (pb + 1 < nbands) stage_band(stage + ((pb + 1) & 1) * HB * tl.stage_row_bytes, src_img, a + (pb + 1) * HB,
                                      min(HB, count - (pb + 1) * HB));
      if (edge) {
        fixup_edges(cur, gs, tl, xb, n);
        __syncthreads();
      }
      scan_rows<Tin>(cur, P, gs, t, tl, gather ? 0 : ch, n, status);
      __syncthreads();
      const int v0 = a + pb * HB;
      for (int c = threadIdx.x; c < tl.sw; c += WS) {
        if (x0 + c >= g.W) break;
        float rv[HB];
        band_rows<K, 0>(P, c, M == Mode::RowsToOut ? t.w_out1 : t.w_row, t, tl, rv);
#pragma unroll
        for (int r = 0; r < HB; ++r) {
          if (r < n) {
            if constexpr (M == Mode::RowsToMid) {
              mid_out[ch * g.mid_ch + (long long)img * g.mid_img + (long long)(v0 + r) * g.mid_row + x0 + c] =
                  __float_as_int(__fadd_rn(rv[r], kMagic)) - kMagicBits;
            } else {
              dst[(long long)img * g.out_img + (long long)(v0 + r) * g.out_row + (long long)(x0 + c) * g.out_px + ch] =
                  rv[r];
            }
          }
        }
      }
    }
    __syncthreads();  // P / stage reuse by the next segment
  }
}

// ---------------------------------------------------------------- column pass from the int32 plane
// ColsFromMid (large radii): thread c <-> strip column c <-> TMEM lane c.  Each
// band of HB rows of the R plane is read once and appended to a TMEM ring of D
// rows (mirrored first band); the k running box sums read their lead/trail
// windows from the ring, except trails older than the ring (lag > D - HB),
// which are re-read from the plane.  All plane
// reads are cp.async copies of the thread's own column into shared-memory rings
// issued tl.pf bands ahead (one commit group per band), so HBM latency is hidden
// without registers and without CTA-wide barriers.
constexpr int SB_NDEEP = 4;  // deep-trail boxes prefetched through shared memory (the largest ones)

// cp.async.wait_group takes an immediate: the few prefetch depths the host picks
__device__ __forceinline__ void cp_async_wait_depth(int n) {
  switch (n) {
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    case 3: cp_async_wait<3>(); break;
    case 5: cp_async_wait<5>(); break;
    case 7: cp_async_wait<7>(); break;
    default: cp_async_wait<0>(); break;
  }
}

template <int K>
__global__ void __launch_bounds__(WS) cols_kernel(const int* __restrict__ mid_in, float* __restrict__ dst, Geometry g,
                                                  Taps t, Tiling tl) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t tmem_base_s;
  // channel varies fastest across CTAs: the channels of one pixel range run together and
  // share the interleaved lines in L2 (reads and partial-sector writes merge there)
  const int ch = blockIdx.x % g.in_px;
  const int sidx = blockIdx.x / g.in_px;
  const int strip = sidx % tl.nstrips;
  const long long item = sidx / tl.nstrips;
  const int x0 = strip * WS;
  const int c = threadIdx.x;
  const bool active = (x0 + c) < g.W;
  const int xc = active ? x0 + c : g.W - 1;  // inactive lanes mirror a valid column (no stores)
  const int wh = g.oy1 - g.oy0;  // rows of each image this launch outputs
  const long long total = (long long)g.nimg * wh;
  const long long T0 = item * tl.rows_per_item;
  const long long T1 = min(T0 + tl.rows_per_item, total);
  const int D = tl.D;
  const int PF = tl.pf;
  int* lring = (int*)smem;          // [PF][HB][WS] lead bands
  int* dring = lring + PF * HB * WS;  // [ndeep][PF][HB][WS] deep trail bands of boxes K-1, K-2, ...
  if (threadIdx.x < 32) tmem_alloc(&tmem_base_s, (uint32_t)tl.tmem_cols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tlane = tmem_base_s + ((uint32_t)(threadIdx.x & ~31) << 16);
  bool deep[K];
#pragma unroll
  for (int i = 0; i < K; ++i) deep[i] = (2 * HB + t.pmax + t.p[i]) > D;  // trail older than the ring

  for (long long T = T0; T < T1;) {
    const int img = (int)(T / wh);
    const int a = g.oy0 + (int)(T - (long long)img * wh);
    const int b = g.oy0 + (int)min((long long)wh, T1 - (long long)img * wh);
    T = (long long)img * wh + (b - g.oy0);
    const int* mcol = mid_in + ch * g.mid_ch + (long long)img * g.mid_img + xc;
    const long long mrow = g.mid_row;
    // 16 rows from plane row v0 into ring band `slot` (rows clamped at the image edges)
    auto fetch = [&](int* ring, int slot, int v0) {
      int* sp = ring + slot * (HB * WS) + c;
      if (v0 >= 0 && v0 + HB <= g.H) {
        const int* p = mcol + (long long)v0 * mrow;
#pragma unroll
        for (int r = 0; r < HB; ++r) {
          cp_async4(sp + r * WS, p);
          p += mrow;
        }
      } else {
#pragma unroll
        for (int r = 0; r < HB; ++r) cp_async4(sp + r * WS, mcol + (long long)min(max(v0 + r, 0), g.H - 1) * mrow);
      }
    };
    const int vstart = a - 1 - t.pmax;
    const int count = (b - a) + 2 * t.pmax + 1;
    const int nbands = (count + HB - 1) / HB;
    const int nout = (b - a + HB - 1) / HB;
    // output band ob is emitted at band iteration ob + W (full bands)
    const int W = (2 * t.pmax + 1 + HB + HB - 1) / HB - 1;
    int box[K];
#pragma unroll
    for (int i = 0; i < K; ++i) box[i] = 0;
    // ring slots of the lead / in-ring trail windows of the next output band, advanced by HB
    // per band with one conditional wrap (D is a multiple of HB)
    int lead_s[K], trail_s[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      lead_s[i] = (t.pmax + 1 + t.p[i]) % D;
      trail_s[i] = (t.pmax - t.p[i]) % D;
    }
    // one cp.async group per band iteration q: lead band q and the deep trails of output
    // band q - W, issued PF - 1 iterations ahead
    auto issue = [&](int q) {
      if (q < nbands) fetch(lring, q % PF, vstart + q * HB);
      const int ob = q - W;
      if (ob >= 0 && ob < nout) {
#pragma unroll
        for (int d = 0; d < SB_NDEEP; ++d) {
          const int i = K - 1 - d;
          if (i >= 0 && d < tl.ndeep) fetch(dring + d * PF * HB * WS, ob % PF, a + ob * HB - t.p[i] - 1);
        }
      }
      cp_async_commit();
    };
    for (int q = 0; q < PF - 1; ++q) issue(q);
    int out_next = a, prod_slot = 0, ob = 0;
    for (int pb = 0; pb < nbands; ++pb) {
      const int n = min(HB, count - pb * HB);
      issue(pb + PF - 1);
      cp_async_wait_depth(PF - 1);  // lead band pb and the deep trails of output band pb - W landed
      uint32_t cur[HB];
      const int* lp = lring + (pb % PF) * (HB * WS) + c;
#pragma unroll
      for (int r = 0; r < HB; ++r) cur[r] = (uint32_t)lp[r * WS];
      tmem_st16(tlane + (uint32_t)prod_slot, cur);
      if (prod_slot == 0) tmem_st16(tlane + (uint32_t)D, cur);
      tmem_wait_st();
      const int produced = pb * HB + n;
      prod_slot += HB;
      prod_slot = prod_slot >= D ? 0 : prod_slot;
      if (produced >= 2 * t.pmax + 1 && produced - n < 2 * t.pmax + 1) {
        // warm-up: the box sums of row a-1, 2*pmax+1 plane rows (L2-resident), 16 loads in flight
        for (int u0 = 0; u0 <= 2 * t.pmax; u0 += HB) {
          int val[HB];
#pragma unroll
          for (int r = 0; r < HB; ++r)
            val[r] = u0 + r <= 2 * t.pmax ? __ldg(mcol + (long long)min(max(vstart + u0 + r, 0), g.H - 1) * mrow) : 0;
#pragma unroll
          for (int r = 0; r < HB; ++r) {
            const int u = u0 + r;
            const int au = u > t.pmax ? u - t.pmax : t.pmax - u;
#pragma unroll
            for (int i = 0; i < K; ++i)
              if (u <= 2 * t.pmax && au <= t.p[i]) box[i] += val[r];
          }
        }
      }
      while (out_next < b) {
        const int nb = min(HB, b - out_next);
        if (produced < (out_next - a) + nb + 2 * t.pmax + 1) break;
        if (pb < ob + W) cp_async_wait_all();  // a short last band can be due before its group
        float ov[HB];
#pragma unroll
        for (int r = 0; r < HB; ++r) ov[r] = 0.0f;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          uint32_t lv[HB], tv[HB];
          tmem_ld16(tlane + (uint32_t)lead_s[i], lv);
          if (!deep[i]) tmem_ld16(tlane + (uint32_t)trail_s[i], tv);
          tmem_wait_ld();
          if (deep[i]) {
            const int d = K - 1 - i;
            if (d < tl.ndeep) {
              const int* tp = dring + d * PF * HB * WS + (ob % PF) * (HB * WS) + c;
#pragma unroll
              for (int r = 0; r < HB; ++r) tv[r] = (uint32_t)tp[r * WS];
            } else {
              const int v0 = out_next - t.p[i] - 1;
#pragma unroll
              for (int r = 0; r < HB; ++r) tv[r] = (uint32_t)__ldg(mcol + (long long)min(max(v0 + r, 0), g.H - 1) * mrow);
            }
          }
          int bx = box[i];
          const float w = t.w_col[i];
#pragma unroll
          for (int r = 0; r < HB; ++r) {
            bx += (int)lv[r] - (int)tv[r];
            ov[r] = fmaf(w, (float)bx, ov[r]);
          }
          box[i] = bx;
          lead_s[i] += HB;
          lead_s[i] = lead_s[i] >= D ? lead_s[i] - D : lead_s[i];
          trail_s[i] += HB;
          trail_s[i] = trail_s[i] >= D ? trail_s[i] - D : trail_s[i];
        }
        if (active) {
          float* dptr = dst + (long long)img * g.out_img + (long long)(out_next - g.oy0) * g.out_row +
                        (long long)(x0 + c) * g.out_px + ch;
          const long long step = g.out_row;
#pragma unroll
          for (int r = 0; r < HB; ++r) {
            if (r < nb) st_stream(dptr, ov[r]);
            dptr += step;
          }
        }
        out_next += nb;
        ++ob;
      }
    }
    cp_async_wait_all();  // the segment's trailing (unused) groups
  }
  tmem_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem_base_s, (uint32_t)tl.tmem_cols);
}

// ---------------------------------------------------------------- fused, warp-specialised
// CTA = NCONS consumer warps (thread c <-> strip column c <-> TMEM lane c) and
// NPROD producer warps.  Producers stage rows with cp.async (one band ahead),
// replicate edge columns and prefix-scan each band into one of two prefix
// buffers; consumers turn a prefix buffer into row values (releasing it
// immediately), append them to the TMEM ring and emit every output band whose
// rows are all present.  Buffers are handed over with mbarriers, so consumers
// never wait on a CTA-wide barrier.
constexpr int NCONS = WS / 32;
constexpr int NPROD = 2;
constexpr int FUSED_THREADS = 32 * (NCONS + NPROD);
constexpr int NSTAGE = 2 * NPROD;  // staged bands (each producer warp double-buffers its own)
constexpr int NPBUF = 2 * NPROD;   // prefix buffers (each producer warp owns two)
// fused kernel: 4 consumer warps + FPROD producer warps (each owns every FPROD-th band)
constexpr int FCONS = WS / 32;
constexpr int FPROD = 4;
constexpr int FTHREADS = 32 * (FCONS + FPROD);
constexpr int FPBUF = 2 * FPROD;

// MINB = 3 (uint8 one-channel float2 path): three CTAs per SM.  The kernel is compiled
// for 80 registers per thread; the producer warpgroup gives registers back
// (setmaxnreg.dec) so the consumer warpgroup can grow (setmaxnreg.inc), and the staged
// band and the output staging box are single-buffered to fit three CTAs' shared memory.
#ifndef SB_F3PREG
#define SB_F3PREG 72
#define SB_F3CREG 88
#endif
constexpr int F3PREG = SB_F3PREG, F3CREG = SB_F3CREG;

// ---- shared-memory counters (acquire / release) and the device watchdog used by the ring kernels
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  sb_perturb();
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// SB_WATCHDOG builds: a wait longer than 2 s prints what it waited for and traps (a hang
// becomes a diagnosable launch error)
#ifdef SB_WATCHDOG
#define SB_WD_START const unsigned long long wd_t0 = gtimer();
#define SB_WD_CHECK(what, a, b)                                                                              \
  if (gtimer() - wd_t0 > 2000000000ull) {                                                                    \
    printf("watchdog: %s block %d warp %d lane %d a=%d b=%d\n", what, (int)blockIdx.x, (int)(threadIdx.x >> 5), \
           (int)(threadIdx.x & 31), (int)(a), (int)(b));                                                     \
    __trap();                                                                                                \
  }
#else
#define SB_WD_START
#define SB_WD_CHECK(what, a, b)
#endif

#ifndef SB_WA_MAXNS
#define SB_WA_MAXNS 256
#endif
// wait until *p > v
__device__ __forceinline__ void wait_above(const uint32_t* p, uint32_t v, bool backoff) {
  unsigned ns = 32;
  SB_WD_START
  while (ld_acquire(p) <= v) {
    SB_WD_CHECK("wait_above", v, ld_acquire(p));
    if (backoff) {
      __nanosleep(ns);
      ns = ns < SB_WA_MAXNS ? 2 * ns : ns;
    }
  }
  sb_perturb();
}
__device__ __forceinline__ void mbar_wait_wd(uint64_t* bar, uint32_t parity, int tag) {
  SB_WD_START
  while (!mbar_test(bar, parity)) {
    SB_WD_CHECK("mbar", tag, parity);
  }
  sb_perturb();
}

// PAIRED (uint8 packed path): eight consumer warps.  Warps q and q + 4 share TMEM lane quadrant
// q and alternate bands: each forms the row values of its own band while the other is still
// in its column pass, takes the column prefix at the end of the previous band from the other
// warp (one shared-memory word per column, monotonic per-quadrant counters), appends its band
// to the ring and forms the output band that its band completes.  Twice the consumer warps per
// SM for the latency-bound row-value / window chains, at 80 registers per thread.
#ifndef SB_FPPREG
#define SB_FPPREG 64
#define SB_FPCREG 88
#endif
constexpr int PTHREADS = FTHREADS + 32 * FCONS;

template <typename Tin, int K, int MINB = 2, bool B2 = false, int PLS = LS, bool PAIRED = false, bool A4 = false>
__global__ void __launch_bounds__(PAIRED ? PTHREADS : FTHREADS, MINB)
    fused_kernel(const Tin* __restrict__ src, float* __restrict__ dst, Geometry g, Taps t, Tiling tl, int* status,
                 const __grid_constant__ CUtensorMap omap) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t tmem_base_s;
  __shared__ __align__(8) uint64_t bar_full[FPBUF], bar_empty[FPBUF];
  // PAIRED hand-offs: bands whose end-of-band column prefix is published (per quadrant), bands
  // each consumer warp has appended to the ring, and the published prefixes (per writer half)
  __shared__ uint32_t pair_cnt[4], stored_cnt[2 * FCONS], seg_cnt[2 * FCONS];
  __shared__ int carry_s[2][WS];
  constexpr int NCW = PAIRED ? 2 * FCONS : FCONS;  // consumer warps
  const int strip = blockIdx.x % tl.nstrips;
  const long long item = blockIdx.x / tl.nstrips;
  const int ch = blockIdx.y;
  const int x0 = strip * WS;
  const int xb = x0 - tl.xoff;
  const int warp = threadIdx.x >> 5;
  const bool producer = warp >= NCW;
  const int wh = g.oy1 - g.oy0;  // rows of each image this launch outputs
  const long long total = (long long)g.nimg * wh;
  const long long T0 = item * tl.rows_per_item;
  const long long T1 = min(T0 + tl.rows_per_item, total);
  const bool packed = (sizeof(Tin) == 1) && tl.packed;
  // staged bands per producer warp: one for the three-CTA uint8 kernel and the small-stride
  // float32 kernel (two CTAs per SM), two otherwise
  constexpr int NSB = (MINB == 3 || (!B2 && PLS == LS_SMALL && sizeof(Tin) == 4)) ? 1 : 2;
  const int pbuf_words = packed ? HB * LSP2 : HB * PLS;  // packed: HB/2 float2 rows
  unsigned char* stage = smem;                                          // FPROD producers x NSB staged bands
  int* Pbase = (int*)(smem + NSB * FPROD * HB * tl.stage_row_bytes);    // FPROD x npb prefix buffers
  // FCONS x 2 output bands of HB x 32 floats (TMA stores; 128-byte aligned shared addresses)
  float* obuf = (float*)(smem + (((smem_u32(smem) + tl.obuf_off + 127u) & ~127u) - smem_u32(smem)));
  const int D = tl.D;

  if (threadIdx.x == 0) {
    for (int i = 0; i < FPROD * tl.npb; ++i) {
      mbar_init(&bar_full[i], 32);  // one producer warp fills a prefix buffer
      mbar_init(&bar_empty[i], 32 * FCONS);
    }
    if constexpr (PAIRED) {
      for (int i = 0; i < 4; ++i) pair_cnt[i] = 0;
      for (int i = 0; i < 2 * FCONS; ++i) stored_cnt[i] = seg_cnt[i] = 0;
    }
  }
  if (warp == 0) tmem_alloc(&tmem_base_s, (uint32_t)tl.tmem_cols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if constexpr (PAIRED) {
    if (producer)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(SB_FPPREG));
    else
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(SB_FPCREG));
  }
  if constexpr (MINB == 3) {
    if (producer)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(F3PREG));
    else
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(F3CREG));
  }

  if (producer) {
    // ------------------------------------------------ producer warps
    // Producer warp pw owns the bands with global index gb = pw (mod FPROD): it stages
    // them into its private pair of buffers (prefetching its next band) and scans
    // them into prefix buffer pw, so the producers never synchronise with each other.
    const int lane = threadIdx.x & 31, pw = warp - NCW;
    const bool edge = (xb < 0) || (xb + tl.L > g.W);
    const int st_lo = max(xb, 0) * g.in_px * g.es;
    const int st_hi = min(xb + tl.L, g.W) * g.in_px * g.es;
    // 16-byte copies for 16-byte aligned rows, 4-byte copies for rows that are 4-byte multiples
    // (a 1000-pixel-wide uint8 image), element copies otherwise
    // (A4 instantiations; the host picks them for sources whose rows are 4-byte multiples)
    const int st_gran = g.aligned16 ? 16 : (A4 ? 4 : 0);
    const int st_hi16 = A4 ? (st_hi & ~(st_gran - 1)) : (g.aligned16 ? (st_hi & ~15) : st_hi);
    const int st_nchunk = A4 ? max(0, (st_hi16 - st_lo) / max(1, st_gran)) : max(0, (st_hi16 - st_lo) >> 4);
    const uint32_t st_magic = 0xFFFFFFFFu / (uint32_t)max(1, st_nchunk) + 1u;
    unsigned char* mystage = stage + pw * NSB * HB * tl.stage_row_bytes;
    uint32_t gb0 = 0;  // global index of the segment's first band
    for (long long T = T0; T < T1;) {
      const int img = (int)(T / wh);
      const int a = g.oy0 + (int)(T - (long long)img * wh);
      const int b = g.oy0 + (int)min((long long)wh, T1 - (long long)img * wh);
      T = (long long)img * wh + (b - g.oy0);
      const Tin* src_img = src + (long long)img * g.in_img;
      const int vstart = a - 1 - t.pmax;
      const int count = (b - a) + 2 * t.pmax + 1;
      const int nbands = (count + HB - 1) / HB;
      const int first = (int)(((uint32_t)pw + FPROD * 64u - gb0 % FPROD) % FPROD);  // first owned band
      __syncwarp();  // every lane is done with the staged band (single-buffer case)
      if (first < nbands)
        issue_stage<Tin, A4>(mystage, src_img, g, tl, xb, vstart + first * HB, min(HB, count - first * HB), st_lo,
                         st_nchunk, st_magic, st_hi16, st_hi, lane, 32, st_gran);
      int sb = 0;
      for (int pb = first; pb < nbands; pb += FPROD, sb ^= 1) {
        const uint32_t gb = gb0 + pb;
        const int n = min(HB, count - pb * HB);
        unsigned char* cur = mystage + (NSB == 2 ? sb : 0) * HB * tl.stage_row_bytes;
        cp_async_wait_all();  // this band landed (the next one is issued below)
        __syncwarp();
        if (NSB == 2 && pb + FPROD < nbands)
          issue_stage<Tin, A4>(mystage + (sb ^ 1) * HB * tl.stage_row_bytes, src_img, g, tl, xb,
                           vstart + (pb + FPROD) * HB, min(HB, count - (pb + FPROD) * HB), st_lo, st_nchunk, st_magic,
                           st_hi16, st_hi, lane, 32, st_gran);
        if (edge) {
          fixup_edges(cur, g, tl, xb, n, lane, 32);
          __syncwarp();
        }
        // this producer's (gb >> 1)-th band -> its buffer (gb >> 1) % npb, used for the
        // ((gb >> 1) / npb)-th time
        const uint32_t kb = gb / FPROD;
        const int pbi = pw * tl.npb + (int)(kb & (uint32_t)(tl.npb - 1));  // npb is 1 or 2
        int* P = Pbase + pbi * pbuf_words;
        mbar_wait_sleep(&bar_empty[pbi], ((kb >> (tl.npb - 1)) & 1) ^ 1);  // consumers done with it
        if (packed)
          scan_rows_b2_dispatch(cur, (float2*)P, tl);
        else
        {
          // uint8 sources only reach this for interleaved channels / long rows; keeping
          // the lane-per-chunk scan there leaves the uint8 kernel's (hot) code unchanged
          if constexpr (sizeof(Tin) == 1)
            scan_rows<Tin>(cur, P, g, t, tl, ch, n, status, 0, 1);
          else
            scan_band8<Tin, PLS>(cur, P, g, t, tl, ch, n, status);
        }
        if (NSB == 1) {  // single staged band: the next one lands while the other producers' bands are used
          __syncwarp();
          if (pb + FPROD < nbands)
            issue_stage<Tin, A4>(mystage, src_img, g, tl, xb, vstart + (pb + FPROD) * HB, min(HB, count - (pb + FPROD) * HB),
                             st_lo, st_nchunk, st_magic, st_hi16, st_hi, lane, 32, st_gran);
        }
        mbar_arrive(&bar_full[pbi]);
      }
      gb0 += (uint32_t)nbands;
    }
  } else if constexpr (PAIRED) {
    // ------------------------------------------------ paired consumer warps (see the template comment)
    const int lane = threadIdx.x & 31, q = warp & 3, hf = warp >> 2;
    const int c = 32 * q + lane;
    const bool active = (x0 + c) < g.W;
    const uint32_t tlane = tmem_base_s + ((uint32_t)(32 * q) << 16);
    const int NBR = D / HB;  // ring bands
    uint32_t gb0 = 0;        // global index of the segment's first band
    uint32_t seg = 0;        // segments completed
    int obsel = 0;
    for (long long T = T0; T < T1; ++seg) {
      const int img = (int)(T / wh);
      const int a = g.oy0 + (int)(T - (long long)img * wh);
      const int b = g.oy0 + (int)min((long long)wh, T1 - (long long)img * wh);
      T = (long long)img * wh + (b - g.oy0);
      const int count = (b - a) + 2 * t.pmax + 1;
      const int nbands = (count + HB - 1) / HB;
      const int nob = (b - a + HB - 1) / HB;  // output bands of the segment
      int ob = 0, obslot = 0;                 // next output band to consider, ob % NBR
      int slot = hf;                          // ring band of this warp's next band (pb % NBR; NBR >= 2)
      bool first = true;
      for (int pb = hf; pb < nbands; pb += 2) {
        const uint32_t gb = gb0 + (uint32_t)pb;
        const int n = min(HB, count - pb * HB);
        const uint32_t kb = gb / FPROD;
        const int pbi = (int)(gb % FPROD) * tl.npb + (int)(kb & (uint32_t)(tl.npb - 1));
        const float2* P = (const float2*)(Pbase + pbi * pbuf_words);
        uint32_t cv[HB];
        {
          // A parity wait is only meaningful once the buffer's previous use (band gb - 4) is
          // over.  Inside a segment the carry chain guarantees it (this warp's previous band
          // gb - 2 needed every earlier band); a warp entering a segment may have been idle for
          // many one-band segments, so it first sees band gb - 2 published.
          if (first && gb >= 2) wait_above(&pair_cnt[q], gb - 2, false);
          mbar_wait(&bar_full[pbi], (kb >> (tl.npb - 1)) & 1);
          float2 r2[HB / 2];
          band_rows_f2<K>(P, c, t, tl, r2);
          mbar_arrive(&bar_empty[pbi]);
          int lp = 0;  // prefix within the band
#pragma unroll
          for (int qq = 0; qq < HB / 2; ++qq) r2[qq] = round_mid2<K>(r2[qq]);  // round to the mid quantum
#pragma unroll
          for (int r = 0; r < HB; ++r) {
            const float v = r < HB / 2 ? r2[r].x : r2[r - HB / 2].y;
            lp += __float_as_int(v) - kMagicBits;
            cv[r] = (uint32_t)lp;
          }
        }
        // column prefix at the end of band gb - 1 (published by the other warp; 0 at a segment
        // start).  Waiting also keeps pair_cnt monotonic: band gb is published after gb - 1.
        if (gb > 0) wait_above(&pair_cnt[q], gb - 1, false);
        const int carry = pb > 0 ? carry_s[hf ^ 1][c] : 0;
#pragma unroll
        for (int r = 0; r < HB; ++r) cv[r] += (uint32_t)carry;
        carry_s[hf][c] = (int)cv[HB - 1];
        __syncwarp();
        if (lane == 0) st_release(&pair_cnt[q], gb + 1);
        // the ring restarts with every segment: the other warp must be out of the previous
        // segment's windows before this warp's first band lands
        if (first && seg > 0) wait_above(&seg_cnt[2 * q + (hf ^ 1)], seg - 1, false);
        first = false;
        SB_ASSERT(slot * HB + HB <= D && D + HB <= tl.tmem_cols);
        tmem_st16(tlane + (uint32_t)(slot * HB), cv);
        if (slot == 0) tmem_st16(tlane + (uint32_t)D, cv);  // mirror: lag windows never wrap
        tmem_wait_st();
        tmem_fence_before();
        __syncwarp();
        if (lane == 0) st_release(&stored_cnt[2 * q + hf], gb + 1);
        slot += 2;
        slot = slot >= NBR ? slot - NBR : slot;
        // output bands completed by this band (band ob needs virtual rows up to 16 ob + nb + 2 pmax)
        while (ob < nob) {
          const int nb = min(HB, (b - a) - ob * HB);
          const int pe = (ob * HB + nb + 2 * t.pmax + 1 + HB - 1) / HB - 1;
          if (pe > pb) break;
          if (pe == pb) {
            // every earlier band is in the ring: this warp's in program order, the other's by count
            if (pb > 0) wait_above(&stored_cnt[2 * q + (hf ^ 1)], gb - 1, false);
            tmem_fence_after();
            const int out_next = a + ob * HB;
            const int out_mod = obslot * HB;
            int lead_s[K], trail_s[K];
#pragma unroll
            for (int i = 0; i < K; ++i) {
              const int l = out_mod + t.pmax + 1 + t.p[i];
              const int tr = out_mod + t.pmax - t.p[i];
              lead_s[i] = l >= D ? l - D : l;
              trail_s[i] = tr >= D ? tr - D : tr;
            }
            float ov[HB];
            column_band_tmem<K>(tlane, lead_s, trail_s, t, ov);
            if (g.out_bulk && nb == HB) {
              float* obp = obuf + (warp * 2 + obsel) * (HB * 32);
              if (lane == 0) bulk_wait_read<1>();  // the store out of this box (two bands ago) has read it
              __syncwarp();
#pragma unroll
              for (int r = 0; r < HB; ++r) obp[r * 32 + lane] = ov[r];
              fence_proxy_async();
              __syncwarp();
              if (lane == 0) {
                tma_store_3d(&omap, obp, x0 + 32 * q, out_next - g.oy0, img);
                bulk_commit();
              }
              obsel ^= 1;
            } else if (active) {
              float* dptr = dst + (long long)img * g.out_img + (long long)(out_next - g.oy0) * g.out_row + (x0 + c);
#pragma unroll
              for (int r = 0; r < HB; ++r) {
                if (r < nb) st_stream(dptr, ov[r]);
                dptr += g.out_row;
              }
            }
          }
          ++ob;
          obslot = obslot + 1 == NBR ? 0 : obslot + 1;
        }
      }
      gb0 += (uint32_t)nbands;
      // this warp has read its last window of the segment (tcgen05.wait::ld precedes the release)
      tmem_fence_before();
      __syncwarp();
      if (lane == 0) st_release(&seg_cnt[2 * q + hf], seg + 1);
    }
    if (lane == 0) bulk_wait_read<0>();
  } else if constexpr (B2) {
    // ------------------------------------------------ consumer warps, two bands per iteration
    // (uint8 packed path): one prefix carry, one 32-column TMEM store, one 32-row output band
    // with 32-row TMEM windows and one staged 32 x 32 box per iteration
    const int c = threadIdx.x, lane = threadIdx.x & 31;
    const bool active = (x0 + c) < g.W;
    const uint32_t tlane = tmem_base_s + ((uint32_t)(threadIdx.x & ~31) << 16);
    uint32_t gb = 0;
    int obsel = 0;
    for (long long T = T0; T < T1;) {
      const int img = (int)(T / wh);
      const int a = g.oy0 + (int)(T - (long long)img * wh);
      const int b = g.oy0 + (int)min((long long)wh, T1 - (long long)img * wh);
      T = (long long)img * wh + (b - g.oy0);
      const int count = (b - a) + 2 * t.pmax + 1;
      const int nbands = (count + HB - 1) / HB;
      int out_next = a, out_mod = 0, prod_slot = 0;
      int cprefix = 0;
      for (int pb = 0; pb < nbands; pb += 2) {
        uint32_t cv[2 * HB];
        int produced = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 0 || pb + h < nbands) {  // the first band of a turn always exists
            const uint32_t kb = gb / FPROD;
            const int pbi = (int)(gb % FPROD) * tl.npb + (int)(kb & (uint32_t)(tl.npb - 1));
            const float2* P = (const float2*)(Pbase + pbi * pbuf_words);
            mbar_wait(&bar_full[pbi], (kb >> (tl.npb - 1)) & 1);
            float2 r2[HB / 2];
            band_rows_f2<K>(P, c, t, tl, r2);
            mbar_arrive(&bar_empty[pbi]);
#pragma unroll
            for (int q = 0; q < HB / 2; ++q) {
              r2[q] = round_mid2<K>(r2[q]);  // round to the mid quantum
              cv[h * HB + q] = __float_as_uint(r2[q].x);
              cv[h * HB + q + HB / 2] = __float_as_uint(r2[q].y);
            }
            produced = (pb + h) * HB + min(HB, count - (pb + h) * HB);
            ++gb;
          } else {
#pragma unroll
            for (int q = 0; q < HB; ++q) cv[h * HB + q] = (uint32_t)kMagicBits;  // zero rows past the end
          }
        }
#pragma unroll
        for (int r = 0; r < 2 * HB; ++r) {
          cprefix += (int)cv[r] - kMagicBits;
          cv[r] = (uint32_t)cprefix;
        }
        SB_ASSERT(prod_slot + 2 * HB <= D && D + 2 * HB <= tl.tmem_cols);
        tmem_st32(tlane + (uint32_t)prod_slot, cv);
        if (prod_slot == 0) tmem_st32(tlane + (uint32_t)D, cv);  // 32-row mirror
        tmem_wait_st();
        prod_slot += 2 * HB;
        prod_slot = prod_slot >= D ? 0 : prod_slot;
        while (out_next < b) {
          const int nb = min(2 * HB, b - out_next);
          if (produced < (out_next - a) + nb + 2 * t.pmax + 1) break;
          float2 o2[HB];
#pragma unroll
          for (int i = 0; i < K; ++i) {
            int l = out_mod + t.pmax + 1 + t.p[i];
            int tr = out_mod + t.pmax - t.p[i];
            l = l >= D ? l - D : l;
            tr = tr >= D ? tr - D : tr;
            SB_ASSERT(l >= 0 && tr >= 0 && l < D && tr < D);
            uint32_t lv[2 * HB], tv[2 * HB];
            tmem_ld32(tlane + (uint32_t)l, lv);
            tmem_ld32(tlane + (uint32_t)tr, tv);
            tmem_wait_ld();
            const float2 w2 = make_float2(t.w_col[i], t.w_col[i]);
#pragma unroll
            for (int r = 0; r < HB; ++r) {
              const float2 d = make_float2(i2f_fast(lv[2 * r] - tv[2 * r]), i2f_fast(lv[2 * r + 1] - tv[2 * r + 1]));
              o2[r] = i == 0 ? __fmul2_rn(w2, d) : __ffma2_rn(w2, d, o2[r]);
            }
          }
          if (g.out_bulk && nb == 2 * HB) {
            float* ob = obuf + (warp * 2 + obsel) * (2 * HB * 32);
            if (lane == 0) bulk_wait_read<1>();  // the stores out of this box (two bands ago) have read it
            __syncwarp();
#pragma unroll
            for (int r = 0; r < HB; ++r) {
              ob[(2 * r) * 32 + lane] = o2[r].x;
              ob[(2 * r + 1) * 32 + lane] = o2[r].y;
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(&omap, ob, x0 + (warp << 5), out_next - g.oy0, img);
              tma_store_3d(&omap, ob + HB * 32, x0 + (warp << 5), out_next + HB - g.oy0, img);
              bulk_commit();
            }
            obsel ^= 1;
          } else if (active) {
            float* dptr = dst + (long long)img * g.out_img + (long long)(out_next - g.oy0) * g.out_row + (x0 + c);
#pragma unroll
            for (int r = 0; r < HB; ++r) {
              if (2 * r < nb) st_stream(dptr, o2[r].x);
              dptr += g.out_row;
              if (2 * r + 1 < nb) st_stream(dptr, o2[r].y);
              dptr += g.out_row;
            }
          }
          out_next += nb;
          out_mod += nb;
          out_mod = out_mod >= D ? out_mod - D : out_mod;
        }
      }
    }
    if ((threadIdx.x & 31) == 0) bulk_wait_read<0>();
  } else {
    // ------------------------------------------------ consumer warps
    const int c = threadIdx.x;
    const bool active = (x0 + c) < g.W;
    const uint32_t tlane = tmem_base_s + ((uint32_t)(threadIdx.x & ~31) << 16);
    uint32_t gb = 0;
    int obsel = 0;
    for (long long T = T0; T < T1;) {
      const int img = (int)(T / wh);
      const int a = g.oy0 + (int)(T - (long long)img * wh);
      const int b = g.oy0 + (int)min((long long)wh, T1 - (long long)img * wh);
      T = (long long)img * wh + (b - g.oy0);
      const int count = (b - a) + 2 * t.pmax + 1;
      const int nbands = (count + HB - 1) / HB;
      int out_next = a, out_mod = 0, prod_slot = 0;
      int cprefix = 0;  // running column prefix of the rounded row values (mid quanta, wraps)
      for (int pb = 0; pb < nbands; ++pb, ++gb) {
        const int n = min(HB, count - pb * HB);
        const uint32_t kb = gb / FPROD;
        const int pbi = (int)(gb % FPROD) * tl.npb + (int)(kb & (uint32_t)(tl.npb - 1));
        const int* P = Pbase + pbi * pbuf_words;
        float rv[HB];
        mbar_wait(&bar_full[pbi], (kb >> (tl.npb - 1)) & 1);
        if (packed) {
          float2 r2[HB / 2];
          band_rows_f2<K>((const float2*)P, c, t, tl, r2);
#pragma unroll
          for (int q = 0; q < HB / 2; ++q) {
            r2[q] = round_mid2<K>(r2[q]);  // round to the mid quantum
            rv[q] = r2[q].x;
            rv[q + HB / 2] = r2[q].y;
          }
        } else {
          band_rows<K, PLS>(P, c, t.w_row, t, tl, rv);
#pragma unroll
          for (int r = 0; r < HB; ++r) rv[r] = __fadd_rn(rv[r], kMagic);  // round to the mid quantum (_rn: never contracted)
        }
        mbar_arrive(&bar_empty[pbi]);
        {
          uint32_t cv[HB];
#pragma unroll
          for (int r = 0; r < HB; ++r) {
            cprefix += __float_as_int(rv[r]) - kMagicBits;
            cv[r] = (uint32_t)cprefix;
          }
          SB_ASSERT(prod_slot + HB <= D && D + HB <= tl.tmem_cols);
          tmem_st16(tlane + (uint32_t)prod_slot, cv);
          if (prod_slot == 0) tmem_st16(tlane + (uint32_t)D, cv);  // mirror: lag windows never wrap
          tmem_wait_st();
        }
        const int produced = pb * HB + n;
        prod_slot += HB;
        prod_slot = prod_slot >= D ? 0 : prod_slot;
        while (out_next < b) {
          const int nb = min(HB, b - out_next);
          if (produced < (out_next - a) + nb + 2 * t.pmax + 1) break;
          int lead_s[K], trail_s[K];
#pragma unroll
          for (int i = 0; i < K; ++i) {
            const int l = out_mod + t.pmax + 1 + t.p[i];
            const int tr = out_mod + t.pmax - t.p[i];
            lead_s[i] = l >= D ? l - D : l;
            trail_s[i] = tr >= D ? tr - D : tr;
          }
          float ov[HB];
          column_band_tmem<K>(tlane, lead_s, trail_s, t, ov);
          if (g.out_bulk && nb == HB) {
            // stage the band (row r of this warp's 32 columns at ob[r][lane]) and let one
            // TMA tensor store write the 16 x 32 box: no per-row address arithmetic
            const int lane = threadIdx.x & 31;
            float* ob = obuf + (warp * NSB + (NSB == 2 ? obsel : 0)) * (HB * 32);
            if (lane == 0) {  // the store out of this buffer (NSB bands ago) has read it
              if (NSB == 2)
                bulk_wait_read<1>();
              else
                bulk_wait_read<0>();
            }
            __syncwarp();
#pragma unroll
            for (int r = 0; r < HB; ++r) ob[r * 32 + lane] = ov[r];
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(&omap, ob, x0 + (warp << 5), out_next - g.oy0, img);
              bulk_commit();
            }
            obsel ^= 1;
          } else if (active) {
            float* dptr = dst + (long long)img * g.out_img + (long long)(out_next - g.oy0) * g.out_row +
                          (long long)(x0 + c) * g.out_px + ch;
            const long long step = g.out_row;
            if (nb == HB) {
#pragma unroll
              for (int r = 0; r < HB; ++r) {
                st_stream(dptr, ov[r]);
                dptr += step;
              }
            } else {
#pragma unroll
              for (int r = 0; r < HB; ++r) {
                if (r < nb) st_stream(dptr, ov[r]);
                dptr += step;
              }
            }
          }
          out_next += nb;
          out_mod += nb;
          out_mod = out_mod >= D ? out_mod - D : out_mod;
        }
      }
    }
    if ((threadIdx.x & 31) == 0) bulk_wait_read<0>();  // shared memory must outlive the stores out of it
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem_base_s, (uint32_t)tl.tmem_cols);
}

// The segments of one CTA's row range: every image the range touches restarts
// its sweep (virtual rows a-1-pmax .. b-1+pmax of output rows [a, b)); gb0 is
// the global index of the segment's first 16-row band.
struct SegIter {
  long long T, T1, wh;
  int oy0, pmax;
  int img, a, b, count, nbands;
  uint32_t gb0;
  bool valid;
  __device__ __forceinline__ void init(long long T0_, long long T1_, long long wh_, int oy0_, int pmax_) {
    T = T0_, T1 = T1_, wh = wh_, oy0 = oy0_, pmax = pmax_, gb0 = 0, nbands = 0;
    load();
  }
  __device__ __forceinline__ void load() {
    valid = T < T1;
    if (!valid) return;
    img = (int)(T / wh);
    a = oy0 + (int)(T - (long long)img * wh);
    b = oy0 + (int)min(wh, T1 - (long long)img * wh);
    count = (b - a) + 2 * pmax + 1;
    nbands = (count + HB - 1) / HB;
  }
  __device__ __forceinline__ void next() {
    T = (long long)img * wh + (b - oy0);
    gb0 += (uint32_t)nbands;
    load();
  }
};
template <typename Unused = void>  // a template: instantiates its kernels only where it is called
const void* fused5_ptr_for(int k) {
  switch (k) {
    case 1: return (const void*)fused_kernel<uint8_t, 1, 2, true>;
    case 2: return (const void*)fused_kernel<uint8_t, 2, 2, true>;
    case 3: return (const void*)fused_kernel<uint8_t, 3, 2, true>;
    case 4: return (const void*)fused_kernel<uint8_t, 4, 2, true>;
    case 5: return (const void*)fused_kernel<uint8_t, 5, 2, true>;
    case 6: return (const void*)fused_kernel<uint8_t, 6, 2, true>;
    case 7: return (const void*)fused_kernel<uint8_t, 7, 2, true>;
    default: return (const void*)fused_kernel<uint8_t, 8, 2, true>;
  }
}

template <typename Unused = void>
const void* fused5w_ptr_for(int k) {  // two-band uint8 kernel with 4-byte staging copies (A4)
  switch (k) {
    case 1: return (const void*)fused_kernel<uint8_t, 1, 2, true, LS, false, true>;
    case 2: return (const void*)fused_kernel<uint8_t, 2, 2, true, LS, false, true>;
    case 3: return (const void*)fused_kernel<uint8_t, 3, 2, true, LS, false, true>;
    case 4: return (const void*)fused_kernel<uint8_t, 4, 2, true, LS, false, true>;
    case 5: return (const void*)fused_kernel<uint8_t, 5, 2, true, LS, false, true>;
    case 6: return (const void*)fused_kernel<uint8_t, 6, 2, true, LS, false, true>;
    case 7: return (const void*)fused_kernel<uint8_t, 7, 2, true, LS, false, true>;
    default: return (const void*)fused_kernel<uint8_t, 8, 2, true, LS, false, true>;
  }
}

template <typename Unused = void>  // a template: instantiates its kernels only where it is called
const void* fusedp_ptr_for(int k) {
  switch (k) {
    case 1: return (const void*)fused_kernel<uint8_t, 1, 2, false, LS, true>;
    case 2: return (const void*)fused_kernel<uint8_t, 2, 2, false, LS, true>;
    case 3: return (const void*)fused_kernel<uint8_t, 3, 2, false, LS, true>;
    case 4: return (const void*)fused_kernel<uint8_t, 4, 2, false, LS, true>;
    case 5: return (const void*)fused_kernel<uint8_t, 5, 2, false, LS, true>;
    case 6: return (const void*)fused_kernel<uint8_t, 6, 2, false, LS, true>;
    case 7: return (const void*)fused_kernel<uint8_t, 7, 2, false, LS, true>;
    default: return (const void*)fused_kernel<uint8_t, 8, 2, false, LS, true>;
  }
}

template <typename Unused = void>  // a template: instantiates its kernels only where it is called
const void* fused3_ptr_for(int k) {
  switch (k) {
    case 1: return (const void*)fused_kernel<uint8_t, 1, 3>;
    case 2: return (const void*)fused_kernel<uint8_t, 2, 3>;
    case 3: return (const void*)fused_kernel<uint8_t, 3, 3>;
    case 4: return (const void*)fused_kernel<uint8_t, 4, 3>;
    case 5: return (const void*)fused_kernel<uint8_t, 5, 3>;
    case 6: return (const void*)fused_kernel<uint8_t, 6, 3>;
    case 7: return (const void*)fused_kernel<uint8_t, 7, 3>;
    default: return (const void*)fused_kernel<uint8_t, 8, 3>;
  }
}

constexpr int FRING = 32;  // max ring slots (512 TMEM columns / HB)

// ---------------------------------------------------------------- column pass, prefix form (large radii)
// ColsFromMid with independent output bands: one CTA per strip and SM, the ring
// in TMEM holds the running column PREFIX C of the R plane (as in the fused
// kernel), so every output band is C(y+p) - C(y-p-1) windows with no running
// state and CG output warp groups emit bands j = g (mod CG) concurrently.
//  * loader warps (4, one per TMEM lane quadrant): plane bands arrive as TMA
//    tensor loads (16 x 128 int32 boxes) tl.pf bands ahead; the loader accumulates C and appends each
//    band to the ring after every output band that reads the overwritten band
//    from TMEM is done (lag tl.lag = span + CG - 1 bands);
//  * trails older than the ring (C5's largest boxes) are read from a shared-memory
//    copy: the loader copies band u = v - NB + tl.copy_e out of TMEM while writing
//    band v, so it is there before any output band needs it and stays there for
//    tl.ds bands (copy_e = lag - span lets the loader run lag - span - CG + 1
//    bands of slack ahead of the output groups).  The host classifies every trail window as ring or copy
//    (tl.deepmask) and falls back to cols_kernel when a window would straddle.
#ifndef SB_CG
#define SB_CG 2
#endif
constexpr int CG = SB_CG;                      // output warp groups
constexpr int C2THREADS = 32 * 4 * (1 + CG);   // loader group + CG output groups
constexpr int C2DONE = 32;  // output-band done barriers: >= lag - span + 1, so no barrier is lapped
constexpr int C2PF = 8;     // max plane-band slots (TMA ring)

// Work units: unit u = (row chunk u / nstrips, strip u % nstrips) covers tall rows
// [rc * Hc, min((rc + 1) * Hc, total)) of one 128-column strip (the tall image stacks the
// batch; Hc = tl.rows_per_item).  CTA b takes units b, b + grid, ... so the CTAs running at
// any moment sweep neighbouring strips over the same rows and every strip's halo columns
// are L2 hits.  A unit splits into segments at image boundaries; every segment restarts
// the sweep (virtual rows a-1-pmax .. b-1+pmax of the output rows [a, b)); gb0 is the
// CTA-global index of the segment's first band (bands of bh rows).
struct WorkIter {
  long long T, Tend, total, wh, Hc;
  int u, nunits, nstrips, oy0, pmax, bh;
  int strip, img, a, b, count, nbands;
  uint32_t gb0;
  bool valid;
  __device__ __forceinline__ void init(long long total_, long long Hc_, int nstrips_, long long wh_, int oy0_,
                                       int pmax_, int bh_ = HB) {
    total = total_, Hc = Hc_, nstrips = nstrips_, wh = wh_, oy0 = oy0_, pmax = pmax_, bh = bh_, gb0 = 0, nbands = 0;
    nunits = (int)((total + Hc - 1) / Hc) * nstrips;
    u = blockIdx.x;
    load_unit();
  }
  __device__ __forceinline__ void load_unit() {
    valid = u < nunits;
    if (!valid) return;
    strip = u % nstrips;
    T = (long long)(u / nstrips) * Hc;
    Tend = min(T + Hc, total);
    load();
  }
  __device__ __forceinline__ void load() {
    img = (int)(T / wh);
    const long long r = T - (long long)img * wh;
    a = oy0 + (int)r;
    b = oy0 + (int)min(wh, r + (Tend - T));
    count = (b - a) + 2 * pmax + 1;
    nbands = (count + bh - 1) / bh;
  }
  __device__ __forceinline__ void next() {
    T += (long long)(b - a);
    gb0 += (uint32_t)nbands;
    if (T < Tend) {
      load();
    } else {
      u += gridDim.x;
      load_unit();
    }
  }
};

// Wide fused sweep (sweep_wide.cu): float32, one channel, radii past fused_kernel's reach.
// 4 row warps + WCG output groups of 4 warps + WPROD producer warps; slot row strides WLS
// (words, = 4 mod 32 so rows are 16 mod 128 bytes apart) bound the staged row length L.
constexpr int WCG = 2;
constexpr int WPROD = 4;
constexpr int WTHREADS = 32 * (4 + 4 * WCG + WPROD);
constexpr int WLS[3] = {516, 676, 900};

// Monotonic counters in shared memory (release / acquire at CTA scope): a count cannot alias
// the way an mbarrier phase parity can when one waiter falls two phases behind.

// Row-tile sweep (sweep_rowtile.cu): uint8, one channel, small radii.  32-row bands; 8 row
// warps (thread = row; two per TMEM lane quadrant), 4 loader warps and TOG output groups of 4
// (thread = column); TRS row-value slots of TB rows x TRSW words (528 B = 16 mod 128).
#ifndef SB_TOG
#define SB_TOG 2
#endif
#ifndef SB_TROWW
#define SB_TROWW 8
#endif
#ifndef SB_TRS
#define SB_TRS 4
#endif
constexpr int TB = 32;
constexpr int TOG = SB_TOG;
constexpr int TROWW = SB_TROWW;
constexpr int TTHREADS = 32 * (TROWW + 4 + 4 * TOG);
constexpr int TRS = SB_TRS;
#ifndef SB_TOBUF
#define SB_TOBUF 2
#endif
constexpr int TOBUF = SB_TOBUF;  // output boxes per output warp (double or single buffered)
constexpr int TRSW = WS + 4;
constexpr int TDONE = 32;  // output-band done barriers

// SPLIT: eight loader warps.  Warps q and q + 4 share lane quadrant q and alternate band pairs
// (pair G goes to half G & 1): each waits for its plane bands, forms the pair's prefix from zero
// and only then takes the running column prefix from the other half (one shared-memory word per
// column, monotonic per-quadrant counters), so the waits, shared-memory loads and scans of
// consecutive pairs overlap.  Ring releases stay in band order (pair_done), and with band
// copies a pair is appended only after the previous pair's copies are out of the ring.
constexpr int C2STHREADS = C2THREADS + 32 * 4;

template <int K, bool SPLIT = false>
__global__ void __launch_bounds__(SPLIT ? C2STHREADS : C2THREADS, 1)
    cols2_kernel(const int* __restrict__ mid_in, float* __restrict__ dst, Geometry g, Taps t, Tiling tl,
                 const __grid_constant__ CUtensorMap omap, const __grid_constant__ CUtensorMap mmap) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t tmem_base_s;
  __shared__ __align__(8) uint64_t lfull[C2PF], lempty[C2PF];
  __shared__ uint32_t ring_cnt[4];  // ring bands written, per lane quadrant (monotonic: cannot alias)
  // output bands finished by output group g in lane quadrant q (monotonic).  The loader of a
  // quadrant waits only for the three output warps that read its TMEM lanes: one ld.acquire per
  // output band instead of an mbarrier all four quadrants arrive on.
  __shared__ uint32_t out_cnt[4][CG];
  // SPLIT hand-offs per lane quadrant: pairs whose end-of-pair column prefix is published,
  // pairs released to the output groups (with their band copies made), and the prefixes
  __shared__ uint32_t lcarry_cnt[4], pair_done[4];
  __shared__ int lcarry_s[2][WS];
  constexpr int NLW = SPLIT ? 8 : 4;  // loader warps
  const int ch = blockIdx.x % g.in_px;
  const int sidx = blockIdx.x / g.in_px;
  const int strip = sidx % tl.nstrips;
  const long long item = sidx / tl.nstrips;
  const int x0 = strip * WS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3;  // TMEM lane quadrant: columns 32q .. 32q+31
  const int c = 32 * q + lane;
  const int xc = (x0 + c) < g.W ? x0 + c : g.W - 1;  // inactive lanes mirror a valid column (no stores)
  const int wh = g.oy1 - g.oy0;
  const long long total = (long long)g.nimg * wh;
  const long long T0 = item * tl.rows_per_item;
  const long long T1 = min(T0 + tl.rows_per_item, total);
  const int D = tl.D, NB = D / HB, PF = tl.pf, DS = tl.ds;
  unsigned char* abase = smem + (((smem_u32(smem) + 127u) & ~127u) - smem_u32(smem));  // TMA: 128-byte aligned
  int* lring = (int*)abase;                   // [PF][2][HB][WS] plane band pairs (TMA tensor loads)
  int* dring = lring + PF * 2 * HB * WS;      // [DS + 1][HB][WS] copies of old ring bands (+ mirror of slot 0)
  float* obuf = (float*)(abase + tl.obuf_off);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) ring_cnt[i] = 0;
    for (int i = 0; i < 4 * CG; ++i) (&out_cnt[0][0])[i] = 0;
    for (int i = 0; i < 4; ++i) lcarry_cnt[i] = pair_done[i] = 0;
    for (int i = 0; i < PF; ++i) {
      mbar_init(&lfull[i], 1);   // the issuing thread's expect_tx + the TMA bytes
      mbar_init(&lempty[i], 4);  // one arrive per loader warp
    }
  }
  if (warp == 0) tmem_alloc(&tmem_base_s, (uint32_t)tl.tmem_cols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tlane = tmem_base_s + ((uint32_t)q << 21);

  if (SPLIT && warp < NLW) {
    // ------------------------------------------------ loader, two halves alternating pairs
    const int h = warp >> 2;
    SegIter sc, so;  // ring bands / the output bands whose completion gates the ring
    sc.init(T0, T1, wh, g.oy0, t.pmax);
    so.init(T0, T1, wh, g.oy0, t.pmax);
    uint32_t v = 0;  // global ring band of the next pair's first band
    uint32_t G = 0;  // global pair index: pair G is staged in TMA slot G % PF, use G / PF
    int og = 0, oob = 0;
    uint32_t ocnt = 0;
    int slot = 0;                           // v % NB
    int cslot = tl.copy_e % NB, dslot = 0;  // as in the one-half loader (every warp tracks them)
    const int dist = PF - 2;                // a half issues its pairs dist pairs ahead (PF even, >= 4)
    for (; sc.valid; sc.next()) {
      const int* mcol = mid_in + ch * g.mid_ch + (long long)sc.img * g.mid_img + xc;
      const long long mrow = g.mid_row;
      const int vstart = sc.a - 1 - t.pmax;
      const int zc = ch * g.nimg + sc.img;
      const int npairs = (sc.nbands + 1) / 2;
      const uint32_t G0 = G;
      // pair pp of this segment, by lane 0 of the q = 0 warp of the half that owns it
      auto issue = [&](int pp) {
        if (q == 0 && lane == 0 && pp < npairs) {
          const uint32_t Gi = G0 + (uint32_t)pp;
          const int is = (int)(Gi % (uint32_t)PF);
          mbar_wait(&lempty[is], ((Gi / (uint32_t)PF) & 1) ^ 1);
          mbar_expect_tx(&lfull[is], 2 * HB * WS * 4);
          tma_load_3d(lring + is * (2 * HB * WS), &mmap, x0, vstart + pp * 2 * HB, zc, &lfull[is]);
        }
      };
      for (int pp = 0; pp < dist && pp < npairs; ++pp)
        if (((G0 + (uint32_t)pp) & 1u) == (uint32_t)h) issue(pp);
      for (int pp = 0; pp < npairs; ++pp, ++G) {
        const int nbp = min(2, sc.nbands - 2 * pp);  // bands in this pair
        bool cp[2] = {false, false};
        if (DS > 0) {
#pragma unroll
          for (int d = 0; d < 2; ++d) cp[d] = d < nbp && (long long)v + d >= (long long)NB - tl.copy_e;
        }
        if ((G & 1u) == (uint32_t)h) {
          issue(pp + dist);
          // every output band reading ring bands v+d - NB from TMEM is done
          while (so.valid && (long long)(so.gb0 + (uint32_t)oob) + tl.lag <= (long long)v + nbp - 1) {
            wait_above(&out_cnt[q][og], ocnt, false);
            if (++og == CG) {
              og = 0;
              ++ocnt;
            }
            if (++oob == (so.b - so.a + HB - 1) / HB) {
              so.next();
              oob = 0;
            }
          }
          tmem_fence_after();
          const int ls = (int)(G % (uint32_t)PF);
          uint32_t cv[2][HB];
          mbar_wait(&lfull[ls], (G / (uint32_t)PF) & 1);
          int cprefix = 0;  // prefix within the pair; the carry of the earlier pairs is added below
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            if (d >= nbp) break;
            const int v0 = vstart + (2 * pp + d) * HB;
            if (v0 >= 0 && v0 + HB <= g.H) {
              const int* lp = lring + ls * (2 * HB * WS) + d * (HB * WS) + c;
              int e[HB];
#pragma unroll
              for (int r = 0; r < HB; ++r) e[r] = lp[r * WS];
              int odd = cprefix;
#pragma unroll
              for (int r = 0; r < HB; r += 2) {
                cv[d][r] = (uint32_t)(odd + e[r]);
                odd = odd + e[r] + e[r + 1];
                cv[d][r + 1] = (uint32_t)odd;
              }
              cprefix = odd;
            } else {
              // rows beyond the image edges replicate the border row (filtering.py:10-13)
#pragma unroll
              for (int r = 0; r < HB; ++r) {
                cprefix += __ldg(mcol + (long long)min(max(v0 + r, 0), g.H - 1) * mrow);
                cv[d][r] = (uint32_t)cprefix;
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&lempty[ls]);
          // the running prefix at the end of pair G - 1 (0 at a segment start); waiting also keeps
          // lcarry_cnt monotonic
          if (G > 0) wait_above(&lcarry_cnt[q], G - 1, false);
          const int carry = pp > 0 ? lcarry_s[h ^ 1][c] : 0;
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            if (d >= nbp) break;
#pragma unroll
            for (int r = 0; r < HB; ++r) cv[d][r] += (uint32_t)carry;
          }
          lcarry_s[h][c] = carry + cprefix;
          __syncwarp();
          if (lane == 0) st_release(&lcarry_cnt[q], G + 1);
          // with band copies, pair G - 1's copies leave the ring before this pair overwrites bands
          if (DS > 0 && G > 0) wait_above(&pair_done[q], G - 1, false);
          {
            int sl = slot;
#pragma unroll
            for (int d = 0; d < 2; ++d) {
              if (d >= nbp) break;
              tmem_st16(tlane + (uint32_t)(sl * HB), cv[d]);
              if (sl == 0) tmem_st16(tlane + (uint32_t)D, cv[d]);  // mirror: lag windows never wrap
              if (++sl == NB) sl = 0;
            }
          }
          tmem_wait_st();
          tmem_fence_before();
          __syncwarp();
          // releases in band order
          if (DS == 0 && G > 0) wait_above(&pair_done[q], G - 1, false);
          if (lane == 0) st_release(&ring_cnt[q], v + (uint32_t)nbp);
          if (DS > 0) {
            uint32_t old[2][HB];
            int cs = cslot;
#pragma unroll
            for (int d = 0; d < 2; ++d) {
              if (d >= nbp) break;
              if (cp[d]) tmem_ld16(tlane + (uint32_t)(cs * HB), old[d]);
              if (++cs == NB) cs = 0;
            }
            tmem_wait_ld();
            int ds2 = dslot;
#pragma unroll
            for (int d = 0; d < 2; ++d) {
              if (d >= nbp) break;
              if (cp[d]) {
                int* dp = dring + ds2 * (HB * WS) + c;
#pragma unroll
                for (int r = 0; r < HB; ++r) dp[r * WS] = (int)old[d][r];
                if (ds2 == 0) {  // mirror of copy slot 0 after the last slot: trail windows never wrap
                  int* mp = dring + DS * (HB * WS) + c;
#pragma unroll
                  for (int r = 0; r < HB; ++r) mp[r * WS] = (int)old[d][r];
                }
                if (++ds2 == DS) ds2 = 0;
              }
            }
            tmem_fence_before();
            __syncwarp();
          }
          if (lane == 0) st_release(&pair_done[q], G + 1);
        }
        // ring / copy positions after this pair (every loader warp, also for the other half's pairs)
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          if (d >= nbp) break;
          if (++slot == NB) slot = 0;
          if (DS > 0) {
            if (cp[d] && ++dslot == DS) dslot = 0;
            if (++cslot == NB) cslot = 0;
          }
        }
        v += (uint32_t)nbp;
      }
    }
  } else if (!SPLIT && warp < 4) {
    // ------------------------------------------------ loader
    SegIter sc, so;  // ring bands / the output bands whose completion gates the ring
    sc.init(T0, T1, wh, g.oy0, t.pmax);
    so.init(T0, T1, wh, g.oy0, t.pmax);
    uint32_t v = 0;  // global ring band
    int og = 0;         // next output band to observe: the ocnt-th band of output group og,
    uint32_t ocnt = 0;  // band oob of segment so
    int oob = 0;
    int slot = 0;
    // plane bands arrive in pairs by TMA (one 32 x 128 box, issued PF-1 pairs ahead by
    // thread 0) into PF slots with full (tx bytes) / empty (one arrive per warp) barriers;
    // a pair shares one lfull wait, one tcgen05.wait::st and one batch of copies
    int lslot = 0, islot = 0;
    uint32_t lph = 0, iph = 0;
    int cslot = tl.copy_e % NB, dslot = 0;  // ring slot (v + copy_e) % NB and copy slot of the next band copy
    for (; sc.valid; sc.next()) {
      const int* mcol = mid_in + ch * g.mid_ch + (long long)sc.img * g.mid_img + xc;
      const long long mrow = g.mid_row;
      const int vstart = sc.a - 1 - t.pmax;
      const int zc = ch * g.nimg + sc.img;
      const int npairs = (sc.nbands + 1) / 2;
      auto issue = [&](int pp) {
        if (threadIdx.x == 0 && pp < npairs) {
          mbar_wait(&lempty[islot], iph ^ 1);
          mbar_expect_tx(&lfull[islot], 2 * HB * WS * 4);
          tma_load_3d(lring + islot * (2 * HB * WS), &mmap, x0, vstart + pp * 2 * HB, zc, &lfull[islot]);
        }
        if (pp < npairs && ++islot == PF) {
          islot = 0;
          iph ^= 1;
        }
      };
      for (int pp = 0; pp < PF - 1; ++pp) issue(pp);
      int cprefix = 0;
      for (int pp = 0; pp < npairs; ++pp) {
        issue(pp + PF - 1);
        const int nbp = min(2, sc.nbands - 2 * pp);  // bands in this pair
        // every output band reading ring bands v+d - NB from TMEM is done
        while (so.valid && (long long)(so.gb0 + (uint32_t)oob) + tl.lag <= (long long)v + nbp - 1) {
          wait_above(&out_cnt[q][og], ocnt, false);
          if (++og == CG) {
            og = 0;
            ++ocnt;
          }
          if (++oob == (so.b - so.a + HB - 1) / HB) {
            so.next();
            oob = 0;
          }
        }
        tmem_fence_after();  // the ring stores below are ordered after the readers' release
        uint32_t cv[2][HB];
        mbar_wait(&lfull[lslot], lph);
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          if (d >= nbp) break;
          const int v0 = vstart + (2 * pp + d) * HB;
          if (v0 >= 0 && v0 + HB <= g.H) {
            const int* lp = lring + lslot * (2 * HB * WS) + d * (HB * WS) + c;
            int e[HB];
#pragma unroll
            for (int r = 0; r < HB; ++r) e[r] = lp[r * WS];
            // running prefix with a two-element stride: odd entries chain by 3-input adds,
            // even entries hang off them (dependency depth 9 instead of 16)
            int odd = cprefix;
#pragma unroll
            for (int r = 0; r < HB; r += 2) {
              cv[d][r] = (uint32_t)(odd + e[r]);
              odd = odd + e[r] + e[r + 1];
              cv[d][r + 1] = (uint32_t)odd;
            }
            cprefix = odd;
          } else {
            // rows beyond the image edges replicate the border row (filtering.py:10-13)
#pragma unroll
            for (int r = 0; r < HB; ++r) {
              cprefix += __ldg(mcol + (long long)min(max(v0 + r, 0), g.H - 1) * mrow);
              cv[d][r] = (uint32_t)cprefix;
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&lempty[lslot]);
        if (++lslot == PF) {
          lslot = 0;
          lph ^= 1;
        }
        const int slot0 = slot;
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          if (d >= nbp) break;
          tmem_st16(tlane + (uint32_t)(slot * HB), cv[d]);
          if (slot == 0) tmem_st16(tlane + (uint32_t)D, cv[d]);  // mirror: lag windows never wrap
          if (++slot == NB) slot = 0;
        }
        tmem_wait_st();
        tmem_fence_before();
        __syncwarp();
        if (lane == 0) st_release(&ring_cnt[q], v + (uint32_t)nbp);  // this quadrant's bands < v + nbp
        (void)slot0;
        if (DS > 0) {
          // after releasing band v: copy band u = v - NB + copy_e out of the ring (its
          // readers wait for band v + 1 or later; see cols_prefix_tiling)
          uint32_t old[2][HB];
          bool cp[2] = {false, false};
          int cs = cslot;
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            if (d >= nbp) break;
            cp[d] = (long long)v + d >= (long long)NB - tl.copy_e;
            if (cp[d]) tmem_ld16(tlane + (uint32_t)(cs * HB), old[d]);
            if (++cs == NB) cs = 0;
          }
          tmem_wait_ld();
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            if (d >= nbp) break;
            if (cp[d]) {
              int* dp = dring + dslot * (HB * WS) + c;
#pragma unroll
              for (int r = 0; r < HB; ++r) dp[r * WS] = (int)old[d][r];
              if (dslot == 0) {  // mirror of copy slot 0 after the last slot: trail windows never wrap
                int* mp = dring + DS * (HB * WS) + c;
#pragma unroll
                for (int r = 0; r < HB; ++r) mp[r * WS] = (int)old[d][r];
              }
              if (++dslot == DS) dslot = 0;
            }
            if (++cslot == NB) cslot = 0;
          }
        }
        v += (uint32_t)nbp;
      }
    }
  } else {
    // ------------------------------------------------ output groups
    const int grp = (warp - NLW) / 4;
    const int ow = warp - NLW;  // output warp 0 .. 4*CG-1 (staging buffers)
    uint32_t onum = 0;
    int obsel = 0;
    SegIter so;
    so.init(T0, T1, wh, g.oy0, t.pmax);
    for (; so.valid; so.next()) {
      const int nout = (so.b - so.a + HB - 1) / HB;
      for (int ob = 0; ob < nout; ++ob, ++onum) {
        if ((int)(onum % CG) != grp) continue;
        const int out_next = so.a + ob * HB;
        const int nb = min(HB, so.b - out_next);
        const uint32_t j = so.gb0 + (uint32_t)ob;  // ring band of the band's deepest trail row
        const uint32_t need = so.gb0 + (uint32_t)((ob * HB + nb + 2 * t.pmax) / HB);
        // one monotonic count per lane quadrant (the loader fills the ring in order).  Without
        // band copies (ring only, e.g. C4) the groups back off so their polling leaves issue
        // slots to the loader (C4 1.231 -> 1.181 ms); with copies (C5) the ring is tight and
        // the loader waits on the groups, so they spin.
        wait_above(&ring_cnt[q], need, DS == 0);
        tmem_fence_after();
        const int base = (int)(j % (uint32_t)NB) * HB;  // ring position of virtual row 16*ob
        float2 o2[HB / 2];
        // boxes in pairs: both boxes' TMEM windows are in flight under one tcgen05.wait
#pragma unroll
        for (int i0 = 0; i0 < K; i0 += 2) {
        uint32_t lvp[2][HB], tvp[2][HB];
#pragma unroll
        for (int d2 = 0; d2 < 2; ++d2) {
          const int i = i0 + d2;
          if (i >= K) break;
          int l = base + t.pmax + 1 + t.p[i];
          l = l >= D ? l - D : l;
          l = l >= D ? l - D : l;
          SB_ASSERT(l >= 0 && l < D);
          tmem_ld16(tlane + (uint32_t)l, lvp[d2]);
          if (!((tl.deepmask >> i) & 1)) {
            int tr = base + t.pmax - t.p[i];
            tr = tr >= D ? tr - D : tr;
            tmem_ld16(tlane + (uint32_t)tr, tvp[d2]);
          }
        }
        tmem_wait_ld();
#pragma unroll
        for (int d2 = 0; d2 < 2; ++d2) {
          const int i = i0 + d2;
          if (i >= K) break;
          uint32_t (&lv)[HB] = lvp[d2];
          uint32_t (&tv)[HB] = tvp[d2];
          const bool deep = (tl.deepmask >> i) & 1;
          if (deep) {
            // virtual rows 16*ob + pmax - p_i .. +15 from the band copies (band j + off/16 on)
            const int off = t.pmax - t.p[i];
            const uint32_t u0 = j + (uint32_t)(off / HB);
            const int r0 = off % HB;
            const int s0 = (int)(u0 % (uint32_t)DS);
            SB_ASSERT(DS > 0 && s0 < DS);
            // rows s0*HB + r0 .. +15 of the linear copy ring (slot 0 is mirrored after slot DS-1)
            const int* p0 = dring + (s0 * HB + r0) * WS + c;
#pragma unroll
            for (int r = 0; r < HB; ++r) tv[r] = (uint32_t)p0[r * WS];
          }
          const float2 w2 = make_float2(t.w_col[i], t.w_col[i]);
#pragma unroll
          for (int r = 0; r < HB / 2; ++r) {
            const float2 d = make_float2(i2f_fast(lv[2 * r] - tv[2 * r]), i2f_fast(lv[2 * r + 1] - tv[2 * r + 1]));
            o2[r] = i == 0 ? __fmul2_rn(w2, d) : __ffma2_rn(w2, d, o2[r]);
          }
        }
        }
        // this warp's windows of the band are read (tcgen05.wait::ld above): the loader may
        // overwrite the ring bands only this band still needed
        tmem_fence_before();
        __syncwarp();
        if (lane == 0) st_release(&out_cnt[q][grp], onum / CG + 1);
        if (g.out_bulk && nb == HB) {
          float* obp = obuf + (ow * 2 + obsel) * (HB * 32);
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
#pragma unroll
          for (int r = 0; r < HB / 2; ++r) {
            obp[(2 * r) * 32 + lane] = o2[r].x;
            obp[(2 * r + 1) * 32 + lane] = o2[r].y;
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&omap, obp, x0 + 32 * q, out_next - g.oy0, so.img);
            bulk_commit();
          }
          obsel ^= 1;
        } else if (x0 + c < g.W) {
          float* dptr = dst + (long long)so.img * g.out_img + (long long)(out_next - g.oy0) * g.out_row +
                        (long long)(x0 + c) * g.out_px + ch;
          const long long step = g.out_row;
#pragma unroll
          for (int r = 0; r < HB / 2; ++r) {
            if (2 * r < nb) st_stream(dptr, o2[r].x);
            dptr += step;
            if (2 * r + 1 < nb) st_stream(dptr, o2[r].y);
            dptr += step;
          }
        }
      }
    }
    // observe the remaining ring bands so no full phase is left pending (not needed for
    // correctness: the CTA ends here) and retire the stores
    if (lane == 0) bulk_wait_read<0>();
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem_base_s, (uint32_t)tl.tmem_cols);
}

// ---------------------------------------------------------------- streaming row pass (large radii)
// RowsToMid for radii too large for the fused sweep.  A CTA owns a band of HB
// rows and streams its full width in chunks of CW columns, so the 2*pmax+1
// halo is paid once per row instead of once per strip: producer warp pw stages
// and prefix-scans rows 8pw..8pw+7 of each chunk (the row prefix carried across
// chunks) into a ring of RL prefix columns; consumer thread c emits column
// o*CW + c of output chunk o once the chunk holding its lead prefix is scanned.
// Virtual column q = x - xs with xs = the first column of the left halo
// (rounded down to 16 so cp.async stays aligned); columns outside [0, W)
// replicate the border (filtering.py:10-13).
constexpr int CW = 128;    // chunk width (= consumer threads)
constexpr int RL = 1024;   // prefix ring length (power of two, >= 3*CW + 2*pmax + 2)

constexpr int NSLOT = RL / CW;  // ring chunk slots; one full/done mbarrier per slot (no phase aliasing)
constexpr int RLS = RL + 4;     // prefix ring row stride in words: 4112 B = 16 (mod 128)
constexpr int SRB_PAD = 16;     // staged rows are CW*4 + 16 bytes apart: 16 (mod 128)
// staged input chunks per producer warp: each warp keeps STG - 1 chunks (8 rows x CW) in flight
// while it scans one, so the bytes in flight per SM cover the DRAM latency
#ifndef SB_STREAM_STAGES
#define SB_STREAM_STAGES 4
#endif
constexpr int STG = SB_STREAM_STAGES;
// float64 sources stage 8-byte elements: two chunks keep the CTA below half an SM's shared memory
constexpr int stream_stages(size_t es) { return es == 8 ? 2 : STG; }
// consumer warps: SRG row groups of CW threads; group rg forms rows [rg * HB / SRG, (rg + 1) * HB / SRG)
// of each output chunk.  Two groups (8 rows per thread, 20 warps per SM instead of 12) measured
// 3.7 % slower on C5 (4.416 vs 4.257 ms): the per-thread address work doubles.  Default 1.
#ifndef SB_STREAM_ROWGROUPS
#define SB_STREAM_ROWGROUPS 1
#endif
constexpr int SRG = SB_STREAM_ROWGROUPS;
constexpr int SCONS = SRG * (CW / 32);
constexpr int STREAM_THREADS = 32 * (SCONS + NPROD);
constexpr int SHB = HB / SRG;  // rows per consumer thread

// The two words a consumer stores for a row pair: the row values rounded to the mid quantum
// (int32 plane), or their float bits (row pass alone).
template <int K, bool TO_OUT>
__device__ __forceinline__ int2 plane_words(float2 rv) {
  if constexpr (TO_OUT) {
    return make_int2(__float_as_int(rv.x), __float_as_int(rv.y));
  } else {
    const float2 q = round_mid2<K>(rv);  // round to the mid quantum
    return make_int2(__float_as_int(q.x) - kMagicBits, __float_as_int(q.y) - kMagicBits);
  }
}

// TO_OUT: the row pass alone (`_filter_rows`, filtering.py:48-64): weights in pixel units and
// the float row values stored as they are (mid_out is then the float destination, g.mid_row its
// row stride), exactly as rows_kernel<.., RowsToOut> forms them.
template <typename Tin, int K, bool TO_OUT = false>
__global__ void __launch_bounds__(STREAM_THREADS, 2)
    stream_rows_kernel(const Tin* __restrict__ src, int* __restrict__ mid_out, Geometry g, Taps t, int xs,
                       int nbands_total, int segw, int* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar_full[NSLOT], bar_done[NSLOT];
  constexpr int STG = stream_stages(sizeof(Tin));  // staged chunks per producer warp (float64: two CTAs per SM)
  const int warp = threadIdx.x >> 5;
  const bool producer = warp >= SCONS;
  // A unit is (band, column segment): segment s covers columns [s * segw, min(W, (s + 1) * segw))
  // and restarts the row prefix at its own left halo, so images with few rows still fill the
  // SMs (segw >= W: one segment, the whole row).
  const int nseg = (g.W + segw - 1) / segw;
  // output chunk o reads prefix columns of input chunks o .. o + lagc
  const int lagc = (CW - 1 - xs + t.pmax) / CW;
  // staged rows and prefix-ring rows are an odd multiple of 16 bytes apart, so the 8 lanes
  // of a 128-bit access phase (8 rows, same chunk) hit 8 distinct bank groups
  // unal: one channel, rows that are not 16-byte multiples, 16-byte aligned base.  A row's
  // chunk is then staged from its start rounded down to 16 bytes (VPR + 1 vectors; the shift is
  // the same for every chunk of the row) and the scan reads element by element behind the
  // shift; a chunk is interior only while the extra vector lies inside the image row.
  const bool unal = g.in_px == 1 && !g.aligned16 && ((size_t)src & 15) == 0;
  const int rowbytes = CW * (int)sizeof(Tin) + SRB_PAD + (unal ? 16 : 0);
  const int pad_el = unal ? (16 + (int)sizeof(Tin) - 1) / (int)sizeof(Tin) : 0;
  __shared__ const Tin* rowp_sh[NPROD][8];
  unsigned char* stage = smem;                           // [NPROD][STG][8][rowbytes]
  int* P = (int*)(smem + NPROD * STG * 8 * rowbytes);    // [HB][RLS]

  if (threadIdx.x == 0) {
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&bar_full[i], 32 * NPROD);
      mbar_init(&bar_done[i], 32 * SCONS);
    }
  }
  __syncthreads();

  const int ch = blockIdx.x % g.in_px;  // channel fastest (see cols_kernel)
  uint32_t cin_ctr = 0, out_ctr = 0;    // input chunks / output chunks completed by this CTA
  const int nblk = gridDim.x / g.in_px;
  for (int unit = blockIdx.x / g.in_px; unit < nbands_total * nseg; unit += nblk) {
    const int band = unit / nseg;
    const int x_begin = (unit - band * nseg) * segw, x_end = min(g.W, x_begin + segw);
    const int qtotal = (x_end - x_begin) - xs + t.pmax;  // virtual columns q = x - x_begin - xs
    const int nin = (qtotal + CW - 1) / CW;
    const int nout = (x_end - x_begin + CW - 1) / CW;
    const long long row0 = (long long)band * HB;
    const int nrows = (int)min((long long)HB, (long long)g.nimg * g.H - row0);
    if (producer) {
      const int lane = threadIdx.x & 31, pw = warp - SCONS;
      unsigned char* mystage = stage + pw * STG * 8 * rowbytes;
      // this warp's 8 source rows (clamped at the end of the tall image) - hoisted per band
      const Tin* rowp[8];
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        const long long trow = row0 + min(8 * pw + rr, nrows - 1);
        const int img = (int)(trow / g.H), v = (int)(trow - (long long)img * g.H);
        rowp[rr] = src + (long long)img * g.in_img + (long long)v * g.in_row + ch;
      }
      const bool vec = g.aligned16 && g.in_px == 1;
      if (unal) {
        __syncwarp();
        if (lane < 8) {
          const long long trow = row0 + min(8 * pw + lane, nrows - 1);
          const int img = (int)(trow / g.H), v = (int)(trow - (long long)img * g.H);
          rowp_sh[pw][lane] = src + (long long)img * g.in_img + (long long)v * g.in_row;
        }
        __syncwarp();
      }
      // this lane's row starts (size_t)row & 15 bytes behind a 16-byte boundary (chunk starts are
      // 16-column multiples, so the shift does not depend on the chunk)
      const int mysh = unal ? (int)((size_t)rowp_sh[pw][lane & 7] & 15) : 0;
      auto issue = [&](int j, int buf) {
        const int xq0 = x_begin + xs + j * CW;  // 16-aligned first column of chunk j
        if (vec && xq0 >= 0 && xq0 + CW <= g.W) {
          // interior chunk: 16-byte copies, 8 rows x VPR vectors (xq0 is a multiple of 16 columns)
          constexpr int VPR = CW * (int)sizeof(Tin) / 16;
#pragma unroll
          for (int it = 0; it < 8 * VPR / 32; ++it) {
            const int idx = lane + 32 * it;
            const int rr = idx / VPR, e4 = idx - rr * VPR;
            cp_async16(mystage + (buf * 8 + rr) * rowbytes + 16 * e4,
                       (const unsigned char*)(rowp[rr] + xq0) + 16 * e4);
          }
        } else if (unal && xq0 >= 0 && xq0 + CW + pad_el <= g.W) {
          constexpr int VPR1 = CW * (int)sizeof(Tin) / 16 + 1;
          for (int idx = lane; idx < 8 * VPR1; idx += 32) {
            const int rr = idx / VPR1, e4 = idx - rr * VPR1;
            const unsigned char* a = (const unsigned char*)(rowp_sh[pw][rr] + xq0);
            cp_async16(mystage + (buf * 8 + rr) * rowbytes + 16 * e4, a - ((size_t)a & 15) + 16 * e4);
          }
        } else {
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) {
            Tin* sp = (Tin*)(mystage + (buf * 8 + rr) * rowbytes + (unal ? (int)((size_t)rowp[rr] & 15) : 0));
            for (int e = lane; e < CW; e += 32) {
              const int x = min(max(xq0 + e, 0), g.W - 1);  // replicate border columns
              const Tin* gp = rowp[rr] + (long long)x * g.in_px;
              if constexpr (sizeof(Tin) == 4) {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(sp + e)), "l"(gp));
              } else {
                sp[e] = *gp;
              }
            }
          }
        }
        cp_async_commit();
      };
      // lane -> row rr = lane & 7 of this warp's 8 and chunk (lane >> 3) + 4*pass of the 8
      // CH-column chunks; the row's running prefix (carry) lives in the 4 lanes of that row
      int carry = 0;
      // one commit group per chunk (empty past the end), so "at most STG - 2 groups pending"
      // always means chunk j has landed
#pragma unroll
      for (int j = 0; j < STG - 1; ++j) {
        if (j < nin)
          issue(j, j);
        else
          cp_async_commit();
      }
      RangeAcc bad;
      int sbuf = 0;  // j % STG
      for (int j = 0; j < nin; ++j) {
        const uint32_t gj = cin_ctr + j;
        cp_async_wait<STG - 2>();
        __syncwarp();  // every lane has read chunk j - 1: its buffer takes chunk j + STG - 1
        if (j + STG - 1 < nin)
          issue(j + STG - 1, sbuf == 0 ? STG - 1 : sbuf - 1);
        else
          cp_async_commit();
        if (j >= NSLOT) {  // ring slot of chunk j last served output chunk j - NSLOT
          const uint32_t go = out_ctr + (j - NSLOT);
          mbar_wait(&bar_done[go % NSLOT], (go / NSLOT) & 1);
        }
        const unsigned char* cur = mystage + sbuf * 8 * rowbytes;
        sbuf = sbuf + 1 == STG ? 0 : sbuf + 1;
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
          const int rr = lane & 7, sc = (lane >> 3) + 4 * pass;
          // the lane's CH elements by 16-byte shared-memory loads (staged rows and sub-chunks are
          // 16-byte aligned for every element size)
          union {
            uint4 q[CH * sizeof(Tin) / 16];
            Tin e[CH];
          } u;
          if (!unal) {
            const uint4* ep = (const uint4*)(cur + rr * rowbytes + sc * CH * (int)sizeof(Tin));
#pragma unroll
            for (int m = 0; m < (int)(CH * sizeof(Tin) / 16); ++m) u.q[m] = ep[m];
          } else {
            const Tin* ee = (const Tin*)(cur + rr * rowbytes + mysh) + sc * CH;
#pragma unroll
            for (int m = 0; m < CH; ++m) u.e[m] = ee[m];
          }
          int v[CH];
          int tot = 0;
#pragma unroll
          for (int m = 0; m < CH; ++m) {
            tot += to_fixed<Tin>(u.e[m], t, bad);
            v[m] = tot;
          }
          // inclusive scan of the chunk totals over the row's 4 lanes (rr, rr+8, rr+16, rr+24)
          int inc = tot;
          int y = __shfl_up_sync(0xffffffffu, inc, 8);
          if (lane >= 8) inc += y;
          y = __shfl_up_sync(0xffffffffu, inc, 16);
          if (lane >= 16) inc += y;
          const int off = carry + inc - tot;
          int* dst = P + (8 * pw + rr) * RLS + ((j * CW + sc * CH) & (RL - 1));
#pragma unroll
          for (int m = 0; m < CH / 4; ++m)
            ((int4*)dst)[m] = make_int4(v[4 * m] + off, v[4 * m + 1] + off, v[4 * m + 2] + off, v[4 * m + 3] + off);
          carry += __shfl_sync(0xffffffffu, inc, rr + 24);  // the row's total over these 4 chunks
        }
        mbar_arrive(&bar_full[gj % NSLOT]);
      }
      report_status(status, bad, t);
    } else {
      const int c = threadIdx.x & (CW - 1);
      const int r0 = (threadIdx.x / CW) * SHB;  // this thread's rows [r0, r0 + SHB) of the band
      // destination of tall row t: a full band inside one image is HB rows one plane row apart
      // (one pointer stepped by the row stride); other bands address every row
      auto midrow_of = [&](int r) {
        const long long trow = row0 + min(r, nrows - 1);
        const int img = (int)(trow / g.H), v = (int)(trow - (long long)img * g.H);
        return mid_out + ch * g.mid_ch + (long long)img * g.mid_img + (long long)v * g.mid_row;
      };
      const bool whole = nrows == HB && (row0 / g.H) == ((row0 + HB - 1) / g.H);
      const size_t mid0g = __cvta_generic_to_global(midrow_of(r0));
      // two output chunks per iteration: one wait (chunks complete in order), both chunks'
      // row values in flight together, then both done-arrivals and stores
      for (int o = 0; o < nout; o += 2) {
        const int no = min(2, nout - o);
        const uint32_t gj = cin_ctr + min(o + no - 1 + lagc, nin - 1);
        mbar_wait(&bar_full[gj % NSLOT], (gj / NSLOT) & 1);
        float2 rv[2][SHB / 2];  // rows r0 + (2r, 2r+1) of chunks o, o+1: packed FMUL2 / FFMA2 / FADD2
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h >= no) break;
          const int x = x_begin + (o + h) * CW + c;
#pragma unroll
          for (int i = 0; i < K; ++i) {
            const int* pl = P + r0 * RLS + ((x - x_begin - xs + t.p[i]) & (RL - 1));
            const int* pt = P + r0 * RLS + ((x - x_begin - xs - t.p[i] - 1) & (RL - 1));
            const float wi = TO_OUT ? t.w_out1[i] : t.w_row[i];
            const float2 w2 = make_float2(wi, wi);
#pragma unroll
            for (int r = 0; r < SHB / 2; ++r) {
              const float2 d = make_float2(i2f_fast((uint32_t)(pl[2 * r * RLS] - pt[2 * r * RLS])),
                                           i2f_fast((uint32_t)(pl[(2 * r + 1) * RLS] - pt[(2 * r + 1) * RLS])));
              rv[h][r] = i == 0 ? __fmul2_rn(w2, d) : __ffma2_rn(w2, d, rv[h][r]);
            }
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h >= no) break;
          const uint32_t go = out_ctr + o + h;
          mbar_arrive(&bar_done[go % NSLOT]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h >= no) break;
          const int x = x_begin + (o + h) * CW + c;
          if (x < x_end) {
            if (whole) {
              // 32-bit element offsets from the band's first row (HB plane rows < 2^31 elements):
              // one IMAD.WIDE per store instead of a 64-bit pointer chain
              const int ms = (int)g.mid_row;
              int idx = x;
#pragma unroll
              for (int r = 0; r < SHB / 2; ++r) {
                const int2 q = plane_words<K, TO_OUT>(rv[h][r]);
                st_global_idx(mid0g, idx, q.x);
                st_global_idx(mid0g, idx + ms, q.y);
                idx += 2 * ms;
              }
            } else {
#pragma unroll
              for (int r = 0; r < SHB / 2; ++r) {
                const int2 q = plane_words<K, TO_OUT>(rv[h][r]);
                if (r0 + 2 * r < nrows) midrow_of(r0 + 2 * r)[x] = q.x;
                if (r0 + 2 * r + 1 < nrows) midrow_of(r0 + 2 * r + 1)[x] = q.y;
              }
            }
          }
        }
      }
    }
    cin_ctr += (uint32_t)nin;
    out_ctr += (uint32_t)nout;
    __syncthreads();  // the next band restarts the ring and the carries
  }
}

// ---------------------------------------------------------------- streaming row pass, interleaved channels
// Sources with C = 2..4 interleaved channels and 16-byte aligned rows (C4; any element type).  The band
// is HB VIRTUAL rows vr = t * C + ch (tall row t, channel ch), so a band touches at most
// HB / C + 2 image rows.  The two producer warps stage those rows ONCE per chunk, interleaved
// as they lie in memory (16-byte cp.async; the per-element 4-byte gather of
// stream_rows_kernel left the consumers waiting for the producers 58 % of the time on C4),
// and each scan lane reads its channel out of the staged row with stride C.  Prefix ring,
// consumers and hand-offs are those of stream_rows_kernel; the int32 plane is
// [channel][tall row][W], dense, below 2^31 elements (32-bit store offsets).
constexpr int mc_rows(int C) { return (HB + C - 1) / C + 1; }

template <typename Tin, int K>
__global__ void __launch_bounds__(STREAM_THREADS, 2)
    stream_rows_mc_kernel(const Tin* __restrict__ src, int* __restrict__ mid_out, Geometry g, Taps t, int xs,
                          int nbands_total, int segw, int unal, int* status) {
  static_assert(SRG == 1, "the interleaved streaming row pass assumes one consumer row group");
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar_full[NSLOT], bar_done[NSLOT];
  constexpr int STG = stream_stages(sizeof(Tin));
  constexpr int ES = (int)sizeof(Tin);
  __shared__ __align__(8) uint64_t sfull[STG];  // staged chunk landed (bulk-copy bytes / edge-chunk arrive)
  __shared__ const Tin* rowp_s[HB / 2 + 2];     // the band's image rows (clamped at the end of the tall image)
  // unal: image rows that are not 16-byte multiples.  Row i is then staged from its chunk start
  // rounded down to 16 bytes (rowsh_s[i] bytes early, the same for every chunk of the row) and
  // padded to 16 bytes behind, so the bulk copies stay aligned; the scan skips the shift.  A
  // chunk counts as interior only if the padding still lies inside the image row.
  __shared__ int rowsh_s[HB / 2 + 2];
  const int warp = threadIdx.x >> 5;
  const bool producer = warp >= SCONS;
  const int C = g.in_px;
  const int nseg = (g.W + segw - 1) / segw;  // column segments per band (see stream_rows_kernel)
  const int lagc = (CW - 1 - xs + t.pmax) / CW;
  const int ntmax = (HB + C - 1) / C + 1;
  const int srb = CW * C * ES + SRB_PAD + (unal ? 16 : 0);  // staged image row: CW pixels of C elements (+ padding)
  const int pad_px = unal ? (16 + C * ES - 1) / (C * ES) : 0;
  unsigned char* stage = smem;                // [STG][ntmax][srb]
  int* P = (int*)(smem + STG * ntmax * srb);  // [HB][RLS]
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&bar_full[i], 32 * NPROD);
      mbar_init(&bar_done[i], 32 * SCONS);
    }
    for (int i = 0; i < STG; ++i) mbar_init(&sfull[i], 1);
  }
  __syncthreads();

  const long long tall = (long long)g.nimg * g.H;
  const long long VR = tall * C;  // virtual rows
  uint32_t cin_ctr = 0, out_ctr = 0;
  for (int unit = blockIdx.x; unit < nbands_total * nseg; unit += gridDim.x) {
    const int band = unit / nseg;
    const int x_begin = (unit - band * nseg) * segw, x_end = min(g.W, x_begin + segw);
    const int qtotal = (x_end - x_begin) - xs + t.pmax;
    const int nin = (qtotal + CW - 1) / CW;
    const int nout = (x_end - x_begin + CW - 1) / CW;
    const long long vr0 = (long long)band * HB;
    const int nrows = (int)min((long long)HB, VR - vr0);
    const long long t_first = vr0 / C;
    const int c_first = (int)(vr0 - t_first * C);
    const int nt = (int)((vr0 + nrows - 1) / C - t_first) + 1;  // image rows of this band
    if (producer) {
      const int lane = threadIdx.x & 31, pw = warp - SCONS, ptid = pw * 32 + lane;
      if (ptid < nt) {
        const long long tt = t_first + ptid;
        const int img = (int)(tt / g.H), v = (int)(tt - (long long)img * g.H);
        const Tin* rp = src + (long long)img * g.in_img + (long long)v * g.in_row;
        rowp_s[ptid] = rp;
        rowsh_s[ptid] = unal ? (int)((size_t)rp & 15) : 0;
      }
      named_bar_sync(1, 32 * NPROD);
      uint32_t tx_band = 0;  // bytes one interior chunk brings in
      for (int i = 0; i < nt; ++i) tx_band += (uint32_t)((rowsh_s[i] + CW * C * ES + 15) & ~15);
      const int my_sh = ptid < nt ? rowsh_s[ptid] : 0;
      const Tin* my_rp = ptid < nt ? rowp_s[ptid] : src;
      // Chunk gc (counted over the CTA's bands) lives in staging buffer gc % STG; its landing is
      // phase gc / STG of sfull[gc % STG].  Interior chunks: one bulk copy per image row, issued
      // by one thread (expect_tx + complete_tx).  Edge chunks (border columns replicated,
      // filtering.py:10-13): 4-byte cp.async by all producer threads, waited for as a group; the
      // issuing thread completes the phase by a plain arrive so every buffer use is one phase.
      auto interior = [&](int j) {
        const int xq0 = x_begin + xs + j * CW;  // 16-aligned first column of chunk j
        return xq0 >= 0 && xq0 + CW + pad_px <= g.W;
      };
      auto issue = [&](int j) {
        const int xq0 = x_begin + xs + j * CW;
        const int buf = (int)((cin_ctr + (uint32_t)j) % STG);
        unsigned char* sbuf = stage + buf * ntmax * srb;
        if (interior(j)) {
          // lane i of the first producer warp copies image row i (the copies issue in parallel;
          // the expect_tx arrive is the phase's only pending arrival, so an early complete_tx
          // cannot complete it)
          if (ptid == 0) mbar_expect_tx(&sfull[buf], tx_band);
          if (ptid < nt)
            bulk_g2s(sbuf + ptid * srb, (const unsigned char*)(my_rp + (long long)xq0 * C) - my_sh,
                     (uint32_t)((my_sh + CW * C * ES + 15) & ~15), &sfull[buf]);
        } else {
          for (int i = 0; i < nt; ++i) {
            const Tin* rp = rowp_s[i];
            for (int e = ptid; e < CW * C; e += 32 * NPROD) {
              const int px = e / C, cc = e - px * C;
              const int x = min(max(xq0 + px, 0), g.W - 1);
              if constexpr (ES == 4)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                                 smem_u32(sbuf + i * srb + rowsh_s[i] + 4 * e)),
                             "l"(rp + (long long)x * C + cc));
              else
                *(Tin*)(sbuf + i * srb + rowsh_s[i] + ES * e) = rp[(long long)x * C + cc];  // visible after the named barrier
            }
          }
          cp_async_commit();
          if (ptid == 0) mbar_arrive(&sfull[buf]);
        }
      };
      // this lane's virtual row: band row 8 pw + rr (clamped), channel cc of staged image row srow
      const int rr = lane & 7;
      const long long vr = vr0 + min(8 * pw + rr, nrows - 1);
      const long long tt = vr / C;
      const int lane_off = (int)(tt - t_first) * srb + rowsh_s[(int)(tt - t_first)] + (int)(vr - tt * C) * ES;
      int carry = 0;
      for (int j = 0; j < STG - 1 && j < nin; ++j) issue(j);
      RangeAcc bad;
      for (int j = 0; j < nin; ++j) {
        const uint32_t gj = cin_ctr + j;
        const int sb = (int)(gj % STG);
        if (!interior(j)) cp_async_wait_all();
        mbar_wait(&sfull[sb], (gj / STG) & 1);
        // both warps have read chunk j - 1 (its buffer takes chunk j + STG - 1), and an edge
        // chunk's copies by the other warp are visible
        named_bar_sync(1, 32 * NPROD);
        if (j + STG - 1 < nin) issue(j + STG - 1);
        if (j >= NSLOT) {
          const uint32_t go = out_ctr + (j - NSLOT);
          mbar_wait(&bar_done[go % NSLOT], (go / NSLOT) & 1);
        }
        const unsigned char* cur = stage + sb * ntmax * srb + lane_off;
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
          const int sc = (lane >> 3) + 4 * pass;
          const Tin* e = (const Tin*)cur + sc * CH * C;
          int v[CH];
          int tot = 0;
#pragma unroll
          for (int m = 0; m < CH; ++m) {
            tot += to_fixed<Tin>(e[m * C], t, bad);
            v[m] = tot;
          }
          int inc = tot;
          int y = __shfl_up_sync(0xffffffffu, inc, 8);
          if (lane >= 8) inc += y;
          y = __shfl_up_sync(0xffffffffu, inc, 16);
          if (lane >= 16) inc += y;
          const int off = carry + inc - tot;
          int* dst = P + (8 * pw + rr) * RLS + ((j * CW + sc * CH) & (RL - 1));
#pragma unroll
          for (int m = 0; m < CH / 4; ++m)
            ((int4*)dst)[m] = make_int4(v[4 * m] + off, v[4 * m + 1] + off, v[4 * m + 2] + off, v[4 * m + 3] + off);
          carry += __shfl_sync(0xffffffffu, inc, rr + 24);
        }
        mbar_arrive(&bar_full[gj % NSLOT]);
      }
      report_status(status, bad, t);
    } else {
      const int c = threadIdx.x;
      const size_t midg = __cvta_generic_to_global(mid_out);
      const int off0 = (int)((long long)c_first * g.mid_ch + t_first * g.mid_row);  // plane offset of band row 0
      const int ch_step = (int)g.mid_ch, wrap_step = (int)(g.mid_row - (long long)C * g.mid_ch);
      for (int o = 0; o < nout; o += 2) {
        const int no = min(2, nout - o);
        const uint32_t gj = cin_ctr + min(o + no - 1 + lagc, nin - 1);
        mbar_wait(&bar_full[gj % NSLOT], (gj / NSLOT) & 1);
        float2 rv[2][HB / 2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h >= no) break;
          const int x = x_begin + (o + h) * CW + c;
#pragma unroll
          for (int i = 0; i < K; ++i) {
            const int* pl = P + ((x - x_begin - xs + t.p[i]) & (RL - 1));
            const int* pt = P + ((x - x_begin - xs - t.p[i] - 1) & (RL - 1));
            const float2 w2 = make_float2(t.w_row[i], t.w_row[i]);
#pragma unroll
            for (int r = 0; r < HB / 2; ++r) {
              const float2 d = make_float2(i2f_fast((uint32_t)(pl[2 * r * RLS] - pt[2 * r * RLS])),
                                           i2f_fast((uint32_t)(pl[(2 * r + 1) * RLS] - pt[(2 * r + 1) * RLS])));
              rv[h][r] = i == 0 ? __fmul2_rn(w2, d) : __ffma2_rn(w2, d, rv[h][r]);
            }
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h >= no) break;
          const uint32_t go = out_ctr + o + h;
          mbar_arrive(&bar_done[go % NSLOT]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h >= no) break;
          const int x = x_begin + (o + h) * CW + c;
          if (x < x_end) {
            int off = off0 + x, cc = c_first;
#pragma unroll
            for (int r = 0; r < HB / 2; ++r) {
              const float2 q = round_mid2<K>(rv[h][r]);  // round to the mid quantum
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                if (2 * r + u < nrows) st_global_idx(midg, off, __float_as_int(u ? q.y : q.x) - kMagicBits);
                ++cc;
                off += cc == C ? wrap_step + ch_step : ch_step;
                cc = cc == C ? 0 : cc;
              }
            }
          }
        }
      }
    }
    cin_ctr += (uint32_t)nin;
    out_ctr += (uint32_t)nout;
    __syncthreads();  // the next band restarts the ring, the carries and the row pointers
  }
}

template <typename Tin>
const void* stream_mc_ptr_for(int k) {
  switch (k) {
    case 1: return (const void*)stream_rows_mc_kernel<Tin, 1>;
    case 2: return (const void*)stream_rows_mc_kernel<Tin, 2>;
    case 3: return (const void*)stream_rows_mc_kernel<Tin, 3>;
    case 4: return (const void*)stream_rows_mc_kernel<Tin, 4>;
    case 5: return (const void*)stream_rows_mc_kernel<Tin, 5>;
    case 6: return (const void*)stream_rows_mc_kernel<Tin, 6>;
    case 7: return (const void*)stream_rows_mc_kernel<Tin, 7>;
    default: return (const void*)stream_rows_mc_kernel<Tin, 8>;
  }
}

template <typename Tin>
const void* stream_out_ptr_for(int k) {
  switch (k) {
    case 1: return (const void*)stream_rows_kernel<Tin, 1, true>;
    case 2: return (const void*)stream_rows_kernel<Tin, 2, true>;
    case 3: return (const void*)stream_rows_kernel<Tin, 3, true>;
    case 4: return (const void*)stream_rows_kernel<Tin, 4, true>;
    case 5: return (const void*)stream_rows_kernel<Tin, 5, true>;
    case 6: return (const void*)stream_rows_kernel<Tin, 6, true>;
    case 7: return (const void*)stream_rows_kernel<Tin, 7, true>;
    default: return (const void*)stream_rows_kernel<Tin, 8, true>;
  }
}

template <typename Tin>  // a template: instantiates its kernels only where it is called
const void* stream_ptr_for(int k) {
#define SB_STREAM(KK) stream_rows_kernel<Tin, KK>
  switch (k) {
    case 1: return (const void*)SB_STREAM(1);
    case 2: return (const void*)SB_STREAM(2);
    case 3: return (const void*)SB_STREAM(3);
    case 4: return (const void*)SB_STREAM(4);
    case 5: return (const void*)SB_STREAM(5);
    case 6: return (const void*)SB_STREAM(6);
    case 7: return (const void*)SB_STREAM(7);
    default: return (const void*)SB_STREAM(8);
  }
#undef SB_STREAM
}

// Kernel pointers per source type, instantiated in sweep_<dtype>.cu (one
// translation unit each, compiled in parallel).
const void* sweep_ptr_u8(Mode m, int k);
const void* sweep_ptr_u16(Mode m, int k);
const void* sweep_ptr_f32(Mode m, int k);
const void* sweep_ptr_f64(Mode m, int k);
int launch_filter_at(const void* src, int src_dtype, long long row_stride, int H, int W, const int* cols, int ncols,
                     const int* pt_col, const int* pt_y, long long npts, float* out, int* R, const TapsG& t,
                     int* status, cudaStream_t st);  // filter_at.cu
// generic two-pass kernels (generic_kernels.cu): any radius < extent, any k <= SB_MAX_K
constexpr size_t kGenericSmemBytes = 200 * 1024;  // longest row prefix the row kernel keeps in shared memory
constexpr int kGenericScratchRows = 296;          // global scratch rows (CTAs) for longer rows
constexpr int kWideSpan = 2048;                   // 2*pmax+1 above this: int64 ("wide") generic arithmetic
size_t generic_rows_scratch_bytes(int W, bool wide);
int launch_rows_generic(const void* src, int src_dtype, void* mid_out, float* dst, const Geometry& g,
                        const TapsG& t, void* scratch, bool wide, int* status, int sms, cudaStream_t st);
int launch_cols_generic(void* mid, float* dst, const Geometry& g, const TapsG& t, bool wide, int sms,
                        cudaStream_t st);
const void* sweep_ptr_cols(int k);   // ColsFromMid (source type unused)
const void* sweep_ptr_cols2(int k);  // ColsFromMid, prefix form
const void* sweep_ptr_cols2s(int k); // ColsFromMid, prefix form, split loader (eight loader warps)
const void* sweep_ptr_stream_f32(int k);  // streaming row pass (float32 sources)
const void* sweep_ptr_stream_f64(int k);  // streaming row pass, one-channel float64 / uint8 / uint16 sources
const void* sweep_ptr_stream_u8(int k);
const void* sweep_ptr_stream_u16(int k);
const void* sweep_ptr_stream_mc(int src_dtype, int k);  // streaming row pass, interleaved channels staged once
const void* sweep_ptr_stream_out(int src_dtype, int k); // streaming row pass alone (float rows out), one channel
const void* sweep_ptr_fused3(int k);      // fused sweep, three CTAs per SM (uint8, one channel)
const void* sweep_ptr_fused5(int k);      // fused sweep, two bands per consumer iteration (uint8, one channel)
const void* sweep_ptr_fusedp(int k);      // fused sweep, paired consumer warps (uint8, one channel)
const void* sweep_ptr_fused5w(int k);     // fused sweep, two bands per turn, 4-byte staging copies (uint8 rows % 4 == 0)
const void* sweep_ptr_fused_f32(int k, int ls);  // fused sweep of float32 sources with prefix stride ls
const void* sweep_ptr_fusedw(int k, int lsw);    // wide fused sweep (sweep_wide.cu), slot stride lsw
const void* sweep_ptr_rowtile(int k);            // uint8 row-tile sweep (sweep_rowtile.cu)

template <typename Tin>
const void* sweep_ptr_for(Mode m, int k) {
#define SB_K_CASES(KERNEL)                                 \
  switch (k) {                                             \
    case 1: return (const void*)KERNEL(1);                 \
    case 2: return (const void*)KERNEL(2);                 \
    case 3: return (const void*)KERNEL(3);                 \
    case 4: return (const void*)KERNEL(4);                 \
    case 5: return (const void*)KERNEL(5);                 \
    case 6: return (const void*)KERNEL(6);                 \
    case 7: return (const void*)KERNEL(7);                 \
    default: return (const void*)KERNEL(8);                \
  }
#define SB_FUSED(KK) fused_kernel<Tin, KK>
#define SB_ROWS_MID(KK) rows_kernel<Tin, KK, Mode::RowsToMid>
#define SB_ROWS_OUT(KK) rows_kernel<Tin, KK, Mode::RowsToOut>
  switch (m) {
    case Mode::Fused: SB_K_CASES(SB_FUSED)
    case Mode::RowsToMid: SB_K_CASES(SB_ROWS_MID)
    case Mode::RowsToOut: SB_K_CASES(SB_ROWS_OUT)
    default: break;
  }
  return nullptr;
#undef SB_FUSED
#undef SB_ROWS_MID
#undef SB_ROWS_OUT
}

template <int PLS>
inline const void* fused_f32_ptr_for(int k) {
#define SB_FF(KK) fused_kernel<float, KK, 2, false, PLS>
  SB_K_CASES(SB_FF)
#undef SB_FF
}

template <typename Unused = void>  // a template: instantiates its kernels only where it is called
const void* cols_ptr_for(int k) {
#define SB_COLS(KK) cols_kernel<KK>
  SB_K_CASES(SB_COLS)
#undef SB_COLS
}

template <typename Unused = void>  // a template: instantiates its kernels only where it is called
const void* cols2_ptr_for(int k) {
#define SB_COLS2(KK) cols2_kernel<KK>
  SB_K_CASES(SB_COLS2)
#undef SB_COLS2
}

template <typename Unused = void>
const void* cols2s_ptr_for(int k) {
#define SB_COLS2S(KK) cols2_kernel<KK, true>
  SB_K_CASES(SB_COLS2S)
#undef SB_COLS2S
#undef SB_K_CASES
}

}  // namespace sb
