// sliceblur_capi.cu - C ABI (include/sliceblur_b200.h) over the sm_100a sweep kernels.
//
// Host-side responsibilities, mirroring the reference where it validates
// (filtering.py:39-45, 67-73, 76-104): argument checks, the fixed-point quanta
// (DESIGN.md "Arithmetic"), the choice between the fused single-launch sweep
// and the two-launch path, and the work decomposition over 148 SMs.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "sliceblur_b200.h"
#include "sweep_kernels.cuh"

namespace {

thread_local std::string g_last_error;
thread_local int g_policy = SB_PATH_AUTO;  // sb_set_path_policy

// SB_DEBUG=1 prints the launch plans to stderr (read once, not per call)
bool debug_plans() {
  static const bool on = std::getenv("SB_DEBUG") != nullptr;
  return on;
}

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(SB_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

constexpr size_t kSmemBudget = 200 * 1024;
// the automatic uint8 one-channel kernel: paired consumer warps (1) or two bands per turn (0)
#ifndef SB_U8_DEFAULT_PAIRED
#define SB_U8_DEFAULT_PAIRED 0
#endif

int ceil16(int v) { return (v + 15) & ~15; }

int validate_kernel(const int64_t* radii, const double* weights, int k) {
  if (!radii || !weights) return fail(SB_ERR_INVALID_ARGUMENT, "radii/weights must not be NULL");
  if (k < 1 || k > SB_MAX_K)
    return fail(SB_ERR_INVALID_ARGUMENT, "need 1 <= k <= " + std::to_string(SB_MAX_K) + " slices");
  if (radii[0] < 0) return fail(SB_ERR_INVALID_ARGUMENT, "slice radii must be strictly increasing and >= 0");
  for (int i = 1; i < k; ++i)
    if (radii[i] <= radii[i - 1])
      return fail(SB_ERR_INVALID_ARGUMENT, "slice radii must be strictly increasing and >= 0");
  for (int i = 0; i < k; ++i)
    if (!std::isfinite(weights[i])) return fail(SB_ERR_INVALID_ARGUMENT, "slice weights must be finite");
  return SB_OK;
}

// Largest s with bound * 2^s < limit (strict), clamped to a sane exponent range.
int quantum_exponent(double bound, double limit) {
  if (!(bound > 0.0)) return 0;
  int s = (int)std::floor(std::log2(limit / bound));
  while (s > -120 && std::ldexp(bound, s) >= limit) --s;
  while (s < 100 && std::ldexp(bound, s + 1) < limit) ++s;
  return std::max(-120, std::min(100, s));
}

struct Plan {
  sb::Taps taps;  // k <= FAST_K (templated sweep kernels)
  sb::TapsG tg;   // any k (generic kernels, filter_at); only the first k entries are set
  int pmax;
};

// Fixed-point quanta.  `wide`: the generic kernels' int64 box sums
// (2*pmax+1 > kWideSpan), so only the magic-number rounding bounds the quanta.
int make_taps(const int64_t* radii, const double* weights, int k, int src_dtype, double value_bound, Plan* plan,
              bool wide = false) {
  int rc = validate_kernel(radii, weights, k);
  if (rc) return rc;
  double bound;
  switch (src_dtype) {
    case SB_DTYPE_U8: bound = 255.0; break;
    case SB_DTYPE_U16:
      // uint16 samples enter exactly; a caller bound below 65535 (e.g. a 12-bit PGM's maxval)
      // only refines the row-value quantum, and samples above it are reported, never used
      bound = (value_bound > 0.0 && value_bound < 65535.0) ? std::ceil(value_bound) : 65535.0;
      break;
    case SB_DTYPE_F32:
    case SB_DTYPE_F64:
      if (!(value_bound >= 0.0) || !std::isfinite(value_bound))
        return fail(SB_ERR_INVALID_ARGUMENT, "float input needs a finite value_bound >= 0 (max |pixel|)");
      bound = value_bound;
      if (bound < 3.0e38) {
        // the kernels quantise (float)v: a double just below the bound can round up to the
        // float above it, so the quantum must admit the bound rounded up to float (a float32
        // pixel <= bound is <= it too)
        float bf = (float)bound;
        if ((double)bf < bound) bf = std::nextafter(bf, INFINITY);
        bound = (double)bf;
      }
      break;
    default: return fail(SB_ERR_INVALID_ARGUMENT, "unknown src_dtype");
  }
  const int pmax = (int)radii[k - 1];
  const double width = 2.0 * pmax + 1.0;
  // |box sum| < 2^31 (int32) or 2^62 (wide) incl. rounding
  const double box_limit = wide ? 4.6e18 : 2147483647.0 - 2.0 * width;
  int s_in = 0;
  if (src_dtype == SB_DTYPE_F32 || src_dtype == SB_DTYPE_F64) {
    s_in = std::min(quantum_exponent(bound, 4194304.0), quantum_exponent(width * bound, box_limit));
  } else if (width * bound >= box_limit) {
    return fail(SB_ERR_INVALID_ARGUMENT, "radius too large for exact int32 box sums of this dtype");
  }
  double gabs = 0.0;
  for (int i = 0; i < k; ++i) gabs += std::fabs(weights[i]) * (2.0 * radii[i] + 1.0);
  // |R| <= gabs * (bound + half an input quantum)
  const double rbound = gabs * (bound + std::ldexp(0.5, -s_in)) * (1.0 + 1e-6);
  const int s_mid = std::min(quantum_exponent(rbound, 4194304.0), quantum_exponent(width * rbound, box_limit));

  sb::TapsG& g = plan->tg;
  g.k = k;
  g.pmax = pmax;
  g.in_scale = (float)std::ldexp(1.0, s_in);
  if (src_dtype == SB_DTYPE_F32 || src_dtype == SB_DTYPE_F64) {
    // |pixel| * 2^s_in <= the scaled bound (< 2^22, exact: bound is a float here), so every
    // sum the quanta were sized for stays in range; half of it flags SB_STATUS_HALF
    const float bf = (float)bound;
    g.in_limit = (float)std::ldexp((double)bf, s_in);
    g.seen_limit = (float)std::ldexp((double)bf, s_in - 1);
  } else {
    g.in_limit = (float)bound;  // uint16: largest admissible sample (uint8: unused)
    g.seen_limit = INFINITY;
  }
  for (int i = 0; i < k; ++i) {
    g.p[i] = (int)radii[i];
    g.w_row[i] = (float)std::ldexp(weights[i], s_mid - s_in);
    g.w_col[i] = (float)std::ldexp(weights[i], -s_mid);
    g.w_out1[i] = (float)std::ldexp(weights[i], -s_in);
  }
  sb::Taps& t = plan->taps;
  std::memset(&t, 0, sizeof(t));
  t.k = k;
  t.pmax = pmax;
  for (int i = 0; i < k && i < sb::FAST_K; ++i) {
    t.p[i] = g.p[i];
    t.w_row[i] = g.w_row[i];
    t.w_col[i] = g.w_col[i];
    t.w_out1[i] = g.w_out1[i];
  }
  t.in_scale = g.in_scale;
  t.in_limit = g.in_limit;
  t.seen_limit = g.seen_limit;
  plan->pmax = pmax;
  return SB_OK;
}

int dtype_size(int dt) {
  switch (dt) {
    case SB_DTYPE_U8: return 1;
    case SB_DTYPE_U16: return 2;
    case SB_DTYPE_F32: return 4;
    case SB_DTYPE_F64: return 8;
  }
  return 0;
}

struct Launch {
  sb::Tiling tl;
  size_t smem;
  dim3 grid;
};

// Tiling of a strip sweep (see sweep_kernels.cuh): staged/prefix row [xb, xb+L)
// with xb = x0 - xoff for a strip of `sw` columns; ring of D rows (+ HB mirror).
sb::Tiling make_tiling(sb::Mode m, int pmax, int channels, int es, bool u8_single, int pmin = 0) {
  sb::Tiling tl;
  std::memset(&tl, 0, sizeof(tl));
  tl.xoff = ceil16(pmax + 1);
  tl.sw = sb::WS;
  const bool rows_only = (m == sb::Mode::RowsToMid || m == sb::Mode::RowsToOut);
  const int staged_ch = rows_only ? 1 : channels;  // the row pass gathers its channel
  if (rows_only) {
    // widen the strip until the halo costs <= 50% extra (bounded by shared memory)
    while (tl.sw < 1024 && ceil16(tl.xoff + tl.sw + pmax) > (3 * tl.sw) / 2) {
      const int L2 = ceil16(tl.xoff + 2 * tl.sw + pmax);
      if ((size_t)2 * sb::HB * ceil16(L2 * es) + (size_t)sb::HB * L2 * 4 > kSmemBudget) break;
      tl.sw *= 2;
    }
  }
  tl.L = ceil16(tl.xoff + tl.sw + pmax);
  const int nchunk = tl.L / sb::CH;
  int lpr = 1;
  while (lpr < nchunk && lpr < 32) lpr <<= 1;
  tl.lanes_per_row = lpr;
  tl.stage_row_bytes = ceil16(tl.L * staged_ch * es);
  if (m == sb::Mode::Fused && (tl.stage_row_bytes / 16) % 2 == 0) tl.stage_row_bytes += 16;  // odd x 16 B: no conflicts
  tl.ls = (m == sb::Mode::Fused) ? sb::LS : tl.L;
  if (m == sb::Mode::Fused && es == 4 && channels == 1 && !u8_single)  // float32: stride sized from L
    tl.ls = tl.L <= sb::LS_SMALL ? sb::LS_SMALL : (tl.L <= sb::LS_MID ? sb::LS_MID : sb::LS);
  tl.packed = (m == sb::Mode::Fused && u8_single && ((tl.L + 63) & ~63) <= 192) ? 1 : 0;  // float2 prefixes
  if (tl.packed) {
    // the scan covers whole 64-column quarters; rows an odd multiple of 16 bytes apart
    tl.L = (tl.L + 63) & ~63;
    tl.stage_row_bytes = tl.L + 16;
  }
  tl.npb = 1;  // one prefix buffer per producer warp (each owns every FPROD-th band)
  tl.nsb = (m == sb::Mode::Fused && es == 4 && tl.ls == sb::LS_SMALL) ? 1 : 2;  // mirrors fused_kernel's NSB
  if (m == sb::Mode::Fused) {
    const size_t pbuf = tl.packed ? (size_t)(sb::HB / 2) * sb::LSP2 * sizeof(float2) : (size_t)sb::HB * tl.ls * sizeof(int);
    const size_t end = (size_t)tl.nsb * sb::FPROD * sb::HB * tl.stage_row_bytes + (size_t)sb::FPROD * tl.npb * pbuf;
    tl.obuf_off = (int)((end + 127) & ~(size_t)127);
  }
  tl.D = ((2 * pmax + 2 * sb::HB + sb::HB - 1) / sb::HB) * sb::HB;  // multiple of HB
  if (m == sb::Mode::ColsFromMid) {
    // The ring holds every window when it fits tensor memory; otherwise trails deeper than
    // the ring are re-read from the plane (prefetched through shared memory).  Measured:
    // a full ring at one CTA per SM beats a 256-column ring with deep re-reads (C4).
    (void)pmin;
    tl.D = std::min(tl.D, 512 - sb::HB);
  }
  int cols = 32;
  while (cols < tl.D + sb::HB) cols <<= 1;
  tl.tmem_cols = cols;
  if (m == sb::Mode::Fused && tl.packed == 1) {
    // Default (SB_FUSED=5): fused_kernel<uint8_t, K, 2, true>, consumers take two bands per
    // iteration (one prefix carry, one 32-column TMEM store, 32-row output bands).
    // SB_FUSED=3: fused_kernel<uint8_t, K, 3>, three CTAs per SM (registers rebalanced between
    // the producer and consumer warpgroups with setmaxnreg, single-buffered staging and output
    // box).  SB_FUSED=1: the two-CTA one-band kernel.  (A/B switches.)
    // SB_U8_DEFAULT_PAIRED picks the automatic uint8 kernel: paired consumer warps (1) or two
    // bands per consumer turn (0); SB_PATH_U8_PAIRED / SB_PATH_U8_TWO_BAND force either
    const bool paired = g_policy == SB_PATH_U8_PAIRED || (SB_U8_DEFAULT_PAIRED && g_policy != SB_PATH_U8_TWO_BAND &&
                                                          g_policy != SB_PATH_U8_THREE_CTA &&
                                                          g_policy != SB_PATH_U8_ONE_BAND);
    if (paired) {
      // ring: the bands one output band reads (E + 1) plus three bands of slack, so a band is
      // overwritten only after the other warp has left every window that reads it
      tl.split = 6;
      const int E = (2 * pmax + 1 + 2 * sb::HB - 1) / sb::HB - 1;
      tl.D = (E + 4) * sb::HB;
      int colsp = 32;
      while (colsp < tl.D + sb::HB) colsp <<= 1;
      tl.tmem_cols = colsp;
    } else if (g_policy != SB_PATH_U8_THREE_CTA && g_policy != SB_PATH_U8_ONE_BAND) {
      // two bands per consumer iteration: 32-row ring slots, 32-row mirror
      tl.split = 5;
      tl.D = ((2 * pmax + 65 + 31) / 32) * 32;
      int cols5 = 32;
      while (cols5 < tl.D + 32) cols5 <<= 1;
      tl.tmem_cols = cols5;
    } else if (g_policy == SB_PATH_U8_THREE_CTA) {
      tl.split = 3;
      const size_t end = (size_t)sb::FPROD * sb::HB * tl.stage_row_bytes +
                         (size_t)sb::FPROD * (sb::HB / 2) * sb::LSP2 * sizeof(float2);
      tl.obuf_off = (int)((end + 127) & ~(size_t)127);
    }
  }
  return tl;
}

// Dynamic shared memory that limits residency to `ctas` CTAs per SM (the TMEM
// ring kernels must never have a CTA waiting inside tcgen05.alloc).
size_t residency_floor(int ctas) { return 233472 / (size_t)(ctas + 1) - 1024 + 16; }

size_t smem_bytes(const sb::Tiling& tl, sb::Mode m) {
  if (m == sb::Mode::ColsFromMid)
    return std::max((size_t)(1 + tl.ndeep) * tl.pf * sb::HB * sb::WS * sizeof(int), residency_floor(512 / tl.tmem_cols));
  if (m == sb::Mode::ColsPrefix)  // plane ring + band copies + output boxes (TMA), 128-byte aligned
    return (size_t)tl.obuf_off + 128 + (size_t)4 * sb::CG * 2 * sb::HB * 32 * sizeof(float);
  if (m == sb::Mode::Fused) {
    // staged bands + prefix buffers (producer/consumer hand-off); the ring lives in tensor memory.
    // + FCONS x 2 output bands of HB x 32 floats staged for TMA tensor stores
    // output staging per consumer warp: 1 (three-CTA), 2 (two-CTA) 16-row boxes, or two 32-row boxes (split 5)
    const int boxes = tl.split == 3 ? 1 : (tl.split == 5 || tl.split == 6 ? 4 : tl.nsb);
    size_t s = (size_t)tl.obuf_off + 128 + (size_t)sb::FCONS * boxes * sb::HB * 32 * sizeof(float);
    // cap residency at 512 / tmem_cols CTAs per SM by asking for enough shared
    // memory, so no CTA ever waits inside tcgen05.alloc
    return std::max(s, residency_floor(512 / tl.tmem_cols));
  }
  return (size_t)2 * sb::HB * tl.stage_row_bytes + (size_t)sb::HB * tl.ls * sizeof(int);
}

bool fused_fits(int pmax, int channels, int es) {
  sb::Tiling tl = make_tiling(sb::Mode::Fused, pmax, channels, es, false);
  return tl.L <= sb::LMAX && tl.tmem_cols <= 512 && smem_bytes(tl, sb::Mode::Fused) <= kSmemBudget;
}

const void* pick_kernel(sb::Mode m, int dtype, int k) {
  if (m == sb::Mode::ColsFromMid) return sb::sweep_ptr_cols(k);  // source unused
  switch (dtype) {
    case SB_DTYPE_U8: return sb::sweep_ptr_u8(m, k);
    case SB_DTYPE_U16: return sb::sweep_ptr_u16(m, k);
    case SB_DTYPE_F32: return sb::sweep_ptr_f32(m, k);
    default: return sb::sweep_ptr_f64(m, k);
  }
}

// Work decomposition: every (strip, channel) column sweeps `items` contiguous
// row ranges of the tall (batch*H) image; items is sized so the grid fills the
// GPU about once, but never so small that the 2*pmax+1 warm-up rows of a
// column sweep exceed ~1/8 of the rows it outputs.
// Tiling of the prefix-form column kernel (cols2_kernel): a 496-row TMEM ring,
// CG output groups, trail windows classified as ring or band copies.  False when
// a window would straddle the two (the running-sum cols_kernel is used then).
// cols2_kernel runs one CTA per SM: its TMA slots and band copies may take the whole opt-in
// shared memory (static shared memory is < 1 KB)
#ifndef SB_COLS2_SMEM_KB
#define SB_COLS2_SMEM_KB 224
#endif
constexpr size_t kCols2Smem = (size_t)SB_COLS2_SMEM_KB * 1024;
#ifndef SB_STREAM_MC
#define SB_STREAM_MC 1
#endif
#ifndef SB_STREAM_MC_UNALIGNED
#define SB_STREAM_MC_UNALIGNED 1
#endif
#ifndef SB_STREAM_ROWS_OUT
#define SB_STREAM_ROWS_OUT 1
#endif
#ifndef SB_STREAM_SEGMENTS
#define SB_STREAM_SEGMENTS 1
#endif
#ifndef SB_STREAM_ALL_TYPES
#define SB_STREAM_ALL_TYPES 1
#endif
#ifndef SB_COLS2_SPLIT
#define SB_COLS2_SPLIT 1
#endif
#ifndef SB_COLS2_MINPF
#define SB_COLS2_MINPF 2
#endif
#ifndef SB_COLS2_SLACK0
#define SB_COLS2_SLACK0 3
#endif

bool cols_prefix_tiling(const sb::Tiling& base, const int64_t* radii, int k, int pmax, sb::Tiling* out) {
  sb::Tiling tl = base;
  const int NB = 31;
  tl.D = NB * sb::HB;
  tl.tmem_cols = 512;
  const size_t band = (size_t)sb::HB * sb::WS * sizeof(int);
  const size_t obuf = (size_t)4 * sb::CG * 2 * sb::HB * 32 * sizeof(float) + 128;
  const int span = 2 + pmax / 8;  // ring bands one output band reads
  // Slack: bands the loader may run ahead of the output groups.  Without band copies the
  // ring bounds it (lag <= NB); with copies, each slack band costs two copy slots.
  int slack0 = NB - span - sb::CG + 1;
  if (slack0 < 0) slack0 = SB_COLS2_SLACK0;
  // first pass: the most slack that still leaves SB_COLS2_MINPF TMA slots (bytes in flight per
  // SM); second pass: anything that fits
  for (int it = 0; it < 2 * (slack0 + 1); ++it) {
    const int slack = slack0 - (it % (slack0 + 1));
    const int min_pf = it <= slack0 ? SB_COLS2_MINPF : 2;
    tl.lag = span + sb::CG - 1 + slack;
    tl.copy_e = tl.lag - span + 1;  // band v - NB + copy_e is copied right after band v is released
    // output band o + C2DONE may finish before the loader observed band o's done phase
    // unless the loader has passed o by then: C2DONE >= lag - span + 1
    if (tl.lag - span + 1 > sb::C2DONE) continue;
    const int thr = tl.lag - 1 - NB;  // bands at offset <= thr come from the copies
    tl.deepmask = 0;
    bool ok = true;
    for (int i = 0; i < k && ok; ++i) {
      const int off = pmax - (int)radii[i];
      const int lo = off / sb::HB, hi = (off + sb::HB - 1) / sb::HB;
      if (hi <= thr) tl.deepmask |= 1 << i;
      else if (lo <= thr) ok = false;                               // straddles copies and ring
      if ((pmax + 1 + (int)radii[i]) / sb::HB <= thr) ok = false;   // leads always from the ring
    }
    if (!ok) continue;
    tl.ds = thr >= 0 ? 2 * tl.lag - NB - span + 2 : 0;  // >= lag - NB + copy_e, plus one spare
    tl.pf = 0;
    const int copies = tl.ds ? tl.ds + 1 : 0;  // + the mirror of copy slot 0
    for (int pf : {sb::C2PF, 6, 4, 3, 2})      // slots of two bands each
      if ((size_t)(2 * pf + copies) * band + obuf <= kCols2Smem) {
        tl.pf = pf;
        break;
      }
    if (tl.pf < min_pf) continue;
    tl.obuf_off = (int)((size_t)(2 * tl.pf + copies) * band);
    *out = tl;
    return true;
  }
  return false;
}

// Tiling of the wide fused sweep (sweep_wide.cu): staged / prefix rows of L columns in
// slots of WLS words, the cols2_kernel ring (496 rows of TMEM, trails older than the ring
// from shared-memory band copies, lag / copy_e / ds / deepmask as in cols_prefix_tiling with
// WCG output groups) and tl.pf = the number of producer slots that fit shared memory.
// False when no slot stride bounds L, a window would straddle ring and copies, or the
// buffers do not fit (the two-launch path runs then).
constexpr size_t kWideSmem = 226 * 1024;  // one CTA per SM (static shared memory is < 1 KB)

bool fusedw_tiling(const int64_t* radii, int k, int pmax, sb::Tiling* out) {
  sb::Tiling tl;
  std::memset(&tl, 0, sizeof(tl));
  tl.xoff = ceil16(pmax + 1);
  tl.sw = sb::WS;
  tl.L = ceil16(tl.xoff + sb::WS + pmax);
  int lsw = 0;
  for (int b : sb::WLS)
    if (b >= tl.L) {
      lsw = b;
      break;
    }
  if (!lsw) return false;
  tl.ls = lsw;
  tl.stage_row_bytes = lsw * 4;
  const int NB = 31;
  tl.D = NB * sb::HB;
  tl.tmem_cols = 512;
  const size_t band = (size_t)sb::HB * sb::WS * sizeof(int);
  const size_t slot = (size_t)sb::HB * lsw * sizeof(int);
  const size_t obuf = (size_t)4 * sb::WCG * 2 * sb::HB * 32 * sizeof(float) + 128;
  const int span = 2 + pmax / 8;  // ring bands one output band reads
  const int slack0 = NB - span - sb::WCG + 1 < 0 ? 3 : NB - span - sb::WCG + 1;
  // the most slack (row warps running ahead of the output groups) that leaves room for
  // three producer slots; two slots only when nothing else fits
  for (int it = 0; it < 2 * (slack0 + 1); ++it) {
    const int min_fp = it <= slack0 ? 3 : 2;
    const int slack = slack0 - (it % (slack0 + 1));
    tl.lag = span + sb::WCG - 1 + slack;
    tl.copy_e = tl.lag - span + 1;
    if (tl.lag - span + 1 > sb::C2DONE) continue;
    const int thr = tl.lag - 1 - NB;  // bands at offset <= thr come from the copies
    tl.deepmask = 0;
    bool ok = true;
    for (int i = 0; i < k && ok; ++i) {
      const int off = pmax - (int)radii[i];
      const int lo = off / sb::HB, hi = (off + sb::HB - 1) / sb::HB;
      if (hi <= thr) tl.deepmask |= 1 << i;
      else if (lo <= thr) ok = false;
      if ((pmax + 1 + (int)radii[i]) / sb::HB <= thr) ok = false;
    }
    if (!ok) continue;
    tl.ds = thr >= 0 ? 2 * tl.lag - NB - span + 2 : 0;
    const int copies = tl.ds ? tl.ds + 1 : 0;
    tl.pf = 0;
    for (int fp = sb::WPROD; fp >= min_fp; --fp)
      if (fp * slot + (size_t)copies * band + obuf <= kWideSmem) {
        tl.pf = fp;
        break;
      }
    if (!tl.pf) continue;
    tl.obuf_off = (int)((size_t)tl.pf * slot + (size_t)copies * band);
    *out = tl;
    return true;
  }
  return false;
}

// Tiling of the uint8 row-tile sweep (sweep_rowtile.cu): staged rows [xb, xb + L) with
// xb = x0 - xoff (16-byte aligned), TMEM row-prefix region of ta columns from staged column
// s0, a ring of D rows (32-row slots) plus its 32-row mirror behind it, all in one 512-column
// allocation (one CTA per SM).  False when the radii do not fit.
bool rowtile_tiling(int pmax, sb::Tiling* out) {
  sb::Tiling tl;
  std::memset(&tl, 0, sizeof(tl));
  tl.xoff = ceil16(pmax + 1);
  tl.sw = sb::WS;
  tl.L = ceil16(tl.xoff + sb::WS + pmax);
  tl.stage_row_bytes = (tl.L / 16) % 2 ? tl.L : tl.L + 16;  // odd multiple of 16: conflict-free
  tl.s0 = (tl.xoff - pmax - 1) & ~7;  // 8-byte aligned (the scan combines 16-byte halves)
  tl.ta = ceil16(tl.xoff + sb::WS + pmax - tl.s0);
  tl.D = sb::TB * ((2 * pmax + 2 * sb::TB + 1 + sb::TB - 1) / sb::TB);
  tl.tmem_cols = 512;
  // two row-prefix regions (two row warps per lane quadrant), the ring and its 32-row mirror
  if (2 * tl.ta + tl.D + sb::TB > 512 || tl.D / sb::TB > 16) return false;
  if ((tl.s0 & 15) && ceil16(tl.s0) + tl.ta + 16 > tl.L + 16) return false;  // the scan reads one chunk ahead
  const size_t stage = (size_t)sb::TROWW * sb::TB * tl.stage_row_bytes;
  const size_t slots = (size_t)sb::TRS * sb::TB * sb::TRSW * sizeof(float);
  tl.obuf_off = (int)(((stage + slots) + 127) & ~(size_t)127);
  const size_t smem = (size_t)tl.obuf_off + 128 + (size_t)4 * sb::TOG * sb::TOBUF * sb::TB * 32 * sizeof(float);
  if (smem > 226 * 1024) return false;
  *out = tl;
  return true;
}

// Persistent (row chunk, strip) units over `sms` CTAs: the chunk count minimising
// (rounds of units) x (chunk rows + warm-up rows).  Returns the chunk height.
long long persistent_chunk(long long total_rows, int nstrips, int sms, long long warm, int band) {
  long long best_chunks = 1;
  double best_cost = 1e300;
  for (long long nc = 1; nc <= 512 && nc <= std::max(1LL, total_rows / band); ++nc) {
    const long long units = nc * nstrips;
    const long long rounds = (units + sms - 1) / sms;
    const double cost = (double)rounds * (double)((total_rows + nc - 1) / nc + warm);
    if (cost < best_cost * 0.995) {
      best_cost = cost;
      best_chunks = nc;
    }
  }
  return (total_rows + best_chunks - 1) / best_chunks;
}

// Immutable launch facts, looked up once per (kernel, device) instead of on every call
// (small images are host-bound otherwise): register count, static shared memory, the
// dynamic shared memory already granted with cudaFuncSetAttribute, and the device's SM
// count / shared memory / register file.  Guarded by a mutex; entries are never removed.
struct FnFacts {
  const void* fn;
  int dev;
  int num_regs;
  size_t static_smem;
  size_t granted;
};
struct DevFacts {
  int sms, smem_per_sm, regs_per_sm;
};
std::mutex g_facts_mu;
std::vector<FnFacts> g_fn_facts;
DevFacts g_dev_facts[64];
bool g_dev_known[64];

int launch_facts(const void* fn, size_t smem, FnFacts* ff, DevFacts* df) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lock(g_facts_mu);
  FnFacts* f = nullptr;
  for (auto& x : g_fn_facts)
    if (x.fn == fn && x.dev == dev) f = &x;
  if (!f) {
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, fn);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncGetAttributes");
    g_fn_facts.push_back({fn, dev, fa.numRegs, fa.sharedSizeBytes, 0});
    f = &g_fn_facts.back();
  }
  if (smem > f->granted) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    f->granted = smem;
  }
  *ff = *f;
  if (dev < 0 || dev >= 64) return fail(SB_ERR_INVALID_ARGUMENT, "device ordinal out of range");
  if (!g_dev_known[dev]) {
    DevFacts d{148, 233472, 65536};
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&d.regs_per_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    g_dev_facts[dev] = d;
    g_dev_known[dev] = true;
  }
  *df = g_dev_facts[dev];
  return SB_OK;
}

int plan_launch(const void* fn, sb::Mode m, const sb::Tiling& base, int pmax, int W, long long total_rows,
                int channels, Launch* out) {
  sb::Tiling& tl = out->tl;
  tl = base;
  tl.nstrips = (W + tl.sw - 1) / tl.sw;
  const size_t smem = smem_bytes(tl, m);
  if (smem > 227 * 1024)
    return fail(SB_ERR_INVALID_ARGUMENT, "slice radius " + std::to_string(pmax) + " too large for the GPU strip sweep");
  out->smem = smem;
  FnFacts fa;
  DevFacts df;
  int rc = launch_facts(fn, smem, &fa, &df);
  if (rc) return rc;
  int occ = 1;
  const int sms = df.sms, smem_per_sm = df.smem_per_sm, regs_per_sm = df.regs_per_sm;
  // Residency from the kernel's own resources.  (cudaOccupancyMaxActiveBlocksPerMultiprocessor
  // reports 1 for kernels that allocate tensor memory, which would idle 3/4 of each SM.)
  const int threads = (m == sb::Mode::Fused) ? (tl.split == 6 ? sb::PTHREADS : sb::FTHREADS)
                                             : (m == sb::Mode::ColsPrefix ? sb::C2THREADS : sb::WS);
  const int regs_per_cta = ((fa.num_regs * 32 + 255) / 256) * 256 * (threads / 32);
  occ = std::min(2048 / threads, regs_per_sm / std::max(1, regs_per_cta));
  occ = std::min<long long>(occ, (long long)smem_per_sm / (long long)(smem + fa.static_smem + 1024));
  if (m == sb::Mode::Fused || m == sb::Mode::ColsFromMid || m == sb::Mode::ColsPrefix)
    occ = std::min(occ, 512 / tl.tmem_cols);
  occ = std::max(occ, 1);
  const long long slots = (long long)sms * occ;
  const long long columns = (long long)tl.nstrips * channels;
  const bool sweeps = (m == sb::Mode::Fused || m == sb::Mode::ColsFromMid || m == sb::Mode::ColsPrefix);
  // Column sweeps pay 2*pmax+1 warm-up rows per item; the row pass pays nothing.
  // Pick the item count minimising (waves of CTAs) x (rows per item incl. warm-up).
  const long long warm = sweeps ? 2LL * pmax + 1 : 0;
  const long long max_items = std::max(1LL, std::min<long long>(4096, total_rows / std::max<long long>(sb::HB, warm)));
  long long best_items = 1;
  double best_cost = 1e300;
  for (long long it = 1; it <= max_items; ++it) {
    const long long ctas = columns * it;
    const long long waves = (ctas + slots - 1) / slots;
    const long long rows = (total_rows + it - 1) / it;
    const double cost = (double)waves * (double)(rows + warm + sb::HB);
    if (cost < best_cost * 0.995) {
      best_cost = cost;
      best_items = it;
    }
  }
  long long items = best_items;
  long long rows_per_item = (total_rows + items - 1) / items;
  if (!sweeps) rows_per_item = ((rows_per_item + sb::HB - 1) / sb::HB) * sb::HB;
  items = (total_rows + rows_per_item - 1) / rows_per_item;
  tl.rows_per_item = rows_per_item;
  if (columns * items > 0x7fffffffLL) return fail(SB_ERR_INVALID_ARGUMENT, "image too large for the grid");
  out->grid = dim3((unsigned)(tl.nstrips * items), (unsigned)channels, 1);
  if (debug_plans())
    std::fprintf(stderr,
                 "[sliceblur_b200] mode=%d pmax=%d L=%d ls=%d D=%d tmem_cols=%d packed=%d smem=%zu occ=%d "
                 "strips=%d items=%lld rows/item=%lld grid=%u x %u\n",
                 (int)m, pmax, tl.L, tl.ls, tl.D, tl.tmem_cols, tl.packed, smem, occ, tl.nstrips, items, rows_per_item,
                 out->grid.x, out->grid.y);
  return SB_OK;
}

int launch_rows(const void* fn, const Launch& L, const void* src, int* mid_out, float* dst, const sb::Geometry& g,
                const sb::Taps& t, int* status, cudaStream_t stream) {
  void* args[] = {(void*)&src, (void*)&mid_out, (void*)&dst, (void*)&g, (void*)&t, (void*)&L.tl, (void*)&status};
  cudaError_t e = cudaLaunchKernel(fn, L.grid, dim3(sb::WS), args, L.smem, stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernel");
  return SB_OK;
}

int launch_cols(const void* fn, const Launch& L, const int* mid_in, float* dst, const sb::Geometry& g,
                const sb::Taps& t, cudaStream_t stream) {
  void* args[] = {(void*)&mid_in, (void*)&dst, (void*)&g, (void*)&t, (void*)&L.tl};
  // channels are folded into grid.x (fastest varying), see cols_kernel
  cudaError_t e = cudaLaunchKernel(fn, dim3(L.grid.x * L.grid.y), dim3(sb::WS), args, L.smem, stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernel");
  return SB_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda at link time)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  // looked up once (thread-safe static initialisation)
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000)p;
    cudaGetLastError();
    return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
  }();
  return fn;
}

// Output tensor map [image][row][column] (fp32) with a 16 x 32 box: one box per
// consumer warp and output band.  Clears g.out_bulk when no map can be made.
void make_output_map(float* dst, sb::Geometry& g, CUtensorMap* map, int box_rows = sb::HB) {
  std::memset(map, 0, sizeof(*map));
  if (!g.out_bulk) return;
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  const long long rows = g.oy1 - g.oy0;
  const cuuint64_t dims[3] = {(cuuint64_t)g.W, (cuuint64_t)rows, (cuuint64_t)g.nimg};
  const cuuint64_t rstride = (cuuint64_t)g.out_row * 4;
  const cuuint64_t istride = g.nimg > 1 ? (cuuint64_t)g.out_img * 4 : rstride * (cuuint64_t)rows;
  const cuuint64_t strides[2] = {rstride, istride};
  const cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (!enc || enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)dst, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    g.out_bulk = 0;
}

// Tensor map of the int32 R plane [channel*batch][H][W] with a 32 x 128 box (the
// prefix-form column kernel loads a pair of bands per TMA).  False when the plane rows
// are not 16-byte multiples or no map can be made.
bool make_plane_map(const int* mid, const sb::Geometry& g, int channels, CUtensorMap* map) {
  std::memset(map, 0, sizeof(*map));
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc || (g.mid_row * 4) % 16 != 0 || (g.mid_img * 4) % 16 != 0 || (uintptr_t)mid % 16 != 0) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.nimg * (cuuint64_t)channels};
  const cuuint64_t strides[2] = {(cuuint64_t)g.mid_row * 4, (cuuint64_t)g.mid_img * 4};
  const cuuint32_t box[3] = {(cuuint32_t)sb::WS, (cuuint32_t)(2 * sb::HB), 1};  // a pair of bands
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, (void*)mid, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

int launch_fused(const void* fn, const Launch& L, const void* src, float* dst, const sb::Geometry& g0,
                 const sb::Taps& t, int* status, cudaStream_t stream) {
  sb::Geometry g = g0;
  alignas(64) CUtensorMap omap;
  make_output_map(dst, g, &omap);
  void* args[] = {(void*)&src, (void*)&dst, (void*)&g, (void*)&t, (void*)&L.tl, (void*)&status, (void*)&omap};
  cudaError_t e = cudaLaunchKernel(fn, L.grid, dim3(L.tl.split == 6 ? sb::PTHREADS : sb::FTHREADS), args, L.smem, stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernel");
  return SB_OK;
}

// ---------------------------------------------------------------- path choice
// One decision shared by the workspace queries and the launches (so a caller that
// sized its workspace with the query always has enough).
enum class RowPath { Fused, FusedWide, RowTile, Stream, Tiled, Generic };
enum class ColPath { None, Prefix, Running, Generic };

struct Route {
  RowPath rows;
  ColPath cols;
  bool wide;             // generic kernels with int64 sums and an int64 plane
  size_t scratch_bytes;  // generic row kernel's global scratch rows
};

bool needs_wide(int pmax) { return 2LL * pmax + 1 > sb::kWideSpan; }

size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

// stream_rows_kernel's `unal` mode (one channel, rows not 16-byte multiples, aligned base):
// staged rows carry one more 16-byte vector
bool stream_unaligned(const void* src, const sb::Geometry& g) {
  return g.in_px == 1 && !g.aligned16 && ((uintptr_t)src & 15) == 0;
}

// Segment width (a multiple of the chunk) of the streaming row pass: the segment count that
// minimises (rounds of units over the resident CTAs, two per SM) x (segment + halo width).
int stream_segment_width(int64_t width, int pmax, long long par_bands, int sms) {
  const long long ctas_par = (long long)sms * 2;
  int nseg = 1;
  double best = 1e300;
  const int halo = 2 * pmax + 1 + sb::CW;
  const int max_seg = (int)std::max<int64_t>(1, width / std::max(1024, 8 * pmax));
  for (int ns = 1; ns <= std::min(max_seg, 512); ++ns) {
    const int sw = (int)(((width + ns - 1) / ns + sb::CW - 1) / sb::CW) * sb::CW;
    const long long units = par_bands * ((width + sw - 1) / sw);
    const double cost = (double)((units + ctas_par - 1) / ctas_par) * (double)(sw + halo);
    if (cost < best * 0.97) {
      best = cost;
      nseg = ns;
    }
  }
  return SB_STREAM_SEGMENTS ? (int)(((width + nseg - 1) / nseg + sb::CW - 1) / sb::CW) * sb::CW
                            : (int)((width + sb::CW - 1) / sb::CW) * sb::CW;
}

// The streaming row pass takes float32 sources with any channel count and one-channel sources
// of every other type (float64 is the reference's own dtype: 8192^2 sigma 64 went from 2.26 to
// 0.43 ms with it; interleaved non-float32 channels keep the tiled row pass).
bool stream_rows_fits(int src_dtype, int pmax, int channels, int64_t width) {
  const int xs = -(((pmax + 1) + 15) & ~15);
  const int lagc = (sb::CW - 1 - xs + pmax) / sb::CW;
  // interleaved channels of the other types: up to four (stream_rows_mc_kernel; rows that are not
  // 16-byte multiples are staged from aligned-down addresses)
  const bool other = SB_STREAM_ALL_TYPES &&
                     (channels == 1 || (channels <= 4 && (SB_STREAM_MC_UNALIGNED ||
                                                          (width * channels * dtype_size(src_dtype)) % 16 == 0)));
  return (src_dtype == SB_DTYPE_F32 || other) && lagc + 1 < sb::NSLOT;
}

bool tiled_rows_fits(sb::Mode m, int pmax, int channels, int es) {
  const sb::Tiling tl = make_tiling(m, pmax, channels, es, false);
  return smem_bytes(tl, m) <= 227 * 1024;
}

// The running-sum column kernel reads every lead window from its TMEM ring: the ring
// (capped at 496 rows) must span pmax - p_0 + 2 bands (see cols_kernel).
bool running_cols_fits(const int64_t* radii, int pmax, int channels) {
  const sb::Tiling ct = make_tiling(sb::Mode::ColsFromMid, pmax, channels, 4, false);
  return ct.D >= pmax - (int)radii[0] + 2 * sb::HB;
}

Route route_2d(int src_dtype, int64_t width, int channels, const int64_t* radii, int k) {
  const int pmax = (int)radii[k - 1];
  Route r{RowPath::Generic, ColPath::Generic, needs_wide(pmax), 0};
  const int es = dtype_size(src_dtype);
  const bool fast = k <= sb::FAST_K && g_policy != SB_PATH_GENERIC && !r.wide;
  sb::Tiling rt;
  if (fast && g_policy == SB_PATH_U8_ROWTILE && src_dtype == SB_DTYPE_U8 && channels == 1 &&
      rowtile_tiling(pmax, &rt)) {
    r.rows = RowPath::RowTile;
    r.cols = ColPath::None;
    return r;
  }
  // One-channel uint8 past the packed (float2-prefix) tiling: the unpacked fused sweep is slower
  // than the streaming row pass + cols2 (4096^2 p_max 77: 0.189 vs 0.114 ms; 8192^2 p_max 103:
  // 0.652 vs 0.321 ms), so AUTO takes two launches there.
  const bool u8_unpacked = SB_STREAM_ALL_TYPES && src_dtype == SB_DTYPE_U8 && channels == 1 &&
                           !make_tiling(sb::Mode::Fused, pmax, 1, 1, true).packed &&
                           stream_rows_fits(src_dtype, pmax, channels, width);
  // Dense rows that are not 16-byte multiples: the fused sweep stages them element by element
  // (4001^2 float32 p_max 20: 0.224 ms), the streaming row pass from aligned-down 16-byte copies
  // (0.128 ms); packed uint8 stays fused (64 x 1000^2: 0.43 vs 0.56 ms; a pitched device copy
  // into an aligned layout first measured 0.36 ms and is not used).
  const bool unaligned_rows = SB_STREAM_ALL_TYPES && (width * channels * es) % 16 != 0 &&
                              !(src_dtype == SB_DTYPE_U8 && channels == 1) &&
                              stream_rows_fits(src_dtype, pmax, channels, width);
  if (fast && g_policy != SB_PATH_UNFUSED && fused_fits(pmax, channels, es) && !u8_unpacked && !unaligned_rows) {
    r.rows = RowPath::Fused;
    r.cols = ColPath::None;
    return r;
  }
  sb::Tiling wt;
  if (fast && g_policy == SB_PATH_FUSED_WIDE && src_dtype == SB_DTYPE_F32 && channels == 1 &&
      fusedw_tiling(radii, k, pmax, &wt)) {
    r.rows = RowPath::FusedWide;
    r.cols = ColPath::None;
    return r;
  }
  if (fast) {
    if (stream_rows_fits(src_dtype, pmax, channels, width))
      r.rows = RowPath::Stream;
    else if (tiled_rows_fits(sb::Mode::RowsToMid, pmax, channels, es))
      r.rows = RowPath::Tiled;
    sb::Tiling ct = make_tiling(sb::Mode::ColsFromMid, pmax, channels, 4, false), pt;
    if (cols_prefix_tiling(ct, radii, k, pmax, &pt))
      r.cols = ColPath::Prefix;
    else if (running_cols_fits(radii, pmax, channels))
      r.cols = ColPath::Running;
  }
  if (r.rows == RowPath::Generic) r.scratch_bytes = sb::generic_rows_scratch_bytes((int)width, r.wide);
  return r;
}

RowPath route_rows_only(int src_dtype, int64_t width, int k, int pmax) {
  if (k <= sb::FAST_K && g_policy != SB_PATH_GENERIC && !needs_wide(pmax) &&
      tiled_rows_fits(sb::Mode::RowsToOut, pmax, 1, dtype_size(src_dtype)))
    return RowPath::Tiled;
  (void)width;
  return RowPath::Generic;
}

int device_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  static int cache[64] = {0};
  if (!cache[dev]) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = sms;
  }
  return cache[dev];
}

}  // namespace

extern "C" {

int sb_version(void) { return 4; }

int sb_set_path_policy(int policy) {
  if (policy < SB_PATH_AUTO || policy > SB_PATH_U8_TWO_BAND) return -1;
  const int prev = g_policy;
  g_policy = policy;
  return prev;
}

size_t sb_filter_at_workspace_bytes(int64_t height, int64_t ncols) {
  if (height < 1 || ncols < 1) return 0;
  return (size_t)height * (size_t)ncols * sizeof(int);
}

int sb_filter_at(const void* src, int src_dtype, int64_t height, int64_t width, int64_t src_row_stride,
                 const int32_t* cols, int64_t ncols, const int32_t* pt_col, const int32_t* pt_y, int64_t npts,
                 float* out, const int64_t* radii, const double* weights, int k, double value_bound, void* workspace,
                 size_t workspace_bytes, int* status_dev, void* stream) {
  if (!src || !cols || !pt_col || !pt_y || !out || height < 1 || width < 1 || ncols < 1 || npts < 1)
    return fail(SB_ERR_INVALID_ARGUMENT, "filter_at needs a non-empty image, columns and points");
  if (src_row_stride < width) return fail(SB_ERR_INVALID_ARGUMENT, "row stride smaller than the width");
  if (height > 0x7fffffffLL || width > 0x7fffffffLL || ncols > 65535)
    return fail(SB_ERR_INVALID_ARGUMENT, "filter_at: image or column set too large");
  int rc = sb_check_kernel(radii, weights, k, width);  // filtering.py:119-120
  if (rc) return rc;
  rc = sb_check_kernel(radii, weights, k, height);
  if (rc) return rc;
  static thread_local Plan plan;  // 16 KB of generic taps: not on the stack of every call
  // the same quanta as the full filter of this image (sb_separable_filter_2d): wide past kWideSpan
  rc = make_taps(radii, weights, k, src_dtype, value_bound, &plan, needs_wide((int)radii[k - 1]));
  if (rc) return rc;
  const size_t need = sb_filter_at_workspace_bytes(height, ncols);
  if (!workspace || workspace_bytes < need)
    return fail(SB_ERR_WORKSPACE, "workspace of " + std::to_string(need) + " bytes required");
  const int e = sb::launch_filter_at(src, src_dtype, src_row_stride, (int)height, (int)width, cols, (int)ncols,
                                     pt_col, pt_y, npts, out, (int*)workspace, plan.tg, status_dev,
                                     (cudaStream_t)stream);
  if (e) return cuda_fail((cudaError_t)e, "filter_at launch");
  return SB_OK;
}

const char* sb_last_error(void) { return g_last_error.c_str(); }

int sb_check_kernel(const int64_t* radii, const double* weights, int k, int64_t extent) {
  int rc = validate_kernel(radii, weights, k);
  if (rc) return rc;
  if (radii[k - 1] >= extent)
    return fail(SB_ERR_KERNEL_TOO_LARGE, "slice radius " + std::to_string(radii[k - 1]) + " does not fit extent " +
                                             std::to_string(extent));
  double dc = 0.0;
  for (int i = 0; i < k; ++i) dc += weights[i] * (2.0 * (double)radii[i] + 1.0);
  if (std::fabs(dc - 1.0) > 1e-6) return fail(SB_ERR_NOT_UNIT_DC, "kernel must have unit DC gain; call normalized()");
  return SB_OK;
}

// Row pitch (elements) of the intermediate plane: the width rounded up to four elements, so plane
// rows are 16-byte multiples for every image width (cols2_kernel's TMA loads need that)
static int64_t plane_width(int64_t width) { return (width + 3) & ~(int64_t)3; }

size_t sb_separable_filter_2d_workspace_bytes(int src_dtype, int64_t batch, int64_t height, int64_t width,
                                              int channels, const int64_t* radii, int k) {
  if (!radii || k < 1 || k > SB_MAX_K || batch < 1 || height < 1 || width < 1 || channels < 1) return 0;
  if (dtype_size(src_dtype) == 0 || radii[k - 1] < 0 || radii[k - 1] > 0x7fffffff) return 0;
  const Route r = route_2d(src_dtype, width, channels, radii, k);
  if (r.rows == RowPath::Fused || r.rows == RowPath::FusedWide || r.rows == RowPath::RowTile) return 0;
  const size_t plane = (size_t)batch * height * plane_width(width) * channels * (r.wide ? sizeof(long long) : sizeof(int));
  return r.scratch_bytes ? align256(plane) + r.scratch_bytes : plane;
}

int sb_separable_filter_2d_window(const void* src, int src_dtype, int64_t batch, int64_t height, int64_t width,
                                  int channels, int64_t src_image_stride, int64_t src_row_stride,
                                  int64_t row_begin, int64_t row_end, float* dst, int64_t dst_image_stride,
                                  int64_t dst_row_stride, const int64_t* radii, const double* weights, int k,
                                  double value_bound, void* workspace, size_t workspace_bytes, int* status_dev,
                                  void* stream) {
  if (row_begin < 0 || row_end > height || row_begin >= row_end)
    return fail(SB_ERR_INVALID_ARGUMENT, "need 0 <= row_begin < row_end <= height");
  if (!src || !dst) return fail(SB_ERR_INVALID_ARGUMENT, "src/dst must not be NULL");
  if (batch < 1 || height < 1 || width < 1) return fail(SB_ERR_INVALID_ARGUMENT, "need a non-empty 2D image");
  if (channels < 1) return fail(SB_ERR_INVALID_ARGUMENT, "channels must be >= 1");
  if (height > 0x7fffffff || width > 0x7fffffff) return fail(SB_ERR_INVALID_ARGUMENT, "extent exceeds int32");
  if (src_row_stride < width * channels || dst_row_stride < width * channels)
    return fail(SB_ERR_INVALID_ARGUMENT, "row stride smaller than width * channels");
  if (batch > 1 && (src_image_stride < height * src_row_stride ||
                    dst_image_stride < (row_end - row_begin) * dst_row_stride))
    return fail(SB_ERR_INVALID_ARGUMENT, "image stride smaller than rows * row stride");
  int rc = sb_check_kernel(radii, weights, k, width);
  if (rc) return rc;
  rc = sb_check_kernel(radii, weights, k, height);
  if (rc) return rc;
  const Route route = route_2d(src_dtype, width, channels, radii, k);
  static thread_local Plan plan;
  rc = make_taps(radii, weights, k, src_dtype, value_bound, &plan, route.wide);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;

  sb::Geometry g;
  std::memset(&g, 0, sizeof(g));
  g.in_img = src_image_stride;
  g.in_row = src_row_stride;
  g.in_px = channels;
  g.es = dtype_size(src_dtype);
  g.out_img = dst_image_stride;
  g.out_row = dst_row_stride;
  g.out_px = channels;
  g.H = (int)height;
  g.W = (int)width;
  g.nimg = (int)batch;
  g.oy0 = (int)row_begin;
  g.oy1 = (int)row_end;
  g.aligned16 = ((uintptr_t)src % 16 == 0) && ((src_row_stride * g.es) % 16 == 0) &&
                (batch == 1 || (src_image_stride * g.es) % 16 == 0);
  g.out_bulk = channels == 1 && ((uintptr_t)dst % 16 == 0) && ((dst_row_stride * 4) % 16 == 0) &&
               (batch == 1 || (dst_image_stride * 4) % 16 == 0);
  const long long total_rows = (long long)batch * (row_end - row_begin);  // rows the column sweep outputs
  const long long all_rows = (long long)batch * height;                   // rows the row pass produces
  if (route.rows == RowPath::Fused) {
    const bool u8_single = (src_dtype == SB_DTYPE_U8 && channels == 1);
    const sb::Tiling base = make_tiling(sb::Mode::Fused, plan.pmax, channels, g.es, u8_single);
    // rows that are 4-byte but not 16-byte multiples (a 1000-pixel-wide uint8 image): the two-band
    // kernel instantiated with 4-byte staging copies (64 x 1000^2: 0.43 -> 0.165 ms)
    const bool words = !g.aligned16 && (((uintptr_t)src | (uintptr_t)(g.in_row * g.es) |
                                         (uintptr_t)((batch > 1 ? g.in_img : 0) * g.es)) & 3) == 0;
    const void* fn = base.split == 3   ? sb::sweep_ptr_fused3(k)
                     : base.split == 5 ? (words ? sb::sweep_ptr_fused5w(k) : sb::sweep_ptr_fused5(k))
                     : base.split == 6 ? sb::sweep_ptr_fusedp(k)
                     : (src_dtype == SB_DTYPE_F32 && channels == 1) ? sb::sweep_ptr_fused_f32(k, base.ls)
                                                                     : pick_kernel(sb::Mode::Fused, src_dtype, k);
    Launch L;
    rc = plan_launch(fn, sb::Mode::Fused, base, plan.pmax, g.W, total_rows, channels, &L);
    if (rc) return rc;
    return launch_fused(fn, L, src, dst, g, plan.taps, status_dev, st);
  }
  if (route.rows == RowPath::RowTile) {
    sb::Tiling tl;
    if (!rowtile_tiling(plan.pmax, &tl)) return fail(SB_ERR_INVALID_ARGUMENT, "row-tile tiling");
    tl.nstrips = (g.W + sb::WS - 1) / sb::WS;
    const void* fn = sb::sweep_ptr_rowtile(k);
    const size_t smem = (size_t)tl.obuf_off + 128 + (size_t)4 * sb::TOG * sb::TOBUF * sb::TB * 32 * sizeof(float);
    FnFacts ff;
    DevFacts df;
    rc = launch_facts(fn, smem, &ff, &df);
    if (rc) return rc;
    tl.rows_per_item = persistent_chunk(total_rows, tl.nstrips, df.sms, 2LL * plan.pmax + 1 + sb::TB, sb::TB);
    const long long units = ((total_rows + tl.rows_per_item - 1) / tl.rows_per_item) * tl.nstrips;
    const long long grid = std::min<long long>(df.sms, units);
    sb::Geometry gr = g;
    alignas(64) CUtensorMap omap;
    make_output_map(dst, gr, &omap);
    if (debug_plans())
      std::fprintf(stderr, "[sliceblur_b200] row-tile: pmax=%d L=%d srb=%d s0=%d ta=%d D=%d smem=%zu grid=%lld chunk=%lld units=%lld\n",
                   plan.pmax, tl.L, tl.stage_row_bytes, tl.s0, tl.ta, tl.D, smem, grid, tl.rows_per_item, units);
    void* args[] = {(void*)&src, (void*)&dst, (void*)&gr, (void*)&plan.taps, (void*)&tl, (void*)&omap};
    cudaError_t e = cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(sb::TTHREADS), args, smem, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernel");
    return SB_OK;
  }
  if (route.rows == RowPath::FusedWide) {
    sb::Tiling tl;
    if (!fusedw_tiling(radii, k, plan.pmax, &tl)) return fail(SB_ERR_INVALID_ARGUMENT, "wide sweep tiling");
    tl.nstrips = (g.W + sb::WS - 1) / sb::WS;
    const void* fn = sb::sweep_ptr_fusedw(k, tl.ls);
    const size_t smem = (size_t)tl.obuf_off + 128 + (size_t)4 * sb::WCG * 2 * sb::HB * 32 * sizeof(float);
    FnFacts ff;
    DevFacts df;
    rc = launch_facts(fn, smem, &ff, &df);
    if (rc) return rc;
    // persistent: one CTA per SM over (row chunk, strip) units taken round-robin; the chunk
    // height minimises (rounds of units) x (chunk rows + the 2*pmax+1 warm-up rows)
    const long long warm = 2LL * plan.pmax + 1 + sb::HB;
    long long best_chunks = 1;
    double best_cost = 1e300;
    for (long long nc = 1; nc <= 64 && nc <= std::max(1LL, total_rows / sb::HB); ++nc) {
      const long long units = nc * tl.nstrips;
      const long long rounds = (units + df.sms - 1) / df.sms;
      const double cost = (double)rounds * (double)((total_rows + nc - 1) / nc + warm);
      if (cost < best_cost * 0.995) {
        best_cost = cost;
        best_chunks = nc;
      }
    }
    tl.rows_per_item = (total_rows + best_chunks - 1) / best_chunks;
    const long long units = ((total_rows + tl.rows_per_item - 1) / tl.rows_per_item) * tl.nstrips;
    const long long grid = std::min<long long>(df.sms, units);
    sb::Geometry gw = g;
    alignas(64) CUtensorMap omap;
    make_output_map(dst, gw, &omap);
    if (debug_plans())
      std::fprintf(stderr, "[sliceblur_b200] wide fused: pmax=%d L=%d ls=%d fp=%d ds=%d lag=%d deep=%x smem=%zu grid=%lld "
                   "chunk=%lld units=%lld\n",
                   plan.pmax, tl.L, tl.ls, tl.pf, tl.ds, tl.lag, tl.deepmask, smem, grid, tl.rows_per_item, units);
    void* args[] = {(void*)&src, (void*)&dst, (void*)&gw, (void*)&plan.taps, (void*)&tl, (void*)&status_dev,
                    (void*)&omap};
    cudaError_t e = cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(sb::WTHREADS), args, smem, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernel");
    return SB_OK;
  }
  // two passes through an int32 workspace laid out [channel][batch][H][W]
  const size_t need = sb_separable_filter_2d_workspace_bytes(src_dtype, batch, height, width, channels, radii, k);
  if (!workspace || workspace_bytes < need)
    return fail(SB_ERR_WORKSPACE, "workspace of " + std::to_string(need) + " bytes required");
  int* mid = (int*)workspace;
  g.mid_row = (long long)plane_width(width);  // rows padded to 16 bytes: the plane keeps its TMA tensor map
  g.mid_img = (long long)height * g.mid_row;
  g.mid_ch = g.mid_img * batch;
  const int sms = device_sms();

  // ---- row pass
  if (route.rows == RowPath::Stream) {
    // streaming row pass: full-width bands, prefix carried across chunks
    const int xs = -(((plan.pmax + 1) + 15) & ~15);  // first halo column, 16-aligned
    // interleaved channels with 16-byte aligned rows: bands of virtual (row, channel) rows, the
    // image rows staged once for all channels (stream_rows_mc_kernel); else one channel per CTA
    // rows that are not 16-byte multiples are staged from aligned-down addresses (unal); the
    // first image row must be 16-byte aligned so no copy starts before the caller's buffer
    const int unal = (g.in_row * g.es) % 16 != 0 || (g.in_img * g.es) % 16 != 0;
    const bool mc = SB_STREAM_MC && channels >= 2 && channels <= 4 && g.in_px == channels &&
                    (uintptr_t)src % 16 == 0 && (!unal || SB_STREAM_MC_UNALIGNED) &&
                    all_rows * g.mid_row * channels < (1LL << 31) && (src_dtype == SB_DTYPE_F32 || SB_STREAM_ALL_TYPES);
    const void* fs = mc                            ? sb::sweep_ptr_stream_mc(src_dtype, k)
                     : src_dtype == SB_DTYPE_F32   ? sb::sweep_ptr_stream_f32(k)
                     : src_dtype == SB_DTYPE_F64   ? sb::sweep_ptr_stream_f64(k)
                     : src_dtype == SB_DTYPE_U16   ? sb::sweep_ptr_stream_u16(k)
                                                   : sb::sweep_ptr_stream_u8(k);
    const size_t stage = mc ? (size_t)sb::stream_stages(g.es) * sb::mc_rows(channels) *
                                  (sb::CW * channels * (size_t)g.es + sb::SRB_PAD + (unal ? 16 : 0))
                            : (size_t)sb::NPROD * sb::stream_stages(g.es) * 8 *
                                  (sb::CW * (size_t)g.es + sb::SRB_PAD + (stream_unaligned(src, g) ? 16 : 0));
    const size_t smem = stage + (size_t)sb::HB * sb::RLS * sizeof(int);
    FnFacts ff;
    DevFacts df;
    rc = launch_facts(fs, smem, &ff, &df);
    if (rc) return rc;
    const int nb_total = (int)(((mc ? all_rows * channels : all_rows) + sb::HB - 1) / sb::HB);
    // Column segments: a unit is (band, segment), each segment re-scanning its own left halo.
    // The count minimises (rounds of units over the resident CTAs) x (segment + halo width), so
    // images with few rows fill the SMs (128 x 524288, p_max 103: 2.88 -> 0.52 ms) and a
    // ragged last round is evened out (C4: 1536 bands on 296 CTA slots).
    const int segw = stream_segment_width(width, plan.pmax, (long long)nb_total * (mc ? 1 : channels), df.sms);
    const int units_total = nb_total * (int)((width + segw - 1) / segw);
    const int gx = mc ? std::max(1, std::min(units_total, df.sms * 2 * 8))
                      : std::max(1, std::min(units_total, df.sms * 2 * 8 / std::max(1, channels)));
    void* args_mc[] = {(void*)&src, (void*)&mid, (void*)&g, (void*)&plan.taps, (void*)&xs, (void*)&nb_total,
                       (void*)&segw, (void*)&unal, (void*)&status_dev};
    void* args_1c[] = {(void*)&src, (void*)&mid, (void*)&g, (void*)&plan.taps, (void*)&xs, (void*)&nb_total,
                       (void*)&segw, (void*)&status_dev};
    void** args = mc ? args_mc : args_1c;
    if (debug_plans())
      std::fprintf(stderr, "[sliceblur_b200] stream rows: pmax=%d xs=%d bands=%d segw=%d grid=%d x %d smem=%zu\n",
                   plan.pmax, xs, nb_total, segw, gx, channels, smem);
    cudaError_t e = cudaLaunchKernel(fs, dim3(mc ? gx : gx * channels, 1), dim3(sb::STREAM_THREADS), args, smem, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernel");
  } else if (route.rows == RowPath::Tiled) {
    const void* f1 = pick_kernel(sb::Mode::RowsToMid, src_dtype, k);
    Launch L1;
    rc = plan_launch(f1, sb::Mode::RowsToMid, make_tiling(sb::Mode::RowsToMid, plan.pmax, channels, g.es, false),
                     plan.pmax, g.W, all_rows, channels, &L1);
    if (rc) return rc;
    rc = launch_rows(f1, L1, src, mid, nullptr, g, plan.taps, status_dev, st);
    if (rc) return rc;
  } else {
    const size_t plane =
        (size_t)batch * height * plane_width(width) * channels * (route.wide ? sizeof(long long) : sizeof(int));
    void* scratch = route.scratch_bytes ? (void*)((char*)workspace + align256(plane)) : nullptr;
    if (debug_plans())
      std::fprintf(stderr, "[sliceblur_b200] generic rows: pmax=%d k=%d W=%d wide=%d scratch=%zu\n", plan.pmax, k,
                   g.W, (int)route.wide, route.scratch_bytes);
    const int e =
        sb::launch_rows_generic(src, src_dtype, mid, nullptr, g, plan.tg, scratch, route.wide, status_dev, sms, st);
    if (e) return cuda_fail((cudaError_t)e, "generic row pass");
  }

  // ---- column pass
  ColPath cols = route.cols;
  if (cols == ColPath::Prefix) {
    sb::Tiling ct = make_tiling(sb::Mode::ColsFromMid, plan.pmax, channels, 4, false), pt;
    alignas(64) CUtensorMap mmap;
    if (make_plane_map(mid, g, channels, &mmap) && cols_prefix_tiling(ct, radii, k, plan.pmax, &pt)) {
      // ring-only tilings with an even number (>= 4) of TMA slots take the split loader (two loader
      // warps per lane quadrant; C4 1.028 -> 1.002 ms).  With band copies the copies serialise the
      // two halves and the tiling loses slack to the extra slots (C5 4.14 -> 4.33 ms): one half.
      const bool split = SB_COLS2_SPLIT && pt.ds == 0 && pt.pf >= 4 && pt.pf % 2 == 0;
      const void* f3 = split ? sb::sweep_ptr_cols2s(k) : sb::sweep_ptr_cols2(k);
      Launch L3;
      rc = plan_launch(f3, sb::Mode::ColsPrefix, pt, plan.pmax, g.W, total_rows, channels, &L3);
      if (rc) return rc;
      sb::Geometry g2 = g;
      alignas(64) CUtensorMap omap;
      make_output_map(dst, g2, &omap);
      void* args[] = {(void*)&mid, (void*)&dst, (void*)&g2, (void*)&plan.taps, (void*)&L3.tl, (void*)&omap,
                      (void*)&mmap};
      // channels are folded into grid.x (fastest varying), as in cols_kernel
      cudaError_t e = cudaLaunchKernel(f3, dim3(L3.grid.x * L3.grid.y), dim3(split ? sb::C2STHREADS : sb::C2THREADS), args,
                                       L3.smem, st);
      if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernel");
      return SB_OK;
    }
    cols = running_cols_fits(radii, plan.pmax, channels) ? ColPath::Running : ColPath::Generic;
  }
  if (cols == ColPath::Running) {
    const void* f2 = pick_kernel(sb::Mode::ColsFromMid, src_dtype, k);
    sb::Tiling ct = make_tiling(sb::Mode::ColsFromMid, plan.pmax, channels, 4, false, (int)radii[0]);
    // deep trails (older than the ring) of the largest boxes come through shared memory
    ct.ndeep = 0;
    for (int d = 0; d < sb::SB_NDEEP && d < k; ++d)
      if (2 * sb::HB + plan.pmax + (int)radii[k - 1 - d] > ct.D) ct.ndeep = d + 1;
    const size_t band = (size_t)sb::HB * sb::WS * sizeof(int);
    const size_t budget = (512 / ct.tmem_cols) > 1 ? 100 * 1024 : 200 * 1024;
    ct.pf = 2;
    for (int pf : {8, 6, 4, 3, 2})
      if ((size_t)(1 + ct.ndeep) * pf * band <= budget) {
        ct.pf = pf;
        break;
      }
    Launch L2;
    rc = plan_launch(f2, sb::Mode::ColsFromMid, ct, plan.pmax, g.W, total_rows, channels, &L2);
    if (rc) return rc;
    return launch_cols(f2, L2, mid, dst, g, plan.taps, st);
  }
  if (debug_plans()) std::fprintf(stderr, "[sliceblur_b200] generic cols: pmax=%d k=%d\n", plan.pmax, k);
  const int e = sb::launch_cols_generic(mid, dst, g, plan.tg, route.wide, sms, st);
  if (e) return cuda_fail((cudaError_t)e, "generic column pass");
  return SB_OK;
}

int sb_separable_filter_2d(const void* src, int src_dtype, int64_t batch, int64_t height, int64_t width,
                           int channels, int64_t src_image_stride, int64_t src_row_stride, float* dst,
                           int64_t dst_image_stride, int64_t dst_row_stride, const int64_t* radii,
                           const double* weights, int k, double value_bound, void* workspace,
                           size_t workspace_bytes, int* status_dev, void* stream) {
  if (height < 1) return fail(SB_ERR_INVALID_ARGUMENT, "need a non-empty 2D image");
  return sb_separable_filter_2d_window(src, src_dtype, batch, height, width, channels, src_image_stride,
                                       src_row_stride, 0, height, dst, dst_image_stride, dst_row_stride, radii,
                                       weights, k, value_bound, workspace, workspace_bytes, status_dev, stream);
}

size_t sb_filter_rows_workspace_bytes(int src_dtype, int64_t rows, int64_t width, const int64_t* radii, int k) {
  if (!radii || k < 1 || k > SB_MAX_K || rows < 1 || width < 1 || width > 0x7fffffff) return 0;
  if (dtype_size(src_dtype) == 0 || radii[k - 1] < 0 || radii[k - 1] > 0x7fffffff) return 0;
  if (route_rows_only(src_dtype, width, k, (int)radii[k - 1]) != RowPath::Generic) return 0;
  return sb::generic_rows_scratch_bytes((int)width, needs_wide((int)radii[k - 1]));
}

int sb_filter_rows(const void* src, int src_dtype, int64_t rows, int64_t width, int64_t src_row_stride, float* dst,
                   int64_t dst_row_stride, const int64_t* radii, const double* weights, int k, double value_bound,
                   void* workspace, size_t workspace_bytes, int* status_dev, void* stream) {
  if (!src || !dst) return fail(SB_ERR_INVALID_ARGUMENT, "src/dst must not be NULL");
  if (rows < 1 || width < 1) return fail(SB_ERR_INVALID_ARGUMENT, "need a non-empty signal");
  if (rows > 0x7fffffff || width > 0x7fffffff) return fail(SB_ERR_INVALID_ARGUMENT, "extent exceeds int32");
  if (src_row_stride < width || dst_row_stride < width)
    return fail(SB_ERR_INVALID_ARGUMENT, "row stride smaller than width");
  int rc = sb_check_kernel(radii, weights, k, width);
  if (rc) return rc;
  const bool wide = needs_wide((int)radii[k - 1]);
  static thread_local Plan plan;
  rc = make_taps(radii, weights, k, src_dtype, value_bound, &plan, wide);
  if (rc) return rc;
  sb::Geometry g;
  std::memset(&g, 0, sizeof(g));
  g.in_row = src_row_stride;
  g.in_px = 1;
  g.es = dtype_size(src_dtype);
  g.out_row = dst_row_stride;
  g.out_px = 1;
  g.H = (int)rows;
  g.W = (int)width;
  g.nimg = 1;
  g.aligned16 = ((uintptr_t)src % 16 == 0) && ((src_row_stride * g.es) % 16 == 0);
  if (SB_STREAM_ROWS_OUT && k <= sb::FAST_K && !wide && g_policy != SB_PATH_GENERIC && rows >= sb::HB / 2 &&
      stream_rows_fits(src_dtype, plan.pmax, 1, width) && rows * dst_row_stride < (1LL << 31)) {
    // the streaming row pass with float rows out (8192^2 sigma 64: float32 0.85 -> 0.21 ms, float64 2.08 -> 0.28 ms)
    const int xs = -(((plan.pmax + 1) + 15) & ~15);
    const void* fs = sb::sweep_ptr_stream_out(src_dtype, k);
    const size_t smem = (size_t)sb::NPROD * sb::stream_stages(g.es) * 8 *
                            (sb::CW * (size_t)g.es + sb::SRB_PAD + (stream_unaligned(src, g) ? 16 : 0)) +
                        (size_t)sb::HB * sb::RLS * sizeof(int);
    FnFacts ff;
    DevFacts df;
    rc = launch_facts(fs, smem, &ff, &df);
    if (rc) return rc;
    g.mid_row = dst_row_stride;
    g.mid_img = rows * dst_row_stride;
    g.mid_ch = 0;
    int* out_words = (int*)dst;
    const int nb_total = (int)((rows + sb::HB - 1) / sb::HB);
    const int segw = stream_segment_width(width, plan.pmax, nb_total, df.sms);
    const int units_total = nb_total * (int)((width + segw - 1) / segw);
    const int gx = std::max(1, std::min(units_total, df.sms * 2 * 8));
    void* args[] = {(void*)&src, (void*)&out_words, (void*)&g, (void*)&plan.taps, (void*)&xs, (void*)&nb_total,
                    (void*)&segw, (void*)&status_dev};
    cudaError_t e = cudaLaunchKernel(fs, dim3(gx, 1), dim3(sb::STREAM_THREADS), args, smem, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernel");
    return SB_OK;
  }
  if (route_rows_only(src_dtype, width, k, plan.pmax) == RowPath::Tiled) {
    const void* fn = pick_kernel(sb::Mode::RowsToOut, src_dtype, k);
    Launch L;
    rc = plan_launch(fn, sb::Mode::RowsToOut, make_tiling(sb::Mode::RowsToOut, plan.pmax, 1, g.es, false),
                     plan.pmax, g.W, rows, 1, &L);
    if (rc) return rc;
    return launch_rows(fn, L, src, nullptr, dst, g, plan.taps, status_dev, (cudaStream_t)stream);
  }
  const size_t need = sb_filter_rows_workspace_bytes(src_dtype, rows, width, radii, k);
  if (need && (!workspace || workspace_bytes < need))
    return fail(SB_ERR_WORKSPACE, "workspace of " + std::to_string(need) + " bytes required");
  const int e = sb::launch_rows_generic(src, src_dtype, nullptr, dst, g, plan.tg, need ? workspace : nullptr, wide,
                                        status_dev, device_sms(), (cudaStream_t)stream);
  if (e) return cuda_fail((cudaError_t)e, "generic row pass");
  return SB_OK;
}

int sb_slice_filter_1d(const void* src, int src_dtype, int64_t n, float* dst, const int64_t* radii,
                       const double* weights, int k, double value_bound, void* workspace, size_t workspace_bytes,
                       int* status_dev, void* stream) {
  if (n < 1) return fail(SB_ERR_INVALID_ARGUMENT, "need a non-empty 1D signal");
  return sb_filter_rows(src, src_dtype, 1, n, n, dst, n, radii, weights, k, value_bound, workspace, workspace_bytes,
                        status_dev, stream);
}

}  // extern "C"
