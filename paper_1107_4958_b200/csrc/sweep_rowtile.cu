// sweep_rowtile.cu - uint8 one-channel fused sweep with the row pass on "thread = row"
// warps that keep their row prefix in tensor memory (the headline C3 config: 256 x 1024^2
// uint8, k = 3, radii 7 / 14 / 23).
//
// Reference: separable_filter_2d (filtering.py:76-104): _filter_rows (filtering.py:48-64)
// over the rows, then over the columns of the result; replicate boundaries
// (filtering.py:10-13).  Same arithmetic as fused_kernel<uint8_t, K, 2, true>, so the
// results are bit-identical: exact row prefixes held as the fp32 numbers 2^23 + prefix, box
// sums by one exact FADD2 per row pair, weighted with FFMA2, rounded to the mid quantum;
// exact int32 column prefixes; box sums C(y+p) - C(y-p-1).
//
// Why: in fused_kernel the consumer warps (thread = column) read the K lead and K trail
// prefixes of every row from shared memory (24 B/px) and are latency- and
// shared-memory-bound.  Here a row warp owns 32 rows of a band as its TMEM lane quadrant:
//  * row warps (0..7; warp w takes bands gb = w mod 8, TMEM lane quadrant w mod 4 and row-prefix
//    region w / 4; thread t = row t of the band): stage
//    the row's [xb, xb + L) bytes with cp.async (the warp's next band is staged right after
//    the scan, so seven other bands hide the latency), prefix-scan them with IDP4A (one per
//    byte) into TMEM columns [0, ta) of its lane, then read the lead / trail windows of
//    every 16 output columns back with unaligned tcgen05.ld.x16 and form the row values in
//    registers; the 32 x 128 band of rounded row values goes to a shared-memory slot
//    (16-byte stores, 8 B/px of shared-memory traffic instead of 24);
//  * loader warps (8..11; thread = column c, TMEM lane c): read the slot's column, accumulate
//    the column prefix C (exact int32, wraps) and append the 32 rows to the ring in TMEM
//    columns [2 ta, 2 ta + D) (first 32 rows mirrored after the end, so every 32-row window is
//    contiguous);
//  * output groups (12..19, TOG groups of four; output band j = g mod TOG): two TMEM windows
//    per box, staged and written by TMA tensor stores.
// Persistent grid, one CTA per SM over (row chunk, strip) units (WorkIter, 32-row bands).
#include "sweep_kernels.cuh"

namespace sb {

#ifndef SB_RT_OUT_BACKOFF
#define SB_RT_OUT_BACKOFF 1
#endif

// Position in the CTA's band list: band pb of segment w, CTA-global index gb.
struct BandCursor {
  WorkIter w;
  int pb;
  uint32_t gb;
  __device__ __forceinline__ void adv() {
    ++gb;
    if (++pb == w.nbands) {
      w.next();
      pb = 0;
    }
  }
};

template <int K>
__global__ void __launch_bounds__(TTHREADS, 1)
    rowtile_kernel(const uint8_t* __restrict__ src, float* __restrict__ dst, Geometry g, Taps t, Tiling tl,
                   const __grid_constant__ CUtensorMap omap) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t tmem_base_s;
  __shared__ __align__(8) uint64_t rfull[TRS];
  __shared__ uint32_t ld_cnt[4];           // bands whose row values loader warp q has read
  __shared__ uint32_t ring_cnt[4];         // ring bands written, per lane quadrant (loader warp q)
  __shared__ uint32_t out_cnt[TOG][4];     // output bands done, per output group and lane quadrant
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3;  // TMEM lane quadrant
  const int wh = g.oy1 - g.oy0;
  const long long total = (long long)g.nimg * wh;
  const int D = tl.D, NBR = D / TB, srb = tl.stage_row_bytes;
  unsigned char* abase = smem + (((smem_u32(smem) + 127u) & ~127u) - smem_u32(smem));  // 128-byte aligned
  unsigned char* stage = abase;                                      // [TROWW][TB][srb] staged rows
  float* rslot = (float*)(abase + TROWW * TB * srb);                 // [TRS][TB][TRSW] row values (bits)
  float* obuf = (float*)(abase + tl.obuf_off);                       // [4 TOG][2][TB][32] output boxes
  if (threadIdx.x == 0) {
    for (int i = 0; i < TRS; ++i) mbar_init(&rfull[i], 32);  // the row warp's lanes
    for (int i = 0; i < 4; ++i) ld_cnt[i] = 0;
    for (int i = 0; i < 4; ++i) ring_cnt[i] = 0;
    for (int i = 0; i < TOG * 4; ++i) out_cnt[i / 4][i % 4] = 0;
  }
  if (warp == 0) tmem_alloc(&tmem_base_s, (uint32_t)tl.tmem_cols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tq = tmem_base_s + ((uint32_t)(32 * q) << 16);  // this warp's lane quadrant, column 0
  const uint32_t tring = tq + (uint32_t)(2 * tl.ta);  // after the two row-prefix regions

  if (warp < TROWW) {
    // ------------------------------------------------ row warps
    unsigned char* stg = stage + (warp * TB + lane) * srb;  // this thread's staged row
    const uint32_t ta0 = tq + (uint32_t)((warp >> 2) * tl.ta);  // TROWW = 4: region 0 only  // row-prefix region of this warp (sub warp >> 2)
    const int nq = tl.L / 16;
    BandCursor cur, nxt;  // the band being processed / the next band to stage (both this warp's)
    cur.w.init(total, tl.rows_per_item, tl.nstrips, wh, g.oy0, t.pmax, TB);
    cur.pb = 0;
    cur.gb = 0;
    for (int i = 0; i < warp && cur.w.valid; ++i) cur.adv();  // bands gb = warp (mod TROWW)
    nxt = cur;
    auto stage_band = [&](const BandCursor& b) {
      const int xb = b.w.strip * WS - tl.xoff;
      const int v = min(max(b.w.a - 1 - t.pmax + b.pb * TB + lane, 0), g.H - 1);
      const uint8_t* grow = src + (long long)b.w.img * g.in_img + (long long)v * g.in_row;
      for (int j = 0; j < nq; ++j) {
        const int col = xb + 16 * j;
        if (g.aligned16 && col >= 0 && col + 16 <= g.W) cp_async16(stg + 16 * j, grow + col);
      }
      cp_async_commit();
    };
    if (nxt.w.valid) stage_band(nxt);
    while (cur.w.valid) {
      const BandCursor b = cur;
      for (int i = 0; i < TROWW && cur.w.valid; ++i) cur.adv();
      nxt = cur;
      const int xb = b.w.strip * WS - tl.xoff;
      cp_async_wait_all();
      if (!g.aligned16 || xb < 0 || xb + tl.L > g.W) {
        // columns outside the image replicate the border (filtering.py:10-13); unaligned
        // rows and partial chunks are copied byte by byte
        const int v = min(max(b.w.a - 1 - t.pmax + b.pb * TB + lane, 0), g.H - 1);
        const uint8_t* grow = src + (long long)b.w.img * g.in_img + (long long)v * g.in_row;
        for (int j = 0; j < nq; ++j) {
          const int col = xb + 16 * j;
          if (g.aligned16 && col >= 0 && col + 16 <= g.W) continue;
          for (int e = 0; e < 16; ++e) stg[16 * j + e] = grow[min(max(col + e, 0), g.W - 1)];
        }
      }
      // prefix of staged bytes [s0, s0 + ta) as 2^23 + prefix (bit pattern 0x4B000000 + prefix),
      // 16 columns per tcgen05.st; s0 is 8-byte aligned, so a group of 16 bytes is the upper
      // half of one 16-byte chunk and the lower half of the next when s0 = 8 (mod 16)
      {
        uint32_t base = 0x4B000000u;
        const unsigned char* sp = stg + (tl.s0 & ~15);
        const bool half = (tl.s0 & 15) != 0;
        uint4 prev = *(const uint4*)sp;
        for (int j = 0; j < tl.ta / 16; ++j) {
          uint32_t wd[4];
          if (half) {
            const uint4 nx = *(const uint4*)(sp + 16 * (j + 1));
            wd[0] = prev.z, wd[1] = prev.w, wd[2] = nx.x, wd[3] = nx.y;
            prev = nx;
          } else {
            const uint4 w4 = *(const uint4*)(sp + 16 * j);
            wd[0] = w4.x, wd[1] = w4.y, wd[2] = w4.z, wd[3] = w4.w;
          }
          uint32_t v[16];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            v[4 * m] = __dp4a(wd[m], 0x00000001u, base);
            v[4 * m + 1] = __dp4a(wd[m], 0x00000101u, base);
            v[4 * m + 2] = __dp4a(wd[m], 0x00010101u, base);
            base = __dp4a(wd[m], 0x01010101u, base);
            v[4 * m + 3] = base;
          }
          tmem_st16(ta0 + (uint32_t)(16 * j), v);
        }
      }
      __syncwarp();
      if (nxt.w.valid) stage_band(nxt);  // the staged row is in TMEM now
      tmem_wait_st();
      // row values of the band's 128 columns -> slot gb mod TRS
      const int slot = (int)(b.gb % TRS);
      // the slot's previous band (gb - TRS) has been read by all four loader warps.  A count,
      // not an mbarrier parity: two row warps share a slot and one may arrive here two uses ahead
      if (b.gb >= TRS)
        for (int l = 0; l < 4; ++l) wait_above(&ld_cnt[l], b.gb - TRS, false);
      float* rrow = rslot + (slot * TB + lane) * TRSW;
      const int off0 = tl.xoff - tl.s0;
#pragma unroll 1
      for (int c0 = 0; c0 < WS; c0 += 16) {
        float2 acc[8];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          uint32_t lv[16], tv[16];
          tmem_ld16(ta0 + (uint32_t)(off0 + c0 + t.p[i]), lv);
          tmem_ld16(ta0 + (uint32_t)(off0 + c0 - t.p[i] - 1), tv);
          tmem_wait_ld();
          const float2 w2 = make_float2(t.w_row[i], t.w_row[i]);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float2 l2 = make_float2(__uint_as_float(lv[2 * j]), __uint_as_float(lv[2 * j + 1]));
            const float2 r2 = make_float2(-__uint_as_float(tv[2 * j]), -__uint_as_float(tv[2 * j + 1]));
            const float2 d = __fadd2_rn(l2, r2);  // exact box sums of columns c0+2j, c0+2j+1
            acc[j] = i == 0 ? __fmul2_rn(w2, d) : __ffma2_rn(w2, d, acc[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const float2 a = round_mid2<K>(acc[j]);  // round to the mid quantum
          const float2 c = round_mid2<K>(acc[j + 1]);
          *(float4*)(rrow + c0 + 2 * j) = make_float4(a.x, a.y, c.x, c.y);
        }
      }
      mbar_arrive(&rfull[slot]);
    }
  } else if (warp < TROWW + 4) {
    // ------------------------------------------------ loader warps: column prefix -> TMEM ring
    const int c = 32 * q + lane;
    WorkIter sc, so;  // ring bands / the output bands whose completion gates the ring
    sc.init(total, tl.rows_per_item, tl.nstrips, wh, g.oy0, t.pmax, TB);
    so.init(total, tl.rows_per_item, tl.nstrips, wh, g.oy0, t.pmax, TB);
    uint32_t gb = 0, onum = 0;
    int oob = 0;
    for (; sc.valid; sc.next()) {
      int cprefix = 0;
      for (int pb = 0; pb < sc.nbands; ++pb, ++gb) {
        const int slot = (int)(gb % TRS);
        mbar_wait_wd(&rfull[slot], (gb / TRS) & 1, 2000000 + (int)gb);
        // ring band gb overwrites band gb - NBR: every output band reading it must be done
        while (so.valid && (long long)so.gb0 + oob + NBR <= (long long)gb) {
          wait_above(&out_cnt[onum % TOG][q], onum / TOG, false);
          ++onum;
          if (++oob == (so.b - so.a + TB - 1) / TB) {
            so.next();
            oob = 0;
          }
        }
        const int rs = (int)(gb % (uint32_t)NBR);
        {
          // column prefix of the slot's 32 rows, in two 16-row halves (registers); odd entries
          // chain by 3-input adds, even entries hang off them
          const float* col = rslot + slot * TB * TRSW + c;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            int e[HB];
#pragma unroll
            for (int r = 0; r < HB; ++r) e[r] = __float_as_int(col[(HB * hh + r) * TRSW]) - kMagicBits;
            if (hh == 1) {
              __syncwarp();
              if (lane == 0) st_release(&ld_cnt[q], gb + 1);
            }
            uint32_t cv[HB];
            int odd = cprefix;
#pragma unroll
            for (int r = 0; r < HB; r += 2) {
              cv[r] = (uint32_t)(odd + e[r]);
              odd = odd + e[r] + e[r + 1];
              cv[r + 1] = (uint32_t)odd;
            }
            cprefix = odd;
            tmem_st16(tring + (uint32_t)(rs * TB + HB * hh), cv);
            if (rs == 0) tmem_st16(tring + (uint32_t)(D + HB * hh), cv);  // mirror: 32-row windows never wrap
          }
        }
        tmem_wait_st();
        tmem_fence_before();
        __syncwarp();
        if (lane == 0) st_release(&ring_cnt[q], gb + 1);
      }
    }
  } else {
    // ------------------------------------------------ output groups
    const int grp = (warp - TROWW - 4) / 4;
    const int ow = warp - TROWW - 4;
    uint32_t onum = 0;
    int obsel = 0;
    WorkIter so;
    so.init(total, tl.rows_per_item, tl.nstrips, wh, g.oy0, t.pmax, TB);
    for (; so.valid; so.next()) {
      const int x0 = so.strip * WS;
      const int c = 32 * q + lane;
      const int nout = (so.b - so.a + TB - 1) / TB;
      for (int ob = 0; ob < nout; ++ob, ++onum) {
        if ((int)(onum % TOG) != grp) continue;
        const int j0 = ob * TB;
        const int nb = min(TB, so.b - so.a - j0);
        const uint32_t need = so.gb0 + (uint32_t)((j0 + nb + 2 * t.pmax) / TB);
        wait_above(&ring_cnt[q], need, SB_RT_OUT_BACKOFF);
        tmem_fence_after();
        const int out_mod = (int)(((so.gb0 + (uint32_t)ob) % (uint32_t)NBR) * TB);
        float2 o2[TB / 2];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          int l = out_mod + t.pmax + 1 + t.p[i];
          int tr = out_mod + t.pmax - t.p[i];
          l = l >= D ? l - D : l;
          tr = tr >= D ? tr - D : tr;
          const float2 w2 = make_float2(t.w_col[i], t.w_col[i]);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {  // two 16-row halves (registers)
            uint32_t lv[HB], tv[HB];
            tmem_ld16(tring + (uint32_t)(l + HB * hh), lv);
            tmem_ld16(tring + (uint32_t)(tr + HB * hh), tv);
            tmem_wait_ld();
#pragma unroll
            for (int r = 0; r < HB / 2; ++r) {
              const float2 d =
                  make_float2(i2f_fast(lv[2 * r] - tv[2 * r]), i2f_fast(lv[2 * r + 1] - tv[2 * r + 1]));
              o2[hh * (HB / 2) + r] = i == 0 ? __fmul2_rn(w2, d) : __ffma2_rn(w2, d, o2[hh * (HB / 2) + r]);
            }
          }
        }
        tmem_fence_before();
        __syncwarp();
        if (lane == 0) st_release(&out_cnt[grp][q], onum / TOG + 1);
        const int out_row = so.a + j0 - g.oy0;
        if (g.out_bulk && nb == TB) {
          float* obp = obuf + (ow * TOBUF + (TOBUF == 2 ? obsel : 0)) * (TB * 32);
          if (lane == 0) {  // the stores out of this box (TOBUF bands ago) have read it
            if (TOBUF == 2)
              bulk_wait_read<1>();
            else
              bulk_wait_read<0>();
          }
          __syncwarp();
#pragma unroll
          for (int r = 0; r < TB / 2; ++r) {
            obp[(2 * r) * 32 + lane] = o2[r].x;
            obp[(2 * r + 1) * 32 + lane] = o2[r].y;
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&omap, obp, x0 + 32 * q, out_row, so.img);
            tma_store_3d(&omap, obp + HB * 32, x0 + 32 * q, out_row + HB, so.img);
            bulk_commit();
          }
          obsel ^= 1;
        } else if (x0 + c < g.W) {
          float* dptr = dst + (long long)so.img * g.out_img + (long long)out_row * g.out_row + (x0 + c);
#pragma unroll
          for (int r = 0; r < TB / 2; ++r) {
            if (2 * r < nb) st_stream(dptr, o2[r].x);
            dptr += g.out_row;
            if (2 * r + 1 < nb) st_stream(dptr, o2[r].y);
            dptr += g.out_row;
          }
        }
      }
    }
    if (lane == 0) bulk_wait_read<0>();
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem_base_s, (uint32_t)tl.tmem_cols);
}

const void* sweep_ptr_rowtile(int k) {
  switch (k) {
    case 1: return (const void*)rowtile_kernel<1>;
    case 2: return (const void*)rowtile_kernel<2>;
    case 3: return (const void*)rowtile_kernel<3>;
    case 4: return (const void*)rowtile_kernel<4>;
    case 5: return (const void*)rowtile_kernel<5>;
    case 6: return (const void*)rowtile_kernel<6>;
    case 7: return (const void*)rowtile_kernel<7>;
    default: return (const void*)rowtile_kernel<8>;
  }
}

// the two-band uint8 fused sweep with 4-byte staging copies (sweep_kernels.cuh, A4), compiled here
// to balance the translation units
const void* sweep_ptr_fused5w(int k) { return fused5w_ptr_for<>(k); }
}  // namespace sb
