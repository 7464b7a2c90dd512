// sweep_wide.cu - one-launch fused sweep for float32 sources whose radii are past the
// reach of fused_kernel (C5: p_max 257), so the row-filtered values never go to HBM.
//
// Reference: separable_filter_2d (filtering.py:76-104) = _filter_rows (filtering.py:48-64)
// over the rows, then over the columns of the result, replicate boundaries
// (filtering.py:10-13).  The arithmetic is the fused sweep's:
// exact int32 row prefixes in the input quantum, row values rounded to the mid quantum,
// exact int32 column prefixes, box sums as prefix differences.
//
// Persistent grid, one CTA per SM, over (row chunk, 128-column strip) units (WorkIter).
// 16 warps, four roles, mbarrier hand-offs only:
//  * staging: band gb lives in slot gb mod FP; one bulk copy (cp.async.bulk) per clamped
//    row stages columns [x0 - xoff, x0 - xoff + L) of its 16 rows, issued by the row warps
//    as soon as they have read the slot's previous band (FP bands in flight);
//  * producers (warps 12..15, rows 4pw .. 4pw+3 of every band): border columns replicated
//    in place, rows prefix-scanned IN PLACE (f32 -> int32 fixed point), so a slot is one
//    16 x LSW word buffer;
//  * row warps (0..3; thread c = strip column c = TMEM lane c): the K box sums of every
//    row of the band from the slot, weighted, rounded to the mid quantum and accumulated
//    into the column prefix C, which is appended to a 496-row ring in tensor memory (the
//    cols2_kernel ring: trail windows older than the ring come from shared-memory copies
//    the row warps take out of TMEM just before eviction);
//  * output groups (warps 4..11, WCG groups of four): output band j = g (mod WCG) is
//    sum_i w_i (C(y+p_i) - C(y-p_i-1)) from two TMEM windows per box, staged and written
//    by TMA tensor stores.
#include "sweep_kernels.cuh"

namespace sb {


// In-place prefix scan of rows r0 .. r0+3 (those < n) of a slot: float32 elements ->
// inclusive int32 prefixes in the input quantum (to_fixed).  Lane (rr, cq) = (lane & 3,
// lane >> 2) takes chunk cg + cq of row r0 + rr, so each 8-lane phase of the 128-bit
// accesses touches 4 rows x 2 chunks = 8 distinct bank groups (LSW*4 = 16 mod 128).  A lane
// reads its whole 16-element chunk before writing it back and no other lane touches the
// chunk, so the scan may overwrite the staged values.
template <int LSW>
__device__ __forceinline__ void scan4_inplace(int* P, const Taps& t, int L, int r0, int n, RangeAcc& bad) {
  const int lane = threadIdx.x & 31;
  const int rr = lane & 3, cq = lane >> 2;
  const int nchunk = L / CH;
  const int r = r0 + rr;
  int running = 0;
  for (int cg = 0; cg < nchunk; cg += 8) {
    const int chunk = cg + cq;
    const bool live = (r < n) && (chunk < nchunk);
    int v[CH];
    int tot = 0;
    int4* p4 = (int4*)(P + r * LSW + chunk * CH);
    if (live) {
      float e[CH];
#pragma unroll
      for (int m = 0; m < CH / 4; ++m) *(int4*)(e + 4 * m) = p4[m];
#pragma unroll
      for (int m = 0; m < CH; ++m) {
        tot += to_fixed<float>(e[m], t, bad);
        v[m] = tot;
      }
    }
    int inc = tot;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const int carry = running + inc - tot;
    if (live) {
#pragma unroll
      for (int m = 0; m < CH / 4; ++m)
        p4[m] = make_int4(v[4 * m] + carry, v[4 * m + 1] + carry, v[4 * m + 2] + carry, v[4 * m + 3] + carry);
    }
    running += __shfl_sync(0xffffffffu, inc, rr + 28);
  }
}

// Stage band (segment s, band pb) into slot P: one bulk copy per clamped row of the 16-byte
// part of columns [max(xb, 0), min(xb + L, W)); the copies complete on `bar`, which the
// calling lane 0 arms with the byte count first (0 bytes when the rows are not 16-byte
// aligned: the producers then copy the elements).  Issued by one warp.
__device__ __forceinline__ void issue_band(int* P, const float* __restrict__ src, const Geometry& g, const Tiling& tl,
                                           const WorkIter& s, int pb, int lsw, uint64_t* bar) {
  const int lane = threadIdx.x & 31;
  const int xb = s.strip * WS - tl.xoff;
  const int lo = max(xb, 0), hi = min(xb + tl.L, g.W);
  const int hi4 = g.aligned16 ? lo + ((hi - lo) & ~3) : lo;
  const int n = min(HB, s.count - pb * HB);
  const int v0 = s.a - 1 - s.pmax + pb * HB;
  fence_proxy_async();  // the slot's generic-proxy accesses (scan, row values) precede the copy
  __syncwarp();
  if (lane == 0) mbar_expect_tx(bar, (uint32_t)(n * (hi4 - lo) * 4));
  __syncwarp();
  if (lane < n && hi4 > lo) {
    const int v = min(max(v0 + lane, 0), g.H - 1);
    bulk_g2s(P + lane * lsw + (lo - xb), src + (long long)s.img * g.in_img + (long long)v * g.in_row + lo,
             (uint32_t)((hi4 - lo) * 4), bar);
  }
}

template <int K, int LSW>
__global__ void __launch_bounds__(WTHREADS, 1)
    fusedw_kernel(const float* __restrict__ src, float* __restrict__ dst, Geometry g, Taps t, Tiling tl, int* status,
                  const __grid_constant__ CUtensorMap omap) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t tmem_base_s;
  __shared__ __align__(8) uint64_t done[C2DONE], sfull[WPROD], pfull[WPROD];
  __shared__ uint32_t ring_cnt[4];  // ring bands written, per lane quadrant (monotonic: cannot alias)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3;  // TMEM lane quadrant: columns 32q .. 32q+31
  const int c = 32 * q + lane;
  const int wh = g.oy1 - g.oy0;
  const long long total = (long long)g.nimg * wh;  // tall-image rows every strip outputs
  const int D = tl.D, NB = D / HB, DS = tl.ds, FP = tl.pf;
  unsigned char* abase = smem + (((smem_u32(smem) + 127u) & ~127u) - smem_u32(smem));  // 128-byte aligned
  int* slots = (int*)abase;                         // [FP][HB][LSW] staged rows -> row prefixes (in place)
  int* dring = slots + FP * HB * LSW;               // [DS + 1][HB][WS] copies of old ring bands (+ mirror)
  float* obuf = (float*)(abase + tl.obuf_off);      // [4 * WCG][2][HB][32] output boxes (TMA stores)
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) ring_cnt[i] = 0;
    for (int i = 0; i < C2DONE; ++i) mbar_init(&done[i], 32 * 4);
    for (int i = 0; i < WPROD; ++i) {
      mbar_init(&sfull[i], 1);       // the issuing lane's expect_tx arrive + the bulk-copy bytes
      mbar_init(&pfull[i], 32 * WPROD);  // every producer thread after its rows' scan
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&tmem_base_s, (uint32_t)tl.tmem_cols);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tlane = tmem_base_s + ((uint32_t)q << 21);

  if (warp >= 4 + 4 * WCG) {
    // ------------------------------------------------ producers
    // every producer warp takes rows 4pw .. 4pw+3 of every band: element copies the bulk
    // copies left out (unaligned rows, the tail past the last 16-byte boundary), border
    // replication, in-place scan; then one arrive per thread on the slot's pfull
    const int pw = warp - (4 + 4 * WCG);
    RangeAcc bad;
    WorkIter s;
    s.init(total, tl.rows_per_item, tl.nstrips, wh, g.oy0, t.pmax);
    uint32_t j = 0;
    for (; s.valid; s.next()) {
      const int xb = s.strip * WS - tl.xoff;
      const float* src_img = src + (long long)s.img * g.in_img;
      const int lo = max(xb, 0), hi = min(xb + tl.L, g.W);
      const int hi4 = g.aligned16 ? lo + ((hi - lo) & ~3) : lo;
      const bool edge = (xb < 0) || (xb + tl.L > g.W);
      const int r0 = 4 * pw;
      for (int pb = 0; pb < s.nbands; ++pb, ++j) {
        const int n = min(HB, s.count - pb * HB);
        const int fs = (int)(j % (uint32_t)FP);
        int* P = slots + fs * (HB * LSW);
        mbar_wait(&sfull[fs], (j / (uint32_t)FP) & 1);
        if (r0 < n) {
          const int v0 = s.a - 1 - t.pmax + pb * HB;
          if (hi4 < hi) {
            for (int r = r0; r < min(r0 + 4, n); ++r) {
              const float* grow = src_img + (long long)min(max(v0 + r, 0), g.H - 1) * g.in_row;
              for (int x = hi4 + lane; x < hi; x += 32) ((float*)P)[r * LSW + (x - xb)] = grow[x];
            }
            __syncwarp();
          }
          if (edge) {
            // replicate the border columns (filtering.py:10-13)
            float* Pf = (float*)P;
            const int left = lo - xb, right0 = hi - xb;
            for (int r = r0; r < min(r0 + 4, n); ++r) {
              const float l0 = Pf[r * LSW + left], rv = Pf[r * LSW + right0 - 1];
              for (int x = lane; x < left; x += 32) Pf[r * LSW + x] = l0;
              for (int x = right0 + lane; x < tl.L; x += 32) Pf[r * LSW + x] = rv;
            }
            __syncwarp();
          }
          scan4_inplace<LSW>(P, t, tl.L, r0, n, bad);
        }
        mbar_arrive(&pfull[fs]);
      }
    }
    report_status(status, bad, t);
  } else if (warp < 4) {
    // ------------------------------------------------ row warps: row values, column prefix, TMEM ring
    WorkIter sc, so;  // ring bands / the output bands whose completion gates the ring
    sc.init(total, tl.rows_per_item, tl.nstrips, wh, g.oy0, t.pmax);
    so.init(total, tl.rows_per_item, tl.nstrips, wh, g.oy0, t.pmax);
    uint32_t v = 0;  // global band (ring band) index
    uint32_t onum = 0;
    int oob = 0;  // next output band to observe: index onum, band oob of segment so
    int slot = 0;
    int cslot = tl.copy_e % NB, dslot = 0;  // ring slot (v + copy_e) % NB and copy slot of the next band copy
    const int base = c + tl.xoff;
    // bands are staged FP ahead: the row warps re-arm a slot as soon as all four have read it
    WorkIter ls;  // next band to stage: band lpb of segment ls, global index jl
    ls.init(total, tl.rows_per_item, tl.nstrips, wh, g.oy0, t.pmax);
    int lpb = 0;
    uint32_t jl = 0;
    auto stage_next = [&]() {
      if (!ls.valid) return;
      const int fs = (int)(jl % (uint32_t)FP);
      if (warp == 0) issue_band(slots + fs * (HB * LSW), src, g, tl, ls, lpb, LSW, &sfull[fs]);
      ++jl;
      if (++lpb == ls.nbands) {
        ls.next();
        lpb = 0;
      }
    };
    for (int i = 0; i < FP; ++i) stage_next();
    for (; sc.valid; sc.next()) {
      int cprefix = 0;
      const int npairs = (sc.nbands + 1) / 2;
      for (int pp = 0; pp < npairs; ++pp) {
        const int nbp = min(2, sc.nbands - 2 * pp);  // bands in this pair
        // every output band reading ring bands v+d - NB from TMEM is done
        while (so.valid && (long long)(so.gb0 + (uint32_t)oob) + tl.lag <= (long long)v + nbp - 1) {
          mbar_wait(&done[onum % C2DONE], (onum / C2DONE) & 1);
          ++onum;
          if (++oob == (so.b - so.a + HB - 1) / HB) {
            so.next();
            oob = 0;
          }
        }
        uint32_t cv[2][HB];
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          if (d >= nbp) break;
          const uint32_t gb = v + (uint32_t)d;
          const int fs = (int)(gb % (uint32_t)FP);
          const int* Ps = slots + fs * (HB * LSW);
          mbar_wait(&pfull[fs], (gb / (uint32_t)FP) & 1);
          float acc[HB];
#pragma unroll
          for (int r = 0; r < HB; ++r) acc[r] = 0.0f;
#pragma unroll
          for (int i = 0; i < K; ++i) {
            const int* pl = Ps + base + t.p[i];
            const int* pt = Ps + base - t.p[i] - 1;
            const float wi = t.w_row[i];
#pragma unroll
            for (int r = 0; r < HB; ++r) acc[r] = fmaf(wi, i2f_fast((uint32_t)(pl[r * LSW] - pt[r * LSW])), acc[r]);
          }
          named_bar_sync(1, 128);  // all row warps are done with the slot: stage band gb + FP into it
          stage_next();
          // round to the mid quantum and accumulate the column prefix (exact int32, wraps);
          // odd entries chain by 3-input adds, even entries hang off them
          int odd = cprefix;
#pragma unroll
          for (int r = 0; r < HB; r += 2) {
            const int e0 = __float_as_int(__fadd_rn(acc[r], kMagic)) - kMagicBits;  // _rn: never contracted
            const int e1 = __float_as_int(__fadd_rn(acc[r + 1], kMagic)) - kMagicBits;
            cv[d][r] = (uint32_t)(odd + e0);
            odd = odd + e0 + e1;
            cv[d][r + 1] = (uint32_t)odd;
          }
          cprefix = odd;
        }
        const int slot0 = slot;
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          if (d >= nbp) break;
          SB_ASSERT(slot * HB + HB <= D);
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
          // readers wait for band v + 1 or later; see fusedw_tiling)
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
              SB_ASSERT(dslot >= 0 && dslot < DS);
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
    const int grp = warp / 4 - 1;
    const int ow = warp - 4;  // output warp 0 .. 4*WCG-1 (staging buffers)
    uint32_t onum = 0;
    int obsel = 0;
    WorkIter so;
    so.init(total, tl.rows_per_item, tl.nstrips, wh, g.oy0, t.pmax);
    for (; so.valid; so.next()) {
      const int x0 = so.strip * WS;
      const int nout = (so.b - so.a + HB - 1) / HB;
      for (int ob = 0; ob < nout; ++ob, ++onum) {
        if ((int)(onum % WCG) != grp) continue;
        const int out_next = so.a + ob * HB;
        const int nb = min(HB, so.b - out_next);
        const uint32_t j = so.gb0 + (uint32_t)ob;  // ring band of the band's deepest trail row
        const uint32_t need = so.gb0 + (uint32_t)((ob * HB + nb + 2 * t.pmax) / HB);
        // the output groups mostly wait for the row warps: back off instead of spinning
        wait_above(&ring_cnt[q], need, true);
        tmem_fence_after();
        const int rbase = (int)(j % (uint32_t)NB) * HB;  // ring position of virtual row 16*ob
        float2 o2[HB / 2];
#pragma unroll
        for (int i0 = 0; i0 < K; i0 += 2) {
          uint32_t lvp[2][HB], tvp[2][HB];
#pragma unroll
          for (int d2 = 0; d2 < 2; ++d2) {
            const int i = i0 + d2;
            if (i >= K) break;
            int l = rbase + t.pmax + 1 + t.p[i];
            l = l >= D ? l - D : l;
            l = l >= D ? l - D : l;
            SB_ASSERT(l >= 0 && l < D);
            tmem_ld16(tlane + (uint32_t)l, lvp[d2]);
            if (!((tl.deepmask >> i) & 1)) {
              int tr = rbase + t.pmax - t.p[i];
              tr = tr >= D ? tr - D : tr;
              tmem_ld16(tlane + (uint32_t)tr, tvp[d2]);
            }
          }
          tmem_wait_ld();
#pragma unroll
          for (int d2 = 0; d2 < 2; ++d2) {
            const int i = i0 + d2;
            if (i >= K) break;
            uint32_t(&lv)[HB] = lvp[d2];
            uint32_t(&tv)[HB] = tvp[d2];
            if ((tl.deepmask >> i) & 1) {
              // virtual rows 16*ob + pmax - p_i .. +15 from the band copies (band j + off/16 on)
              const int off = t.pmax - t.p[i];
              const uint32_t u0 = j + (uint32_t)(off / HB);
              const int r0 = off % HB;
              const int s0 = (int)(u0 % (uint32_t)DS);
              SB_ASSERT(DS > 0 && s0 < DS);
              const int* p0 = dring + (s0 * HB + r0) * WS + c;
#pragma unroll
              for (int r = 0; r < HB; ++r) tv[r] = (uint32_t)p0[r * WS];
            }
            const float2 w2 = make_float2(t.w_col[i], t.w_col[i]);
#pragma unroll
            for (int r = 0; r < HB / 2; ++r) {
              const float2 dd =
                  make_float2(i2f_fast(lv[2 * r] - tv[2 * r]), i2f_fast(lv[2 * r + 1] - tv[2 * r + 1]));
              o2[r] = i == 0 ? __fmul2_rn(w2, dd) : __ffma2_rn(w2, dd, o2[r]);
            }
          }
        }
        tmem_fence_before();
        mbar_arrive(&done[onum % C2DONE]);
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
          float* dptr = dst + (long long)so.img * g.out_img + (long long)(out_next - g.oy0) * g.out_row + (x0 + c);
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
    if (lane == 0) bulk_wait_read<0>();
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem_base_s, (uint32_t)tl.tmem_cols);
}

template <int LSW>
const void* fusedw_ptr_for(int k) {
  switch (k) {
    case 1: return (const void*)fusedw_kernel<1, LSW>;
    case 2: return (const void*)fusedw_kernel<2, LSW>;
    case 3: return (const void*)fusedw_kernel<3, LSW>;
    case 4: return (const void*)fusedw_kernel<4, LSW>;
    case 5: return (const void*)fusedw_kernel<5, LSW>;
    case 6: return (const void*)fusedw_kernel<6, LSW>;
    case 7: return (const void*)fusedw_kernel<7, LSW>;
    default: return (const void*)fusedw_kernel<8, LSW>;
  }
}

const void* sweep_ptr_fusedw(int k, int lsw) {
  if (lsw == WLS[0]) return fusedw_ptr_for<WLS[0]>(k);
  if (lsw == WLS[1]) return fusedw_ptr_for<WLS[1]>(k);
  return fusedw_ptr_for<WLS[2]>(k);
}

}  // namespace sb
