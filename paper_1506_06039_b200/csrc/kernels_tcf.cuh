// kernels_tcf.cuh -- the exact tensor-core coarse search (kernels_tc.cuh) with the operand
// preparation fused in: the search reads the LEVEL-0 frames itself.
//
// k_tc_coarse multiplies operand planes that k_tc_prep wrote to HBM (147 KB per C2 frame,
// written and read back) and loads them one 32-column strip at a time, the MMA warp
// stalling at every strip boundary for the copy.  Here builder warps produce the strips
// in shared memory straight from the raw frame rows (2^L x 2^L block sums -> 7-bit / byte
// parts, the same layout k_tc_prep writes), while the tensor cores work:
//
//   warp 0      MMA issuer (as k_tc_coarse), additionally waiting, per super-stage, for the
//               32-row chunks of the strip its pairs read (abuilt[c]) and committing, once
//               its pairs are past a chunk, the chunk's release (afree[c], tcgen05.commit:
//               arrives when those MMAs have completed)
//   warp 1      B producer: the B-tile ring from the per-template table (bulk copies)
//   warps 2..7  A builders: strip st+1's chunk c as soon as strip st's MMAs released it
//               (a single strip buffer: the build trails the MMAs by about one chunk);
//               frame energies on the way: total, edge rows, edge columns, the
//               squares of the four corner blocks (to global scratch)
//
// The epilogue first turns the energy partials into g_a for every lag (the corner tables'
// 2-D prefix = the DP of P:35) in the shared memory the strips used, then proceeds exactly
// as k_tc_coarse's: h -> N -> f -> argmin (S4).  Levels 0 and 1 (levels = 2 keeps
// k_tc_prep, which also writes the level-1 image).
//
// Measured (B200, C2, 1,184 frames alone): 0.46 us/frame against 0.33 for k_tc_prep +
// k_tc_coarse: the builders' global loads are latency-bound (1.15 TB/s, 166 registers per
// thread, one CTA per SM) and the tensor pipe waits (27 % active); an L2 prefetch two chunks
// ahead made it slower.  Opt-in (MOCO_TC_FUSED=1); bit-identical to the two-kernel search.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels_tc.cuh"

namespace moco {

constexpr int TCF_BUILDERS = 6;   // warps 2..7
constexpr int TCF_MAXCH = 16;     // 32-row chunks per strip (R <= 512)

struct TcfArgs {
  TcArgs t;                  // G and ga unused
  const uint16_t *frames;    // level-0 frames of the batch, row pitch n
  int64_t fstride;           // elements
  int n;                     // raw row pitch (elements)
  u64 *corner;               // [B][4][w][w] squares of the corner blocks (row/col 0 unused)
  int offE;                  // shared-memory offsets: energy partials, barriers
  int offBars;
  int nch;                   // 32-row chunks per strip = ceil(R / 32)
};

// shared-memory need of the epilogue (D1 staging, keys, g_a, corner tables)
__host__ __device__ inline int tcf_epi_bytes(const TcGeom &g) {
  const int nfr = g.GG * g.F;
  return g.GG * g.NT * 128 * 33 * 4 + g.GG * 128 * 16 + nfr * g.W * g.W * 8 + nfr * 4 * g.w * g.w * 8;
}

template <int L>
__global__ void __launch_bounds__(TC_THREADS, 1) k_tc_fused(TcfArgs fa) {
  const TcArgs &a = fa.t;
  const TcGeom &g = a.g;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int F = g.F, hw = g.hw, w = g.w, mc = g.mc, nc = g.nc, N = g.N, N1 = g.N1, NT = g.NT, GG = g.GG;
  const int NSS = g.nss, ICH = g.ICH, NCH = fa.nch, R = g.R;
  const int nfr = GG * F;
  unsigned char *As = smem;                                   // [GG] strips of 2 planes
  unsigned char *Bring = As + GG * g.stripB;                  // [NSS][ICH][N*32]
  u64 *etot = reinterpret_cast<u64 *>(smem + fa.offE);        // [nfr]
  u64 *erow = etot + nfr;                                     // [nfr][2 hw]: top rows, bottom rows (from the bottom)
  u64 *ecol = erow + nfr * 2 * hw;                            // [nfr][2 hw]: left cols, right cols (from the right)
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + fa.offBars);
  uint64_t *full = bars, *empty = bars + NSS, *abuilt = bars + 2 * NSS, *afree = abuilt + NCH;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(afree + NCH);
  const int grp0 = blockIdx.x * GG;
  const int ngroups = (a.B + F - 1) / F;
  const int gcount = min(GG, ngroups - grp0);
  const int per_strip = g.npairs / ICH;
  const int nsuper = g.nstrips * per_strip;
  const int64_t fi0 = (int64_t)grp0 * F;

  if (warp == 0) tmem_alloc(tmem_holder, g.tmem_cols);
  for (int k = tid; k < nfr * (1 + 4 * hw); k += TC_THREADS) etot[k] = 0;
  if (tid == 0) {
    for (int s = 0; s < NSS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int c = 0; c < NCH; ++c) {
      mbar_init(&abuilt[c], TCF_BUILDERS);
      mbar_init(&afree[c], 1);
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = *tmem_holder;

  if (warp == 0) {
    // ---------------- MMA issuer
    const uint32_t idesc = idesc_i8(128, N);
    const uint64_t bd0 = umma_desc(smem_u32(Bring), 128, 256);
    const uint64_t ad0 = umma_desc(smem_u32(As), g.planeB, 128);
    const uint32_t blo0 = (uint32_t)bd0, bhi = (uint32_t)(bd0 >> 32);
    const uint32_t alo0 = (uint32_t)ad0, ahi = (uint32_t)(ad0 >> 32);
    const uint32_t rowstep = (32u * F) >> 4;
    const uint32_t tilestep = (uint32_t)(N * 32) >> 4;
    const uint32_t sstep = (uint32_t)ICH * tilestep;
    const int ntg = gcount * NT;
    uint32_t aoff[4], tcol[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gg = j / NT, k = j % NT;
      aoff[j] = (uint32_t)(gg * g.stripB >> 4) + (uint32_t)(k * g.ST) * rowstep;
      tcol[j] = taddr + (uint32_t)(j * g.TS);
    }
    const int span = NT * g.ST;   // plane rows one pair's A tiles cover
    int ss = 0, round = 0;
    for (int st = 0; st < g.nstrips; ++st) {
      int nbuilt = 0, nfreed = 0;
      uint32_t arow = alo0;
      for (int u = 0; u < per_strip; ++u) {
        const int i0 = u * ICH;
        const int need = min(NCH, (2 * (i0 + ICH - 1) + span - 1) / 32 + 1);
        while (nbuilt < need) {
          mbar_wait(&abuilt[nbuilt], st & 1);
          ++nbuilt;
        }
        mbar_wait(&full[ss], round & 1);
        tc_fence_after();
        uint32_t blo = blo0 + (uint32_t)ss * sstep;
        for (int q = 0; q < ICH; ++q, blo += tilestep, arow += 2 * rowstep) {
          const uint32_t acc = (st | u | q) != 0 ? 1u : 0u;
          if (ntg == 4) {
            mma_i8_x4_elect(tcol[0], tcol[1], tcol[2], tcol[3], arow + aoff[0], arow + aoff[1], arow + aoff[2],
                            arow + aoff[3], ahi, blo, bhi, idesc, acc);
          } else if (ntg == 2) {
            mma_i8_x2_elect(tcol[0], tcol[1], arow + aoff[0], arow + aoff[1], ahi, blo, bhi, idesc, acc);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < ntg) mma_i8_elect(tcol[j], arow + aoff[j], ahi, blo, bhi, idesc, acc);
          }
        }
        mma_commit_elect(&empty[ss]);
        // chunks wholly below the next pair's first row are released once these MMAs are done
        const int freeable = u + 1 < per_strip ? min(NCH, (2 * (i0 + ICH)) / 32) : NCH;
        // every chunk's phase of this strip is consumed before it is released (rows past the
        // last pair's tiles are built but never read)
        while (nbuilt < freeable) {
          mbar_wait(&abuilt[nbuilt], st & 1);
          ++nbuilt;
        }
        while (nfreed < freeable) {
          mma_commit_elect(&afree[nfreed]);
          ++nfreed;
        }
        __syncwarp();
        if (++ss == NSS) { ss = 0; ++round; }
      }
    }
  } else if (warp == 1) {
    // ---------------- B producer: the ring of B tiles, one bulk copy per super-stage
    const uint32_t bytes = (uint32_t)(ICH * N * 32);
    int st = 0, i0 = 0;
    for (int u = 0; u < nsuper; ++u) {
      const int slot = u % NSS, rnd = u / NSS;
      if (rnd > 0) mbar_wait(&empty[slot], (rnd - 1) & 1);
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[slot], bytes);
        bulk_g2s(Bring + slot * ICH * N * 32, a.Btab + ((int64_t)st * g.npairs + i0) * (N * 32), bytes, &full[slot]);
      }
      __syncwarp();
      i0 += ICH;
      if (i0 >= g.npairs) { i0 = 0; ++st; }
    }
  } else {
    // ---------------- A builders.  Each thread keeps one frame fl (tpf = 192 / nfr threads
    // per frame) and one 8-column chunk cc4 of the strip (tpf is a multiple of 4), walking
    // rows; task = (plane row, cc4), 4 lane-consecutive tasks read 4 x 16 raw columns of one
    // raw row pair.  Loads of 4 tasks are issued before any is used.  Energies accumulate
    // in registers (total, edge columns) and reach shared memory once at the end; edge-row
    // sums (lane-quad reduced) and corner squares as they occur.
    const int bt = (warp - 2) * 32 + lane;
    const uint32_t pm = g.sb == 7 ? 0x007F007Fu : 0x00FF00FFu, sb = (uint32_t)g.sb;
    const int tpf = (TCF_BUILDERS * 32) / nfr;
    const int fl = bt / tpf, pt0 = bt - fl * tpf;
    const int cc4 = pt0 & 3;
    const int gg = fl / F, f = fl - gg * F;
    const int64_t fi = fi0 + fl;
    const bool frame_live = gg < gcount && fi < a.B;
    const uint16_t *Fr = fa.frames + (frame_live ? fi : 0) * fa.fstride;
    u64 rtot = 0, eL[8], eR[8];
#pragma unroll
    for (int x = 0; x < 8; ++x) eL[x] = eR[x] = 0;
    constexpr int KB = 4;   // tasks in flight per thread
    for (int st = 0; st < g.nstrips; ++st) {
      const bool edgeL = 32 * st < hw, edgeR = 32 * st + 32 > nc - hw;
      const int ccg = 4 * st + cc4;   // coarse 8-column chunk of the row
      for (int c = 0; c < NCH; ++c) {
        if (st > 0) mbar_wait(&afree[c], (st - 1) & 1);
        const int pr0 = 32 * c, nrow = min(32, R - pr0);
        for (int pb = pt0; pb < 128; pb += KB * tpf) {   // 32 rows x 4 chunks per frame
          uint32_t P[KB][4];
          int prs[KB];
          bool inr[KB], live[KB];
#pragma unroll
          for (int q = 0; q < KB; ++q) {
            const int pt = pb + q * tpf, prl = pt >> 2;
            prs[q] = pr0 + prl;
            const int cr = prs[q] - hw;
            inr[q] = pt < 128 && prl < nrow;
            live[q] = inr[q] && frame_live && cr >= 0 && cr < mc;
            P[q][0] = P[q][1] = P[q][2] = P[q][3] = 0;
            if (live[q]) coarse8<L>(Fr + (int64_t)(cr << L) * fa.n + ((ccg * 8) << L), fa.n, P[q]);
          }
#pragma unroll
          for (int q = 0; q < KB; ++q) {
            const int pr = prs[q], cr = pr - hw;
            if (inr[q]) {
              const uint32_t h0 = (P[q][0] >> sb) & pm, h1 = (P[q][1] >> sb) & pm;
              const uint32_t h2 = (P[q][2] >> sb) & pm, h3 = (P[q][3] >> sb) & pm;
              const uint2 hi = make_uint2(__byte_perm(h0, h1, 0x6420), __byte_perm(h2, h3, 0x6420));
              const uint2 lo = make_uint2(__byte_perm(P[q][0] & pm, P[q][1] & pm, 0x6420),
                                          __byte_perm(P[q][2] & pm, P[q][3] & pm, 0x6420));
              unsigned char *dst = As + gg * g.stripB + ((cc4 >> 1) * R + pr) * (32 * F) + f * 32 + (cc4 & 1) * 8;
              *reinterpret_cast<uint2 *>(dst) = hi;
              *reinterpret_cast<uint2 *>(dst + 16) = lo;
            }
            uint32_t v[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) { v[2 * k] = P[q][k] & 0xffffu; v[2 * k + 1] = P[q][k] >> 16; }
            u64 rs = 0;
#pragma unroll
            for (int x = 0; x < 8; ++x) rs += (u64)(v[x] * v[x]);   // each < 2^32
            rtot += rs;
            // edge rows: the row's sum over the lane quad (the strip's 4 chunks of the row;
            // all four lanes have the same q, row and liveness)
            u64 rq = rs + __shfl_xor_sync(0xffffffffu, rs, 1);   // warp-uniform: every lane shuffles
            rq += __shfl_xor_sync(0xffffffffu, rq, 2);
            if (live[q] && cc4 == 0 && (cr < hw || cr >= mc - hw)) {
              if (cr < hw) atomicAdd(&erow[fl * 2 * hw + cr], rq);
              if (cr >= mc - hw) atomicAdd(&erow[fl * 2 * hw + hw + (mc - 1 - cr)], rq);
            }
            if ((edgeL || edgeR) && live[q]) {
#pragma unroll
              for (int x = 0; x < 8; ++x) {
                const int j = 8 * ccg + x;
                const bool lf = j < hw, rt = j >= nc - hw;
                if (!(lf || rt)) continue;
                const u64 sq = (u64)(v[x] * v[x]);
                if (lf) eL[x] += sq;
                if (rt) eR[x] += sq;
                if (cr < hw || cr >= mc - hw) {   // corner squares (the tables of)
                  u64 *cb = fa.corner + fi * 4 * w * w;
                  if (cr < hw && lf) cb[(0 * w + cr + 1) * w + j + 1] = sq;
                  if (cr < hw && rt) cb[(1 * w + cr + 1) * w + nc - j] = sq;
                  if (cr >= mc - hw && lf) cb[(2 * w + mc - cr) * w + j + 1] = sq;
                  if (cr >= mc - hw && rt) cb[(3 * w + mc - cr) * w + nc - j] = sq;
                }
              }
            }
          }
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&abuilt[c]);
      }
    }
    // flush the register-held energies (the edge chunks of the thread's column: first / last strip)
    if (frame_live) {
      if (rtot) atomicAdd(&etot[fl], rtot);
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const int jl = 8 * cc4 + x, jr = 8 * (4 * (g.nstrips - 1) + cc4) + x;
        if (eL[x] && jl < hw) atomicAdd(&ecol[fl * 2 * hw + jl], eL[x]);
        if (eR[x] && jr >= nc - hw) atomicAdd(&ecol[fl * 2 * hw + hw + (nc - 1 - jr)], eR[x]);
      }
    }
  }
  // all MMAs done -> accumulators final
  {
    const int last = nsuper - 1;
    mbar_wait(&empty[last % NSS], (last / NSS) & 1);
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // ---- epilogue part 1: g_a for every lag of every frame (the DP of P:35 in each corner)
  const int W = g.W, CS = w * w;
  uint32_t *D1s = reinterpret_cast<uint32_t *>(smem);
  Key *keys = reinterpret_cast<Key *>(smem + GG * NT * 128 * 33 * 4);
  u64 *gas = reinterpret_cast<u64 *>(keys + GG * 128);
  u64 *cor = gas + nfr * W * W;   // [nfr][4][w][w]
  {
    for (int k = tid; k < nfr * 4 * CS; k += TC_THREADS) {
      const int fl = k / (4 * CS), r = k - fl * 4 * CS;
      const int pp = (r % CS) / w, qq = r % w;
      const bool ok = fl < gcount * F && fi0 + fl < a.B && pp > 0 && qq > 0;
      cor[k] = ok ? fa.corner[(fi0 + fl) * 4 * CS + r] : 0;
    }
    __syncthreads();
    for (int k = tid; k < nfr * 4; k += TC_THREADS) {   // strips: 1-D prefix sums
      u64 *e = (k & 2) ? ecol : erow;
      u64 *p = e + (k >> 2) * 2 * hw + (k & 1) * hw;
      for (int q = 1; q < hw; ++q) p[q] += p[q - 1];
    }
    for (int k = tid; k < nfr * 4 * w; k += TC_THREADS) {   // corners: 2-D prefix, rows
      u64 *c = cor + (k / w) * CS + (k % w) * w;
      for (int q = 1; q < w; ++q) c[q] += c[q - 1];
    }
    __syncthreads();
    for (int k = tid; k < nfr * 4 * w; k += TC_THREADS) {   // then columns
      u64 *c = cor + (k / w) * CS + (k % w);
      for (int p = 1; p < w; ++p) c[p * w] += c[(p - 1) * w];
    }
    __syncthreads();
    for (int k = tid; k < nfr * W * W; k += TC_THREADS) {
      const int fl = k / (W * W), lag = k - fl * W * W;
      const int s = lag / W - hw, t = lag % W - hw;
      const u64 *re = erow + fl * 2 * hw, *ce = ecol + fl * 2 * hw;
      const u64 rex = s > 0 ? re[s - 1] : (s < 0 ? re[hw + (-s) - 1] : 0);
      const u64 cex = t > 0 ? ce[t - 1] : (t < 0 ? ce[hw + (-t) - 1] : 0);
      u64 corner = 0;
      if (s != 0 && t != 0) {
        const int quad = (s < 0 ? 2 : 0) | (t < 0 ? 1 : 0);
        corner = cor[(fl * 4 + quad) * CS + abs(s) * w + abs(t)];
      }
      gas[k] = etot[fl] - rex - cex + corner;
    }
    __syncthreads();
  }

  // ---- epilogue part 2: as k_tc_coarse: h -> N -> f -> argmin (S4)
  const int m = (warp & 3) * 32 + lane;
  const int sl = m / (2 * F), rho = m % (2 * F);
  const int f = rho >> 1, pa = rho & 1;
  Key best[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) best[q] = Key{~0ull, ~0u};
  for (int c = 0; c < g.Wt; c += 16) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int gg = (warp >> 2) + 2 * q;
      if (gg >= GG) continue;
      for (int k = 0; k < NT; ++k) {
        uint32_t yh[16], yl[16];
        const uint32_t tbase = taddr + ((uint32_t)((warp & 3) * 32) << 16) + (gg * NT + k) * g.TS + N1;
        tmem_ld16(tbase + c, yh);
        tmem_ld16(tbase + g.Wt + c, yl);
        tmem_wait_ld();
        uint32_t *dst = D1s + ((gg * NT + k) * 128 + m) * 33;
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) { dst[qq] = yh[qq]; dst[16 + qq] = yl[qq]; }
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int gg = (warp >> 2) + 2 * q;
      if (gg >= GG) continue;
      const int64_t fi = (int64_t)(grp0 + gg) * F + f;
      Key bk = best[q];
      for (int k = 0; k < NT; ++k) {
        const int s = -hw + k * g.ST + sl;
        const bool valid = gg < gcount && s <= hw && fi < a.B;
        const int mp = sl + 1 < g.ST ? m + 2 * F : m + 2 * F - 128;
        const int kp = sl + 1 < g.ST ? k : k + 1;
        const bool haveP = kp < NT;
        uint32_t xh[16], xl[16];
        const uint32_t tbase = taddr + ((uint32_t)((warp & 3) * 32) << 16) + (gg * NT + k) * g.TS;
        tmem_ld16(tbase + c, xh);
        tmem_ld16(tbase + g.Wt + c, xl);
        tmem_wait_ld();
        const uint32_t *src = D1s + ((gg * NT + (haveP ? kp : 0)) * 128 + (haveP ? mp : 0)) * 33;
        if (haveP) {
#pragma unroll
          for (int qq = 0; qq < 16; ++qq) { xh[qq] += src[qq]; xl[qq] += src[16 + qq]; }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t mh = pa ? xh[j + 8] : xh[j], ml = pa ? xl[j + 8] : xl[j];
          const uint32_t ph = __shfl_xor_sync(0xffffffffu, pa ? xh[j] : xh[j + 8], 1);
          const uint32_t pl = __shfl_xor_sync(0xffffffffu, pa ? xl[j] : xl[j + 8], 1);
          const int ti = c + j + (pa ? 8 : 0);
          if (!valid || ti >= W) continue;
          const int sbits = g.sb;
          const u64 h = pa == 0 ? ((u64)mh << (2 * sbits)) + (((u64)ml + (u64)ph) << sbits) + (u64)pl
                                : ((u64)ph << (2 * sbits)) + (((u64)pl + (u64)mh) << sbits) + (u64)ml;
          const int lag = (s + hw) * W + ti;
          const u64 Nn = gas[(fi - fi0) * W * W + lag] + a.gb[lag] - 2 * h;
          const int t = ti - hw;
          const double area = (double)((mc - abs(s)) * (nc - abs(t)));
          const double fv = (double)Nn / (a.scale * area);
          if (a.grid_out) a.grid_out[fi * W * W + lag] = fv;
          const Key kk{(u64)__double_as_longlong(fv), (unsigned)lag};
          if (key_less(kk, bk)) bk = kk;
        }
      }
      best[q] = bk;
    }
    __syncthreads();
  }
  tc_fence_before();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int gg = (warp >> 2) + 2 * q;
    if (gg < GG) keys[gg * 128 + m] = best[q];
  }
  __syncthreads();
  if (tid < GG * F) {
    const int gg = tid / F, ff = tid % F;
    const int fo = (grp0 + gg) * F + ff;
    if (gg < gcount && fo < a.B && a.shift_out) {
      Key b{~0ull, ~0u};
      for (int q = 2 * ff; q < 128; q += 2 * F) {
        if (key_less(keys[gg * 128 + q], b)) b = keys[gg * 128 + q];
        if (key_less(keys[gg * 128 + q + 1], b)) b = keys[gg * 128 + q + 1];
      }
      const int s = (int)(b.idx / W) - hw, t = (int)(b.idx % W) - hw;
      a.shift_out[2 * fo] = s;
      a.shift_out[2 * fo + 1] = t;
      if (a.f_out) a.f_out[fo] = __longlong_as_double((long long)b.f);
      if (a.flags) a.flags[fo] = (abs(s) == hw || abs(t) == hw) ? 1 : 0;
    }
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc(taddr, g.tmem_cols);
}

// Shared-memory layout of k_tc_fused for geometry g; false if it does not fit.
inline bool tcf_layout(const TcGeom &g, int *smem, int *offE, int *offBars, int *nch) {
  const int main = g.GG * g.stripB + g.nss * g.ICH * g.N * 32;
  const int epi = tcf_epi_bytes(g);
  const int A = (std::max(main, epi) + 15) / 16 * 16;
  const int nfr = g.GG * g.F;
  const int E = nfr * (1 + 4 * g.hw) * 8;
  *nch = (g.R + 31) / 32;
  if (*nch > TCF_MAXCH) return false;
  *offE = A;
  *offBars = A + (E + 15) / 16 * 16;
  *smem = 1024 + *offBars + (2 * g.nss + 2 * *nch) * 8 + 16;
  return *smem <= 227 * 1024;
}

}  // namespace moco
