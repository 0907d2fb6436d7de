// kernels_rtc.cuh -- S5 refine sums on the 5th-gen tensor cores (tcgen05, kind::i8).
//
// The +-1 refinement at level l needs, per frame f and each of
// the nine candidates (u, v) around the doubled coarse shift (S, T) = 2 s_{l+1},
//   H_f(u,v)  = sum_{i<ml, j<nl} a_f[i+S+u][j+T+v] b[i][j]        (cross term)
//   GA_f(u,v) = sum_{i<ml, j<nl} a_f[i+S+u][j+T+v]^2              (frame energy)
// with a_f = 0 outside the frame.  Substituting p = (i+u+1, j+v+1) on the extended grid
// P = [0, ml+2) x [0, nl+2):
//   H_f(c) = sum_p A_f[p] Bt_c[p],   A_f[p] = a_f[p_r+S-1][p_c+T-1],
//                                    Bt_c[p] = b[p_r-u'][p_c-v'],  c = 3u'+v', u' = u+1
// -- one GEMM D[(frame, part)][(c, part)] = sum_p over the pixels p, for a batch of 64
// frames: M = 128 rows (7-bit hi parts of 64 frames, then lo parts), N = 32 columns
// (hi parts of the nine shifted templates, then lo parts; 14 zero columns), K = the
// pixels in 32-column steps.  The exact integer recombination
//   H = 2^14 D[hi][hi] + 2^7 (D[hi][lo] + D[lo][hi]) + D[lo][lo]
// is the same hi/lo split the coarse search uses (values < 2^14, kernels_tc.cuh).
// int32 accumulators are split into `nsets` row classes (p_r mod nsets) so no
// accumulator sums more than 2^31 / 127^2 products.  GA comes from the converter
// warps, which touch every sample once anyway: per-row totals and the four edge
// columns, binned by row class (rows 0, 1, ml, ml+1, interior), then combined per
// candidate in the epilogue.
//
// Per CTA (64 frames x a part of the rows), warp-specialised; a stage is one grid row
// p_r x a chunk of 7 K-steps:
//   warp 0   one bulk copy per stage of its 7 template B tiles (precomputed table,
//            L2-resident) into the operand stage;
//   warp 1   MMA issuer: 7 MMAs (M128 N32 K32) per stage into accumulator set p_r mod nsets;
//   warps 2-9 converters, 8 frames each: their raw rows (frame row p_r+S_f-1, 240
//            columns from the 8-aligned column below p_c+T_f-1) by 16-byte LDGSTS with
//            zero fill, RTC_NSR-1 stages ahead; then u16 -> int8 hi/lo A tiles in the
//            core-matrix layout, and the GA bins.  (One TMA box per frame row was
//            tried first: 64 small boxes per stage left the kernel at ~1.3 TB/s.)
// Epilogue (warps 2-5, one TMEM lane each): sets summed in 64 bits, parts recombined,
// atomically added to acc[f][0..17] (the layout k_refine_pick reads).
#pragma once

#include <cmath>

namespace moco {

#ifdef MOCO_RTC_TIMING
#define RT_T(...) __VA_ARGS__
#else
#define RT_T(...)
#endif

constexpr int RTC_F = 64;                 // frames per CTA
constexpr int RTC_KC = 7;                 // K-steps (32 grid columns) per stage
constexpr int RTC_BOXW = 240;             // raw box width (u16): 32*KC + 7 misalignment
#ifndef RTC_NSR
#define RTC_NSR 4
#endif
#ifndef RTC_NSO
#define RTC_NSO 2
#endif
constexpr int RTC_NS = RTC_NSR;           // raw ring depth
constexpr int RTC_NO = RTC_NSO;           // operand ring depth
constexpr int RTC_CW = 8;                 // converter warps
constexpr int RTC_THREADS = 32 * (2 + RTC_CW);
constexpr int RTC_RAW_SLOT = 512;         // bytes per frame in a raw stage (480 used, 128-B aligned)
constexpr int RTC_RAW_STAGE = RTC_F * RTC_RAW_SLOT;
constexpr int RTC_A_STAGE = RTC_KC * 4096;   // A tiles: 128 rows x 32 B per K-step
constexpr int RTC_B_STAGE = RTC_KC * 1024;   // B tiles: 32 rows x 32 B per K-step
constexpr int RTC_OP_STAGE = RTC_A_STAGE + RTC_B_STAGE;
constexpr int RTC_BINS_OFF = 1024;        // [64][5 row classes][5] u64
constexpr int RTC_RAW_OFF = 14336;
constexpr int RTC_OP_OFF = RTC_RAW_OFF + RTC_NS * RTC_RAW_STAGE;
constexpr int RTC_SMEM = RTC_OP_OFF + RTC_NO * RTC_OP_STAGE + 1024;   // + alignment slack

struct RtcGeom {
  int ml, nl;
  int nsteps;   // K-steps per grid row: ceil((nl+2)/32)
  int nch;      // stages per grid row: ceil(nsteps/KC)
  int nsets;    // accumulator sets (power of 2, <= 16)
};

inline bool rtc_make(RtcGeom *g, int ml, int nl, int vb) {
  if (vb > 14 || ml < 4 || nl < 8 || nl % 8 != 0) return false;
  g->ml = ml;
  g->nl = nl;
  g->nsteps = (nl + 2 + 31) / 32;
  g->nch = (g->nsteps + RTC_KC - 1) / RTC_KC;
  const double per_row = (double)(nl + 2) * 127.0 * 127.0;
  int ns = 1;
  while (ns <= 16 && std::ceil((double)(ml + 2) / ns) * per_row >= 2147483648.0) ns <<= 1;
  if (ns > 16) return false;
  g->nsets = ns;
  return true;
}

// Template candidate tiles, one per (grid row p_r, K-step k): rows n = pb*16 + c
// (c < 9: part pb of Bt_c, c >= 9: zero), K-major core matrices, LBO 512 / SBO 128.
__global__ void k_rtc_table(const uint16_t *__restrict__ b, int pitch, int ml, int nl, int nsteps, uint8_t *tab) {
  const int64_t total = (int64_t)(ml + 2) * nsteps * 1024;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = e >> 10;
    const int off = (int)(e & 1023);
    const int pr = (int)(tile / nsteps), k = (int)(tile % nsteps);
    const int half = off >> 9, r = off & 511;
    const int n = (r >> 7) * 8 + ((r & 127) >> 4), x = half * 16 + (r & 15);
    const int pb = n >> 4, c = n & 15;
    uint8_t v = 0;
    if (c < 9) {
      const int i = pr - c / 3, j = 32 * k + x - c % 3;
      if (i >= 0 && i < ml && j >= 0 && j < nl) {
        const uint32_t val = b[(int64_t)i * pitch + j];
        v = (uint8_t)(pb == 0 ? (val >> 7) : (val & 127u));
      }
    }
    tab[e] = v;
  }
}

struct RtcArgs {
  const uint16_t *img;      // level-l frames
  int64_t fstride;          // elements between frames
  int pitch;                // elements between rows
  const uint8_t *tab;       // [ml+2][nsteps][1024]
  u64 *acc;                 // [B][18]: H for the nine candidates, then GA (atomically added)
  const int32_t *shift_in;  // [B][2] at level l+1
  int B;
  int parts;                // row parts per 64-frame group
  int rows_per_part;
  RtcGeom g;
};

__device__ __forceinline__ void rtc_stage(const RtcGeom &g, int r0, int i, int &pr, int &k0, int &kc) {
  pr = r0 + i / g.nch;
  k0 = (i % g.nch) * RTC_KC;
  kc = min(RTC_KC, g.nsteps - k0);
}

__global__ void __launch_bounds__(RTC_THREADS, 1) k_refine_tc(RtcArgs a) {
  extern __shared__ __align__(1024) unsigned char rtc_raw[];
  unsigned char *smem = rtc_raw + ((1024u - (smem_u32(rtc_raw) & 1023u)) & 1023u);
  uint64_t *afull = reinterpret_cast<uint64_t *>(smem), *aempty = afull + RTC_NO;
  uint64_t *done = aempty + RTC_NO;
  uint32_t *holder = reinterpret_cast<uint32_t *>(smem + 128);
  int *Ssh = reinterpret_cast<int *>(smem + 256), *Tsh = reinterpret_cast<int *>(smem + 512);
  u64 *bins = reinterpret_cast<u64 *>(smem + RTC_BINS_OFF);
  unsigned char *raw = smem + RTC_RAW_OFF, *ops = smem + RTC_OP_OFF;
  const RtcGeom &g = a.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = blockIdx.x / a.parts, part = blockIdx.x % a.parts;
  const int f0 = grp * RTC_F, nf = min(RTC_F, a.B - f0);
  const int r0 = part * a.rows_per_part, r1 = min(g.ml + 2, r0 + a.rows_per_part);
  const int nstage = (r1 - r0) * g.nch;
  const int nsets_used = min(g.nsets, r1 - r0);

  for (int k = tid; k < RTC_F * 25; k += RTC_THREADS) bins[k] = 0;
  if (tid < RTC_F) {
    int S = 0, T = 0;
    if (tid < nf) {
      S = 2 * a.shift_in[2 * (f0 + tid)];
      T = 2 * a.shift_in[2 * (f0 + tid) + 1];
    }
    Ssh[tid] = S;
    Tsh[tid] = T;
  }
  if (warp == 1) tmem_alloc(holder, 32 * g.nsets);
  if (tid == 0) {
    for (int s = 0; s < RTC_NO; ++s) {
      mbar_init(&afull[s], RTC_CW + 1);
      mbar_init(&aempty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = *holder;

  if (warp == 0) {
    // ---------------- loads
    for (int i = 0; i < nstage; ++i) {
      int pr, k0, kc;
      rtc_stage(g, r0, i, pr, k0, kc);
      const int so = i % RTC_NO, ro = i / RTC_NO;
      if (ro > 0) mbar_wait(&aempty[so], (ro - 1) & 1);
      if (lane == 0) {
        mbar_arrive_expect_tx(&afull[so], (uint32_t)(kc * 1024));
        bulk_g2s(ops + so * RTC_OP_STAGE + RTC_A_STAGE, a.tab + ((int64_t)pr * g.nsteps + k0) * 1024,
                 (uint32_t)(kc * 1024), &afull[so]);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    const uint32_t idesc = idesc_i8(128, 32);
    const uint64_t ad0 = umma_desc(smem_u32(ops), 2048, 128);
    const uint64_t bd0 = umma_desc(smem_u32(ops + RTC_A_STAGE), 512, 128);
    const uint32_t ahi = (uint32_t)(ad0 >> 32), bhi = (uint32_t)(bd0 >> 32);
    for (int i = 0; i < nstage; ++i) {
      const int s = i % RTC_NO, rnd = i / RTC_NO;
      int pr, k0, kc;
      rtc_stage(g, r0, i, pr, k0, kc);
      mbar_wait(&afull[s], rnd & 1);
      tc_fence_after();
      const int rr = pr - r0;
      const uint32_t d = taddr + (uint32_t)((rr & (g.nsets - 1)) * 32);
      const bool first = rr < g.nsets && k0 == 0;
      const uint32_t alo = (uint32_t)ad0 + (uint32_t)(s * RTC_OP_STAGE >> 4);
      const uint32_t blo = (uint32_t)bd0 + (uint32_t)(s * RTC_OP_STAGE >> 4);
      for (int k = 0; k < kc; ++k)
        mma_i8_elect(d, alo + (uint32_t)(k * 4096 >> 4), ahi, blo + (uint32_t)(k * 1024 >> 4), bhi, idesc,
                     (first && k == 0) ? 0u : 1u);
      mma_commit_elect(&aempty[s]);
      __syncwarp();
    }
    mma_commit_elect(done);
    __syncwarp();
  } else {
    // ---------------- converters: lane = (frame f of the warp's 8, K-half phase kq)
    const int cw = warp - 2, f = cw * 8 + (lane & 7), kq = lane >> 3;
    const bool fv = f < nf;
    const int o = (Tsh[f] - 1) & 7;                  // box element of grid column 32*k0
    const uint32_t sh = (uint32_t)(o & 1) * 16;
    const int nl2 = g.nl + 2;
    u64 tot = 0, e0 = 0, e1 = 0, e2 = 0, e3 = 0;
    RT_T(uint64_t w_data = 0, w_empty = 0, w_conv = 0, w_fence = 0, w_issue = 0; const uint64_t tbeg = gtimer();)
    // raw rows of this warp's 8 frames: 16-byte LDGSTS with zero fill outside the frame
    // (a 16-byte block at an 8-aligned column is entirely inside or outside), issued
    // RTC_NS-1 stages ahead; a warp reads only the slots it filled: __syncwarp suffices
    auto issue = [&](int j) {
      if (j < nstage) {
        int pr, k0, kc;
        rtc_stage(g, r0, j, pr, k0, kc);
        unsigned char *rs = raw + (j % RTC_NS) * RTC_RAW_STAGE;
        for (int k = lane; k < 8 * (RTC_BOXW / 8); k += 32) {
          const int fl = k / (RTC_BOXW / 8), q = k % (RTC_BOXW / 8), ff = cw * 8 + fl;
          const int x = 32 * k0 + Tsh[ff] - 1, xb = x - (x & 7) + 8 * q, y = pr + Ssh[ff] - 1;
          const bool ok = ff < nf && y >= 0 && y < g.ml && xb >= 0 && xb < g.nl;
#ifdef RTC_SAMEFRAME
          const uint16_t *src = ok ? a.img + (int64_t)(f0) * a.fstride + (int64_t)y * a.pitch + xb : a.img;
#else
          const uint16_t *src = ok ? a.img + (int64_t)(f0 + ff) * a.fstride + (int64_t)y * a.pitch + xb : a.img;
#endif
          cp_async16_zfill(rs + ff * RTC_RAW_SLOT + 16 * q, src, ok ? 16u : 0u);
        }
      }
      cp_async_commit();
    };
    for (int j = 0; j < RTC_NS - 1; ++j) issue(j);
    for (int i = 0; i < nstage; ++i) {
      const int s = i % RTC_NS;
      int pr, k0, kc;
      rtc_stage(g, r0, i, pr, k0, kc);
      const int so = i % RTC_NO, ro = i / RTC_NO;
      RT_T(uint64_t t0 = gtimer();)
      cp_async_wait<RTC_NS - 2>();
      __syncwarp();
      RT_T(uint64_t t1 = gtimer(); w_data += t1 - t0;)
      if (ro > 0) mbar_wait(&aempty[so], (ro - 1) & 1);
      RT_T(uint64_t t2 = gtimer(); w_empty += t2 - t1;)
      const uint32_t rb = smem_u32(raw + s * RTC_RAW_STAGE + f * RTC_RAW_SLOT) + (uint32_t)(o >> 1) * 4;
      unsigned char *A = ops + so * RTC_OP_STAGE;
#ifdef RTC_NOCONV
      for (int kh = kq; kh < 0; kh += 4) {
#else
      for (int kh = kq; kh < 2 * kc; kh += 4) {
#endif
        const int pc0 = 32 * k0 + 16 * kh;   // grid columns pc0 .. pc0+15
        uint32_t w[9], v2[8];
#pragma unroll
        for (int q = 0; q < 9; ++q) w[q] = lds32(rb + (uint32_t)(32 * kh + 4 * q));
#pragma unroll
        for (int q = 0; q < 8; ++q) v2[q] = __funnelshift_r(w[q], w[q + 1], sh);
        if (!fv) {
#pragma unroll
          for (int q = 0; q < 8; ++q) v2[q] = 0;
        } else if (pc0 + 16 > nl2) {   // grid columns >= nl+2 carry no template: zero
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int c = pc0 + 2 * q;
            if (c >= nl2) v2[q] = 0;
            else if (c + 1 >= nl2) v2[q] &= 0xffffu;
          }
        }
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const uint32_t x0 = v2[2 * p], x1 = v2[2 * p + 1];
          lo[p] = __byte_perm(x0 & 0x007F007Fu, x1 & 0x007F007Fu, 0x6420);
          hi[p] = __byte_perm((x0 >> 7) & 0x007F007Fu, (x1 >> 7) & 0x007F007Fu, 0x6420);
        }
        unsigned char *tile = A + (kh >> 1) * 4096 + (kh & 1) * 2048 + (f & 7) * 16;
        *reinterpret_cast<uint4 *>(tile + (f >> 3) * 128) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4 *>(tile + (8 + (f >> 3)) * 128) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        // frame energy: the 16 squares (each < 2^28) in two 32-bit halves
        uint32_t sa = 0, sb = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t x = v2[q], y = v2[q + 4];
          sa += (x & 0xffffu) * (x & 0xffffu) + (x >> 16) * (x >> 16);
          sb += (y & 0xffffu) * (y & 0xffffu) + (y >> 16) * (y >> 16);
        }
        tot += (u64)sa + (u64)sb;
        if (pc0 == 0) {
          e0 += (u64)((v2[0] & 0xffffu) * (v2[0] & 0xffffu));
          e1 += (u64)((v2[0] >> 16) * (v2[0] >> 16));
        }
        if (pc0 <= g.nl && g.nl < pc0 + 16) {   // nl % 8 == 0: columns nl, nl+1 share one word
          const uint32_t x = (g.nl - pc0) == 0 ? v2[0] : v2[4];
          e2 += (u64)((x & 0xffffu) * (x & 0xffffu));
          e3 += (u64)((x >> 16) * (x >> 16));
        }
      }
      RT_T(uint64_t t3 = gtimer(); w_conv += t3 - t2;)
      fence_proxy_async();   // A tiles written by the generic proxy, read by the tensor core
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[so]);
      RT_T(uint64_t t4 = gtimer(); w_fence += t4 - t3;)
      issue(i + RTC_NS - 1);   // into the slot read in the previous iteration
      RT_T(w_issue += gtimer() - t4;)
      // end of a grid row: flush the row-class bins when the class changes next
      if (k0 + kc == g.nsteps) {
        const int cls = pr < 2 ? pr : (pr >= g.ml ? pr - g.ml + 2 : 4);
        if (cls != 4 || pr + 1 == g.ml || pr + 1 == r1) {
          if (fv) {
            u64 *bn = bins + (f * 5 + cls) * 5;
            atomicAdd(reinterpret_cast<unsigned long long *>(bn + 0), (unsigned long long)tot);
            atomicAdd(reinterpret_cast<unsigned long long *>(bn + 1), (unsigned long long)e0);
            atomicAdd(reinterpret_cast<unsigned long long *>(bn + 2), (unsigned long long)e1);
            atomicAdd(reinterpret_cast<unsigned long long *>(bn + 3), (unsigned long long)e2);
            atomicAdd(reinterpret_cast<unsigned long long *>(bn + 4), (unsigned long long)e3);
          }
          tot = e0 = e1 = e2 = e3 = 0;
        }
      }
    }
    RT_T(if (blockIdx.x == 0 && lane == 0 && (warp == 2 || warp == 9)) printf("RTT warp %d nstage %d total %llu data %llu aempty %llu conv %llu fence %llu issue %llu\n", warp, nstage, (unsigned long long)(gtimer() - tbeg), (unsigned long long)w_data, (unsigned long long)w_empty, (unsigned long long)w_conv, (unsigned long long)w_fence, (unsigned long long)w_issue);)
  }

  // ---------------- epilogue
  mbar_wait(done, 0);
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  u64 *Es = reinterpret_cast<u64 *>(raw);   // [128][18]: (pb = hi, c < 9), (pb = lo, c < 9)
  if (warp >= 2 && warp < 6) {
    const int sub = warp & 3, m = sub * 32 + lane;
    u64 eh[9], el[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) { eh[c] = 0; el[c] = 0; }
    for (int st = 0; st < nsets_used; ++st) {
      uint32_t x[16], y[16];
      const uint32_t tb = taddr + ((uint32_t)(sub * 32) << 16) + (uint32_t)(st * 32);
      tmem_ld16(tb, x);
      tmem_ld16(tb + 16, y);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 9; ++c) { eh[c] += x[c]; el[c] += y[c]; }
    }
#pragma unroll
    for (int c = 0; c < 9; ++c) { Es[m * 18 + c] = eh[c]; Es[m * 18 + 9 + c] = el[c]; }
  }
  __syncthreads();
  for (int k = tid; k < RTC_F * 9; k += RTC_THREADS) {
    const int ff = k / 9, c = k % 9;
    if (ff >= nf) continue;
    const u64 *ph = Es + ff * 18, *pl = Es + (64 + ff) * 18;
    const u64 H = (ph[c] << 14) + ((ph[9 + c] + pl[c]) << 7) + pl[9 + c];
    // GA: row classes of u' (0: rows 0,1,int; 1: 1,int,ml; 2: int,ml,ml+1), minus the
    // two grid columns outside [v', v'+nl) (0: nl,nl+1; 1: 0,nl+1; 2: 0,1)
    const int up = c / 3, vp = c % 3;
    const int ex1 = vp == 0 ? 3 : 1, ex2 = vp == 2 ? 2 : 4;
    const u64 *bn = bins + ff * 25;
    u64 GA = 0;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int cls = up == 0 ? (q == 0 ? 0 : q == 1 ? 1 : 4) : up == 1 ? (q == 0 ? 1 : q == 1 ? 4 : 2)
                                                                          : (q == 0 ? 4 : q == 1 ? 2 : 3);
      GA += bn[cls * 5] - bn[cls * 5 + ex1] - bn[cls * 5 + ex2];
    }
    u64 *acc = a.acc + (int64_t)(f0 + ff) * 18;
    atomicAdd(reinterpret_cast<unsigned long long *>(acc + c), (unsigned long long)H);
    atomicAdd(reinterpret_cast<unsigned long long *>(acc + 9 + c), (unsigned long long)GA);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(taddr, 32 * g.nsets);
}

}  // namespace moco
