// kernels_rtc.cuh -- S5 refine sums on the 5th-gen tensor cores (tcgen05, kind::i8),
// conversion-free: the raw u16 frame rows ARE the A operand.
//
// The +-1 refinement at level l needs, per frame f and each of
// the nine candidates (u, v) around the doubled coarse shift (S, T) = 2 s_{l+1},
//   H_f(u,v)  = sum_{i<ml, j<nl} a_f[i+S+u][j+T+v] b[i][j]        (cross term)
//   GA_f(u,v) = sum_{i<ml, j<nl} a_f[i+S+u][j+T+v]^2              (frame energy)
// with a_f = 0 outside the frame.  On the extended grid (p_r, p_c) in [0, ml+2) x
// [0, nl+2), A_f[p_r][p_c] = a_f[p_r+S-1][p_c+T-1], and with u' = u+1, v' = v+1:
//   H_f(u',v') = sum_{i<ml} sum_{p_c} A_f[i+u'][p_c] b[i][p_c-v'].
//
// A little-endian u16 row is an int8 row of interleaved (low byte, high byte) pairs.
// Fed to tcgen05.mma.kind::i8 unchanged, with three B rows per candidate
//   type a: (b_lo, 0)   -> sum a_lo b_lo                  (weight 1)
//   type b: (b_hi, b_lo)-> sum a_lo b_hi + a_hi b_lo       (weight 2^8)
//   type c: (0, b_hi)   -> sum a_hi b_hi                  (weight 2^16)
// the cross term is H = D_a + 2^8 D_b + 2^16 D_c exactly (values < 2^14: bytes <= 255,
// all products of u8 x u8 in int32 accumulators) -- no per-pixel work for H at all.
//
// MMA shape: M = 128 = 16 frames x 8 consecutive grid rows (one 8-row group per frame),
// N = 64 = 6 template rows x 3 column shifts v' x 3 types (54 used), K = 32 bytes =
// 16 pixels.  The A tiles are TMA boxes {64 pixels, 32 grid rows} per frame written with
// the 128-byte swizzle: each box row is one 128-byte K-major row (64 pixels), the boxes
// 1024-byte aligned, and the UMMA descriptor (layout SWIZZLE_128B, SBO = box size) starts
// at row 6q of every box for row group q and at byte 32k for K-step k -- the swizzle
// phase follows the address bits, so the window slides freely.  A row group G (template
// rows 6G..6G+5) needs grid rows 6G..6G+7; in D, entry (frame, r_rel; t_rel, v', type) is
// useful when u' = r_rel - t_rel is 0, 1 or 2.  A frame's box starts at the 8-aligned
// column below T-1, so the grid column of box pixel e is e - o with o = (T-1) mod 8
// (odd: T is even); frames are bucketed by o (k_rtc_bucket) and the template table holds
// one pre-shifted copy per class.  int32 accumulators alternate between `nsets` TMEM sets
// by row group.  GA is the only per-pixel CUDA-core work: one warp per frame sums a^2
// from the staged (swizzled) boxes, grid rows binned by class 0, 1, ml, ml+1, interior,
// the four edge columns kept apart; the epilogue combines the bins per candidate.
//
// Work unit: a CTA takes 16 frames of one alignment class x a range of row groups; a
// stage = 5 row groups (32 grid rows) x 4 K-steps (64 pixels):
//   warp 0     TMA: one box per frame + one bulk copy of B tiles per row group;
//   warp 1     MMA issuer: 5 x 4 MMAs (M128 N64 K32) per stage;
//   warps 2-17 GA, one frame each, from the same staged boxes;
// double-buffered stages; epilogue: TMEM -> per-row partial H -> 8-lane shuffle sums.
// C2, 2 368 frames: 467 us against 584 us for the CUDA-core kernel (an earlier variant
// with a dimension-reordered, 16-byte-row tensor map took 616 us: TMA-row bound); in the
// three-stream pipeline 1.40 -> 1.48 M frames/s.  DESIGN.md section 11.
#pragma once

#include <cmath>

namespace moco {

#ifdef MOCO_RTC_TIMING
__device__ __forceinline__ uint64_t gtimer_rt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define gtimer gtimer_rt
#endif
#ifdef MOCO_RTC_TIMING
#define RT_T(...) __VA_ARGS__
#else
#define RT_T(...)
#endif

constexpr int RTC_F = 16;                  // frames per CTA (core-matrix groups of M)
#ifndef RTC_RGROUPS
#define RTC_RGROUPS 5
#endif
constexpr int RTC_RG = RTC_RGROUPS;                  // row groups (6 template rows each) per stage
constexpr int RTC_R = (6 * RTC_RG + 2 + 7) / 8 * 8;  // grid rows per stage box (6 RG + 2 used)
#ifndef RTC_NSTAGE
#define RTC_NSTAGE 2
#endif
constexpr int RTC_KS = 4;                  // K-steps (16 pixels) per stage: one 128-byte row
constexpr int RTC_NST = RTC_NSTAGE;        // ring depth
constexpr int RTC_CH = 2 * RTC_KS;         // 8-pixel chunks per stage box
#ifndef RTC_GA_WARPS
#define RTC_GA_WARPS 16
#endif
// GA split: 1 = the GA warps sum a^2 over every staged pixel (grid rows [0, ml+2), box
// columns [0, 16 nk), i.e. grid columns [-o, 16 nk - o)) with one uniform path, and the
// pick kernel (k_refine_pick, ga_total) subtracts the columns outside the grid and
// separates the rows 0, 1, ml, ml+1 and the columns 0, 1, nl, nl+1 from the frame itself
// (a few hundred pixels per frame); 0 = row-class bins and edge columns here
#ifndef RTC_GA_TOTAL
#define RTC_GA_TOTAL 1
#endif
constexpr int RTC_CW = RTC_GA_WARPS;       // GA warps (16 / RTC_CW frames each)
constexpr int RTC_THREADS = 32 * (2 + RTC_CW);
constexpr int RTC_SLOT = RTC_R * 128;                        // bytes per frame box: R rows of 128 B (SW128)
constexpr int RTC_RAW = RTC_F * RTC_SLOT;                     // A stage
constexpr int RTC_BT = 2048;                                  // one B tile: 64 rows x 32 B
constexpr int RTC_STAGE = RTC_RAW + RTC_RG * RTC_KS * RTC_BT;
constexpr int RTC_BINS_OFF = 1024;         // [16][5 row classes][5] u64
constexpr int RTC_ST_OFF = 5120;           // after the bins (16 x 25 x 8 = 3200 B), 1024-aligned
constexpr int RTC_SMEM = RTC_ST_OFF + RTC_NST * RTC_STAGE + 1024;  // + alignment slack
static_assert(RTC_SLOT % 1024 == 0 && RTC_R % 8 == 0, "SWIZZLE_128B boxes must be 1024-byte aligned");
static_assert(RTC_BINS_OFF + RTC_F * 25 * 8 <= RTC_ST_OFF && RTC_ST_OFF % 1024 == 0, "bins overlap the stages");
static_assert(RTC_SMEM <= 227 * 1024, "shared memory");
static_assert(RTC_CH % 4 == 0 && RTC_NST * 2 * 8 + 8 <= 128, "chunk lanes, barrier space");

struct RtcGeom {
  int ml, nl;
  int nk;       // K-steps per grid row: ceil((nl + 2 + 7) / 16)
  int nstrips;  // ceil(nk / KS)
  int ng;       // row groups: ceil(ml / 6)
  int nsets;    // accumulator sets (power of 2, <= 8: 64 TMEM columns each)
};

inline bool rtc_make(RtcGeom *g, int ml, int nl, int vb) {
  if (vb > 14 || ml < 6 || nl < 8 || nl % 8 != 0) return false;
  g->ml = ml;
  g->nl = nl;
  g->nk = (nl + 2 + 7 + 15) / 16;
  g->nstrips = (g->nk + RTC_KS - 1) / RTC_KS;
  g->ng = (ml + 5) / 6;
  // one D entry adds, per row group, nk*16 products of bytes (type a: <= 255*255)
  const double per_group = (double)g->nk * 16.0 * 255.0 * 255.0;
  int ns = 1;
  while (ns <= 8 && std::ceil((double)g->ng / ns) * per_group >= 2147483648.0) ns <<= 1;
  if (ns > 8) return false;
  g->nsets = ns;
  return true;
}
inline size_t rtc_table_bytes(const RtcGeom &g) { return (size_t)4 * g.ng * g.nk * RTC_BT; }

// B tiles per (class c: o = 2c+1, row group G, K-step j): row n = (t*3 + v')*3 + type
// (54..63 zero), byte k of the step = pixel k>>1, byte k&1 (0: low, 1: high) of A; the
// pixel's grid column is 16j + (k>>1) - o.  Layout [half][64 rows][16 B] (LBO 1024, SBO 128).
__global__ void k_rtc_table(const uint16_t *__restrict__ b, int pitch, int ml, int nl, int ng, int nk, uint8_t *tab) {
  const int64_t total = (int64_t)4 * ng * nk * RTC_BT;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = e / RTC_BT;
    const int off = (int)(e % RTC_BT);
    const int c = (int)(tile / ((int64_t)ng * nk)), rem = (int)(tile % ((int64_t)ng * nk));
    const int G = rem / nk, j = rem % nk;
    const int half = off >> 10, n = (off & 1023) >> 4, kb = off & 15;
    const int k = half * 16 + kb;
    uint8_t v = 0;
    if (n < 54) {
      const int tv = n / 3, type = n % 3, t = tv / 3, vp = tv % 3;
      const int i = 6 * G + t, pc = 16 * j + (k >> 1) - (2 * c + 1), jc = pc - vp;
      if (i < ml && jc >= 0 && jc < nl) {
        const uint32_t bv = b[(int64_t)i * pitch + jc];
        const uint32_t lo = bv & 255u, hi = bv >> 8;
        const int byte = k & 1;
        v = (uint8_t)(type == 0 ? (byte ? 0u : lo) : type == 1 ? (byte ? lo : hi) : (byte ? hi : 0u));
      }
    }
    tab[e] = v;
  }
}

// Frames of a batch bucketed by alignment class o = (T-1) mod 8 in {1,3,5,7}:
// meta[0..3] = class counts, meta[4..8] = first CTA group of each class (prefix of
// ceil(count/16)); perm = frame indices, class-major.  One block.
__global__ void __launch_bounds__(1024) k_rtc_bucket(const int32_t *__restrict__ shift_in, int B, int *perm,
                                                     int *meta) {
  __shared__ int cnt[4], base[4], fill[4];
  if (threadIdx.x < 4) { cnt[threadIdx.x] = 0; fill[threadIdx.x] = 0; }
  __syncthreads();
  for (int f = threadIdx.x; f < B; f += blockDim.x) atomicAdd(&cnt[((2 * shift_in[2 * f + 1] - 1) & 7) >> 1], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int b0 = 0, g0 = 0;
    for (int c = 0; c < 4; ++c) {
      base[c] = b0;
      meta[c] = cnt[c];
      meta[4 + c] = g0;
      b0 += cnt[c];
      g0 += (cnt[c] + RTC_F - 1) / RTC_F;
    }
    meta[8] = g0;
  }
  __syncthreads();
  for (int f = threadIdx.x; f < B; f += blockDim.x) {
    const int c = ((2 * shift_in[2 * f + 1] - 1) & 7) >> 1;
    perm[base[c] + atomicAdd(&fill[c], 1)] = f;
  }
}

// u16 frames [frames][rows][cols] (row pitch, frame stride in elements), box {64 columns,
// rows, 1 frame} written with the 128-byte swizzle: each box row is one 128-byte K-major
// row of the A operand (64 pixels = 128 interleaved low/high bytes), zero fill outside.
inline bool tmap_u16_sw128(CUtensorMap *tm, const void *base, int cols, int rows, int64_t frames, int pitch,
                           int64_t fstride, int box_rows) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)frames};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch * 2, (cuuint64_t)fstride * 2};
  const cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void *>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// UMMA shared-memory descriptor, K-major, 128-byte swizzle (layout type 2): rows of 128 B
// in 1024-byte atoms, SBO = byte distance between 8-row groups; the start address may
// sit at any row of an atom (the XOR phase comes from the address bits).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Four MMAs into one accumulator (the four K-steps of a row group): one elect, one
// predicate for the first (accumulate = acc0), the other three accumulate.
__device__ __forceinline__ void mma_i8_k4_elect(uint32_t d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                                uint32_t ahi, uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3,
                                                uint32_t bhi, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 da0, da1, da2, da3, db0, db1, db2, db3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %12, 0;\n\t"
      "mov.b64 da0, {%1, %5};\n\t"
      "mov.b64 da1, {%2, %5};\n\t"
      "mov.b64 da2, {%3, %5};\n\t"
      "mov.b64 da3, {%4, %5};\n\t"
      "mov.b64 db0, {%6, %10};\n\t"
      "mov.b64 db1, {%7, %10};\n\t"
      "mov.b64 db2, {%8, %10};\n\t"
      "mov.b64 db3, {%9, %10};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], da0, db0, %11, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], da1, db1, %11, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], da2, db2, %11, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], da3, db3, %11, 1;\n\t}" ::"r"(d),
      "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(ahi), "r"(b0), "r"(b1), "r"(b2), "r"(b3), "r"(bhi), "r"(idesc),
      "r"(acc0)
      : "memory");
}

struct RtcArgs {
  const uint8_t *tab;       // rtc_table_bytes
  u64 *acc;                 // [B][18]: H for the nine candidates, then GA (atomically added)
  const int32_t *shift_in;  // [B][2] at level l+1
  const int *perm;          // [B] class-major frame order
  const int *meta;          // k_rtc_bucket output
  int B;
  int parts;                // row-group ranges per 16-frame group
  int groups_per_part;      // multiple of RTC_RG
  RtcGeom g;
};

__global__ void __launch_bounds__(RTC_THREADS, 1) k_refine_tc(const __grid_constant__ CUtensorMap tmF, RtcArgs a) {
  extern __shared__ __align__(1024) unsigned char rtc_raw[];
  unsigned char *smem = rtc_raw + ((1024u - (smem_u32(rtc_raw) & 1023u)) & 1023u);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem), *empty = full + RTC_NST, *done = full + 2 * RTC_NST;
  uint32_t *holder = reinterpret_cast<uint32_t *>(smem + 128);
  int *Ssh = reinterpret_cast<int *>(smem + 256), *Tsh = reinterpret_cast<int *>(smem + 320);
  int *Fid = reinterpret_cast<int *>(smem + 384);
  u64 *bins = reinterpret_cast<u64 *>(smem + RTC_BINS_OFF);
  unsigned char *stg = smem + RTC_ST_OFF;
  const RtcGeom &g = a.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // (class, group in class, part) of this CTA
  const int gidx = blockIdx.x / a.parts, part = blockIdx.x % a.parts;
  if (gidx >= a.meta[8]) return;
  int cls = 0;
  while (cls < 3 && gidx >= a.meta[5 + cls]) ++cls;
  const int gic = gidx - a.meta[4 + cls];
  int cbase = 0;
  for (int c = 0; c < cls; ++c) cbase += a.meta[c];
  const int f0 = cbase + gic * RTC_F, nf = min(RTC_F, a.meta[cls] - gic * RTC_F);
  const int o = 2 * cls + 1;
  const int G0 = part * a.groups_per_part, G1 = min(g.ng, G0 + a.groups_per_part);
  const int nblk = (G1 - G0 + RTC_RG - 1) / RTC_RG;   // row-group blocks (stages per strip)
  const int nstage = max(0, nblk) * g.nstrips;
  const int tcols = max(64, 64 * g.nsets);
  RT_T(const uint64_t t_beg = gtimer(); uint64_t w_a = 0, w_b = 0; uint64_t t0;)

  for (int k = tid; k < RTC_F * 25; k += RTC_THREADS) bins[k] = 0;
  if (tid < RTC_F) {
    int S = 0, T = 0, fi = -1;
    if (tid < nf) {
      fi = a.perm[f0 + tid];
      S = 2 * a.shift_in[2 * fi];
      T = 2 * a.shift_in[2 * fi + 1];
    }
    Ssh[tid] = S;
    Tsh[tid] = T;
    Fid[tid] = fi;
  }
  if (warp == 1) tmem_alloc(holder, tcols);
  if (tid == 0) {
    for (int s = 0; s < RTC_NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + RTC_CW);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = *holder;

  if (warp == 0) {
    // ---------------- loads: one box per frame, B tiles per row group
    for (int i = 0; i < nstage; ++i) {
      const int s = i % RTC_NST, rnd = i / RTC_NST;
      const int gb = G0 + (i / g.nstrips) * RTC_RG, j0 = (i % g.nstrips) * RTC_KS;
      const int ngr = min(RTC_RG, G1 - gb), kc = min(RTC_KS, g.nk - j0);
      RT_T(t0 = gtimer();)
      if (rnd > 0) mbar_wait(&empty[s], (rnd - 1) & 1);
      RT_T(w_a += gtimer() - t0;)
#ifdef RTC_DIAG_NOB   // (diagnostic builds, results wrong: no B tiles loaded)
      if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)(nf * RTC_SLOT));
#else
      if (lane == 0)
        mbar_arrive_expect_tx(&full[s], (uint32_t)(nf * RTC_SLOT + ngr * kc * RTC_BT));
#endif
      __syncwarp();
      unsigned char *st = stg + s * RTC_STAGE;
      if (lane < nf) {
        const int x0 = (Tsh[lane] - 1) - ((Tsh[lane] - 1) & 7) + 16 * j0;   // 8-aligned column below T-1
        tma_load3(st + lane * RTC_SLOT, &tmF, x0, 6 * gb + Ssh[lane] - 1, Fid[lane], &full[s]);
      }
#ifndef RTC_DIAG_NOB
      if (lane == 0)
#else
      if (false)
#endif
        for (int q = 0; q < ngr; ++q)
          bulk_g2s(st + RTC_RAW + q * RTC_KS * RTC_BT,
                   a.tab + (((int64_t)cls * g.ng + gb + q) * g.nk + j0) * RTC_BT, (uint32_t)(kc * RTC_BT),
                   &full[s]);
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    const uint32_t idesc = idesc_i8(128, 64);
    const uint64_t ad0 = umma_desc_sw128(smem_u32(stg), RTC_SLOT);
    const uint64_t bd0 = umma_desc(smem_u32(stg + RTC_RAW), 1024, 128);
    const uint32_t ahi = (uint32_t)(ad0 >> 32), bhi = (uint32_t)(bd0 >> 32);
    for (int i = 0; i < nstage; ++i) {
      const int s = i % RTC_NST, rnd = i / RTC_NST;
      const int gb = G0 + (i / g.nstrips) * RTC_RG, j0 = (i % g.nstrips) * RTC_KS;
      const int ngr = min(RTC_RG, G1 - gb), kc = min(RTC_KS, g.nk - j0);
      RT_T(t0 = gtimer();)
      mbar_wait(&full[s], rnd & 1);
      RT_T(w_a += gtimer() - t0;)
      tc_fence_after();
      const uint32_t alo = (uint32_t)ad0 + (uint32_t)(s * RTC_STAGE >> 4);
      const uint32_t blo = (uint32_t)bd0 + (uint32_t)(s * RTC_STAGE >> 4);
#ifndef RTC_DIAG_NOMMA   // (diagnostic builds, results wrong: tools/rtc_diag.sh)
      for (int q = 0; q < ngr; ++q) {
#else
      for (int q = 0; q < 0; ++q) {
#endif
        const int G = gb + q, Gr = G - G0;
        // sets by the part-relative group index: the epilogue reads sets 0 .. nsets_used-1
        const uint32_t d = taddr + (uint32_t)((Gr & (g.nsets - 1)) * 64);
        // A: bytes 32k .. 32k+31 of rows 6q .. 6q+7 of every frame box
        const uint32_t aq = alo + (uint32_t)((6 * q * 128) >> 4), bq = blo + (uint32_t)((q * RTC_KS * RTC_BT) >> 4);
        const uint32_t acc0 = (Gr < g.nsets && j0 == 0) ? 0u : 1u;
        if (kc == 4) {
          mma_i8_k4_elect(d, aq, aq + 2, aq + 4, aq + 6, ahi, bq, bq + (RTC_BT >> 4), bq + 2 * (RTC_BT >> 4),
                          bq + 3 * (RTC_BT >> 4), bhi, idesc, acc0);
        } else {
          for (int k = 0; k < kc; ++k)
            mma_i8_elect(d, aq + (uint32_t)(2 * k), ahi, bq + (uint32_t)(k * (RTC_BT >> 4)), bhi, idesc,
                         k == 0 ? acc0 : 1u);
        }
      }
      mma_commit_elect(&empty[s]);
      __syncwarp();
    }
    mma_commit_elect(done);
    __syncwarp();
  } else {
    // ---------------- GA warps: warp w = frame w; lane = (row rr & 7, chunk ch & 3), so
    // each 8-lane phase of a 16-byte load reads 128 contiguous bytes (frame boxes are a
    // multiple of 128 B apart: lanes on different frames would share banks)
    const int cw = warp - 2;
    constexpr int FPW = RTC_F / RTC_CW;             // frames per GA warp
    const int nl2 = g.nl + 2;
    const int lr = lane & 7, lc = lane >> 3;
    u64 tot[FPW], e0[FPW], e1[FPW], e2[FPW], e3[FPW];   // interior rows, per frame of this warp
#pragma unroll
    for (int k = 0; k < FPW; ++k) tot[k] = e0[k] = e1[k] = e2[k] = e3[k] = 0;
    for (int i = 0; i < nstage; ++i) {
      const int s = i % RTC_NST, rnd = i / RTC_NST;
      const int gb = G0 + (i / g.nstrips) * RTC_RG, j0 = (i % g.nstrips) * RTC_KS;
      const int ngr = min(RTC_RG, G1 - gb), kc = min(RTC_KS, g.nk - j0);
      // grid rows of this stage's row groups: [6gb, 6(gb+ngr)); the last group also owns
      // rows ml, ml+1 (the two below the template)
      const int r_lo = 6 * gb, r_hi = (gb + ngr == g.ng) ? g.ml + 2 : min(g.ml, 6 * (gb + ngr));
      RT_T(t0 = gtimer();)
      mbar_wait(&full[s], rnd & 1);
      RT_T(w_a += gtimer() - t0;)
#ifndef RTC_DIAG_NOGA
      const int nrow = r_hi - r_lo, nch = 2 * kc;
#else
      const int nrow = 0, nch = 0;
#endif
      // interior stage (no grid row 0, 1, ml, ml+1 and no edge column: about 2/3 of the
      // stages at C2): no per-chunk tests; a^2 = a * a_lo + 2^8 a * a_hi as two 16x8-bit
      // dot products per word (bytes regrouped by one PRMT); per stage and lane 32 words,
      // each product pair < 2^23 for a < 2^14, so the 32-bit sums cannot wrap
#ifndef RTC_DIAG_FASTONLY
      const bool fast = kc == RTC_KS && r_lo >= 2 && r_hi <= g.ml && 16 * j0 - o > 1 &&
                        16 * j0 + 8 * RTC_CH - o <= g.nl;
#else
      const bool fast = true;   // (diagnostic: edge stages summed as interior ones)
#endif
#pragma unroll
      for (int fk = 0; fk < FPW; ++fk) {
        const int f = cw + fk * RTC_CW;
        if (f >= nf) continue;
        const unsigned char *st = stg + s * RTC_STAGE + f * RTC_SLOT;
#if RTC_GA_TOTAL
        (void)fast;
        {
          uint4 q4[RTC_R / 8][RTC_CH / 4];
#pragma unroll
          for (int rq = 0; rq < RTC_R / 8; ++rq) {
            const int br = rq * 8 + lr;
#pragma unroll
            for (int cb = 0; cb < RTC_CH / 4; ++cb)
              q4[rq][cb] = (br < nrow && cb * 4 + lc < nch)
                               ? *reinterpret_cast<const uint4 *>(st + br * 128 + (((cb * 4 + lc) ^ lr) << 4))
                               : make_uint4(0, 0, 0, 0);
          }
          uint32_t slo = 0, shi = 0;
#pragma unroll
          for (int rq = 0; rq < RTC_R / 8; ++rq)
#pragma unroll
            for (int cb = 0; cb < RTC_CH / 4; ++cb) {
              const uint32_t wv[4] = {q4[rq][cb].x, q4[rq][cb].y, q4[rq][cb].z, q4[rq][cb].w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t pb = __byte_perm(wv[q], 0, 0x3120);
                slo = __dp2a_lo(wv[q], pb, slo);
                shi = __dp2a_hi(wv[q], pb, shi);
              }
            }
          tot[fk] += (u64)slo + ((u64)shi << 8);
          continue;
        }
#endif
        if (fast) {
          uint4 q4[RTC_R / 8][RTC_CH / 4];
#pragma unroll
          for (int rq = 0; rq < RTC_R / 8; ++rq) {
            const int br = rq * 8 + lr;   // box row = grid row - r_lo (r_lo = 6 gb)
#pragma unroll
            for (int cb = 0; cb < RTC_CH / 4; ++cb)
              q4[rq][cb] = br < nrow ? *reinterpret_cast<const uint4 *>(st + br * 128 + (((cb * 4 + lc) ^ lr) << 4))
                                     : make_uint4(0, 0, 0, 0);
          }
          uint32_t slo = 0, shi = 0;
#pragma unroll
          for (int rq = 0; rq < RTC_R / 8; ++rq)
#pragma unroll
            for (int cb = 0; cb < RTC_CH / 4; ++cb) {
              const uint32_t wv[4] = {q4[rq][cb].x, q4[rq][cb].y, q4[rq][cb].z, q4[rq][cb].w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t pb = __byte_perm(wv[q], 0, 0x3120);   // (lo0, lo1, hi0, hi1)
                slo = __dp2a_lo(wv[q], pb, slo);
                shi = __dp2a_hi(wv[q], pb, shi);
              }
            }
          tot[fk] += (u64)slo + ((u64)shi << 8);
          continue;
        }
#pragma unroll
        for (int rq = 0; rq < RTC_R / 8; ++rq) {   // fixed trip count: loads of all row blocks in flight
          const int rb = rq * 8;
          if (rb >= nrow) break;
          const int rr = rb + lr;
          const int pr = r_lo + rr;
          const int rc = pr < 2 ? pr : (pr >= g.ml ? pr - g.ml + 2 : 4);
          uint4 q4[RTC_CH / 4];
#pragma unroll
          for (int cb = 0; cb < RTC_CH / 4; ++cb) {
            const int ch = cb * 4 + lc;
            const int br = pr - 6 * gb;   // box row; its 16-byte chunk ch sits at ch ^ (row & 7)
            q4[cb] = (rr < nrow && ch < nch)
                         ? *reinterpret_cast<const uint4 *>(st + br * 128 + ((ch ^ (br & 7)) << 4))
                         : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int cb = 0; cb < RTC_CH / 4; ++cb) {
            const int ch = cb * 4 + lc;
            if (rr >= nrow || ch >= nch) continue;
            const int pc0 = 16 * j0 + 8 * ch - o;   // grid column of the chunk's first pixel
            const uint32_t wv[4] = {q4[cb].x, q4[cb].y, q4[cb].z, q4[cb].w};
            if (rc == 4 && pc0 > 1 && pc0 + 8 <= g.nl) {
              // interior chunk: eight squares, no masks (each pair of squares < 2^29)
              uint32_t sa = 0, sb = 0;
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                sa += (wv[q] & 0xffffu) * (wv[q] & 0xffffu) + (wv[q] >> 16) * (wv[q] >> 16);
                sb += (wv[q + 2] & 0xffffu) * (wv[q + 2] & 0xffffu) + (wv[q + 2] >> 16) * (wv[q + 2] >> 16);
              }
              tot[fk] += (u64)sa + sb;
              continue;
            }
            u64 t8 = 0;
            uint32_t sq[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) {
              const uint32_t v = (x & 1) ? (wv[x >> 1] >> 16) : (wv[x >> 1] & 0xffffu);
              const int c = pc0 + x;
              sq[x] = (c >= 0 && c < nl2) ? v * v : 0u;
              t8 += sq[x];
            }
            u64 c0 = 0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
            for (int x = 0; x < 8; ++x) {
              if (pc0 + x == 0) c0 = sq[x];
              if (pc0 + x == 1) c1 = sq[x];
              if (pc0 + x == g.nl) c2 = sq[x];
              if (pc0 + x == g.nl + 1) c3 = sq[x];
            }
            if (rc == 4) {
              tot[fk] += t8; e0[fk] += c0; e1[fk] += c1; e2[fk] += c2; e3[fk] += c3;
            } else {
              u64 *bn = bins + (f * 5 + rc) * 5;
              atomicAdd(reinterpret_cast<unsigned long long *>(bn + 0), (unsigned long long)t8);
              atomicAdd(reinterpret_cast<unsigned long long *>(bn + 1), (unsigned long long)c0);
              atomicAdd(reinterpret_cast<unsigned long long *>(bn + 2), (unsigned long long)c1);
              atomicAdd(reinterpret_cast<unsigned long long *>(bn + 3), (unsigned long long)c2);
              atomicAdd(reinterpret_cast<unsigned long long *>(bn + 4), (unsigned long long)c3);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
#if RTC_GA_TOTAL
#pragma unroll
    for (int fk = 0; fk < FPW; ++fk) {
      const int f = cw + fk * RTC_CW;
      const u64 t = warp_sum(tot[fk]);
      if (f < nf && lane == 0)
        atomicAdd(reinterpret_cast<unsigned long long *>(a.acc + (int64_t)Fid[f] * 18 + 9), (unsigned long long)t);
    }
    (void)e0; (void)e1; (void)e2; (void)e3;
#else
#pragma unroll
    for (int fk = 0; fk < FPW; ++fk) {
      const int f = cw + fk * RTC_CW;
      const u64 t = warp_sum(tot[fk]), a0 = warp_sum(e0[fk]), a1 = warp_sum(e1[fk]), a2 = warp_sum(e2[fk]),
                a3 = warp_sum(e3[fk]);
      if (f < nf && lane == 0) {
        u64 *bn = bins + (f * 5 + 4) * 5;
        atomicAdd(reinterpret_cast<unsigned long long *>(bn + 0), (unsigned long long)t);
        atomicAdd(reinterpret_cast<unsigned long long *>(bn + 1), (unsigned long long)a0);
        atomicAdd(reinterpret_cast<unsigned long long *>(bn + 2), (unsigned long long)a1);
        atomicAdd(reinterpret_cast<unsigned long long *>(bn + 3), (unsigned long long)a2);
        atomicAdd(reinterpret_cast<unsigned long long *>(bn + 4), (unsigned long long)a3);
      }
    }
#endif
  }

  // ---------------- epilogue: TMEM lane m = f*8 + r_rel; warp (m / 32) reads 32 lanes
  RT_T(const uint64_t t_main = gtimer() - t_beg;)
  mbar_wait(done, 0);
  RT_T(const uint64_t t_done = gtimer() - t_beg;)
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  RT_T(const uint64_t t_sync = gtimer() - t_beg; uint64_t t_tm = 0;)
  tc_fence_after();
  const int nsets_used = min(g.nsets, max(0, G1 - G0));
  if (warp >= 2 && warp < 6) {
    const int sw = warp & 3, m = sw * 32 + lane, ff = m >> 3, rr = m & 7;
    // w[t*3 + v'] = D_a + 2^8 D_b + 2^16 D_c of this row (all sets), compile-time indices
    u64 w[18];
#pragma unroll
    for (int c = 0; c < 18; ++c) w[c] = 0;
    for (int st = 0; st < nsets_used; ++st) {
#pragma unroll
      for (int cb = 0; cb < 4; cb += 2) {   // 32 columns per wait: n = cb*16 .. cb*16+31
        uint32_t x[32];
        tmem_ld16(taddr + ((uint32_t)(sw * 32) << 16) + (uint32_t)(st * 64 + cb * 16), *reinterpret_cast<uint32_t (*)[16]>(x));
        tmem_ld16(taddr + ((uint32_t)(sw * 32) << 16) + (uint32_t)(st * 64 + cb * 16 + 16),
                  *reinterpret_cast<uint32_t (*)[16]>(x + 16));
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const int n = cb * 16 + q;
          if (n < 54) w[n / 3] += (u64)x[q] << (8 * (n % 3));
        }
      }
    }
    // candidate (u', v') takes template row t = rr - u' of this grid row: branch-free selects
    u64 hp[9];
#pragma unroll
    for (int up = 0; up < 3; ++up) {
      const int t = rr - up;
#pragma unroll
      for (int vp = 0; vp < 3; ++vp) {
        u64 v = 0;
#pragma unroll
        for (int tt = 0; tt < 6; ++tt) v = (t == tt) ? w[tt * 3 + vp] : v;
        hp[up * 3 + vp] = v;
      }
    }
    RT_T(t_tm = gtimer() - t_beg;)
    // sum the 8 grid rows of the frame (lanes ff*8 .. ff*8+7 of this warp)
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      u64 v = hp[c];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      hp[c] = v;
    }
    if (rr == 0 && ff < nf) {
      u64 *acc = a.acc + (int64_t)Fid[ff] * 18;
#pragma unroll
      for (int c = 0; c < 9; ++c) atomicAdd(reinterpret_cast<unsigned long long *>(acc + c), (unsigned long long)hp[c]);
    }
  }
  RT_T(const uint64_t t_h = gtimer() - t_beg;)
  // GA per candidate from the bins: row classes of u' (0: rows 0,1,int; 1: 1,int,ml;
  // 2: int,ml,ml+1), minus the two grid columns outside [v', v'+nl) (0: nl,nl+1;
  // 1: 0,nl+1; 2: 0,1)
#if !RTC_GA_TOTAL
  for (int k = tid; k < RTC_F * 9; k += RTC_THREADS) {
    const int ff = k / 9, c = k % 9;
    if (ff >= nf) continue;
    const int up = c / 3, vp = c % 3;
    const int ex1 = vp == 0 ? 3 : 1, ex2 = vp == 2 ? 2 : 4;
    const u64 *bn = bins + ff * 25;
    u64 GA = 0;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int rc = up == 0 ? (q == 0 ? 0 : q == 1 ? 1 : 4) : up == 1 ? (q == 0 ? 1 : q == 1 ? 4 : 2)
                                                                         : (q == 0 ? 4 : q == 1 ? 2 : 3);
      GA += bn[rc * 5] - bn[rc * 5 + ex1] - bn[rc * 5 + ex2];
    }
    atomicAdd(reinterpret_cast<unsigned long long *>(a.acc + (int64_t)Fid[ff] * 18 + 9 + c), (unsigned long long)GA);
  }
#endif
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(taddr, tcols);
  RT_T(if (blockIdx.x < 3 && lane == 0 && warp < 4) printf("RTT cta %d warp %d nstage %d main %llu done %llu sync %llu tmem %llu h %llu total %llu wait %llu\n", blockIdx.x, warp, nstage, (unsigned long long)t_main, (unsigned long long)t_done, (unsigned long long)t_sync, (unsigned long long)t_tm, (unsigned long long)t_h, (unsigned long long)(gtimer() - t_beg), (unsigned long long)w_a);)
}

}  // namespace moco
