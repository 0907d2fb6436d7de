// kernels_tc.cuh -- exact coarse search on the 5th-gen tensor cores (tcgen05, kind::i8).
//
// The cross term of P:37, h(s,t) = sum_{(i,j) in D_{s,t}} a[i+s][j+t] b[i][j], is a
// dense contraction once written per template row i and frame column j' = j+t:
//
//     h(s,t) = sum_i sum_j' a[i+s][j'] * b[i][j'-t]        (a, b zero outside the image)
//
// For each PAIR of template rows (i, i+1) and each 32-column strip of j' this is one MMA
//     D[(s',f,pa), (d,pb,t)] += A[(s',f,pa), j'] * B[j', (d,pb,t)]
// with M rows = (A-row lag s', frame f, part pa) -- A is a sliding window over the
// frame's rows (row i+s'), addressed purely through the UMMA shared-memory descriptor,
// so the Hankel structure costs no data movement -- and N columns = (d, part pb, lag t):
// B is the Toeplitz expansion of template rows i (d = 0) and i+1 (d = 1), generated in
// shared memory per step.  Frame row i+s' meets template row i+1 at lag s'-1, so
//     h(s,t) = D[(s,.,.), (0,.,t)] + D[(s+1,.,.), (1,.,t)]
// (A-row lags s' in [-(w-1), w]).  Pairing halves the MMA instructions and the A-operand
// shared-memory reads per multiply-accumulate.
//
// Exactness: coarse values < 2^14 (bits + 2L <= 14) are split into two
// 7-bit parts v = 128*hi + lo, values < 2^16 into their two bytes (sb = 8), so every u8
// product is exact and every int32 accumulator (one product per template-row pair and
// column) stays below (2^sb - 1)^2 * ceil(m_c/2) * n_c < 2^31.  The epilogue recombines
// h = 2^(2 sb) D_hh + 2^sb (D_hl + D_lh) + D_ll in 64-bit integers, so
// N = g_a + g_b - 2h is EXACT and f = fl(N / (16^L A)) is bit-identical to the
// oracle's -- no certification step is needed.
//
//   K_prep  k_tc_prep    raw frames -> 2^L x 2^L block sums -> int8 hi/lo planes in the
//                        MMA operand layout (one HBM read of the frame), plus the frame
//                        energy table g_a for every coarse lag (strip/corner DP)
//   K_tc    k_tc_coarse  tcgen05 MMAs into TMEM, then epilogue: h, N, f, argmin (R4)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "kernels_direct.cuh"

namespace moco {

// ------------------------------------------------------------------ geometry
struct TcGeom {
  int mc, nc, w, hw, W, L;
  int F;        // frames per operand group (1, 2, 4): core matrix = 4/F rows x (F frames x 2 parts)
  int ST;       // lag rows s per 128-row M tile = 64 / F
  int NT;       // M tiles
  int Wt;       // t lags padded to a multiple of 8 (16 with MOCO_TC_WT16=1)
  int N1;       // columns per template row = 2 * Wt (parts x lags)
  int N;        // 2 * N1: a template-row pair
  int R;        // rows per operand plane = mc + NT*ST (plane row = frame row + hw)
  int nstrips;  // 32-column strips of j'
  int planeB;   // bytes per 16-column plane = R * 32 * F
  int stripB;   // 2 planes
  int TPAD, TP; // padded template parts: TP = nc + 2*TPAD bytes per row, zeros in the pads
  int SEGB;     // bytes of one template part row a strip's B tiles read: 32 + 2*TPAD
  int stg;      // 1: the producers build B tiles from a staged template band (no tile table)
  int nss;      // ring slots (= active producer warps): 7 when building, TC_TSLOTS when copying
  int sb;       // bits per operand part: 7 (coarse values < 2^14) or 8 (< 2^16)
  int TS;       // TMEM columns between accumulator tiles (N, or 256 when there is room)
  int ICH;      // template-row pairs per super-stage (one ring slot per producer warp)
  int ctas;     // CTAs per SM the geometry is sized for
  int npairs;   // ceil(mc / 2)
  int GG;       // operand groups per CTA
  int tmem_cols;
  int smem;     // dynamic shared memory bytes
  int prep_smem, prep_smem1;   // k_tc_prep dynamic shared memory: F frames / one frame per CTA
};

struct TcPlan {
  bool ready = false;
  bool tpl_ready = false;
  TcGeom g;
  int64_t cap = 0;          // frames per batch
  uint8_t *G = nullptr;     // operand planes for cap frames
  u64 *ga = nullptr;        // [cap][W*W] frame energies
  uint8_t *G2 = nullptr;    // second buffers: the prep of batch k+1 overlaps batch k
  u64 *ga2 = nullptr;
  uint8_t *T8 = nullptr;    // template parts [2][mc][nc]
  uint8_t *Btab = nullptr;  // the B tiles of every (strip, pair), built once per template (or null)
  // fused search (kernels_tcf.cuh, levels <= 1): layout and the corner-square scratch
  bool fused = false;
  int f_smem = 0, f_offE = 0, f_offBars = 0, f_nch = 0;
  u64 *corner = nullptr;    // [cap][4][w][w]
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// 16-byte LDGSTS (L1-bypassing) into shared memory, per-thread commit groups
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// Programmatic dependent launch (the closed-loop chain): let the next kernel of the stream
// be scheduled now, then wait until the previous one has completed and its writes are
// visible.  Both are no-ops for a kernel launched without the PDL attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t *holder, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(holder)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// D[tmem] (+)= A[smem] * B[smem], int8 x int8 -> int32, issued by one thread.
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-uniform variants: every lane executes the asm, one elected lane issues.
// Descriptors are passed as (low word, high word); only the low word (start
// address) changes inside the main loop.
__device__ __forceinline__ void mma_i8_elect(uint32_t tmem_d, uint32_t alo, uint32_t ahi, uint32_t blo,
                                             uint32_t bhi, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %7, 0;\n\t"
      "mov.b64 da, {%1, %2};\n\t"
      "mov.b64 db, {%3, %4};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %5, p;\n\t}" ::"r"(tmem_d),
      "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(0), "r"(accumulate)
      : "memory");
}
// Four MMAs sharing one B tile (the four operand groups of a template-row pair): one
// elect, one predicate, four issues -- a quarter of the per-MMA issue overhead.
__device__ __forceinline__ void mma_i8_x4_elect(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3, uint32_t a0,
                                                uint32_t a1, uint32_t a2, uint32_t a3, uint32_t ahi, uint32_t blo,
                                                uint32_t bhi, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 da0, da1, da2, da3, db;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %13, 0;\n\t"
      "mov.b64 da0, {%4, %8};\n\t"
      "mov.b64 da1, {%5, %8};\n\t"
      "mov.b64 da2, {%6, %8};\n\t"
      "mov.b64 da3, {%7, %8};\n\t"
      "mov.b64 db, {%9, %10};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], da0, db, %11, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%1], da1, db, %11, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%2], da2, db, %11, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%3], da3, db, %11, p;\n\t}" ::"r"(t0),
      "r"(t1), "r"(t2), "r"(t3), "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc),
      "r"(0), "r"(accumulate)
      : "memory");
}
// Two MMAs sharing one B tile (two M tiles of one operand group, C1-C3's geometry).
__device__ __forceinline__ void mma_i8_x2_elect(uint32_t t0, uint32_t t1, uint32_t a0, uint32_t a1, uint32_t ahi,
                                                uint32_t blo, uint32_t bhi, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 da0, da1, db;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %9, 0;\n\t"
      "mov.b64 da0, {%2, %4};\n\t"
      "mov.b64 da1, {%3, %4};\n\t"
      "mov.b64 db, {%5, %6};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], da0, db, %7, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%1], da1, db, %7, p;\n\t}" ::"r"(t0),
      "r"(t1), "r"(a0), "r"(a1), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(0), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, no swizzle: core matrices of 8 rows x 16 B
// (128 contiguous bytes); LBO = byte distance between the two 16-byte K halves,
// SBO = byte distance between consecutive 8-row groups; version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
// Instruction descriptor: u8 x u8 -> s32, K-major A and B, M=128, N.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// ---------------------------------------------------------------- K_prep
struct TcPrepArgs {
  const uint16_t *frames;   // level-0 frames, row pitch = n
  int64_t fstride;
  int n;                    // raw row pitch (elements)
  int B;                    // frames in this batch
  TcGeom g;
  uint8_t *G;               // [groups][nstrips][2][R][F][2][16]
  u64 *ga;                  // [B][W*W]
  int fp;                   // frames per CTA: g.F, or 1 (the CTA then fits beside the search)
  uint16_t *img1;           // L = 2: also write the level-1 image (2x2 sums) here, or null
  int64_t fs1;              // its frame stride and row pitch (elements)
  int p1;
};

// 8 consecutive coarse values (2^L x 2^L block sums) of one coarse row as 4 pair-words.
template <int L>
__device__ __forceinline__ void coarse8(const uint16_t *base, int n, uint32_t (&P)[4]) {
  if constexpr (L == 0) {
    const uint4 u = __ldcs(reinterpret_cast<const uint4 *>(base));
    P[0] = u.x; P[1] = u.y; P[2] = u.z; P[3] = u.w;
  } else {
    constexpr int bs = 1 << L, nv = bs;           // raw 16-byte vectors per raw row (8 bs samples)
    uint32_t s[4 * nv];                           // raw column pairs summed over the bs rows
#pragma unroll
    for (int k = 0; k < 4 * nv; ++k) s[k] = 0;
#pragma unroll
    for (int dy = 0; dy < bs; ++dy)
#pragma unroll
      for (int q = 0; q < nv; ++q) {
        const uint4 u = __ldcs(reinterpret_cast<const uint4 *>(base + (int64_t)dy * n + q * 8));
        s[4 * q + 0] += u.x; s[4 * q + 1] += u.y; s[4 * q + 2] += u.z; s[4 * q + 3] += u.w;   // halves < 2^14: no carry
      }
    if constexpr (L == 1) {
      // coarse values k, k+1 are the half sums of words s[k], s[k+1]: gather the low
      // halves and the high halves of the two words with one byte-permute each and add
      // (each half < 2^14: no carry into the other half)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        P[k] = __byte_perm(s[2 * k], s[2 * k + 1], 0x5410) + __byte_perm(s[2 * k], s[2 * k + 1], 0x7632);
      return;
    }
    // fold: coarse value k = both halves of its bs/2 raw pair words
    uint32_t c[8];
    constexpr int wpc = bs / 2;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t acc = 0;
#pragma unroll
      for (int j = 0; j < wpc; ++j) acc += (s[k * wpc + j] & 0xffffu) + (s[k * wpc + j] >> 16);
      c[k] = acc;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) P[k] = c[2 * k] | (c[2 * k + 1] << 16);
  }
}

// L = 2 with the level-1 image written on the way (replaces the separate level 0 -> 1
// downsample, which read the frames a second time): raw rows 0-1 and 2-3 of the 4-row band
// summed apart; level-1 value j of each row pair = both halves of pair word j (< 2^14);
// the 4x4 coarse value k = both halves of the sum of the two level-1 pair words 2k', 2k'+1
// (each half < 2^15, the coarse value < 2^16) -- the same sums, regrouped.
__device__ __forceinline__ void coarse8_l2_emit(const uint16_t *base, int n, uint16_t *o1, int p1,
                                                uint32_t (&P)[4]) {
  uint32_t sa[16], sb[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) sa[k] = sb[k] = 0;
#pragma unroll
  for (int dy = 0; dy < 4; ++dy)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 u = __ldcs(reinterpret_cast<const uint4 *>(base + (int64_t)dy * n + q * 8));
      uint32_t *s = dy < 2 ? sa : sb;
      s[4 * q + 0] += u.x; s[4 * q + 1] += u.y; s[4 * q + 2] += u.z; s[4 * q + 3] += u.w;
    }
  uint32_t wa[8], wb[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    wa[k] = __byte_perm(sa[2 * k], sa[2 * k + 1], 0x5410) + __byte_perm(sa[2 * k], sa[2 * k + 1], 0x7632);
    wb[k] = __byte_perm(sb[2 * k], sb[2 * k + 1], 0x5410) + __byte_perm(sb[2 * k], sb[2 * k + 1], 0x7632);
  }
  uint4 *ra = reinterpret_cast<uint4 *>(o1), *rb = reinterpret_cast<uint4 *>(o1 + p1);
  ra[0] = make_uint4(wa[0], wa[1], wa[2], wa[3]); ra[1] = make_uint4(wa[4], wa[5], wa[6], wa[7]);
  rb[0] = make_uint4(wb[0], wb[1], wb[2], wb[3]); rb[1] = make_uint4(wb[4], wb[5], wb[6], wb[7]);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t x0 = wa[2 * k] + wb[2 * k], x1 = wa[2 * k + 1] + wb[2 * k + 1];
    P[k] = __byte_perm(x0, x1, 0x5410) + __byte_perm(x0, x1, 0x7632);
  }
}

template <int L>
// One CTA per operand group of F frames.  Shared: per frame, edge-row and edge-column
// sums of a^2, the four (hw+1)^2 corner tables and the total.
#ifndef TC_PREP_RPP
#define TC_PREP_RPP 2
#endif
#ifndef TC_PREP_MINB
#define TC_PREP_MINB 4
#endif
__global__ void __launch_bounds__(256, TC_PREP_MINB) k_tc_prep(TcPrepArgs a) {
  const TcGeom &g = a.g;
  extern __shared__ __align__(16) unsigned char smem[];
  const int F = g.F, FP = a.fp, hw = g.hw, w = g.w, mc = g.mc, nc = g.nc, W = g.W;
  const int CS = w * w;                       // corner table size per quad (index 0 = empty)
  u64 *rowE = reinterpret_cast<u64 *>(smem);  // [FP][2*hw]  top rows 0..hw-1, bottom rows from the bottom
  u64 *colE = rowE + FP * 2 * hw;             // [FP][2*hw]
  u64 *cor = colE + FP * 2 * hw;              // [FP][4][w][w]
  u64 *tot = cor + FP * 4 * CS;               // [FP]
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int k = tid; k < FP * (4 * hw + 4 * CS + 1); k += nth) rowE[k] = 0;
  __syncthreads();
  // warp = one (frame, plane row) item at a time, lanes = 8-column chunks of the coarse
  // row: every load instruction reads 512 contiguous bytes of a raw row (L >= 1 folds
  // 2^L raw rows); energies: row sums by warp reduction, edge columns by atomics on
  // distinct addresses, corner tables by plain stores
  const int warp = tid >> 5, lane = tid & 31, nwarp = nth >> 5;
  const int nchunk = nc >> 3;
  // FP (frames per CTA: F, or 1 so that a CTA fits beside the search kernel) divides the
  // warp count, so a warp always works on the same frame fl = warp % FP; edge-column
  // energies accumulate in registers (a lane owns at most one left-edge and one
  // right-edge chunk) and are added to shared memory once at the end.  The operand
  // planes keep the search's layout: group grp = fi / F, slot f = fi % F.
  const int fl = warp % FP;
  const int fi = (int)blockIdx.x * FP + fl;
  const int grp = fi / F, f = fi - grp * F;
  const uint16_t *frame = a.frames + (int64_t)(fi < a.B ? fi : 0) * a.fstride;
  // this warp's edge-column sums (left hw, right hw), owned by the warp: no atomics
  u64 *ce = tot + FP + warp * 2 * hw;
  for (int k = lane; k < 2 * hw; k += 32) ce[k] = 0;
  __syncwarp();
  u64 ftot = 0;
  // coarse rows of <= 256 values: each lane owns one 8-column chunk, so its edge-column
  // squares (< 2^28 each: coarse values < 2^14) accumulate in 32-bit registers and are
  // flushed to the warp's shared sums every 16 rows
  const bool one_chunk = nchunk <= 32 && g.sb == 7;   // 32-bit edge accumulators: 14-bit values only
  uint32_t eacc[8];
#pragma unroll
  for (int x = 0; x < 8; ++x) eacc[x] = 0;
  auto flush_edges = [&]() {
    const int c0 = lane * 8;
    if (lane < nchunk && (c0 < hw || c0 + 8 > nc - hw)) {
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const int c = c0 + x;
        if (c < hw) ce[c] += eacc[x];
        if (c >= nc - hw) ce[hw + (nc - 1 - c)] += eacc[x];
        eacc[x] = 0;
      }
    }
  };
  auto item = [&](int pr, const uint32_t (&P)[4], int cc, bool live, u64 &rs) {
    const int cr = pr - hw;
    // parts of g.sb bits (7: v = 128 hi + lo; 8: the two bytes of a 16-bit coarse value)
    const uint32_t pm = g.sb == 7 ? 0x007F007Fu : 0x00FF00FFu, sb = (uint32_t)g.sb;
    const uint32_t h0 = (P[0] >> sb) & pm, h1 = (P[1] >> sb) & pm;
    const uint32_t h2 = (P[2] >> sb) & pm, h3 = (P[3] >> sb) & pm;
    const uint2 hi = make_uint2(__byte_perm(h0, h1, 0x6420), __byte_perm(h2, h3, 0x6420));
    const uint2 lo = make_uint2(__byte_perm(P[0] & pm, P[1] & pm, 0x6420),
                                __byte_perm(P[2] & pm, P[3] & pm, 0x6420));
    uint8_t *dst = a.G + ((((int64_t)grp * g.nstrips + (cc >> 2)) * 2 + ((cc >> 1) & 1)) * g.R + pr) * (32 * F) +
                   f * 32 + (cc & 1) * 8;
    *reinterpret_cast<uint2 *>(dst) = hi;
    *reinterpret_cast<uint2 *>(dst + 16) = lo;
    if (!live) return;
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) { v[2 * k] = P[k] & 0xffffu; v[2 * k + 1] = P[k] >> 16; }
    if (g.sb == 7) {
      uint32_t cs = 0;
#pragma unroll
      for (int x = 0; x < 8; ++x) cs += v[x] * v[x];   // 8 terms < 2^28: < 2^31
      rs += cs;
    } else {
#pragma unroll
      for (int x = 0; x < 8; ++x) rs += (u64)(v[x] * v[x]);   // each < 2^32
    }
    const int c0 = cc * 8;
    const bool eL = c0 < hw, eR = c0 + 8 > nc - hw;
    if (!(eL || eR)) return;
    if (one_chunk) {
#pragma unroll
      for (int x = 0; x < 8; ++x) eacc[x] += v[x] * v[x];
    } else {
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const int c = c0 + x;
        const u64 v2 = (u64)(v[x] * v[x]);
        if (c < hw) ce[c] += v2;                        // distinct columns per lane
        if (c >= nc - hw) ce[hw + (nc - 1 - c)] += v2;
      }
    }
    const bool top = cr < hw, bot = cr >= mc - hw;
    if (!(top || bot)) return;
    for (int x = 0; x < 8; ++x) {   // corner tables of the DP: plain stores
      const int c = c0 + x;
      const bool lf = c < hw, rt = c >= nc - hw;
      const u64 v2 = (u64)(v[x] * v[x]);
      for (int qb = 0; qb < 2; ++qb) {
        if (!(qb ? bot : top)) continue;
        const int pp = qb ? mc - cr : cr + 1;
        for (int qr = 0; qr < 2; ++qr) {
          if (!(qr ? rt : lf)) continue;
          const int qq = qr ? nc - c : c + 1;
          cor[((fl * 4) + (qb * 2 + qr)) * CS + pp * w + qq] = v2;
        }
      }
    }
  };
  auto row_done = [&](int pr, bool live, u64 rs) {
    if (!live) return;
    const int cr = pr - hw;
    rs = warp_sum(rs);
    if (lane == 0) {
      ftot += rs;
      if (cr < hw) rowE[fl * 2 * hw + cr] = rs;
      if (cr >= mc - hw) rowE[fl * 2 * hw + hw + (mc - 1 - cr)] = rs;
    }
  };
  // plane rows pr = warp / F, + nwarp / F, ...; TC_PREP_RPP rows per pass (loads first)
  const int pstep = nwarp / FP;
  int nrows = 0;
  for (int pr0 = warp / FP; pr0 < g.R; pr0 += TC_PREP_RPP * pstep) {
    if (one_chunk && nrows + TC_PREP_RPP > 16) {   // <= 16 rows of squares per flush
      flush_edges();
      nrows = 0;
    }
    nrows += TC_PREP_RPP;
    bool live[TC_PREP_RPP];
    u64 rs[TC_PREP_RPP];
#pragma unroll
    for (int q = 0; q < TC_PREP_RPP; ++q) {
      const int pr = pr0 + q * pstep;
      live[q] = fi < a.B && pr < g.R && pr - hw >= 0 && pr - hw < mc;
      rs[q] = 0;
    }
    for (int cc = lane; cc < nchunk; cc += 32) {
      uint32_t P[TC_PREP_RPP][4];
#pragma unroll
      for (int q = 0; q < TC_PREP_RPP; ++q) {
        const int pr = pr0 + q * pstep;
        P[q][0] = P[q][1] = P[q][2] = P[q][3] = 0;
        if (!live[q]) continue;
        const uint16_t *src = frame + (int64_t)((pr - hw) << L) * a.n + ((cc * 8) << L);
        if constexpr (L == 2) {
          if (a.img1)
            coarse8_l2_emit(src, a.n, a.img1 + (int64_t)fi * a.fs1 + (int64_t)(2 * (pr - hw)) * a.p1 + cc * 16, a.p1,
                            P[q]);
          else
            coarse8<L>(src, a.n, P[q]);
        } else {
          coarse8<L>(src, a.n, P[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < TC_PREP_RPP; ++q) {
        const int pr = pr0 + q * pstep;
        if (pr < g.R) item(pr, P[q], cc, live[q], rs[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < TC_PREP_RPP; ++q) {
      const int pr = pr0 + q * pstep;
      if (pr < g.R) row_done(pr, live[q], rs[q]);
    }
  }
  // flush this warp's edge-column and total energies
  if (one_chunk) flush_edges();
  __syncwarp();
  for (int k = lane; k < 2 * hw; k += 32) atomicAdd(&colE[fl * 2 * hw + k], ce[k]);
  if (lane == 0) atomicAdd(&tot[fl], ftot);
  __syncthreads();
  // prefix sums: edge strips (1-D), corners (2-D, the DP of P:35 in each corner)
  for (int k = tid; k < FP * 4; k += nth) {
    u64 *e = (k & 2) ? colE : rowE;
    u64 *p = e + (k >> 2) * 2 * hw + (k & 1) * hw;
    for (int q = 1; q < hw; ++q) p[q] += p[q - 1];
  }
  for (int k = tid; k < FP * 4 * w; k += nth) {
    u64 *c = cor + (k / w) * CS + (k % w) * w;
    for (int q = 1; q < w; ++q) c[q] += c[q - 1];
  }
  __syncthreads();
  for (int k = tid; k < FP * 4 * w; k += nth) {
    u64 *c = cor + (k / w) * CS + (k % w);
    for (int p = 1; p < w; ++p) c[p * w] += c[(p - 1) * w];
  }
  __syncthreads();
  for (int k = tid; k < FP * W * W; k += nth) {
    const int f = k / (W * W), lag = k % (W * W);
    const int fi = (int)blockIdx.x * FP + f;
    if (fi >= a.B) continue;
    const int s = lag / W - hw, t = lag % W - hw;
    const u64 *re = rowE + f * 2 * hw, *ce = colE + f * 2 * hw;
    // rows of the frame outside the frame-side rectangle of D_{s,t}:
    // top s rows when s > 0, bottom |s| rows when s < 0 (likewise columns for t)
    const u64 rex = s > 0 ? re[s - 1] : (s < 0 ? re[hw + (-s) - 1] : 0);
    const u64 cex = t > 0 ? ce[t - 1] : (t < 0 ? ce[hw + (-t) - 1] : 0);
    u64 corner = 0;
    if (s != 0 && t != 0) {
      const int quad = (s < 0 ? 2 : 0) | (t < 0 ? 1 : 0);
      corner = cor[(f * 4 + quad) * CS + abs(s) * w + abs(t)];
    }
    a.ga[(int64_t)fi * W * W + lag] = tot[f] - rex - cex + corner;
  }
}

// ---------------------------------------------------------------- K_tc
struct TcArgs {
  const uint8_t *G;
  const uint8_t *T8;     // template parts [2][mc][nc]
  const uint8_t *Btab;   // [nstrips][npairs][N*32] precomputed B tiles, or null: built by the producers
  const u64 *ga;         // [B][W*W]
  const u64 *gb;         // [W*W]
  TcGeom g;
  double scale;          // 16^L
  int B;
  int32_t *shift_out;    // [B][2] or null
  double *f_out;         // [B] or null
  uint8_t *flags;        // [B] or null
  double *grid_out;      // [B][W*W] or null: f for every coarse lag
};

// One CTA = GG operand groups (GG*F frames), warp-specialised, no block barrier in
// the main loop.  Work is handed over in super-stages of ICH consecutive template
// rows (ICH B tiles): one full/empty mbarrier handshake per super-stage.  Super-stage
// u is built by producer p = u mod 7 into ITS OWN ring slot p: every barrier is then
// waited on in phase order by exactly one producer and by the MMA warp, so a parity
// wait can never alias a phase two completions away.
//   warp 0           MMA issuer (warp-uniform loop, one elected lane issues): per
//                    32-column strip one bulk copy per group, then per super-stage
//                    wait full[ss], issue ICH*GG*NT MMAs, commit to empty[ss];
//   warps 1..7       producers: warp p builds super-stages u == p-1 (mod 7) straight
//                    from the zero-padded template parts in global memory (L1/L2
//                    resident), then arrives on full[ss].
// Producers depend only on the template, so they run up to NSS super-stages ahead,
// across strip boundaries; the strip reload stall is covered by the second CTA on
// the SM.
#ifdef MOCO_TC_TIMING   // debug builds only: per-CTA phase times, printed for a few CTAs
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TC_T(...) __VA_ARGS__
#else
#define TC_T(...)
#endif
constexpr int TC_THREADS = 256;
constexpr int TC_PRODUCERS = 7;
constexpr int TC_TSLOTS = 4;   // ring slots with the B-tile table (copies are cheap; fewer slots, larger super-stages)

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

template <int CPL>   // B chunks (16 bytes) per producer lane per tile = 2N/32
__global__ void __launch_bounds__(TC_THREADS, 3) k_tc_coarse(TcArgs a) {   // <= 85 registers: 3 CTAs/SM fit
  const TcGeom &g = a.g;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int F = g.F, hw = g.hw, mc = g.mc, nc = g.nc, N = g.N, N1 = g.N1, NT = g.NT, GG = g.GG;
  const int NSS = g.nss;                                       // one ring slot per active producer warp
  const int ICH = g.ICH;
  unsigned char *As = smem;                                   // [GG] strips of 2 planes
  unsigned char *Bring = As + GG * g.stripB;                  // [NSS][ICH][N*32]
  const int SEGB = g.SEGB, PAIRB = 4 * SEGB;
  unsigned char *Stg = Bring + NSS * ICH * N * 32;            // [NSS][2][ICH][pb][d][SEGB] (g.stg only)
  uint64_t *bars = reinterpret_cast<uint64_t *>(Stg + (g.stg ? NSS * 2 * ICH * PAIRB : 0));
  uint64_t *full = bars, *empty = bars + NSS, *aload = bars + 2 * NSS;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 2 * NSS + 1);
  const int grp0 = blockIdx.x * GG;
  const int ngroups = (a.B + F - 1) / F;
  const int gcount = min(GG, ngroups - grp0);
  const int per_strip = g.npairs / ICH;
  const int nsuper = g.nstrips * per_strip;

  TC_T(const uint64_t t_start = gtimer(); const long long c_start = clock64(); uint64_t w_strip = 0, w_full = 0, w_empty = 0, t_issue = 0;)
  if (warp == 0) tmem_alloc(tmem_holder, g.tmem_cols);
  if (tid == 0) {
    for (int s = 0; s < NSS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(aload, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = *tmem_holder;

  if (warp == 0) {
    // ---------------- MMA issuer (whole warp walks the loop, warp-uniform; the
    // elect is inside the asm so no per-instruction ELECT loop is generated)
    const uint32_t idesc = idesc_i8(128, N);
    const uint64_t bd0 = umma_desc(smem_u32(Bring), 128, 256);
    const uint64_t ad0 = umma_desc(smem_u32(As), g.planeB, 128);
    const uint32_t blo0 = (uint32_t)bd0, bhi = (uint32_t)(bd0 >> 32);
    const uint32_t alo0 = (uint32_t)ad0, ahi = (uint32_t)(ad0 >> 32);
    const uint32_t rowstep = (32u * F) >> 4;         // descriptor units per plane row
    const uint32_t tilestep = (uint32_t)(N * 32) >> 4;
    const uint32_t sstep = (uint32_t)ICH * tilestep;
    // per-MMA (group gg, M tile k) A offsets and TMEM columns, j = gg*NT + k < 4
    const int ntg = gcount * NT;
    uint32_t aoff[4], tcol[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gg = j / NT, k = j % NT;
      aoff[j] = (uint32_t)(gg * g.stripB >> 4) + (uint32_t)(k * g.ST) * rowstep;
      tcol[j] = taddr + (uint32_t)(j * g.TS);
    }
    if (elect_one()) {   // the epilogue's frame energies: HBM -> L2 while the MMAs run
      const uintptr_t b0 = (uintptr_t)(a.ga + (int64_t)grp0 * F * g.W * g.W) & ~(uintptr_t)15;
      const uintptr_t b1 = (uintptr_t)(a.ga + (int64_t)min((grp0 + gcount) * F, a.B) * g.W * g.W) & ~(uintptr_t)15;
      if (b1 > b0) bulk_prefetch_l2(reinterpret_cast<const void *>(b0), (uint32_t)(b1 - b0));
    }
    __syncwarp();
    const int nst = g.nstrips;
    int ss = 0, round = 0;              // slot (= producer) and slot use of the super-stage
    int pss = NSS - 1, pround = -1;     // of the previous super-stage
    for (int st = 0; st < nst; ++st) {
      TC_T(uint64_t t0 = gtimer();)
      if (st > 0) mbar_wait(&empty[pss], pround & 1);   // strip buffers free
      TC_T(w_empty += gtimer() - t0;)
      if (elect_one()) {
        mbar_arrive_expect_tx(aload, (uint32_t)(gcount * g.stripB));
        for (int gg = 0; gg < gcount; ++gg)
          bulk_g2s(As + gg * g.stripB, a.G + ((int64_t)(grp0 + gg) * nst + st) * g.stripB,
                   (uint32_t)g.stripB, aload);
        // the next strip streams from HBM into L2 while this one is multiplied
        if (st + 1 < nst)
          for (int gg = 0; gg < gcount; ++gg)
            bulk_prefetch_l2(a.G + ((int64_t)(grp0 + gg) * nst + st + 1) * g.stripB, (uint32_t)g.stripB);
      }
      __syncwarp();
      TC_T(t0 = gtimer();)
      mbar_wait(aload, st & 1);
      TC_T(w_strip += gtimer() - t0;)
      tc_fence_after();
      uint32_t arow = alo0;             // A descriptor low word at the pair's first template row
      for (int u = 0; u < per_strip; ++u) {
        TC_T(t0 = gtimer();)
        mbar_wait(&full[ss], round & 1);
        TC_T(w_full += gtimer() - t0;)
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
        __syncwarp();
        pss = ss;
        pround = round;
        if (++ss == NSS) { ss = 0; ++round; }
      }
    }
    TC_T(t_issue = gtimer();)
  } else {
    // ---------------- B producers: tile of pair (i, i+1), row n = (d, pb, t)
    const int p = warp - 1;
    int srcoff[CPL];
    uint32_t live = 0;
    // chunk c of this lane: row n = (lane&7) + 8*(lane>>4) + 16c, half h = (lane>>3)&1,
    // 512 bytes apart; each 8-lane phase of a 16-byte store covers all 32 banks
    const int dst0 = (lane >> 4) * 256 + ((lane >> 3) & 1) * 128 + (lane & 7) * 16;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int n = (lane & 7) + 8 * (lane >> 4) + 16 * q, h = (lane >> 3) & 1;
      const int d = n >= N1 ? 1 : 0, r = n - d * N1;
      const int pb = r >= g.Wt ? 1 : 0, ti = r - pb * g.Wt;
      if (ti < g.W) live |= 1u << q;
      // bytes b_pb[i+d][J0 + 16h - t + x], x = 0..15, from the 4-aligned word below
      const int col = 16 * h - (ti - hw) + g.TPAD;          // in the staged band [J0, J0 + SEGB)
      srcoff[q] = (pb * 2 + d) * SEGB + col;
    }
    int st = p / per_strip, i0 = (p % per_strip) * ICH;   // strip, first pair of the super-stage
    const int ss = p;
    if (a.Btab) {
      // B tiles precomputed per template: one bulk copy of the super-stage's ICH tiles
      const uint32_t bytes = (uint32_t)(ICH * N * 32);
      int round = 0;
      for (int u = p; p < NSS && u < nsuper; u += NSS, ++round) {
        if (round > 0) mbar_wait(&empty[ss], (round - 1) & 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[ss], bytes);
          bulk_g2s(Bring + ss * ICH * N * 32, a.Btab + ((int64_t)st * g.npairs + i0) * (N * 32), bytes, &full[ss]);
        }
        __syncwarp();
        i0 += NSS * ICH;
        while (i0 >= g.npairs) { i0 -= g.npairs; ++st; }
      }
    } else {
    // The band of template-part rows a super-stage reads (ICH pairs x 2 parts x 2 rows x
    // SEGB bytes) is staged in shared memory with LDGSTS one super-stage ahead: the tile
    // build then waits on shared-memory latency only (the T8 band of a strip does not
    // stay L1-resident next to the strips and the ring, so direct loads went to L2).
    unsigned char *stg = Stg + p * 2 * ICH * PAIRB;
    const int nchunk = ICH * PAIRB / 16, segc = SEGB / 16;
    auto stage_band = [&](int st_, int i0_, unsigned char *dst) {
      for (int k = lane; k < nchunk; k += 32) {
        const int q = k / (4 * segc), r = k % (4 * segc);
        const int seg = r / segc, c16 = r % segc;   // seg = pb*2 + d
        const uint8_t *src = a.T8 + (int64_t)(seg >> 1) * (mc + 2) * g.TP +
                             (int64_t)(2 * (i0_ + q) + (seg & 1)) * g.TP + st_ * 32 + c16 * 16;
        cp_async16(dst + q * PAIRB + seg * SEGB + c16 * 16, src);
      }
      cp_async_commit();
    };
    stage_band(st, i0, stg);
    int round = 0;
    for (int u = p; u < nsuper; u += TC_PRODUCERS, ++round) {
      // next super-stage of this warp: TC_PRODUCERS super-stages later
      int nst = st, ni0 = i0 + TC_PRODUCERS * ICH;
      while (ni0 >= g.npairs) { ni0 -= g.npairs; ++nst; }
      unsigned char *cur = stg + (round & 1) * ICH * PAIRB;
      __syncwarp();   // every lane is done reading the other buffer (previous round)
      if (u + TC_PRODUCERS < nsuper) stage_band(nst, ni0, stg + ((round + 1) & 1) * ICH * PAIRB);
      else cp_async_commit();
      if (round > 0) mbar_wait(&empty[ss], (round - 1) & 1);
      cp_async_wait<1>();
      __syncwarp();
      unsigned char *Bs = Bring + ss * ICH * N * 32;
#ifdef MOCO_TC_NOPROD   // timing experiments: MMAs on stale B tiles
      for (int q = 0; q < 0; ++q) {
#else
      for (int q = 0; q < ICH; ++q) {
#endif
        const unsigned char *rowbase = cur + q * PAIRB;
        unsigned char *Bt = Bs + q * N * 32 + dst0;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const uint32_t *wp = reinterpret_cast<const uint32_t *>(rowbase + (srcoff[c] & ~3));
          const uint32_t sh = (srcoff[c] & 3) * 8;
          uint4 outv = make_uint4(0, 0, 0, 0);
          if ((live >> c) & 1u) {
            const uint32_t w0 = wp[0], w1 = wp[1], w2 = wp[2], w3 = wp[3], w4 = wp[4];
            outv.x = __funnelshift_r(w0, w1, sh);
            outv.y = __funnelshift_r(w1, w2, sh);
            outv.z = __funnelshift_r(w2, w3, sh);
            outv.w = __funnelshift_r(w3, w4, sh);
          }
          *reinterpret_cast<uint4 *>(Bt + c * 512) = outv;
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[ss]);
      st = nst;
      i0 = ni0;
    }
    cp_async_wait<0>();
    }
  }
  // all MMAs done -> accumulators final.  Every warp must be converged before the
  // .sync.aligned TMEM loads (threads can leave the mbarrier spin at different times).
  {
    const int last = nsuper - 1;
    mbar_wait(&empty[last % NSS], (last / NSS) & 1);
  }
  __syncwarp();
  TC_T(const uint64_t t_mma = gtimer(); const long long c_mma = clock64();)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // ---- epilogue: h -> N -> f -> argmin (S4), per frame.  Warp w reads TMEM lanes
  // 32*(w%4).. of the tiles of groups gg = w/4, w/4 + 2, ...  Per 16-column chunk the
  // d = 1 halves are first staged in shared memory (the strips are free now), so each
  // row can add its partner row s'+1 (next lane block, or the next M tile).
  const int W = g.W;
  const int m = (warp & 3) * 32 + lane;     // accumulator row = TMEM lane
  const int sl = m / (2 * F), rho = m % (2 * F);
  const int f = rho >> 1, pa = rho & 1;
  // [GG*NT][128][33 words]: (pb hi 16 | pb lo 16), rows padded to 33 words so the 32
  // lanes (consecutive rows) of a warp hit 32 different banks
  uint32_t *D1s = reinterpret_cast<uint32_t *>(smem);
  Key *keys = reinterpret_cast<Key *>(smem + GG * NT * 128 * 33 * 4);
  // the frame energies of this CTA's frames, staged once with coalesced loads (per-lag
  // loads straight from global memory, one row s per lane, were the epilogue's cost)
  u64 *gas = reinterpret_cast<u64 *>(keys + GG * 128);
  const int64_t fi0 = (int64_t)grp0 * F;
  {
    const int64_t nga = (int64_t)min(gcount * F, a.B - (int)fi0) * W * W;
    const u64 *src = a.ga + fi0 * W * W;
    for (int64_t k = tid; k < nga; k += TC_THREADS) gas[k] = src[k];
  }
  __syncthreads();
  Key best[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) best[q] = Key{~0ull, ~0u};
  for (int c = 0; c < g.Wt; c += 16) {
    // stage the d = 1 columns of this chunk
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
      const int fi = (grp0 + gg) * F + f;
      Key bk = best[q];
      for (int k = 0; k < NT; ++k) {
        const int s = -hw + k * g.ST + sl;
        // both rows of the (hi, lo) lane pair evaluate lags: hi lane the first 8 columns of
        // the chunk, lo lane the last 8 (each has the pair's four part sums after the swap)
        const bool valid = gg < gcount && s <= hw && fi < a.B;
        // partner row s' = s + 1: same tile, 2F lanes further, or the next tile's first block
        const int mp = sl + 1 < g.ST ? m + 2 * F : m + 2 * F - 128;
        const int kp = sl + 1 < g.ST ? k : k + 1;
        const bool haveP = kp < NT;   // s + 1 <= hw + 1 always lies inside the NT*ST lag rows
        uint32_t xh[16], xl[16];
        const uint32_t tbase = taddr + ((uint32_t)((warp & 3) * 32) << 16) + (gg * NT + k) * g.TS;
        tmem_ld16(tbase + c, xh);             // d = 0, pb = hi
        tmem_ld16(tbase + g.Wt + c, xl);      // d = 0, pb = lo
        tmem_wait_ld();
        const uint32_t *src = D1s + ((gg * NT + (haveP ? kp : 0)) * 128 + (haveP ? mp : 0)) * 33;
        if (haveP) {
#pragma unroll
          for (int qq = 0; qq < 16; ++qq) { xh[qq] += src[qq]; xl[qq] += src[16 + qq]; }   // each < 2^31: no wrap
        }
        // the (hi, lo) lane pair splits the chunk: iteration j, hi lane column j, lo lane
        // column j+8; each sends its partner the part sums of the partner's column
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t mh = pa ? xh[j + 8] : xh[j], ml = pa ? xl[j + 8] : xl[j];
          const uint32_t ph = __shfl_xor_sync(0xffffffffu, pa ? xh[j] : xh[j + 8], 1);
          const uint32_t pl = __shfl_xor_sync(0xffffffffu, pa ? xl[j] : xl[j + 8], 1);
          const int ti = c + j + (pa ? 8 : 0);
          if (!valid || ti >= W) continue;
          const int sb = g.sb;   // h = 2^(2 sb) D_hh + 2^sb (D_hl + D_lh) + D_ll
          const u64 h = pa == 0 ? ((u64)mh << (2 * sb)) + (((u64)ml + (u64)ph) << sb) + (u64)pl
                                : ((u64)ph << (2 * sb)) + (((u64)pl + (u64)mh) << sb) + (u64)ml;
          const int lag = (s + hw) * W + ti;
          const u64 Nn = gas[(fi - fi0) * W * W + lag] + a.gb[lag] - 2 * h;
          const int t = ti - hw;
          const double area = (double)((mc - abs(s)) * (nc - abs(t)));
          const double fv = (double)Nn / (a.scale * area);
          if (a.grid_out) a.grid_out[(int64_t)fi * W * W + lag] = fv;
          const Key kk{(u64)__double_as_longlong(fv), (unsigned)lag};
          if (key_less(kk, bk)) bk = kk;
        }
      }
      best[q] = bk;
    }
    __syncthreads();   // D1s is restaged by the next chunk
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
      for (int q = 2 * ff; q < 128; q += 2 * F) {   // both lanes of each row pair
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
  TC_T(if (tid == 0 && (blockIdx.x % 149 == 0)) printf("TCT cta %d mma_cycles %lld total %llu mma_done %llu issue_end %llu wait_strip %llu wait_full %llu wait_empty %llu\n", blockIdx.x, c_mma - c_start, (unsigned long long)(gtimer() - t_start), (unsigned long long)(t_mma - t_start), (unsigned long long)(t_issue - t_start), (unsigned long long)w_strip, (unsigned long long)w_full, (unsigned long long)w_empty);)
}

// The B tile of every (strip st, pair i), as the producers would build it: row n = (d,
// pb, t), half h: bytes T8[pb][2i+d][TPAD + 32 st + 16h - (t - hw) + x], zero rows for
// t >= W; core-matrix layout (n>>3)*256 + h*128 + (n&7)*16.
__global__ void k_tc_btab(const uint8_t *__restrict__ T8, TcGeom g, uint8_t *__restrict__ tab) {
  const int tile = g.N * 32;
  const int64_t total = (int64_t)g.nstrips * g.npairs * tile;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int off = (int)(e % tile);
    const int64_t ti_ = e / tile;
    const int st = (int)(ti_ / g.npairs), i = (int)(ti_ % g.npairs);
    const int n = (off >> 8) * 8 + ((off & 127) >> 4), h = (off >> 7) & 1, x = off & 15;
    const int d = n >= g.N1 ? 1 : 0, r = n - d * g.N1;
    const int pb = r >= g.Wt ? 1 : 0, t = r - pb * g.Wt;
    uint8_t v = 0;
    if (t < g.W)
      v = T8[(int64_t)pb * (g.mc + 2) * g.TP + (int64_t)(2 * i + d) * g.TP + 32 * st + 16 * h - (t - g.hw) + g.TPAD + x];
    tab[e] = v;
  }
}

// template parts for the B operand, zero-padded rows: T8[pb][i][TPAD + j] =
// (b >> sb, b & (2^sb - 1))[pb] for j in [0, nc), 0 in the pads
__global__ void k_tc_template(const uint16_t *__restrict__ b, int pitch, int mc, int nc, int TPAD, int TP, int sb,
                              uint8_t *T8) {
  const int rows = mc + 2;   // zero rows past the template (second row of an odd-mc pair)
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 2 * rows * TP; e += gridDim.x * blockDim.x) {
    const int pb = e / (rows * TP), r = e % (rows * TP);
    const int i = r / TP, j = r % TP - TPAD;
    uint8_t v = 0;
    if (j >= 0 && j < nc && i < mc) {
      const uint32_t x = b[(int64_t)i * pitch + j];
      v = (uint8_t)(pb == 0 ? (x >> sb) : (x & ((1u << sb) - 1u)));
    }
    T8[e] = v;
  }
}

// ---------------------------------------------------------------- host side
inline bool tc_make_geom(TcGeom *gp, int w, int mc, int nc, int L, int vb) {
  TcGeom g{};
  g.mc = mc; g.nc = nc; g.w = w; g.hw = w - 1; g.W = 2 * w - 1; g.L = L;
  g.sb = vb <= 14 ? 7 : 8;
  // t lags padded to a multiple of 8 (N = 4 Wt: a multiple of 32, so N/16 producer chunks
  // per lane is one of the even instantiations); the epilogue reads 16-column chunks past
  // Wt, inside the TMEM allocation and ignored.  MOCO_TC_WT16=1: pad to 16 (round 1)
  const char *w16 = getenv("MOCO_TC_WT16");
  g.Wt = (w16 && atoi(w16)) ? (g.W + 15) / 16 * 16 : (g.W + 7) / 8 * 8;
  g.N1 = 2 * g.Wt;
  g.N = 2 * g.N1;
  if (g.N > 256) return false;
  const int lagrows = g.W + 1;   // A-row lags s' in [-(w-1), w]
  // One CTA per SM by default (measured on B200: more operand groups per
  // CTA -- each B tile feeds more MMAs -- beat two CTAs overlapping their strip loads).
  const char *ce = getenv("MOCO_TC_CTAS");   // tuning experiments: CTAs per SM target
  const int ctas = ce ? std::max(1, atoi(ce)) : 1;
  const int smem_cap = (228 * 1024) / ctas - 1024, tmem_cap = 512 / ctas;
  // frames per group: the fewest padded lag rows with NT*N within TMEM; ties -> F = 1
  // (measured with B tiles from the per-template table: C1 1.027 -> 1.048 M, C3 868 -> 921 k
  // frames/s over F = 2)
  int bestF = 0, bestRows = 1 << 30;
  const char *fe = getenv("MOCO_TC_F");   // tuning experiments
  for (int F : {1, 2, 4}) {
    if (fe && atoi(fe) != F) continue;
    const int ST = 64 / F, NT = (lagrows + ST - 1) / ST;
    if (NT * g.N > tmem_cap) continue;
    if (NT * ST < bestRows) { bestRows = NT * ST; bestF = F; }
  }
  if (!bestF) return false;
  g.F = bestF; g.ST = 64 / g.F; g.NT = (lagrows + g.ST - 1) / g.ST;
  g.R = mc + g.NT * g.ST;
  g.nstrips = (nc + 31) / 32;
  g.planeB = g.R * 32 * g.F;
  g.stripB = 2 * g.planeB;
  g.TPAD = (g.hw + 8 + 15) / 16 * 16;
  g.TP = nc + 2 * g.TPAD;
  g.npairs = (mc + 1) / 2;
  g.SEGB = 32 + 2 * g.TPAD;
  // B tiles from the per-template table unless MOCO_TC_BTAB=0 (then the band staging area)
  const char *bte = getenv("MOCO_TC_BTAB");
  g.stg = (bte && atoi(bte) == 0) ? 1 : 0;
  const char *nse = getenv("MOCO_TC_SLOTS");   // tuning: ring slots when copying tiles
  // (levels = 0, C1: 2 slots let the super-stages grow to 8 pairs, 1.237 -> 1.274 M frames/s;
  // at C2-C4 2 and 4 slots measure the same within 1.5 %)
  g.nss = g.stg ? TC_PRODUCERS : (nse ? std::max(2, std::min(TC_PRODUCERS, atoi(nse))) : (L == 0 ? 2 : TC_TSLOTS));
  auto smem_for = [&](int GG, int ICH) {
    return 1024 + GG * g.stripB + g.nss * ICH * g.N * 32 + g.stg * TC_PRODUCERS * 2 * ICH * 4 * g.SEGB +
           (2 * g.nss + 1) * 8 + 16;
  };
  // two CTAs per SM (one loads its next strip while the other computes): as many
  // groups per CTA as half of shared memory and half of TMEM allow, then the largest
  // super-stage (ICH | npairs) that still fits; the epilogue's staging of the d = 1
  // accumulator halves (GG*NT*128*32 words + keys) must fit in the same memory
  g.GG = 0;
  g.ctas = ctas;
  for (int GG = 4; GG >= 1 && !g.GG; --GG) {
    if (GG * g.NT * g.N > tmem_cap || GG * g.NT > 4) continue;
    for (int ICH = 8; ICH >= 1; ICH /= 2) {
      const int sm = smem_for(GG, ICH);
      if (g.npairs % ICH == 0 && sm <= smem_cap && GG * g.NT * 128 * 132 + GG * 128 * 16 + GG * g.F * g.W * g.W * 8 <= sm - 1024 - 256) {
        g.GG = GG;
        g.ICH = ICH;
        break;
      }
    }
  }
  if (!g.GG) return false;
  g.TS = g.N;   // (256-column-aligned tiles measured no faster)
  int cols = 32;
  while (cols < g.GG * g.NT * g.TS) cols <<= 1;
  g.tmem_cols = cols;
  g.smem = smem_for(g.GG, g.ICH);
  g.prep_smem = (g.F * (4 * g.hw + 4 * w * w + 1) + 8 * 2 * g.hw) * 8;   // + per-warp edge-column sums
  g.prep_smem1 = ((4 * g.hw + 4 * w * w + 1) + 8 * 2 * g.hw) * 8;        // one frame per CTA
  *gp = g;
  return true;
}

inline bool tc_supported(int dtype, int bits, int levels, int w, int mc, int nc) {
  const int vb = bits + 2 * levels;
  if (dtype != 1 /*MOCO_U16*/ || vb > 16) return false;
  // an int32 accumulator adds one part product per template-row pair and column
  const int64_t pmax = vb <= 14 ? 127 : 255;
  if (nc % 32 != 0 || (int64_t)((mc + 1) / 2) * nc * pmax * pmax >= ((int64_t)1 << 31)) return false;
  TcGeom g;
  return tc_make_geom(&g, w, mc, nc, levels, vb);
}
// AUTO policy (from measurement): the tensor-core search wherever it is
// supported; otherwise the FFT path for 16-bit data (exact after certification), with
// the CUDA-core direct search for float32 data.
inline bool tc_auto_prefers(int w) { (void)w; return true; }
inline bool fft_auto_prefers(int w, bool tc_ok) { (void)w; return !tc_ok; }

inline int tc_init(TcPlan *tc, int w, int mc, int nc, int L, int vb, int64_t cap) {
  if (!tc_make_geom(&tc->g, w, mc, nc, L, vb)) return -1;
  const TcGeom &g = tc->g;
  tc->cap = cap;
  const int64_t groups = (cap + g.F - 1) / g.F;
  if (cudaMalloc(&tc->G, (size_t)groups * g.nstrips * g.stripB) != cudaSuccess) return -1;
  if (cudaMalloc(&tc->ga, (size_t)cap * g.W * g.W * sizeof(u64)) != cudaSuccess) return -1;
  if (cudaMalloc(&tc->G2, (size_t)groups * g.nstrips * g.stripB) != cudaSuccess ||
      cudaMalloc(&tc->ga2, (size_t)cap * g.W * g.W * sizeof(u64)) != cudaSuccess) {
    cudaGetLastError();   // optional: without them batches run back to back
    if (tc->G2) cudaFree(tc->G2);
    tc->G2 = nullptr;
    tc->ga2 = nullptr;
  }
  if (cudaMalloc(&tc->T8, (size_t)2 * (mc + 2) * g.TP) != cudaSuccess) return -1;
  // precomputed B tiles (MOCO_TC_BTAB=0: the producer warps build them per CTA)
  if (!g.stg && cudaMalloc(&tc->Btab, (size_t)g.nstrips * g.npairs * g.N * 32) != cudaSuccess) return -1;
  if (smem_attr(k_tc_coarse<2>, g.smem) != cudaSuccess ||
      smem_attr(k_tc_coarse<4>, g.smem) != cudaSuccess ||
      smem_attr(k_tc_coarse<10>, g.smem) != cudaSuccess ||
      smem_attr(k_tc_coarse<14>, g.smem) != cudaSuccess ||
      smem_attr(k_tc_coarse<6>, g.smem) != cudaSuccess ||
      smem_attr(k_tc_coarse<8>, g.smem) != cudaSuccess ||
      smem_attr(k_tc_coarse<12>, g.smem) != cudaSuccess ||
      smem_attr(k_tc_coarse<16>, g.smem) != cudaSuccess)
    return -1;
  if (smem_attr(k_tc_prep<0>, g.prep_smem) != cudaSuccess ||
      smem_attr(k_tc_prep<1>, g.prep_smem) != cudaSuccess ||
      smem_attr(k_tc_prep<2>, g.prep_smem) != cudaSuccess)
    return -1;
  tc->ready = true;
  return 0;
}

inline int tc_set_template(TcPlan *tc, const uint16_t *tpl_coarse, int pitch, cudaStream_t st) {
  const TcGeom &g = tc->g;
  k_tc_template<<<128, 256, 0, st>>>(tpl_coarse, pitch, g.mc, g.nc, g.TPAD, g.TP, g.sb, tc->T8);
  if (tc->Btab) k_tc_btab<<<512, 256, 0, st>>>(tc->T8, g, tc->Btab);
  if (cudaGetLastError() != cudaSuccess) return -1;
  tc->tpl_ready = true;
  return 0;
}

inline void tc_free(TcPlan *tc) {
  if (tc->G) cudaFree(tc->G);
  if (tc->ga) cudaFree(tc->ga);
  if (tc->G2) cudaFree(tc->G2);
  if (tc->ga2) cudaFree(tc->ga2);
  tc->G2 = nullptr; tc->ga2 = nullptr;
  if (tc->T8) cudaFree(tc->T8);
  if (tc->Btab) cudaFree(tc->Btab);
  if (tc->corner) cudaFree(tc->corner);
  tc->corner = nullptr;
  tc->G = nullptr; tc->ga = nullptr; tc->T8 = nullptr; tc->Btab = nullptr;
  tc->ready = tc->tpl_ready = false;
}

}  // namespace moco
