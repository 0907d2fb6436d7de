// kernels_tc.cuh -- exact coarse search on the 5th-gen tensor cores (tcgen05, kind::i8).
//
// The cross term of P:37, h(s,t) = sum_{(i,j) in D_{s,t}} a[i+s][j+t] b[i][j], is a
// dense contraction once written per template row i and frame column j' = j+t:
//
//     h(s,t) = sum_i sum_j' a[i+s][j'] * b[i][j'-t]        (a, b zero outside the image)
//
// For each template row i and each 32-column strip of j' this is one MMA
//     D[(s,f,pa), (pb,t)] += A[(s,f,pa), j'] * B[j', (pb,t)]
// with M rows = (lag s, frame f, part pa) -- A is a sliding window over the frame's
// rows (row i+s), addressed purely through the UMMA shared-memory descriptor, so the
// Hankel structure costs no data movement -- and N columns = (part pb, lag t): B is
// the Toeplitz expansion of template row i, generated in shared memory per step.
//
// Exactness: coarse values are < 2^14 (bits + 2L <= 14); each is split
// into two 7-bit parts v = 128*hi + lo, both in [0,127], so every int8 product is exact
// and every int32 accumulator stays below 127^2 * m_c * n_c < 2^31.  The epilogue
// recombines h = 2^14 D_hh + 2^7 (D_hl + D_lh) + D_ll in 64-bit integers, so
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

#include "kernels_direct.cuh"

namespace moco {

// ------------------------------------------------------------------ geometry
struct TcGeom {
  int mc, nc, w, hw, W, L;
  int F;        // frames per operand group (1, 2, 4): core matrix = 4/F rows x (F frames x 2 parts)
  int ST;       // lag rows s per 128-row M tile = 64 / F
  int NT;       // M tiles
  int Wt;       // t lags padded to a multiple of 16
  int N;        // 2 * Wt
  int R;        // rows per operand plane = mc + NT*ST (plane row = frame row + hw)
  int nstrips;  // 32-column strips of j'
  int planeB;   // bytes per 16-column plane = R * 32 * F
  int stripB;   // 2 planes
  int OFF, TSW; // template strip: columns [J0-OFF, J0-OFF+TSW)
  int NS;       // B ring stages (2 batches of NS/2 template rows)
  int GG;       // operand groups per CTA
  int tmem_cols;
  int smem;     // dynamic shared memory bytes
  int prep_smem;
};

struct TcPlan {
  bool ready = false;
  bool tpl_ready = false;
  TcGeom g;
  int64_t cap = 0;          // frames per batch
  uint8_t *G = nullptr;     // operand planes for cap frames
  u64 *ga = nullptr;        // [cap][W*W] frame energies
  uint8_t *T8 = nullptr;    // template parts [2][mc][nc]
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
};

// One CTA per operand group of F frames.  Shared: per frame, edge-row and edge-column
// sums of a^2, the four (hw+1)^2 corner tables and the total.
template <int L>
__global__ void __launch_bounds__(256) k_tc_prep(TcPrepArgs a) {
  const TcGeom &g = a.g;
  extern __shared__ __align__(16) unsigned char smem[];
  const int F = g.F, hw = g.hw, w = g.w, mc = g.mc, nc = g.nc, W = g.W;
  const int CS = w * w;                       // corner table size per quad (index 0 = empty)
  u64 *rowE = reinterpret_cast<u64 *>(smem);  // [F][2*hw]  top rows 0..hw-1, bottom rows from the bottom
  u64 *colE = rowE + F * 2 * hw;              // [F][2*hw]
  u64 *cor = colE + F * 2 * hw;               // [F][4][w][w]
  u64 *tot = cor + F * 4 * CS;                // [F]
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int k = tid; k < F * (4 * hw + 4 * CS + 1); k += nth) rowE[k] = 0;
  __syncthreads();
  const int grp = blockIdx.x;
  const int items = g.nstrips * 2 * g.R * F;
  constexpr int bs = 1 << L;
  u64 mytot[4] = {0, 0, 0, 0};
  for (int it = tid; it < items; it += nth) {
    const int f = it % F;
    int rest = it / F;
    const int r = rest % g.R;
    rest /= g.R;
    const int kc = rest & 1, st = rest >> 1;
    const int fi = grp * F + f;
    const int cr = r - hw;
    const int c0 = st * 32 + kc * 16;
    uint32_t v[16];
#pragma unroll
    for (int x = 0; x < 16; ++x) v[x] = 0;
    const bool live = fi < a.B && cr >= 0 && cr < mc && c0 < nc;
    if (live) {
      const uint16_t *base = a.frames + (int64_t)fi * a.fstride + (int64_t)(cr * bs) * a.n + c0 * bs;
#pragma unroll
      for (int dy = 0; dy < bs; ++dy) {
        const uint16_t *row = base + (int64_t)dy * a.n;
        // 16 coarse columns = 16*bs raw samples = 2*bs 16-byte vectors (nc % 32 == 0)
#pragma unroll
        for (int q = 0; q < 2 * bs; ++q) {
          const uint4 u = *reinterpret_cast<const uint4 *>(row + q * 8);
          const uint32_t ws[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const uint32_t s = (ws[e >> 1] >> (16 * (e & 1))) & 0xffffu;
            const int x = (q * 8 + e) / bs;   // coarse column within the 16
            v[x] += s;
          }
        }
      }
#pragma unroll
      for (int x = 0; x < 16; ++x)
        if (c0 + x >= nc) v[x] = 0;
    }
    // int8 parts, 16 bytes each
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      hi[q] = lo[q] = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        hi[q] |= (v[4 * q + e] >> 7) << (8 * e);
        lo[q] |= (v[4 * q + e] & 127u) << (8 * e);
      }
    }
    uint8_t *dst = a.G + ((((int64_t)grp * g.nstrips + st) * 2 + kc) * g.R + r) * (32 * F) + f * 32;
    *reinterpret_cast<uint4 *>(dst) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4 *>(dst + 16) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    if (!live) continue;
    // energies (S2): totals, edge strips, corners
    uint32_t rs = 0;
#pragma unroll
    for (int x = 0; x < 16; ++x) rs += v[x] * v[x];   // < 16 * 2^28 = 2^32
    mytot[f] += rs;
    const bool top = cr < hw, bot = cr >= mc - hw;
    if (top) atomicAdd(&rowE[f * 2 * hw + cr], (u64)rs);
    if (bot) atomicAdd(&rowE[f * 2 * hw + hw + (mc - 1 - cr)], (u64)rs);
#pragma unroll
    for (int x = 0; x < 16; ++x) {
      const int c = c0 + x;
      if (c >= nc) break;
      const bool lf = c < hw, rt = c >= nc - hw;
      if (!(lf || rt)) continue;
      const u64 v2 = (u64)(v[x] * v[x]);
      if (lf) atomicAdd(&colE[f * 2 * hw + c], v2);
      if (rt) atomicAdd(&colE[f * 2 * hw + hw + (nc - 1 - c)], v2);
      if (top || bot) {
        for (int qb = 0; qb < 2; ++qb) {
          if (!(qb ? bot : top)) continue;
          const int p = qb ? mc - cr : cr + 1;
          for (int qr = 0; qr < 2; ++qr) {
            if (!(qr ? rt : lf)) continue;
            const int qq = qr ? nc - c : c + 1;
            cor[((f * 4) + (qb * 2 + qr)) * CS + p * w + qq] = v2;
          }
        }
      }
    }
  }
  // totals
  for (int f = 0; f < F; ++f) {
    const u64 s = warp_sum(mytot[f]);
    if ((tid & 31) == 0) atomicAdd(&tot[f], s);
  }
  __syncthreads();
  // prefix sums: edge strips (1-D), corners (2-D, the DP of P:35 in each corner)
  for (int k = tid; k < F * 4; k += nth) {
    u64 *e = (k & 2) ? colE : rowE;
    u64 *p = e + (k >> 2) * 2 * hw + (k & 1) * hw;
    for (int q = 1; q < hw; ++q) p[q] += p[q - 1];
  }
  for (int k = tid; k < F * 4 * w; k += nth) {
    u64 *c = cor + (k / w) * CS + (k % w) * w;
    for (int q = 1; q < w; ++q) c[q] += c[q - 1];
  }
  __syncthreads();
  for (int k = tid; k < F * 4 * w; k += nth) {
    u64 *c = cor + (k / w) * CS + (k % w);
    for (int p = 1; p < w; ++p) c[p * w] += c[(p - 1) * w];
  }
  __syncthreads();
  for (int k = tid; k < F * W * W; k += nth) {
    const int f = k / (W * W), lag = k % (W * W);
    const int fi = grp * F + f;
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

// One CTA = GG operand groups (GG*F frames) sharing every generated B tile.
// 256 threads: all generate B tiles for ICH template rows at a time into a ring of
// NS = 2*ICH stages, thread 0 issues the MMAs of the batch and commits each stage to
// its `empty` mbarrier, so generation of batch b+1 overlaps the MMAs of batch b.
__global__ void __launch_bounds__(256, 1) k_tc_coarse(TcArgs a) {
  const TcGeom &g = a.g;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nth = blockDim.x;
  const int F = g.F, hw = g.hw, mc = g.mc, nc = g.nc, N = g.N, NT = g.NT, NS = g.NS, GG = g.GG;
  const int ICH = NS / 2;
  unsigned char *As = smem;                                   // [GG] strips of 2 planes
  unsigned char *TS = As + GG * g.stripB;                     // [2][mc][TSW]
  unsigned char *Bring = TS + 2 * mc * g.TSW;                 // [NS][N*32]
  uint64_t *bars = reinterpret_cast<uint64_t *>(Bring + NS * N * 32);   // empty[NS], aload
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + NS + 1);
  Key *keys = reinterpret_cast<Key *>(smem);                 // epilogue: aliases the strips
  const int grp0 = blockIdx.x * GG;
  const int ngroups = (a.B + F - 1) / F;
  const int gcount = min(GG, ngroups - grp0);

  if (warp == 0) tmem_alloc(tmem_holder, g.tmem_cols);
  if (tid == 0) {
    for (int s = 0; s < NS + 1; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = *tmem_holder;
  const uint32_t idesc = idesc_i8(128, N);
  const uint32_t As_u = smem_u32(As);
  const uint32_t B_u = smem_u32(Bring);
  uint64_t *aload = &bars[NS];

  int it = 0;
  for (int st = 0; st < g.nstrips; ++st) {
    const int J0 = st * 32;
    if (tid == 0) {
      mbar_arrive_expect_tx(aload, (uint32_t)(gcount * g.stripB));
      for (int gg = 0; gg < gcount; ++gg)
        bulk_g2s(As + gg * g.stripB, a.G + ((int64_t)(grp0 + gg) * g.nstrips + st) * g.stripB,
                 (uint32_t)g.stripB, aload);
    }
    // template strip: TS[pb][i][x] = b_pb[i][J0 - OFF + x] (0 outside the image)
    {
      const int vec = g.TSW / 16;
      const int total = 2 * mc * vec;
      for (int e = tid; e < total; e += nth) {
        const int x16 = e % vec;
        const int row = e / vec;   // pb*mc + i
        const int col = J0 - g.OFF + x16 * 16;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (col >= 0 && col + 16 <= nc) v = *reinterpret_cast<const uint4 *>(a.T8 + (int64_t)row * nc + col);
        *reinterpret_cast<uint4 *>(TS + row * g.TSW + x16 * 16) = v;
      }
    }
    mbar_wait(aload, st & 1);
    __syncthreads();
    for (int i0 = 0; i0 < mc; i0 += ICH) {
      const int nI = min(ICH, mc - i0);
      // ring slots of this batch must have been consumed by the MMAs of batch-2
      for (int q = 0; q < nI; ++q) {
        const int j = it + q;
        if (j >= NS) mbar_wait(&bars[j % NS], ((j / NS) - 1) & 1);
      }
      // B tiles: N rows (pb, t) x 32 bytes: B[(pb,t)][k] = b_pb[i][J0 + k - t]
      for (int c = tid; c < nI * 2 * N; c += nth) {
        const int q = c / (2 * N), cc = c % (2 * N);
        const int n = cc >> 1, h = cc & 1;
        const int pb = n / g.Wt, ti = n % g.Wt;
        unsigned char *Bt = Bring + ((it + q) % NS) * N * 32;
        uint4 outv = make_uint4(0, 0, 0, 0);
        if (ti < g.W) {
          const int o = 16 * h - (ti - hw) + g.OFF;
          const uint32_t *wp =
              reinterpret_cast<const uint32_t *>(TS + (pb * mc + i0 + q) * g.TSW + (o & ~3));
          const uint32_t sh = (o & 3) * 8;
          const uint32_t w0 = wp[0], w1 = wp[1], w2 = wp[2], w3 = wp[3], w4 = wp[4];
          outv.x = __funnelshift_r(w0, w1, sh);
          outv.y = __funnelshift_r(w1, w2, sh);
          outv.z = __funnelshift_r(w2, w3, sh);
          outv.w = __funnelshift_r(w3, w4, sh);
        }
        *reinterpret_cast<uint4 *>(Bt + (n >> 3) * 256 + h * 128 + (n & 7) * 16) = outv;
      }
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        for (int q = 0; q < nI; ++q) {
          const int stage = (it + q) % NS;
          const int i = i0 + q;
          const uint64_t bdesc = umma_desc(B_u + stage * N * 32, 128, 256);
          for (int gg = 0; gg < gcount; ++gg)
            for (int k = 0; k < NT; ++k) {
              const uint64_t adesc =
                  umma_desc(As_u + gg * g.stripB + (i + k * g.ST) * 32 * F, g.planeB, 128);
              mma_i8(taddr + (gg * NT + k) * N, adesc, bdesc, idesc, (st | i) != 0 ? 1u : 0u);
            }
          mma_commit(&bars[stage]);
        }
      }
      it += nI;
    }
    // every MMA of this strip has completed before the strip buffers are reused
    const int last = it - 1;
    mbar_wait(&bars[last % NS], (last / NS) & 1);
  }
  tc_fence_after();

  // ---- epilogue: h -> N -> f -> argmin (S4), per frame.  Warp w reads TMEM lanes
  // 32*(w%4).. of the tiles of groups gg = w/4, w/4 + 2, ...
  const int W = g.W;
  const int m = (warp & 3) * 32 + lane;     // accumulator row = TMEM lane
  const int sl = m / (2 * F), rho = m % (2 * F);
  const int f = rho >> 1, pa = rho & 1;
  Key best[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    best[q] = Key{~0ull, ~0u};
    const int gg = (warp >> 2) + 2 * q;
    if (gg >= GG) continue;
    const int fi = (grp0 + gg) * F + f;
    Key bk{~0ull, ~0u};
    for (int k = 0; k < NT; ++k) {
      const int s = -hw + k * g.ST + sl;
      const bool valid = gg < gcount && pa == 0 && s <= hw && fi < a.B;
      for (int c = 0; c < g.Wt; c += 16) {
        uint32_t xh[16], xl[16];
        const uint32_t tbase = taddr + ((uint32_t)((warp & 3) * 32) << 16) + (gg * NT + k) * N;
        tmem_ld16(tbase + c, xh);             // pb = hi
        tmem_ld16(tbase + g.Wt + c, xl);      // pb = lo
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint32_t ph = __shfl_xor_sync(0xffffffffu, xh[q], 1);   // partner row: pa = lo
          const uint32_t pl = __shfl_xor_sync(0xffffffffu, xl[q], 1);
          const int ti = c + q;
          if (!valid || ti >= W) continue;
          const u64 h = ((u64)xh[q] << 14) + (((u64)xl[q] + (u64)ph) << 7) + (u64)pl;
          const int lag = (s + hw) * W + ti;
          const u64 Nn = a.ga[(int64_t)fi * W * W + lag] + a.gb[lag] - 2 * h;
          const int t = ti - hw;
          const double area = (double)((mc - abs(s)) * (nc - abs(t)));
          const double fv = (double)Nn / (a.scale * area);
          if (a.grid_out) a.grid_out[(int64_t)fi * W * W + lag] = fv;
          const Key kk{(u64)__double_as_longlong(fv), (unsigned)lag};
          if (key_less(kk, bk)) bk = kk;
        }
      }
    }
    best[q] = bk;
  }
  tc_fence_before();
  fence_proxy_async();
  __syncthreads();   // strip buffers are now free for the key table
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
      for (int q = 2 * ff; q < 128; q += 2 * F)
        if (key_less(keys[gg * 128 + q], b)) b = keys[gg * 128 + q];
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

// template parts for the B operand: T8[0] = b >> 7, T8[1] = b & 127 (coarse template)
__global__ void k_tc_template(const uint16_t *__restrict__ b, int pitch, int mc, int nc, uint8_t *T8) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < mc * nc; e += gridDim.x * blockDim.x) {
    const int i = e / nc, j = e % nc;
    const uint32_t v = b[(int64_t)i * pitch + j];
    T8[e] = (uint8_t)(v >> 7);
    T8[mc * nc + e] = (uint8_t)(v & 127u);
  }
}

// ---------------------------------------------------------------- host side
inline bool tc_make_geom(TcGeom *gp, int w, int mc, int nc, int L) {
  TcGeom g{};
  g.mc = mc; g.nc = nc; g.w = w; g.hw = w - 1; g.W = 2 * w - 1; g.L = L;
  g.Wt = (g.W + 15) / 16 * 16;
  g.N = 2 * g.Wt;
  if (g.N > 256) return false;
  // frames per group: the largest F with the fewest padded lag rows and NT*N <= 256
  int bestF = 0, bestRows = 1 << 30;
  for (int F : {4, 2, 1}) {
    const int ST = 64 / F, NT = (g.W + ST - 1) / ST;
    if (NT * g.N > 256) continue;
    if (NT * ST < bestRows) { bestRows = NT * ST; bestF = F; }
  }
  if (!bestF) return false;
  g.F = bestF; g.ST = 64 / g.F; g.NT = (g.W + g.ST - 1) / g.ST;
  g.R = mc + g.NT * g.ST;
  g.nstrips = (nc + 31) / 32;
  g.planeB = g.R * 32 * g.F;
  g.stripB = 2 * g.planeB;
  g.OFF = (g.hw + 15) / 16 * 16;
  g.TSW = (16 + g.hw + g.OFF + 20 + 15) / 16 * 16;
  auto smem_for = [&](int GG, int NS) {
    return 1024 + GG * g.stripB + 2 * mc * g.TSW + NS * g.N * 32 + (NS + 1) * 8 + 16;
  };
  // as many groups per CTA as shared memory (227 KB) and TMEM (512 columns) allow
  g.NS = 16;
  g.GG = 0;
  for (int GG = 8; GG >= 1 && !g.GG; --GG) {
    if (GG * g.NT * g.N > 512) continue;
    for (int NS = 16; NS >= 4; NS -= 4)
      if (smem_for(GG, NS) <= 227 * 1024 && GG * 128 * 16 <= GG * g.stripB) {
        g.GG = GG;
        g.NS = NS;
        break;
      }
  }
  if (!g.GG) return false;
  int cols = 32;
  while (cols < g.GG * g.NT * g.N) cols <<= 1;
  g.tmem_cols = cols;
  g.smem = smem_for(g.GG, g.NS);
  g.prep_smem = (g.F * (4 * g.hw + 4 * w * w + 1)) * 8;
  *gp = g;
  return true;
}

inline bool tc_supported(int dtype, int bits, int levels, int w, int mc, int nc) {
  if (dtype != 1 /*MOCO_U16*/ || bits + 2 * levels > 14) return false;
  if (nc % 32 != 0 || (int64_t)mc * nc * 127 * 127 >= ((int64_t)1 << 31)) return false;
  TcGeom g;
  return tc_make_geom(&g, w, mc, nc, levels);
}
// AUTO policy: the tensor-core search wherever it is supported.
inline bool tc_auto_prefers(int w) { (void)w; return true; }

inline int tc_init(TcPlan *tc, int w, int mc, int nc, int L, int64_t cap) {
  if (!tc_make_geom(&tc->g, w, mc, nc, L)) return -1;
  const TcGeom &g = tc->g;
  tc->cap = cap;
  const int64_t groups = (cap + g.F - 1) / g.F;
  if (cudaMalloc(&tc->G, (size_t)groups * g.nstrips * g.stripB) != cudaSuccess) return -1;
  if (cudaMalloc(&tc->ga, (size_t)cap * g.W * g.W * sizeof(u64)) != cudaSuccess) return -1;
  if (cudaMalloc(&tc->T8, (size_t)2 * mc * nc) != cudaSuccess) return -1;
  if (cudaFuncSetAttribute(k_tc_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize, g.smem) != cudaSuccess)
    return -1;
  if (cudaFuncSetAttribute(k_tc_prep<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, g.prep_smem) != cudaSuccess ||
      cudaFuncSetAttribute(k_tc_prep<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, g.prep_smem) != cudaSuccess ||
      cudaFuncSetAttribute(k_tc_prep<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, g.prep_smem) != cudaSuccess)
    return -1;
  tc->ready = true;
  return 0;
}

inline int tc_set_template(TcPlan *tc, const uint16_t *tpl_coarse, int pitch, cudaStream_t st) {
  const TcGeom &g = tc->g;
  k_tc_template<<<64, 256, 0, st>>>(tpl_coarse, pitch, g.mc, g.nc, tc->T8);
  if (cudaGetLastError() != cudaSuccess) return -1;
  tc->tpl_ready = true;
  return 0;
}

inline void tc_free(TcPlan *tc) {
  if (tc->G) cudaFree(tc->G);
  if (tc->ga) cudaFree(tc->ga);
  if (tc->T8) cudaFree(tc->T8);
  tc->G = nullptr; tc->ga = nullptr; tc->T8 = nullptr;
  tc->ready = tc->tpl_ready = false;
}

}  // namespace moco
