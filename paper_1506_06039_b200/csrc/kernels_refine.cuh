// kernels_refine.cuh -- S5 refine (+ S6 apply) for MOCO_U16.
//
// At each finer level l the nine candidates (s,t) = (S+u, T+v), u,v in {-1,0,1},
// with (S,T) = 2 x the shift of level l+1 ("multiply the optimal (s,t) by 2 and
// do a local search"), are scored exactly through the decomposition of P:31:
//
//     N(s,t) = GA(s,t) + GB(s,t) - 2 H(s,t)
//     H(s,t)  = sum_{(i,j) in D_{s,t}} a[i+s][j+t] b[i][j]       (cross term)
//     GA(s,t) = sum_{(i,j) in D_{s,t}} a[i+s][j+t]^2             (frame energy)
//     GB(s,t) = sum_{(i,j) in D_{s,t}} b[i][j]^2                 (template energy)
//
// Template-stationary design: the template is read ONCE per plan call, not once per
// frame.  K_sum (k_refine_sums) gives each CTA a fixed tile of template rows
// [r0, r1) x 256 columns in shared memory; a producer warp streams, frame after frame,
// the matching frame rows [r0+S-1, r1+S+1) into a TMA ring, and each consumer warp
// takes one frame at a time (lane = 8 template columns, all rows of the tile, frame
// rows kept in registers).  TMA tensor boxes start at the 16-byte aligned column
// x0 <= T-1 and are zero-filled outside the frame, so with a_pad = 0 outside
//     H(s,t)  = sum_{tile (i,j)} a_pad[i+s][j+t] b[i][j]
//     GA(s,t) = sum_{tile (i,j)} a_pad[i+s][j+t]^2
// -- one uniform loop (specialised on the misalignment T-1-x0).  The warp's 18 sums
// go to the frame's 64-bit accumulators with one atomic add each.
// K_pick (k_refine_pick) then forms N = GA + GB - 2H per candidate (GB from the
// plan's 2-D prefix table of b^2), takes the argmin with key (f, s, t), re-zeroes the
// accumulators and, at level 0, writes the corrected frame c[i][j] = a[i+s][j+t]
// (0 outside) with 16-byte streaming stores.
// Everything is exact in integers, so f = fl(N / (16^l A)) is the oracle's value.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "kernels_tc.cuh"

namespace moco {

// 2-D prefix of b^2: P[i][j] = sum_{i' < i, j' < j} b[i'][j']^2, (m+1) x (n+1), once per plan.
// Pass 1 (rows) then pass 2 (columns), one thread per row / column.
// 2-D prefix of b^2, P[i][j] = sum_{i'<i, j'<j} b[i'][j']^2, (m+1) x (n+1): a warp per row
// (warp scans over 32-column chunks, coalesced), then the column pass in row segments
// (each thread scans a segment of its column, the segment totals are prefixed, a second
// pass adds them): independent loads in flight instead of one dependent chain per column.
__global__ void k_prefix2d_rows(const uint16_t *__restrict__ b, int pitch, int m, int n, u64 *__restrict__ P) {
  const int n1 = n + 1, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i <= m; i += nw) {
    u64 *row = P + (int64_t)i * n1;
    if (lane == 0) row[0] = 0;
    u64 carry = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      u64 v = 0;
      if (i > 0 && j < n) {
        const u64 x = b[(int64_t)(i - 1) * pitch + j];
        v = x * x;
      }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u64 t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
      }
      v += carry;
      if (j < n) row[j + 1] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
}
constexpr int PF_SEG = 16;   // row segments of the column pass
__global__ void k_prefix2d_cols(int m, int n, u64 *__restrict__ P) {
  // block: 32 columns x PF_SEG segments
  __shared__ u64 seg[PF_SEG][33];
  const int n1 = n + 1, m1 = m + 1;
  const int c = threadIdx.x & 31, sg = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + c;
  const int rows = (m1 + PF_SEG - 1) / PF_SEG, r0 = sg * rows, r1 = min(m1, r0 + rows);
  u64 acc = 0;
  if (j <= n)
    for (int i = r0; i < r1; ++i) acc += P[(int64_t)i * n1 + j];
  seg[sg][c] = acc;
  __syncthreads();
  u64 off = 0;
  for (int k = 0; k < sg; ++k) off += seg[k][c];
  if (j <= n)
    for (int i = r0; i < r1; ++i) {
      off += P[(int64_t)i * n1 + j];
      P[(int64_t)i * n1 + j] = off;
    }
}

struct RefineSumArgs {
  const uint16_t *tpl;      // level-l template
  int tpitch;
  int ml, nl;
  int B;
  const int32_t *shift_in;  // [B][2] at level l+1
  u64 *acc;                 // [B][18]: H for the 9 candidates, then GA
  int rt;                   // template rows per tile (<= RS_MAXRT)
  int nrt;                  // row tiles
  int stages;               // ring depth
  int wide;                 // 1: flush 32-bit partials after every row (values >= 2^13)
};

#ifndef RS_CTW
#define RS_CTW 256
#endif
constexpr int RS_CT = RS_CTW;         // template columns per tile (a warp walks it in 256-column halves)
constexpr int RS_BOX = RS_CT == 512 ? 176 : 136;   // frame box columns: the boxes cover CT + 9
constexpr int RS_NBOX = RS_CT == 512 ? 3 : 2;
constexpr int RS_MAXRT = 16;
constexpr int RS_CW = 12;             // consumer warps (frames in flight per CTA)
constexpr int RS_THREADS = 32 * (1 + RS_CW);

// staged frame box: (rt+2) rows x RS_BOX columns, padded to 128 bytes (TMA destination alignment)
__host__ __device__ inline int rs_box_elems(int rt) { return ((rt + 2) * RS_BOX * 2 + 127) / 128 * 64; }
__host__ __device__ inline int rs_stage_bytes(int rt) { return RS_NBOX * rs_box_elems(rt) * 2; }
inline int rs_smem_bytes(int rt, int stages) { return 1024 + RS_MAXRT * RS_CT * 2 + stages * rs_stage_bytes(rt) + RS_CW * 32 * 19 * 4; }

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// TMA tensor load of a 3-D box (x = column, y = row, z = frame), zero fill out of bounds.
__device__ __forceinline__ void tma_load3(void *dst, const CUtensorMap *tm, int x, int y, int z, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap *tm, int x, int y, int z, const void *src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(tm)),
               "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
               : "memory");
}
// L2 eviction-priority policies (createpolicy) and the hinted copies that use them.
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load3_hint(void *dst, const CUtensorMap *tm, int x, int y, int z, uint64_t *bar,
                                               uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
      "{%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st_global_hint(void *p, const uint4 &v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }


// Frame row window for template columns j0..j0+7: the 10 samples at frame columns
// j0+T-1 .. j0+T+8 (staged columns j0+OFFA .. j0+OFFA+9), plus the three 8-wide sums
// of their squares for v = -1, 0, +1.
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// Frame row window for template columns j0..j0+7: the 10 samples at frame columns
// j0+T-1 .. j0+T+8, i.e. staged columns c+OFFA .. c+OFFA+9.  Six 32-bit words from the
// word offset OFFA/2 (per-word shared addresses: the window may cross a box), then
// one runtime funnel shift per word pair for odd OFFA -- the same code for every
// misalignment, so concurrently running warps share one instruction stream.
__device__ __forceinline__ void rs_frame10(const uint32_t (&wa)[6], uint32_t roff, uint32_t sh, uint32_t (&v)[10],
                                           uint32_t (&wsum)[3]) {
  uint32_t w[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) w[q] = lds32(wa[q] + roff);
#pragma unroll
  for (int m = 0; m < 5; ++m) {
    const uint32_t u = __funnelshift_r(w[m], w[m + 1], sh);
    v[2 * m] = u & 0xffffu;
    v[2 * m + 1] = u >> 16;
  }
  uint32_t sq[10];
#pragma unroll
  for (int x = 0; x < 10; ++x) sq[x] = v[x] * v[x];
  uint32_t mid = 0;
#pragma unroll
  for (int x = 1; x < 9; ++x) mid += sq[x];
  wsum[0] = mid - sq[8] + sq[0];   // v = -1
  wsum[1] = mid;                   // v =  0
  wsum[2] = mid - sq[1] + sq[9];   // v = +1
}

__device__ __forceinline__ void load_tpl8(const uint16_t *p, uint32_t (&bv)[8]) {
  const uint4 bq = *reinterpret_cast<const uint4 *>(p);
  const uint32_t bw[4] = {bq.x, bq.y, bq.z, bq.w};
#pragma unroll
  for (int x = 0; x < 8; ++x) bv[x] = (x & 1) ? (bw[x >> 1] >> 16) : (bw[x >> 1] & 0xffffu);
}

// One template row against the three frame rows (u = -1, 0, +1).
__device__ __forceinline__ void h_row(const uint32_t (&bv)[8], const uint32_t (&f0)[10], const uint32_t (&f1)[10],
                                      const uint32_t (&f2)[10], const uint32_t (&w0)[3], const uint32_t (&w1)[3],
                                      const uint32_t (&w2)[3], uint32_t (&H)[9], uint32_t (&GA)[9]) {
#pragma unroll
  for (int v = 0; v < 3; ++v) {
    uint32_t h0 = H[v], h1 = H[3 + v], h2 = H[6 + v];
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      h0 += f0[x + v] * bv[x];
      h1 += f1[x + v] * bv[x];
      h2 += f2[x + v] * bv[x];
    }
    H[v] = h0; H[3 + v] = h1; H[6 + v] = h2;
    GA[v] += w0[v]; GA[3 + v] += w1[v]; GA[6 + v] += w2[v];
  }
}

// One frame on one warp: rows 0..nr-1 of the tile against staged frame rows 0..nr+1,
// the tile's columns walked in halves of 256 (lane = 8 columns of a half).
// Staged row k of box b starts at Fs + b*rs_box_elems(rt) + k*RS_BOX.
template <bool WIDE>
__device__ __forceinline__ void rs_frame(const uint16_t *Tt, const uint16_t *Fs, int rt, int nr, int ncols, int offa,
                                         uint32_t (&H)[9], uint32_t (&GA)[9], u64 (&H64)[9], u64 (&G64)[9]) {
  const int lane = threadIdx.x & 31;
  const int be = rs_box_elems(rt);
  const uint32_t fbase = (uint32_t)__cvta_generic_to_shared(Fs);
  const uint32_t sh = (uint32_t)(offa & 1) * 16;
  auto fl = [&]() {
    if (WIDE) {
#pragma unroll
      for (int q = 0; q < 9; ++q) { H64[q] += H[q]; G64[q] += GA[q]; H[q] = 0; GA[q] = 0; }
    }
  };
  for (int c = lane * 8; c < ncols; c += 256) {   // ncols % 8 == 0: a lane's 8 columns are all in or all out
    uint32_t wa[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const int col = c + (offa & ~1) + 2 * q;
      wa[q] = fbase + (uint32_t)(((col / RS_BOX) * be + (col % RS_BOX)) * 2);
    }
    const uint16_t *tp = Tt + c;
    uint32_t fa[10], fb[10], fc[10], wa0[3], wb[3], wc[3], bv[8];
    auto ld = [&](int k, uint32_t (&v)[10], uint32_t (&w)[3]) { rs_frame10(wa, (uint32_t)(k * RS_BOX * 2), sh, v, w); };
    ld(0, fa, wa0);
    ld(1, fb, wb);
    int q = 0;
    for (; q + 3 <= nr; q += 3) {
      ld(q + 2, fc, wc); load_tpl8(tp + q * RS_CT, bv); h_row(bv, fa, fb, fc, wa0, wb, wc, H, GA); fl();
      ld(q + 3, fa, wa0); load_tpl8(tp + (q + 1) * RS_CT, bv); h_row(bv, fb, fc, fa, wb, wc, wa0, H, GA); fl();
      ld(q + 4, fb, wb); load_tpl8(tp + (q + 2) * RS_CT, bv); h_row(bv, fc, fa, fb, wc, wa0, wb, H, GA); fl();
    }
    if (q < nr) { ld(q + 2, fc, wc); load_tpl8(tp + q * RS_CT, bv); h_row(bv, fa, fb, fc, wa0, wb, wc, H, GA); fl(); ++q; }
    if (q < nr) { ld(q + 2, fa, wa0); load_tpl8(tp + q * RS_CT, bv); h_row(bv, fb, fc, fa, wb, wc, wa0, H, GA); fl(); }
  }
}

template <bool WIDE>
__global__ void __launch_bounds__(RS_THREADS, 1)
    k_refine_sums(const __grid_constant__ CUtensorMap tmF, RefineSumArgs a) {
  pdl_enter();
  extern __shared__ __align__(1024) unsigned char rs_smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(rs_smem);   // [32]
  uint64_t *empty = full + 32;                               // [32], then int[32] stage misalignments
  uint16_t *Tt = reinterpret_cast<uint16_t *>(rs_smem + 1024);
  unsigned char *ring = rs_smem + 1024 + RS_MAXRT * RS_CT * 2;
  const int RT = a.rt, NS = a.stages, SB = rs_stage_bytes(RT);
  uint32_t *red = reinterpret_cast<uint32_t *>(ring + NS * SB);   // [RS_CW][32][19]
  const int ml = a.ml, nl = a.nl;
  const int rtile = blockIdx.x % a.nrt, ctile = blockIdx.x / a.nrt;
  const int r0 = (int)((int64_t)rtile * ml / a.nrt), nr = (int)((int64_t)(rtile + 1) * ml / a.nrt) - r0;
  const int c0 = ctile * RS_CT;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // the template tile, zero outside the template
  for (int e = tid; e < RS_MAXRT * RS_CT; e += blockDim.x) {
    const int r = e / RS_CT, c = e % RS_CT;
    Tt[e] = (r < nr && c0 + c < nl) ? a.tpl[(int64_t)(r0 + r) * a.tpitch + c0 + c] : (uint16_t)0;
  }
  if (tid == 0) {
    for (int k = 0; k < NS; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], 1);
      reinterpret_cast<int *>(empty + 32)[32 + k] = -1;
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (nr <= 0) return;
  int *stg_offa = reinterpret_cast<int *>(empty + 32);   // [32] misalignment of the frame in each stage
  int *stg_tag = stg_offa + 32;                           // [32] frame a stage was last issued for
  // (a parity wait alone can alias: a consumer may start waiting on a stage while its
  // previous use is still in flight, two phases behind; the tag orders it first)
  if (warp == 0) {
    // ---------------- producer: frame f's rows [r0+S-1, r0+nr+S+1) into stage f % NS.
    // Lanes 0..7 each own every 8th frame (independent stages), so eight frames are
    // waited for and issued per pass; shifts are read 32 frames at a time.
    const uint32_t bytes = (uint32_t)(RS_NBOX * (RT + 2) * RS_BOX * 2);   // full boxes
    for (int f32 = 0; f32 < a.B; f32 += 32) {
      int2 sv = make_int2(0, 0);
      if (f32 + lane < a.B) sv = reinterpret_cast<const int2 *>(a.shift_in)[f32 + lane];
      for (int k0 = 0; k0 < 32; k0 += 8) {
        const int sx = __shfl_sync(0xffffffffu, sv.x, k0 + (lane & 7));
        const int sy = __shfl_sync(0xffffffffu, sv.y, k0 + (lane & 7));
        const int f = f32 + k0 + lane;
        if (lane < 8 && f < a.B) {
          const int S = 2 * sx, T = 2 * sy;
          const int stg = f % NS;
          if (f >= NS) mbar_wait(&empty[stg], ((f / NS) - 1) & 1);
          const int x0 = c0 + (T - 1) - ((T - 1) & 7);
          uint16_t *Fs = reinterpret_cast<uint16_t *>(ring + stg * SB);
          stg_offa[stg] = (T - 1) & 7;
          *reinterpret_cast<volatile int *>(&stg_tag[stg]) = f;
          mbar_arrive_expect_tx(&full[stg], bytes);
#pragma unroll
          for (int bx = 0; bx < RS_NBOX; ++bx)
            tma_load3(Fs + bx * rs_box_elems(RT), &tmF, x0 + bx * RS_BOX, r0 + S - 1, f, &full[stg]);
        }
        __syncwarp();
      }
    }
    return;
  }
  // ---------------- consumers: warp w takes frames w-1, w-1+RS_CW, ...
  const int cw = warp - 1;
  uint32_t *rw = red + cw * 32 * 19;
  for (int f = cw; f < a.B; f += RS_CW) {
    const int stg = f % NS;
    while (*reinterpret_cast<volatile int *>(&stg_tag[stg]) != f) __nanosleep(32);
    mbar_wait(&full[stg], (f / NS) & 1);
    const int offa = stg_offa[stg];
    const uint16_t *Fs = reinterpret_cast<const uint16_t *>(ring + stg * SB);
    uint32_t H[9], GA[9];
    u64 H64[9], G64[9];   // 64-bit flush targets, live only when WIDE
#pragma unroll
    for (int q = 0; q < 9; ++q) { H[q] = 0; GA[q] = 0; }
    if (WIDE) {
#pragma unroll
      for (int q = 0; q < 9; ++q) { H64[q] = 0; G64[q] = 0; }
    }
#ifndef RS_NOCOMPUTE
    rs_frame<WIDE>(Tt, Fs, RT, nr, min(RS_CT, nl - c0), offa, H, GA, H64, G64);
#else
    H[0] += Fs[lane] + offa;
#endif
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stg]);   // the staged rows are no longer read
    u64 *acc = a.acc + (int64_t)f * 18;
    if (!WIDE) {
      // lane sums < 2^31 (<= 64 products < 2^24 each): transpose through shared memory,
      // lanes 0..17 add one column of 32 in 64 bits
#pragma unroll
      for (int q = 0; q < 9; ++q) { rw[lane * 19 + q] = H[q]; rw[lane * 19 + 9 + q] = GA[q]; }
      __syncwarp();
      if (lane < 18) {
        u64 sum = 0;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) sum += rw[k * 19 + lane];
        atomicAdd(acc + lane, sum);
      }
      __syncwarp();
    } else {
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const u64 h = warp_sum(H64[q]), g = warp_sum(G64[q]);
        if (lane == 0) { atomicAdd(acc + q, h); atomicAdd(acc + 9 + q, g); }
      }
    }
  }
}

struct RefinePickArgs {
  const uint16_t *frames;   // level-l images (apply source at level 0)
  int64_t fstride;
  int pitch;
  const u64 *pb2;           // [(ml+1)][(nl+1)] prefix of b^2
  int ml, nl;
  double scale;             // 16^l
  int B;
  const int32_t *shift_in;  // [B][2] at level l+1
  u64 *acc;                 // [B][18], re-zeroed here
  int32_t *shift_out;       // [B][2] at level l
  double *f_out;            // [B] or null
  uint16_t *corrected;      // [B][ml][nl] or null (level 0)
  int parts;                // CTAs per frame (apply rows split among them)
  int ga_total;             // 1: acc[9] holds the tensor-core refine's a^2 sum over its staged
                            // pixels (grid rows [0, ml+2), grid columns [-o, kw-o)); the
                            // nine GA are completed here (ga_pieces).  0: acc[9..17] are GA
  int kw;                   // 16 n_k: staged columns per grid row (ga_total)
  const u64 *gbin;          // ga_total: [B][26] pieces from k_ga_pieces, or null (computed here)
};

// GA pieces of frame f for ga_total (kernels_rtc.cuh, RTC_GA_TOTAL): on the extended grid
// A[p_r][p_c] = a[p_r+S-1][p_c+T-1] (0 outside the frame), o = (T-1) mod 8,
//   bins[rc][0]   = sum of A^2 over grid row class rc (0: row 0, 1: row 1, 2: row ml,
//                   3: row ml+1, 4: rows 2..ml-1) and grid columns [0, nl+2),
//   bins[rc][1+k] = A^2 at grid column (0, 1, nl, nl+1)[k] summed over the rows of class rc;
// the interior total is the staged sum minus the staged columns outside [0, nl+2) minus
// the four class rows.  Reads rows 0, 1, ml, ml+1 and, per grid row, the two 16-byte chunks
// at the left edge and the (kw - nl)/8 chunks at the right edge.
// (bins[20], the interior-row total, needs the refine's sum: ga_finish)
__device__ __forceinline__ void ga_pieces(const RefinePickArgs &a, int64_t f, int S, int T,
                                          u64 *bins /* smem [26] */) {
  const int tid = threadIdx.x, nth = blockDim.x, ml = a.ml, nl = a.nl, nl2 = nl + 2;
  if (tid < 26) bins[tid] = 0;
  __syncthreads();
  const uint16_t *A = a.frames + f * a.fstride;
  const int o = (T - 1) & 7, x0 = (T - 1) - o;   // frame column of staged column 0 (grid column -o)
  // (1) the four class rows over grid columns [0, nl+2)
  // (16-byte chunks from x0: chunk k holds grid columns 8k-o .. 8k-o+7)
  u64 r0 = 0, r1 = 0, r2 = 0, r3 = 0;
  const int nchk = (nl2 + o + 7) >> 3;
  for (int k = tid; k < 4 * nchk; k += nth) {
    const int r = k / nchk, ch = k - r * nchk;
    const int fr = (r < 2 ? r : ml + r - 2) + S - 1, fc0 = x0 + 8 * ch;
    if (fr < 0 || fr >= ml || fc0 < 0 || fc0 >= nl) continue;
    const uint4 u = *reinterpret_cast<const uint4 *>(A + (int64_t)fr * a.pitch + fc0);
    const uint32_t wv[4] = {u.x, u.y, u.z, u.w};
    uint32_t q = 0;   // eight squares of < 2^16 values would overflow: 32-bit per pair below
    u64 qs = 0;
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const uint32_t v = (x & 1) ? (wv[x >> 1] >> 16) : (wv[x >> 1] & 0xffffu);
      const int pc = 8 * ch + x - o;
      q = (pc >= 0 && pc < nl2) ? v * v : 0u;
      qs += q;
    }
    if (r == 0) r0 += qs; else if (r == 1) r1 += qs; else if (r == 2) r2 += qs; else r3 += qs;
  }
  // (2) per grid row: staged columns outside [0, nl+2) and the four edge columns
  u64 X = 0, i0 = 0, i1 = 0, i2 = 0, i3 = 0;
  const int cr0 = max(2, nl >> 3), ncs = a.kw >> 3;   // right-edge chunks [cr0, ncs), left [0, 2)
  for (int pr = tid; pr < ml + 2; pr += nth) {
    const int fr = pr + S - 1;
    if (fr < 0 || fr >= ml) continue;
    const uint16_t *row = A + (int64_t)fr * a.pitch;
    const int rc = pr < 2 ? pr : (pr >= ml ? pr - ml + 2 : 4);
    u64 c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    for (int q = 0; q < 2 + 3; ++q) {
      const int ch = q < 2 ? q : cr0 + q - 2;
      if (ch >= ncs || (q >= 2 && ch < 2)) continue;
      const int fc0 = x0 + 8 * ch;
      if (fc0 < 0 || fc0 >= nl) continue;   // 8-aligned: the chunk is wholly in or out of the row
      const uint4 u = *reinterpret_cast<const uint4 *>(row + fc0);
      const uint32_t wv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const u64 v = (x & 1) ? (wv[x >> 1] >> 16) : (wv[x >> 1] & 0xffffu), sq = v * v;
        const int pc = 8 * ch + x - o;
        if (pc < 0 || pc >= nl2) X += sq;
        else if (pc == 0) c0 += sq;
        else if (pc == 1) c1 += sq;
        else if (pc == nl) c2 += sq;
        else if (pc == nl + 1) c3 += sq;
      }
    }
    if (rc == 4) {
      i0 += c0; i1 += c1; i2 += c2; i3 += c3;
    } else {
      atomicAdd(reinterpret_cast<unsigned long long *>(bins + rc * 5 + 1), (unsigned long long)c0);
      atomicAdd(reinterpret_cast<unsigned long long *>(bins + rc * 5 + 2), (unsigned long long)c1);
      atomicAdd(reinterpret_cast<unsigned long long *>(bins + rc * 5 + 3), (unsigned long long)c2);
      atomicAdd(reinterpret_cast<unsigned long long *>(bins + rc * 5 + 4), (unsigned long long)c3);
    }
  }
  r0 = warp_sum(r0); r1 = warp_sum(r1); r2 = warp_sum(r2); r3 = warp_sum(r3);
  X = warp_sum(X); i0 = warp_sum(i0); i1 = warp_sum(i1); i2 = warp_sum(i2); i3 = warp_sum(i3);
  if ((tid & 31) == 0) {
    unsigned long long *b = reinterpret_cast<unsigned long long *>(bins);
    atomicAdd(b + 0, (unsigned long long)r0); atomicAdd(b + 5, (unsigned long long)r1);
    atomicAdd(b + 10, (unsigned long long)r2); atomicAdd(b + 15, (unsigned long long)r3);
    atomicAdd(b + 25, (unsigned long long)X);
    atomicAdd(b + 21, (unsigned long long)i0); atomicAdd(b + 22, (unsigned long long)i1);
    atomicAdd(b + 23, (unsigned long long)i2); atomicAdd(b + 24, (unsigned long long)i3);
  }
  __syncthreads();
}
__device__ __forceinline__ void ga_finish(u64 *bins, u64 total) {
  if (threadIdx.x == 0) bins[20] = total - bins[25] - bins[0] - bins[5] - bins[10] - bins[15];
  __syncthreads();
}

// The GA pieces of a batch ahead of the pick (align_tc_pipelined: on the pick stream once
// the shifts the refine starts from exist, so it runs beside the refine sums).
__global__ void __launch_bounds__(128) k_ga_pieces(RefinePickArgs a, u64 *out) {
  __shared__ u64 bins[26];
  const int64_t f = blockIdx.x;
  const int S = 2 * a.shift_in[2 * f], T = 2 * a.shift_in[2 * f + 1];
  ga_pieces(a, f, S, T, bins);
  if (threadIdx.x < 26) out[f * 26 + threadIdx.x] = bins[threadIdx.x];
}

template <int SH>
__device__ __forceinline__ void pick_apply_rows(const uint16_t *A, uint16_t *O, int pitch, int s, int t, int ml,
                                                int nl, int r0, int r1) {
  // output chunk (i, 8-column group j0): source samples a[i+s][j0+t .. j0+t+7]; the two
  // aligned vectors at ab = j0 + t - SH cover them (ab is a multiple of 8, so each vector
  // lies wholly inside or wholly outside the row); out-of-frame samples are 0
  const int groups = nl >> 3;
  constexpr int U = 4;
  if (groups <= (int)blockDim.x) {
    // a thread keeps one column group and walks rows: no per-element division, the
    // column tests once per thread
    const int rstep = blockDim.x / groups;
    if ((int)threadIdx.x >= rstep * groups) return;
    const int jj = (threadIdx.x % groups) * 8, ab = jj + t - SH;
    const bool lok = ab >= 0 && ab + 8 <= nl, hok = SH && ab + 8 >= 0 && ab + 16 <= nl;
    const uint16_t *src = A + ab;
    uint16_t *dst = O + jj;
    for (int i0 = r0 + (int)threadIdx.x / groups; i0 < r1; i0 += U * rstep) {
      uint4 lo[U], hi[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int i = i0 + k * rstep, r = i + s;
        const bool rok = i < r1 && r >= 0 && r < ml;
        const uint16_t *row = src + (int64_t)(rok ? r : 0) * pitch;
        lo[k] = (rok && lok) ? __ldcs(reinterpret_cast<const uint4 *>(row)) : make_uint4(0, 0, 0, 0);
        hi[k] = (rok && hok) ? __ldcs(reinterpret_cast<const uint4 *>(row + 8)) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int i = i0 + k * rstep;
        if (i >= r1) continue;
        const uint32_t w[8] = {lo[k].x, lo[k].y, lo[k].z, lo[k].w, hi[k].x, hi[k].y, hi[k].z, hi[k].w};
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int e2 = SH + 2 * q;
          o[q] = (e2 & 1) ? __funnelshift_r(w[e2 >> 1], w[(e2 >> 1) + 1], 16) : w[e2 >> 1];
        }
        __stcs(reinterpret_cast<uint4 *>(dst + (int64_t)i * nl), make_uint4(o[0], o[1], o[2], o[3]));
      }
    }
    return;
  }
  const int total = (r1 - r0) * groups;
  for (int e0 = threadIdx.x; e0 < total; e0 += U * blockDim.x) {
    uint4 lo[U], hi[U];
    int ii[U], jj[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int e = e0 + k * blockDim.x;
      const int ec = e < total ? e : 0;
      ii[k] = r0 + ec / groups;
      jj[k] = (ec % groups) * 8;
      const int r = ii[k] + s, ab = jj[k] + t - SH;
      const bool rok = e < total && r >= 0 && r < ml;
      const uint16_t *row = A + (int64_t)(rok ? r : 0) * pitch;
      lo[k] = (rok && ab >= 0 && ab + 8 <= nl) ? __ldcs(reinterpret_cast<const uint4 *>(row + ab)) : make_uint4(0, 0, 0, 0);
      hi[k] = (SH && rok && ab + 8 >= 0 && ab + 16 <= nl) ? __ldcs(reinterpret_cast<const uint4 *>(row + ab + 8))
                                                          : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int e = e0 + k * blockDim.x;
      if (e >= total) continue;
      const uint32_t w[8] = {lo[k].x, lo[k].y, lo[k].z, lo[k].w, hi[k].x, hi[k].y, hi[k].z, hi[k].w};
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e2 = SH + 2 * q;
        o[q] = (e2 & 1) ? __funnelshift_r(w[e2 >> 1], w[(e2 >> 1) + 1], 16) : w[e2 >> 1];
      }
      __stcs(reinterpret_cast<uint4 *>(O + (int64_t)ii[k] * nl + jj[k]), make_uint4(o[0], o[1], o[2], o[3]));
    }
  }
}

// CTA (frame f, part) with gridDim.x = B * parts: argmin of the nine candidates (every
// part computes it; part 0 stores it), then (level 0) rows [part ml/parts, ...) of the
// corrected frame -- small batches (the closed-loop case) spread one frame over many SMs.
__global__ void __launch_bounds__(256) k_refine_pick(RefinePickArgs a) {
  __shared__ int res[2];
  __shared__ u64 gbins[26];
  pdl_enter();
  const int parts = a.parts;
  const int64_t f = blockIdx.x / parts;
  const int part = blockIdx.x % parts;
  const int S = 2 * a.shift_in[2 * f], T = 2 * a.shift_in[2 * f + 1];
  const int ml = a.ml, nl = a.nl;
  if (a.ga_total) {
    if (a.gbin) {
      if (threadIdx.x < 26) gbins[threadIdx.x] = a.gbin[f * 26 + threadIdx.x];
      __syncthreads();
    } else {
      ga_pieces(a, f, S, T, gbins);
    }
    ga_finish(gbins, a.acc[f * 18 + 9]);
  }
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    u64 *acc = a.acc + f * 18;
    Key k{~0ull, ~0u};
    if (lane < 9) {
      const int c = lane;
      const u64 h = acc[c];
      u64 ga;
      if (a.ga_total) {
        // row classes of u' (0: rows 0, 1, interior; 1: 1, interior, ml; 2: interior, ml,
        // ml+1) minus the two grid columns outside [v', v'+nl) (0: nl, nl+1; 1: 0, nl+1; 2: 0, 1)
        const int up = c / 3, vp = c % 3, ex1 = vp == 0 ? 3 : 1, ex2 = vp == 2 ? 2 : 4;
        const int q0 = up == 0 ? 0 : (up == 1 ? 1 : 4), q1 = up == 0 ? 1 : (up == 1 ? 4 : 2), q2 = up == 0 ? 4 : (up == 1 ? 2 : 3);
        ga = gbins[q0 * 5] - gbins[q0 * 5 + ex1] - gbins[q0 * 5 + ex2] + gbins[q1 * 5] - gbins[q1 * 5 + ex1] -
             gbins[q1 * 5 + ex2] + gbins[q2 * 5] - gbins[q2 * 5 + ex1] - gbins[q2 * 5 + ex2];
      } else {
        ga = acc[9 + c];
      }
      const int s = S + c / 3 - 1, t = T + c % 3 - 1, n1 = nl + 1;
      const int i0 = max(0, -s), i1 = ml - max(0, s), j0 = max(0, -t), j1 = nl - max(0, t);
      const u64 gb = a.pb2[(int64_t)i1 * n1 + j1] - a.pb2[(int64_t)i0 * n1 + j1] -
                     a.pb2[(int64_t)i1 * n1 + j0] + a.pb2[(int64_t)i0 * n1 + j0];
      const u64 N = ga + gb - 2 * h;
      const double area = (double)((ml - abs(s)) * (nl - abs(t)));
      const double fv = (double)N / (a.scale * area);
      k = Key{(u64)__double_as_longlong(fv), (unsigned)c};   // rank == (s,t) lexicographic order
    }
    k = warp_min_key(k);
    if (lane == 0) {
      const int s = S + (int)(k.idx / 3) - 1, t = T + (int)(k.idx % 3) - 1;
      if (part == 0) {
        a.shift_out[2 * f] = s;
        a.shift_out[2 * f + 1] = t;
        if (a.f_out) a.f_out[f] = __longlong_as_double((long long)k.f);
      }
      res[0] = s;
      res[1] = t;
    }
  }
  if (parts == 1 && threadIdx.x < 18) a.acc[f * 18 + threadIdx.x] = 0;   // ready for the next call
  if (!a.corrected) return;
  __syncthreads();
  const int s = res[0], t = res[1];
  const uint16_t *A = a.frames + f * a.fstride;
  uint16_t *O = a.corrected + f * (int64_t)ml * nl;
  const int r0 = (int)((int64_t)part * ml / parts), r1 = (int)((int64_t)(part + 1) * ml / parts);
  switch (t & 7) {
    case 0: pick_apply_rows<0>(A, O, a.pitch, s, t, ml, nl, r0, r1); break;
    case 1: pick_apply_rows<1>(A, O, a.pitch, s, t, ml, nl, r0, r1); break;
    case 2: pick_apply_rows<2>(A, O, a.pitch, s, t, ml, nl, r0, r1); break;
    case 3: pick_apply_rows<3>(A, O, a.pitch, s, t, ml, nl, r0, r1); break;
    case 4: pick_apply_rows<4>(A, O, a.pitch, s, t, ml, nl, r0, r1); break;
    case 5: pick_apply_rows<5>(A, O, a.pitch, s, t, ml, nl, r0, r1); break;
    case 6: pick_apply_rows<6>(A, O, a.pitch, s, t, ml, nl, r0, r1); break;
    default: pick_apply_rows<7>(A, O, a.pitch, s, t, ml, nl, r0, r1); break;
  }
}

// -------------------------------------------------------------- host helpers
// Tensor maps (driver entry point fetched through the runtime: no -lcuda).
inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}
// 3-D u16 tensor [frames][rows][cols] with row pitch `pitch` and frame stride `fstride`
// (elements); box = bw columns x bh rows x 1 frame; out-of-bounds elements read as 0.
inline bool tmap_u16_3d(CUtensorMap *tm, const void *base, int cols, int rows, int64_t frames, int pitch,
                        int64_t fstride, int bw, int bh) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)frames};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch * 2, (cuuint64_t)fstride * 2};
  const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void *>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace moco
