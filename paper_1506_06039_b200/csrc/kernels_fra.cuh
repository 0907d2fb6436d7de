// kernels_fra.cuh -- S5 refine + S4 pick + S6 apply at the last pyramid level with the
// frame RESIDENT on chip: one thread-block cluster per frame, each CTA holding a band of
// the frame's rows in shared memory, so the frame crosses HBM exactly once for the refine
// sums, the argmin and the corrected-frame write (frame in + corrected out: the roofline
// bytes of the step).  Replaces k_refine_tc + k_ga_pieces +
// k_refine_pick (which read the frame twice) where it fits.
//
// The +-1 refinement ("f_{2s+u,2t+v} are computed for u,v in {0,-1,1}"), with
// (S, T) = 2 (s, t) of the coarser level, needs per frame and candidate (u, v)
//   H(u,v)  = sum_{i<ml, j<nl} a[i+S+u][j+T+v] b[i][j]      (cross term)
//   GA(u,v) = sum_{i<ml, j<nl} a[i+S+u][j+T+v]^2            (frame energy)
// with a = 0 outside the frame; GB(u,v) comes from the plan's 2-D prefix table of b^2 and
// N = GA + GB - 2H, f = N / (16^l Area), argmin of the key (f, s, t) (R4).
//
// Work layout (v4).  Cluster c takes frames c, c + nclusters, ...; CTA q of the cluster
// holds frame rows [q rpc, (q+1) rpc) (Q = 8 at 512^2: 64-row bands) in one of three band
// slices (bulk copies in 16-row chunks, one "full" mbarrier per chunk and one "released"
// mbarrier per slice; the last warp to release a slice loads the frame three ahead into
// it), two zero guard rows on either side, and accumulates every (template row i, frame
// row r = i+S+u) pair with r in its band.  Eight compute warps: a row of nl/8 16-byte
// chunks spans WPR warps (one chunk per lane), the CTA's template rows split into
// RB = 8/WPR contiguous row blocks.  A lane keeps the three frame rows i+S-1, i+S, i+S+1
// of its chunk in registers (sliding window, one 16-byte shared load per template row)
// and reads the template straight from global memory (L2-resident, prefetched three rows
// ahead) out of per-plan copies, shifted so that the 12 template pixels under its chunk
// at the column shifts T-1, T, T+1 are one 16-byte-aligned run, and pre-split into dp2a
// operands (k_fra_tcopy).  The nine H sums are 16x8-bit dot products: the u16 frame word
// (two pixels) is the 16-bit operand of dp2a as it sits in memory, the template word
// regrouped into (lo, lo, hi, hi) bytes, so H = sum dp2a_lo + 2^8 sum dp2a_hi exactly
// (values < 2^14; 32-bit partials flushed every FRA_HFLUSH rows).  GA: dp2a pair sums of
// a^2 over the rows every u pairs, minus per v the strip columns outside the template's
// range; the <= 2 rows at each end that only some u pair by one warp.  Per-warp butterfly
// reduction of the 12 sums; each CTA pushes its partials into every CTA of the cluster
// (DSMEM stores) and arrives on the cluster barrier, computes the NEXT frame's partials,
// and only then waits (software pipelining: a CTA that is ahead keeps working); every
// warp takes the argmin from its local copy and the CTA writes the corrected rows whose
// source rows it holds straight from shared memory.
// Measured (C2, 1,184 frames): 0.66 us/frame on 120 SMs (15 clusters of 8 at one CTA per
// SM) against 0.34 for k_refine_tc + k_ga_pieces + k_refine_pick: opt-in (MOCO_FRA=1),
// bit-identical.
#pragma once

namespace moco {

constexpr int FRA_CW = 8;                        // compute warps
constexpr int FRA_THREADS = 32 * FRA_CW;         // (the last warp to release a slice issues its next frame)
constexpr int FRA_CR = 16;                       // frame rows per slice chunk
constexpr int FRA_MAXCH = 16;                    // slice chunks at most
constexpr int FRA_GUARD = 2;                     // zero rows above and below the band
constexpr int FRA_HDR = 10 * 1024;              // barriers, partials, reduction scratch
constexpr int FRA_NBUF = 3;                      // frame slices per CTA (frames in flight)
constexpr int FRA_HFLUSH = 96;                   // template rows per 32-bit H partial (vb <= 14)

struct FraGeom {
  int Q;          // CTAs per cluster = per frame
  int rpc;        // frame rows per CTA
  int nchunk;     // slice chunks per CTA
  int NCH;        // 16-byte chunks per row (nl / 8)
  int WPR;        // warps per row (ceil(NCH / 32)), a power of two <= 8
  int RB;         // row blocks = FRA_CW / WPR
  int slice_bytes, smem;
  int m;          // template-copy margin, 8-pixel blocks
  int WT;         // template-copy row length (pixels)
  int gflush;     // frame rows per 32-bit dp2a pair sum of a^2
  int ncl;        // clusters launched (co-resident clusters, from the occupancy query)
};

struct FraArgs {
  const uint16_t *frames;   // level-l images, row pitch `pitch`, frame stride `fstride` (elements)
  int64_t fstride;
  int pitch;
  const uint32_t *tcopy;    // [4][E/O][ml][WT/2] shifted, pre-split template copies (k_fra_tcopy)
  const u64 *pb2;           // 2-D prefix table of b^2, (ml+1) x (nl+1)
  int ml, nl;
  double scale;             // 16^l
  int B;
  const int32_t *shift_in;  // [B][2] at level l+1
  int32_t *shift_out;       // [B][2] at level l
  double *f_out;            // [B] or null
  uint16_t *corrected;      // [B][ml][nl] or null (level 0)
  FraGeom g;
};

// Geometry for an ml x nl level with |T| <= tmax: the smallest cluster (<= 8 CTAs) whose
// CTA holds FRA_NBUF row bands; nl a multiple of 8 with at most 32 FRA_CW chunks per row,
// pitches multiples of 8 samples, values < 2^vb, vb <= 14.
inline bool fra_make(FraGeom *g, int ml, int nl, int pitch, int vb, int tmax) {
  if (vb > 14 || nl % 8 != 0 || pitch % 8 != 0 || ml < 4) return false;
  const int NCH = nl / 8;
  if (NCH > 32 * FRA_CW) return false;
  int WPR = 1;
  while (32 * WPR < NCH) WPR *= 2;
  int pick = 0;
  for (int Q = 1; Q <= 8 && !pick; Q *= 2) {
    const int rpc = (ml + Q - 1) / Q;
    const int nchunk = (rpc + FRA_CR - 1) / FRA_CR;
    const int slice = (nchunk * FRA_CR + 2 * FRA_GUARD) * pitch * 2;
    if (nchunk <= FRA_MAXCH && FRA_HDR + FRA_NBUF * slice <= 227 * 1024) pick = Q;
  }
  if (!pick) return false;
  g->Q = pick;
  g->rpc = (ml + pick - 1) / pick;
  g->nchunk = (g->rpc + FRA_CR - 1) / FRA_CR;
  g->NCH = NCH; g->WPR = WPR; g->RB = FRA_CW / WPR;
  g->slice_bytes = (g->nchunk * FRA_CR + 2 * FRA_GUARD) * pitch * 2;
  g->smem = FRA_HDR + FRA_NBUF * g->slice_bytes;
  g->m = tmax / 8 + 2;
  g->WT = nl + 16 * g->m + 16;
  // a 16-byte chunk adds <= 8 (2^vb - 1) 255 to a 32-bit dp2a pair sum per row
  g->gflush = (int)std::max(1.0, std::min(1024.0, std::floor(4294967295.0 / (8.0 * (std::ldexp(1.0, vb) - 1.0) * 255.0))));
  g->ncl = 0;
  return true;
}
inline size_t fra_tcopy_bytes(const FraGeom &g, int ml) { return (size_t)8 * ml * (g.WT / 2) * 4; }

// (lo0, lo1, hi0, hi1) bytes of a word holding two u16 pixels: the 8-bit operand of dp2a
__host__ __device__ __forceinline__ uint32_t fra_split_pair(uint32_t p0, uint32_t p1) {
  return (p0 & 255u) | ((p1 & 255u) << 8) | ((p0 >> 8) << 16) | ((p1 >> 8) << 24);
}

// Shifted, pre-split template copies.  Copy k (SH = 2k in {0,2,4,6}) is the template row
// shifted so that pixel p holds b[i][p + SH - OFF] (0 outside the template), OFF = 2 + 8m;
// a lane with frame chunk c and column shift T (even; SH = (-T) mod 8, kT = (-T - SH)/8)
// finds the template pixels [8c - T - 2, 8c - T + 10) at copy pixels p0 + [0, 12),
// p0 = 8(c + kT + m).  Stored as dp2a operands, WW = WT/2 words per row:
//   E_k[i][q] = split(pixels 2q+2, 2q+3)   (the pairs under the lane's pixels at v = 0)
//   O_k[i][q] = split(pixels 2q+1, 2q+2)   (v = +1: O[j], v = -1: O[j+1])
// so a lane reads E[q0 .. q0+3] and O[q0 .. q0+4], q0 = p0/2: 16-byte aligned.
// Layout [k][E/O][ml][WW] u32.
__global__ void k_fra_tcopy(const uint16_t *__restrict__ b, int pitch, int ml, int nl, int m, int WT,
                            uint32_t *__restrict__ out) {
  const int WW = WT / 2;
  const int64_t per = (int64_t)ml * WW, total = 8 * per;
  const int off = 2 + 8 * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int ke = (int)(e / per), k = ke >> 1, odd = ke & 1;
    const int64_t r = e % per;
    const int i = (int)(r / WW), q = (int)(r % WW);
    const int p = 2 * q + (odd ? 1 : 2);   // first pixel of the pair (copy coordinates)
    const int x0 = p + 2 * k - off, x1 = x0 + 1;
    const uint32_t v0 = (x0 >= 0 && x0 < nl) ? b[(int64_t)i * pitch + x0] : 0u;
    const uint32_t v1 = (x1 >= 0 && x1 < nl) ? b[(int64_t)i * pitch + x1] : 0u;
    out[e] = fra_split_pair(v0, v1);
  }
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ u64 ld_dsmem_u64(const void *local, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  u64 v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(ra) : "memory");
  return v;
}
// named barrier of the compute warps only
__device__ __forceinline__ void fra_bar_compute() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * FRA_CW) : "memory");
}

__device__ __forceinline__ uint32_t fra_split(uint32_t w) { return __byte_perm(w, 0, 0x3120); }

// one template row's dp2a operands under the lane's chunk: E[0..3] (v = 0), O[0..4]
struct FraT {
  uint32_t e[4], o[5];
};
__device__ __forceinline__ void fra_ldt(FraT &t, const uint32_t *pe, const uint32_t *po) {
  const uint4 x = __ldg(reinterpret_cast<const uint4 *>(pe));
  const uint4 y = __ldg(reinterpret_cast<const uint4 *>(po));
  t.e[0] = x.x; t.e[1] = x.y; t.e[2] = x.z; t.e[3] = x.w;
  t.o[0] = y.x; t.o[1] = y.y; t.o[2] = y.z; t.o[3] = y.w;
  t.o[4] = __ldg(po + 4);
}

// One template row against the frame rows i+S-1, i+S, i+S+1 (am, a0, ap): candidate
// q = 3(u+1) + (v+1).  Frame pixel 8c+2k+e meets template pixel 8c+2k+e-T-v.
__device__ __forceinline__ void fra_row(const FraT &t, const uint4 &am, const uint4 &a0, const uint4 &ap,
                                        uint32_t (&lo)[9], uint32_t (&hi)[9]) {
  const uint32_t aw[3][4] = {{am.x, am.y, am.z, am.w}, {a0.x, a0.y, a0.z, a0.w}, {ap.x, ap.y, ap.z, ap.w}};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t sp[3] = {t.o[k + 1], t.e[k], t.o[k]};   // v = -1, 0, +1
#pragma unroll
    for (int up = 0; up < 3; ++up)
#pragma unroll
      for (int vp = 0; vp < 3; ++vp) {
        lo[up * 3 + vp] = __dp2a_lo(aw[up][k], sp[vp], lo[up * 3 + vp]);
        hi[up * 3 + vp] = __dp2a_hi(aw[up][k], sp[vp], hi[up * 3 + vp]);
      }
  }
}

// H over template rows [ba, bb): fr0 = slice address of frame row 0 at this lane's chunk,
// te / to = the lane's E / O template words of row 0 (row stride WW words).
__device__ __forceinline__ void fra_h(const unsigned char *fr0, int pitch2, const uint32_t *te, const uint32_t *to,
                                      int WW, int ba, int bb, int S, u64 (&H)[9]) {
#pragma unroll
  for (int q = 0; q < 9; ++q) H[q] = 0;
  if (ba >= bb) return;
  auto lda = [&](int r) { return *reinterpret_cast<const uint4 *>(fr0 + (ptrdiff_t)r * pitch2); };
  auto ldt = [&](FraT &t, int i) {
    const int64_t o = (int64_t)min(i, bb - 1) * WW;
    fra_ldt(t, te + o, to + o);
  };
  uint4 A0 = lda(ba + S - 1), A1 = lda(ba + S), A2;
  FraT T0, T1, T2;
  ldt(T0, ba);
  ldt(T1, ba + 1);
  ldt(T2, ba + 2);
  int i = ba;
  while (i < bb) {
    const int se = min(bb, i + FRA_HFLUSH);
    uint32_t lo[9], hi[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) lo[q] = hi[q] = 0;
    // three rows per round so the window rotates through named registers (no moves)
    for (; i + 3 <= se; i += 3) {
      A2 = lda(i + S + 1);
      fra_row(T0, A0, A1, A2, lo, hi);
      ldt(T0, i + 3);
      A0 = lda(i + S + 2);
      fra_row(T1, A1, A2, A0, lo, hi);
      ldt(T1, i + 4);
      A1 = lda(i + S + 3);
      fra_row(T2, A2, A0, A1, lo, hi);
      ldt(T2, i + 5);
    }
    if (i < se) {   // the block's last one or two rows (FRA_HFLUSH % 3 == 0)
      A2 = lda(i + S + 1);
      fra_row(T0, A0, A1, A2, lo, hi);
      if (i + 1 < se) {
        A0 = lda(i + S + 2);
        fra_row(T1, A1, A2, A0, lo, hi);
      }
      i = se;
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) H[q] += (u64)lo[q] + ((u64)hi[q] << 8);
  }
}
static_assert(FRA_HFLUSH % 3 == 0, "H flush interval must keep the window rotation");

// Warp reduce-scatter of 16 values: lanes 2j and 2j+1 return the warp sum of value j.
__device__ __forceinline__ u64 fra_reduce16(u64 (&v)[16], int lane) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const bool up = lane & 16;
    const u64 send = up ? v[k] : v[k + 8], keep = up ? v[k + 8] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool up = lane & 8;
    const u64 send = up ? v[k] : v[k + 4], keep = up ? v[k + 4] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const bool up = lane & 4;
    const u64 send = up ? v[k] : v[k + 2], keep = up ? v[k + 2] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  {
    const bool up = lane & 2;
    const u64 send = up ? v[0] : v[1], keep = up ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// Corrected rows r in [rlo, rhi) (stepping rstep) of the band: out[r-s][j] = a[r][j+t] (0
// outside), 16-byte streaming stores; the lane's output chunk q and its two source blocks
// are fixed for the frame.
template <int SH>
__device__ __forceinline__ void fra_apply_rows(const unsigned char *srow0, int pitch2, uint16_t *O, int rlo, int rhi,
                                               int rstep, int s, int nl, int q, int bl, bool okl, bool okh) {
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int r = rlo; r < rhi; r += rstep) {
    const unsigned char *src = srow0 + (ptrdiff_t)r * pitch2 + 16 * bl;
    const uint4 lo = okl ? *reinterpret_cast<const uint4 *>(src) : z;
    const uint4 hi = (SH && okh) ? *reinterpret_cast<const uint4 *>(src + 16) : z;
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint32_t ov[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e2 = SH + 2 * k;
      ov[k] = (e2 & 1) ? __funnelshift_r(w[e2 >> 1], w[(e2 >> 1) + 1], 16) : w[e2 >> 1];
    }
    __stcs(reinterpret_cast<uint4 *>(O + (int64_t)(r - s) * nl + 8 * q), make_uint4(ov[0], ov[1], ov[2], ov[3]));
  }
}

// Per-CTA shared memory: header (chunk barriers per slice, the cluster's partials per
// frame slot, reduction scratch), then FRA_NBUF slices.
constexpr int FRA_OFF_CNT = FRA_NBUF * FRA_MAXCH * 8 + FRA_NBUF * 8;   // [NBUF] int: warps done with a slice
constexpr int FRA_NSLOT = 4;                                        // partial slots (frames in the exchange)
constexpr int FRA_OFF_PART = 1024;                                  // [NSLOT][8 ranks][24] u64
constexpr int FRA_OFF_RED = FRA_OFF_PART + FRA_NSLOT * 8 * 24 * 8;  // [2][FRA_CW][12] u64
constexpr int FRA_OFF_REDE = FRA_OFF_RED + 2 * FRA_CW * 12 * 8;     // [2][16] u64
static_assert(FRA_OFF_REDE + 2 * 16 * 8 <= FRA_HDR, "fra header");

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire;" ::: "memory"); }
__device__ __forceinline__ void st_dsmem_u64(void *local, uint32_t rank, u64 v) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"(v) : "memory");
}

// Frame j of a cluster lives in slice j % FRA_NBUF.  Per CTA and frame: H and GA partials
// -> pushed into every CTA's partial slot j % 3 -> cluster barrier arrive; the barrier is
// waited for only after the NEXT frame's partials (software pipelining: a CTA that is
// ahead keeps computing instead of waiting), then every compute warp takes the argmin
// from its local copy of the cluster's partials and the CTA writes its corrected rows.
__global__ void __launch_bounds__(FRA_THREADS, 1) k_refine_frame(FraArgs a) {
  static_assert(FRA_OFF_CNT + FRA_NBUF * 4 <= FRA_OFF_PART, "fra header");
  extern __shared__ __align__(1024) unsigned char fra_raw[];
  unsigned char *smem = fra_raw;
  const FraGeom &g = a.g;
  uint64_t *fbar = reinterpret_cast<uint64_t *>(smem);              // [NBUF][MAXCH] slice chunk landed
  uint64_t *ebar = fbar + FRA_NBUF * FRA_MAXCH;                     // [NBUF] slice released (FRA_CW warps)
  int *dcnt = reinterpret_cast<int *>(smem + FRA_OFF_CNT);          // [NBUF] warps done with the slice
  u64 *part = reinterpret_cast<u64 *>(smem + FRA_OFF_PART);         // [3][8][24]: H 0..8, GA core 9..11, edge 12..20
  u64 *red = reinterpret_cast<u64 *>(smem + FRA_OFF_RED);           // [2][FRA_CW][12]
  u64 *rede = reinterpret_cast<u64 *>(smem + FRA_OFF_REDE);         // [2][16]
  unsigned char *slices = smem + FRA_HDR;                           // [NBUF] guard rows, band rows, guard rows
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int cl = (int)cluster_id_x();
  const int ml = a.ml, nl = a.nl, NCH = g.NCH, RB = g.RB, WPR = g.WPR, WT = g.WT, Q = g.Q;
  const int R0 = (int)rank * g.rpc, R1 = min(ml, R0 + g.rpc);
  const int pitch2 = a.pitch * 2;
  const int nf = cl < a.B ? (a.B - cl + g.ncl - 1) / g.ncl : 0;   // frames of this cluster
  // slice address of frame row 0 (row R0 sits after the guard rows)
  auto srow0_of = [&](int j) {
    return slices + (size_t)(j % FRA_NBUF) * g.slice_bytes + (ptrdiff_t)(FRA_GUARD - R0) * pitch2;
  };

  if (tid == 0) {
    for (int k = 0; k < FRA_NBUF * FRA_MAXCH; ++k) mbar_init(&fbar[k], 1);
    for (int k = 0; k < FRA_NBUF; ++k) {
      mbar_init(&ebar[k], FRA_CW);
      dcnt[k] = 0;
    }
    fence_mbar_init();
  }
  // zero the slices once: guard rows and never-loaded tail rows must read as 0
  for (int e = tid; e < FRA_NBUF * g.slice_bytes / 16; e += FRA_THREADS)
    reinterpret_cast<uint4 *>(slices)[e] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  __syncthreads();
  cluster_arrive();   // every CTA of the cluster runs before any partial is pushed
  cluster_wait();

  // frame j's band rows into slice j % NBUF (bulk copies, one mbarrier per 16-row chunk)
  auto issue = [&](int j) {
    const int f = cl + j * g.ncl, bf = j % FRA_NBUF;
    const int S = 2 * a.shift_in[2 * f];
    const int need0 = max(0, S - 1), need1 = min(ml, ml + S + 1);
    unsigned char *slice = slices + (size_t)bf * g.slice_bytes;
    for (int k = 0; k < g.nchunk; ++k) {
      uint64_t *fb = &fbar[bf * FRA_MAXCH + k];
      const int r0 = R0 + k * FRA_CR, r1 = min(R1, r0 + FRA_CR);
      if (r0 < r1 && r0 < need1 && r1 > need0) {
        const uint32_t bytes = (uint32_t)((r1 - r0) * pitch2);
        mbar_arrive_expect_tx(fb, bytes);
        bulk_g2s(slice + (size_t)(FRA_GUARD + k * FRA_CR) * pitch2,
                 a.frames + (int64_t)f * a.fstride + (int64_t)r0 * a.pitch, bytes, fb);
      } else {
        mbar_arrive(fb);
      }
    }
  };
  if (tid == 0)
    for (int j = 0; j < min(nf, FRA_NBUF); ++j) issue(j);

  // ================================================================== compute warps
  const int rb = warp / WPR, wc = warp % WPR;
  const int c = wc * 32 + lane;          // 16-byte chunk column of this lane
  const bool act = c < NCH;
  const int cc = act ? c : 0;

  // GB of candidate `lane` (< 9) of frame j from the 2-D prefix table of b^2
  auto gb_of = [&](int j) -> u64 {
    if (lane >= 9 || j >= nf) return 0;
    const int f = cl + j * g.ncl;
    const int s = 2 * a.shift_in[2 * f] + lane / 3 - 1, t = 2 * a.shift_in[2 * f + 1] + lane % 3 - 1;
    const int n1 = nl + 1, ci0 = max(0, -s), ci1 = ml - max(0, s), cj0 = max(0, -t), cj1 = nl - max(0, t);
    return a.pb2[(int64_t)ci1 * n1 + cj1] - a.pb2[(int64_t)ci0 * n1 + cj1] - a.pb2[(int64_t)ci1 * n1 + cj0] +
           a.pb2[(int64_t)ci0 * n1 + cj0];
  };

  // ---- H and GA partials of frame j, reduced over the CTA and pushed to every CTA
  auto partials = [&](int j) {
    const int f = cl + j * g.ncl, bf = j % FRA_NBUF;
    const uint32_t fpar = (uint32_t)((j / FRA_NBUF) & 1);
    uint64_t *fb = fbar + bf * FRA_MAXCH;
    const int S = 2 * a.shift_in[2 * f], T = 2 * a.shift_in[2 * f + 1];
    const unsigned char *srow0 = srow0_of(j);
    const unsigned char *fr0 = srow0 + 16 * cc;
    // the CTA's template rows [i0, i1) (those pairing with a frame row of the band), split
    // into RB contiguous blocks; each block waits for the chunks holding its frame rows
    const int i0 = max(0, R0 - S - 1), i1 = max(i0, min(ml, R1 - S + 1));
    const int BL = (i1 - i0 + RB - 1) / RB;
    const int ba = min(i1, i0 + rb * BL), bb = min(i1, ba + BL);
    u64 H[9];
    {
      const int ra = max(R0, ba + S - 1), rz = min(R1, bb + S + 1);
      if (ba < bb && ra < rz)
        for (int k = (ra - R0) / FRA_CR; k <= (rz - 1 - R0) / FRA_CR; ++k) mbar_wait(&fb[k], fpar);
      const int SH = (-T) & 7, kT = (-T - SH) >> 3, WW = WT >> 1;
      const uint32_t *te = a.tcopy + (int64_t)(SH >> 1) * 2 * ml * WW + 4 * (cc + kT + g.m);
      if (act) fra_h(fr0, pitch2, te, te + (int64_t)ml * WW, WW, ba, bb, S, H);
      else {
#pragma unroll
        for (int q = 0; q < 9; ++q) H[q] = 0;
      }
    }
    for (int k = 0; k < g.nchunk; ++k) mbar_wait(&fb[k], fpar);
    // GA over the rows every u pairs (the core): every column's a^2 by dp2a pair sums,
    // minus per v the columns outside the template's range (the strips)
    const int RI0 = max(0, S + 1), RI1 = min(ml, ml + S - 1);   // rows of every u
    const int RU0 = max(0, S - 1), RU1 = min(ml, ml + S + 1);   // rows of some u
    const int ra = max(R0, RI0), rz = min(R1, RI1);
    u64 gv[3];
    {
      u64 gall = 0;
      if (act) {
        uint32_t glo = 0, ghi = 0;
        int cnt = 0;
        for (int r = ra + rb; r < rz; r += RB) {
          const uint4 v = *reinterpret_cast<const uint4 *>(fr0 + (ptrdiff_t)r * pitch2);
          const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t sp = fra_split(wv[k]);
            glo = __dp2a_lo(wv[k], sp, glo);
            ghi = __dp2a_hi(wv[k], sp, ghi);
          }
          if (++cnt == g.gflush) {
            gall += (u64)glo + ((u64)ghi << 8);
            glo = ghi = 0;
            cnt = 0;
          }
        }
        gall += (u64)glo + ((u64)ghi << 8);
      }
      // strip columns (outside the range of some v): left [0, XL), right [XR, nl); every
      // compute warp takes the core rows = warp mod FRA_CW, a lane one strip column
      const int XL = min(nl, max(0, T + 1)), XR = max(0, min(nl, nl + T - 1));
      const int ns = XL + (nl - XR);
      u64 ex[3] = {0, 0, 0};
      for (int ci = lane; ci < ns; ci += 32) {
        const int col = ci < XL ? ci : XR + (ci - XL);
        u64 cs = 0;
        for (int r = ra + warp; r < rz; r += FRA_CW) {
          const uint32_t px = *reinterpret_cast<const uint16_t *>(srow0 + (ptrdiff_t)r * pitch2 + 2 * col);
          cs += (u64)(px * px);
        }
#pragma unroll
        for (int vp = 0; vp < 3; ++vp) {
          const int jj = col - T - (vp - 1);
          ex[vp] += (jj < 0 || jj >= nl) ? cs : 0ull;
        }
      }
#pragma unroll
      for (int vp = 0; vp < 3; ++vp) gv[vp] = gall - ex[vp];   // mod 2^64: the sums are exact
    }
    const int p2 = j & 1;
    {
      u64 v16[16];
#pragma unroll
      for (int q = 0; q < 9; ++q) v16[q] = H[q];
#pragma unroll
      for (int q = 0; q < 3; ++q) v16[9 + q] = gv[q];
#pragma unroll
      for (int q = 12; q < 16; ++q) v16[q] = 0;
      const u64 sum = fra_reduce16(v16, lane);
      const int idx = (lane >> 1) & 15;
      if (!(lane & 1) && idx < 12) red[(p2 * FRA_CW + warp) * 12 + idx] = sum;
    }
    // GA over the <= 4 rows only some u pair (warp 0): exact per-(u,v) sums
    if (warp == 0) {
      u64 e[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) e[q] = 0;
      for (int r = max(R0, RU0); r < min(R1, RU1); ++r) {
        if (r >= RI0 && r < RI1) {   // rows of every u: core (skip to the bottom edge)
          r = max(r, min(R1, RI1) - 1);
          continue;
        }
        for (int ch = lane; ch < NCH; ch += 32) {
          const uint4 v = *reinterpret_cast<const uint4 *>(srow0 + (ptrdiff_t)r * pitch2 + 16 * ch);
          const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
          u64 sv[3] = {0, 0, 0};
#pragma unroll
          for (int x = 0; x < 8; ++x) {
            const uint32_t px = (x & 1) ? (wv[x >> 1] >> 16) : (wv[x >> 1] & 0xffffu);
#pragma unroll
            for (int vp = 0; vp < 3; ++vp) {
              const int jj = 8 * ch + x - T - (vp - 1);
              sv[vp] += (jj >= 0 && jj < nl) ? (u64)(px * px) : 0ull;
            }
          }
#pragma unroll
          for (int up = 0; up < 3; ++up) {
            const int i = r - S - (up - 1);   // template row paired with frame row r at u
            if (i < 0 || i >= ml) continue;
#pragma unroll
            for (int vp = 0; vp < 3; ++vp) e[up * 3 + vp] += sv[vp];
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 9; ++q) e[q] = warp_sum(e[q]);
      if (lane < 9) {
        u64 x = 0;
#pragma unroll
        for (int q = 0; q < 9; ++q) x = lane == q ? e[q] : x;
        rede[p2 * 16 + lane] = x;
      }
    }
    fra_bar_compute();
    if (tid < 21) {   // push this CTA's partials into slot j % 3 of every CTA of the cluster
      u64 v = 0;
      if (tid < 12) {
#pragma unroll 4
        for (int w = 0; w < FRA_CW; ++w) v += red[(p2 * FRA_CW + w) * 12 + tid];
      } else {
        v = rede[p2 * 16 + tid - 12];
      }
      u64 *dst = part + ((j % FRA_NSLOT) * 8 + rank) * 24 + tid;
      for (int q = 0; q < Q; ++q) st_dsmem_u64(dst, (uint32_t)q, v);
    }
  };

  // ---- argmin of frame j from the local copy of the cluster's partials (every warp), apply
  auto finish = [&](int j, u64 gb) {
    const int f = cl + j * g.ncl, bf = j % FRA_NBUF;
    const int S = 2 * a.shift_in[2 * f], T = 2 * a.shift_in[2 * f + 1];
    Key key{~0ull, ~0u};
    if (lane < 9) {
      const u64 *sl = part + (j % FRA_NSLOT) * 8 * 24;
      u64 h = 0, gav = 0;
      const int vp = lane % 3;
      for (int q = 0; q < Q; ++q) {
        h += sl[q * 24 + lane];
        gav += sl[q * 24 + 9 + vp] + sl[q * 24 + 12 + lane];
      }
      const int s = S + lane / 3 - 1, t = T + vp - 1;
      const u64 N = gav + gb - 2 * h;
      const double area = (double)((ml - abs(s)) * (nl - abs(t)));
      const double fv = (double)N / (a.scale * area);
      key = Key{(u64)__double_as_longlong(fv), (unsigned)lane};   // rank == (s,t) lexicographic
    }
    key = warp_min_key(key);
    const int s = S + (int)(key.idx / 3) - 1, t = T + (int)(key.idx % 3) - 1;
    if (rank == 0 && warp == 0 && lane == 0) {
      a.shift_out[2 * f] = s;
      a.shift_out[2 * f + 1] = t;
      if (a.f_out) a.f_out[f] = __longlong_as_double((long long)key.f);
    }
    // apply (level 0): corrected rows from the resident band
    if (a.corrected) {
      const unsigned char *srow0 = srow0_of(j);
      uint16_t *O = a.corrected + (int64_t)f * ml * nl;
      if (act) {   // zero rows of this CTA's index band (no source row in the frame)
        for (int o = R0 + rb; o < min(R1, -s); o += RB)
          __stcs(reinterpret_cast<uint4 *>(O + (int64_t)o * nl + 8 * cc), make_uint4(0, 0, 0, 0));
        for (int o = max(R0, ml - s) + rb; o < R1; o += RB)
          __stcs(reinterpret_cast<uint4 *>(O + (int64_t)o * nl + 8 * cc), make_uint4(0, 0, 0, 0));
      }
      const int SHa = t & 7, ab = 8 * cc + t - SHa, bl = ab >> 3;
      const bool okl = bl >= 0 && bl < NCH, okh = bl + 1 >= 0 && bl + 1 < NCH;
      const int r0 = max(R0, max(0, s)), r1 = min(R1, min(ml, ml + s));
      if (act && r0 < r1) {
        const int rs = r0 + ((rb - r0) & (RB - 1));   // the rows = rb mod RB (RB a power of two)
        switch (SHa) {
          case 0: fra_apply_rows<0>(srow0, pitch2, O, rs, r1, RB, s, nl, cc, bl, okl, okh); break;
          case 1: fra_apply_rows<1>(srow0, pitch2, O, rs, r1, RB, s, nl, cc, bl, okl, okh); break;
          case 2: fra_apply_rows<2>(srow0, pitch2, O, rs, r1, RB, s, nl, cc, bl, okl, okh); break;
          case 3: fra_apply_rows<3>(srow0, pitch2, O, rs, r1, RB, s, nl, cc, bl, okl, okh); break;
          case 4: fra_apply_rows<4>(srow0, pitch2, O, rs, r1, RB, s, nl, cc, bl, okl, okh); break;
          case 5: fra_apply_rows<5>(srow0, pitch2, O, rs, r1, RB, s, nl, cc, bl, okl, okh); break;
          case 6: fra_apply_rows<6>(srow0, pitch2, O, rs, r1, RB, s, nl, cc, bl, okl, okh); break;
          default: fra_apply_rows<7>(srow0, pitch2, O, rs, r1, RB, s, nl, cc, bl, okl, okh); break;
        }
      }
    }
    // release the slice; the last warp to do so loads frame j + NBUF into it (the mbarrier
    // orders every warp's reads of the slice before the bulk copies' writes)
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&ebar[bf]);
      if (atomicAdd(&dcnt[bf], 1) == FRA_CW - 1) {
        dcnt[bf] = 0;
        mbar_wait(&ebar[bf], (uint32_t)((j / FRA_NBUF) & 1));
        if (j + FRA_NBUF < nf) issue(j + FRA_NBUF);
      }
    }
  };

  // Per thread: P(0) A(0), then for each j: P(j+1) W(j) A(j+1) F(j) -- P = partials pushed,
  // A / W = cluster barrier arrive (release) / wait (acquire), F = argmin + apply.  The
  // arrive right after the wait keeps the release fence clear of the apply's global stores.
  // Slot j % 4 is rewritten by P(j+4), after W(j+2), i.e. after every thread's A(j+2),
  // which follows its F(j): no CTA still reads it.
  if (nf > 0) {
    u64 gb_cur = gb_of(0);
    partials(0);
    cluster_arrive();
    for (int j = 0; j < nf; ++j) {
      const u64 gb_next = gb_of(j + 1);
      if (j + 1 < nf) partials(j + 1);
      cluster_wait();   // frame j: every CTA's partials are in
      if (j + 1 < nf) cluster_arrive();
      finish(j, gb_cur);
      gb_cur = gb_next;
    }
  }
}

}  // namespace moco
