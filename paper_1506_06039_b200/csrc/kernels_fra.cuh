// kernels_fra.cuh -- S5 refine + S4 pick + S6 apply at the last pyramid level with the
// frame RESIDENT on chip: one thread-block cluster per frame, each CTA holding a band of
// the frame's rows in shared memory, so the frame crosses HBM exactly once for the refine
// sums, the argmin and the corrected-frame write (frame in + corrected out: the roofline
// bytes of the step).
//
// The +-1 refinement ("f_{2s+u,2t+v} are computed for u,v in {0,-1,1}"), with
// (S, T) = 2 (s, t) of the coarser level, needs per frame and candidate (u, v)
//   H(u,v)  = sum_{i<ml, j<nl} a[i+S+u][j+T+v] b[i][j]      (cross term)
//   GA(u,v) = sum_{i<ml, j<nl} a[i+S+u][j+T+v]^2            (frame energy)
// with a = 0 outside the frame; GB(u,v) comes from the plan's 2-D prefix table of b^2 and
// N = GA + GB - 2H, f = N / (16^l Area), argmin of the key (f, s, t) (R4).
//
// Work layout.  Cluster c takes frames c, c + nclusters, ...; CTA q of the cluster holds
// frame rows [q rpc, (q+1) rpc) (bulk copies in 16-row chunks, one "full" and one "empty"
// mbarrier each, two zero guard rows on either side) and accumulates every (template row
// i, frame row r = i+S+u) pair with r in its band.  Warp 8 is the producer (bulk copies);
// warps 0-7 compute.  The CTA's template rows are split into RB contiguous row blocks, one
// per group of WPR warps (a row of nl/8 16-byte chunks spans WPR warps, one chunk per
// lane); each row block streams its template rows through its own two-slot sub-ring.  A
// lane keeps the three frame rows i+S-1, i+S, i+S+1 of its chunk in registers (sliding
// window, one 16-byte shared load per template row) and forms the nine H sums with 16x8-bit
// dot products: the u16 frame word (two pixels) is the 16-bit operand of dp2a as it sits
// in memory, the template word regrouped into (lo, lo, hi, hi) bytes, so H = sum dp2a_lo +
// 2^8 sum dp2a_hi exactly (values < 2^14; 32-bit partials flushed every sub-ring slot).
// GA: per-pixel column sums over the rows every u pairs (64-bit IMAD.WIDE), masked per v
// once per frame; the <= 4 edge rows separately.  The CTAs exchange their 18 partial sums
// through distributed shared memory (one cluster barrier per frame), every CTA takes the
// same argmin, and each writes the corrected rows whose source rows it holds (zero rows:
// those of its own index band with no source) straight from shared memory, releasing each
// chunk to the producer for the next frame's rows.
#pragma once

namespace moco {

constexpr int FRA_CW = 8;                        // compute warps
constexpr int FRA_THREADS = 32 * (FRA_CW + 1);   // + one producer warp
constexpr int FRA_CR = 16;                       // frame rows per slice chunk
constexpr int FRA_TRB = 8;                       // template rows per sub-ring slot
constexpr int FRA_NS = 2;                        // slots per sub-ring
constexpr int FRA_MAXCH = 16;                    // slice chunks at most
constexpr int FRA_GUARD = 2;                     // zero rows above and below the band
constexpr int FRA_HDR = 4096;                    // barriers, partials, reduction scratch

struct FraGeom {
  int Q;          // CTAs per cluster = per frame
  int rpc;        // frame rows per CTA
  int nchunk;     // slice chunks per CTA
  int NCH;        // 16-byte chunks per row (nl / 8)
  int WPR;        // warps per row (ceil(NCH / 32)), a power of two <= 8
  int RB;         // row blocks = FRA_CW / WPR
  int slice_bytes, tslot_bytes, smem;
  int ncl;        // clusters launched (co-resident clusters, from the occupancy query)
};

struct FraArgs {
  const uint16_t *frames;   // level-l images, row pitch `pitch`, frame stride `fstride` (elements)
  int64_t fstride;
  int pitch;
  const uint16_t *tpl;      // level-l template, row pitch tpitch
  int tpitch;
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

// Geometry for an ml x nl level: the smallest cluster (<= 8 CTAs) whose row bands fit
// 144 KB of shared memory next to the template sub-rings; nl a multiple of 8 with at most
// 256 chunks per row, pitches multiples of 8 samples, values < 2^14.
inline bool fra_make(FraGeom *g, int ml, int nl, int pitch, int tpitch, int vb) {
  if (vb > 14 || nl % 8 != 0 || pitch % 8 != 0 || tpitch % 8 != 0 || ml < 4) return false;
  const int NCH = nl / 8;
  if (NCH > 32 * FRA_CW) return false;
  int WPR = 1;
  while (32 * WPR < NCH) WPR *= 2;
  for (int Q = 1; Q <= 8; Q *= 2) {
    const int rpc = (ml + Q - 1) / Q;
    const int nchunk = (rpc + FRA_CR - 1) / FRA_CR;
    const int slice = (nchunk * FRA_CR + 2 * FRA_GUARD) * pitch * 2;
    if (nchunk > FRA_MAXCH || slice > 144 * 1024) continue;
    g->Q = Q; g->rpc = rpc; g->nchunk = nchunk; g->NCH = NCH; g->WPR = WPR; g->RB = FRA_CW / WPR;
    g->slice_bytes = slice;
    g->tslot_bytes = FRA_TRB * tpitch * 2;
    g->smem = FRA_HDR + slice + g->RB * FRA_NS * g->tslot_bytes;
    g->ncl = 0;
    return g->smem <= 227 * 1024;
  }
  return false;
}

// (not .aligned: the producer warp reaches it from a lane-0-only code path)
__device__ __forceinline__ void cluster_arrive_wait() {
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
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
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// named barrier of the compute warps only
__device__ __forceinline__ void fra_bar_compute() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * FRA_CW) : "memory");
}

// (lo0, lo1, hi0, hi1) bytes of a word holding two u16 pixels: the 8-bit operand of dp2a
__device__ __forceinline__ uint32_t fra_split(uint32_t w) { return __byte_perm(w, 0, 0x3120); }

// One template row (three 16-byte blocks around the lane's chunk: b0-1, b0, b0+1) against
// the frame rows i+S-1, i+S, i+S+1 (a0, a1, a2).  SH = (8c - T) mod 8 (T even).
template <int SH>
__device__ __forceinline__ void fra_row(const uint4 &t0, const uint4 &t1, const uint4 &t2, const uint4 &a0,
                                        const uint4 &a1, const uint4 &a2, uint32_t (&lo)[9], uint32_t (&hi)[9]) {
  const uint32_t W[12] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w, t2.x, t2.y, t2.z, t2.w};
  uint32_t sp[3][4];   // [v+1][k]: template pair under frame pixels (8c+2k, 8c+2k+1) at shift T+v
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int e = 4 + SH / 2 + k;
    sp[1][k] = fra_split(W[e]);                                  // v = 0:  columns 8c+2k-T, +1
    sp[2][k] = fra_split(__funnelshift_r(W[e - 1], W[e], 16));   // v = +1: one column left
    sp[0][k] = fra_split(__funnelshift_r(W[e], W[e + 1], 16));   // v = -1: one column right
  }
  const uint32_t aw[3][4] = {{a0.x, a0.y, a0.z, a0.w}, {a1.x, a1.y, a1.z, a1.w}, {a2.x, a2.y, a2.z, a2.w}};
#pragma unroll
  for (int up = 0; up < 3; ++up)
#pragma unroll
    for (int vp = 0; vp < 3; ++vp)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        lo[up * 3 + vp] = __dp2a_lo(aw[up][k], sp[vp][k], lo[up * 3 + vp]);
        hi[up * 3 + vp] = __dp2a_hi(aw[up][k], sp[vp][k], hi[up * 3 + vp]);
      }
}

// H over the template rows [ia, ib) held in one sub-ring slot (slot row 0 = row ia): the
// sliding window (a0, a1, a2) = frame rows (ia+S-1, ia+S, ia+S+1) continues across slots.
// srow0 = slice address of frame row 0.
template <int SH>
__device__ __forceinline__ void fra_hslot(const unsigned char *slot, int tpitch2, const unsigned char *srow0,
                                          int pitch2, int ia, int ib, int S, int c, int b0, bool ok0, bool ok1,
                                          bool ok2, uint4 &a0, uint4 &a1, uint4 &a2, u64 (&H)[9], u64 (&Hh)[9]) {
  uint32_t lo[9], hi[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) lo[q] = hi[q] = 0;
  const uint4 z = make_uint4(0, 0, 0, 0);
  // three rows per round so the window rotates through named registers (no moves)
  for (int i = ia; i < ib; i += 3) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int ii = i + d;
      if (ii >= ib) break;
      const unsigned char *tr = slot + (size_t)(ii - ia) * tpitch2 + 16 * b0;
      const uint4 t0 = ok0 ? *reinterpret_cast<const uint4 *>(tr - 16) : z;
      const uint4 t1 = ok1 ? *reinterpret_cast<const uint4 *>(tr) : z;
      const uint4 t2 = ok2 ? *reinterpret_cast<const uint4 *>(tr + 16) : z;
      const uint4 an = *reinterpret_cast<const uint4 *>(srow0 + (ptrdiff_t)(ii + S + 1) * pitch2 + 16 * c);
      if (d == 0) { a2 = an; fra_row<SH>(t0, t1, t2, a0, a1, a2, lo, hi); }
      if (d == 1) { a0 = an; fra_row<SH>(t0, t1, t2, a1, a2, a0, lo, hi); }
      if (d == 2) { a1 = an; fra_row<SH>(t0, t1, t2, a2, a0, a1, lo, hi); }
    }
    // restore the order (a0, a1, a2) = frame rows (i'+S-1, i'+S, i'+S+1) of the next row i'
    const int done = min(3, ib - i);
    if (done == 1) { const uint4 x = a0; a0 = a1; a1 = a2; a2 = x; }
    else if (done == 2) { const uint4 x = a2; a2 = a1; a1 = a0; a0 = x; }
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    H[q] += lo[q];
    Hh[q] += hi[q];
  }
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

__global__ void __launch_bounds__(FRA_THREADS, 1) k_refine_frame(FraArgs a) {
  extern __shared__ __align__(1024) unsigned char fra_raw[];
  unsigned char *smem = fra_raw;
  const FraGeom &g = a.g;
  uint64_t *fbar = reinterpret_cast<uint64_t *>(smem);         // [FRA_MAXCH] slice chunk landed
  uint64_t *ebar = fbar + FRA_MAXCH;                           // [FRA_MAXCH] slice chunk released
  uint64_t *tfull = ebar + FRA_MAXCH;                          // [8][NS] sub-ring slot landed
  uint64_t *tempty = tfull + 8 * FRA_NS;                       // [8][NS] sub-ring slot released
  u64 *part = reinterpret_cast<u64 *>(smem + 512);             // [2][32]: H 0..8, GA 9..17
  u64 *red = reinterpret_cast<u64 *>(smem + 1024);             // [8 warps][18]
  int *res = reinterpret_cast<int *>(smem + 2304);             // s, t
  unsigned char *slice = smem + FRA_HDR;                       // guard rows, band rows, guard rows
  unsigned char *tring = slice + g.slice_bytes;                // [RB][NS] slots
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int cl = (int)cluster_id_x();
  const int ml = a.ml, nl = a.nl, NCH = g.NCH, RB = g.RB, WPR = g.WPR;
  const int R0 = (int)rank * g.rpc, R1 = min(ml, R0 + g.rpc);
  const int pitch2 = a.pitch * 2, tpitch2 = a.tpitch * 2;
  // slice address of frame row 0 (row R0 sits after the guard rows)
  const unsigned char *srow0 = slice + (ptrdiff_t)(FRA_GUARD - R0) * pitch2;

  if (tid == 0) {
    for (int k = 0; k < FRA_MAXCH; ++k) {
      mbar_init(&fbar[k], 1);
      mbar_init(&ebar[k], FRA_CW);
    }
    for (int k = 0; k < 8 * FRA_NS; ++k) {
      mbar_init(&tfull[k], 1);
      mbar_init(&tempty[k], WPR);
    }
    fence_mbar_init();
  }
  // zero the whole slice once: guard rows and never-loaded tail rows must read as 0
  for (int e = tid; e < g.slice_bytes / 16; e += FRA_THREADS)
    reinterpret_cast<uint4 *>(slice)[e] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  __syncthreads();

  // frame rows paired with some template row: [max(0,S-1), min(ml, ml+S+1)); the CTA's
  // template rows: [max(0, R0-S-1), min(ml, R1-S+1)), split into RB contiguous blocks
  auto t_range = [&](int S, int &i0, int &i1) {
    i0 = max(0, R0 - S - 1);
    i1 = max(i0, min(ml, R1 - S + 1));
  };
  auto blk = [&](int i0, int i1, int b, int &ba, int &bb) {
    const int BL = (i1 - i0 + RB - 1) / RB;
    ba = min(i1, i0 + b * BL);
    bb = min(i1, ba + BL);
  };

  if (warp == FRA_CW) {
    // ================================================================ producer warp
    if (lane != 0) {   // (idle lanes still take part in every cluster barrier)
      for (int f = cl; f < a.B; f += g.ncl) cluster_arrive_wait();
      cluster_arrive_wait();
      return;
    }
    auto issue_chunk = [&](int f, int S, int k) {
      const int r0 = R0 + k * FRA_CR, r1 = min(R1, r0 + FRA_CR);
      const int need0 = max(0, S - 1), need1 = min(ml, ml + S + 1);
      if (r0 < r1 && r0 < need1 && r1 > need0) {
        const uint32_t bytes = (uint32_t)((r1 - r0) * pitch2);
        mbar_arrive_expect_tx(&fbar[k], bytes);
        bulk_g2s(slice + (size_t)(FRA_GUARD + k * FRA_CR) * pitch2,
                 a.frames + (int64_t)f * a.fstride + (int64_t)r0 * a.pitch, bytes, &fbar[k]);
      } else {
        mbar_arrive(&fbar[k]);
      }
    };
    int tcb[8];   // template slots used so far, per row block
    for (int b = 0; b < 8; ++b) tcb[b] = 0;
    // issue template slots [from, to) of every row block of a frame, each once its slot is free
    auto issue_slots = [&](int i0, int i1, int from, int to) {
      int next[8];
      for (int b = 0; b < RB; ++b) next[b] = from;
      for (;;) {
        bool any = false;
        for (int b = 0; b < RB; ++b) {
          int ba, bb;
          blk(i0, i1, b, ba, bb);
          const int nck = (bb - ba + FRA_TRB - 1) / FRA_TRB;
          if (next[b] >= min(to, nck)) continue;
          any = true;
          const int gi = tcb[b] + next[b];
          uint64_t *eb = &tempty[b * FRA_NS + gi % FRA_NS];
          if (gi >= FRA_NS && !mbar_test(eb, (uint32_t)((gi / FRA_NS - 1) & 1))) continue;
          const int ra = ba + next[b] * FRA_TRB, rz = min(bb, ra + FRA_TRB);
          uint64_t *fb = &tfull[b * FRA_NS + gi % FRA_NS];
          const uint32_t bytes = (uint32_t)((rz - ra) * tpitch2);
          mbar_arrive_expect_tx(fb, bytes);
          bulk_g2s(tring + (size_t)(b * FRA_NS + gi % FRA_NS) * g.tslot_bytes, a.tpl + (int64_t)ra * a.tpitch,
                   bytes, fb);
          ++next[b];
        }
        if (!any) break;
      }
    };
    int f = cl;
    if (f < a.B) {
      const int S = 2 * a.shift_in[2 * f];
      for (int k = 0; k < g.nchunk; ++k) issue_chunk(f, S, k);
      int i0, i1;
      t_range(S, i0, i1);
      issue_slots(i0, i1, 0, FRA_NS);
    }
    for (int it = 0; f < a.B; ++it, f += g.ncl) {
      const int S = 2 * a.shift_in[2 * f];
      int i0, i1;
      t_range(S, i0, i1);
      issue_slots(i0, i1, FRA_NS, 1 << 30);
      for (int b = 0; b < RB; ++b) {
        int ba, bb;
        blk(i0, i1, b, ba, bb);
        tcb[b] += (bb - ba + FRA_TRB - 1) / FRA_TRB;
      }
      cluster_arrive_wait();   // (frame f: the compute warps are past H)
      const int fn = f + g.ncl;
      if (fn < a.B) {
        const int Sn = 2 * a.shift_in[2 * fn];
        int j0, j1;
        t_range(Sn, j0, j1);
        issue_slots(j0, j1, 0, FRA_NS);
        for (int k = 0; k < g.nchunk; ++k) {
          mbar_wait(&ebar[k], (uint32_t)(it & 1));   // frame f is done with chunk k
          issue_chunk(fn, Sn, k);
        }
      }
    }
    cluster_arrive_wait();
    return;
  }

  // ================================================================== compute warps
  const int rb = warp / WPR, wc = warp % WPR;
  const int c = wc * 32 + lane;          // 16-byte chunk column of this lane
  const bool act = c < NCH;
  const int cc = act ? c : 0;
  int tcb[8];
  for (int b = 0; b < 8; ++b) tcb[b] = 0;
  int f = cl;
  for (int it = 0; f < a.B; ++it, f += g.ncl) {
    const int S = 2 * a.shift_in[2 * f], T = 2 * a.shift_in[2 * f + 1];
    int i0, i1;
    t_range(S, i0, i1);
    const uint32_t fpar = (uint32_t)(it & 1);
    // ---------------- H over this warp group's template row block
    u64 H[9], Hh[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) H[q] = Hh[q] = 0;
    {
      int ba, bb;
      blk(i0, i1, rb, ba, bb);
      const int nck = (bb - ba + FRA_TRB - 1) / FRA_TRB;
      if (nck > 0) {   // frame chunks holding rows [ba+S-1, bb+S+1) of the band
        const int ra = max(R0, ba + S - 1), rz = min(R1, bb + S + 1);
        if (ra < rz)
          for (int k = (ra - R0) / FRA_CR; k <= (rz - 1 - R0) / FRA_CR; ++k) mbar_wait(&fbar[k], fpar);
      }
      const int b0 = (8 * cc - T) >> 3, SH = (8 * cc - T) & 7;
      const bool ok0 = b0 - 1 >= 0 && b0 - 1 < NCH, ok1 = b0 >= 0 && b0 < NCH, ok2 = b0 + 1 >= 0 && b0 + 1 < NCH;
      uint4 a0 = make_uint4(0, 0, 0, 0), a1 = a0, a2 = a0;
      if (nck > 0) {
        a0 = *reinterpret_cast<const uint4 *>(srow0 + (ptrdiff_t)(ba + S - 1) * pitch2 + 16 * cc);
        a1 = *reinterpret_cast<const uint4 *>(srow0 + (ptrdiff_t)(ba + S) * pitch2 + 16 * cc);
      }
      for (int j = 0; j < nck; ++j) {
        const int gi = tcb[rb] + j, sl = rb * FRA_NS + gi % FRA_NS;
        mbar_wait(&tfull[sl], (uint32_t)((gi / FRA_NS) & 1));
        const unsigned char *slot = tring + (size_t)sl * g.tslot_bytes;
        const int ia = ba + j * FRA_TRB, ib = min(bb, ia + FRA_TRB);
        if (act) {
          switch (SH) {
            case 0: fra_hslot<0>(slot, tpitch2, srow0, pitch2, ia, ib, S, cc, b0, ok0, ok1, ok2, a0, a1, a2, H, Hh); break;
            case 2: fra_hslot<2>(slot, tpitch2, srow0, pitch2, ia, ib, S, cc, b0, ok0, ok1, ok2, a0, a1, a2, H, Hh); break;
            case 4: fra_hslot<4>(slot, tpitch2, srow0, pitch2, ia, ib, S, cc, b0, ok0, ok1, ok2, a0, a1, a2, H, Hh); break;
            default: fra_hslot<6>(slot, tpitch2, srow0, pitch2, ia, ib, S, cc, b0, ok0, ok1, ok2, a0, a1, a2, H, Hh); break;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[sl]);
      }
    }
    for (int b = 0; b < RB; ++b) {
      int ba, bb;
      blk(i0, i1, b, ba, bb);
      tcb[b] += (bb - ba + FRA_TRB - 1) / FRA_TRB;
    }
    // ---------------- GA: per-pixel column sums over the rows every u pairs, masked per v
    u64 ga[9], cs[8];
#pragma unroll
    for (int q = 0; q < 9; ++q) ga[q] = 0;
#pragma unroll
    for (int x = 0; x < 8; ++x) cs[x] = 0;
    const int rlo = max(R0, max(0, S - 1)), rhi = min(R1, min(ml, ml + S + 1));
    if (rlo < rhi)
      for (int k = (rlo - R0) / FRA_CR; k <= (rhi - 1 - R0) / FRA_CR; ++k) mbar_wait(&fbar[k], fpar);
    if (act) {
      for (int r = rlo + rb; r < rhi; r += RB) {
        const uint4 v = *reinterpret_cast<const uint4 *>(srow0 + (ptrdiff_t)r * pitch2 + 16 * cc);
        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
        uint32_t px[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) px[x] = (x & 1) ? (wv[x >> 1] >> 16) : (wv[x >> 1] & 0xffffu);
        if (r >= S + 1 && r < ml + S - 1) {   // every u pairs this row (warp-uniform branch)
#pragma unroll
          for (int x = 0; x < 8; ++x) cs[x] += (u64)px[x] * px[x];
        } else {
#pragma unroll
          for (int up = 0; up < 3; ++up) {
            const int i = r - S - (up - 1);
            if (i < 0 || i >= ml) continue;
#pragma unroll
            for (int vp = 0; vp < 3; ++vp) {
              u64 s8 = 0;
#pragma unroll
              for (int x = 0; x < 8; ++x) {
                const int j = 8 * cc + x - T - (vp - 1);
                s8 += (j >= 0 && j < nl) ? (u64)px[x] * px[x] : 0ull;
              }
              ga[up * 3 + vp] += s8;
            }
          }
        }
      }
#pragma unroll
      for (int vp = 0; vp < 3; ++vp) {
        u64 s = 0;
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const int j = 8 * cc + x - T - (vp - 1);
          s += (j >= 0 && j < nl) ? cs[x] : 0ull;
        }
#pragma unroll
        for (int up = 0; up < 3; ++up) ga[up * 3 + vp] += s;
      }
    }
    // ---------------- block reduction -> this CTA's partials, then the cluster's sums
    u64 v18[18];
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      v18[q] = H[q] + (Hh[q] << 8);
      v18[9 + q] = ga[q];
    }
#pragma unroll
    for (int q = 0; q < 18; ++q) v18[q] = warp_sum(v18[q]);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 18; ++q) red[warp * 18 + q] = v18[q];
    fra_bar_compute();
    u64 *pp = part + (it & 1) * 32;
    if (tid < 18) {
      u64 s = 0;
      for (int w = 0; w < FRA_CW; ++w) s += red[w * 18 + tid];
      pp[tid] = s;
    }
    cluster_arrive_wait();
    if (warp == 0) {
      Key key{~0ull, ~0u};
      if (lane < 9) {
        u64 h = 0, gav = 0;
        for (int q = 0; q < g.Q; ++q) {
          h += ld_dsmem_u64(pp + lane, (uint32_t)q);
          gav += ld_dsmem_u64(pp + 9 + lane, (uint32_t)q);
        }
        const int s = S + lane / 3 - 1, t = T + lane % 3 - 1, n1 = nl + 1;
        const int ci0 = max(0, -s), ci1 = ml - max(0, s), cj0 = max(0, -t), cj1 = nl - max(0, t);
        const u64 gb = a.pb2[(int64_t)ci1 * n1 + cj1] - a.pb2[(int64_t)ci0 * n1 + cj1] -
                       a.pb2[(int64_t)ci1 * n1 + cj0] + a.pb2[(int64_t)ci0 * n1 + cj0];
        const u64 N = gav + gb - 2 * h;
        const double area = (double)((ml - abs(s)) * (nl - abs(t)));
        const double fv = (double)N / (a.scale * area);
        key = Key{(u64)__double_as_longlong(fv), (unsigned)lane};   // rank == (s,t) lexicographic
      }
      key = warp_min_key(key);
      if (lane == 0) {
        const int s = S + (int)(key.idx / 3) - 1, t = T + (int)(key.idx % 3) - 1;
        res[0] = s;
        res[1] = t;
        if (rank == 0) {
          a.shift_out[2 * f] = s;
          a.shift_out[2 * f + 1] = t;
          if (a.f_out) a.f_out[f] = __longlong_as_double((long long)key.f);
        }
      }
    }
    fra_bar_compute();
    const int s = res[0], t = res[1];
    // every chunk landed this frame (skipped ones by a plain arrive): wait for all, so that
    // no chunk barrier is waited on after the producer recycles it
    for (int k = 0; k < g.nchunk; ++k) mbar_wait(&fbar[k], fpar);
    // ---------------- apply (level 0): corrected rows from the resident band; each chunk
    // is released to the producer once its rows are written
    if (a.corrected) {
      uint16_t *O = a.corrected + (int64_t)f * ml * nl;
      if (act)   // zero rows of this CTA's index band (no source row in the frame)
        for (int o = R0 + rb; o < R1; o += RB)
          if (o + s < 0 || o + s >= ml)
            __stcs(reinterpret_cast<uint4 *>(O + (int64_t)o * nl + 8 * cc), make_uint4(0, 0, 0, 0));
      const int SHa = t & 7, ab = 8 * cc + t - SHa, bl = ab >> 3;
      const bool okl = bl >= 0 && bl < NCH, okh = bl + 1 >= 0 && bl + 1 < NCH;
      for (int k = 0; k < g.nchunk; ++k) {
        const int r0 = max(R0 + k * FRA_CR, max(0, s)), r1 = min(min(R1, R0 + (k + 1) * FRA_CR), min(ml, ml + s));
        if (act && r0 < r1) {
          const int rs = r0 + ((rb - r0) % RB + RB) % RB;   // the rows = rb mod RB
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
        __syncwarp();
        if (lane == 0) mbar_arrive(&ebar[k]);
      }
    } else {
      __syncwarp();
      if (lane == 0)
        for (int k = 0; k < g.nchunk; ++k) mbar_arrive(&ebar[k]);
    }
  }
  // no CTA leaves while another may still read its partials
  cluster_arrive_wait();
}

}  // namespace moco
