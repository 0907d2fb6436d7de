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
// Layout of the work: cluster c takes frames c, c + nclusters, ...; CTA q of the cluster
// holds frame rows [q rpc, (q+1) rpc) (bulk copies in 16-row chunks, one mbarrier each)
// and accumulates the (template row i, frame row r = i+S+u) pairs of its rows.  The nine
// H sums run on CUDA cores with 16x8-bit dot products: a u16 frame word (two pixels) is
// the 16-bit operand of dp2a as it sits in memory, the template word is regrouped into
// (lo, lo, hi, hi) bytes, so H = sum dp2a_lo + 2^8 sum dp2a_hi exactly (values < 2^14,
// 32-bit partials flushed to 64 bits every template chunk).  Template rows stream through
// a two-slot shared-memory ring (16 rows per slot, L2-resident).  The CTAs exchange their
// 18 partial sums through distributed shared memory (one cluster barrier per frame), every
// CTA takes the same argmin, and each writes the corrected rows whose source rows it holds
// (zero rows: the rows of its own index band with no source), straight from shared memory;
// the freed chunks then receive the next frame's rows.
#pragma once

namespace moco {

constexpr int FRA_THREADS = 256;
constexpr int FRA_CR = 16;       // frame rows per slice chunk (one mbarrier each)
constexpr int FRA_TR = 16;       // template rows per ring slot
constexpr int FRA_MAXCH = 16;    // slice chunks at most (rpc <= 256)
constexpr int FRA_SLICE_OFF = 4096;

struct FraGeom {
  int Q;          // CTAs per cluster = per frame
  int rpc;        // frame rows per CTA
  int nchunk;     // slice chunks per CTA
  int NCH;        // 8-pixel chunks per row (nl / 8)
  int PH;         // row phases: FRA_THREADS / NCH
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
// 144 KB of shared memory next to the template ring; nl a multiple of 8 with at most
// 256 chunks per row, values < 2^14.
inline bool fra_make(FraGeom *g, int ml, int nl, int pitch, int tpitch, int vb) {
  if (vb > 14 || nl % 8 != 0 || pitch % 8 != 0 || tpitch % 8 != 0 || ml < 4) return false;
  const int NCH = nl / 8;
  if (NCH > FRA_THREADS) return false;
  int PH = FRA_THREADS / NCH;
  if (PH > 16) PH = 16;
  while (FRA_TR % PH) --PH;   // rows of a ring slot split evenly over the phases
  for (int Q = 1; Q <= 8; Q *= 2) {
    const int rpc = (ml + Q - 1) / Q;
    const int nchunk = (rpc + FRA_CR - 1) / FRA_CR;
    const int slice = nchunk * FRA_CR * pitch * 2;
    if (nchunk > FRA_MAXCH || slice > 144 * 1024) continue;
    g->Q = Q; g->rpc = rpc; g->nchunk = nchunk; g->NCH = NCH; g->PH = PH;
    g->slice_bytes = slice;
    g->tslot_bytes = FRA_TR * tpitch * 2;
    g->smem = FRA_SLICE_OFF + slice + 2 * g->tslot_bytes;
    g->ncl = 0;
    return g->smem <= 227 * 1024;
  }
  return false;
}

__device__ __forceinline__ void cluster_arrive_wait() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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

// (lo0, lo1, hi0, hi1) bytes of a word holding two u16 pixels: the 8-bit operand of dp2a
__device__ __forceinline__ uint32_t fra_split(uint32_t w) { return __byte_perm(w, 0, 0x3120); }

// One template row (three 16-byte blocks around the thread's chunk: b0-1, b0, b0+1) against
// the frame rows i+S-1, i+S, i+S+1 of the thread's chunk.  SH = (8c - T) mod 8 (T even).
template <int SH>
__device__ __forceinline__ void fra_row(const uint4 &t0, const uint4 &t1, const uint4 &t2, const uint4 (&a)[3],
                                        uint32_t (&lo)[9], uint32_t (&hi)[9]) {
  const uint32_t W[12] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w, t2.x, t2.y, t2.z, t2.w};
  uint32_t sp[3][4];   // [v+1][k]: template pair under frame pixels (8c+2k, 8c+2k+1) at shift T+v
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int e = 4 + SH / 2 + k;
    sp[1][k] = fra_split(W[e]);                                  // v = 0:  columns 8c+2k-T, +1
    sp[2][k] = fra_split(__funnelshift_r(W[e - 1], W[e], 16));   // v = +1: one column left
    sp[0][k] = fra_split(__funnelshift_r(W[e], W[e + 1], 16));   // v = -1: one column right
  }
#pragma unroll
  for (int up = 0; up < 3; ++up) {
    const uint32_t aw[4] = {a[up].x, a[up].y, a[up].z, a[up].w};
#pragma unroll
    for (int vp = 0; vp < 3; ++vp)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        lo[up * 3 + vp] = __dp2a_lo(aw[k], sp[vp][k], lo[up * 3 + vp]);
        hi[up * 3 + vp] = __dp2a_hi(aw[k], sp[vp][k], hi[up * 3 + vp]);
      }
  }
}

struct FraCtx {
  const unsigned char *slice;   // this CTA's frame rows [R0, R1), row stride pitch*2 bytes
  uint64_t *fbar;
  int R0, R1, pitch2, it;
  int ready;                    // slice chunks this thread has seen land (this frame)
  __device__ __forceinline__ uint4 row(int r, int c) {
    if (r < R0 || r >= R1) return make_uint4(0, 0, 0, 0);
    const int k = (r - R0) / FRA_CR;
    while (ready <= k) {
      mbar_wait(&fbar[ready], (uint32_t)(it & 1));
      ++ready;
    }
    return *reinterpret_cast<const uint4 *>(slice + (size_t)(r - R0) * pitch2 + 16 * c);
  }
};

// This thread's template rows [ia, ib) of the current ring slot (row ia = slot row ra).
template <int SH>
__device__ __forceinline__ void fra_hrows(FraCtx &X, const unsigned char *tslot, int ra, int ia, int ib, int S,
                                          int c, int b0, int NCH, int tpitch2, u64 (&H)[9], u64 (&Hh)[9]) {
  uint32_t lo[9], hi[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) lo[q] = hi[q] = 0;
  uint4 a[3];
  a[0] = X.row(ia + S - 1, c);
  a[1] = X.row(ia + S, c);
  a[2] = X.row(ia + S + 1, c);
  const bool ok0 = b0 - 1 >= 0 && b0 - 1 < NCH, ok1 = b0 >= 0 && b0 < NCH, ok2 = b0 + 1 >= 0 && b0 + 1 < NCH;
  for (int i = ia; i < ib; ++i) {
    if (i > ia) {
      a[0] = a[1];
      a[1] = a[2];
      a[2] = X.row(i + S + 1, c);
    }
    const unsigned char *tr = tslot + (size_t)(ra + i - ia) * tpitch2;
    const uint4 z = make_uint4(0, 0, 0, 0);
    const uint4 t0 = ok0 ? *reinterpret_cast<const uint4 *>(tr + 16 * (b0 - 1)) : z;
    const uint4 t1 = ok1 ? *reinterpret_cast<const uint4 *>(tr + 16 * b0) : z;
    const uint4 t2 = ok2 ? *reinterpret_cast<const uint4 *>(tr + 16 * (b0 + 1)) : z;
    fra_row<SH>(t0, t1, t2, a, lo, hi);
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    H[q] += lo[q];
    Hh[q] += hi[q];
  }
}

// Corrected rows of one slice chunk: out[o][j] = a[o+s][j+t] (0 outside), source rows in
// [rlo, rhi) of this CTA; 16-byte streaming stores.
template <int SH>
__device__ __forceinline__ void fra_apply_rows(FraCtx &X, uint16_t *O, int rlo, int rhi, int s, int t, int ml,
                                               int nl, int NCH) {
  const int items = (rhi - rlo) * NCH;
  for (int e = threadIdx.x; e < items; e += FRA_THREADS) {
    const int r = rlo + e / NCH, q = e % NCH;
    const int o = r - s;
    const int ab = 8 * q + t - SH;   // multiple of 8: blocks wholly in or out of the row
    const int bl = ab >> 3;
    const uint4 z = make_uint4(0, 0, 0, 0);
    const uint4 lo = (bl >= 0 && bl < NCH) ? X.row(r, bl) : z;
    const uint4 hi = (SH && bl + 1 >= 0 && bl + 1 < NCH) ? X.row(r, bl + 1) : z;
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint32_t ov[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e2 = SH + 2 * k;
      ov[k] = (e2 & 1) ? __funnelshift_r(w[e2 >> 1], w[(e2 >> 1) + 1], 16) : w[e2 >> 1];
    }
    __stcs(reinterpret_cast<uint4 *>(O + (int64_t)o * nl + 8 * q), make_uint4(ov[0], ov[1], ov[2], ov[3]));
  }
}

__global__ void __launch_bounds__(FRA_THREADS, 1) k_refine_frame(FraArgs a) {
  extern __shared__ __align__(1024) unsigned char fra_raw[];
  unsigned char *smem = fra_raw;
  uint64_t *fbar = reinterpret_cast<uint64_t *>(smem);         // [FRA_MAXCH]
  uint64_t *tbar = fbar + FRA_MAXCH;                           // [2]
  u64 *part = reinterpret_cast<u64 *>(smem + 256);             // [2][32]: H 0..8, GA 9..17
  u64 *red = reinterpret_cast<u64 *>(smem + 1024);             // [8 warps][18]
  int *res = reinterpret_cast<int *>(smem + 2304);             // s, t
  unsigned char *slice = smem + FRA_SLICE_OFF;
  unsigned char *tring = slice + a.g.slice_bytes;
  const FraGeom &g = a.g;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int cl = (int)cluster_id_x();
  const int ml = a.ml, nl = a.nl, NCH = g.NCH, PH = g.PH;
  const int R0 = (int)rank * g.rpc, R1 = min(ml, R0 + g.rpc);
  const int pitch2 = a.pitch * 2, tpitch2 = a.tpitch * 2;
  const int c = tid % NCH, ph = tid / NCH;   // chunk column, row phase
  const bool hthr = ph < PH;
  const int RPP = FRA_TR / PH;               // template rows per phase per ring slot

  if (tid == 0) {
    for (int k = 0; k < FRA_MAXCH; ++k) mbar_init(&fbar[k], 1);
    mbar_init(&tbar[0], 1);
    mbar_init(&tbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // producer helpers (thread 0): rows needed by frame f with coarse shift S: the union
  // over u of the rows paired with a template row, [max(0,S-1), min(ml, ml+S+1))
  auto issue_chunk = [&](int f, int S, int k) {
    const int r0 = R0 + k * FRA_CR, r1 = min(R1, r0 + FRA_CR);
    const int need0 = max(0, S - 1), need1 = min(ml, ml + S + 1);
    if (r0 < r1 && r0 < need1 && r1 > need0) {
      const uint32_t bytes = (uint32_t)((r1 - r0) * pitch2);
      mbar_arrive_expect_tx(&fbar[k], bytes);
      bulk_g2s(slice + (size_t)k * FRA_CR * pitch2, a.frames + (int64_t)f * a.fstride + (int64_t)r0 * a.pitch,
               bytes, &fbar[k]);
    } else {
      mbar_arrive(&fbar[k]);
    }
  };
  auto t_range = [&](int S, int &i0, int &i1) {
    i0 = max(0, R0 - S - 1);
    i1 = min(ml, R1 - S + 1);
    if (i1 < i0) i1 = i0;
  };
  auto issue_tchunk = [&](int i0, int i1, int k, int slotidx) {
    const int ra = i0 + k * FRA_TR, rb = min(i1, ra + FRA_TR);
    const int slot = slotidx & 1;
    const uint32_t bytes = (uint32_t)((rb - ra) * tpitch2);
    mbar_arrive_expect_tx(&tbar[slot], bytes);
    bulk_g2s(tring + (size_t)slot * g.tslot_bytes, a.tpl + (int64_t)ra * a.tpitch, bytes, &tbar[slot]);
  };

  int tcount = 0;   // template ring slots used so far (slot = tcount & 1, parity = (tcount >> 1) & 1)
  int f = cl;
  if (tid == 0 && f < a.B) {
    const int S = 2 * a.shift_in[2 * f];
    for (int k = 0; k < g.nchunk; ++k) issue_chunk(f, S, k);
    int i0, i1;
    t_range(S, i0, i1);
    const int ntc = (i1 - i0 + FRA_TR - 1) / FRA_TR;
    for (int k = 0; k < min(2, ntc); ++k) issue_tchunk(i0, i1, k, tcount + k);
  }
  for (int it = 0; f < a.B; ++it, f += g.ncl) {
    const int S = 2 * a.shift_in[2 * f], T = 2 * a.shift_in[2 * f + 1];
    int i0, i1;
    t_range(S, i0, i1);
    const int ntc = (i1 - i0 + FRA_TR - 1) / FRA_TR;
    FraCtx X{slice, fbar, R0, R1, pitch2, it, 0};
    // ---------------- H: template chunks through the ring
    u64 H[9], Hh[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) H[q] = Hh[q] = 0;
    const int b0 = (8 * c - T) >> 3, SH = (8 * c - T) & 7;
    for (int k = 0; k < ntc; ++k) {
      const int si = tcount + k;
      mbar_wait(&tbar[si & 1], (uint32_t)((si >> 1) & 1));
      const unsigned char *ts = tring + (size_t)(si & 1) * g.tslot_bytes;
      if (hthr) {
        const int ra = ph * RPP, ia = i0 + k * FRA_TR + ra, ib = min(i1, ia + RPP);
        if (ia < ib) {
          switch (SH) {
            case 0: fra_hrows<0>(X, ts, ra, ia, ib, S, c, b0, NCH, tpitch2, H, Hh); break;
            case 2: fra_hrows<2>(X, ts, ra, ia, ib, S, c, b0, NCH, tpitch2, H, Hh); break;
            case 4: fra_hrows<4>(X, ts, ra, ia, ib, S, c, b0, NCH, tpitch2, H, Hh); break;
            default: fra_hrows<6>(X, ts, ra, ia, ib, S, c, b0, NCH, tpitch2, H, Hh); break;
          }
        }
      }
      __syncthreads();
      if (tid == 0 && k + 2 < ntc) issue_tchunk(i0, i1, k + 2, si + 2);
    }
    tcount += ntc;
    // ---------------- GA: a^2 over the rows and columns each candidate pairs with b
    u64 ga[9], gint = 0;
#pragma unroll
    for (int q = 0; q < 9; ++q) ga[q] = 0;
    if (hthr) {
      const bool cint = 8 * c >= T + 1 && 8 * c + 8 <= nl + T - 1;   // all 8 columns valid for every v
      const int rlo = max(R0, max(0, S - 1)), rhi = min(R1, min(ml, ml + S + 1));
      for (int r = rlo + ph; r < rhi; r += PH) {
        const uint4 v = X.row(r, c);
        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
        uint32_t sq[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const uint32_t p = (x & 1) ? (wv[x >> 1] >> 16) : (wv[x >> 1] & 0xffffu);
          sq[x] = p * p;
        }
        if (cint && r >= S + 1 && r < ml + S - 1) {
          u64 s8 = 0;
#pragma unroll
          for (int x = 0; x < 8; ++x) s8 += sq[x];
          gint += s8;
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
                const int j = 8 * c + x - T - (vp - 1);
                s8 += (j >= 0 && j < nl) ? sq[x] : 0u;
              }
              ga[up * 3 + vp] += s8;
            }
          }
        }
      }
    }
    // ---------------- block reduction -> this CTA's partials, then the cluster's sums
    u64 v18[18];
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      v18[q] = H[q] + (Hh[q] << 8);
      v18[9 + q] = ga[q] + gint;
    }
#pragma unroll
    for (int q = 0; q < 18; ++q) v18[q] = warp_sum(v18[q]);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 18; ++q) red[warp * 18 + q] = v18[q];
    __syncthreads();
    u64 *pp = part + (it & 1) * 32;
    if (tid < 18) {
      u64 s = 0;
      for (int w = 0; w < FRA_THREADS / 32; ++w) s += red[w * 18 + tid];
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
    __syncthreads();
    const int s = res[0], t = res[1];
    // every chunk of this frame has landed (needed ones were waited for by H/GA, the others
    // completed with a plain arrive): catch up, so that no thread ever waits on a chunk
    // barrier after it has been recycled for the next frame
    while (X.ready < g.nchunk) {
      mbar_wait(&fbar[X.ready], (uint32_t)(it & 1));
      ++X.ready;
    }
    __syncthreads();   // (before thread 0 recycles any chunk for the next frame)
    // ---------------- next frame: template ring (free: every H row is done)
    const int fn = f + g.ncl;
    int Sn = 0;
    if (fn < a.B) {
      Sn = 2 * a.shift_in[2 * fn];
      if (tid == 0) {
        int j0, j1;
        t_range(Sn, j0, j1);
        const int ntn = (j1 - j0 + FRA_TR - 1) / FRA_TR;
        for (int k = 0; k < min(2, ntn); ++k) issue_tchunk(j0, j1, k, tcount + k);
      }
    }
    // ---------------- apply (level 0): corrected rows from the resident slice; every
    // chunk released to the next frame's rows once its rows are written
    if (a.corrected) {
      uint16_t *O = a.corrected + (int64_t)f * ml * nl;
      // zero rows of this CTA's index band: no source row in the frame
      {
        const int zr = (R1 - R0) * NCH;
        for (int e = tid; e < zr; e += FRA_THREADS) {
          const int o = R0 + e / NCH, q = e % NCH;
          if (o + s < 0 || o + s >= ml)
            __stcs(reinterpret_cast<uint4 *>(O + (int64_t)o * nl + 8 * q), make_uint4(0, 0, 0, 0));
        }
      }
      for (int k = 0; k < g.nchunk; ++k) {
        const int r0 = max(R0 + k * FRA_CR, max(0, s)), r1 = min(min(R1, R0 + (k + 1) * FRA_CR), min(ml, ml + s));
        if (r0 < r1) {
          switch (t & 7) {
            case 0: fra_apply_rows<0>(X, O, r0, r1, s, t, ml, nl, NCH); break;
            case 1: fra_apply_rows<1>(X, O, r0, r1, s, t, ml, nl, NCH); break;
            case 2: fra_apply_rows<2>(X, O, r0, r1, s, t, ml, nl, NCH); break;
            case 3: fra_apply_rows<3>(X, O, r0, r1, s, t, ml, nl, NCH); break;
            case 4: fra_apply_rows<4>(X, O, r0, r1, s, t, ml, nl, NCH); break;
            case 5: fra_apply_rows<5>(X, O, r0, r1, s, t, ml, nl, NCH); break;
            case 6: fra_apply_rows<6>(X, O, r0, r1, s, t, ml, nl, NCH); break;
            default: fra_apply_rows<7>(X, O, r0, r1, s, t, ml, nl, NCH); break;
          }
          __syncthreads();
        }
        if (tid == 0 && fn < a.B) issue_chunk(fn, Sn, k);
      }
    } else if (tid == 0 && fn < a.B) {   // (the slice is no longer read: H, GA done)
      for (int k = 0; k < g.nchunk; ++k) issue_chunk(fn, Sn, k);
    }
    __syncthreads();
  }
  // no CTA leaves while another may still read its partials
  cluster_arrive_wait();
}

}  // namespace moco
