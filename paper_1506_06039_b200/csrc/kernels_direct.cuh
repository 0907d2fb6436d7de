// kernels_direct.cuh -- CUDA-core kernels of the moco hot path (sm_100a).
//
// Exact integer arithmetic for MOCO_U16 (every N_{s,t} is computed exactly in
// 64-bit integers, then f = fl(N / (16^l * Area)) -- the same correctly
// rounded quotient the fp64 oracle produces, so results are bit-identical);
// fp64 accumulation for MOCO_F32.
//
//   K1 k_downsample_*   2x2 block SUM (u16) / mean (fp64) per level (R1)
//   K2 k_template_energy  sum_{D_{s,t}} b^2 for every coarse lag
//   K3+K4d+K5 k_coarse    frame energy g_a (strip/corner form of the DP of
//                         P:33-35), direct cross term h, score
//                         and deterministic argmin with key (f, s, t) (R4)
//   K6 k_refine           f_{2s+u,2t+v}, u,v in {0,-1,1} exactly
//   K7 k_apply            corrected[i][j] = a[i+s][j+t] or 0
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <type_traits>
#include <utility>

namespace moco {

typedef unsigned long long u64;

// cudaFuncAttributeMaxDynamicSharedMemorySize is a property of the function on a device,
// shared by every plan of the process: only ever RAISE it (a plan with a smaller geometry
// created later must not lower the limit under an earlier plan's launches).
inline cudaError_t smem_attr(const void *fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void *>, int> set;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  int &cur = set[{dev, fn}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}
template <class K>
inline cudaError_t smem_attr(K *fn, int bytes) { return smem_attr((const void *)fn, bytes); }

// ---------------------------------------------------------------- key helpers
// f >= 0, so the IEEE-754 bit pattern of the double orders like an unsigned
// integer; idx = (s+w-1)*(2w-1) + (t+w-1) (or the candidate rank in refine)
// orders like (s, t) lexicographically.  min over (fbits, idx) = argmin of the
// key (f, s, t).
struct Key {
  u64 f;
  unsigned idx;
};
__device__ __forceinline__ bool key_less(const Key &a, const Key &b) {
  return a.f < b.f || (a.f == b.f && a.idx < b.idx);
}
__device__ __forceinline__ Key warp_min_key(Key k) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Key other;
    other.f = __shfl_xor_sync(0xffffffffu, k.f, o);
    other.idx = __shfl_xor_sync(0xffffffffu, k.idx, o);
    if (key_less(other, k)) k = other;
  }
  return k;
}
// Block-wide min; every thread gets the result.  `red` holds >= 32 Keys.
__device__ __forceinline__ Key block_min_key(Key k, Key *red) {
  k = warp_min_key(k);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = k;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  if (wid == 0) {
    Key v = lane < nw ? red[lane] : Key{~0ull, ~0u};
    v = warp_min_key(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Value type of a level image: u16 samples -> uint32 arithmetic, float ->
// double, double -> double.
template <class In> struct Arith;
template <> struct Arith<uint16_t> {
  typedef uint32_t V;
  typedef u64 Acc;
};
template <> struct Arith<float> {
  typedef double V;
  typedef double Acc;
};
template <> struct Arith<double> {
  typedef double V;
  typedef double Acc;
};

// ------------------------------------------------------------------------- K1
// out[r][c] = in[2r][2c] + in[2r][2c+1] + in[2r+1][2c] + in[2r+1][2c+1]  (u16 block sums)
// 4 outputs per thread from one 16-byte load of each of the two source rows.
__global__ void k_downsample_u16(const uint16_t *__restrict__ in, int64_t in_fstride, int in_pitch,
                                 int mi, int ni, uint16_t *__restrict__ out, int64_t out_fstride,
                                 int out_pitch, int mo, int no, int B) {
  const int groups = (no + 3) >> 2;
  const int64_t total = (int64_t)B * mo * groups;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int cg = (int)(g % groups);
    const int64_t fr = g / groups;
    const int r = (int)(fr % mo);
    const int64_t f = fr / mo;
    const uint16_t *r0 = in + f * in_fstride + (int64_t)(2 * r) * in_pitch;
    const uint16_t *r1 = r0 + in_pitch;
    const int c0 = cg * 4;
    uint16_t o[4];
    if (2 * c0 + 8 <= ni && ((2 * c0) & 7) == 0) {
      const uint4 x = *reinterpret_cast<const uint4 *>(r0 + 2 * c0);
      const uint4 y = *reinterpret_cast<const uint4 *>(r1 + 2 * c0);
      const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        o[k] = (uint16_t)((xs[k] & 0xffffu) + (xs[k] >> 16) + (ys[k] & 0xffffu) + (ys[k] >> 16));
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = c0 + k;
        o[k] = c < no ? (uint16_t)(r0[2 * c] + r0[2 * c + 1] + r1[2 * c] + r1[2 * c + 1]) : 0;
      }
    }
    uint16_t *dst = out + f * out_fstride + (int64_t)r * out_pitch + c0;
    if (c0 + 4 <= out_pitch) {
      uint2 v;
      v.x = (uint32_t)o[0] | ((uint32_t)o[1] << 16);
      v.y = (uint32_t)o[2] | ((uint32_t)o[3] << 16);
      *reinterpret_cast<uint2 *>(dst) = v;
    } else {
      for (int k = 0; k < 4 && c0 + k < out_pitch; ++k) dst[k] = o[k];
    }
  }
}

// fp32/fp64 -> fp64 2x2 MEAN, summed in the oracle's order ((x00+x01)+x10)+x11 / 4.
template <class In>
__global__ void k_downsample_mean(const In *__restrict__ in, int64_t in_fstride, int in_pitch,
                                  int mi, int ni, double *__restrict__ out, int64_t out_fstride,
                                  int out_pitch, int mo, int no, int B) {
  const int64_t total = (int64_t)B * mo * no;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(g % no);
    const int64_t fr = g / no;
    const int r = (int)(fr % mo);
    const int64_t f = fr / mo;
    const In *r0 = in + f * in_fstride + (int64_t)(2 * r) * in_pitch;
    const In *r1 = r0 + in_pitch;
    const double v = (((double)r0[2 * c] + (double)r0[2 * c + 1]) + (double)r1[2 * c]) +
                     (double)r1[2 * c + 1];
    out[f * out_fstride + (int64_t)r * out_pitch + c] = v / 4.0;
  }
}

// ------------------------------------------------------------------------- K2
// gb[s][t] = sum over the template rectangle of D_{s,t} of b^2:
//   rows [max(0,-s), mc - max(0,s)), cols [max(0,-t), nc - max(0,t)).
// One block per lag; once per plan.
template <class In>
__global__ void k_template_energy(const In *__restrict__ b, int pitch, int mc, int nc, int w,
                                  typename Arith<In>::Acc *__restrict__ gb) {
  typedef typename Arith<In>::Acc Acc;
  typedef typename Arith<In>::V V;
  const int W = 2 * w - 1;
  const int s = (int)(blockIdx.x / W) - (w - 1), t = (int)(blockIdx.x % W) - (w - 1);
  const int i0 = max(0, -s), i1 = mc - max(0, s), j0 = max(0, -t), j1 = nc - max(0, t);
  Acc acc = 0;
  for (int i = i0; i < i1; ++i)
    for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
      const V v = (V)b[(int64_t)i * pitch + j];
      acc += (Acc)(v * v);
    }
  __shared__ Acc red[32];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc tot = 0;
    for (int k = 0; k < (int)(blockDim.x + 31) / 32; ++k) tot += red[k];
    gb[blockIdx.x] = tot;
  }
}

// ---------------------------------------------------------------- K3+K4d+K5
// One CTA per frame.  Shared memory:
//   ga[W*W]      frame energy per lag (strip/corner form of the DP)
//   hs[SC*W]     cross-term partials for the current chunk of lag rows
//   band region  template rows [r0, r0+BR) and frame rows
//                [r0-(w-1), r0+BR+(w-1)) zero-padded by w-1 columns each side,
//                so that a_pad[i+s][j+t] = 0 outside the frame and
//                h(s,t) = sum_{i,j} a_pad[i+s][j+t] * b[i][j]
//   (the band region first hosts the four corner tables of a^2)
struct CoarseArgs {
  const void *frames;   // coarse images, [B] x fstride elements, row pitch `pitch`
  int64_t fstride;
  int pitch;
  const void *tpl;      // coarse template, row pitch tpitch
  int tpitch;
  const void *gb;       // W*W template energies
  int mc, nc, w;
  double scale;         // 16^L for u16 block sums, 1 for means
  int B;
  int br;               // band rows
  int sc;               // lag rows per chunk
  int fpitch;           // smem frame-band row pitch (elements)
  int32_t *shift_out;   // [B][2] or null
  double *f_out;        // [B] or null
  double *grid_out;     // [B][W*W] or null
  uint8_t *flags;       // [B] or null
};

constexpr int KT = 8;  // consecutive t-lags per thread

template <class In>
__device__ __forceinline__ typename Arith<In>::V ldv(const In *p) {
  return (typename Arith<In>::V)(*p);
}

// WIDE: coarse values may reach 16 bits, so a product can reach 2^32 and is
// accumulated straight into 64 bits.  Otherwise (values < 2^14, products
// < 2^28) up to 16 products are summed in 32 bits before widening.
template <class In, bool WIDE>
__global__ void __launch_bounds__(512) k_coarse(CoarseArgs a) {
  typedef typename Arith<In>::V V;
  typedef typename Arith<In>::Acc Acc;
  extern __shared__ __align__(16) unsigned char smem[];
  const int w = a.w, W = 2 * w - 1, mc = a.mc, nc = a.nc;
  const int hw = w - 1;
  Acc *ga = reinterpret_cast<Acc *>(smem);                 // W*W
  Acc *hs = ga + W * W;                                    // sc*W
  Key *red = reinterpret_cast<Key *>(hs + a.sc * W);       // 32
  Acc *misc = reinterpret_cast<Acc *>(red + 32);           // 4*w + 1 (strips) + 32
  unsigned char *band = reinterpret_cast<unsigned char *>(misc + 4 * w + 1 + 32);
  const int64_t f = blockIdx.x;
  const In *A = reinterpret_cast<const In *>(a.frames) + f * a.fstride;
  const In *Bt = reinterpret_cast<const In *>(a.tpl);
  const int tid = threadIdx.x, nth = blockDim.x;

  // ---- frame energy g_a (S2).  g_a(s,t) = Total - RowEx(s) - ColEx(t) + Corner(s,t):
  // the rows/cols of the frame outside the frame-side rectangle of D_{s,t}
  // (top s rows if s>0, bottom |s| if s<0; left t cols if t>0, right |t| if t<0).
  Acc *rowTop = misc, *rowBot = misc + w, *colL = misc + 2 * w, *colR = misc + 3 * w;
  Acc *total = misc + 4 * w;
  Acc *wred = misc + 4 * w + 1;
  {
    // total
    Acc acc = 0;
    for (int64_t e = tid; e < (int64_t)mc * nc; e += nth) {
      const int r = (int)(e / nc), c = (int)(e % nc);
      const V v = ldv(A + (int64_t)r * a.pitch + c);
      acc += (Acc)(v * v);
    }
    acc = warp_sum(acc);
    if ((tid & 31) == 0) wred[tid >> 5] = acc;
    // strip sums of the first/last w-1 rows and cols (one thread each)
    for (int k = tid; k < 4 * hw; k += nth) {
      const int kind = k / hw, q = k % hw;
      Acc s = 0;
      if (kind < 2) {
        const int r = kind == 0 ? q : mc - 1 - q;
        for (int c = 0; c < nc; ++c) {
          const V v = ldv(A + (int64_t)r * a.pitch + c);
          s += (Acc)(v * v);
        }
      } else {
        const int c = kind == 2 ? q : nc - 1 - q;
        for (int r = 0; r < mc; ++r) {
          const V v = ldv(A + (int64_t)r * a.pitch + c);
          s += (Acc)(v * v);
        }
      }
      // stash per-row/col sums at index q+1; prefix below
      Acc *dst = kind == 0 ? rowTop : kind == 1 ? rowBot : kind == 2 ? colL : colR;
      dst[q + 1] = s;
    }
    // four corner tables of a^2, oriented so index (p,q) counts from the corner
    Acc *cor = reinterpret_cast<Acc *>(band);  // 4 * w * w, index [quad][p][q], p,q in 0..w-1
    for (int k = tid; k < 4 * w * w; k += nth) {
      const int quad = k / (w * w), p = (k / w) % w, q = k % w;
      Acc v2 = 0;
      if (p > 0 && q > 0) {
        const int r = (quad & 2) ? mc - p : p - 1;   // quad bit1: bottom rows
        const int c = (quad & 1) ? nc - q : q - 1;   // quad bit0: right cols
        const V v = ldv(A + (int64_t)r * a.pitch + c);
        v2 = (Acc)(v * v);
      }
      cor[k] = v2;
    }
    __syncthreads();
    if (tid == 0) {
      Acc tot = 0;
      for (int k = 0; k < (nth + 31) / 32; ++k) tot += wred[k];
      *total = tot;
    }
    if (tid < 4) {
      Acc *dst = tid == 0 ? rowTop : tid == 1 ? rowBot : tid == 2 ? colL : colR;
      dst[0] = 0;
      for (int q = 1; q < w; ++q) dst[q] += dst[q - 1];
    }
    // 2D inclusive prefix per corner: rows then columns (the DP of P:35 run in each corner)
    for (int k = tid; k < 4 * w; k += nth) {
      Acc *c = cor + (k / w) * w * w + (k % w) * w;
      for (int q = 1; q < w; ++q) c[q] += c[q - 1];
    }
    __syncthreads();
    for (int k = tid; k < 4 * w; k += nth) {
      Acc *c = cor + (k / w) * w * w + (k % w);
      for (int p = 1; p < w; ++p) c[p * w] += c[(p - 1) * w];
    }
    __syncthreads();
    for (int k = tid; k < W * W; k += nth) {
      const int s = k / W - hw, t = k % W - hw;
      const Acc rex = s > 0 ? rowTop[s] : (s < 0 ? rowBot[-s] : (Acc)0);
      const Acc cex = t > 0 ? colL[t] : (t < 0 ? colR[-t] : (Acc)0);
      Acc corner = 0;
      if (s != 0 && t != 0) {
        const int quad = (s < 0 ? 2 : 0) | (t < 0 ? 1 : 0);
        corner = cor[quad * w * w + abs(s) * w + abs(t)];
      }
      ga[k] = *total - rex - cex + corner;
    }
    __syncthreads();
  }

  // ---- cross term h by direct sums (S3, K4d), chunked over lag rows
  const int G = (W + KT - 1) / KT;
  In *tb = reinterpret_cast<In *>(band);
  const int br = a.br, FP = a.fpitch;
  In *fb = tb + br * nc;
  Key best{~0ull, ~0u};
  for (int s_lo = 0; s_lo < W; s_lo += a.sc) {
    const int SC = min(a.sc, W - s_lo);
    const int tasks = SC * G;
    const int R = max(1, nth / tasks);
    const int task = tid % tasks, rg = tid / tasks;
    const bool active = rg < R && tid < tasks * R;
    const int si = s_lo + task / G;           // lag-row index, s = si - hw
    const int g = task % G;                   // t-lags [g*KT, g*KT+KT) - hw
    for (int k = tid; k < SC * W; k += nth) hs[k] = 0;
    Acc acc64[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) acc64[k] = 0;
    for (int r0 = 0; r0 < mc; r0 += br) {
      const int nb = min(br, mc - r0);
      __syncthreads();
      for (int e = tid; e < nb * nc; e += nth) {
        const int i = e / nc, j = e % nc;
        tb[e] = Bt[(int64_t)(r0 + i) * a.tpitch + j];
      }
      const int fr0 = r0 - hw, nfr = nb + 2 * hw;
      for (int e = tid; e < nfr * FP; e += nth) {
        const int i = e / FP, jj = e % FP - hw;
        const int r = fr0 + i;
        In v = (In)0;
        if (r >= 0 && r < mc && jj >= 0 && jj < nc) v = A[(int64_t)r * a.pitch + jj];
        fb[e] = v;
      }
      __syncthreads();
      if (!active) continue;
      for (int i = rg; i < nb; i += R) {
        const In *brow = tb + i * nc;
        // frame row (r0+i) + s  ->  band row i + hw + s = i + si
        const In *arow = fb + (i + si) * FP + g * KT;
        if constexpr (sizeof(In) == 2 && !WIDE) {
          uint32_t acc32[KT];
#pragma unroll
          for (int k = 0; k < KT; ++k) acc32[k] = 0;
          V win[2 * KT];
#pragma unroll
          for (int k = 0; k < KT; ++k) win[KT + k] = ldv(arow + k);
          for (int j0 = 0; j0 < nc; j0 += KT) {
#pragma unroll
            for (int k = 0; k < KT; ++k) {
              win[k] = win[KT + k];
              win[KT + k] = ldv(arow + j0 + KT + k);
            }
#pragma unroll
            for (int jj = 0; jj < KT; ++jj) {
              const V bv = (j0 + jj < nc) ? ldv(brow + j0 + jj) : 0u;
#pragma unroll
              for (int k = 0; k < KT; ++k) acc32[k] += win[jj + k] * bv;
            }
            if ((j0 & (2 * KT - 1)) == KT || j0 + KT >= nc) {   // <= 16 products per flush
#pragma unroll
              for (int k = 0; k < KT; ++k) {
                acc64[k] += acc32[k];
                acc32[k] = 0;
              }
            }
          }
        } else {
          V win[2 * KT];
#pragma unroll
          for (int k = 0; k < KT; ++k) win[KT + k] = ldv(arow + k);
          for (int j0 = 0; j0 < nc; j0 += KT) {
#pragma unroll
            for (int k = 0; k < KT; ++k) {
              win[k] = win[KT + k];
              win[KT + k] = ldv(arow + j0 + KT + k);
            }
#pragma unroll
            for (int jj = 0; jj < KT; ++jj) {
              const V bv = (j0 + jj < nc) ? ldv(brow + j0 + jj) : (V)0;
#pragma unroll
              for (int k = 0; k < KT; ++k) acc64[k] += (Acc)win[jj + k] * (Acc)bv;
            }
          }
        }
      }
    }
    __syncthreads();
    if (active) {
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        const int ti = g * KT + k;
        if (ti < W) {
          if constexpr (std::is_same<Acc, u64>::value)
            atomicAdd(reinterpret_cast<u64 *>(&hs[(si - s_lo) * W + ti]), (u64)acc64[k]);
          else
            atomicAdd(reinterpret_cast<double *>(&hs[(si - s_lo) * W + ti]), (double)acc64[k]);
        }
      }
    }
    __syncthreads();
    // ---- score (S4) and running argmin over this chunk of lag rows
    const Acc *gbt = reinterpret_cast<const Acc *>(a.gb);
    for (int k = tid; k < SC * W; k += nth) {
      const int lag = s_lo * W + k;
      const int s = lag / W - hw, t = lag % W - hw;
      const Acc N = ga[lag] + gbt[lag] - 2 * hs[k];
      const double area = (double)((mc - abs(s)) * (nc - abs(t)));
      double fv = (double)N / (a.scale * area);
      if (fv < 0) fv = 0;   // fp64 path only: rounding residue of the 3-term form
      if (a.grid_out) a.grid_out[f * W * W + lag] = fv;
      Key kk{(u64)__double_as_longlong(fv), (unsigned)lag};
      if (key_less(kk, best)) best = kk;
    }
  }
  best = block_min_key(best, red);
  if (tid == 0) {
    const int s = (int)(best.idx / W) - hw, t = (int)(best.idx % W) - hw;
    if (a.shift_out) {
      a.shift_out[2 * f] = s;
      a.shift_out[2 * f + 1] = t;
    }
    if (a.f_out) a.f_out[f] = __longlong_as_double((long long)best.f);
    if (a.flags) a.flags[f] = (abs(s) == hw || abs(t) == hw) ? 1 : 0;
  }
}

// ------------------------------------------------------------------------- K6
// One CTA per frame: the nine candidates (2s+u, 2t+v), u,v in {-1,0,1}, at
// level l, each N by direct exact summation over its own overlap.
struct RefineArgs {
  const void *frames;  // level-l frame images
  int64_t fstride;
  int pitch;
  const void *tpl;
  int tpitch;
  int ml, nl;
  double scale;        // 16^l (u16 block sums) or 1
  int B;
  const int32_t *shift_in;   // [B][2] at level l+1
  int32_t *shift_out;        // [B][2] at level l
  double *f_out;             // [B] or null (f of the winner at level l)
};

template <class In>
__global__ void __launch_bounds__(256) k_refine(RefineArgs a) {
  typedef typename Arith<In>::Acc Acc;
  typedef typename Arith<In>::V V;
  const int64_t f = blockIdx.x;
  const In *A = reinterpret_cast<const In *>(a.frames) + f * a.fstride;
  const In *Bt = reinterpret_cast<const In *>(a.tpl);
  const int S = 2 * a.shift_in[2 * f], T = 2 * a.shift_in[2 * f + 1];
  const int ml = a.ml, nl = a.nl;
  Acc acc[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) acc[c] = 0;
  // template rows that can overlap any candidate: i + S + u in [0, ml) for some u
  const int ilo = max(0, -S - 1), ihi = min(ml, ml - S + 1);
  const int jlo = max(0, -T - 1), jhi = min(nl, nl - T + 1);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = ilo + wid; i < ihi; i += nw) {
    for (int j = jlo + lane; j < jhi; j += 32) {
      const V bv = (V)Bt[(int64_t)i * a.tpitch + j];
#pragma unroll
      for (int u = -1; u <= 1; ++u) {
        const int r = i + S + u;
        if (r < 0 || r >= ml) continue;
        const In *arow = A + (int64_t)r * a.pitch;
#pragma unroll
        for (int v = -1; v <= 1; ++v) {
          const int c = j + T + v;
          if (c < 0 || c >= nl) continue;
          const V av = (V)arow[c];
          if constexpr (sizeof(In) == 2) {
            const uint32_t d = av > bv ? av - bv : bv - av;
            acc[(u + 1) * 3 + (v + 1)] += (Acc)(d * d);
          } else {
            const double d = (double)av - (double)bv;
            acc[(u + 1) * 3 + (v + 1)] += d * d;
          }
        }
      }
    }
  }
  __shared__ Acc part[9][32];
  __shared__ Key red[32];
#pragma unroll
  for (int c = 0; c < 9; ++c) {
    const Acc v = warp_sum(acc[c]);
    if (lane == 0) part[c][wid] = v;
  }
  __syncthreads();
  Key k{~0ull, ~0u};
  if (threadIdx.x < 9) {
    Acc N = 0;
    for (int q = 0; q < nw; ++q) N += part[threadIdx.x][q];
    const int u = threadIdx.x / 3 - 1, v = threadIdx.x % 3 - 1;
    const int s = S + u, t = T + v;
    const double area = (double)((ml - abs(s)) * (nl - abs(t)));
    const double fv = (double)N / (a.scale * area);
    // candidate rank in (s,t) lexicographic order == threadIdx.x (u-major, v-minor)
    k = Key{(u64)__double_as_longlong(fv), (unsigned)threadIdx.x};
  }
  k = block_min_key(k, red);
  if (threadIdx.x == 0) {
    a.shift_out[2 * f] = S + (int)(k.idx / 3) - 1;
    a.shift_out[2 * f + 1] = T + (int)(k.idx % 3) - 1;
    if (a.f_out) a.f_out[f] = __longlong_as_double((long long)k.f);
  }
}

// ------------------------------------------------------------------------- K7
// corrected[i][j] = a[i+s][j+t] if in range else 0, 16 bytes of output per thread.
// Rows are `pitch` elements apart (a multiple of 16 bytes); columns >= n are written as 0.
template <class E>
__global__ void k_apply(const E *__restrict__ in, E *__restrict__ out, int m, int n, int pitch,
                        const int32_t *__restrict__ shifts, int B) {
  constexpr int V = 16 / sizeof(E);
  const int groups = pitch / V;
  const int64_t total = (int64_t)B * m * groups;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int cg = (int)(g % groups);
    const int64_t fr = g / groups;
    const int i = (int)(fr % m);
    const int64_t f = fr / m;
    const int s = shifts[2 * f], t = shifts[2 * f + 1];
    const int r = i + s;
    E o[V];
    if (r < 0 || r >= m) {
#pragma unroll
      for (int k = 0; k < V; ++k) o[k] = (E)0;
    } else {
      const E *src = in + f * (int64_t)m * pitch + (int64_t)r * pitch;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int c = cg * V + k + t;
        o[k] = (c >= 0 && c < n && cg * V + k < n) ? src[c] : (E)0;
      }
    }
    *reinterpret_cast<uint4 *>(out + f * (int64_t)m * pitch + (int64_t)i * pitch + cg * V) =
        *reinterpret_cast<const uint4 *>(o);
  }
}

}  // namespace moco

namespace moco {
// ---------------------------------------------------------------- peak probes
// Throughput microbenchmarks for the ALU roofs bench.py reports (SURVEY.md section 2.5
// "MB"): every thread runs `iters` x 8 independent dependency chains of one instruction
// kind; ops are counted as the instruction's arithmetic (FFMA/DFMA = 2 flops, IMAD = 2
// ops, IDP.2A = 4 ops: two 16x8-bit products and two adds).
template <int KIND>
__global__ void __launch_bounds__(256) k_probe(int iters, uint32_t seed, uint32_t *sink) {
  const uint32_t t = threadIdx.x + seed;
  if (KIND == 0) {
    float a[8], b = __uint_as_float(0x3f800001u + (t & 7)), c = 1e-7f;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = (float)(t + k);
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 1234.5f) sink[0] = 1;
  } else if (KIND == 1) {
    uint32_t a[8], b = 3u + (t & 7), c = t;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = t + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = a[k] * b + c;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= a[k];
    if (s == 0x12345u) sink[0] = s;
  } else if (KIND == 2) {
    uint32_t a[8], b = 0x01020304u ^ t, c = t * 7u;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = t + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = __dp2a_lo(c + k, b, a[k]);
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= a[k];
    if (s == 0x12345u) sink[0] = s;
  } else {
    double a[8], b = 1.0 + 1e-9 * (t & 7), c = 1e-12;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = (double)(t + k);
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 1234.5) sink[0] = 1;
  }
}
}  // namespace moco

namespace moco {
// ---------------------------------------------------------------- mean image (reports)
// mean[p] = (1/T) sum_f frames[f][p] (Fig. 2, "the mean of every image"); exact
// 64-bit integer sums for uint16, fp64 for float32; one division per pixel.
template <class E>
__global__ void __launch_bounds__(256) k_mean_image(const E *__restrict__ fr, int64_t T, int64_t mn,
                                                    double *__restrict__ out) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < mn; p += (int64_t)gridDim.x * blockDim.x) {
    if (std::is_same<E, uint16_t>::value) {
      u64 s = 0;
      for (int64_t f = 0; f < T; ++f) s += (u64)fr[f * mn + p];
      out[p] = (double)s / (double)T;
    } else {
      double s = 0;
      for (int64_t f = 0; f < T; ++f) s += (double)fr[f * mn + p];
      out[p] = s / (double)T;
    }
  }
}
}  // namespace moco
