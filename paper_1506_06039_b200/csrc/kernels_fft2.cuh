// kernels_fft2.cuh -- the FFT path of S3/S4 (the paper's method) for transform
// lengths with a two-pass register plan (kernels_fft.cuh Plan2p: 240, 256, 288, 300, 320,
// 360 -- every BASELINE config and the paper's default w = min(m,n)/3 at 256^2 coarse).
//
// Same mathematics as kernels_fft.cuh (H = IFFT2(FFT2(a_pad) . conj(FFT2(b_pad))),
// h(s,t) = H[s mod Mr][t mod Mc], certified candidate set, exact rescoring), laid out for
// the SM instead of for generality:
//
//   k_fft2_rows<P,L>  one read of the frame (bulk copies into shared memory): 2^L x 2^L
//                     block sums (S1, exact; L <= 1: levels = 2 runs on the level-1 image
//                     the level-1 refine reads anyway), the frame-energy partials of
//                     P:33-35 (row sums, edge columns, the row prefixes of the four corner
//                     blocks) and the row FFTs of two coarse rows packed per complex
//                     transform -> S[f][k][row]
//   k_fft2_cols<P>    per column bin: FFT_Mr, times conj(B^)/(Mr Mc), IFFT_Mr, keep the
//                     2w-1 lag rows -> P[f][s][k]
//   k_fft2_score<P>   per group of lag rows: IFFT_Mc of two packed lag rows, g_a of every
//                     lag from the energy partials (total - strips + corner),
//                     certified interval of f~; the LAST block of a frame (global counter)
//                     takes the candidate set Q and, when |Q| > 1 (or levels = 0, where
//                     f_min is the coarse f), re-scores Q exactly: N = sum_D (a - b)^2 in
//                     64-bit integers, straight from the level-0 frame.
//
// Transforms (N = N1 N2, n = n2 + N2 n1, k = k1 + N1 k2) run in place in shared memory with
// the two index orders of one padded array, row r of N2+1 slots (the gap spreads the
// stride-(N2+1) accesses over the banks):
//     natural order   element n at ix(n)  = (N2+1) (n / N2) + n % N2
//     k1-major order  element k at pos(k) = (N2+1) (k % N1) + k / N1
// The forward transform takes natural order to k1-major order (pass 1: radix-N1 over n1 per
// n2, twiddle; pass 2: radix-N2 over n2 per k1, both writing back to the addresses they
// read); the inverse takes k1-major order back to natural order (the same passes
// transposed).  No index arithmetic inside the passes beyond constant offsets, and no data
// movement between them.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels_fft.cuh"
#include "kernels_tc.cuh"

namespace moco {

constexpr int F2_THREADS = 288;
constexpr int F2_WARPS = F2_THREADS / 32;

template <int P>
struct F2 {
  static constexpr int N1 = Plan2p<P>::N1, N2 = Plan2p<P>::N2, N = N1 * N2, R = N2 + 1;
  // transforms per block (one thread per (transform, n2) in the wider pass)
  static constexpr int NF = F2_THREADS / (N1 > N2 ? N1 : N2) < 16 ? F2_THREADS / (N1 > N2 ? N1 : N2) : 16;
  static constexpr int STRIDE = (N1 * R) | 1;   // slots per transform (odd: bank spread)
  __device__ static __forceinline__ int ix(int n) { return n + n / N2; }
  __device__ static __forceinline__ int pos(int k) { return R * (k % N1) + k / N1; }
};

// ------------------------------------------------ packed-fp32 complex arithmetic (sm_100)
// A complex value is one 64-bit register pair (re, im); add/sub/mul/fma.rn.f32x2 do both
// halves in one instruction (FADD2/FMUL2/FFMA2), and ptxas folds the operand swaps and
// broadcasts below into the instructions' swizzle modifiers.
struct c2 { unsigned long long v; };
__device__ __forceinline__ c2 c2of(float2 z) { c2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(z.x), "f"(z.y)); return r; }
__device__ __forceinline__ float2 f2of(c2 a) { float2 z; asm("mov.b64 {%0, %1}, %2;" : "=f"(z.x), "=f"(z.y) : "l"(a.v)); return z; }
__device__ __forceinline__ c2 c2mk(float x, float y) { return c2of(make_float2(x, y)); }
__device__ __forceinline__ c2 operator+(c2 a, c2 b) { c2 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v)); return r; }
__device__ __forceinline__ c2 operator-(c2 a, c2 b) { c2 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v)); return r; }
__device__ __forceinline__ c2 mul2(c2 a, c2 b) { c2 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v)); return r; }
__device__ __forceinline__ c2 fma2(c2 a, c2 b, c2 c) {
  c2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}
__device__ __forceinline__ c2 swp(c2 a) { const float2 z = f2of(a); return c2mk(z.y, z.x); }
// z * (c + i s) = z c + (i s) z, (i s) z = (-s z.y, s z.x) = swap(z) * (-s, s)
__device__ __forceinline__ c2 cmul2(c2 z, float c, float s) { return fma2(z, c2mk(c, c), mul2(swp(z), c2mk(-s, s))); }
// m + (i s) u
__device__ __forceinline__ c2 addi(c2 m, c2 u, float s) { return fma2(swp(u), c2mk(-s, s), m); }

// z e^{SIGN 2 pi i m / N} with m a compile-time constant after unrolling: the quarter
// turns are swaps and sign changes, the rest two packed instructions
template <int N, int SIGN>
__device__ __forceinline__ c2 rotc(c2 z, int m) {
  if (m == 0) return z;
  if (N % 4 == 0 && m == N / 4) return mul2(swp(z), c2mk(-(float)SIGN, (float)SIGN));
  if (N % 2 == 0 && m == N / 2) return mul2(z, c2mk(-1.f, -1.f));
  if (N % 4 == 0 && m == 3 * N / 4) return mul2(swp(z), c2mk((float)SIGN, -(float)SIGN));
  const float2 cs = twk<N>(m);
  return cmul2(z, cs.x, (float)SIGN * cs.y);
}

template <int N, int SIGN>
struct D2;
template <int SIGN>
struct D2<2, SIGN> {
  static __device__ __forceinline__ void run(c2 (&v)[2]) {
    const c2 a = v[0], b = v[1];
    v[0] = a + b;
    v[1] = a - b;
  }
};
template <int SIGN>
struct D2<3, SIGN> {
  static __device__ __forceinline__ void run(c2 (&v)[3]) {
    const float s1 = (float)SIGN * 0.86602540378443865f;
    const c2 t = v[1] + v[2], u = v[1] - v[2];
    const c2 m = fma2(t, c2mk(-0.5f, -0.5f), v[0]);
    v[0] = v[0] + t;
    v[1] = addi(m, u, s1);
    v[2] = addi(m, u, -s1);
  }
};
template <int SIGN>
struct D2<4, SIGN> {
  static __device__ __forceinline__ void run(c2 (&v)[4]) {
    const c2 t0 = v[0] + v[2], t1 = v[0] - v[2], t2 = v[1] + v[3], d = v[1] - v[3];
    v[0] = t0 + t2;
    v[2] = t0 - t2;
    v[1] = addi(t1, d, (float)SIGN);
    v[3] = addi(t1, d, -(float)SIGN);
  }
};
template <int SIGN>
struct D2<5, SIGN> {
  static __device__ __forceinline__ void run(c2 (&v)[5]) {
    const float c1 = 0.30901699437494742f, c2_ = -0.80901699437494742f;
    const float s1 = (float)SIGN * 0.95105651629515357f, s2 = (float)SIGN * 0.58778525229247313f;
    const c2 a = v[0];
    const c2 t1 = v[1] + v[4], u1 = v[1] - v[4];
    const c2 t2 = v[2] + v[3], u2 = v[2] - v[3];
    v[0] = a + (t1 + t2);
    const c2 m1 = fma2(t2, c2mk(c2_, c2_), fma2(t1, c2mk(c1, c1), a));
    const c2 m2 = fma2(t2, c2mk(c1, c1), fma2(t1, c2mk(c2_, c2_), a));
    // r1 = i (s1 u1 + s2 u2), r2 = i (s2 u1 - s1 u2)
    const c2 r1 = fma2(swp(u2), c2mk(-s2, s2), mul2(swp(u1), c2mk(-s1, s1)));
    const c2 r2 = fma2(swp(u2), c2mk(s1, -s1), mul2(swp(u1), c2mk(-s2, s2)));
    v[1] = m1 + r1;
    v[4] = m1 - r1;
    v[2] = m2 + r2;
    v[3] = m2 - r2;
  }
};
template <int N1, int N2, int SIGN>
struct D2CT {
  static __device__ __forceinline__ void run(c2 (&v)[N1 * N2]) {
    constexpr int N = N1 * N2;
    c2 t[N1][N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) {
      c2 u[N1];
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) u[n1] = v[N2 * n1 + n2];
      D2<N1, SIGN>::run(u);
#pragma unroll
      for (int k1 = 0; k1 < N1; ++k1) t[k1][n2] = rotc<N, SIGN>(u[k1], (n2 * k1) % N);
    }
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) {
      D2<N2, SIGN>::run(t[k1]);
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) v[k1 + N1 * k2] = t[k1][k2];
    }
  }
};
template <int SIGN> struct D2<8, SIGN> : D2CT<2, 4, SIGN> {};
template <int SIGN> struct D2<9, SIGN> : D2CT<3, 3, SIGN> {};
template <int SIGN> struct D2<12, SIGN> : D2CT<3, 4, SIGN> {};
template <int SIGN> struct D2<15, SIGN> : D2CT<3, 5, SIGN> {};
template <int SIGN> struct D2<16, SIGN> : D2CT<4, 4, SIGN> {};
template <int SIGN> struct D2<18, SIGN> : D2CT<2, 9, SIGN> {};
template <int SIGN> struct D2<20, SIGN> : D2CT<4, 5, SIGN> {};

__device__ __forceinline__ c2 lds2(const float2 *p) { return c2of(*p); }
__device__ __forceinline__ void sts2(float2 *p, c2 a) { *p = f2of(a); }

// Forward: x natural -> X k1-major, X[k] = sum_n x[n] e^{-2 pi i n k / N}.  tw[m] =
// e^{-2 pi i m / N}.  nfft <= NF transforms at x + q * STRIDE.  All threads; ends synced.
template <int P>
__device__ __forceinline__ void f2_fwd(float2 *x, const float2 *tw, int nfft) {
  using G = F2<P>;
  constexpr int N1 = G::N1, N2 = G::N2, R = G::R, S = G::STRIDE;
  __syncthreads();
  for (int task = threadIdx.x; task < nfft * N2; task += blockDim.x) {
    const int q = task / N2, n2 = task - q * N2;
    float2 *b = x + q * S + n2;
    c2 v[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) v[n1] = lds2(b + R * n1);
    D2<N1, -1>::run(v);
    sts2(b, v[0]);
#pragma unroll
    for (int k1 = 1; k1 < N1; ++k1) {
      const float2 t = tw[n2 * k1];
      sts2(b + R * k1, cmul2(v[k1], t.x, t.y));
    }
  }
  __syncthreads();
  for (int task = threadIdx.x; task < nfft * N1; task += blockDim.x) {
    const int q = task / N1, k1 = task - q * N1;
    float2 *b = x + q * S + R * k1;
    c2 u[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) u[n2] = lds2(b + n2);
    D2<N2, -1>::run(u);
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) sts2(b + k2, u[k2]);
  }
  __syncthreads();
}

// Inverse: X k1-major -> x natural, x[n] = sum_k X[k] e^{+2 pi i n k / N} (unnormalised).
template <int P>
__device__ __forceinline__ void f2_inv(float2 *x, const float2 *tw, int nfft) {
  using G = F2<P>;
  constexpr int N1 = G::N1, N2 = G::N2, R = G::R, S = G::STRIDE;
  __syncthreads();
  for (int task = threadIdx.x; task < nfft * N1; task += blockDim.x) {
    const int q = task / N1, k1 = task - q * N1;
    float2 *b = x + q * S + R * k1;
    c2 u[N2];
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) u[k2] = lds2(b + k2);
    D2<N2, 1>::run(u);   // over k2 -> n2
    sts2(b, u[0]);
#pragma unroll
    for (int n2 = 1; n2 < N2; ++n2) {
      const float2 t = tw[k1 * n2];
      sts2(b + n2, cmul2(u[n2], t.x, -t.y));
    }
  }
  __syncthreads();
  for (int task = threadIdx.x; task < nfft * N2; task += blockDim.x) {
    const int q = task / N2, n2 = task - q * N2;
    float2 *b = x + q * S + n2;
    c2 v[N1];
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) v[k1] = lds2(b + R * k1);
    D2<N1, 1>::run(v);   // over k1 -> n1
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) sts2(b + R * n1, v[n1]);
  }
  __syncthreads();
}

// inclusive warp scan of u64
__device__ __forceinline__ u64 warp_scan_incl(u64 v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u64 t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Per-frame energy scratch (u64), for a frame of coarse size mc x nc and hw = w - 1:
//   [0]                       total sum of a^2                                    (atomic)
//   [1, 1+hw)                 top rows i:           sum_j a^2[i][j]
//   [1+hw, 1+2hw)             bottom rows (distance d from the last row)
//   [1+2hw, 1+3hw)            left columns j:       sum_i a^2[i][j]               (atomic)
//   [1+3hw, 1+4hw)            right columns (distance d from the last column)     (atomic)
//   [1+4hw + (quad*hw + i)*hw + (a-1)]  corner row prefixes: sum of a^2 over the first a
//                             columns from the quad's side of its i-th row from its edge
//                             (quad = bottom*2 + right)
// The atomic slots are zero on entry; the pick re-zeroes them.  Each frame holds two such
// sets: the squares a^2 (g_a) and the values a themselves (S_a, for the mean removal).
__host__ __device__ constexpr int f2_esz(int hw) { return 1 + 4 * hw + 4 * hw * hw; }
__host__ __device__ constexpr int f2_esz2(int hw) { return 2 * f2_esz(hw); }

struct F2RowsArgs {
  const uint16_t *frames;   // level-0 frames (levels L) or coarse images (L = 0)
  int64_t fstride;
  int pitch;
  int mc, nc, hw, Kc, mcp;
  int per;                  // row pairs per block (<= NF)
  const float2 *tw;         // [Mc]
  float2 *S;                // [B][Kc][mcp]
  u64 *E;                   // [B][2 esz] energy and linear partials
  const long long *mu;      // [0]: the integer mean removed from the frames (k_tpl_stats)
};

// raw bytes a k_fft2_rows block stages: 2 per row pairs x 2^L raw rows of 2^L nc samples
__host__ __device__ constexpr int f2_stage_bytes(int per, int L, int nc) { return 2 * per * (1 << L) * (1 << L) * nc * 2; }
constexpr int F2_STAGE_MAX = 64 * 1024;

// two blocks per SM (<= 113 registers, 36 B of spills): one block's bulk copy overlaps the
// other's transforms (126 registers and one block per SM before: C3 161 -> 106 us per
// 256 frames, the whole FFT path 723 -> 825 k frames/s)
template <int P, int L>
__global__ void __launch_bounds__(F2_THREADS, 2) k_fft2_rows(F2RowsArgs a) {
  pdl_enter();
  static_assert(L == 0 || L == 1, "2x2 block sums at most (levels = 2 runs on the level-1 image)");
  using G = F2<P>;
  constexpr int Mc = G::N, S = G::STRIDE, N2 = G::N2, D = 1 << L;
  extern __shared__ __align__(128) unsigned char f2sm[];
  __shared__ __align__(8) uint64_t bar[2];
  const int hw = a.hw, nc = a.nc, mc = a.mc;
  const int nrb = (a.mcp / 2 + a.per - 1) / a.per;
  const int64_t f = blockIdx.x / nrb;
  const int p0 = (blockIdx.x - (int)(f * nrb)) * a.per;
  const int np = min(a.per, a.mcp / 2 - p0), nr = 2 * np;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the block's raw rows (D per coarse row, D nc samples each), staged by bulk copies
  uint16_t *stg = reinterpret_cast<uint16_t *>(f2sm);
  float2 *tw = reinterpret_cast<float2 *>(f2sm + f2_stage_bytes(a.per, L, nc));
  float2 *x = tw + Mc;
  const int rawrow = D * nc;
  const int nraw = D * max(0, min(nr, mc - 2 * p0));
  const uint16_t *Fr = a.frames + f * a.fstride + (int64_t)(D * 2 * p0) * a.pitch;
  // two barriers: the raw rows of the first round of row pairs (one per warp) and the
  // rest, so that the first round starts while the second is still in flight
  const int n0 = min(nraw, 2 * D * F2_WARPS), n1 = nraw - n0;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&bar[0], (uint32_t)(n0 * rawrow * 2));
      if (n1 > 0) mbar_arrive_expect_tx(&bar[1], (uint32_t)(n1 * rawrow * 2));
    }
    __syncwarp();
    for (int r = lane; r < nraw; r += 32)
      bulk_g2s(stg + (size_t)r * rawrow, Fr + (int64_t)r * a.pitch, (uint32_t)(rawrow * 2), &bar[r < n0 ? 0 : 1]);
  }
  for (int k = threadIdx.x; k < Mc; k += blockDim.x) tw[k] = a.tw[k];
  // zero columns [nc, Mc) of every transform of the block
  const int tail = Mc - nc;
  for (int e = threadIdx.x; e < np * tail; e += blockDim.x) {
    const int q = e / tail, j = nc + (e - q * tail);
    x[q * S + G::ix(j)] = make_float2(0.f, 0.f);
  }
  // a warp per coarse row pair (one complex transform), a lane per 8 coarse columns; the
  // lane's first and last chunks hold the edge columns (hw <= 256), whose squares it
  // accumulates over its rows
  const int nch = nc >> 3;
  const int cl = lane, cr = lane + 32 * ((nch - 1 - lane) >> 5);
  const bool hasL = lane < nch && 8 * cl < hw, hasR = lane < nch && 8 * cr + 8 > nc - hw;
  // squares (g_a) and values (S_a) of the edge columns, per lane
  // (values: 32-bit, < 2^16 x 2 rows x 2 NF rows per block)
  u64 eL[8], eR[8];
  uint32_t lL[8], lR[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { eL[k] = eR[k] = 0; lL[k] = lR[k] = 0; }
  u64 wtot = 0, wlin = 0;
  u64 *E = a.E + f * f2_esz2(hw), *EL = E + f2_esz(hw);
  const int mu = (int)a.mu[0];
  // two-sided mean removal (the template shifted too): the linear partials (S_a) per lag
  // are needed; one-sided: only the frame total (for ||a - mu||_2)
  const bool lin = a.mu[3] != 0;
  // 8 coarse values of coarse row rl (block-local), columns 8c .. 8c+7, from the staged rows
  auto load8 = [&](int rl, int c, uint32_t (&v)[8]) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = 0;
    if (2 * p0 + rl >= mc) return;
    const uint16_t *Rr = stg + (size_t)(D * rl) * rawrow;
    if constexpr (L == 0) {
      const uint4 q4 = *reinterpret_cast<const uint4 *>(Rr + 8 * c);
      const uint32_t wv[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) { v[2 * k] = wv[k] & 0xffffu; v[2 * k + 1] = wv[k] >> 16; }
    } else {
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const uint4 u0 = *reinterpret_cast<const uint4 *>(Rr + 16 * c + 8 * g);
        const uint4 u1 = *reinterpret_cast<const uint4 *>(Rr + rawrow + 16 * c + 8 * g);
        const uint32_t w0[4] = {u0.x, u0.y, u0.z, u0.w}, w1[4] = {u1.x, u1.y, u1.z, u1.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          v[4 * g + k] = (w0[k] & 0xffffu) + (w0[k] >> 16) + (w1[k] & 0xffffu) + (w1[k] >> 16);
      }
    }
  };
  for (int q = warp; q < np; q += F2_WARPS) {
    if (q < F2_WARPS) mbar_wait(&bar[0], 0);
    else if (q < 2 * F2_WARPS && n1 > 0) mbar_wait(&bar[1], 0);
    float2 *xq = x + q * S;
    const int r0 = 2 * (p0 + q);
    const float m0 = r0 < mc ? (float)mu : 0.f, m1 = r0 + 1 < mc ? (float)mu : 0.f;
    u64 rs0 = 0, rs1 = 0;
    uint32_t ls0 = 0, ls1 = 0;   // < 2^16 x nc / 32 per lane
    for (int c = lane; c < nch; c += 32) {
      uint32_t v0[8], v1[8];
      load8(2 * q, c, v0);
      load8(2 * q + 1, c, v1);
      // natural-order slots of columns 8c .. 8c+7 (at most one row break of the padding);
      // the transforms see a - mu on the support (exact in fp32), 0 outside
      const int j0 = 8 * c, q0 = j0 / N2, brk = (q0 + 1) * N2 - j0;
      float2 *xc = xq + j0 + q0;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        xc[k + (k >= brk ? 1 : 0)] = make_float2((float)v0[k] - m0, (float)v1[k] - m1);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t s0 = v0[k] * v0[k], s1 = v1[k] * v1[k];   // < 2^32 (coarse values < 2^16)
        rs0 += s0;
        rs1 += s1;
        ls0 += v0[k];
        ls1 += v1[k];
        if (hasL && c == cl) { eL[k] += (u64)s0 + s1; lL[k] += v0[k] + v1[k]; }
        if (hasR && c == cr) { eR[k] += (u64)s0 + s1; lR[k] += v0[k] + v1[k]; }
      }
    }
    rs0 = warp_sum(rs0);
    rs1 = warp_sum(rs1);
    if (mu) {
      ls0 = warp_sum(ls0);
      ls1 = warp_sum(ls1);
    }
    if (lane < 2) {
      const int r = r0 + lane;
      const u64 rs = lane ? rs1 : rs0, ls = lane ? ls1 : ls0;
      if (r < mc) {
        wtot += rs;
        wlin += ls;
        if (r < hw) { E[1 + r] = rs; if (lin) EL[1 + r] = ls; }
        if (r >= mc - hw) { E[1 + hw + (mc - 1 - r)] = rs; if (lin) EL[1 + hw + (mc - 1 - r)] = ls; }
      }
    }
  }
  if (lane < 2 && wtot) atomicAdd(&E[0], wtot);
  if (lane < 2 && wlin) atomicAdd(&EL[0], wlin);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int jl = 8 * cl + k, jr = 8 * cr + k;
    if (hasL && jl < hw) {
      if (eL[k]) atomicAdd(&E[1 + 2 * hw + jl], eL[k]);
      if (lin && lL[k]) atomicAdd(&EL[1 + 2 * hw + jl], (u64)lL[k]);
    }
    if (hasR && jr < nc && jr >= nc - hw) {
      if (eR[k]) atomicAdd(&E[1 + 3 * hw + (nc - 1 - jr)], eR[k]);
      if (lin && lR[k]) atomicAdd(&EL[1 + 3 * hw + (nc - 1 - jr)], (u64)lR[k]);
    }
  }
  __syncthreads();
  // corner row prefixes (squares and values): a warp per (corner row, side), scanning the
  // hw columns (the frame value is the transform input plus mu)
  for (int t = warp; t < 2 * nr; t += F2_WARPS) {
    const int rl = t >> 1, right = t & 1, r = 2 * p0 + rl;
    if (r >= mc) continue;
    const float *xr = reinterpret_cast<const float *>(x + (rl >> 1) * S) + (rl & 1);
    for (int bot = 0; bot < 2; ++bot) {
      const int i = bot ? mc - 1 - r : r;
      if (i >= hw) continue;
      u64 *o = E + 1 + 4 * hw + ((2 * bot + right) * hw + i) * hw;
      u64 *ol = EL + 1 + 4 * hw + ((2 * bot + right) * hw + i) * hw;
      u64 carry = 0, carryl = 0;
      for (int a0 = 0; a0 < hw; a0 += 32) {
        const int aa = a0 + lane;
        u64 v2 = 0, v1 = 0;
        if (aa < hw) {
          const uint32_t v = (uint32_t)((int)xr[2 * G::ix(right ? nc - 1 - aa : aa)] + mu);
          v2 = (u64)(v * v);
          v1 = v;
        }
        const u64 sc = warp_scan_incl(v2) + carry;
        if (aa < hw) o[aa] = sc;
        carry = __shfl_sync(0xffffffffu, sc, 31);
        if (lin) {
          const u64 scl = warp_scan_incl(v1) + carryl;
          if (aa < hw) ol[aa] = scl;
          carryl = __shfl_sync(0xffffffffu, scl, 31);
        }
      }
    }
  }
  f2_fwd<P>(x, tw, np);
  // unpack the two real rows' spectra into S[f][k][row]: warps over k, lanes over rows
  {
    float2 *Sk = a.S + f * a.Kc * a.mcp + 2 * p0 + lane + (int64_t)warp * a.mcp;
    const int q = lane >> 1;
    const bool odd = lane & 1;
    const float2 *xq = x + q * S;
    const int64_t step = (int64_t)F2_WARPS * a.mcp;
    for (int k = warp; k < a.Kc; k += F2_WARPS, Sk += step) {
      if (lane >= nr) continue;
      const unsigned uk = (unsigned)k, un = (unsigned)(k == 0 ? 0 : Mc - k);
      const float2 zk = xq[G::R * (uk % G::N1) + uk / G::N1];
      const float2 zn = xq[G::R * (un % G::N1) + un / G::N1];
      // X0 = (Z[k] + conj Z[-k]) / 2, X1 = (Z[k] - conj Z[-k]) / 2i
      *Sk = odd ? make_float2(0.5f * (zk.y + zn.y), -0.5f * (zk.x - zn.x))
                : make_float2(0.5f * (zk.x + zn.x), 0.5f * (zk.y - zn.y));
    }
  }
}

struct F2ColsArgs {
  const float2 *S;          // [B][Kc][mcp]
  int mc, Kc, mcp, W, hw;
  int Mc;                   // row transform length (Hermitian weights of the stored bins)
  int lin;                  // mean removal on: also the values' corner tables
  int per;                  // column bins per block (<= NF)
  const float2 *tw;         // [Mr]
  const float2 *Bc;         // [Kc][Mr] conj(B^)/(Mr Mc)   (frames)
  float2 *P;                // [B][W][Kc]                  (frames)
  float2 *Bout;             // template mode: Bc out, or null
  float scale;              // template mode: 1/(Mr Mc)
  u64 *E;                   // [B][esz] energy partials: the corner row prefixes become 2-D
                            // corner sums here (split over the frame's blocks)
  double *ynorm;            // [B] sum over the full spectrum of |Y|^2, Y the product the
                            // inverse transform gets (the certification bound's inverse term)
};

// four blocks per SM (<= 56 registers; the 360-point instantiation needs 66 and ran three
// blocks: w = 85 435 -> 457 k frames/s)
template <int P>
__global__ void __launch_bounds__(F2_THREADS, 4) k_fft2_cols(F2ColsArgs a) {
  pdl_enter();
  using G = F2<P>;
  constexpr int Mr = G::N, S = G::STRIDE;
  extern __shared__ __align__(128) unsigned char f2sm[];
  float2 *tw = reinterpret_cast<float2 *>(f2sm);
  float2 *x = tw + Mr;
  const int ncb = (a.Kc + a.per - 1) / a.per;
  const int64_t f = blockIdx.x / ncb;
  const int k0 = (blockIdx.x - (int)(f * ncb)) * a.per;
  const int nk = min(a.per, a.Kc - k0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < Mr; k += blockDim.x) tw[k] = a.tw[k];
  // a warp per column bin: rows u (natural order), 4 loads in flight per lane
  const float2 *Sf = a.S + (f * a.Kc + k0) * a.mcp;
  for (int q = warp; q < nk; q += F2_WARPS) {
    float2 *xq = x + q * S;
    for (int u0 = 0; u0 < Mr; u0 += 128) {
      float2 v[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int u = u0 + 32 * h + lane;
        v[h] = u < a.mc ? __ldcg(Sf + (int64_t)q * a.mcp + u) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int u = u0 + 32 * h + lane;
        if (u < Mr) xq[G::ix(u)] = v[h];
      }
    }
  }
  if (a.E) {
    // corner tables of the DP: the row prefixes RP[quad][i][a] of k_fft2_rows become
    // CP[quad][p-1][a] = sum_{i<p} RP[quad][i][a], in place; this block scans its share of
    // the 4 hw columns (quad, a) (both sets -- squares and values -- when the mean is
    // removed from both sides).  hw >= 24: lanes over columns (adjacent a: coalesced), warps over segments of the hw
    // rows -- each warp sums its segment, the segment sums are scanned through shared
    // memory, a second pass writes the prefixes (w = 85 382 -> 434 k, C3 844 -> 876 k
    // frames/s); smaller hw: a warp scan per column (one 32-row chunk; C2 897 vs 889 k)
    __shared__ u64 segsum[F2_WARPS][32];
    const int hw = a.hw, ncol = (a.lin ? 8 : 4) * hw;
    const int cpb = (ncol + ncb - 1) / ncb, c0 = (blockIdx.x - (int)(f * ncb)) * cpb, c1 = min(ncol, c0 + cpb);
    u64 *RP = a.E + f * f2_esz2(hw) + 1 + 4 * hw;
    auto colp = [&](int c) {
      const int set = c / (4 * hw), cq = c - set * 4 * hw;
      const int quad = cq / hw, aa = cq - quad * hw;
      return RP + (int64_t)set * f2_esz(hw) + (int64_t)quad * hw * hw + aa;
    };
    if (hw < 24) {
      for (int c = c0 + warp; c < c1; c += F2_WARPS) {
        u64 *col = colp(c);
        const u64 v = lane < hw ? col[(int64_t)lane * hw] : 0;
        const u64 sc = warp_scan_incl(v);
        if (lane < hw) col[(int64_t)lane * hw] = sc;
      }
    } else {
      const int seg = (hw + F2_WARPS - 1) / F2_WARPS, i0 = min(hw, warp * seg), i1 = min(hw, i0 + seg);
      for (int cg = c0; cg < c1; cg += 32) {
        const int c = cg + lane;
        u64 *col = c < c1 ? colp(c) : RP;
        u64 sum = 0;
        if (c < c1)
          for (int i = i0; i < i1; ++i) sum += col[(int64_t)i * hw];
        segsum[warp][lane] = sum;
        __syncthreads();
        u64 carry = 0;
        for (int w2 = 0; w2 < warp; ++w2) carry += segsum[w2][lane];
        if (c < c1)
          for (int i = i0; i < i1; ++i) {
            carry += col[(int64_t)i * hw];
            col[(int64_t)i * hw] = carry;
          }
        __syncthreads();
      }
    }
  }
  f2_fwd<P>(x, tw, nk);
  if (a.Bout) {
    for (int q = warp; q < nk; q += F2_WARPS)
      for (int u = lane; u < Mr; u += 32) {
        const float2 v = x[q * S + G::pos(u)];
        a.Bout[(int64_t)(k0 + q) * Mr + u] = make_float2(v.x * a.scale, -v.y * a.scale);
      }
    return;
  }
  double ysq = 0.0;
  for (int q = warp; q < nk; q += F2_WARPS) {
    const float2 *Bk = a.Bc + (int64_t)(k0 + q) * Mr;
    // a stored bin k stands for k and Mc - k of the Hermitian full spectrum
    const int kk = k0 + q;
    const double wk = (kk == 0 || 2 * kk == a.Mc) ? 1.0 : 2.0;
    double yq = 0.0;
    for (int u = lane; u < Mr; u += 32) {
      float2 *c = x + q * S + G::pos(u);
      const float2 y = cmul(*c, __ldg(Bk + u));
      *c = y;
      yq += (double)y.x * y.x + (double)y.y * y.y;
    }
    ysq += wk * yq;
  }
  if (a.ynorm) {
    ysq = warp_sum(ysq);
    if (lane == 0 && ysq > 0) atomicAdd(a.ynorm + f, ysq);
  }
  f2_inv<P>(x, tw, nk);
  float2 *Pf = a.P + f * a.W * a.Kc + k0;
  for (int e = threadIdx.x; e < a.W * nk; e += blockDim.x) {
    const int si = e / nk, q = e - si * nk;
    int u = si - a.hw;
    u += u < 0 ? Mr : 0;
    Pf[(int64_t)si * a.Kc + q] = x[q * S + G::ix(u)];
  }
}

struct F2ScoreArgs {
  const float2 *P;          // [B][W][Kc]
  const float2 *tw;         // [Mc]
  int mc, nc, hw, W, Kc;
  int per;                  // lag-row pairs per block (<= NF)
  const u64 *E;             // [B][esz] energy partials (k_fft2_rows)
  u64 *Ew;                  // the same, written: the pick re-zeroes the accumulated slots
  const u64 *gb;            // [W*W] template energies
  double scale;             // 16^L
  double eps_f, eps_i;      // eps_h = ||a'||_2 (eps_f ||b'||_2 + eps_i ||b'||_1) (kernels_fft.cuh)
  const unsigned long long *b1;   // (unused by k_fft2_score: the mean-removed norms come from tst)
  const long long *tst;     // [3] mu, ||b - mu||_1, ||b - mu||_2^2 (k_tpl_stats)
  const long long *gl;      // [W*W] template linear sums per lag (k_energy_u16_t<false> on the template)
  double *ynorm;            // [B] |Y|^2 summed over the full spectrum (k_fft2_cols), re-zeroed by the pick
  double sqrtN;             // sqrt(Mr Mc)
  const uint16_t *frames;   // level-0 frames (exact rescoring through block sums)
  int64_t fstride;
  int pitch;
  int L;                    // block-sum levels from `frames` to the coarse level (0 or 1)
  const uint16_t *tpl;      // coarse template
  int tpitch;
  float *lb;                // [B][W*W]
  float *rmin;              // [B][W] per lag row: the minimum of its lb values
  int *ub;                  // [B] float bits, FFT_UB_INIT between calls
  int *cnt;                 // [B] finished blocks, 0 between calls
  int32_t *shift_out;       // [B][2]
  double *f_out;            // [B] or null (levels = 0: f_min is the coarse f)
  uint8_t *flags;           // [B] or null
  int *qcount;              // [B] or null
  float *h_out;             // [B][W*W] or null (diagnostics)
  int *qn;                  // [B] candidates left for k_fft2_rescore (0: resolved; -1: all lags)
  int *ql;                  // [B][FFT_QCAP] their lags
  u64 *nacc;                // [B][max(FFT_QCAP, W*W)] exact N partial sums, zero between calls
  int *cnt2;                // [B] finished k_fft2_rescore blocks, 0 between calls
  int rparts;               // k_fft2_rescore blocks per frame
};

// coarse value (2^L x 2^L block sum) at coarse column jj of the coarse row whose first raw
// row is ar: D raw rows, D adjacent samples each (4- / 8-byte aligned loads)
template <int L>
__device__ __forceinline__ uint32_t f2_coarse_at(const uint16_t *ar, int pitch, int jj) {
  if constexpr (L == 0) {
    return __ldg(ar + jj);
  } else if constexpr (L == 1) {
    const uint32_t u0 = __ldg(reinterpret_cast<const uint32_t *>(ar + 2 * jj));
    const uint32_t u1 = __ldg(reinterpret_cast<const uint32_t *>(ar + pitch + 2 * jj));
    return (u0 & 0xffffu) + (u0 >> 16) + (u1 & 0xffffu) + (u1 >> 16);
  } else {
    uint32_t v = 0;
#pragma unroll
    for (int dy = 0; dy < 4; ++dy) {
      const uint2 u = __ldg(reinterpret_cast<const uint2 *>(ar + (int64_t)dy * pitch + 4 * jj));
      v += (u.x & 0xffffu) + (u.x >> 16) + (u.y & 0xffffu) + (u.y >> 16);
    }
    return v;
  }
}

// partial exact N(s,t) = sum over the coarse rows [r0, r1) of D_{s,t} of
// (a_c[i+s][j+t] - b_c[i][j])^2, a_c the 2^L x 2^L block sums of the level-0 frame,
// in 64-bit integers; all threads of the block; result to thread 0.  Warps over rows (four
// in flight), lanes over columns.
template <int L>
__device__ u64 f2_exact_N(const F2ScoreArgs &a, int64_t f, int s, int t, int r0, int r1, u64 *red) {
  constexpr int D = 1 << L;
  const int mc = a.mc, nc = a.nc;
  const int i0 = max(r0, max(0, -s)), i1 = min(r1, mc - max(0, s)), j0 = max(0, -t), j1 = nc - max(0, t);
  const uint16_t *Fr = a.frames + f * a.fstride;
  const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  u64 acc = 0;
  for (int i = i0 + 4 * wid; i < i1; i += 4 * nw) {
    for (int j = j0 + lane; j < j1; j += 32) {
      uint32_t av[4], bv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int ii = min(i + q, i1 - 1);
        av[q] = f2_coarse_at<L>(Fr + (int64_t)(D * (ii + s)) * a.pitch, a.pitch, j + t);
        bv[q] = __ldg(a.tpl + (int64_t)ii * a.tpitch + j);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int d = (int)av[q] - (int)bv[q];
        if (i + q < i1) acc += (u64)((uint32_t)(d * d));   // |d| < 2^16
      }
    }
  }
  acc = warp_sum(acc);
  __syncthreads();
  if (lane == 0) red[wid] = acc;
  __syncthreads();
  u64 tot = 0;
  if (threadIdx.x == 0)
    for (int k = 0; k < nw; ++k) tot += red[k];
  return tot;
}

// Partial exact N over the coarse rows [r0, r1) for EVERY lag of a box s in [s0, s0+ns),
// t in [t0, t0+nt) (ns, nt <= 3) in one pass: the template value b_c[i][j] is loaded once
// per pixel, each box row's frame values once per lane (two words) and shifted to the box
// columns with warp shuffles.  acc[ds*3+dt] per thread (u64), not yet reduced.
template <int L>
__device__ __forceinline__ void f2_exact_box(const F2ScoreArgs &a, int64_t f, int s0, int ns, int t0, int nt, int r0,
                                             int r1, u64 (&acc)[9]) {
  constexpr int D = 1 << L;
  const int mc = a.mc, nc = a.nc;
  const uint16_t *Fr = a.frames + f * a.fstride;
  const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = r0 + wid; i < r1; i += nw) {
    const uint16_t *br = a.tpl + (int64_t)i * a.tpitch;
    for (int jb = 0; jb < nc; jb += 32) {
      const int j = jb + lane;
      const int bv = j < nc ? (int)__ldg(br + j) : 0;
#pragma unroll
      for (int ds = 0; ds < 3; ++ds) {
        if (ds >= ns) break;
        const int fr = i + s0 + ds;   // frame row (warp-uniform)
        if (fr < 0 || fr >= mc) continue;
        const uint16_t *ar = Fr + (int64_t)(D * fr) * a.pitch;
        const int c0 = j + t0, c1 = c0 + 32;
        const uint32_t v0 = (c0 >= 0 && c0 < nc) ? f2_coarse_at<L>(ar, a.pitch, c0) : 0u;
        const uint32_t v1 = (c1 >= 0 && c1 < nc) ? f2_coarse_at<L>(ar, a.pitch, c1) : 0u;
#pragma unroll
        for (int dt = 0; dt < 3; ++dt) {
          const uint32_t x0 = __shfl_sync(0xffffffffu, v0, (lane + dt) & 31);
          const uint32_t x1 = __shfl_sync(0xffffffffu, v1, (lane + dt) & 31);
          if (dt >= nt) continue;
          const int fc = j + t0 + dt;   // frame column of this lane's pixel at lag t0 + dt
          if (j >= nc || fc < 0 || fc >= nc) continue;
          const int d = (int)(lane + dt < 32 ? x0 : x1) - bv;
          acc[ds * 3 + dt] += (u64)((uint32_t)(d * d));   // |d| < 2^16
        }
      }
    }
  }
}

// four blocks per SM (<= 56 registers, no spills; 68 and three blocks before: w = 85
// 370 -> 381 k frames/s).  Five for k_fft2_cols spills its radix-20 codelets and is slower.
template <int P>
__global__ void __launch_bounds__(F2_THREADS, 4) k_fft2_score(F2ScoreArgs a) {
  pdl_enter();
  using G = F2<P>;
  constexpr int Mc = G::N, S = G::STRIDE;
  extern __shared__ __align__(128) unsigned char f2sm[];
  const int W = a.W, hw = a.hw;
  float2 *tw = reinterpret_cast<float2 *>(f2sm);
  float2 *x = tw + Mc;
  u64 *RX = reinterpret_cast<u64 *>(x + G::NF * S);   // [W] excluded-row energy per s
  u64 *CX = RX + W;                                   // [W] excluded-column energy per t
  u64 *RXl = CX + W, *CXl = RXl + W;                  // [W] the same for the values (S_a)
  double *rinv = reinterpret_cast<double *>(CXl + W);                   // [W]
  double *cinv = rinv + W;                                               // [W]
  __shared__ float redf[32];
  __shared__ int qn, qlist[FFT_QCAP], last;
  const int npairs = (W + 1) / 2, npb = (npairs + a.per - 1) / a.per;
  const int64_t f = blockIdx.x / npb;
  const int p0 = (blockIdx.x - (int)(f * npb)) * a.per;
  const int np = min(a.per, npairs - p0), s0 = 2 * p0, nr = min(2 * np, W - s0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const u64 *E = a.E + f * f2_esz2(hw), *EL = E + f2_esz(hw);
  for (int k = threadIdx.x; k < Mc; k += blockDim.x) tw[k] = a.tw[k];
  // packed lag rows, Hermitian extension of each half spectrum: x = row s1 + i row s2, in
  // k1-major order for the inverse transform; a warp per pair
  const float2 *Pf = a.P + (f * W + s0) * a.Kc;
  for (int q = warp; q < np; q += F2_WARPS) {
    const bool two = 2 * q + 1 < nr;
    const float2 *P1 = Pf + (int64_t)(2 * q) * a.Kc, *P2 = P1 + a.Kc;
    for (int k = lane; k < Mc; k += 32) {
      const bool lo = k < a.Kc;
      const int kk = lo ? k : Mc - k;
      float2 v1 = __ldcg(P1 + kk);
      float2 v2 = two ? __ldcg(P2 + kk) : make_float2(0.f, 0.f);
      if (!lo) { v1.y = -v1.y; v2.y = -v2.y; }
      x[q * S + G::pos(k)] = make_float2(v1.x - v2.y, v1.y + v2.x);
    }
  }
  // energies and linear sums: the excluded strips by warp scans of the edge row /
  // column sums
  const bool lin = a.tst[3] != 0;   // two-sided mean removal: S_a per lag
  if (warp < (lin ? 8 : 4)) {   // (warp & 3): 0 top rows, 1 bottom rows, 2 left cols, 3 right cols; warp >= 4: values
    const int side = warp & 3;
    u64 *o = warp < 4 ? (side < 2 ? RX : CX) : (side < 2 ? RXl : CXl);
    const u64 *src = (warp < 4 ? E : EL) + 1 + side * hw;
    if ((side & 1) && lane == 0) o[hw] = 0;
    u64 carry = 0;
    for (int d0 = 0; d0 < hw; d0 += 32) {
      const int d = d0 + lane;
      const u64 sc = warp_scan_incl(d < hw ? src[d] : 0) + carry;
      if (d < hw) o[(side & 1) ? hw - d - 1 : hw + d + 1] = sc;   // s > 0 excludes the top rows
      carry = __shfl_sync(0xffffffffu, sc, 31);
    }
  }
  for (int k = threadIdx.x; k < W; k += blockDim.x) {
    rinv[k] = 1.0 / (a.scale * (double)(a.mc - abs(k - hw)));
    cinv[k] = 1.0 / (double)(a.nc - abs(k - hw));
  }
  f2_inv<P>(x, tw, np);
  // The transforms saw a' = a - mu_a and b' = b - mu_b on the supports, so
  //   h = sum_D a b = h' + mu_b S_a + mu_a S_b - mu_a mu_b A         (exact integers aside h')
  // with S_a, S_b the frame / template sums over D's two rectangles (two-sided: mu_a = mu_b
  // = mu; one-sided: mu_b = 0, no S_a).  Error of h~ = h~' + [correction]: the derived
  // bound with the shifted norms, plus the rounding of the fp64 sum; the fp64 evaluation of
  // N~ = g_a + g_b - 2 h~ adds its own.
  const u64 tot = E[0], totl = EL[0];
  const long long mu = a.tst[0], mub = a.tst[3];
  const long long n_sup = (long long)a.mc * a.nc;
  const double a2p = (double)((long long)tot - 2 * mu * (long long)totl + mu * mu * n_sup);   // ||a - mu||_2^2
  // forward terms through Cauchy-Schwarz with ||b'||_2; the inverse transform's term from
  // the computed spectrum norm: ||E_inv||_2 <= Ci u sqrt(N) ||Y~||_2
  const double epsh = (sqrt(a2p) * (1.0 + 1e-12)) * a.eps_f * sqrt((double)a.tst[2]) * (1.0 + 1e-12) +
                      a.eps_i * a.sqrtN * sqrt(a.ynorm[f]) * (1.0 + 1e-9);
  constexpr double U53 = 1.1102230246251565e-16;   // 2^-53
  float best = 3.0e38f;
  float *lbf = a.lb + f * W * W;
  for (int rl = warp; rl < nr; rl += F2_WARPS) {
    const int si = s0 + rl, s = si - hw;
    const float *xr = reinterpret_cast<const float *>(x + (rl >> 1) * S) + (rl & 1);
    const double ri = rinv[si];
    const u64 rx = RX[si], rxl = lin ? RXl[si] : 0;
    const int64_t cq = (int64_t)(s < 0 ? 2 : 0) * hw * hw;
    const u64 *CPq = E + 1 + 4 * hw + cq, *CPl = EL + 1 + 4 * hw + cq;
    float rowlb = 3.0e38f;
    // the lag's global operands (2-D corner sum of the frame, template energy and sum),
    // loaded one lane iteration ahead so their latency overlaps the previous lag's math
    auto ldlag = [&](int ti, u64 &cv, u64 &gbv, long long &glv) {
      const int t = ti - hw, lag = si * W + ti;
      cv = 0;
      if (s != 0 && t != 0)   // 2-D corner sums of the excluded |s| x |t| corner (k_fft2_cols)
        cv = __ldg(CPq + (t < 0 ? hw * hw : 0) + (int64_t)(abs(s) - 1) * hw + abs(t) - 1);
      gbv = __ldg(a.gb + lag);
      glv = mu ? __ldg(a.gl + lag) : 0;
    };
    u64 cv_n = 0, gb_n = 0;
    long long gl_n = 0;
    if (lane < W) ldlag(lane, cv_n, gb_n, gl_n);
    for (int ti = lane; ti < W; ti += 32) {
      const u64 cv = cv_n, gbv = gb_n;
      const long long glv = gl_n;
      if (ti + 32 < W) ldlag(ti + 32, cv_n, gb_n, gl_n);
      const int t = ti - hw;
      const int tt = t < 0 ? t + Mc : t;
      const float hp = xr[2 * G::ix(tt)];
      const int lag = si * W + ti;
      u64 ga = tot - rx - CX[ti] + cv, sa = lin ? totl - rxl - CXl[ti] : 0;
      if (lin && s != 0 && t != 0)
        sa += __ldg(CPl + (t < 0 ? hw * hw : 0) + (int64_t)(abs(s) - 1) * hw + abs(t) - 1);
      const long long area = (long long)(a.mc - abs(s)) * (a.nc - abs(t));
      const long long corr = mu ? mub * (long long)sa + mu * (glv - mub * area) : 0;
      const double h = (double)hp + (double)corr;
      if (a.h_out) a.h_out[f * W * W + lag] = (float)h;
      const double gsum = (double)ga + (double)gbv;
      const double hdev = epsh + 2 * U53 * (fabs((double)hp) + fabs((double)corr));   // |h~ - h|
      const double inv = ri * cinv[ti];
      const double fa = (gsum - 2.0 * h) * inv;
      const double del = (2.0 * hdev + 4 * U53 * (gsum + 2.0 * fabs(h))) * inv;
      best = fminf(best, (float)(fa + del) * (1.0f + 1e-6f));
      const float lbv = (float)(fa - del) * (1.0f - 1e-6f);
      lbf[lag] = lbv;
      rowlb = fminf(rowlb, lbv);
    }
    for (int o = 16; o > 0; o >>= 1) rowlb = fminf(rowlb, __shfl_xor_sync(0xffffffffu, rowlb, o));
    if (lane == 0) a.rmin[f * W + si] = rowlb;
  }
  for (int o = 16; o > 0; o >>= 1) best = fminf(best, __shfl_xor_sync(0xffffffffu, best, o));
  if (lane == 0) redf[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = 3.0e38f;
    for (int k = 0; k < F2_WARPS; ++k) b = fminf(b, redf[k]);
    atomicMin(a.ub + f, __float_as_int(fmaxf(b, 0.f)));
    __threadfence();
    last = atomicAdd(a.cnt + f, 1) == npb - 1;
    qn = 0;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the last block of the frame: candidate set Q = {lag : f~ - delta <= min(f~ + delta)}
  // (only the lag rows whose minimum lower bound reaches thr are scanned: the same set)
  const float thr = __int_as_float(atomicAdd(a.ub + f, 0));
  __shared__ int nrows, rlist[F2_THREADS];
  for (int r0 = 0; r0 < W; r0 += F2_THREADS) {
    if (threadIdx.x == 0) nrows = 0;
    __syncthreads();
    const int si = r0 + threadIdx.x;
    if (si < W && __ldcg(a.rmin + f * W + si) <= thr) rlist[atomicAdd(&nrows, 1)] = si;
    __syncthreads();
    for (int k = warp; k < nrows; k += F2_WARPS) {
      const int base = rlist[k] * W;
      for (int ti = lane; ti < W; ti += 32)
        if (__ldcg(lbf + base + ti) <= thr) {
          const int q = atomicAdd(&qn, 1);
          if (q < FFT_QCAP) qlist[q] = base + ti;
        }
    }
    __syncthreads();
  }
  const int nq = qn;
  const bool all = nq > FFT_QCAP;
  if (threadIdx.x == 0) {
    if (nq == 1 && !a.f_out) {   // the one candidate is the exact argmin
      const int s = qlist[0] / W - hw, t = qlist[0] % W - hw;
      a.shift_out[2 * f] = s;
      a.shift_out[2 * f + 1] = t;
      if (a.flags) a.flags[f] = (uint8_t)((abs(s) == hw || abs(t) == hw) ? 1 : 0);
      a.qn[f] = 0;
    } else {
      a.qn[f] = all ? -1 : nq;   // exact rescoring by k_fft2_rescore
    }
    if (a.qcount) a.qcount[f] = nq;
    a.ub[f] = FFT_UB_INIT;
    a.cnt[f] = 0;
  }
  if (!(nq == 1 && !a.f_out) && !all)
    for (int k = threadIdx.x; k < nq; k += blockDim.x) a.ql[f * FFT_QCAP + k] = qlist[k];
  // re-zero the accumulated energy slots (total, edge columns) for the next call
  if (threadIdx.x == 0) a.ynorm[f] = 0.0;
  u64 *Ew = a.Ew + f * f2_esz2(hw);
  for (int st2 = 0; st2 < 2; ++st2) {
    u64 *e = Ew + st2 * f2_esz(hw);
    if (threadIdx.x == 0) e[0] = 0;
    for (int k = threadIdx.x; k < 2 * hw; k += blockDim.x) e[1 + 2 * hw + k] = 0;
  }
}

// Exact rescoring of the certified candidates (S4): blocks (frame, row part); frames whose
// candidate set k_fft2_score resolved exit at once.  Candidates inside a 3 x 3 box of lags
// (the usual case: the neighbours of the optimum) are scored in one pass over the part's
// rows; others one lag at a time.  Partial N -> 64-bit atomics; the last part of a frame
// takes the argmin of the key (f, s, t) over the exact values and writes the outputs.
template <int L>
__global__ void __launch_bounds__(256) k_fft2_rescore(F2ScoreArgs a) {
  __shared__ u64 red[32];
  __shared__ u64 bred[8][9];
  __shared__ int last, box[4];
  pdl_enter();
  const int64_t f = blockIdx.x / a.rparts;
  const int part = blockIdx.x - (int)(f * a.rparts);
  const int qn = a.qn[f];
  if (qn == 0) return;
  const int W = a.W, hw = a.hw;
  const bool all = qn < 0;
  const int ncand = all ? W * W : qn;
  const int rows = (a.mc + a.rparts - 1) / a.rparts, r0 = part * rows, r1 = min(a.mc, r0 + rows);
  const int *ql = a.ql + f * FFT_QCAP;
  u64 *acc = a.nacc + f * (int64_t)max(FFT_QCAP, W * W);
  if (threadIdx.x == 0) {
    int smin = 1 << 30, smax = -(1 << 30), tmin = 1 << 30, tmax = -(1 << 30);
    for (int c = 0; c < (all ? 0 : ncand); ++c) {
      const int s = ql[c] / W - hw, t = ql[c] % W - hw;
      smin = min(smin, s); smax = max(smax, s); tmin = min(tmin, t); tmax = max(tmax, t);
    }
    box[0] = smin; box[1] = smax - smin + 1; box[2] = tmin; box[3] = tmax - tmin + 1;
  }
  __syncthreads();
  const bool boxed = !all && box[1] <= 3 && box[3] <= 3;
  if (boxed) {
    // slots of the box lags: acc[ds * 3 + dt]; the last block maps candidates to them
    u64 v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = 0;
    f2_exact_box<L>(a, f, box[0], box[1], box[2], box[3], r0, r1, v);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const u64 x = warp_sum(v[k]);
      if (lane == 0) bred[wid][k] = x;
    }
    __syncthreads();
    if (threadIdx.x < 9) {
      u64 x = 0;
      for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) x += bred[w2][threadIdx.x];
      if (x) atomicAdd(acc + threadIdx.x, x);
    }
  } else {
    for (int c = 0; c < ncand; ++c) {
      const int lag = all ? c : ql[c];
      const u64 part_n = f2_exact_N<L>(a, f, lag / W - hw, lag % W - hw, r0, r1, red);
      if (threadIdx.x == 0 && part_n) atomicAdd(acc + c, part_n);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(a.cnt2 + f, 1) == a.rparts - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  Key bk{~0ull, ~0u};
  for (int c = threadIdx.x; c < ncand; c += blockDim.x) {
    const int lag = all ? c : ql[c];
    const int s = lag / W - hw, t = lag % W - hw;
    const int slot = boxed ? (s - box[0]) * 3 + (t - box[2]) : c;
    const u64 N = __ldcg(acc + slot);
    const double area = (double)((a.mc - abs(s)) * (a.nc - abs(t)));
    const Key kk{(u64)__double_as_longlong((double)N / (a.scale * area)), (unsigned)lag};
    if (key_less(kk, bk)) bk = kk;
  }
  __shared__ Key kred[32];
  bk = block_min_key(bk, kred);
  // re-zero the accumulators for the next call
  for (int k = threadIdx.x; k < (boxed ? 9 : ncand); k += blockDim.x) acc[k] = 0;
  if (threadIdx.x == 0) {
    const int s = (int)(bk.idx / W) - hw, t = (int)(bk.idx % W) - hw;
    a.shift_out[2 * f] = s;
    a.shift_out[2 * f + 1] = t;
    if (a.f_out) a.f_out[f] = __longlong_as_double((long long)bk.f);
    if (a.flags) a.flags[f] = (uint8_t)(((abs(s) == hw || abs(t) == hw) ? 1 : 0) | (all ? 2 : 0));
    a.qn[f] = 0;
    a.cnt2[f] = 0;
  }
}

}  // namespace moco
