// kernels_fft.cuh -- S3 by FFT cross-correlation (the paper's method), with a
// certified candidate set and exact rescoring (S4), for MOCO_U16.
//
// The cross term of P:31 for every coarse lag,
//     h(s,t) = sum_{(i,j) in D_{s,t}} a[i+s][j+t] b[i][j],
// is a circular cross-correlation once a and b are zero-padded to Mr x Mc with
// Mr >= m_c + w - 1 and Mc >= n_c + w - 1 (no wrap-around for |s|,|t| <= w-1):
//     H = IFFT2( FFT2(a_pad) . conj(FFT2(b_pad)) ),   h(s,t) = H[s mod Mr][t mod Mc]
// (the paper writes it with the rotated template b^ and pad m+w; the two are
// the same numbers -- pinned in tests/test_oracle_pins.py).  The sizes are products of
// 2, 3, 4, 5 (288 = 4*4*2*3*3 for 256 + 31 or + 63) and every 1-D transform is a
// shared-memory Stockham autosort FFT (natural order in and out, no bit reversal).
//
//   k_fft_rows    two real rows packed as one complex row -> FFT_Mc -> Hermitian halves,
//                 stored column-major per frame: S[f][k][row], k in [0, Mc/2]
//   k_fft_cols    per column bin k: FFT_Mr over rows, times conj(B^)/(Mr Mc), IFFT_Mr,
//                 keep only the 2w-1 lag rows: P[f][s+w-1][k]   (template: store conj(B^))
//   k_fft_score   per frame: two lag rows packed -> IFFT_Mc -> h~(s,t); then the
//                 certified search of S4 (below) and exact rescoring
//
// fp32 certification (S4): with |h~ - h| <= eps_h = u ||a||_2 (Cf ||b||_2 + Ci ||b||_1)
// (u = 2^-24; Cf, Ci derived from the transforms' stage structure), the
// score f~ = (g_a + g_b - 2 h~) / (16^L A) is within delta = 2 eps_h / (16^L A) of the
// exact f.  Every lag whose interval [f~ - delta, f~ + delta] reaches below
// min(f~ + delta) is re-scored EXACTLY (64-bit integer direct sum of P:31) and the argmin
// of the key (f, s, t) is taken over those exact values -- the result is the exact
// method's, bit for bit.  More than FFT_QCAP candidates: every lag is re-scored (flag
// bit 1).  The template spectrum is computed in fp64 (direct separable DFT) and rounded
// once to fp32.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "kernels_direct.cuh"

namespace moco {

// ---------------------------------------------------------------- error bound
// First-order bound on the fp32 cross term, DESIGN.md §5.  A transform is a product of
// stages; a stage whose outputs are computed with |fl(y_k) - y_k| <= rho u sum_j |z_j|
// over its radix-r block has ||fl(Az) - Az||_2 <= mu ||A||_2 ||z||_2 with mu = sqrt(r) rho
// u, and a diagonal twiddle stage (rounded constant, two roundings per component) mu = 3u.
// Summed over the stages (the unnormalised stages multiply to ||F||_2 = sqrt(N)):
//   ||fl(F x) - F x||_2 <= kappa u sqrt(N) ||x||_2.
// rho per butterfly as written (kernels_fft.cuh dft_small / Dft, kernels_fft2.cuh D2):
// radix 2: 1, radix 4 (two add layers, +-i exact): 2, radix 3 (depth 3 and one rounded
// constant): 4, radix 5 (depth 4 and rounded constants): 8.
inline double fft_mu(int r) {
  return r == 2 ? std::sqrt(2.0) * 1 : r == 4 ? 2.0 * 2 : r == 3 ? std::sqrt(3.0) * 4 : std::sqrt(5.0) * 8;
}
// kappa of a codelet of length n (kernels_fft.cuh DftCT splits, innermost radices 2-5)
inline double fft_kappa_codelet(int n) {
  switch (n) {
    case 2: case 3: case 4: case 5: return fft_mu(n);
    case 8: return fft_mu(2) + 3 + fft_mu(4);
    case 9: return fft_mu(3) + 3 + fft_mu(3);
    case 12: return fft_mu(3) + 3 + fft_mu(4);
    case 15: return fft_mu(3) + 3 + fft_mu(5);
    case 16: return fft_mu(4) + 3 + fft_mu(4);
    case 18: return fft_mu(2) + 3 + fft_kappa_codelet(9);
    case 20: return fft_mu(4) + 3 + fft_mu(5);
    default: return 1e30;
  }
}
constexpr int FFT_QCAP = 64;
constexpr int FFT_UB_INIT = 0x7f7f7f7f;   // ~3.4e38f: a.ub between calls
constexpr int FFT_MAXST = 10;

struct FftLen {
  int N, nst;
  int rad[FFT_MAXST];
};

// smallest N >= lo with N = 2^a 3^b 5^c, factored into radices 4, 2, 3, 5
inline bool fft_len_make(int lo, FftLen *L) {
  for (int N = lo; N < 4 * lo + 64; ++N) {
    int x = N, c4 = 0, c2 = 0, c3 = 0, c5 = 0;
    while (x % 4 == 0) { x /= 4; ++c4; }
    while (x % 2 == 0) { x /= 2; ++c2; }
    while (x % 3 == 0) { x /= 3; ++c3; }
    while (x % 5 == 0) { x /= 5; ++c5; }
    if (x != 1 || c4 + c2 + c3 + c5 > FFT_MAXST) continue;
    L->N = N;
    L->nst = 0;
    for (int k = 0; k < c4; ++k) L->rad[L->nst++] = 4;
    for (int k = 0; k < c2; ++k) L->rad[L->nst++] = 2;
    for (int k = 0; k < c3; ++k) L->rad[L->nst++] = 3;
    for (int k = 0; k < c5; ++k) L->rad[L->nst++] = 5;
    return true;
  }
  return false;
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

// In-place R-point DFT, sign -1 (forward) or +1 (inverse).
template <int R>
__device__ __forceinline__ void dft_small(float2 (&v)[5], float sign) {
  if constexpr (R == 2) {
    const float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    const float2 a = cadd(v[0], v[2]), b = csub(v[0], v[2]);
    const float2 c = cadd(v[1], v[3]), d = csub(v[1], v[3]);
    // -i*sign*d for the forward (sign=-1) gives -i d
    const float2 jd = make_float2(-sign * d.y, sign * d.x);   // i*sign*d
    v[0] = cadd(a, c);
    v[2] = csub(a, c);
    v[1] = cadd(b, jd);
    v[3] = csub(b, jd);
  } else if constexpr (R == 3) {
    const float c1 = -0.5f, s1 = sign * 0.86602540378443865f;
    const float2 a = v[0], b = v[1], c = v[2];
    const float2 t = cadd(b, c), u = csub(b, c);
    v[0] = cadd(a, t);
    const float2 m = make_float2(a.x + c1 * t.x, a.y + c1 * t.y);
    const float2 r = make_float2(-s1 * u.y, s1 * u.x);   // i*s1*u
    v[1] = cadd(m, r);
    v[2] = csub(m, r);
  } else {   // R == 5
    const float c1 = 0.30901699437494742f, c2 = -0.80901699437494742f;
    const float s1 = sign * 0.95105651629515357f, s2 = sign * 0.58778525229247313f;
    const float2 a = v[0];
    const float2 t1 = cadd(v[1], v[4]), u1 = csub(v[1], v[4]);
    const float2 t2 = cadd(v[2], v[3]), u2 = csub(v[2], v[3]);
    v[0] = cadd(a, cadd(t1, t2));
    const float2 m1 = make_float2(a.x + c1 * t1.x + c2 * t2.x, a.y + c1 * t1.y + c2 * t2.y);
    const float2 m2 = make_float2(a.x + c2 * t1.x + c1 * t2.x, a.y + c2 * t1.y + c1 * t2.y);
    const float2 r1 = make_float2(-(s1 * u1.y + s2 * u2.y), s1 * u1.x + s2 * u2.x);   // i(s1 u1 + s2 u2)
    const float2 r2 = make_float2(-(s2 * u1.y - s1 * u2.y), s2 * u1.x - s1 * u2.x);   // i(s2 u1 - s1 u2)
    v[1] = cadd(m1, r1);
    v[4] = csub(m1, r1);
    v[2] = cadd(m2, r2);
    v[3] = csub(m2, r2);
  }
}

// q = x / d for x, d < 2^16 via multiply-high by the magic m = floor((2^32 - 1) / d) + 1
__device__ __forceinline__ uint32_t fdiv16(uint32_t x, uint32_t m) { return __umulhi(x, m); }

template <int R>
__device__ __forceinline__ void fft_stage(const float2 *x, float2 *y, const float2 *tw, int N, int Ns, int nfft,
                                          float sign) {
  const int nb = N / R, tstep = N / (Ns * R);
  const uint32_t mnb = 0xffffffffu / (uint32_t)nb + 1u, mns = 0xffffffffu / (uint32_t)Ns + 1u;
  for (int e = threadIdx.x; e < nfft * nb; e += blockDim.x) {
    const int f = (int)fdiv16((uint32_t)e, mnb), j = e - f * nb;
    const float2 *in = x + f * N;
    float2 *out = y + f * N;
    const int jq = Ns == 1 ? j : (int)fdiv16((uint32_t)j, mns);
    const int k = j - jq * Ns;
    float2 v[5];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = in[j + r * nb];
#pragma unroll
    for (int r = 1; r < R; ++r) {
      float2 t = tw[k * r * tstep];   // exp(-2 pi i k r / (Ns R)); k r tstep < N
      if (sign > 0) t.y = -t.y;
      v[r] = cmul(v[r], t);
    }
    dft_small<R>(v, sign);
    const int o = jq * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) out[o + r * Ns] = v[r];
  }
}

// ------------------------------------------------------------ register codelets
// Small DFTs held in registers, natural order in and out,
//   X[k] = sum_n v[n] e^{SIGN 2 pi i n k / N}   (SIGN = -1 forward, +1 inverse),
// N = 2, 3, 4, 5 written out, larger N composed by Cooley-Tukey N = N1 x N2 at compile time
// (n = N2 n1 + n2, k = k1 + N1 k2) with the twiddles e^{SIGN 2 pi i n2 k1 / N} as float
// constants (cos, sin)(2 pi m / N) -- every index is a compile-time constant after
// unrolling, so the tables fold into immediates.
__device__ __forceinline__ float2 mul_i(float2 z, float s) { return make_float2(-s * z.y, s * z.x); }   // (s i) z
template <int SIGN>
__device__ __forceinline__ float2 rot(float2 z, float2 cs) {   // z * e^{SIGN i theta}, cs = (cos, sin) theta
  const float sn = (float)SIGN * cs.y;
  return make_float2(z.x * cs.x - z.y * sn, z.x * sn + z.y * cs.x);
}
template <int N>
__device__ __forceinline__ float2 twk(int m);
template <>
__device__ __forceinline__ float2 twk<8>(int m) {
  constexpr float C[8] = {1.0f, 0.707106781f, 0.0f, -0.707106781f, -1.0f, -0.707106781f, 0.0f, 0.707106781f};
  constexpr float S[8] = {0.0f, 0.707106781f, 1.0f, 0.707106781f, 0.0f, -0.707106781f, -1.0f, -0.707106781f};
  return make_float2(C[m], S[m]);
}
template <>
__device__ __forceinline__ float2 twk<9>(int m) {
  constexpr float C[9] = {1.0f, 0.766044443f, 0.173648178f, -0.5f, -0.939692621f, -0.939692621f, -0.5f, 0.173648178f, 0.766044443f};
  constexpr float S[9] = {0.0f, 0.64278761f, 0.984807753f, 0.866025404f, 0.342020143f, -0.342020143f, -0.866025404f, -0.984807753f, -0.64278761f};
  return make_float2(C[m], S[m]);
}
template <>
__device__ __forceinline__ float2 twk<12>(int m) {
  constexpr float C[12] = {1.0f, 0.866025404f, 0.5f, 0.0f, -0.5f, -0.866025404f, -1.0f, -0.866025404f, -0.5f, 0.0f, 0.5f, 0.866025404f};
  constexpr float S[12] = {0.0f, 0.5f, 0.866025404f, 1.0f, 0.866025404f, 0.5f, 0.0f, -0.5f, -0.866025404f, -1.0f, -0.866025404f, -0.5f};
  return make_float2(C[m], S[m]);
}
template <>
__device__ __forceinline__ float2 twk<15>(int m) {
  constexpr float C[15] = {1.0f, 0.913545458f, 0.669130606f, 0.309016994f, -0.104528463f, -0.5f, -0.809016994f, -0.978147601f, -0.978147601f, -0.809016994f, -0.5f, -0.104528463f, 0.309016994f, 0.669130606f, 0.913545458f};
  constexpr float S[15] = {0.0f, 0.406736643f, 0.743144825f, 0.951056516f, 0.994521895f, 0.866025404f, 0.587785252f, 0.207911691f, -0.207911691f, -0.587785252f, -0.866025404f, -0.994521895f, -0.951056516f, -0.743144825f, -0.406736643f};
  return make_float2(C[m], S[m]);
}
template <>
__device__ __forceinline__ float2 twk<16>(int m) {
  constexpr float C[16] = {1.0f, 0.923879533f, 0.707106781f, 0.382683432f, 0.0f, -0.382683432f, -0.707106781f, -0.923879533f, -1.0f, -0.923879533f, -0.707106781f, -0.382683432f, 0.0f, 0.382683432f, 0.707106781f, 0.923879533f};
  constexpr float S[16] = {0.0f, 0.382683432f, 0.707106781f, 0.923879533f, 1.0f, 0.923879533f, 0.707106781f, 0.382683432f, 0.0f, -0.382683432f, -0.707106781f, -0.923879533f, -1.0f, -0.923879533f, -0.707106781f, -0.382683432f};
  return make_float2(C[m], S[m]);
}
template <>
__device__ __forceinline__ float2 twk<18>(int m) {
  constexpr float C[18] = {1.0f, 0.939692621f, 0.766044443f, 0.5f, 0.173648178f, -0.173648178f, -0.5f, -0.766044443f, -0.939692621f, -1.0f, -0.939692621f, -0.766044443f, -0.5f, -0.173648178f, 0.173648178f, 0.5f, 0.766044443f, 0.939692621f};
  constexpr float S[18] = {0.0f, 0.342020143f, 0.64278761f, 0.866025404f, 0.984807753f, 0.984807753f, 0.866025404f, 0.64278761f, 0.342020143f, 0.0f, -0.342020143f, -0.64278761f, -0.866025404f, -0.984807753f, -0.984807753f, -0.866025404f, -0.64278761f, -0.342020143f};
  return make_float2(C[m], S[m]);
}
template <>
__device__ __forceinline__ float2 twk<20>(int m) {
  constexpr float C[20] = {1.0f, 0.951056516f, 0.809016994f, 0.587785252f, 0.309016994f, 0.0f, -0.309016994f, -0.587785252f, -0.809016994f, -0.951056516f, -1.0f, -0.951056516f, -0.809016994f, -0.587785252f, -0.309016994f, 0.0f, 0.309016994f, 0.587785252f, 0.809016994f, 0.951056516f};
  constexpr float S[20] = {0.0f, 0.309016994f, 0.587785252f, 0.809016994f, 0.951056516f, 1.0f, 0.951056516f, 0.809016994f, 0.587785252f, 0.309016994f, 0.0f, -0.309016994f, -0.587785252f, -0.809016994f, -0.951056516f, -1.0f, -0.951056516f, -0.809016994f, -0.587785252f, -0.309016994f};
  return make_float2(C[m], S[m]);
}

template <int N, int SIGN>
struct Dft;
template <int SIGN>
struct Dft<2, SIGN> {
  static __device__ __forceinline__ void run(float2 (&v)[2]) {
    const float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};
template <int SIGN>
struct Dft<3, SIGN> {
  static __device__ __forceinline__ void run(float2 (&v)[3]) {
    const float s1 = (float)SIGN * 0.86602540378443865f;
    const float2 t = cadd(v[1], v[2]), u = csub(v[1], v[2]);
    const float2 m = make_float2(v[0].x - 0.5f * t.x, v[0].y - 0.5f * t.y);
    const float2 r = mul_i(u, s1);
    v[0] = cadd(v[0], t);
    v[1] = cadd(m, r);
    v[2] = csub(m, r);
  }
};
template <int SIGN>
struct Dft<4, SIGN> {
  static __device__ __forceinline__ void run(float2 (&v)[4]) {
    const float2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]), t2 = cadd(v[1], v[3]);
    const float2 t3 = mul_i(csub(v[1], v[3]), (float)SIGN);
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  }
};
template <int SIGN>
struct Dft<5, SIGN> {
  static __device__ __forceinline__ void run(float2 (&v)[5]) {
    const float c1 = 0.30901699437494742f, c2 = -0.80901699437494742f;
    const float s1 = (float)SIGN * 0.95105651629515357f, s2 = (float)SIGN * 0.58778525229247313f;
    const float2 a = v[0];
    const float2 t1 = cadd(v[1], v[4]), u1 = csub(v[1], v[4]);
    const float2 t2 = cadd(v[2], v[3]), u2 = csub(v[2], v[3]);
    v[0] = cadd(a, cadd(t1, t2));
    const float2 m1 = make_float2(a.x + c1 * t1.x + c2 * t2.x, a.y + c1 * t1.y + c2 * t2.y);
    const float2 m2 = make_float2(a.x + c2 * t1.x + c1 * t2.x, a.y + c2 * t1.y + c1 * t2.y);
    const float2 r1 = make_float2(-(s1 * u1.y + s2 * u2.y), s1 * u1.x + s2 * u2.x);   // i (s1 u1 + s2 u2)
    const float2 r2 = make_float2(-(s2 * u1.y - s1 * u2.y), s2 * u1.x - s1 * u2.x);   // i (s2 u1 - s1 u2)
    v[1] = cadd(m1, r1);
    v[4] = csub(m1, r1);
    v[2] = cadd(m2, r2);
    v[3] = csub(m2, r2);
  }
};
template <int N1, int N2, int SIGN>
struct DftCT {
  static __device__ __forceinline__ void run(float2 (&v)[N1 * N2]) {
    constexpr int N = N1 * N2;
    float2 t[N1][N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) {
      float2 u[N1];
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) u[n1] = v[N2 * n1 + n2];
      Dft<N1, SIGN>::run(u);
#pragma unroll
      for (int k1 = 0; k1 < N1; ++k1) t[k1][n2] = (n2 * k1 == 0) ? u[k1] : rot<SIGN>(u[k1], twk<N>((n2 * k1) % N));
    }
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) {
      Dft<N2, SIGN>::run(t[k1]);
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) v[k1 + N1 * k2] = t[k1][k2];
    }
  }
};
template <int SIGN> struct Dft<8, SIGN> : DftCT<2, 4, SIGN> {};
template <int SIGN> struct Dft<9, SIGN> : DftCT<3, 3, SIGN> {};
template <int SIGN> struct Dft<12, SIGN> : DftCT<3, 4, SIGN> {};
template <int SIGN> struct Dft<15, SIGN> : DftCT<3, 5, SIGN> {};
template <int SIGN> struct Dft<16, SIGN> : DftCT<4, 4, SIGN> {};
template <int SIGN> struct Dft<18, SIGN> : DftCT<2, 9, SIGN> {};
template <int SIGN> struct Dft<20, SIGN> : DftCT<4, 5, SIGN> {};

// nfft transforms of length N = N1 x N2 in two register passes: pass 1, one thread per
// (transform, n2): radix-N1 over n1 of x[N2 n1 + n2], times e^{SIGN 2 pi i n2 k1 / N} (the
// smem table tw[m] = e^{-2 pi i m / N}), into y at n2 + RP k1 (rows padded to RP elements so
// that pass 2 reads are bank-conflict free); pass 2, one thread per (transform, k1):
// radix-N2 over n2 -> X[k1 + N1 k2] back into x in natural order.  y holds nfft*(N+FFT_YPAD).
constexpr int FFT_YPAD = 40;
template <int N1, int N2, int SIGN>
__device__ void fft2p(float2 *x, float2 *y, const float2 *tw, int nfft) {
  constexpr int N = N1 * N2, RP = (N2 & 1) ? N2 + 2 : N2 + 1, YS = N + FFT_YPAD;
  static_assert(N1 * RP <= YS, "scratch row padding");
  for (int task = threadIdx.x; task < nfft * N2; task += blockDim.x) {
    const int q = task / N2, n2 = task - q * N2;
    const float2 *in = x + q * N + n2;
    float2 v[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) v[n1] = in[N2 * n1];
    Dft<N1, SIGN>::run(v);
    float2 *out = y + q * YS + n2;
    out[0] = v[0];
#pragma unroll
    for (int k1 = 1; k1 < N1; ++k1) {
      float2 t = tw[n2 * k1];   // n2 k1 <= (N2-1)(N1-1) < N
      if (SIGN > 0) t.y = -t.y;
      out[RP * k1] = cmul(v[k1], t);
    }
  }
  __syncthreads();
  for (int task = threadIdx.x; task < nfft * N1; task += blockDim.x) {
    const int q = task / N1, k1 = task - q * N1;
    const float2 *in = y + q * YS + RP * k1;
    float2 u[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) u[n2] = in[n2];
    Dft<N2, SIGN>::run(u);
    float2 *out = x + q * N + k1;
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) out[N1 * k2] = u[k2];
  }
  __syncthreads();
}
// The lengths with a two-pass register plan, P -> (N1, N2), N1 N2 = N (P = 0: the generic
// shared-memory Stockham passes).  Each kernel that transforms is instantiated per plan,
// so a kernel carries the code of one plan only (all of them inlined together thrashed
// the instruction cache: 288-point rows 363 -> 435 us).
constexpr int FFT_NPLAN = 7;
__host__ __device__ constexpr int fft_plan_of(int N) {
  return N == 288 ? 1 : N == 360 ? 2 : N == 300 ? 3 : N == 320 ? 4 : N == 240 ? 5 : N == 256 ? 6 : 0;
}
template <int P> struct Plan2p { static constexpr int N1 = 1, N2 = 1; };
template <> struct Plan2p<1> { static constexpr int N1 = 16, N2 = 18; };
template <> struct Plan2p<2> { static constexpr int N1 = 20, N2 = 18; };
template <> struct Plan2p<3> { static constexpr int N1 = 20, N2 = 15; };
template <> struct Plan2p<4> { static constexpr int N1 = 16, N2 = 20; };
template <> struct Plan2p<5> { static constexpr int N1 = 16, N2 = 15; };
template <> struct Plan2p<6> { static constexpr int N1 = 16, N2 = 16; };

// nfft transforms of length L.N stored contiguously in x; y is scratch of the same
// size.  Returns the buffer holding the result.  All threads of the block take part.
template <int P>
__device__ float2 *fft_batch(float2 *x, float2 *y, const float2 *tw, const FftLen &L, int nfft, float sign) {
  if constexpr (P > 0) {   // register two-pass plan (x in, x out; y holds nfft * (N + FFT_YPAD))
    if (sign < 0) fft2p<Plan2p<P>::N1, Plan2p<P>::N2, -1>(x, y, tw, nfft);
    else fft2p<Plan2p<P>::N1, Plan2p<P>::N2, 1>(x, y, tw, nfft);
    return x;
  }
  int Ns = 1;
  for (int st = 0; st < L.nst; ++st) {
    const int R = L.rad[st];
    switch (R) {
      case 2: fft_stage<2>(x, y, tw, L.N, Ns, nfft, sign); break;
      case 3: fft_stage<3>(x, y, tw, L.N, Ns, nfft, sign); break;
      case 4: fft_stage<4>(x, y, tw, L.N, Ns, nfft, sign); break;
      default: fft_stage<5>(x, y, tw, L.N, Ns, nfft, sign); break;
    }
    __syncthreads();
    float2 *t = x; x = y; y = t;
    Ns *= R;
  }
  return x;
}

// twiddles exp(-2 pi i k / N), k < N, computed in double
__global__ void k_fft_twiddles(float2 *tw, int N) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
    double s, c;
    sincospi(-2.0 * k / N, &s, &c);
    tw[k] = make_float2((float)c, (float)s);
  }
}

// Template spectrum in fp64 (once per template), separable direct DFT:
//   R[i][k] = sum_j b[i][j] e^{-2 pi i j k / Mc}                (k < Kc)
//   Bc[k][u] = conj(sum_i R[i][k] e^{-2 pi i i u / Mr}) / (Mr Mc), rounded once to fp32
// twiddles by sincospi in double; |rounding error| ~ 1e-16 relative to ||b||_1, far
// below the fp32 rounding of the result.
// Template statistics for the mean-removed FFT path (kernels_fft2.cuh): with `mean` set,
// mu = round(sum b / (mc nc)) (else 0), then ||b - mu||_1 and ||b - mu||_2^2 over the
// template's support.  st[0] = mu, st[1] = ||b'||_1, st[2] = ||b'||_2^2.  One block.
__global__ void k_tpl_stats(const uint16_t *__restrict__ b, int pitch, int mc, int nc, int mean,
                            long long *__restrict__ st) {
  __shared__ unsigned long long red[32];
  __shared__ long long mu_s;
  unsigned long long acc = 0;
  for (int e = threadIdx.x; e < mc * nc; e += blockDim.x) acc += b[(int64_t)(e / nc) * pitch + e % nc];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
    const unsigned long long n = (unsigned long long)mc * nc;
    mu_s = mean ? (long long)((t + n / 2) / n) : 0;
  }
  __syncthreads();
  // mean 1: both sides shifted by mu (b' = b - mu); mean 2: the frames only (b' = b)
  const long long mu = mean == 1 ? mu_s : 0;
  unsigned long long a1 = 0, a2 = 0;
  for (int e = threadIdx.x; e < mc * nc; e += blockDim.x) {
    const long long d = (long long)b[(int64_t)(e / nc) * pitch + e % nc] - mu;
    a1 += (unsigned long long)(d < 0 ? -d : d);
    a2 += (unsigned long long)(d * d);
  }
  for (int o = 16; o > 0; o >>= 1) {
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  __syncthreads();
  __shared__ unsigned long long r1[32], r2[32];
  if ((threadIdx.x & 31) == 0) { r1[threadIdx.x >> 5] = a1; r2[threadIdx.x >> 5] = a2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t1 = 0, t2 = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { t1 += r1[k]; t2 += r2[k]; }
    st[0] = mu_s;   // the frames' shift
    st[1] = (long long)t1;
    st[2] = (long long)t2;
    st[3] = mu;     // the template's shift
  }
}
__global__ void k_tpl_dft_rows(const uint16_t *__restrict__ b, int pitch, int nc, int Mc, int Kc,
                               double2 *__restrict__ R, const long long *__restrict__ mu) {
  extern __shared__ double2 tw64[];
  for (int m = threadIdx.x; m < Mc; m += blockDim.x) {
    double s_, c_;
    sincospi(-2.0 * m / Mc, &s_, &c_);
    tw64[m] = make_double2(c_, s_);
  }
  __syncthreads();
  const int i = blockIdx.x;
  double *row = reinterpret_cast<double *>(tw64 + Mc);   // the template row (minus mu), staged once
  const double m0 = mu ? (double)mu[3] : 0.0;   // k_tpl_stats: the template's shift
  for (int j = threadIdx.x; j < nc; j += blockDim.x) row[j] = (double)b[(int64_t)i * pitch + j] - m0;
  __syncthreads();
  for (int k = threadIdx.x; k < Kc; k += blockDim.x) {
    double re = 0, im = 0;
    int m = 0;
    for (int j = 0; j < nc; ++j) {
      const double v = row[j];
      re += v * tw64[m].x;
      im += v * tw64[m].y;
      m += k;
      if (m >= Mc) m -= Mc;
    }
    R[(int64_t)i * Kc + k] = make_double2(re, im);
  }
}
__global__ void k_tpl_dft_cols(const double2 *__restrict__ R, int mc, int Mr, int Mc, int Kc, float2 *__restrict__ Bc,
                               unsigned long long *__restrict__ b1, const uint16_t *__restrict__ b, int pitch, int nc) {
  extern __shared__ double2 tw64[];
  for (int m = threadIdx.x; m < Mr; m += blockDim.x) {
    double s_, c_;
    sincospi(-2.0 * m / Mr, &s_, &c_);
    tw64[m] = make_double2(c_, s_);
  }
  __syncthreads();
  const int k = blockIdx.x;
  double2 *col = tw64 + Mr;   // the column R[.][k], staged once
  for (int i = threadIdx.x; i < mc; i += blockDim.x) col[i] = R[(int64_t)i * Kc + k];
  __syncthreads();
  const double scale = 1.0 / ((double)Mr * (double)Mc);
  for (int u = threadIdx.x; u < Mr; u += blockDim.x) {
    double re = 0, im = 0;
    int m = 0;
    for (int i = 0; i < mc; ++i) {
      const double2 r = col[i];
      const double2 t = tw64[m];
      re += r.x * t.x - r.y * t.y;
      im += r.x * t.y + r.y * t.x;
      m += u;
      if (m >= Mr) m -= Mr;
    }
    Bc[(int64_t)k * Mr + u] = make_float2((float)(re * scale), (float)(-im * scale));
  }
  if (k == 0 && b1) {   // ||b||_1 of the coarse template (non-negative samples): sum b
    unsigned long long acc = 0;
    for (int e = threadIdx.x; e < mc * nc; e += blockDim.x) acc += b[(int64_t)(e / nc) * pitch + e % nc];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(b1, acc);
  }
}

struct FftGeom {
  int mc, nc, w, hw, W;
  FftLen Lr, Lc;   // column length Mr (over rows), row length Mc (over columns)
  int Kc;          // Mc/2 + 1 column bins kept
  int mcp;         // rows stored per column of S (mc rounded up to even)
};

constexpr int FFT_ROWS_PAIRS = 8;   // row pairs per k_fft_rows block
constexpr int FFT_COLS = 8;         // column bins per k_fft_cols block
constexpr int FFT_THREADS = 256;

// ---------------------------------------------------------------- forward rows
// S[f][k][r] = sum_j a_f[r][j] exp(-2 pi i j k / Mc), k in [0, Kc), r in [0, mcp)
template <int P>
__global__ void __launch_bounds__(FFT_THREADS) k_fft_rows(const uint16_t *__restrict__ img, int64_t fstride,
                                                          int pitch, FftGeom g, const float2 *__restrict__ twc,
                                                          float2 *__restrict__ S, int per) {
  extern __shared__ __align__(16) float2 fsm[];
  const int Mc = g.Lc.N;
  float2 *tw = fsm;
  float2 *x = tw + Mc, *y = x + FFT_ROWS_PAIRS * Mc;   // y: FFT_ROWS_PAIRS * (Mc + FFT_YPAD)
  const int nrb = (g.mcp / 2 + per - 1) / per;   // per <= FFT_ROWS_PAIRS row pairs per block
  const int f = blockIdx.x / nrb, rb = blockIdx.x % nrb;
  const int p0 = rb * per, np = min(per, g.mcp / 2 - p0);
  for (int k = threadIdx.x; k < Mc; k += blockDim.x) tw[k] = twc[k];
  const uint16_t *A = img + (int64_t)f * fstride;
  for (int e = threadIdx.x; e < np * Mc; e += blockDim.x) {
    const int q = e / Mc, j = e - q * Mc;
    const int r0 = 2 * (p0 + q), r1 = r0 + 1;
    float re = 0.f, im = 0.f;
    if (j < g.nc) {
      if (r0 < g.mc) re = (float)A[(int64_t)r0 * pitch + j];
      if (r1 < g.mc) im = (float)A[(int64_t)r1 * pitch + j];
    }
    x[q * Mc + j] = make_float2(re, im);
  }
  __syncthreads();
  const float2 *Z = fft_batch<P>(x, y, tw, g.Lc, np, -1.f);
  // unpack the two real rows' spectra; store column-major S[f][k][row]
  float2 *Sf = S + (int64_t)f * g.Kc * g.mcp;
  for (int e = threadIdx.x; e < g.Kc * np; e += blockDim.x) {
    const int k = e / np, q = e - k * np;
    const float2 zk = Z[q * Mc + k], zn = conjf2(Z[q * Mc + (Mc - k) % Mc]);
    const float2 x0 = make_float2(0.5f * (zk.x + zn.x), 0.5f * (zk.y + zn.y));
    const float2 d = make_float2(0.5f * (zk.x - zn.x), 0.5f * (zk.y - zn.y));
    const float2 x1 = make_float2(d.y, -d.x);   // d / i
    float2 *dst = Sf + (int64_t)k * g.mcp + 2 * (p0 + q);
    dst[0] = x0;
    dst[1] = x1;
  }
}

// ---------------------------------------------------------------- columns
// mode 0 (frames): P[f][s+hw][k] = (1/(Mr Mc)) sum_u X[u][k] Bc[k][u] e^{+2 pi i u s / Mr}
//                  for s in [-hw, hw], X = FFT over rows of S[f][k][*]
// mode 1 (template): Bc[k][u] = conj(X[u][k]) / (Mr Mc)
template <int PL>
__global__ void __launch_bounds__(FFT_THREADS) k_fft_cols(const float2 *__restrict__ S, FftGeom g,
                                                          const float2 *__restrict__ twr, float2 *__restrict__ Bc,
                                                          float2 *__restrict__ P, int mode, int per) {
  extern __shared__ __align__(16) float2 fsm[];
  const int Mr = g.Lr.N;
  float2 *tw = fsm;
  float2 *x = tw + Mr, *y = x + FFT_COLS * Mr;
  const int ncb = (g.Kc + per - 1) / per;   // per <= FFT_COLS column bins per block
  const int f = blockIdx.x / ncb, cb = blockIdx.x % ncb;
  const int k0 = cb * per, nk = min(per, g.Kc - k0);
  for (int k = threadIdx.x; k < Mr; k += blockDim.x) tw[k] = twr[k];
  const float2 *Sf = S + (int64_t)f * g.Kc * g.mcp;
  for (int e = threadIdx.x; e < nk * Mr; e += blockDim.x) {
    const int q = e / Mr, u = e - q * Mr;
    x[q * Mr + u] = u < g.mc ? Sf[(int64_t)(k0 + q) * g.mcp + u] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  float2 *X = fft_batch<PL>(x, y, tw, g.Lr, nk, -1.f);
  const float scale = 1.0f / ((float)Mr * (float)g.Lc.N);
  if (mode == 1) {
    for (int e = threadIdx.x; e < nk * Mr; e += blockDim.x) {
      const int q = e / Mr, u = e - q * Mr;
      const float2 v = X[q * Mr + u];
      Bc[(int64_t)(k0 + q) * Mr + u] = make_float2(v.x * scale, -v.y * scale);
    }
    return;
  }
  for (int e = threadIdx.x; e < nk * Mr; e += blockDim.x) {
    const int q = e / Mr, u = e - q * Mr;
    X[q * Mr + u] = cmul(X[q * Mr + u], Bc[(int64_t)(k0 + q) * Mr + u]);
  }
  __syncthreads();
  float2 *other = X == x ? y : x;
  const float2 *Hc = fft_batch<PL>(X, other, tw, g.Lr, nk, +1.f);
  float2 *Pf = P + (int64_t)f * g.W * g.Kc;
  for (int e = threadIdx.x; e < g.W * nk; e += blockDim.x) {
    const int si = e / nk, q = e - si * nk;
    const int u = (si - g.hw + Mr) % Mr;
    Pf[(int64_t)si * g.Kc + k0 + q] = Hc[q * Mr + u];
  }
}

// ---------------------------------------------------------------- score + certify
struct FftScoreArgs {
  const float2 *P;          // [B][W][Kc]
  const float2 *twc;        // [Mc]
  const uint16_t *img;      // coarse frames (exact rescoring)
  int64_t fstride;
  int pitch;
  const uint16_t *tpl;      // coarse template
  int tpitch;
  const u64 *ga;            // [B][W*W]
  const u64 *gb;            // [W*W]
  FftGeom g;
  double scale;             // 16^L
  double eps_f, eps_i;      // Cf u, Ci u: eps_h = ||a||_2 (eps_f ||b||_2 + eps_i ||b||_1)
  const unsigned long long *b1;   // ||b||_1 of the coarse template (device)
  int B;
  int32_t *shift_out;       // [B][2]
  double *f_out;            // [B] or null
  uint8_t *flags;           // [B] or null
  int *qcount;              // [B] or null: candidates re-scored (diagnostics)
  float *h_out;             // [B][W*W] or null: the fp32 FFT cross term h~ (diagnostics)
  float *lb;                // [B][W*W] lower bounds f~ - delta (split, small-batch path)
  int *ub;                  // [B] min(f~ + delta) as float bits, kept at +inf between calls
};

// exact h(s,t) for one lag, 64-bit, all threads of the block; result to thread 0
__device__ u64 exact_h(const FftScoreArgs &a, const uint16_t *A, int s, int t, u64 *red) {
  const int mc = a.g.mc, nc = a.g.nc;
  const int i0 = max(0, -s), i1 = mc - max(0, s), j0 = max(0, -t), j1 = nc - max(0, t);
  // warps over rows, lanes over columns (coalesced), four independent rows in flight
  const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  u64 acc = 0;
  for (int i = i0 + wid; i < i1; i += 4 * nw) {
    const uint16_t *ar[4], *br[4];
    bool ok[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int ii = i + q * nw;
      ok[q] = ii < i1;
      ar[q] = A + (int64_t)((ok[q] ? ii : i) + s) * a.pitch + t;
      br[q] = a.tpl + (int64_t)(ok[q] ? ii : i) * a.tpitch;
    }
    for (int j = j0 + lane; j < j1; j += 32) {
#pragma unroll
      for (int q = 0; q < 4; ++q)   // products < 2^32 (coarse values < 2^16), sums in 64 bits
        if (ok[q]) acc += (u64)((uint32_t)ar[q][j] * br[q][j]);
    }
  }
  acc = warp_sum(acc);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  u64 tot = 0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) tot += red[k];
  return tot;
}

// Candidate set Q = {lag : lower bound <= thr} (lower bounds in lbs, shared or global),
// exact 64-bit rescoring of Q (all lags past FFT_QCAP), argmin key (f, s, t) (S4).
// qn_s must be zero on entry (set before the block barrier that precedes the call).
__device__ __forceinline__ void fft_pick_tail(const FftScoreArgs &a, int64_t f, const float *lbs, float thr, u64 *red,
                                              int *qn_s, int *qlist) {
  const FftGeom &g = a.g;
  const int W = g.W, hw = g.hw;
  const u64 *gaf = a.ga + f * W * W;
  for (int lag = threadIdx.x; lag < W * W; lag += blockDim.x) {
    if (lbs[lag] <= thr) {
      const int q = atomicAdd(qn_s, 1);
      if (q < FFT_QCAP) qlist[q] = lag;
    }
  }
  __syncthreads();
  const int nq = *qn_s;
  const bool all = nq > FFT_QCAP;
  const int ncand = all ? W * W : nq;
  const uint16_t *A = a.img + f * a.fstride;
  Key bk{~0ull, ~0u};
  for (int c = 0; c < ncand; ++c) {
    const int lag = all ? c : qlist[c];
    const int s = lag / W - hw, t = lag % W - hw;
    const u64 h = exact_h(a, A, s, t, red);
    if (threadIdx.x == 0) {
      const u64 N = gaf[lag] + a.gb[lag] - 2 * h;
      const double area = (double)((g.mc - abs(s)) * (g.nc - abs(t)));
      const double fv = (double)N / (a.scale * area);
      const Key kk{(u64)__double_as_longlong(fv), (unsigned)lag};
      if (key_less(kk, bk)) bk = kk;
    }
  }
  if (threadIdx.x == 0) {
    const int s = (int)(bk.idx / W) - hw, t = (int)(bk.idx % W) - hw;
    a.shift_out[2 * f] = s;
    a.shift_out[2 * f + 1] = t;
    if (a.f_out) a.f_out[f] = __longlong_as_double((long long)bk.f);
    if (a.flags) a.flags[f] = (uint8_t)(((abs(s) == hw || abs(t) == hw) ? 1 : 0) | (all ? 2 : 0));
    if (a.qcount) a.qcount[f] = nq;
  }
}

template <int P>
__global__ void __launch_bounds__(1024) k_fft_score(FftScoreArgs a) {
  extern __shared__ __align__(16) float2 fsm[];
  const FftGeom &g = a.g;
  const int Mc = g.Lc.N, W = g.W, hw = g.hw;
  float2 *tw = fsm;
  float2 *x = tw + Mc, *y = x + FFT_ROWS_PAIRS * Mc;
  float *hb = reinterpret_cast<float *>(y + FFT_ROWS_PAIRS * (Mc + FFT_YPAD));   // [W][W] h~
  __shared__ u64 red[32];
  __shared__ float fmin_hi_s;
  __shared__ int qn;
  __shared__ int qlist[FFT_QCAP];
  const int64_t f = blockIdx.x;
  for (int k = threadIdx.x; k < Mc; k += blockDim.x) tw[k] = a.twc[k];
  const float2 *Pf = a.P + f * W * g.Kc;
  const int npairs = (W + 1) / 2;
  for (int p0 = 0; p0 < npairs; p0 += FFT_ROWS_PAIRS) {
    const int np = min(FFT_ROWS_PAIRS, npairs - p0);
    __syncthreads();
    for (int e = threadIdx.x; e < np * Mc; e += blockDim.x) {
      const int q = e / Mc, k = e - q * Mc;
      const int s1 = 2 * (p0 + q), s2 = s1 + 1;
      // Hermitian extension of each lag row's half spectrum, packed as re + i*im
      const bool lo = k < g.Kc;
      const int kk = lo ? k : Mc - k;
      float2 v1 = Pf[(int64_t)s1 * g.Kc + kk];
      float2 v2 = s2 < W ? Pf[(int64_t)s2 * g.Kc + kk] : make_float2(0.f, 0.f);
      if (!lo) { v1.y = -v1.y; v2.y = -v2.y; }
      x[q * Mc + k] = make_float2(v1.x - v2.y, v1.y + v2.x);
    }
    __syncthreads();
    const float2 *Hr = fft_batch<P>(x, y, tw, g.Lc, np, +1.f);
    for (int e = threadIdx.x; e < np * W; e += blockDim.x) {
      const int q = e / W, ti = e - q * W;
      const int s1 = 2 * (p0 + q), s2 = s1 + 1;
      const float2 v = Hr[q * Mc + (ti - hw + Mc) % Mc];
      hb[s1 * W + ti] = v.x;
      if (s2 < W) hb[s2 * W + ti] = v.y;
    }
  }
  __syncthreads();
  if (a.h_out)
    for (int lag = threadIdx.x; lag < W * W; lag += blockDim.x) a.h_out[f * W * W + lag] = hb[lag];
  // scores with certified error intervals.  1/(16^L A) = rinv[s] * cinv[t]; pass 1 takes
  // min(f~ + delta) and leaves the lower bound f~ - delta of every lag in hb for pass 2
  double *rinv = reinterpret_cast<double *>(hb + ((W * W + 1) & ~1));   // [W]
  double *cinv = rinv + W;                                              // [W]
  for (int k = threadIdx.x; k < W; k += blockDim.x) {
    rinv[k] = 1.0 / (a.scale * (double)(g.mc - abs(k - hw)));
    cinv[k] = 1.0 / (double)(g.nc - abs(k - hw));
  }
  __syncthreads();
  const u64 *gaf = a.ga + f * W * W;
  const double na = sqrt((double)gaf[hw * W + hw]) * (1.0 + 1e-12);
  const double eps2 = 2.0 * na * (a.eps_f * sqrt((double)a.gb[hw * W + hw]) * (1.0 + 1e-12) + a.eps_i * (double)*a.b1);
  float best = 3.0e38f;
  for (int lag = threadIdx.x; lag < W * W; lag += blockDim.x) {
    const int si = lag / W, ti = lag - si * W;
    const double inv = rinv[si] * cinv[ti];
    const double fa = ((double)gaf[lag] + (double)a.gb[lag] - 2.0 * (double)hb[lag]) * inv;
    const double del = eps2 * inv;
    best = fminf(best, (float)(fa + del) * (1.0f + 1e-6f));
    hb[lag] = (float)(fa - del) * (1.0f - 1e-6f);
  }
  for (int o = 16; o > 0; o >>= 1) best = fminf(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) reinterpret_cast<float *>(red)[threadIdx.x >> 5] = best;
  if (threadIdx.x == 0) qn = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = 3.0e38f;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) b = fminf(b, reinterpret_cast<float *>(red)[k]);
    fmin_hi_s = b;
  }
  __syncthreads();
  fft_pick_tail(a, f, hb, fmin_hi_s, red, &qn, qlist);
}

// Small batches (the closed-loop case): the score step spread over many blocks.
// k_fft_score_rows: block (frame f, group of FFT_ROWS_PAIRS lag-row pairs) -> inverse FFT
// of its lag rows and the certified interval of each of its lags (same arithmetic as
// k_fft_score): lower bound to a.lb, min of the upper bounds by atomicMin into a.ub[f]
// (non-negative floats order like their bit patterns).
template <int P>
__global__ void __launch_bounds__(FFT_THREADS) k_fft_score_rows(FftScoreArgs a, int per) {
  extern __shared__ __align__(16) float2 fsm[];
  const FftGeom &g = a.g;
  const int Mc = g.Lc.N, W = g.W, hw = g.hw;
  float2 *tw = fsm;
  float2 *x = tw + Mc, *y = x + FFT_ROWS_PAIRS * Mc;
  __shared__ float redf[FFT_THREADS / 32];
  const int npairs = (W + 1) / 2, npb = (npairs + per - 1) / per;
  const int64_t f = blockIdx.x / npb;
  const int p0 = (blockIdx.x % npb) * per, np = min(per, npairs - p0);
  for (int k = threadIdx.x; k < Mc; k += blockDim.x) tw[k] = a.twc[k];
  const float2 *Pf = a.P + f * W * g.Kc;
  for (int e = threadIdx.x; e < np * Mc; e += blockDim.x) {
    const int q = e / Mc, k = e - q * Mc;
    const int s1 = 2 * (p0 + q), s2 = s1 + 1;
    const bool lo = k < g.Kc;
    const int kk = lo ? k : Mc - k;
    float2 v1 = Pf[(int64_t)s1 * g.Kc + kk];
    float2 v2 = s2 < W ? Pf[(int64_t)s2 * g.Kc + kk] : make_float2(0.f, 0.f);
    if (!lo) { v1.y = -v1.y; v2.y = -v2.y; }
    x[q * Mc + k] = make_float2(v1.x - v2.y, v1.y + v2.x);
  }
  __syncthreads();
  const float2 *Hr = fft_batch<P>(x, y, tw, g.Lc, np, +1.f);
  const u64 *gaf = a.ga + f * W * W;
  const double na = sqrt((double)gaf[hw * W + hw]) * (1.0 + 1e-12);
  const double eps2 = 2.0 * na * (a.eps_f * sqrt((double)a.gb[hw * W + hw]) * (1.0 + 1e-12) + a.eps_i * (double)*a.b1);
  float best = 3.0e38f;
  for (int e = threadIdx.x; e < np * 2 * W; e += blockDim.x) {
    const int q = e / (2 * W), r = e - q * 2 * W, half = r / W, ti = r - half * W;
    const int si = 2 * (p0 + q) + half;
    if (si >= W) continue;
    const float2 v = Hr[q * Mc + (ti - hw + Mc) % Mc];
    const float h = half ? v.y : v.x;
    const int lag = si * W + ti;
    if (a.h_out) a.h_out[f * W * W + lag] = h;
    const double inv = (1.0 / (a.scale * (double)(g.mc - abs(si - hw)))) * (1.0 / (double)(g.nc - abs(ti - hw)));
    const double fa = ((double)gaf[lag] + (double)a.gb[lag] - 2.0 * (double)h) * inv;
    const double del = eps2 * inv;
    best = fminf(best, (float)(fa + del) * (1.0f + 1e-6f));
    a.lb[f * W * W + lag] = (float)(fa - del) * (1.0f - 1e-6f);
  }
  for (int o = 16; o > 0; o >>= 1) best = fminf(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) redf[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = 3.0e38f;
    for (int k = 0; k < FFT_THREADS / 32; ++k) b = fminf(b, redf[k]);
    atomicMin(a.ub + f, __float_as_int(fmaxf(b, 0.f)));
  }
}

// k_fft_score_pick: one block per frame: Q from the lower bounds, exact rescoring, argmin;
// a.ub[f] is put back to "+inf" for the next call.
__global__ void __launch_bounds__(1024) k_fft_score_pick(FftScoreArgs a) {
  __shared__ u64 red[32];
  __shared__ int qn;
  __shared__ int qlist[FFT_QCAP];
  const int64_t f = blockIdx.x;
  const float thr = __int_as_float(a.ub[f]);
  if (threadIdx.x == 0) qn = 0;
  __syncthreads();
  fft_pick_tail(a, f, a.lb + f * a.g.W * a.g.W, thr, red, &qn, qlist);
  if (threadIdx.x == 0) a.ub[f] = FFT_UB_INIT;
}

// ---------------------------------------------------------------- frame energies
// g_a(s,t) = sum over the frame-side rectangle of D_{s,t} of a^2 for every coarse lag
// (P:32-35): total minus the excluded edge strips plus the doubly excluded corner --
// the paper's DP of P:35 run in each corner (a (w x w) prefix table per corner, built
// one quadrant at a time so any w fits in shared memory).  One block per frame.
// Small batches: the row pass of k_energy_u16 split over blocks (frame f, row band),
// partial sums into a per-frame scratch [4 hw + 1] (row edges stored, column edges and
// the total added atomically); k_energy_fin then does the rest per frame and clears it.
__global__ void __launch_bounds__(256) k_energy_rows(const uint16_t *__restrict__ img, int64_t fstride, int pitch,
                                                     int mc, int nc, int w, int rpb, u64 *__restrict__ scr) {
  const int hw = w - 1;
  const int nb = (mc + rpb - 1) / rpb;
  const int64_t f = blockIdx.x / nb;
  const int r0 = (blockIdx.x % nb) * rpb, r1 = min(mc, r0 + rpb);
  u64 *rowE = scr + f * (4 * hw + 1), *colE = rowE + 2 * hw, *tot = colE + 2 * hw;
  const uint16_t *A = img + f * fstride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  u64 mytot = 0;
  for (int r = r0 + warp; r < r1; r += nwarp) {
    u64 rs = 0;
    const uint16_t *row = A + (int64_t)r * pitch;
#pragma unroll 4
    for (int c = lane; c < nc; c += 32) {
      const u64 v2 = (u64)row[c] * row[c];
      rs += v2;
      if (c < hw) atomicAdd(reinterpret_cast<unsigned long long *>(&colE[c]), (unsigned long long)v2);
      if (c >= nc - hw)
        atomicAdd(reinterpret_cast<unsigned long long *>(&colE[hw + (nc - 1 - c)]), (unsigned long long)v2);
    }
    rs = warp_sum(rs);
    if (lane == 0) {
      mytot += rs;
      if (r < hw) rowE[r] = rs;
      if (r >= mc - hw) rowE[hw + (mc - 1 - r)] = rs;
    }
  }
  if (lane == 0 && mytot) atomicAdd(reinterpret_cast<unsigned long long *>(tot), (unsigned long long)mytot);
}

// SQ = true: g(s,t) = sum over the frame-side rectangle of D_{s,t} of a^2 (the energies);
// SQ = false: the same sums of a itself (the template's linear lag sums of the mean
// removal, kernels_fft2.cuh).  One block per image.
// flip = 1 stores g(-s,-t) at lag (s,t): the TEMPLATE-side rectangle of D_{s,t} (g_b and the
// template's linear sums).
template <bool SQ>
__global__ void __launch_bounds__(1024) k_energy_u16_t(const uint16_t *__restrict__ img, int64_t fstride, int pitch,
                                                      int mc, int nc, int w, u64 *__restrict__ ga,
                                                      u64 *__restrict__ part, int flip = 0) {
  extern __shared__ __align__(16) u64 esm[];
  const int hw = w - 1, W = 2 * w - 1, CS = w * w;
  u64 *rowE = esm;                 // [2 hw]: top rows, bottom rows (from the bottom)
  u64 *colE = rowE + 2 * hw;       // [2 hw]
  u64 *cor = colE + 2 * hw;        // [w][w]: one quadrant at a time
  u64 *tot = cor + CS;             // [1]
  for (int k = threadIdx.x; k < 4 * hw + CS + 1; k += blockDim.x) esm[k] = 0;
  __syncthreads();
  const uint16_t *A = img + (int64_t)blockIdx.x * fstride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  u64 mytot = 0;
  if (part) {   // the row pass was done by k_energy_rows: take its sums and clear them
    u64 *pf = part + (int64_t)blockIdx.x * (4 * hw + 1);
    __syncthreads();
    for (int k = threadIdx.x; k < 4 * hw + 1; k += blockDim.x) {
      esm[k < 4 * hw ? k : 4 * hw + CS] = pf[k];
      pf[k] = 0;
    }
  } else {
    // row pass: warp per row, lane per 8-column chunk (16-byte loads: the coarse images'
    // pitch is a multiple of 8 samples); squares of the edge columns accumulate in the
    // lane's registers (a lane holds at most one left-edge and one right-edge chunk for
    // hw <= 256) and reach shared memory once per frame
    const int nchunk = (nc + 7) >> 3;
    const int cl = lane, cr = lane + 32 * ((nchunk - 1 - lane) >> 5);   // the lane's first / last chunk
    const bool hasL = lane < nchunk && 8 * cl < hw, hasR = lane < nchunk && 8 * cr + 8 > nc - hw;
    u64 eL[8], eR[8];
#pragma unroll
    for (int x = 0; x < 8; ++x) eL[x] = eR[x] = 0;
    for (int r = warp; r < mc; r += nwarp) {
      const uint16_t *row = A + (int64_t)r * pitch;
      u64 rs = 0;
      for (int c = lane; c < nchunk; c += 32) {
        const uint4 q = *reinterpret_cast<const uint4 *>(row + 8 * c);
        const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
        uint32_t sq[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const uint32_t v = (x & 1) ? (wv[x >> 1] >> 16) : (wv[x >> 1] & 0xffffu);
          sq[x] = 8 * c + x < nc ? (SQ ? v * v : v) : 0u;   // < 2^32
          rs += sq[x];
        }
        if (c == cl && hasL)
#pragma unroll
          for (int x = 0; x < 8; ++x) eL[x] += sq[x];
        if (c == cr && hasR)
#pragma unroll
          for (int x = 0; x < 8; ++x) eR[x] += sq[x];
      }
      rs = warp_sum(rs);
      if (lane == 0) {
        mytot += rs;
        if (r < hw) rowE[r] = rs;
        if (r >= mc - hw) rowE[hw + (mc - 1 - r)] = rs;
      }
    }
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const int c0 = 8 * cl + x, c1 = 8 * cr + x;
      if (hasL && c0 < hw) atomicAdd(&colE[c0], eL[x]);
      if (hasR && c1 < nc && c1 >= nc - hw) atomicAdd(&colE[hw + (nc - 1 - c1)], eR[x]);
    }
    if (lane == 0) atomicAdd(tot, mytot);
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    u64 *e = (threadIdx.x & 2) ? colE : rowE;
    u64 *p = e + (threadIdx.x & 1) * hw;
    for (int q = 1; q < hw; ++q) p[q] += p[q - 1];
  }
  __syncthreads();
  u64 *gf = ga + (int64_t)blockIdx.x * W * W;
  for (int lag = threadIdx.x; lag < W * W; lag += blockDim.x) {
    const int s = lag / W - hw, t = lag % W - hw;
    const u64 rex = s > 0 ? rowE[s - 1] : (s < 0 ? rowE[hw + (-s) - 1] : 0);
    const u64 cex = t > 0 ? colE[t - 1] : (t < 0 ? colE[hw + (-t) - 1] : 0);
    gf[flip ? W * W - 1 - lag : lag] = *tot - rex - cex;
  }
  // corners: quadrant (s<0 ? 2 : 0) | (t<0 ? 1 : 0) -- s > 0 excludes the TOP rows, t > 0
  // the LEFT columns; table[p][q] = sum of a^2 over the p x q corner block
  for (int quad = 0; quad < 4; ++quad) {
    const bool bot = quad & 2, rt = quad & 1;
    __syncthreads();
    for (int e = threadIdx.x; e < CS; e += blockDim.x) {
      const int pp = e / w, qq = e % w;
      u64 v2 = 0;
      if (pp > 0 && qq > 0) {
        const int r = bot ? mc - pp : pp - 1, c = rt ? nc - qq : qq - 1;
        const u64 v = A[(int64_t)r * pitch + c];
        v2 = SQ ? v * v : v;
      }
      cor[e] = v2;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < w; k += blockDim.x)
      for (int q = 1; q < w; ++q) cor[k * w + q] += cor[k * w + q - 1];
    __syncthreads();
    for (int k = threadIdx.x; k < w; k += blockDim.x)
      for (int p = 1; p < w; ++p) cor[p * w + k] += cor[(p - 1) * w + k];
    __syncthreads();
    for (int e = threadIdx.x; e < hw * hw; e += blockDim.x) {
      const int as = e / hw + 1, at = e % hw + 1;
      const int s = bot ? -as : as, t = rt ? -at : at;
      const int lg = (s + hw) * W + (t + hw);
      gf[flip ? W * W - 1 - lg : lg] += cor[as * w + at];
    }
  }
}
#define k_energy_u16 k_energy_u16_t<true>

}  // namespace moco
