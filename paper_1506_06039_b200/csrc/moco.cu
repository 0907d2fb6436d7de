// moco.cu -- host side of libmoco.so: the C-ABI declared in include/moco.h.
//
// Plans, workspace, stream-ordered launches of the hot-path kernels
// (kernels_direct.cuh, kernels_tc.cuh) and the host-buffer end-to-end path.
// No CPU fallback: every step of the path runs in the kernels; a CUDA failure
// is reported as MOCO_ECUDA.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <new>
#include <type_traits>
#include <vector>

#include "moco.h"
#include "kernels_direct.cuh"
#include "kernels_tc.cuh"
#include "kernels_refine.cuh"
#include "kernels_rtc.cuh"
#include "kernels_fft.cuh"
#include "kernels_fft2.cuh"
#include "kernels_tcf.cuh"
#include "kernels_fra.cuh"

using namespace moco;

// Kernel launch, optionally with programmatic dependent launch (PDL): the kernel may be
// scheduled while the stream's previous kernel finishes; it calls pdl_enter() first
// (griddepcontrol.wait), so it still sees every write of its predecessor.
template <typename... KArgs, typename... Args>
static cudaError_t launchk(bool pdl, void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                           Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

static thread_local char g_err[512] = "";

static int set_cuda_err(cudaError_t e, const char *what) {
  snprintf(g_err, sizeof(g_err), "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
  return MOCO_ECUDA;
}
#define CK(x)                                        \
  do {                                               \
    cudaError_t e_ = (x);                            \
    if (e_ != cudaSuccess) return set_cuda_err(e_, #x); \
  } while (0)
#define CKL(name)                                            \
  do {                                                       \
    cudaError_t e_ = cudaGetLastError();                     \
    if (e_ != cudaSuccess) return set_cuda_err(e_, name);    \
  } while (0)

struct moco_plan {
  int m, n, w, W, levels, dtype, bits, device;
  int algo;                   // resolved MOCO_ALGO_*
  bool algo_forced;           // set by moco_plan_set_algo (no per-call routing)
  int ml[3], nl[3], pitch[3]; // per level dims and row pitch (elements)
  size_t esz[3];              // element size per level
  void *tpl[3];               // template pyramid
  void *gb;                   // W*W template energies (u64 or double)
  u64 *pb2[3];                // refine levels: 2-D prefix of b^2 [(ml+1)][(nl+1)]
  int rstages[3];             // refine levels: bulk-copy ring depth
  int rrt[3], rnrt[3];        // refine levels: template rows per tile, row tiles
  u64 *racc;                  // refine accumulators [cap][18] (kept zero between calls)
  RtcGeom rtc[3];             // tensor-core refine geometry per level (kernels_rtc.cuh)
  bool pdl_now = false;       // inside a closed-loop (latency-route) call: kernels chained by PDL
  FraGeom fra;                // frame-resident refine + pick + apply at level 0 (kernels_fra.cuh)
  bool fra_ok;
  uint32_t *fra_tc = nullptr; // its shifted, pre-split template copies (k_fra_tcopy)
  uint8_t *rtab[3];           // its template candidate tiles, or null: CUDA-core refine
  int *rperm, *rmeta;         // its per-batch alignment-class bucketing
  int nsm;                    // multiprocessors of the plan's device
  int64_t cap;                // frames per internal batch
  void *scratch[3];           // frame pyramid levels 1..L for one batch
  int32_t *sh[3];             // per-level shifts for one batch
  bool has_tpl;
  // rows of n samples that are not a multiple of 16 bytes: frames are staged through
  // buffers with the padded level-0 pitch (pitch[0] > n)
  bool stage;
  void *stage_in, *stage_out;
  // tuning / cross-check switches, read from the environment ONCE at plan creation
  // (DESIGN.md §8 table) -- no getenv on the per-batch launch path
  struct {
    int rtc = -1;          // MOCO_RTC: -1 default, 0 CUDA-core refine sums, 1 force tensor cores
    int rtc_parts = 0;     // MOCO_RTC_PARTS (0: cost model)
    int prep_fp = 0;       // MOCO_PREP_FP=1: k_tc_prep one frame per CTA (co-resides with the search)
    int pdl = 2;           // MOCO_PDL: programmatic dependent launch 0 off, 1 closed-loop route only,
                           // 2 also every FFT sub-batch chain (w = 85 467 -> 470 k frames/s)
    int fra = 0;           // MOCO_FRA=1: level-0 refine + pick + apply by the frame-resident
                           // cluster kernel k_refine_frame (one HBM read per frame, but bound by
                           // CUDA-core dot products and cluster synchronisation: 0.66 us/frame
                           // alone vs 0.34 for k_refine_tc + k_ga_pieces + k_refine_pick,
                           // DESIGN.md section 11) instead of the tensor-core refine + pick
    int fra_min = 64;      // MOCO_FRA_MIN: smallest batch for k_refine_frame
    bool nofuse_ds = false, ga_inpick = false, nopipe = false;
    bool fft_v1 = false;   // MOCO_FFT_V1=1: the generic FFT kernels (kernels_fft.cuh) for every length
    int fft_mean = -1;     // MOCO_FFT_MEAN=0/1/2: mean removal on the FFT path off / two-sided /
                           // frames only (default: fft_mean_mode)
    int tc_fused = 0;      // MOCO_TC_FUSED=1: k_tc_fused (operand strips built in the search kernel,
                           // kernels_tcf.cuh; measured slower: C2 1.38 vs 1.83 M frames/s)
  } knob;
  bool simple_refine;         // MOCO_REFINE=simple: unfused K6/K7 (cross-check in tests)
  int simple_level;           // MOCO_REFINE=simpleN: simple K6 at level N only (debug)
  int64_t launches;
  // coarse kernel launch geometry
  int c_threads, c_sc, c_br, c_fpitch;
  size_t c_smem;
  // tensor-core path state
  TcPlan tc;
  // FFT path state (kernels_fft.cuh)
  struct {
    bool ready = false, tpl_ready = false;
    FftGeom g;
    float2 *twr = nullptr, *twc = nullptr, *Bc = nullptr, *S = nullptr, *P = nullptr;
    u64 *ga = nullptr;
    int *qc = nullptr;
    u64 *epart = nullptr;       // small batches: row-pass energy partials [cap][4 hw + 1], kept zero
    float *lb = nullptr;        // small-batch split score: lower bounds [cap][W*W]
    float *rmin = nullptr;      // kernels_fft2.cuh: per lag row, the minimum lower bound [2][cap][W]
    int *ub = nullptr;          // and min upper bound per frame [cap]
    cudaStream_t side = nullptr;   // small batches: frame energies beside the FFT
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int64_t cap = 0;
    double bound_Cf = 0, bound_Ci = 0;   // eps_h = u ||a||_2 (Cf ||b||_2 + Ci ||b||_1)
    double2 *R64 = nullptr;     // template spectrum rows in fp64 [mc][Kc] (k_tpl_dft_rows)
    unsigned long long *b1 = nullptr;   // ||b||_1 of the coarse template
    // mean removal (v2): the transforms see a - mu and b - mu on the supports, the score adds
    // back mu (S_a + S_b) - mu^2 A exactly (kernels_fft2.cuh)
    long long *tst = nullptr;   // [4] mu_a, ||b - mu_b||_1, ||b - mu_b||_2^2, mu_b (k_tpl_stats)
    long long *gl = nullptr;    // [W*W] template linear sums per lag (k_energy_u16_t<false>, flipped)
    double *ynorm = nullptr;    // [2 cap] spectrum norms (k_fft2_cols), kept zero
    int smem_rows = 0, smem_cols = 0, smem_score = 0, smem_energy = 0;
    int pc = 0, pr = 0;         // register FFT plans of the row (Mc) and column (Mr) lengths
    // kernels_fft2.cuh (both lengths with a register plan, n_c % 8 == 0): the frame-to-
    // spectrum row kernel reads the level-0 frames itself (no downsample, no g_a kernel)
    bool v2 = false;
    u64 *E = nullptr;           // energy partials [cap][f2_esz(hw)], accumulated slots kept zero
    int *cnt = nullptr;         // finished score blocks per frame [cap], kept zero
    int *qn = nullptr, *ql = nullptr, *cnt2 = nullptr;   // k_fft2_rescore hand-over [cap], kept zero
    u64 *nacc = nullptr;        // its exact N partial sums [cap][max(QCAP, W^2)], kept zero
    int smem2_rows = 0, smem2_cols = 0, smem2_score = 0;
    // sub-batches alternate between two streams and two scratch sets (S, P, E, lb, ub, cnt
    // hold 2 x cap frames): one sub-batch's kernel tails overlap the other's work
    cudaStream_t ss[2] = {nullptr, nullptr};
    cudaEvent_t ev_j[2] = {nullptr, nullptr};
  } fft;
  // two-stream batch pipeline (align_tc_pipelined)
  bool pipe_ready;
  cudaStream_t ps[3];
  cudaEvent_t pe_prep[2], pe_free[2], pe_sums[2], pe_pick[2], pe_start, pe_end, pe_end2;
  int32_t *sh1b;              // second level-1 shift buffer (pipeline)
  int32_t *sh2b[2];           // coarse shifts at level 2 (pipeline, levels = 2)
  void *scratch1b;            // second level-1 image buffer (pipeline, levels = 2)
  u64 *racc2;                 // second refine accumulator buffer (pipeline)
  u64 *gbin[2];               // GA pieces per frame [cap][26] (pipeline, k_ga_pieces)
  // end-to-end staging
  bool host_ready;
  int64_t host_ch;
  void *slot_in[3], *slot_out[3];
  int32_t *slot_sh[3];
  double *slot_f[3];
  uint8_t *slot_flags[3];
  cudaStream_t hs[3];
  cudaEvent_t ev_in[3], ev_done[3], ev_free[3];
  // live per-kernel timing (moco_profile_*)
  bool prof_on;
  struct ProfRec { int kind; cudaEvent_t a, b; };
  std::vector<ProfRec> prof_live;
  std::vector<cudaEvent_t> prof_pool;
};

static cudaEvent_t prof_event(moco_plan *p) {
  if (!p->prof_pool.empty()) {
    cudaEvent_t e = p->prof_pool.back();
    p->prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
// Bracket one launch with events on its stream when profiling is on.
struct ProfScope {
  moco_plan *p;
  cudaStream_t st;
  int kind;
  cudaEvent_t a = nullptr;
  ProfScope(moco_plan *p_, int kind_, cudaStream_t st_) : p(p_), st(st_), kind(kind_) {
    if (p->prof_on) {
      a = prof_event(p);
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = prof_event(p);
      cudaEventRecord(b, st);
      p->prof_live.push_back({kind, a, b});
    }
  }
};

static int round_up(int x, int a) { return (x + a - 1) / a * a; }

static size_t coarse_smem(const moco_plan *p, int sc, int br, int fpitch) {
  const int w = p->w, W = p->W, L = p->levels;
  const size_t acc = 8;
  const size_t e = p->esz[L];
  size_t band = std::max((size_t)4 * w * w * acc,
                         (size_t)br * p->nl[L] * e + (size_t)(br + 2 * (w - 1)) * fpitch * e);
  size_t sz = (size_t)W * W * acc + (size_t)sc * W * acc + 32 * sizeof(Key) +
              (size_t)(4 * w + 1 + 32) * acc;
  sz = (sz + 15) / 16 * 16;
  return sz + band;
}

// Exported functions take their C linkage from the declarations in moco.h.

int moco_abi_version(void) { return MOCO_ABI_VERSION; }

int moco_probe_peaks(int device, double *out, int n) {
  if (!out || n < 0) return MOCO_EINVAL;
  CK(cudaSetDevice(device));
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  uint32_t *sink = nullptr;
  CK(cudaMalloc(&sink, 16));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int iters = 4096, blocks = nsm * 8;
  const double ops_per_inst[4] = {2.0, 2.0, 4.0, 2.0};
  int rc = MOCO_OK;
  for (int k = 0; k < 4 && k < n && rc == MOCO_OK; ++k) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      switch (k) {
        case 0: k_probe<0><<<blocks, 256>>>(iters, rep, sink); break;
        case 1: k_probe<1><<<blocks, 256>>>(iters, rep, sink); break;
        case 2: k_probe<2><<<blocks, 256>>>(iters, rep, sink); break;
        default: k_probe<3><<<blocks, (unsigned)256>>>(iters / 8, rep, sink); break;
      }
      cudaEventRecord(e1);
      if (cudaEventSynchronize(e1) != cudaSuccess) { rc = set_cuda_err(cudaGetLastError(), "k_probe"); break; }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0) best = std::min(best, ms);
    }
    const double insts = (double)blocks * 256 * 8 * (k == 3 ? iters / 8 : iters);
    out[k] = insts * ops_per_inst[k] / (best * 1e-3);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  return rc;
}

int moco_mean_image(const void *d_frames, int64_t T, int m, int n, int dtype, double *d_mean, moco_stream_t stream) {
  if (T < 1 || m < 1 || n < 1 || !d_frames || !d_mean || (dtype != MOCO_U16 && dtype != MOCO_F32)) return MOCO_EINVAL;
  const int64_t mn = (int64_t)m * n;
  const unsigned grid = (unsigned)std::min<int64_t>((mn + 255) / 256, 148 * 16);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == MOCO_U16) k_mean_image<uint16_t><<<grid, 256, 0, st>>>((const uint16_t *)d_frames, T, mn, d_mean);
  else k_mean_image<float><<<grid, 256, 0, st>>>((const float *)d_frames, T, mn, d_mean);
  CKL("k_mean_image");
  return MOCO_OK;
}

int moco_auto_config(int m, int n, int *w, int *levels) {
  if (!w || !levels || m < 1 || n < 1) return MOCO_EINVAL;
  const int L = (m > 256 || n > 256) ? 1 : 0;
  const int wc = std::min(m >> L, n >> L) / 3;  // P:49 min(m,n)/3, at the coarse level (R16)
  if (wc < 1) return MOCO_EINVAL;
  *w = wc;
  *levels = L;
  return MOCO_OK;
}

const char *moco_strerror(int code) {
  switch (code) {
    case MOCO_OK: return "ok";
    case MOCO_EINVAL: return "invalid argument";
    case MOCO_ENOMEM: return "out of memory";
    case MOCO_ECUDA: return "CUDA error";
    case MOCO_ESTATE: return "invalid call order (template not set)";
    default: return "unknown moco status";
  }
}

const char *moco_last_cuda_error(void) { return g_err; }

int64_t moco_last_launch_count(const moco_plan *p) { return p ? p->launches : 0; }

static void plan_free(moco_plan *p) {
  if (!p) return;
  for (int l = 0; l < 3; ++l) {
    if (p->tpl[l]) cudaFree(p->tpl[l]);
    if (p->scratch[l]) cudaFree(p->scratch[l]);
    if (p->sh[l]) cudaFree(p->sh[l]);
  }
  if (p->gb) cudaFree(p->gb);
  if (p->racc) cudaFree(p->racc);
  if (p->fra_tc) cudaFree(p->fra_tc);
  for (int l = 0; l < 3; ++l) {
    if (p->pb2[l]) cudaFree(p->pb2[l]);
    if (p->rtab[l]) cudaFree(p->rtab[l]);
  }
  if (p->rperm) cudaFree(p->rperm);
  if (p->stage_in) cudaFree(p->stage_in);
  if (p->stage_out) cudaFree(p->stage_out);
  if (p->rmeta) cudaFree(p->rmeta);
  tc_free(&p->tc);
  for (void *q : {(void *)p->fft.twr, (void *)p->fft.twc, (void *)p->fft.Bc, (void *)p->fft.S, (void *)p->fft.P,
                  (void *)p->fft.ga, (void *)p->fft.qc, (void *)p->fft.lb, (void *)p->fft.rmin, (void *)p->fft.ub, (void *)p->fft.epart})
    if (q) cudaFree(q);
  if (p->fft.side) cudaStreamDestroy(p->fft.side);
  if (p->fft.ev_fork) cudaEventDestroy(p->fft.ev_fork);
  if (p->fft.ev_join) cudaEventDestroy(p->fft.ev_join);
  for (int k = 0; k < 3; ++k) {
    if (p->slot_in[k]) cudaFree(p->slot_in[k]);
    if (p->slot_out[k]) cudaFree(p->slot_out[k]);
    if (p->slot_sh[k]) cudaFree(p->slot_sh[k]);
    if (p->slot_f[k]) cudaFree(p->slot_f[k]);
    if (p->slot_flags[k]) cudaFree(p->slot_flags[k]);
    if (p->ev_in[k]) cudaEventDestroy(p->ev_in[k]);
    if (p->ev_done[k]) cudaEventDestroy(p->ev_done[k]);
    if (p->ev_free[k]) cudaEventDestroy(p->ev_free[k]);
  }
  for (int k = 0; k < 3; ++k)
    if (p->hs[k]) cudaStreamDestroy(p->hs[k]);
  for (int k = 0; k < 3; ++k)
    if (p->ps[k]) cudaStreamDestroy(p->ps[k]);
  for (int k = 0; k < 2; ++k)
    for (cudaEvent_t e : {p->pe_prep[k], p->pe_free[k], p->pe_sums[k], p->pe_pick[k]})
      if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {p->pe_start, p->pe_end, p->pe_end2})
    if (e) cudaEventDestroy(e);
  if (p->sh1b) cudaFree(p->sh1b);
  for (int k = 0; k < 2; ++k)
    if (p->sh2b[k]) cudaFree(p->sh2b[k]);
  if (p->scratch1b) cudaFree(p->scratch1b);
  if (p->racc2) cudaFree(p->racc2);
  for (int k = 0; k < 2; ++k)
    if (p->gbin[k]) cudaFree(p->gbin[k]);
  for (int k = 0; k < 2; ++k) {
    if (p->fft.ss[k]) cudaStreamDestroy(p->fft.ss[k]);
    if (p->fft.ev_j[k]) cudaEventDestroy(p->fft.ev_j[k]);
  }
  if (p->fft.R64) cudaFree(p->fft.R64);
  if (p->fft.tst) cudaFree(p->fft.tst);
  if (p->fft.gl) cudaFree(p->fft.gl);
  if (p->fft.ynorm) cudaFree(p->fft.ynorm);
  if (p->fft.b1) cudaFree(p->fft.b1);
  if (p->fft.E) cudaFree(p->fft.E);
  if (p->fft.cnt) cudaFree(p->fft.cnt);
  if (p->fft.qn) cudaFree(p->fft.qn);
  if (p->fft.ql) cudaFree(p->fft.ql);
  if (p->fft.cnt2) cudaFree(p->fft.cnt2);
  if (p->fft.nacc) cudaFree(p->fft.nacc);
  for (auto &r : p->prof_live) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : p->prof_pool) cudaEventDestroy(e);
  delete p;
}

// ---------------------------------------------------------------- FFT path (S3 by FFT)
// call fn(std::integral_constant<int, P>) for the kernel instantiation of FFT plan P
template <class Fn>
static void fft_dispatch(int plan, Fn &&fn) {
  switch (plan) {
    case 1: fn(std::integral_constant<int, 1>{}); break;
    case 2: fn(std::integral_constant<int, 2>{}); break;
    case 3: fn(std::integral_constant<int, 3>{}); break;
    case 4: fn(std::integral_constant<int, 4>{}); break;
    case 5: fn(std::integral_constant<int, 5>{}); break;
    case 6: fn(std::integral_constant<int, 6>{}); break;
    default: fn(std::integral_constant<int, 0>{}); break;
  }
}
static bool fft_supported(const moco_plan *p) {
  if (p->dtype != MOCO_U16 || p->w - 1 > 248) return false;   // (k_energy_u16: edge chunks in one lane round)
  const int L = p->levels;
  FftLen a, b;
  return fft_len_make(p->ml[L] + p->w - 1, &a) && fft_len_make(p->nl[L] + p->w - 1, &b);
}

// row pairs per k_fft2_rows block: at most NF transforms and F2_STAGE_MAX staged raw bytes
static int fft2_rows_per_max(int NF, int L, int nc) {
  return std::max(1, std::min(NF, F2_STAGE_MAX / f2_stage_bytes(1, L, nc)));
}
static int fft2_rows_smem(int P_N, int NF, int STRIDE, int per, int L, int nc, int hw) {
  return f2_stage_bytes(per, L, nc) + (P_N + NF * STRIDE) * 8 + 2 * NF * 8 + 2 * hw * 8;
}

// kappa of one 1-D transform of length L.N as the kernels compute it: a two-pass register
// plan (N1 codelet, twiddle stage, N2 codelet) or the generic radix-2/3/4/5 Stockham stages
static double fft_kappa_len(const FftLen &L, int plan) {
  int n1 = 0, n2 = 0;
  switch (plan) {
    case 1: n1 = Plan2p<1>::N1; n2 = Plan2p<1>::N2; break;
    case 2: n1 = Plan2p<2>::N1; n2 = Plan2p<2>::N2; break;
    case 3: n1 = Plan2p<3>::N1; n2 = Plan2p<3>::N2; break;
    case 4: n1 = Plan2p<4>::N1; n2 = Plan2p<4>::N2; break;
    case 5: n1 = Plan2p<5>::N1; n2 = Plan2p<5>::N2; break;
    case 6: n1 = Plan2p<6>::N1; n2 = Plan2p<6>::N2; break;
    default: break;
  }
  if (n1) return fft_kappa_codelet(n1) + 3 + fft_kappa_codelet(n2);
  double k = 0;
  for (int st = 0; st < L.nst; ++st) k += fft_mu(L.rad[st]) + 3;
  return k;
}
// Constants of eps_h = u ||a||_2 (Cf ||b||_2 + Ci ||b||_1), DESIGN.md §5.  Per lag, the
// errors made before the inverse transform -- the forward 2-D transform of a (row
// transforms, unpack of the packed real rows, column transforms), the fp32 rounding of the
// fp64 template spectrum (1) and of the spectrum product (2 sqrt 2) -- reach h(s,t) as a
// correlation with b, so Cauchy-Schwarz bounds them by ||.||_2 ||b||_2; the inverse
// transform's own rounding (columns, packing of two lag rows, rows) is bounded through
// ||Y||_2 <= ||a||_2 ||b||_1 / sqrt(N).  x 1.1 for the second-order terms (each first-order
// term is ~ kappa u ~ 1e-5 relative).
static void fft_bound_C(const FftLen &Lr, int pr, const FftLen &Lc, int pc, double *Cf, double *Ci) {
  const double kr = fft_kappa_len(Lr, pr), kc = fft_kappa_len(Lc, pc);
  *Cf = 1.1 * ((kc + 1 + kr) + 1 + 2 * std::sqrt(2.0));
  *Ci = 1.1 * (kr + 1 + kc);
}

static int fft_init(moco_plan *p) {
  auto &F = p->fft;
  if (F.ready) return MOCO_OK;
  const int L = p->levels;
  FftGeom &g = F.g;
  g.mc = p->ml[L]; g.nc = p->nl[L]; g.w = p->w; g.hw = p->w - 1; g.W = p->W;
  if (!fft_len_make(g.mc + g.hw, &g.Lr) || !fft_len_make(g.nc + g.hw, &g.Lc)) return MOCO_EINVAL;
  g.Kc = g.Lc.N / 2 + 1;
  g.mcp = (g.mc + 1) / 2 * 2;
  F.pc = fft_plan_of(g.Lc.N);
  F.pr = fft_plan_of(g.Lr.N);
  F.v2 = F.pc > 0 && F.pr > 0 && g.nc % 8 == 0 && !p->knob.fft_v1;
  const size_t esz = (size_t)f2_esz2(g.hw) * 8;
  // sub-batches sized so the spectra stay in L2 (about 80 MB)
  const size_t per = F.v2 ? (size_t)g.Kc * g.mcp * 8 + (size_t)g.W * g.Kc * 8 + (size_t)g.W * g.W * 4 + esz
                          : (size_t)g.Kc * g.mcp * 8 + (size_t)g.W * g.Kc * 8 + (size_t)g.W * g.W * 8;
  size_t budget = (size_t)(F.v2 ? 160u : 80u) << 20;   // per set (v2: two sets); measured: 40 -> 160 MB per set C3 595 -> 628 k, w = 85 306 -> 348 k frames/s
  if (const char *mb = getenv("MOCO_FFT_MB")) budget = (size_t)std::max(4, atoi(mb)) << 20;   // tuning (plan creation)
  F.cap = std::max<int64_t>(1, std::min<int64_t>(p->cap, (int64_t)(budget / per)));
  const int64_t nset = F.v2 ? 2 : 1;   // v2: two scratch sets (two streams)
  const int Mr = g.Lr.N, Mc = g.Lc.N;
  auto al = [&](void **q, size_t bytes) {
    if (cudaMalloc(q, bytes) != cudaSuccess) { cudaGetLastError(); return false; }
    return true;
  };
  if (!al((void **)&F.R64, (size_t)g.mc * g.Kc * 16) || !al((void **)&F.b1, 8) || !al((void **)&F.tst, 4 * 8) ||
      !al((void **)&F.gl, (size_t)g.W * g.W * 8))
    return MOCO_ENOMEM;
  if (!al((void **)&F.twr, Mr * 8) || !al((void **)&F.twc, Mc * 8) || !al((void **)&F.Bc, (size_t)g.Kc * Mr * 8) ||
      !al((void **)&F.S, (size_t)nset * F.cap * g.Kc * g.mcp * 8) ||
      !al((void **)&F.P, (size_t)nset * F.cap * g.W * g.Kc * 8) ||
      !al((void **)&F.ga, (size_t)F.cap * g.W * g.W * 8) || !al((void **)&F.qc, (size_t)p->cap * sizeof(int)) ||
      !al((void **)&F.lb, (size_t)nset * F.cap * g.W * g.W * 4) || !al((void **)&F.rmin, (size_t)nset * F.cap * g.W * 4) ||
      !al((void **)&F.ub, (size_t)nset * F.cap * sizeof(int)) ||
      !al((void **)&F.epart, (size_t)F.cap * (4 * g.hw + 1) * 8))
    return MOCO_ENOMEM;
  CK(cudaMemset(F.epart, 0, (size_t)F.cap * (4 * g.hw + 1) * 8));
  if (F.v2) {
    if (!al((void **)&F.E, (size_t)2 * F.cap * esz) || !al((void **)&F.cnt, (size_t)2 * F.cap * sizeof(int)))
      return MOCO_ENOMEM;
    CK(cudaMemset(F.E, 0, (size_t)2 * F.cap * esz));
    CK(cudaMemset(F.cnt, 0, (size_t)2 * F.cap * sizeof(int)));
    const size_t nslots = (size_t)std::max(FFT_QCAP, g.W * g.W);
    if (!al((void **)&F.qn, (size_t)2 * F.cap * sizeof(int)) || !al((void **)&F.cnt2, (size_t)2 * F.cap * sizeof(int)) ||
        !al((void **)&F.ql, (size_t)2 * F.cap * FFT_QCAP * sizeof(int)) || !al((void **)&F.nacc, (size_t)2 * F.cap * nslots * 8))
      return MOCO_ENOMEM;
    CK(cudaMemset(F.qn, 0, (size_t)2 * F.cap * sizeof(int)));
    CK(cudaMemset(F.cnt2, 0, (size_t)2 * F.cap * sizeof(int)));
    CK(cudaMemset(F.nacc, 0, (size_t)2 * F.cap * nslots * 8));
    if (!al((void **)&F.ynorm, (size_t)2 * F.cap * 8)) return MOCO_ENOMEM;
    CK(cudaMemset(F.ynorm, 0, (size_t)2 * F.cap * 8));
    for (int k = 0; k < 2; ++k) {
      CK(cudaStreamCreateWithFlags(&F.ss[k], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&F.ev_j[k], cudaEventDisableTiming));
    }
  }
  CK(cudaMemset(F.ub, 0x7f, (size_t)nset * F.cap * sizeof(int)));   // FFT_UB_INIT
  CK(cudaStreamCreateWithFlags(&F.side, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&F.ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&F.ev_join, cudaEventDisableTiming));
  // derived first-order bound |h~ - h| <= C u ||a||_2 ||b||_1 (kernels_fft.cuh)
  fft_bound_C(g.Lr, F.pr, g.Lc, F.pc, &F.bound_Cf, &F.bound_Ci);
  // (the scratch half of each transform buffer carries FFT_YPAD extra elements per
  // transform: the padded rows of the two-pass register plans, kernels_fft.cuh fft2p)
  F.smem_rows = (Mc + FFT_ROWS_PAIRS * Mc + FFT_ROWS_PAIRS * (Mc + FFT_YPAD)) * 8;
  F.smem_cols = (Mr + FFT_COLS * Mr + FFT_COLS * (Mr + FFT_YPAD)) * 8;
  F.smem_score = (Mc + FFT_ROWS_PAIRS * Mc + FFT_ROWS_PAIRS * (Mc + FFT_YPAD)) * 8 + ((g.W * g.W + 1) & ~1) * 4 + 2 * g.W * 8;
  F.smem_energy = (4 * g.hw + g.w * g.w + 1) * 8;
  if (F.smem_score > 227 * 1024 || F.smem_energy > 227 * 1024) return MOCO_EINVAL;
  int rc_attr = MOCO_OK;
  if (F.v2) {
    fft_dispatch(F.pc, [&](auto PC) {
      constexpr int P = decltype(PC)::value;
      if constexpr (P > 0) {
        using G = F2<P>;
        const int LK = std::min(L, 1);
        const int stg = std::max(f2_stage_bytes(fft2_rows_per_max(G::NF, LK, g.nc), LK, g.nc),
                                 f2_stage_bytes(fft2_rows_per_max(G::NF, 0, g.nc), 0, g.nc));
        F.smem2_rows = stg + (G::N + G::NF * G::STRIDE) * 8 + 2 * G::NF * 8 + 2 * g.hw * 8;
        F.smem2_score = (G::N + G::NF * G::STRIDE) * 8 + 4 * g.W * 8 + 2 * g.W * 8;
        if (smem_attr(k_fft2_rows<P, 0>, F.smem2_rows) != cudaSuccess ||
            smem_attr(k_fft2_rows<P, 1>, F.smem2_rows) != cudaSuccess ||
            smem_attr(k_fft2_score<P>, F.smem2_score) != cudaSuccess)
          rc_attr = set_cuda_err(cudaGetLastError(), "fft2 kernel attributes");
      }
    });
    fft_dispatch(F.pr, [&](auto PR) {
      constexpr int P = decltype(PR)::value;
      if constexpr (P > 0) {
        using G = F2<P>;
        F.smem2_cols = (G::N + G::NF * G::STRIDE) * 8;
        if (smem_attr(k_fft2_cols<P>, F.smem2_cols) != cudaSuccess)
          rc_attr = set_cuda_err(cudaGetLastError(), "fft2 kernel attributes");
      }
    });
    if (F.smem2_score > 227 * 1024) return MOCO_EINVAL;
  }
  fft_dispatch(F.pc, [&](auto PC) {
    constexpr int P = decltype(PC)::value;
    if (smem_attr(k_fft_rows<P>, F.smem_rows) != cudaSuccess || smem_attr(k_fft_score_rows<P>, F.smem_rows) != cudaSuccess ||
        smem_attr(k_fft_score<P>, F.smem_score) != cudaSuccess)
      rc_attr = set_cuda_err(cudaGetLastError(), "fft kernel attributes");
  });
  fft_dispatch(F.pr, [&](auto PR) {
    constexpr int P = decltype(PR)::value;
    if (smem_attr(k_fft_cols<P>, F.smem_cols) != cudaSuccess) rc_attr = set_cuda_err(cudaGetLastError(), "fft kernel attributes");
  });
  if (rc_attr) return rc_attr;
  CK(smem_attr(k_energy_u16, F.smem_energy));
  CK(smem_attr(k_energy_u16_t<false>, F.smem_energy));
  k_fft_twiddles<<<(Mr + 255) / 256, 256>>>(F.twr, Mr);
  k_fft_twiddles<<<(Mc + 255) / 256, 256>>>(F.twc, Mc);
  CKL("k_fft_twiddles");
  CK(cudaDeviceSynchronize());
  F.ready = true;
  return MOCO_OK;
}

// ---- kernels_fft2.cuh launches (F.v2)
// mean removal on the register-plan FFT path (kernels_fft2.cuh): 0 off, 1 two-sided (frames
// and template shifted by the template's mean mu; the frames' value strips and corner
// tables cost a second set of scans), 2 one-sided (the frames only: h = h' + mu S_b, S_b per
// plan; one frame total).  Measured (B200, u16 frames/s, modes 0 / 1 / 2): C2 602 / 749 /
// 757 k, C4 294 / 303 / 309 k, w = 85 320 / 290 / 342 k, C1 (levels = 0, every frame
// re-scores its winner anyway) 798 / 764 / 788 k.  Default: 2 for levels >= 1, else 0.
static int fft_mean_mode(const moco_plan *p) {
  if (!p->fft.v2) return 0;
  if (p->knob.fft_mean >= 0) return p->knob.fft_mean;
  return p->levels >= 1 ? 2 : 0;
}

static F2RowsArgs fft2_rows_args(const moco_plan *p, const void *img, int64_t fstride, int pitch, int per, int set) {
  const auto &F = p->fft;
  const FftGeom &g = F.g;
  F2RowsArgs a{};
  a.frames = (const uint16_t *)img; a.fstride = fstride; a.pitch = pitch;
  a.mc = g.mc; a.nc = g.nc; a.hw = g.hw; a.Kc = g.Kc; a.mcp = g.mcp;
  a.per = per; a.tw = F.twc; a.S = F.S + (int64_t)set * F.cap * g.Kc * g.mcp;
  a.E = nullptr;
  return a;
}
template <int PC>
static void fft2_rows_launch(const F2RowsArgs &a, int L, int64_t nblk, int hw, cudaStream_t st, bool pdl = false) {
  using G = F2<PC>;
  const int smem = fft2_rows_smem(G::N, G::NF, G::STRIDE, a.per, L, a.nc, hw);
  if (L == 0) launchk(pdl, k_fft2_rows<PC, 0>, (unsigned)nblk, F2_THREADS, smem, st, a);
  else launchk(pdl, k_fft2_rows<PC, 1>, (unsigned)nblk, F2_THREADS, smem, st, a);
}


// One sub-batch of nb level-0 frames through the three kernels of kernels_fft2.cuh, with
// scratch set `set`, on stream st.
// fr: the sub-batch's level-0 frames (levels <= 1) or level-1 images (levels = 2, LK = 1)
static int fft2_sub(moco_plan *p, const char *fr, int64_t fstride, int pitch, int64_t nb, int set,
                    int32_t *shift_out, double *f_out, uint8_t *flags, float *h_out, int *qcount,
                    cudaStream_t st) {
  auto &F = p->fft;
  const FftGeom &g = F.g;
  const int L = p->levels, LK = std::min(L, 1);
  const int64_t so = (int64_t)set * F.cap;
  // PDL through the sub-batch's chain (rows -> cols -> score -> rescore): the closed-loop
  // route, and (MOCO_PDL=2, the default) every sub-batch
  const bool pdl = p->pdl_now || (p->knob.pdl >= 2 && !p->prof_on);
  float2 *Pset = F.P + so * g.W * g.Kc;
  fft_dispatch(F.pc, [&](auto PC) {
    constexpr int P = decltype(PC)::value;
    if constexpr (P > 0) {
      // transforms per block: as many as fit, fewer when the batch cannot fill the SMs
      const int npair = g.mcp / 2;
      const int per = (int)std::max<int64_t>(1, std::min<int64_t>(fft2_rows_per_max(F2<P>::NF, LK, g.nc),
                                                                  nb * npair / p->nsm));
      F2RowsArgs a = fft2_rows_args(p, fr, fstride, pitch, per, set);
      a.E = F.E + so * f2_esz2(g.hw);
      a.mu = F.tst;
      ProfScope ps(p, MOCO_K_PREP, st);
      fft2_rows_launch<P>(a, LK, nb * ((npair + per - 1) / per), g.hw, st, pdl);
    }
  });
  CKL("k_fft2_rows");
  fft_dispatch(F.pr, [&](auto PR) {
    constexpr int P = decltype(PR)::value;
    if constexpr (P > 0) {
      constexpr int NF = F2<P>::NF;
      // even split of the Kc bins over the fewest blocks of <= NF
      int per = (int)std::max<int64_t>(1, std::min<int64_t>(NF, nb * g.Kc / p->nsm));
      const int nblk = (g.Kc + per - 1) / per;
      per = (g.Kc + nblk - 1) / nblk;
      F2ColsArgs c{};
      c.S = F.S + so * g.Kc * g.mcp; c.mc = g.mc; c.Kc = g.Kc; c.mcp = g.mcp; c.W = g.W; c.hw = g.hw;
      c.per = per; c.tw = F.twr; c.Bc = F.Bc; c.P = Pset; c.Bout = nullptr; c.scale = 0.f;
      c.E = F.E + so * f2_esz2(g.hw);
      c.Mc = g.Lc.N;
      c.lin = fft_mean_mode(p) == 1 ? 1 : 0;
      c.ynorm = F.ynorm + so;
      ProfScope ps(p, MOCO_K_COARSE, st);
      launchk(pdl, k_fft2_cols<P>, (unsigned)(nb * nblk), F2_THREADS, F.smem2_cols, st, c);
    }
  });
  CKL("k_fft2_cols");
  fft_dispatch(F.pc, [&](auto PC) {
    constexpr int P = decltype(PC)::value;
    if constexpr (P > 0) {
      constexpr int NF = F2<P>::NF;
      const int npairs = (g.W + 1) / 2;
      // several blocks per SM: the per-block energy set-up is small, the transforms few
      int per = (int)std::max<int64_t>(1, std::min<int64_t>(NF, nb * npairs / (4 * p->nsm)));
      const int nblk = (npairs + per - 1) / per;
      per = (npairs + nblk - 1) / nblk;
      F2ScoreArgs a{};
      a.P = Pset; a.tw = F.twc; a.mc = g.mc; a.nc = g.nc; a.hw = g.hw; a.W = g.W; a.Kc = g.Kc;
      a.per = per; a.E = F.E + so * f2_esz2(g.hw); a.Ew = F.E + so * f2_esz2(g.hw); a.gb = (const u64 *)p->gb;
      a.tst = F.tst; a.gl = F.gl; a.ynorm = F.ynorm + so; a.sqrtN = std::sqrt((double)g.Lr.N * (double)g.Lc.N);
      a.scale = (double)(1u << (4 * L)); a.eps_f = std::ldexp(F.bound_Cf, -24); a.eps_i = std::ldexp(F.bound_Ci, -24); a.b1 = F.b1;
      a.frames = (const uint16_t *)fr; a.fstride = fstride; a.pitch = pitch; a.L = LK;
      a.tpl = (const uint16_t *)p->tpl[L]; a.tpitch = p->pitch[L];
      a.lb = F.lb + so * g.W * g.W; a.rmin = F.rmin + so * g.W; a.ub = F.ub + so; a.cnt = F.cnt + so;
      a.shift_out = shift_out; a.f_out = f_out; a.flags = flags; a.qcount = qcount; a.h_out = h_out;
      a.qn = F.qn + so; a.ql = F.ql + so * FFT_QCAP; a.cnt2 = F.cnt2 + so;
      a.nacc = F.nacc + so * (int64_t)std::max(FFT_QCAP, g.W * g.W);
      // row parts per frame: 16 rows each for full batches, down to 2 rows when few frames
      // (the closed-loop call: the exact sums are latency-bound, one block per part)
      a.rparts = (int)std::max<int64_t>(1, std::min<int64_t>(g.mc / 2, std::max<int64_t>(g.mc / 16, 4 * p->nsm / nb)));
      ProfScope ps(p, MOCO_K_SCORE, st);
      launchk(pdl, k_fft2_score<P>, (unsigned)(nb * nblk), F2_THREADS, F.smem2_score, st, a);
      const unsigned rg = (unsigned)(nb * a.rparts);
      if (LK == 0) launchk(pdl, k_fft2_rescore<0>, rg, 256, 0, st, a);
      else launchk(pdl, k_fft2_rescore<1>, rg, 256, 0, st, a);
    }
  });
  CKL("k_fft2_score");
  p->launches += 4;
  return MOCO_OK;
}

// S1-S4 by FFT for B level-0 frames (kernels_fft2.cuh): rows (block sums, energies, row
// FFTs), columns (times the template spectrum), score + certified pick, per sub-batch of
// <= F.cap frames; several sub-batches alternate between two streams (fork/join with the
// caller's stream, graph-capturable).  img1: levels = 2, the level-1 images out.
static int launch_fft2(moco_plan *p, const void *frames, int64_t fstride, int pitch, int64_t B, int32_t *shift_out,
                       double *f_out, uint8_t *flags, cudaStream_t st, float *h_out = nullptr,
                       int *qcount = nullptr) {
  auto &F = p->fft;
  const FftGeom &g = F.g;
  const int64_t nsub = (B + F.cap - 1) / F.cap;
  const bool two = nsub > 1;
  if (two) {
    CK(cudaEventRecord(F.ev_fork, st));
    for (int k = 0; k < 2; ++k) CK(cudaStreamWaitEvent(F.ss[k], F.ev_fork, 0));
  }
  for (int64_t k = 0; k < nsub; ++k) {
    const int64_t b0 = k * F.cap, nb = std::min<int64_t>(F.cap, B - b0);
    const int set = two ? (int)(k & 1) : 0;
    const int rc = fft2_sub(p, (const char *)frames + b0 * fstride * 2, fstride, pitch, nb, set, shift_out + 2 * b0,
                            f_out ? f_out + b0 : nullptr, flags ? flags + b0 : nullptr,
                            h_out ? h_out + b0 * g.W * g.W : nullptr, qcount ? qcount + b0 : nullptr,
                            two ? F.ss[set] : st);
    if (rc) return rc;
  }
  if (two) {
    for (int k = 0; k < 2; ++k) {
      CK(cudaEventRecord(F.ev_j[k], F.ss[k]));
      CK(cudaStreamWaitEvent(st, F.ev_j[k], 0));
    }
  }
  return MOCO_OK;
}

// template spectrum conj(B^)/(Mr Mc), column-major [k][u] (once per template), computed
// in fp64 by a direct separable DFT and rounded once (the error bound of kernels_fft.cuh
// counts that single rounding), and ||b||_1
static int fft_set_template(moco_plan *p, cudaStream_t st) {
  auto &F = p->fft;
  const int L = p->levels;
  const FftGeom &g = F.g;
  const int Mr = g.Lr.N, Mc = g.Lc.N;
  CK(cudaMemsetAsync(F.b1, 0, 8, st));
  // v2: the spectrum of b - mu (mean removal); the generic kernels use b itself (mu = 0)
  const int mean = fft_mean_mode(p);
  k_tpl_stats<<<1, 1024, 0, st>>>((const uint16_t *)p->tpl[L], p->pitch[L], g.mc, g.nc, mean, F.tst);
  if (mean)
    k_energy_u16_t<false><<<1, 1024, (4 * g.hw + g.w * g.w + 1) * 8, st>>>(   // (w - 1 <= 248: fft_supported)
        (const uint16_t *)p->tpl[L], 0, p->pitch[L], g.mc, g.nc, g.w, (u64 *)F.gl, nullptr, 1);
  k_tpl_dft_rows<<<g.mc, 256, Mc * 16 + g.nc * 8, st>>>((const uint16_t *)p->tpl[L], p->pitch[L], g.nc, Mc, g.Kc,
                                                          F.R64, F.tst);
  k_tpl_dft_cols<<<g.Kc, 256, (Mr + g.mc) * 16, st>>>(F.R64, g.mc, Mr, Mc, g.Kc, F.Bc, F.b1, (const uint16_t *)p->tpl[L],
                                            p->pitch[L], g.nc);
  CKL("fft template spectrum");
  F.tpl_ready = true;
  return MOCO_OK;
}

[[maybe_unused]] static int fft_set_template_fp32(moco_plan *p, cudaStream_t st) {
  auto &F = p->fft;
  const int L = p->levels;
  const FftGeom &g = F.g;
  const int nrb = (g.mcp / 2 + FFT_ROWS_PAIRS - 1) / FFT_ROWS_PAIRS;
  const int ncb = (g.Kc + FFT_COLS - 1) / FFT_COLS;
  fft_dispatch(F.pc, [&](auto PC) {
    k_fft_rows<decltype(PC)::value><<<nrb, FFT_THREADS, F.smem_rows, st>>>((const uint16_t *)p->tpl[L], 0, p->pitch[L],
                                                                           g, F.twc, F.S, FFT_ROWS_PAIRS);
  });
  fft_dispatch(F.pr, [&](auto PR) {
    k_fft_cols<decltype(PR)::value><<<ncb, FFT_THREADS, F.smem_cols, st>>>(F.S, g, F.twr, F.Bc, nullptr, 1, FFT_COLS);
  });
  CKL("fft_set_template");
  F.tpl_ready = true;
  return MOCO_OK;
}

// S3+S4 by FFT with certification, for B coarse frames (level-L images).
static int launch_fft(moco_plan *p, const void *img, int64_t fstride, int pitch, int64_t B, int32_t *shift_out,
                      double *f_out, uint8_t *flags, cudaStream_t st, float *h_out = nullptr,
                      int *qcount = nullptr) {
  auto &F = p->fft;
  const FftGeom &g = F.g;
  const int L = p->levels;
  for (int64_t b0 = 0; b0 < B; b0 += F.cap) {
    const int64_t nb = std::min<int64_t>(F.cap, B - b0);
    const uint16_t *im = (const uint16_t *)img + b0 * fstride;
    // small batches (closed loop): a whole SM per frame for the per-frame kernels, the
    // frame energies on a side stream beside the FFT, the score step split over blocks
    const bool small = nb * (((g.W + 1) / 2 + FFT_ROWS_PAIRS - 1) / FFT_ROWS_PAIRS) <= p->nsm;
    // transforms per block: fewer when the batch alone cannot fill the SMs
    const int rper = small ? std::max(1, std::min(FFT_ROWS_PAIRS, (int)(nb * (g.mcp / 2) / p->nsm))) : FFT_ROWS_PAIRS;
    const int cper = small ? std::max(1, std::min(FFT_COLS, (int)(nb * g.Kc / p->nsm))) : FFT_COLS;
    const int sper = small ? std::max(1, std::min(FFT_ROWS_PAIRS, (int)(nb * ((g.W + 1) / 2) / p->nsm))) : FFT_ROWS_PAIRS;
    const int nrb = (g.mcp / 2 + rper - 1) / rper, ncb = (g.Kc + cper - 1) / cper;
    const int npb = ((g.W + 1) / 2 + sper - 1) / sper;
    cudaStream_t se = st;
    if (small) {
      CK(cudaEventRecord(F.ev_fork, st));
      CK(cudaStreamWaitEvent(F.side, F.ev_fork, 0));
      se = F.side;
    }
    {
      ProfScope ps(p, MOCO_K_PREP, se);
      const int eth = nb < p->nsm ? 1024 : 256;
      if (small) {   // row pass over ~all SMs, then the per-frame remainder
        const int rpb = std::max<int>(8, (int)((nb * g.mc + p->nsm - 1) / p->nsm));
        k_energy_rows<<<(unsigned)(nb * ((g.mc + rpb - 1) / rpb)), 256, 0, se>>>(im, fstride, pitch, g.mc, g.nc,
                                                                                  g.w, rpb, F.epart);
        k_energy_u16<<<(unsigned)nb, eth, F.smem_energy, se>>>(im, fstride, pitch, g.mc, g.nc, g.w, F.ga, F.epart);
      } else {
        k_energy_u16<<<(unsigned)nb, eth, F.smem_energy, se>>>(im, fstride, pitch, g.mc, g.nc, g.w, F.ga, nullptr);
      }
    }
    if (small) CK(cudaEventRecord(F.ev_join, se));
    {
      ProfScope ps(p, MOCO_K_COARSE, st);
      fft_dispatch(F.pc, [&](auto PC) {
        k_fft_rows<decltype(PC)::value><<<(unsigned)(nb * nrb), FFT_THREADS, F.smem_rows, st>>>(im, fstride, pitch, g,
                                                                                               F.twc, F.S, rper);
      });
      fft_dispatch(F.pr, [&](auto PR) {
        k_fft_cols<decltype(PR)::value><<<(unsigned)(nb * ncb), FFT_THREADS, F.smem_cols, st>>>(F.S, g, F.twr, F.Bc,
                                                                                               F.P, 0, cper);
      });
    }
    if (small) CK(cudaStreamWaitEvent(st, F.ev_join, 0));
    FftScoreArgs a;
    a.P = F.P; a.twc = F.twc; a.img = im; a.fstride = fstride; a.pitch = pitch;
    a.tpl = (const uint16_t *)p->tpl[L]; a.tpitch = p->pitch[L];
    a.ga = F.ga; a.gb = (const u64 *)p->gb; a.g = g;
    a.scale = (double)(1u << (4 * L)); a.eps_f = std::ldexp(F.bound_Cf, -24); a.eps_i = std::ldexp(F.bound_Ci, -24); a.b1 = F.b1; a.B = (int)nb;
    a.shift_out = shift_out + 2 * b0; a.f_out = f_out ? f_out + b0 : nullptr;
    a.flags = flags ? flags + b0 : nullptr;
    a.qcount = qcount ? qcount + b0 : F.qc + b0;
    a.h_out = h_out ? h_out + b0 * g.W * g.W : nullptr;
    a.lb = F.lb; a.ub = F.ub;
    {
      ProfScope ps(p, MOCO_K_SCORE, st);
      if (small) {
        fft_dispatch(F.pc, [&](auto PC) {
          k_fft_score_rows<decltype(PC)::value><<<(unsigned)(nb * npb), FFT_THREADS, F.smem_rows, st>>>(a, sper);
        });
        k_fft_score_pick<<<(unsigned)nb, 1024, 0, st>>>(a);
      } else {
        fft_dispatch(F.pc, [&](auto PC) {
          k_fft_score<decltype(PC)::value><<<(unsigned)nb, nb < p->nsm ? 1024 : FFT_THREADS, F.smem_score, st>>>(a);
        });
      }
    }
    p->launches += small ? 6 : 4;
    CKL("fft path");
  }
  return MOCO_OK;
}

// Fused tensor-core search (kernels_tcf.cuh): levels <= 1, B tiles from the table, the
// layout fits; needs the corner-square scratch for a batch.  Failure just leaves the
// two-kernel path (k_tc_prep + k_tc_coarse).
static void tcf_setup(moco_plan *p) {
  TcPlan &tc = p->tc;
  const TcGeom &g = tc.g;
  if (p->levels > 1 || g.stg || !p->knob.tc_fused) return;
  if (!tcf_layout(g, &tc.f_smem, &tc.f_offE, &tc.f_offBars, &tc.f_nch)) return;
  if (cudaMalloc(&tc.corner, (size_t)p->cap * 4 * g.w * g.w * sizeof(u64)) != cudaSuccess) {
    cudaGetLastError();
    tc.corner = nullptr;
    return;
  }
  if (smem_attr(k_tc_fused<0>, tc.f_smem) != cudaSuccess || smem_attr(k_tc_fused<1>, tc.f_smem) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  tc.fused = true;
}

static int pipe_create(moco_plan *p) {
  // MOCO_PRIO="xyz": stream priorities of (prep, main, pick), 1 = highest, 0 = lowest (tuning)
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  const char *pr = getenv("MOCO_PRIO");
  for (int k = 0; k < 3; ++k) {
    const int pv = (pr && (int)strlen(pr) > k && pr[k] == '1') ? hi : lo;
    CK(cudaStreamCreateWithPriority(&p->ps[k], cudaStreamNonBlocking, pv));
  }
  for (int k = 0; k < 2; ++k) {
    CK(cudaEventCreateWithFlags(&p->pe_prep[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p->pe_free[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p->pe_sums[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p->pe_pick[k], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&p->pe_start, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&p->pe_end, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&p->pe_end2, cudaEventDisableTiming));
  p->pipe_ready = true;
  return MOCO_OK;
}

int moco_plan_create(moco_plan **out, int m, int n, int w, int levels, int dtype, int bits,
                     int device) {
  if (!out) return MOCO_EINVAL;
  *out = nullptr;
  if (levels < 0 || levels > 2) return MOCO_EINVAL;
  if (dtype != MOCO_U16 && dtype != MOCO_F32) return MOCO_EINVAL;
  if (dtype == MOCO_U16 && (bits < 1 || bits > 16 || bits + 2 * levels > 16)) return MOCO_EINVAL;
  if (m < (2 << levels) || n < (2 << levels)) return MOCO_EINVAL;
  const size_t e0 = dtype == MOCO_U16 ? 2 : 4;
  const int mL = m >> levels, nL = n >> levels;
  if (w < 1 || w >= std::min(mL, nL)) return MOCO_EINVAL;
  if (w > 64 && dtype != MOCO_U16) return MOCO_EINVAL;   // w > 64: FFT path only
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    snprintf(g_err, sizeof(g_err), "no CUDA device %d (count %d)", device, ndev);
    return MOCO_ECUDA;
  }
  CK(cudaSetDevice(device));
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  moco_plan *p = new (std::nothrow) moco_plan();
  if (!p) return MOCO_ENOMEM;
  p->nsm = nsm;
  p->m = m; p->n = n; p->w = w; p->W = 2 * w - 1; p->levels = levels; p->dtype = dtype;
  p->bits = dtype == MOCO_U16 ? bits : 0; p->device = device;
  {
    const char *e = getenv("MOCO_REFINE");
    p->simple_refine = e && strcmp(e, "simple") == 0;
    p->simple_level = (e && strncmp(e, "simple", 6) == 0 && e[6] >= '0' && e[6] <= '9') ? e[6] - '0' : -1;
    if (const char *v = getenv("MOCO_RTC")) p->knob.rtc = atoi(v) ? 1 : 0;
    if (const char *v = getenv("MOCO_RTC_PARTS")) p->knob.rtc_parts = std::max(0, atoi(v));
    p->knob.nofuse_ds = getenv("MOCO_NOFUSE_DS") != nullptr;
    p->knob.ga_inpick = getenv("MOCO_GA_INPICK") != nullptr;
    p->knob.nopipe = getenv("MOCO_NOPIPE") != nullptr;
    p->knob.fft_v1 = getenv("MOCO_FFT_V1") != nullptr;
    if (const char *v = getenv("MOCO_TC_FUSED")) p->knob.tc_fused = atoi(v);
    if (const char *v = getenv("MOCO_FFT_MEAN")) p->knob.fft_mean = std::min(2, std::max(0, atoi(v)));
    if (const char *v = getenv("MOCO_FRA")) p->knob.fra = atoi(v);
    if (const char *v = getenv("MOCO_PDL")) p->knob.pdl = atoi(v);
    if (const char *v = getenv("MOCO_PREP_FP")) p->knob.prep_fp = atoi(v);
    if (const char *v = getenv("MOCO_FRA_MIN")) p->knob.fra_min = std::max(1, atoi(v));
  }
  for (int l = 0; l <= levels; ++l) {
    p->ml[l] = m >> l;
    p->nl[l] = n >> l;
    p->pitch[l] = l == 0 ? round_up(n, (int)(16 / e0)) : round_up(p->nl[l], 8);
    p->esz[l] = dtype == MOCO_U16 ? 2 : (l == 0 ? 4 : 8);
  }
  // coarse kernel geometry (K3+K4d+K5)
  const int W = p->W, G = (W + KT - 1) / KT;
  p->c_sc = std::min(W, std::max(1, 4096 / W));
  p->c_br = 16;
  p->c_fpitch = round_up(p->nl[levels] + W + 2 * KT, 8);
  const int tasks = p->c_sc * G;
  p->c_threads = std::min(512, std::max(64, round_up(tasks, 32)));
  p->c_smem = coarse_smem(p, p->c_sc, p->c_br, p->c_fpitch);
  if (p->c_smem > 227 * 1024 && w <= 64) { plan_free(p); return MOCO_EINVAL; }   // (w > 64: FFT only)
  // workspace: template pyramid, tables, one batch of frame pyramid levels
  int rc = MOCO_OK;
  auto alloc = [&](void **ptr, size_t bytes) {
    if (rc != MOCO_OK) return;
    if (cudaMalloc(ptr, bytes) != cudaSuccess) { cudaGetLastError(); rc = MOCO_ENOMEM; }
  };
  for (int l = 0; l <= levels; ++l) alloc(&p->tpl[l], (size_t)p->ml[l] * p->pitch[l] * p->esz[l]);
  alloc(&p->gb, (size_t)W * W * 8);
  size_t per_frame = 0;
  for (int l = 1; l <= levels; ++l) per_frame += (size_t)p->ml[l] * p->pitch[l] * p->esz[l];
  p->stage = p->pitch[0] != n;
  if (p->stage) per_frame += (size_t)2 * m * p->pitch[0] * e0;
  // tensor-core operand planes + lag energies (upper bound: rows <= m_L + 128, int8 hi/lo)
  if (dtype == MOCO_U16) per_frame += (size_t)2 * (p->ml[levels] + 128) * p->nl[levels] + (size_t)W * W * 8;
  size_t budget = (size_t)1 << 30;   // internal batch scratch (B200: 180 GB HBM)
  if (const char *bm = getenv("MOCO_BATCH_MB")) budget = (size_t)std::max(64, atoi(bm)) << 20;   // tuning
  p->cap = per_frame ? std::max<int64_t>(1, (int64_t)(budget / per_frame)) : (int64_t)1 << 20;
  p->cap = std::min<int64_t>(p->cap, (int64_t)1 << 20);
  for (int l = 1; l <= levels; ++l)
    alloc(&p->scratch[l], (size_t)p->cap * p->ml[l] * p->pitch[l] * p->esz[l]);
  for (int l = 0; l <= levels; ++l) alloc((void **)&p->sh[l], (size_t)p->cap * 2 * sizeof(int32_t));
  if (p->stage) {
    alloc(&p->stage_in, (size_t)p->cap * m * p->pitch[0] * e0);
    alloc(&p->stage_out, (size_t)p->cap * m * p->pitch[0] * e0);
  }
  if (dtype == MOCO_U16 && levels > 0) {
    alloc((void **)&p->racc, (size_t)p->cap * 18 * sizeof(u64));
    alloc((void **)&p->racc2, (size_t)p->cap * 18 * sizeof(u64));
    alloc((void **)&p->sh1b, (size_t)p->cap * 2 * sizeof(int32_t));
    for (int k = 0; k < 2; ++k) alloc((void **)&p->gbin[k], (size_t)p->cap * 26 * sizeof(u64));
    if (levels == 2) {   // align_tc_pipelined at two levels: coarse shifts, level-1 images
      for (int k = 0; k < 2; ++k) alloc((void **)&p->sh2b[k], (size_t)p->cap * 2 * sizeof(int32_t));
      alloc(&p->scratch1b, (size_t)p->cap * p->ml[1] * p->pitch[1] * p->esz[1]);
    }
    if (rc == MOCO_OK && (cudaMemset(p->racc, 0, (size_t)p->cap * 18 * sizeof(u64)) != cudaSuccess ||
                          cudaMemset(p->racc2, 0, (size_t)p->cap * 18 * sizeof(u64)) != cudaSuccess))
      rc = MOCO_ENOMEM;
  }
  if (dtype == MOCO_U16)
    for (int l = 0; l < levels; ++l) {
      alloc((void **)&p->pb2[l], (size_t)(p->ml[l] + 1) * (p->nl[l] + 1) * sizeof(u64));
      // template-stationary refine (kernels_refine.cuh): row tiles x 256-column tiles
      // sized to about one CTA per SM, rows per tile <= RS_MAXRT; ring as deep as fits
      const int nct = (p->nl[l] + RS_CT - 1) / RS_CT;
      int nrt = std::min(p->ml[l], std::max(1, nsm / nct));
      int rt = (p->ml[l] + nrt - 1) / nrt;
      if (rt > RS_MAXRT) {
        rt = RS_MAXRT;
        nrt = (p->ml[l] + rt - 1) / rt;
      }
      p->rrt[l] = rt;
      p->rnrt[l] = nrt;
      // (ring within ~150 KB: a 37 KB operand-prep CTA of the next batch fits beside it)
      p->rstages[l] = std::min(32, (150 * 1024 - rs_smem_bytes(rt, 0)) / rs_stage_bytes(rt));
      // tensor-core refine sums (kernels_rtc.cuh) where they apply; MOCO_RTC=0 selects the
      // CUDA-core kernel (parity cross-check)
      if (p->knob.rtc != 0 && rtc_make(&p->rtc[l], p->ml[l], p->nl[l], bits + 2 * l)) {
        const size_t tb = rtc_table_bytes(p->rtc[l]);
        if (cudaMalloc((void **)&p->rtab[l], tb) != cudaSuccess ||
            (!p->rperm && (cudaMalloc((void **)&p->rperm, (size_t)p->cap * sizeof(int)) != cudaSuccess ||
                           cudaMalloc((void **)&p->rmeta, 16 * sizeof(int)) != cudaSuccess))) {
          cudaGetLastError();
          if (p->rtab[l]) cudaFree(p->rtab[l]);
          p->rtab[l] = nullptr;
        }
      }
    }
  if (rc != MOCO_OK) { plan_free(p); return rc; }
  // refine kernels' shared-memory limits, on this plan's device (function attributes are
  // per device: a process may hold plans on several GPUs)
  if (dtype == MOCO_U16 && levels > 0) {
    int smem = 0;
    bool any_rtc = false;
    for (int l = 0; l < levels; ++l) {
      smem = std::max(smem, rs_smem_bytes(p->rrt[l], p->rstages[l]));
      any_rtc = any_rtc || p->rtab[l] != nullptr;
    }
    if (smem_attr(k_refine_sums<false>, smem) != cudaSuccess ||
        smem_attr(k_refine_sums<true>, smem) != cudaSuccess ||
        (any_rtc &&
         smem_attr(k_refine_tc, RTC_SMEM) != cudaSuccess)) {
      plan_free(p);
      return set_cuda_err(cudaGetLastError(), "refine kernel attributes");
    }
  }
  // frame-resident level-0 refine + apply (kernels_fra.cuh): clusters of Q CTAs, as many
  // as can be co-resident (occupancy query with the cluster launch configuration)
  if (dtype == MOCO_U16 && levels > 0 && !p->stage && p->knob.fra &&
      fra_make(&p->fra, p->ml[0], p->nl[0], p->pitch[0], bits, 2 * (levels == 1 ? w - 1 : 2 * w - 1))) {
    if (smem_attr(k_refine_frame, p->fra.smem) == cudaSuccess &&
        cudaMalloc((void **)&p->fra_tc, fra_tcopy_bytes(p->fra, p->ml[0])) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = p->fra.Q; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(p->fra.Q * (nsm / p->fra.Q));
      cfg.blockDim = dim3(FRA_THREADS);
      cfg.dynamicSmemBytes = p->fra.smem;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, k_refine_frame, &cfg) == cudaSuccess && ncl > 0) {
        p->fra.ncl = ncl;
        p->fra_ok = true;
      }
    }
    cudaGetLastError();
  }
  p->algo = MOCO_ALGO_DIRECT;
  const bool tc_ok = tc_supported(p->dtype, p->bits, p->levels, p->w, p->ml[levels], p->nl[levels]);
  if (tc_ok && tc_auto_prefers(p->w)) {
    if (tc_init(&p->tc, p->w, p->ml[levels], p->nl[levels], levels, p->bits + 2 * levels, p->cap) == 0) {
      p->algo = MOCO_ALGO_TC;
      tcf_setup(p);
      // whole waves of the tensor-core search per internal batch (CTAs/SM x GG*F frames)
      const int64_t wave = (int64_t)nsm * p->tc.g.ctas * p->tc.g.GG * p->tc.g.F;
      // one wave per internal batch when the search is short and the batches pipeline
      // (levels > 0, N <= 192: C2 1.70 -> 1.77 M,
      // C4 399 -> 412 k; the finer batches keep the three streams busier), whole waves up
      // to the scratch budget otherwise (C3, N = 256: 985 vs 871 k with one wave)
      // (levels = 0 pipelines too, align_tc_pipelined0, in batches of one wave -- 592 frames
      // at C1 with four frames per CTA: 1.503 -> 1.524 M frames/s; with the round-1 lag
      // padding two waves of 296 frames, 1.297 -> 1.326 M; MOCO_PIPE0_WAVES=0 one batch per call)
      int64_t wv0 = 1;
      if (const char *v = getenv("MOCO_PIPE0_WAVES")) wv0 = std::max<int64_t>(0, atoi(v));   // 0: off
      if (p->cap >= wave)
        p->cap = (p->tc.g.N <= 192 && (levels > 0 || wv0 > 0) ? (levels > 0 ? 1 : wv0) : p->cap / wave) * wave;
      if (const char *bw = getenv("MOCO_BATCH_WAVES"))   // tuning: waves per internal batch
        p->cap = std::min<int64_t>(p->cap, std::max(1, atoi(bw)) * wave);
    } else {
      cudaGetLastError();
    }
  }
  if (p->algo == MOCO_ALGO_DIRECT && fft_supported(p) && (w > 64 || fft_auto_prefers(p->w, tc_ok))) {
    if (fft_init(p) == MOCO_OK) p->algo = MOCO_ALGO_FFT;
    else cudaGetLastError();
  } else if (p->algo == MOCO_ALGO_TC && fft_supported(p)) {
    if (fft_init(p) != MOCO_OK) cudaGetLastError();   // latency route for small calls (optional)
  }
  if (w > 64 && p->algo != MOCO_ALGO_FFT) { plan_free(p); return MOCO_EINVAL; }
  // streams and events of the batch pipeline (align_tc_pipelined) are created here, so
  // that moco_align_batch never allocates (moco.h) and can be captured in a CUDA graph
  if (dtype == MOCO_U16 && (levels > 0 || p->algo == MOCO_ALGO_TC)) {
    const int prc = pipe_create(p);
    if (prc) { plan_free(p); return prc; }
  }
  *out = p;
  return MOCO_OK;
}

int moco_plan_set_algo(moco_plan *p, int algo) {
  if (!p) return MOCO_EINVAL;
  if (algo == MOCO_ALGO_DIRECT) {
    if (p->w > 64) return MOCO_EINVAL;
    p->algo = algo;
    return MOCO_OK;
  }
  if (algo == MOCO_ALGO_FFT) {
    if (!fft_supported(p)) return MOCO_EINVAL;
    CK(cudaSetDevice(p->device));
    int rc = fft_init(p);
    if (rc) return rc;
    if (p->has_tpl && !p->fft.tpl_ready) {
      rc = fft_set_template(p, 0);
      if (rc) return rc;
      CK(cudaDeviceSynchronize());
    }
    p->algo = MOCO_ALGO_FFT;
    return MOCO_OK;
  }
  const int L = p->levels;
  if (algo == MOCO_ALGO_TC || algo == MOCO_ALGO_AUTO) {
    const bool ok = tc_supported(p->dtype, p->bits, L, p->w, p->ml[L], p->nl[L]);
    if (algo == MOCO_ALGO_AUTO && !(ok && tc_auto_prefers(p->w))) {
      if (fft_supported(p) && (p->w > 64 || fft_auto_prefers(p->w, ok))) return moco_plan_set_algo(p, MOCO_ALGO_FFT);
      return moco_plan_set_algo(p, MOCO_ALGO_DIRECT);
    }
    if (!ok) return MOCO_EINVAL;
    CK(cudaSetDevice(p->device));
    if (!p->tc.ready && tc_init(&p->tc, p->w, p->ml[L], p->nl[L], L, p->bits + 2 * L, p->cap) != 0) return MOCO_ENOMEM;
    if (p->has_tpl && !p->tc.tpl_ready) {
      if (tc_set_template(&p->tc, (const uint16_t *)p->tpl[L], p->pitch[L], 0) != 0)
        return set_cuda_err(cudaGetLastError(), "tc_set_template");
      CK(cudaDeviceSynchronize());
    }
    p->algo = MOCO_ALGO_TC;
    p->algo_forced = algo == MOCO_ALGO_TC;
    return MOCO_OK;
  }
  return MOCO_EINVAL;
}

int moco_plan_get_algo(const moco_plan *p) { return p ? p->algo : MOCO_EINVAL; }

int moco_profile_enable(moco_plan *p, int on) {
  if (!p) return MOCO_EINVAL;
  p->prof_on = on != 0;
  return MOCO_OK;
}

int moco_profile_read(moco_plan *p, double *ms, int64_t *launches, int n) {
  if (!p || n < 0 || (n > 0 && (!ms || !launches))) return MOCO_EINVAL;
  for (int k = 0; k < n; ++k) { ms[k] = 0; launches[k] = 0; }
  for (auto &r : p->prof_live) {
    CK(cudaEventSynchronize(r.b));
    float t = 0;
    CK(cudaEventElapsedTime(&t, r.a, r.b));
    if (r.kind < n) { ms[r.kind] += t; launches[r.kind] += 1; }
    p->prof_pool.push_back(r.a);
    p->prof_pool.push_back(r.b);
  }
  p->prof_live.clear();
  return MOCO_OK;
}

int moco_plan_destroy(moco_plan *p) {
  if (!p) return MOCO_OK;
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  plan_free(p);
  return MOCO_OK;
}

static int grid_for(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

// K1: level l -> l+1 for `B` frames.  src/dst are level images with the
// plan's pitch/fstride conventions.
static int launch_downsample(moco_plan *p, int l, const void *src, int64_t src_fstride, void *dst,
                             int64_t B, cudaStream_t st) {
  const int mi = p->ml[l], ni = p->nl[l], mo = p->ml[l + 1], no = p->nl[l + 1];
  const int64_t dst_fstride = (int64_t)mo * p->pitch[l + 1];
  ProfScope ps(p, MOCO_K_DOWNSAMPLE, st);
  if (p->dtype == MOCO_U16) {
    const int64_t work = B * mo * ((no + 3) / 4);
    k_downsample_u16<<<grid_for(work, 256), 256, 0, st>>>(
        (const uint16_t *)src, src_fstride, p->pitch[l], mi, ni, (uint16_t *)dst, dst_fstride,
        p->pitch[l + 1], mo, no, (int)B);
  } else if (l == 0) {
    k_downsample_mean<float><<<grid_for(B * mo * no, 256), 256, 0, st>>>(
        (const float *)src, src_fstride, p->pitch[l], mi, ni, (double *)dst, dst_fstride,
        p->pitch[l + 1], mo, no, (int)B);
  } else {
    k_downsample_mean<double><<<grid_for(B * mo * no, 256), 256, 0, st>>>(
        (const double *)src, src_fstride, p->pitch[l], mi, ni, (double *)dst, dst_fstride,
        p->pitch[l + 1], mo, no, (int)B);
  }
  p->launches++;
  CKL("k_downsample");
  return MOCO_OK;
}

template <class In, bool WIDE>
static int launch_coarse_t(moco_plan *p, const CoarseArgs &a, cudaStream_t st) {
  static bool attr_done[8] = {false};   // per-device attribute is set once per process
  (void)attr_done;
  CK(smem_attr(k_coarse<In, WIDE>, (int)p->c_smem));
  ProfScope ps(p, MOCO_K_COARSE, st);
  k_coarse<In, WIDE><<<a.B, p->c_threads, p->c_smem, st>>>(a);
  p->launches++;
  CKL("k_coarse");
  return MOCO_OK;
}

static int launch_coarse(moco_plan *p, const void *img, int64_t fstride, int pitch, int64_t B,
                         int32_t *shift_out, double *f_out, double *grid_out, uint8_t *flags,
                         cudaStream_t st) {
  const int L = p->levels;
  CoarseArgs a;
  a.frames = img; a.fstride = fstride; a.pitch = pitch;
  a.tpl = p->tpl[L]; a.tpitch = p->pitch[L];
  a.gb = p->gb;
  a.mc = p->ml[L]; a.nc = p->nl[L]; a.w = p->w;
  a.scale = p->dtype == MOCO_U16 ? (double)(1u << (4 * L)) : 1.0;
  a.B = (int)B; a.br = p->c_br; a.sc = p->c_sc; a.fpitch = p->c_fpitch;
  a.shift_out = shift_out; a.f_out = f_out; a.grid_out = grid_out; a.flags = flags;
  if (p->dtype == MOCO_U16) {
    if (p->bits + 2 * L <= 14) return launch_coarse_t<uint16_t, false>(p, a, st);
    return launch_coarse_t<uint16_t, true>(p, a, st);
  }
  if (L == 0) return launch_coarse_t<float, false>(p, a, st);
  return launch_coarse_t<double, false>(p, a, st);
}

static int launch_refine(moco_plan *p, int l, const void *img, int64_t fstride, int64_t B,
                         const int32_t *sin, int32_t *sout, double *fout, cudaStream_t st) {
  RefineArgs a;
  a.frames = img; a.fstride = fstride; a.pitch = p->pitch[l];
  a.tpl = p->tpl[l]; a.tpitch = p->pitch[l];
  a.ml = p->ml[l]; a.nl = p->nl[l];
  a.scale = p->dtype == MOCO_U16 ? (double)(1u << (4 * l)) : 1.0;
  a.B = (int)B; a.shift_in = sin; a.shift_out = sout; a.f_out = fout;
  ProfScope ps(p, MOCO_K_REFINE, st);
  if (p->dtype == MOCO_U16) k_refine<uint16_t><<<(unsigned)B, 256, 0, st>>>(a);
  else if (l == 0) k_refine<float><<<(unsigned)B, 256, 0, st>>>(a);
  else k_refine<double><<<(unsigned)B, 256, 0, st>>>(a);
  p->launches++;
  CKL("k_refine");
  return MOCO_OK;
}

// K6 (+K7 at level 0): template-stationary u16 refine (kernels_refine.cuh):
// k_refine_sums (per-frame sums) then k_refine_pick (argmin + apply).
// the tensor-core refine sums serve batches of >= 256 frames (the CUDA-core kernel's 148
// template tiles spread small ones better; MOCO_RTC=1 forces it at any size: parity tests)
static bool use_rtc(const moco_plan *p, int l, int64_t B) {
  return p->rtab[l] != nullptr && (B >= 256 || p->knob.rtc == 1);
}

// GA pieces of a batch (k_ga_pieces) for the tensor-core refine at level l.
static int launch_ga_pieces(moco_plan *p, int l, const void *img, int64_t fstride, int64_t B, const int32_t *sin,
                            u64 *out, cudaStream_t st) {
  RefinePickArgs b{};
  b.frames = (const uint16_t *)img; b.fstride = fstride; b.pitch = p->pitch[l];
  b.ml = p->ml[l]; b.nl = p->nl[l]; b.B = (int)B; b.shift_in = sin;
  b.ga_total = 1; b.kw = 16 * p->rtc[l].nk;
  {
    ProfScope ps(p, MOCO_K_APPLY, st);
    k_ga_pieces<<<(unsigned)B, 128, 0, st>>>(b, out);
  }
  p->launches++;
  CKL("k_ga_pieces");
  return MOCO_OK;
}

static int launch_refine_h(moco_plan *p, int l, const void *img, int64_t fstride, int64_t B,
                           const int32_t *sin, int32_t *sout, double *fout, void *corr, cudaStream_t st,
                           u64 *racc = nullptr, cudaStream_t st_pick = nullptr, cudaEvent_t ev_sums = nullptr,
                           const u64 *gbin = nullptr) {
  const int vb = p->bits + 2 * l;
  if (!racc) racc = p->racc;
  RefineSumArgs a;
  a.tpl = (const uint16_t *)p->tpl[l]; a.tpitch = p->pitch[l];
  a.ml = p->ml[l]; a.nl = p->nl[l];
  a.B = (int)B; a.shift_in = sin; a.acc = racc;
  a.rt = p->rrt[l]; a.nrt = p->rnrt[l]; a.stages = p->rstages[l];
  // 32-bit lane partials hold (256-column halves) x rt rows x 8 products, each
  // <= (2^vb - 1)^2, unless flushed to 64 bits after every row
  {
    const double halves = (double)((std::min(a.nl, RS_CT) + 255) / 256);
    const double mx = (std::ldexp(1.0, vb) - 1.0) * (std::ldexp(1.0, vb) - 1.0);
    a.wide = halves * a.rt * 8.0 * mx >= 4294967296.0 ? 1 : 0;
  }
  CUtensorMap tmF;
  // the tensor-core kernel parallelises over 16-frame groups: small batches (the closed
  // loop) keep the CUDA-core kernel, whose 148 template tiles spread even one frame
  // (MOCO_RTC=1 forces the tensor-core kernel at any size: parity tests)
  const bool rtc = use_rtc(p, l, B);
  if (rtc ? !tmap_u16_sw128(&tmF, img, a.nl, a.ml, B, p->pitch[l], fstride, RTC_R)
          : !tmap_u16_3d(&tmF, img, a.nl, a.ml, B, p->pitch[l], fstride, RS_BOX, a.rt + 2)) {
    snprintf(g_err, sizeof(g_err), "cuTensorMapEncodeTiled failed (refine level %d)", l);
    return MOCO_ECUDA;
  }
  RefinePickArgs b;
  b.frames = (const uint16_t *)img; b.fstride = fstride; b.pitch = p->pitch[l];
  b.pb2 = p->pb2[l]; b.ml = p->ml[l]; b.nl = p->nl[l];
  b.scale = (double)(1u << (4 * l));
  b.B = (int)B; b.shift_in = sin; b.acc = racc; b.shift_out = sout; b.f_out = fout;
  b.corrected = (uint16_t *)corr;
  // small batches: several CTAs per frame for the apply (the accumulators are then
  // cleared by a memset after the pick instead of by the single CTA)
  b.parts = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(16, p->ml[l] / 4), p->nsm / std::max<int64_t>(1, B)));
  if (!corr) b.parts = 1;
  b.ga_total = 0;
  b.kw = 0;
  b.gbin = nullptr;
  if (rtc) {
    ProfScope ps(p, MOCO_K_REFINE, st);
    k_rtc_bucket<<<1, 1024, 0, st>>>(sin, (int)B, p->rperm, p->rmeta);
    RtcArgs r;
    r.tab = p->rtab[l]; r.acc = racc; r.shift_in = sin; r.perm = p->rperm; r.meta = p->rmeta;
    r.B = (int)B; r.g = p->rtc[l];
    b.ga_total = RTC_GA_TOTAL;   // the pick completes GA from the staged-pixel total
    b.kw = 16 * p->rtc[l].nk;
    b.gbin = gbin;
    // row-group ranges per 16-frame group (whole stages): the fewest that bring the last
    // wave near full
    const int64_t groups = (B + RTC_F - 1) / RTC_F + 4;   // upper bound over the 4 classes
    const int nblk = (p->rtc[l].ng + RTC_RG - 1) / RTC_RG;
    int best = 1;
    double bestc = 1e30;
    for (int parts = 1; parts <= 16 && parts <= nblk; ++parts) {
      // waves x CTA time; a CTA's fixed part (TMEM, barriers, epilogue) measured at about
      // 8 % of a whole frame group's stages (C2)
      const double waves = std::ceil((double)(groups * parts) / p->nsm);
      const double cost = waves * (0.08 + 1.0 / parts);
      if (cost < bestc) { bestc = cost; best = parts; }
    }
    if (p->knob.rtc_parts) best = std::min(nblk, p->knob.rtc_parts);   // tuning
    r.groups_per_part = (nblk + best - 1) / best * RTC_RG;
    r.parts = (p->rtc[l].ng + r.groups_per_part - 1) / r.groups_per_part;
    k_refine_tc<<<(unsigned)(groups * r.parts), RTC_THREADS, RTC_SMEM, st>>>(tmF, r);
  } else {
    ProfScope ps(p, MOCO_K_REFINE, st);
    const int smem = rs_smem_bytes(a.rt, a.stages);
    const int nct = (a.nl + RS_CT - 1) / RS_CT;
    if (a.wide) launchk(p->pdl_now, k_refine_sums<true>, (unsigned)(a.nrt * nct), RS_THREADS, smem, st, tmF, a);
    else launchk(p->pdl_now, k_refine_sums<false>, (unsigned)(a.nrt * nct), RS_THREADS, smem, st, tmF, a);
  }
  p->launches++;
  CKL(rtc ? "k_refine_tc" : "k_refine_sums");
  if (st_pick) {   // pick/apply on another stream (align_tc_pipelined)
    CK(cudaEventRecord(ev_sums, st));
    CK(cudaStreamWaitEvent(st_pick, ev_sums, 0));
    st = st_pick;
  }
  {
    ProfScope ps(p, MOCO_K_APPLY, st);
    launchk(p->pdl_now && !st_pick, k_refine_pick, (unsigned)(B * b.parts), 256, 0, st, b);
  }
  p->launches++;
  CKL("k_refine_pick");
  if (b.parts > 1) CK(cudaMemsetAsync(racc, 0, (size_t)B * 18 * sizeof(u64), st));
  return MOCO_OK;
}

static bool fused_ok(const moco_plan *p, int l) {
  if (p->simple_refine || p->simple_level == l || p->dtype != MOCO_U16) return false;
  // 32-bit partial sums: one template row adds 8 products (or one 8-square window sum)
  const double dmax = (double)((1u << (p->bits + 2 * l)) - 1);
  if (8.0 * dmax * dmax >= 2147483648.0) return false;   // one row's 8 products in 32 bits
  return p->nl[l] % 8 == 0 && p->rstages[l] >= 2 && p->racc;
}

static int launch_apply(moco_plan *p, const void *in, void *out, const int32_t *sh, int64_t B,
                        cudaStream_t st) {
  ProfScope ps(p, MOCO_K_APPLY, st);
  if (p->dtype == MOCO_U16) {
    const int64_t work = B * p->m * (p->pitch[0] / 8);
    k_apply<uint16_t><<<grid_for(work, 256), 256, 0, st>>>((const uint16_t *)in, (uint16_t *)out,
                                                           p->m, p->n, p->pitch[0], sh, (int)B);
  } else {
    const int64_t work = B * p->m * (p->pitch[0] / 4);
    k_apply<float><<<grid_for(work, 256), 256, 0, st>>>((const float *)in, (float *)out, p->m,
                                                        p->n, p->pitch[0], sh, (int)B);
  }
  p->launches++;
  CKL("k_apply");
  return MOCO_OK;
}

int moco_set_template(moco_plan *p, const void *d_template, moco_stream_t stream) {
  if (!p || !d_template) return MOCO_EINVAL;
  CK(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t row0 = (size_t)p->n * p->esz[0];
  CK(cudaMemcpy2DAsync(p->tpl[0], (size_t)p->pitch[0] * p->esz[0], d_template, row0, row0, p->m,
                       cudaMemcpyDeviceToDevice, st));
  for (int l = 0; l < p->levels; ++l) {
    int rc = launch_downsample(p, l, p->tpl[l], 0, p->tpl[l + 1], 1, st);
    if (rc) return rc;
  }
  const int L = p->levels;
  const int esm = (4 * (p->w - 1) + p->w * p->w + 1) * 8;   // k_energy_u16_t shared memory
  if (p->dtype == MOCO_U16 && p->w - 1 <= 248) {   // g_b by the strip/corner DP of P:33-35, one block
    CK(smem_attr(k_energy_u16_t<true>, esm));
    CK(smem_attr(k_energy_u16_t<false>, esm));
    k_energy_u16_t<true><<<1, 1024, esm, st>>>((const uint16_t *)p->tpl[L], 0, p->pitch[L], p->ml[L], p->nl[L], p->w,
                                               (u64 *)p->gb, nullptr, 1);
  } else if (p->dtype == MOCO_U16)
    k_template_energy<uint16_t><<<p->W * p->W, 256, 0, st>>>(
        (const uint16_t *)p->tpl[L], p->pitch[L], p->ml[L], p->nl[L], p->w, (u64 *)p->gb);
  else if (L == 0)
    k_template_energy<float><<<p->W * p->W, 256, 0, st>>>(
        (const float *)p->tpl[L], p->pitch[L], p->ml[L], p->nl[L], p->w, (double *)p->gb);
  else
    k_template_energy<double><<<p->W * p->W, 256, 0, st>>>(
        (const double *)p->tpl[L], p->pitch[L], p->ml[L], p->nl[L], p->w, (double *)p->gb);
  CKL("k_template_energy");
  if (p->dtype == MOCO_U16)
    for (int l = 0; l < L; ++l) {
      k_prefix2d_rows<<<(p->ml[l] + 8) / 8, 256, 0, st>>>((const uint16_t *)p->tpl[l], p->pitch[l],
                                                               p->ml[l], p->nl[l], p->pb2[l]);
      k_prefix2d_cols<<<(p->nl[l] + 32) / 32, 32 * PF_SEG, 0, st>>>(p->ml[l], p->nl[l], p->pb2[l]);
      CKL("k_prefix2d");
      if (p->rtab[l]) {
        k_rtc_table<<<1024, 256, 0, st>>>((const uint16_t *)p->tpl[l], p->pitch[l], p->ml[l], p->nl[l],
                                          p->rtc[l].ng, p->rtc[l].nk, p->rtab[l]);
        CKL("k_rtc_table");
      }
    }
  if (p->fra_ok) {
    k_fra_tcopy<<<1024, 256, 0, st>>>((const uint16_t *)p->tpl[0], p->pitch[0], p->ml[0], p->nl[0], p->fra.m,
                                      p->fra.WT, p->fra_tc);
    CKL("k_fra_tcopy");
  }
  if (p->tc.ready) {
    if (tc_set_template(&p->tc, (const uint16_t *)p->tpl[L], p->pitch[L], st) != 0)
      return set_cuda_err(cudaGetLastError(), "tc_set_template");
  }
  if (p->fft.ready) {
    const int rc = fft_set_template(p, st);
    if (rc) return rc;
  }
  p->has_tpl = true;
  return MOCO_OK;
}

static int check_align_args(moco_plan *p, const void *frames, int64_t T) {
  if (!p || T < 0) return MOCO_EINVAL;
  if (T > 0 && !frames) return MOCO_EINVAL;
  if (((uintptr_t)frames & 15) != 0) return MOCO_EINVAL;
  if (!p->has_tpl) return MOCO_ESTATE;
  return MOCO_OK;
}

// Tensor-core coarse search (kernels_tc.cuh) straight from the level-0 frames:
// K_prep (operand planes G + lag energies ga) then K_tc.
// levels = 2: the operand preparation also writes the level-1 image (the refine at level
// 1 reads it) when the level-2 band covers it exactly
static bool prep_emits_l1(const moco_plan *p) {
  if (p->levels != 2 || p->dtype != MOCO_U16 || p->knob.nofuse_ds) return false;
  return p->ml[1] == 2 * p->ml[2] && p->nl[1] == 2 * p->nl[2] && p->nl[2] % 8 == 0 && p->pitch[1] % 8 == 0;
}

static int launch_tc_prep(moco_plan *p, const void *frames_b, int64_t B, uint8_t *G, u64 *ga, cudaStream_t st,
                          void *img1 = nullptr) {
  const TcGeom &g = p->tc.g;
  const int64_t groups = (B + g.F - 1) / g.F;
  TcPrepArgs pa;
  pa.frames = (const uint16_t *)frames_b; pa.fstride = (int64_t)p->m * p->n; pa.n = p->n;
  pa.B = (int)B; pa.g = g; pa.G = G; pa.ga = ga;
  // one frame per CTA (MOCO_PREP_FP=1): the CTA's shared memory then fits in what the
  // search kernel leaves free on its SM, so the prep of the next batch can co-run with it
  pa.fp = p->knob.prep_fp == 1 ? 1 : g.F;
  const int psm = pa.fp == 1 ? g.prep_smem1 : g.prep_smem;
  const unsigned pgrid = (unsigned)(groups * g.F / pa.fp);
  pa.img1 = (uint16_t *)img1; pa.fs1 = (int64_t)p->ml[1] * p->pitch[1]; pa.p1 = p->pitch[1];
  {
    ProfScope ps(p, MOCO_K_PREP, st);
    if (p->levels == 0) k_tc_prep<0><<<pgrid, 256, psm, st>>>(pa);
    else if (p->levels == 1) k_tc_prep<1><<<pgrid, 256, psm, st>>>(pa);
    else k_tc_prep<2><<<pgrid, 256, psm, st>>>(pa);
  }
  p->launches++;
  CKL("k_tc_prep");
  return MOCO_OK;
}

static int launch_tc_coarse(moco_plan *p, int64_t B, const uint8_t *G, const u64 *ga, int32_t *shift_out,
                            double *f_out, uint8_t *flags, double *grid_out, cudaStream_t st) {
  const TcGeom &g = p->tc.g;
  const int64_t groups = (B + g.F - 1) / g.F;
  TcArgs ta;
  ta.G = G; ta.T8 = p->tc.T8; ta.Btab = p->tc.Btab; ta.ga = ga; ta.gb = (const u64 *)p->gb; ta.g = g;
  ta.scale = (double)(1u << (4 * p->levels)); ta.B = (int)B;
  ta.shift_out = shift_out; ta.f_out = f_out; ta.flags = flags; ta.grid_out = grid_out;
  {
    ProfScope ps(p, MOCO_K_COARSE, st);
    const unsigned grid = (unsigned)((groups + g.GG - 1) / g.GG);
    switch (g.N / 16) {   // chunks per producer lane = 2N/32 (N = 128 / 192 / 256 for C2 / C1 / C3)
      case 2: k_tc_coarse<2><<<grid, TC_THREADS, g.smem, st>>>(ta); break;
      case 4: k_tc_coarse<4><<<grid, TC_THREADS, g.smem, st>>>(ta); break;
      case 10: k_tc_coarse<10><<<grid, TC_THREADS, g.smem, st>>>(ta); break;
      case 14: k_tc_coarse<14><<<grid, TC_THREADS, g.smem, st>>>(ta); break;
      case 6: k_tc_coarse<6><<<grid, TC_THREADS, g.smem, st>>>(ta); break;
      case 8: k_tc_coarse<8><<<grid, TC_THREADS, g.smem, st>>>(ta); break;
      case 12: k_tc_coarse<12><<<grid, TC_THREADS, g.smem, st>>>(ta); break;
      default: k_tc_coarse<16><<<grid, TC_THREADS, g.smem, st>>>(ta); break;
    }
  }
  p->launches++;
  CKL("k_tc_coarse");
  return MOCO_OK;
}

// The fused search (k_tc_fused) on B level-0 frames with row pitch n.
static int launch_tc_fused(moco_plan *p, const void *frames_b, int64_t B, int32_t *shift_out, double *f_out,
                           uint8_t *flags, double *grid_out, cudaStream_t st) {
  const TcPlan &tc = p->tc;
  const TcGeom &g = tc.g;
  const int64_t groups = (B + g.F - 1) / g.F;
  TcfArgs fa;
  fa.t.G = nullptr; fa.t.T8 = tc.T8; fa.t.Btab = tc.Btab; fa.t.ga = nullptr; fa.t.gb = (const u64 *)p->gb;
  fa.t.g = g; fa.t.scale = (double)(1u << (4 * p->levels)); fa.t.B = (int)B;
  fa.t.shift_out = shift_out; fa.t.f_out = f_out; fa.t.flags = flags; fa.t.grid_out = grid_out;
  fa.frames = (const uint16_t *)frames_b; fa.fstride = (int64_t)p->m * p->n; fa.n = p->n;
  fa.corner = tc.corner; fa.offE = tc.f_offE; fa.offBars = tc.f_offBars; fa.nch = tc.f_nch;
  {
    ProfScope ps(p, MOCO_K_COARSE, st);
    const unsigned grid = (unsigned)((groups + g.GG - 1) / g.GG);
    if (p->levels == 0) k_tc_fused<0><<<grid, TC_THREADS, tc.f_smem, st>>>(fa);
    else k_tc_fused<1><<<grid, TC_THREADS, tc.f_smem, st>>>(fa);
  }
  p->launches++;
  CKL("k_tc_fused");
  return MOCO_OK;
}

static int launch_tc(moco_plan *p, const void *frames_b, int64_t B, int32_t *shift_out, double *f_out,
                     uint8_t *flags, double *grid_out, cudaStream_t st, void *img1 = nullptr) {
  if (p->tc.fused && !img1) return launch_tc_fused(p, frames_b, B, shift_out, f_out, flags, grid_out, st);
  int rc = launch_tc_prep(p, frames_b, B, p->tc.G, p->tc.ga, st, img1);
  if (rc) return rc;
  return launch_tc_coarse(p, B, p->tc.G, p->tc.ga, shift_out, f_out, flags, grid_out, st);
}

// Level-0 refine + pick + apply with the frame resident in a thread-block cluster.
static bool use_fra(const moco_plan *p, int l, int64_t B) {
  return l == 0 && p->fra_ok && B >= p->knob.fra_min && fused_ok(p, 0);
}

static int launch_fra(moco_plan *p, const void *img, int64_t fstride, int64_t B, const int32_t *sin, int32_t *sout,
                      double *fout, void *corr, cudaStream_t st) {
  FraArgs a;
  a.frames = (const uint16_t *)img; a.fstride = fstride; a.pitch = p->pitch[0];
  a.tcopy = p->fra_tc;
  a.pb2 = p->pb2[0]; a.ml = p->ml[0]; a.nl = p->nl[0]; a.scale = 1.0;
  a.B = (int)B; a.shift_in = sin; a.shift_out = sout; a.f_out = fout;
  a.corrected = (uint16_t *)corr;
  a.g = p->fra;
  a.g.ncl = (int)std::min<int64_t>(p->fra.ncl, B);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p->fra.Q; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)(a.g.ncl * p->fra.Q));
  cfg.blockDim = dim3(FRA_THREADS);
  cfg.dynamicSmemBytes = p->fra.smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  {
    ProfScope ps(p, MOCO_K_APPLY, st);
    CK(cudaLaunchKernelEx(&cfg, k_refine_frame, a));
  }
  p->launches++;
  CKL("k_refine_frame");
  return MOCO_OK;
}

// S5 refine at levels L-1..0, then S6 apply (fused into the level-0 refine when possible).
static int refine_levels(moco_plan *p, const void *const *img, const int64_t *fstride, int64_t B,
                         int32_t *shifts_b, double *fmin_b, void *corr_b, cudaStream_t st) {
  const int L = p->levels;
  if (L == 0) return corr_b ? launch_apply(p, img[0], corr_b, shifts_b, B, st) : MOCO_OK;
  for (int l = L - 1; l >= 0; --l) {
    int32_t *so = l == 0 ? shifts_b : p->sh[l];
    double *fo = l == 0 ? fmin_b : nullptr;
    int rc;
    if (use_fra(p, l, B))
      rc = launch_fra(p, img[0], fstride[0], B, p->sh[1], so, fo, corr_b, st);
    else if (fused_ok(p, l))
      rc = launch_refine_h(p, l, img[l], fstride[l], B, p->sh[l + 1], so, fo, l == 0 ? corr_b : nullptr, st);
    else
      rc = launch_refine(p, l, img[l], fstride[l], B, p->sh[l + 1], so, fo, st);
    if (rc) return rc;
  }
  if (corr_b && !fused_ok(p, 0)) return launch_apply(p, img[0], corr_b, shifts_b, B, st);
  return MOCO_OK;
}

// One internal batch [f0, f0+B) of device frames.
static int run_batch(moco_plan *p, const void *frames_b, int64_t B, int32_t *shifts_b,
                     double *fmin_b, void *corr_b, uint8_t *flags_b, double *grid_b,
                     cudaStream_t st) {
  const int L = p->levels;
  const void *img[3];
  int64_t fstride[3];
  img[0] = frames_b;
  fstride[0] = (int64_t)p->m * p->pitch[0];
  for (int l = 1; l <= L; ++l) {
    img[l] = p->scratch[l];
    fstride[l] = (int64_t)p->ml[l] * p->pitch[l];
  }
  const bool tc = p->algo == MOCO_ALGO_TC;
  // the FFT row kernel of kernels_fft2.cuh reads the level-0 frames (and writes level 1)
  const bool fft2 = p->algo == MOCO_ALGO_FFT && p->fft.v2 && !grid_b && p->dtype == MOCO_U16;
  if (fft2) {
    // levels = 2: the level-1 images (the level-1 refine reads them) feed the FFT rows
    if (L == 2) {
      int rc = launch_downsample(p, 0, frames_b, fstride[0], p->scratch[1], B, st);
      if (rc) return rc;
    }
    int rc = launch_fft2(p, img[L == 2 ? 1 : 0], fstride[L == 2 ? 1 : 0], p->pitch[L == 2 ? 1 : 0], B,
                         L == 0 ? shifts_b : p->sh[L], L == 0 ? fmin_b : nullptr, flags_b, st);
    if (rc) return rc;
    return refine_levels(p, img, fstride, B, shifts_b, fmin_b, corr_b, st);
  }
  // the tensor-core search block-sums the level-0 frames itself; only the levels the
  // refine steps read (1..L-1) are materialised
  const bool emit1 = tc && !grid_b && prep_emits_l1(p);   // level 1 written by the operand prep
  for (int l = 0; l < (tc ? L - 1 : L); ++l) {
    if (emit1) break;
    int rc = launch_downsample(p, l, img[l], fstride[l], p->scratch[l + 1], B, st);
    if (rc) return rc;
  }
  if (tc) {
    int rc = grid_b ? launch_tc(p, frames_b, B, nullptr, nullptr, nullptr, grid_b, st)
                    : launch_tc(p, frames_b, B, L == 0 ? shifts_b : p->sh[L], L == 0 ? fmin_b : nullptr,
                                flags_b, nullptr, st, emit1 ? p->scratch[1] : nullptr);
    if (rc || grid_b) return rc;
    return refine_levels(p, img, fstride, B, shifts_b, fmin_b, corr_b, st);
  }
  if (grid_b) {
    if (p->w > 64) return MOCO_EINVAL;   // no exact all-lag path for w > 64
    return launch_coarse(p, img[L], fstride[L], p->pitch[L], B, nullptr, nullptr, grid_b, nullptr, st);
  }
  if (p->algo == MOCO_ALGO_FFT) {
    int rc = launch_fft(p, img[L], fstride[L], p->pitch[L], B, L == 0 ? shifts_b : p->sh[L],
                        L == 0 ? fmin_b : nullptr, flags_b, st);
    if (rc) return rc;
    return refine_levels(p, img, fstride, B, shifts_b, fmin_b, corr_b, st);
  }
  int32_t *sc_out = L == 0 ? shifts_b : p->sh[L];
  int rc = launch_coarse(p, img[L], fstride[L], p->pitch[L], B, sc_out, L == 0 ? fmin_b : nullptr,
                         nullptr, flags_b, st);
  if (rc) return rc;
  return refine_levels(p, img, fstride, B, shifts_b, fmin_b, corr_b, st);
}

// run_batch on caller frames with unpadded rows: plans whose rows are not a multiple of
// 16 bytes (p->stage) copy the batch into the padded-pitch staging buffer first and the
// corrected frames back out (stream-ordered 2-D copies); otherwise a plain run_batch.
static const void *stage_frames(moco_plan *p, const void *frames_b, int64_t B, cudaStream_t st, int *rc) {
  *rc = MOCO_OK;
  if (!p->stage) return frames_b;
  const size_t row = (size_t)p->n * p->esz[0], dpitch = (size_t)p->pitch[0] * p->esz[0];
  cudaError_t e = cudaMemcpy2DAsync(p->stage_in, dpitch, frames_b, row, row, (size_t)B * p->m,
                                    cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) *rc = set_cuda_err(e, "stage frames in");
  return p->stage_in;
}

static int run_batch_user(moco_plan *p, const void *frames_b, int64_t B, int32_t *shifts_b, double *fmin_b,
                          void *corr_b, uint8_t *flags_b, double *grid_b, cudaStream_t st) {
  int rc;
  const void *src = stage_frames(p, frames_b, B, st, &rc);
  if (rc) return rc;
  rc = run_batch(p, src, B, shifts_b, fmin_b, (p->stage && corr_b) ? p->stage_out : corr_b, flags_b, grid_b, st);
  if (rc || !p->stage || !corr_b) return rc;
  const size_t row = (size_t)p->n * p->esz[0], spitch = (size_t)p->pitch[0] * p->esz[0];
  CK(cudaMemcpy2DAsync(corr_b, row, p->stage_out, spitch, row, (size_t)B * p->m, cudaMemcpyDeviceToDevice, st));
  return MOCO_OK;
}

// Several internal batches on the tensor-core path (levels = 1): the HBM-bound operand
// preparation of batch k+1 runs on a second stream into the other G/ga buffer while the
// tensor-core search, refine and apply of batch k run on the main stream, so the
// memory-bound and the compute-bound kernels share the SMs.  Stream-ordered with respect
// to the caller's stream on entry and exit.
constexpr int64_t LAT_T = 16;   // calls with at most this many frames take the latency route

static int align_tc_pipelined(moco_plan *p, const void *d_frames, int64_t T, int32_t *d_shifts, double *d_fmin,
                              void *d_corrected, uint8_t *d_flags, cudaStream_t user) {
  if (!p->pipe_ready) return MOCO_ESTATE;   // created by moco_plan_create
  // prep stream | main stream (TC search, refine sums) | pick/apply stream.  Per batch
  // parity: operand planes G/ga, coarse shifts and refine accumulators are double-
  // buffered; a buffer is reused two batches later, after the events below.
  cudaStream_t sp = p->ps[0], sm = p->ps[1], sa = p->ps[2];
  CK(cudaEventRecord(p->pe_start, user));
  for (int k = 0; k < 3; ++k) CK(cudaStreamWaitEvent(p->ps[k], p->pe_start, 0));
  const size_t fbytes = (size_t)p->m * p->n * p->esz[0];
  uint8_t *G[2] = {p->tc.G, p->tc.G2};
  u64 *ga[2] = {p->tc.ga, p->tc.ga2};
  int32_t *sh1[2] = {p->sh[1], p->sh1b};
  u64 *racc[2] = {p->racc, p->racc2};
  // levels = 2: the coarse search lands at level 2 (sh2b), the level-1 image of the batch
  // is downsampled on the prep stream (scratch[1] / scratch1b) and refined on the main
  // stream (its pick too, since the level-0 refine reads its shifts) into sh1
  const bool two = p->levels == 2;
  void *img1[2] = {p->scratch[1], p->scratch1b};
  const int64_t fs1 = (int64_t)p->ml[1] * p->pitch[1];
  int64_t k = 0;
  for (int64_t f0 = 0; f0 < T; f0 += p->cap, ++k) {
    const int64_t B = std::min<int64_t>(p->cap, T - f0);
    const int buf = (int)(k & 1);
    const char *fr = (const char *)d_frames + f0 * fbytes;
    const bool fused = p->tc.fused && !two;
    const bool emit1 = two && prep_emits_l1(p);
    int rc = MOCO_OK;
    if (!fused) {
      if (k >= 2) CK(cudaStreamWaitEvent(sp, p->pe_free[buf], 0));
      rc = launch_tc_prep(p, fr, B, G[buf], ga[buf], sp, emit1 ? img1[buf] : nullptr);
      if (rc) return rc;
      if (two && !emit1) {
        rc = launch_downsample(p, 0, fr, (int64_t)p->m * p->n, img1[buf], B, sp);
        if (rc) return rc;
      }
      CK(cudaEventRecord(p->pe_prep[buf], sp));
      CK(cudaStreamWaitEvent(sm, p->pe_prep[buf], 0));
    }
    if (k >= 2) CK(cudaStreamWaitEvent(sm, p->pe_pick[buf], 0));   // sh1/racc of batch k-2 consumed
    int32_t *sc = two ? p->sh2b[buf] : sh1[buf];
    rc = fused ? launch_tc_fused(p, fr, B, sc, nullptr, d_flags ? d_flags + f0 : nullptr, nullptr, sm)
               : launch_tc_coarse(p, B, G[buf], ga[buf], sc, nullptr, d_flags ? d_flags + f0 : nullptr, nullptr, sm);
    if (rc) return rc;
    if (two) {
      rc = launch_refine_h(p, 1, img1[buf], fs1, B, sc, sh1[buf], nullptr, nullptr, sm, racc[buf]);
      if (rc) return rc;
    }
    CK(cudaEventRecord(p->pe_free[buf], sm));
    // the pick's GA pieces on the pick stream, beside the refine sums -- when the TC search
    // is short (N <= 128: C2 1.66 -> 1.70 M); behind a long one (C3, N = 256) the pick has
    // slack and the side kernel only slows the refine on the critical stream (982 -> 939 k)
    if (use_fra(p, 0, B)) {
      rc = launch_fra(p, fr, (int64_t)p->m * p->n, B, sh1[buf], d_shifts + 2 * f0, d_fmin + f0,
                      d_corrected ? (char *)d_corrected + f0 * fbytes : nullptr, sm);
      if (rc) return rc;
      CK(cudaEventRecord(p->pe_sums[buf], sm));
      CK(cudaStreamWaitEvent(sa, p->pe_sums[buf], 0));
      CK(cudaEventRecord(p->pe_pick[buf], sa));
      continue;
    }
    const u64 *gb = nullptr;
    if (use_rtc(p, 0, B) && p->gbin[buf] && RTC_GA_TOTAL && p->tc.g.N <= 128 && !p->knob.ga_inpick) {
      CK(cudaStreamWaitEvent(sa, p->pe_free[buf], 0));
      rc = launch_ga_pieces(p, 0, fr, (int64_t)p->m * p->n, B, sh1[buf], p->gbin[buf], sa);
      if (rc) return rc;
      gb = p->gbin[buf];
    }
    rc = launch_refine_h(p, 0, fr, (int64_t)p->m * p->n, B, sh1[buf], d_shifts + 2 * f0, d_fmin + f0,
                         d_corrected ? (char *)d_corrected + f0 * fbytes : nullptr, sm, racc[buf], sa,
                         p->pe_sums[buf], gb);
    if (rc) return rc;
    CK(cudaEventRecord(p->pe_pick[buf], sa));
  }
  CK(cudaEventRecord(p->pe_end, sm));
  CK(cudaEventRecord(p->pe_end2, sa));
  CK(cudaStreamWaitEvent(user, p->pe_end, 0));
  CK(cudaStreamWaitEvent(user, p->pe_end2, 0));
  return MOCO_OK;
}

// levels = 0 (C1: no refine): the operand prep of batch k+1 on a second stream beside the
// tensor-core search of batch k (at N <= 192 the search leaves room on its SM for prep
// CTAs), the apply of batch k on a third stream beside the search of batch k+1.
static int align_tc_pipelined0(moco_plan *p, const void *d_frames, int64_t T, int32_t *d_shifts, double *d_fmin,
                               void *d_corrected, uint8_t *d_flags, cudaStream_t user) {
  if (!p->pipe_ready) return MOCO_ESTATE;
  cudaStream_t sp = p->ps[0], sm = p->ps[1], sa = p->ps[2];
  CK(cudaEventRecord(p->pe_start, user));
  for (int k = 0; k < 3; ++k) CK(cudaStreamWaitEvent(p->ps[k], p->pe_start, 0));
  const size_t fbytes = (size_t)p->m * p->n * p->esz[0];
  uint8_t *G[2] = {p->tc.G, p->tc.G2};
  u64 *ga[2] = {p->tc.ga, p->tc.ga2};
  int64_t k = 0;
  for (int64_t f0 = 0; f0 < T; f0 += p->cap, ++k) {
    const int64_t B = std::min<int64_t>(p->cap, T - f0);
    const int buf = (int)(k & 1);
    const char *fr = (const char *)d_frames + f0 * fbytes;
    if (k >= 2) CK(cudaStreamWaitEvent(sp, p->pe_free[buf], 0));   // search k-2 is done with G/ga[buf]
    int rc = launch_tc_prep(p, fr, B, G[buf], ga[buf], sp);
    if (rc) return rc;
    CK(cudaEventRecord(p->pe_prep[buf], sp));
    CK(cudaStreamWaitEvent(sm, p->pe_prep[buf], 0));
    rc = launch_tc_coarse(p, B, G[buf], ga[buf], d_shifts + 2 * f0, d_fmin + f0, d_flags ? d_flags + f0 : nullptr,
                          nullptr, sm);
    if (rc) return rc;
    CK(cudaEventRecord(p->pe_free[buf], sm));
    if (d_corrected) {
      CK(cudaStreamWaitEvent(sa, p->pe_free[buf], 0));
      rc = launch_apply(p, fr, (char *)d_corrected + f0 * fbytes, d_shifts + 2 * f0, B, sa);
      if (rc) return rc;
    }
  }
  CK(cudaEventRecord(p->pe_end, sm));
  CK(cudaEventRecord(p->pe_end2, sa));
  CK(cudaStreamWaitEvent(user, p->pe_end, 0));
  CK(cudaStreamWaitEvent(user, p->pe_end2, 0));
  return MOCO_OK;
}

int moco_align_batch(moco_plan *p, const void *d_frames, int64_t T, int32_t *d_shifts,
                     double *d_fmin, void *d_corrected, uint8_t *d_flags, moco_stream_t stream) {
  int rc = check_align_args(p, d_frames, T);
  if (rc) return rc;
  if (T > 0 && (!d_shifts || !d_fmin)) return MOCO_EINVAL;
  if (((uintptr_t)d_corrected & 15) != 0) return MOCO_EINVAL;
  if (d_corrected && d_corrected == d_frames) return MOCO_EINVAL;
  CK(cudaSetDevice(p->device));
  p->launches = 0;
  const size_t fbytes = (size_t)p->m * p->n * p->esz[0];
  // closed-loop sizes: the FFT path spreads one frame over many SMs (DESIGN.md §8 latency)
  if (p->algo == MOCO_ALGO_TC && T <= LAT_T && p->fft.ready && p->fft.tpl_ready && !p->algo_forced) {
    p->algo = MOCO_ALGO_FFT;
    p->pdl_now = p->knob.pdl != 0 && !p->prof_on;   // (profiling events between kernels: plain launches)
    for (int64_t f0 = 0; f0 < T && rc == MOCO_OK; f0 += p->cap) {
      const int64_t B = std::min<int64_t>(p->cap, T - f0);
      rc = run_batch_user(p, (const char *)d_frames + f0 * fbytes, B, d_shifts + 2 * f0, d_fmin + f0,
                     d_corrected ? (char *)d_corrected + f0 * fbytes : nullptr,
                     d_flags ? d_flags + f0 : nullptr, nullptr, (cudaStream_t)stream);
    }
    p->algo = MOCO_ALGO_TC;
    p->pdl_now = false;
    return rc;
  }
  if (p->algo == MOCO_ALGO_TC && T > p->cap && p->tc.G2 && p->levels == 0 && !p->stage && !p->knob.nopipe &&
      p->dtype == MOCO_U16)
    return align_tc_pipelined0(p, d_frames, T, d_shifts, d_fmin, d_corrected, d_flags, (cudaStream_t)stream);
  if (p->algo == MOCO_ALGO_TC && T > p->cap && p->tc.G2 && p->racc2 && p->sh1b && fused_ok(p, 0) &&
      (p->levels == 1 || (p->levels == 2 && p->scratch1b && p->sh2b[1] && fused_ok(p, 1))) && !p->knob.nopipe)
    return align_tc_pipelined(p, d_frames, T, d_shifts, d_fmin, d_corrected, d_flags, (cudaStream_t)stream);
  for (int64_t f0 = 0; f0 < T; f0 += p->cap) {
    const int64_t B = std::min<int64_t>(p->cap, T - f0);
    rc = run_batch_user(p, (const char *)d_frames + f0 * fbytes, B, d_shifts + 2 * f0, d_fmin + f0,
                   d_corrected ? (char *)d_corrected + f0 * fbytes : nullptr,
                   d_flags ? d_flags + f0 : nullptr, nullptr, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return MOCO_OK;
}

int moco_score_grid(moco_plan *p, const void *d_frames, int64_t T, double *d_f,
                    moco_stream_t stream) {
  int rc = check_align_args(p, d_frames, T);
  if (rc) return rc;
  if (T > 0 && !d_f) return MOCO_EINVAL;
  CK(cudaSetDevice(p->device));
  p->launches = 0;
  const size_t fbytes = (size_t)p->m * p->n * p->esz[0];
  const int64_t WW = (int64_t)p->W * p->W;
  for (int64_t f0 = 0; f0 < T; f0 += p->cap) {
    const int64_t B = std::min<int64_t>(p->cap, T - f0);
    rc = run_batch_user(p, (const char *)d_frames + f0 * fbytes, B, nullptr, nullptr, nullptr, nullptr,
                   d_f + f0 * WW, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return MOCO_OK;
}

int moco_fft_bound(const moco_plan *p, double *Cf, double *Ci) {
  if (!p || !Cf || !Ci || !p->fft.ready) return MOCO_EINVAL;
  *Cf = p->fft.bound_Cf;
  *Ci = p->fft.bound_Ci;
  return MOCO_OK;
}

int moco_fft_means(const moco_plan *p, int64_t *mu_a, int64_t *mu_b) {
  if (!p || !mu_a || !mu_b || !p->fft.ready || !p->fft.tpl_ready || !p->fft.tst) return MOCO_EINVAL;
  CK(cudaSetDevice(p->device));
  long long t[4];
  CK(cudaMemcpy(t, p->fft.tst, sizeof t, cudaMemcpyDeviceToHost));
  *mu_a = t[0];
  *mu_b = t[3];
  return MOCO_OK;
}

int moco_fft_cross(moco_plan *p, const void *d_frames, int64_t T, float *d_h, int32_t *d_shifts,
                   int32_t *d_qcount, moco_stream_t stream) {
  int rc = check_align_args(p, d_frames, T);
  if (rc) return rc;
  if (T > 0 && (!d_h || !d_shifts)) return MOCO_EINVAL;
  if (!fft_supported(p)) return MOCO_EINVAL;
  CK(cudaSetDevice(p->device));
  rc = fft_init(p);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (!p->fft.tpl_ready) {
    rc = fft_set_template(p, st);
    if (rc) return rc;
  }
  p->launches = 0;
  const int L = p->levels;
  const size_t fbytes = (size_t)p->m * p->n * p->esz[0];
  const int64_t WW = (int64_t)p->W * p->W;
  for (int64_t f0 = 0; f0 < T; f0 += p->cap) {
    const int64_t B = std::min<int64_t>(p->cap, T - f0);
    const void *img = stage_frames(p, (const char *)d_frames + f0 * fbytes, B, st, &rc);
    if (rc) return rc;
    int64_t fs = (int64_t)p->m * p->pitch[0];
    if (p->fft.v2) {
      int lin = 0;
      if (L == 2) {
        rc = launch_downsample(p, 0, img, fs, p->scratch[1], B, st);
        if (rc) return rc;
        img = p->scratch[1];
        fs = (int64_t)p->ml[1] * p->pitch[1];
        lin = 1;
      }
      rc = launch_fft2(p, img, fs, p->pitch[lin], B, d_shifts + 2 * f0, nullptr, nullptr, st, d_h + f0 * WW,
                       d_qcount ? d_qcount + f0 : nullptr);
      if (rc) return rc;
      continue;
    }
    for (int l = 0; l < L; ++l) {
      rc = launch_downsample(p, l, img, fs, p->scratch[l + 1], B, st);
      if (rc) return rc;
      img = p->scratch[l + 1];
      fs = (int64_t)p->ml[l + 1] * p->pitch[l + 1];
    }
    rc = launch_fft(p, img, fs, p->pitch[L], B, d_shifts + 2 * f0, nullptr, nullptr, st, d_h + f0 * WW,
                    d_qcount ? d_qcount + f0 : nullptr);
    if (rc) return rc;
  }
  return MOCO_OK;
}

int moco_align_host(moco_plan *p, const void *h_frames, int64_t T, int32_t *h_shifts,
                    double *h_fmin, void *h_corrected, uint8_t *h_flags) {
  if (!p || T < 0) return MOCO_EINVAL;
  if (T == 0) return MOCO_OK;
  if (!h_frames || !h_shifts || !h_fmin) return MOCO_EINVAL;
  if (!p->has_tpl) return MOCO_ESTATE;
  CK(cudaSetDevice(p->device));
  const size_t fbytes = (size_t)p->m * p->n * p->esz[0];
  if (!p->host_ready) {
    // chunks of ~128 MiB of frames, capped by the plan's batch capacity; three slots so
    // the copy of chunk k+1 in, the kernels of chunk k and the copy of chunk k-1 out
    // all overlap (PCIe is full duplex).  Compute stays on ONE stream (the plan's
    // scratch is shared).
    p->host_ch = std::max<int64_t>(1, std::min<int64_t>(p->cap, ((int64_t)128 << 20) / (int64_t)fbytes));
    for (int k = 0; k < 3; ++k) {
      if (cudaMalloc(&p->slot_in[k], p->host_ch * fbytes) != cudaSuccess ||
          cudaMalloc(&p->slot_out[k], p->host_ch * fbytes) != cudaSuccess ||
          cudaMalloc((void **)&p->slot_sh[k], p->host_ch * 2 * sizeof(int32_t)) != cudaSuccess ||
          cudaMalloc((void **)&p->slot_f[k], p->host_ch * sizeof(double)) != cudaSuccess ||
          cudaMalloc((void **)&p->slot_flags[k], p->host_ch) != cudaSuccess) {
        cudaGetLastError();
        return MOCO_ENOMEM;
      }
    }
    for (int k = 0; k < 3; ++k) CK(cudaStreamCreateWithFlags(&p->hs[k], cudaStreamNonBlocking));
    for (int k = 0; k < 3; ++k) {
      CK(cudaEventCreateWithFlags(&p->ev_in[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&p->ev_done[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&p->ev_free[k], cudaEventDisableTiming));
    }
    p->host_ready = true;
  }
  cudaStream_t s_in = p->hs[0], s_comp = p->hs[1], s_out = p->hs[2];
  int64_t total_launches = 0;
  int64_t chunk = 0;
  for (int64_t f0 = 0; f0 < T; f0 += p->host_ch, ++chunk) {
    const int k = (int)(chunk % 3);
    const int64_t B = std::min<int64_t>(p->host_ch, T - f0);
    if (chunk >= 3) CK(cudaStreamWaitEvent(s_in, p->ev_free[k], 0));
    CK(cudaMemcpyAsync(p->slot_in[k], (const char *)h_frames + f0 * fbytes, B * fbytes,
                       cudaMemcpyHostToDevice, s_in));
    CK(cudaEventRecord(p->ev_in[k], s_in));
    CK(cudaStreamWaitEvent(s_comp, p->ev_in[k], 0));
    if (chunk >= 3) CK(cudaStreamWaitEvent(s_comp, p->ev_free[k], 0));
    int rc = moco_align_batch(p, p->slot_in[k], B, p->slot_sh[k], p->slot_f[k],
                              h_corrected ? p->slot_out[k] : nullptr,
                              h_flags ? p->slot_flags[k] : nullptr, s_comp);
    if (rc) return rc;
    total_launches += p->launches;
    CK(cudaEventRecord(p->ev_done[k], s_comp));
    CK(cudaStreamWaitEvent(s_out, p->ev_done[k], 0));
    CK(cudaMemcpyAsync(h_shifts + 2 * f0, p->slot_sh[k], B * 2 * sizeof(int32_t),
                       cudaMemcpyDeviceToHost, s_out));
    CK(cudaMemcpyAsync(h_fmin + f0, p->slot_f[k], B * sizeof(double), cudaMemcpyDeviceToHost, s_out));
    if (h_corrected)
      CK(cudaMemcpyAsync((char *)h_corrected + f0 * fbytes, p->slot_out[k], B * fbytes,
                         cudaMemcpyDeviceToHost, s_out));
    if (h_flags) CK(cudaMemcpyAsync(h_flags + f0, p->slot_flags[k], B, cudaMemcpyDeviceToHost, s_out));
    CK(cudaEventRecord(p->ev_free[k], s_out));
  }
  CK(cudaStreamSynchronize(s_out));
  p->launches = total_launches;
  return MOCO_OK;
}

