/*
 * moco.h -- C-ABI of the B200-native moco hot path (libmoco.so).
 *
 * The operation (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   For every frame a of a stack and a fixed template b, find the integer
 *   shift (s,t) with max(|s|,|t|) < w minimising
 *       f_{s,t} = (1/Area(D_{s,t})) * sum_{(i,j) in D_{s,t}} (a_{i+s,j+t} - b_{i,j})^2
 *   over the overlap D_{s,t}, on frames downsampled by 2x2 block means
 *   `levels` times, then "multiply the optimal (s,t) by 2 and do a
 *   local search" over f_{2s+u,2t+v}, u,v in {0,-1,1}, once per finer level
 *   (P:30), and finally apply the shift with zero fill.
 *
 * Conventions (DESIGN.md §3 readings):
 *   - w is the strict bound at the COARSEST level: |s|,|t| <= w-1 there (R2, R3).
 *   - D_{s,t} pairs template pixel (i,j) with frame pixel (i+s, j+t) (0-based):
 *     a frame equal to the template translated by (+dy,+dx) returns (dy,dx)
 *     with f = 0, and corrected[i][j] = a[i+s][j+t] (R12).
 *   - Ties in f are broken by the smallest (s,t) in lexicographic order (R4);
 *     f is compared as the fp64 value fl(N / Area) (R5).
 *   - Returned shifts are full-resolution pixels; f_min is f at level 0 (R11).
 *   - Odd dimensions: the trailing row/column is dropped at each level (R1).
 *
 * Data layout: every image is row-major, rows of n elements, no padding.  Rows
 *   whose byte length is not a multiple of 16 (e.g. the paper's 416x460 video,
 *   P:62) are accepted: such plans stage each internal batch through a
 *   padded-pitch device buffer with stream-ordered 2-D copies.
 *   Frames: T consecutive m*n images.  MOCO_U16: uint16 samples holding
 *   integers < 2^bits.  MOCO_F32: float32 samples.
 *
 * Ownership: all `d_` pointers are CUDA device memory owned by the caller and
 *   must stay valid until the stream reaches the call; `h_` pointers are host
 *   memory (pinned host memory gets the full copy bandwidth).  The plan owns
 *   its template pyramid, tables and workspace.  Calls are stream-ordered and
 *   asynchronous unless stated; one in-flight call per plan (use one plan per
 *   stream for concurrency).  Results are independent of batch size, stream
 *   and GPU count.
 *
 * Errors: every function returns MOCO_OK (0) or a negative code; no call
 *   aborts the process; there is NO CPU fallback -- a missing device or a
 *   kernel failure is reported as MOCO_ECUDA (see moco_last_cuda_error()).
 */
#ifndef MOCO_H_
#define MOCO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOCO_ABI_VERSION 1

typedef struct moco_plan moco_plan;   /* opaque, library-owned */
typedef void *moco_stream_t;          /* a cudaStream_t (NULL = legacy default stream) */

enum moco_dtype { MOCO_U16 = 1, MOCO_F32 = 2 };

enum moco_status {
  MOCO_OK = 0,
  MOCO_EINVAL = -1,  /* bad argument (see each call)                         */
  MOCO_ENOMEM = -2,  /* device or pinned-host allocation failed               */
  MOCO_ECUDA = -3,   /* CUDA runtime/kernel error; text in moco_last_cuda_error */
  MOCO_ESTATE = -4   /* call order violated (e.g. align before set_template)  */
};

/* Coarse-search algorithm for S3 (the cross term).  AUTO picks by problem
 * size from measurement. */
enum moco_algo { MOCO_ALGO_AUTO = 0, MOCO_ALGO_DIRECT = 1, MOCO_ALGO_TC = 2, MOCO_ALGO_FFT = 3 };

/* Per-frame flag bits written to d_flags/h_flags when non-NULL. */
#define MOCO_FLAG_EDGE 0x1u     /* coarse argmin on the window edge |s| or |t| = w-1 */
#define MOCO_FLAG_FULL 0x2u     /* FFT path: certified candidate set exceeded its cap, every
                                   coarse lag was re-scored exactly (result still exact) */

/*
 * moco_plan_create -- validate the problem and allocate the workspace.
 *   m, n    frame rows/cols at full resolution.
 *   w       strict shift bound at the coarsest level.
 *   levels  number of 2x2 downsamplings, 0..2 (levels >= 3 rejected: P:49
 *           "downsampling 3 and 4 times causes severe errors").
 *   dtype   MOCO_U16 or MOCO_F32.
 *   bits    MOCO_U16: sample bit depth, 1..16, with bits + 2*levels <= 16 (so
 *           level-l block sums fit 16 bits); ignored for MOCO_F32.
 *   device  CUDA device ordinal the plan lives on.
 * EINVAL when: out == NULL; levels not in {0,1,2}; m or n < 2^(levels+1);
 *   w < 1 or w >= min(m_L, n_L) with m_L = floor(m / 2^levels); unknown dtype;
 *   bits out of range.
 * ENOMEM when workspace allocation fails.  No kernel is launched; every stream,
 * event and buffer moco_align_batch uses is created here.
 */
int moco_plan_create(moco_plan **out, int m, int n, int w, int levels, int dtype,
                     int bits, int device);

/*
 * moco_auto_config -- the paper's default settings for an m x n video (P:49,
 * section 3): "If the images are larger than 256x256, we downsample once,
 * otherwise, we do not downsample" -> *levels = 1 if m > 256 or n > 256, else 0;
 * "a maximum translation width of min(m,n)/3" -> *w = floor(min(m_L, n_L) / 3)
 * at the coarsest level (m_L = floor(m / 2^levels); reading R16: w is
 * the coarse-level bound, R2).  The paper's template is "the first image in the
 * video": pass the first frame as d_template to moco_set_template.
 * Host-only arithmetic.  EINVAL on NULL outputs or when no w >= 1 fits
 * (min(m_L, n_L) < 3).
 */
int moco_auto_config(int m, int n, int *w, int *levels);

/* Force the coarse-search algorithm (tests/benchmarks); EINVAL if unsupported
 * for this plan (MOCO_ALGO_TC needs MOCO_U16 with bits + 2*levels <= 14;
 * MOCO_ALGO_FFT needs MOCO_U16; MOCO_ALGO_DIRECT needs w <= 64). */
int moco_plan_set_algo(moco_plan *p, int algo);
/* Algorithm AUTO resolved to for this plan (MOCO_ALGO_DIRECT, _TC or _FFT). */
int moco_plan_get_algo(const moco_plan *p);

/*
 * moco_set_template -- copy the m*n template b (dtype of the plan, device
 * memory) into the plan and build its pyramid and energy tables (S0, once per
 * plan; "the first two sums", "The template used for every video").
 * May be called again to replace the template.  EINVAL on NULL.
 */
int moco_set_template(moco_plan *p, const void *d_template, moco_stream_t stream);

/*
 * moco_align_batch -- the hot path (S1..S7) for T frames resident on the device.
 *   d_frames     T*m*n samples, 16-byte aligned.
 *   d_shifts     out, int32 [T][2] = (s, t) per frame, full resolution.
 *   d_fmin       out, double [T] = f_{s,t} at level 0 for the returned shift.
 *   d_corrected  out or NULL: T*m*n samples, corrected[i][j] = a[i+s][j+t]
 *                in range else 0 (bit copy).  Must not alias d_frames.
 *   d_flags      out or NULL: uint8 [T], MOCO_FLAG_* bits.
 * T == 0 is a no-op; T < 0, NULL required pointers or misalignment -> EINVAL;
 * ESTATE before moco_set_template.  Never allocates; loops over internal
 * batches sized to the plan's workspace.  The outputs may be any memory the
 * device can store to -- including another GPU's buffer mapped into this
 * device's address space (CUDA symmetric memory / peer mappings): the kernels
 * that produce each frame's record store it there directly, which is how the
 * multi-GPU results gather is fused into the hot path (dist.PeerResults,
 * SURVEY.md 8(e)); at levels = 0 the apply reads d_shifts back (over the same
 * mapping).
 */
int moco_align_batch(moco_plan *p, const void *d_frames, int64_t T, int32_t *d_shifts,
                     double *d_fmin, void *d_corrected, uint8_t *d_flags,
                     moco_stream_t stream);

/*
 * moco_align_host -- end-to-end entry point: frames in HOST memory, results
 * back in host memory.  Streams chunks host->device, runs moco_align_batch on
 * each and copies results back, overlapping the copies with compute on
 * internal streams.  Synchronous: returns after every result is in host
 * memory.  Same arguments/meaning as moco_align_batch with h_ host pointers
 * (h_corrected and h_flags may be NULL).  Allocates its device staging
 * buffers on first use (ENOMEM on failure).
 */
int moco_align_host(moco_plan *p, const void *h_frames, int64_t T, int32_t *h_shifts,
                    double *h_fmin, void *h_corrected, uint8_t *h_flags);

/*
 * moco_score_grid -- the coarse-level ScoreGrid: for each of T device frames,
 * d_f[k][s+w-1][t+w-1] = f_{s,t} at the coarsest level for every
 * max(|s|,|t|) < w ("comparing every possible translation").
 * d_f is double [T][2w-1][2w-1].  Same errors as moco_align_batch.
 */
int moco_score_grid(moco_plan *p, const void *d_frames, int64_t T, double *d_f,
                    moco_stream_t stream);

/*
 * moco_fft_cross -- diagnostics of the FFT path (S3 by FFT): for each of T
 * device frames, d_h[k][s+w-1][t+w-1] = the fp32 FFT cross term h~(s,t) at the
 * coarsest level (float [T][2w-1][2w-1]), d_shifts[k] = the certified exact coarse
 * argmin (int32 [T][2], coarse pixels), d_qcount[k] = how many lags were re-scored
 * exactly (int32 [T], may be NULL).  Works whatever algorithm the plan uses; EINVAL
 * for non-U16 plans.  Same other errors as moco_align_batch.
 */
int moco_fft_cross(moco_plan *p, const void *d_frames, int64_t T, float *d_h, int32_t *d_shifts,
                   int32_t *d_qcount, moco_stream_t stream);

/*
 * moco_fft_bound -- the constants of the FFT path's certified error bound (DESIGN.md §5,
 * SURVEY.md §8(c)-O6): for every coarse lag
 *     |h~(s,t) - h(s,t)| <= u (Cf ||a'||_2 ||b'||_2 + Ci sqrt(Mr Mc) ||Y~||_2),  u = 2^-24,
 * a' = a - mu_a, b' = b - mu_b on the supports (moco_fft_means), Y~ the computed spectrum
 * product the inverse transform receives.  Cf covers the forward transforms (per-stage and
 * twiddle rounding, the fp64 template spectrum rounded once to fp32, the product), Ci the
 * inverse.  Cf, Ci: host outputs.  MOCO_EINVAL if the plan has no FFT path.
 */
int moco_fft_bound(const moco_plan *p, double *Cf, double *Ci);

/*
 * moco_fft_means -- the mean removal of the FFT path: the transforms see
 * a - mu_a (frames) and b - mu_b (template) on the supports, and the exact integer
 * correction h = h' + mu_b S_a + mu_a S_b - mu_a mu_b A restores the cross term.  mu_a is
 * the coarse template's rounded mean (0 when mean removal is off); mu_b = mu_a (two-sided)
 * or 0 (frames only).  Host outputs; reads the plan's device copy (synchronises the plan's
 * device).  MOCO_EINVAL if the plan has no FFT path or no template yet.
 */
int moco_fft_means(const moco_plan *p, int64_t *mu_a, int64_t *mu_b);

/*
 * moco_mean_image -- report helper (Fig. 2 caption:
 * "the mean of every image"): d_mean[i*n + j] = (1/T) sum_k frames[k][i][j] for T device
 * frames of m x n samples (dtype MOCO_U16 or MOCO_F32, rows of n samples, no padding).
 * uint16: exact 64-bit sums, one fp64 division per pixel; float32: fp64 sums.  d_mean is
 * double [m][n], device memory.  Stream-ordered.  EINVAL on T < 1, m or n < 1, NULL
 * pointers or an unknown dtype.
 */
int moco_mean_image(const void *d_frames, int64_t T, int m, int n, int dtype, double *d_mean,
                    moco_stream_t stream);

/*
 * moco_probe_peaks -- measured arithmetic throughput of `device` (not part of the hot
 * path; the ALU roofs bench.py reports, SURVEY.md section 2.5 "MB"): out[0] FFMA
 * flop/s, out[1] IMAD int ops/s, out[2] IDP.2A (16x8-bit dot product) ops/s,
 * out[3] DFMA flop/s, each from a saturating microbenchmark (8 chains per thread, 8
 * CTAs of 256 threads per SM, best of 2 timed runs).  Fills min(n, 4) entries;
 * synchronous.  EINVAL on NULL out, ECUDA on a device error.
 */
int moco_probe_peaks(int device, double *out, int n);

/* Number of kernel launches the last moco_align_batch/moco_score_grid issued. */
int64_t moco_last_launch_count(const moco_plan *p);

/*
 * Live per-kernel timing (bench.py's roofline).  When enabled, every launch
 * of the plan is bracketed by CUDA events recorded on the launching stream;
 * moco_profile_read synchronises those events and returns, per kernel kind
 * (enum moco_kernel), the accumulated device milliseconds and launch counts
 * since the last reset, then resets.  n = number of array slots (>= MOCO_K_COUNT
 * fills all).  EINVAL on NULL plan.
 */
enum moco_kernel {
  MOCO_K_DOWNSAMPLE = 0,  /* K1 */
  MOCO_K_COARSE = 1,      /* K3+K4d+K5 direct, or the tensor-core search */
  MOCO_K_REFINE = 2,      /* K6 */
  MOCO_K_APPLY = 3,       /* K7 */
  MOCO_K_PREP = 4,        /* tensor-core operand preparation */
  MOCO_K_SCORE = 5,       /* tensor-core score + argmin epilogue */
  MOCO_K_COUNT = 6
};
int moco_profile_enable(moco_plan *p, int on);
int moco_profile_read(moco_plan *p, double *ms, int64_t *launches, int n);

/* Release everything the plan owns (synchronises its device work). NULL ok. */
int moco_plan_destroy(moco_plan *p);

/* Static text for a status code. */
const char *moco_strerror(int code);
/* Text of the last CUDA error seen by any call on this thread ("" if none). */
const char *moco_last_cuda_error(void);
/* MOCO_ABI_VERSION of the loaded library. */
int moco_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MOCO_H_ */
