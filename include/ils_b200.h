/*
 * ils_b200.h -- C ABI of the B200-native ILS smoothing hot path.
 *
 * The reference (ilsmooth, pure Python) has no native ABI; its seam is the
 * Python API (pkg/src/ilsmooth/__init__.py:44-61) plus the FFT seam
 * solver._fft2/_ifft2 (solver.py:24-30).  Each entry point below states the
 * reference interface it replaces.  All functions are plain C: pointers,
 * sizes, POD structs; no torch types.  Device pointers are CUDA global memory
 * on the plan's device; `stream` is a cudaStream_t passed as void*.
 *
 * Errors are status codes here and exceptions in the Python layer:
 *   ILS_EINVAL, ILS_ENONFINITE_INPUT, ILS_EUNSUPPORTED -> ValueError
 *   ILS_ENONFINITE                                     -> NumericalError
 * (errors.py:10-15; raise sites image.py:43-44, smoother.py:166-167,
 *  solver.py:119-125).  ils_last_error() returns a thread-local message.
 */
#ifndef ILS_B200_H
#define ILS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ILS_ABI_VERSION 1

#if defined(__GNUC__)
#define ILS_API __attribute__((visibility("default")))
#else
#define ILS_API
#endif

typedef enum {
  ILS_OK = 0,
  ILS_EINVAL = 1,           /* bad parameters / shapes / plan mismatch -> ValueError */
  ILS_ENONFINITE_INPUT = 2, /* non-finite input plane -> ValueError (image.py:43-44) */
  ILS_ENONFINITE = 3,       /* non-finite iterate -> NumericalError (smoother.py:166-167) */
  ILS_ECUDA = 4,            /* CUDA runtime failure */
  ILS_EUNSUPPORTED = 5      /* a side has a prime factor > 4096 (fp32) / 2048 (fp64) -> ValueError */
} ils_status;

typedef enum { ILS_CHARBONNIER = 0, ILS_WELSCH = 1, ILS_SOFT = 2 /* HQS plans only */ } ils_penalty_kind;
typedef enum { ILS_F32 = 0, ILS_F64 = 1 } ils_dtype;

/* Value of a device status word that saw no failure (memset pattern 0x7f). */
#define ILS_STATUS_CLEAN 0x7f7f7f7f

/* SmoothParams (smoother.py:31-62) + penalty (penalty.py:47-105), flattened.
 * c must already be resolved (SmoothParams.curvature, smoother.py:60-62). */
typedef struct {
  int32_t kind;  /* ils_penalty_kind */
  double p;      /* Charbonnier exponent, (0, 1]       (penalty.py:54-56) */
  double eps;    /* Charbonnier eps > 0                  (penalty.py:57-58) */
  double gamma;  /* Welsch gamma > 0                     (penalty.py:84-86) */
  double lam;    /* lambda > 0, finite                   (smoother.py:47-48) */
  double c;      /* curvature >= min_curvature(1-1e-12) (smoother.py:51-56) */
  int32_t iters; /* >= 1                                 (smoother.py:49-50) */
} ils_params;

typedef struct ils_plan ils_plan;

/* make_plan(height, width, lam, c) (solver.py:78-106) for a batch of `batch`
 * planes of height x width, computing in `dtype` on CUDA `device`.  Holds the
 * FFT radix plans, twiddle tables and the 1-D spectral-denominator tables.
 * Immutable after creation; safe to share across threads and streams. */
ILS_API ils_status ils_plan_create(ils_plan** out, int32_t batch, int32_t height, int32_t width, const ils_params* params,
                           int32_t dtype, int32_t device);
ILS_API void ils_plan_destroy(ils_plan* plan);

/* HqsParams (hqs.py:27-47): the penalty-splitting baseline for the L1
 * gradient objective.  beta0 = 0 selects the default 2*lam.  A plan from
 * ils_hqs_plan_create runs hqs_smooth_plane (hqs.py:50-66) through
 * ils_smooth / ils_smooth_host: per iteration n the field step
 * m = soft_threshold(grad u, lam / (2 beta_n)) is fused into the row pass
 * and the u-step solve_ls(lam = 2 beta_n, c = 1) uses the per-iteration
 * denominator 1 + beta_n (wy + wx), beta_n = beta0 kappa^n.  No energy trace. */
typedef struct {
  double lam;    /* > 0, finite */
  double beta0;  /* > 0 finite, or 0 for 2*lam */
  double kappa;  /* > 1, finite */
  int32_t iters; /* >= 1 */
} ils_hqs_params;
ILS_API ils_status ils_hqs_plan_create(ils_plan** out, int32_t batch, int32_t height, int32_t width,
                                       const ils_hqs_params* params, int32_t dtype, int32_t device);

/* Bytes of device workspace one in-flight ils_smooth/ils_solve_ls call needs
 * (two half spectra + trace partials).  One workspace per concurrent call. */
ILS_API ils_status ils_workspace_size(const ils_plan* plan, size_t* bytes);

/* smooth_plane / smooth_color(PER_CHANNEL_RGB) (smoother.py:132-217): all
 * params.iters ILS iterations on `batch` planes.  f_dev/u_dev: planar
 * [batch][height][width] with rows contiguous and `plane_stride` elements
 * between planes.  status_dev (int32, device): set to ILS_STATUS_CLEAN, then
 * atomically lowered to the first non-finite iteration (0 = input).
 * energies_dev (double, device, optional): (iters+1) x batch energies,
 * iteration-major (smoother.py:93-101, 161, 168-169).  Asynchronous. */
ILS_API ils_status ils_smooth(const ils_plan* plan, const void* f_dev, void* u_dev, int64_t plane_stride, void* workspace,
                      void* stream, int32_t* status_dev, double* energies_dev);

/* Same, with HOST buffers: `nbatches` consecutive batches of plan.batch
 * planes (plane_stride elements apart) are copied in, smoothed and copied
 * out, pipelined so batch k+1's host->device copy and batch k-1's
 * device->host copy overlap batch k's kernels, and consecutive batches run
 * on two compute lanes (the caller's stream + workspace, and an internal
 * stream whose workspace lives in io_dev).  Blocks until done, then decodes the status words: returns
 * ILS_ENONFINITE_INPUT / ILS_ENONFINITE with *bad_iter = first bad iteration
 * (-1 when clean).  workspace: ils_workspace_size bytes; io_dev:
 * ils_host_io_size bytes of device memory (I/O slots + second workspace).  Host buffers should be pinned
 * (cudaHostAlloc) for the copies to overlap. */
ILS_API ils_status ils_host_io_size(const ils_plan* plan, size_t* bytes);
ILS_API ils_status ils_smooth_host(const ils_plan* plan, const void* f_host, void* u_host, int64_t plane_stride,
                                   int32_t nbatches, void* workspace, void* io_dev, void* stream, int32_t* bad_iter);

/* Applications (applications.py).  ils_smooth_epilogue = ils_smooth whose
 * final pass writes clip01(u + k (f - u)) instead of u (kind
 * ILS_EPI_DETAIL): detail_enhance (:80-93) with k = DetailBoost.k, and the
 * clip01 of clipart_clean / texture_smooth (:186-207) with k = 0. */
typedef enum { ILS_EPI_NONE = 0, ILS_EPI_DETAIL = 1 } ils_epilogue_kind;
typedef struct {
  int32_t kind; /* ils_epilogue_kind */
  double k;     /* boost, finite >= 0 (applications.py:29-31) */
} ils_epilogue;
ILS_API ils_status ils_smooth_epilogue(const ils_plan* plan, const void* f_dev, void* u_dev, int64_t plane_stride,
                                       void* workspace, void* stream, int32_t* status_dev, const ils_epilogue* epi);
/* gaussian_blur (applications.py:210-222) of `batch` planes: separable,
 * radius ceil(3 sigma) <= 128, replicate edges, axis 0 then axis 1.
 * tmp: batch * plane_stride elements of device scratch.  x may equal y. */
ILS_API ils_status ils_gaussian_blur(const void* x, void* y, void* tmp, int32_t batch, int32_t height, int32_t width,
                                     int64_t plane_stride, double sigma, int32_t dtype, void* stream);

/* 8-bit interleaved frames, the reference's PNG/PPM pixel path fused into
 * the first and last passes (formats.py:25-27 read v/255, write
 * floor(clip01(u)*255 + 0.5); image.py MultiImage.from_array channel split).
 * f_dev / u_dev: frames [batch/channels][H][W][channels] bytes on the plan's
 * device; plan batch = frames * channels.  Same result as smoothing the
 * planes v/255 with ils_smooth and quantising u.  No energy trace. */
ILS_API ils_status ils_smooth_u8(const ils_plan* plan, const uint8_t* f_dev, uint8_t* u_dev, int32_t channels,
                                 void* workspace, void* stream, int32_t* status_dev);
/* ils_smooth_host for 8-bit frames: nbatches consecutive batches of
 * batch/channels frames, pipelined as ils_smooth_host (io_dev:
 * ils_host_io_size bytes). */
ILS_API ils_status ils_smooth_host_u8(const ils_plan* plan, const uint8_t* f_host, uint8_t* u_host, int32_t channels,
                                      int32_t nbatches, void* workspace, void* io_dev, void* stream,
                                      int32_t* bad_iter);

/* One pass of the ils_smooth launch sequence on its own (roofline timing and
 * profiling).  pass & 3: 0 = row pass from f (iteration 0), 1 = column solve
 * pass, 2 = fused row pass (iteration >= 1), 3 = final row pass writing u.
 * pass & 4 selects which of the workspace's two half spectra is current:
 * 0 writes spectrum A; 1 solves the current one in place; 2 reads the
 * current one and writes the other; 3 reads the current one.  The ils_smooth
 * sequence is therefore 0, 1, 2, 5, 6, 1, 2, 5, ..., ending with 3 or 7
 * (same results, bit for bit, as ils_smooth). */
ILS_API ils_status ils_launch_pass(const ils_plan* plan, int32_t pass, const void* f_dev, void* u_dev,
                                   int64_t plane_stride, void* workspace, void* stream, int32_t* status_dev);

/* solve_ls(plan, f, mu_x, mu_y) (solver.py:109-134): one least-squares
 * solve per plane.  status_dev is lowered to 1/2/3 when f/mu_x/mu_y hold a
 * non-finite value (solver.py:119-125). */
ILS_API ils_status ils_solve_ls(const ils_plan* plan, const void* f_dev, const void* mu_x_dev, const void* mu_y_dev,
                        void* u_dev, int64_t plane_stride, void* workspace, void* stream, int32_t* status_dev);

/* The hand-written real 2-D transforms on their own (the FFT seam
 * solver._fft2/_ifft2, restricted to real data): rfft2 writes the half
 * spectrum [batch][height][width/2+1] (complex, interleaved) with row pitch
 * `spec_pitch` complex elements; irfft2 is its normalised inverse.
 * irfft2 destroys its input spectrum. */
ILS_API ils_status ils_rfft2(const ils_plan* plan, const void* x_dev, int64_t plane_stride, void* spec_dev, int64_t spec_pitch,
                     void* stream);
ILS_API ils_status ils_irfft2(const ils_plan* plan, void* spec_dev, int64_t spec_pitch, void* x_dev, int64_t plane_stride,
                      void* stream);

/* BT.601 conversion of [frames][3][plane] in place (image.py:110-128);
 * used by ColorMode.LUMINANCE_ONLY (smoother.py:195-202). */
ILS_API ils_status ils_rgb_yuv(void* planes_dev, int32_t dtype, int64_t plane_stride, int64_t npx, int32_t frames,
                       int32_t inverse, void* stream);

/* ---- standalone field kernels (the reference exports these steps as
 * functions, __init__.py:44-61; inside ils_smooth they are fused into the row
 * pass and never touch memory).  Planar [batch][height][width], plane_stride
 * elements apart, dtype ILS_F32/ILS_F64, asynchronous on `stream`.  The fp64
 * gradients and adjoint are bit-identical to the reference's numpy. */
/* grad_x / grad_y (solver.py:33-40): periodic forward differences; gx or gy may be NULL. */
ILS_API ils_status ils_grad(const void* u_dev, void* gx_dev, void* gy_dev, int32_t batch, int32_t height,
                            int32_t width, int64_t plane_stride, int32_t dtype, void* stream);
/* adjoint_accumulate (solver.py:43-49): roll(mu_x,1,1) - mu_x + roll(mu_y,1,0) - mu_y. */
ILS_API ils_status ils_adjoint_accumulate(const void* mu_x_dev, const void* mu_y_dev, void* out_dev, int32_t batch,
                                          int32_t height, int32_t width, int64_t plane_stride, int32_t dtype,
                                          void* stream);
/* aux_update (penalty.py:117-126): out = c x - phi'(x) over n elements; params
 * kind/p/eps/gamma/c (c checked against the penalty's minimum curvature,
 * penalty.py:108-114, -> ILS_EINVAL); lam and iters must be valid but unused. */
ILS_API ils_status ils_aux_update(const ils_params* params, const void* x_dev, void* out_dev, int64_t n,
                                  int32_t dtype, void* stream);
/* energy (smoother.py:93-101): out_dev[b] = sum (u-f)^2 + lam (sum phi(grad_x u) +
 * sum phi(grad_y u)) per plane, f64, deterministic.  Only the penalty fields of
 * params are validated (lam: any finite value; c, iters unused).  scratch:
 * ILS_ENERGY_SCRATCH(batch) bytes of device memory. */
#define ILS_ENERGY_SCRATCH(batch) ((size_t)(batch) * 256u * 3u * sizeof(double))
ILS_API ils_status ils_energy(const ils_params* params, const void* u_dev, const void* f_dev, int32_t batch,
                              int32_t height, int32_t width, int64_t plane_stride, int32_t dtype, double* out_dev,
                              void* scratch, void* stream);

/* tonemap_single / tonemap_multi (applications.py:132-183) on the GPU: log10
 * of the luminance (+ log_offset), the ILS base smoothing of all scales as
 * ONE batched launch sequence with a per-plane lambda (plan batch = nscales;
 * its penalty, c and iters are TonemapParams.base_params', its lam is
 * replaced by lam[s] per plane), the base compression (_compress_base,
 * :111-118) and the recolouring (_recolor, :121-129) -- float64 in and out:
 * lum [H][W], rgb and out [3][H][W].  scalars_dev (3 doubles) receives the
 * coarsest base's max, its spread (max - min) and target_range / spread; the
 * caller raises NumericalError when spread < 1e-9 (:113-116).  workspace:
 * ils_tonemap_workspace_size bytes.  Asynchronous. */
typedef struct {
  int32_t nscales;      /* 1 (tonemap_single) or 3 (tonemap_multi, fine to coarse) */
  double lam[3];        /* base smoothing lambda per scale */
  double weights[3];    /* detail weights, finest first (multi) */
  double target_range;  /* > 0 */
  double saturation;    /* (0, 1] */
  double log_offset;    /* > 0 */
} ils_tonemap_params;
ILS_API ils_status ils_tonemap_workspace_size(const ils_plan* plan, size_t* bytes);
ILS_API ils_status ils_tonemap(const ils_plan* plan, const double* lum_dev, const double* rgb_dev, double* out_dev,
                               const ils_tonemap_params* params, void* workspace, void* stream, int32_t* status_dev,
                               double* scalars_dev);

/* detail_enhance's boost (applications.py:90-92) on n elements: out =
 * clip01(u + k (f - u)) (ILS_EPI_DETAIL's arithmetic, for planes that did not
 * come out of ils_smooth_epilogue, e.g. the LUMINANCE_ONLY round trip). */
ILS_API ils_status ils_detail_boost(const void* f_dev, const void* u_dev, void* out_dev, int64_t n, double k,
                                    int32_t dtype, void* stream);
/* Element-wise dtype conversion of n values (round to nearest even): the
 * drop-in's float64 host planes <-> the fp32 compute planes (as_plane's
 * float64 contract, image.py:36-45; output fresh float64, solver.py:134). */
ILS_API ils_status ils_convert(const void* src_dev, int32_t src_dtype, void* dst_dev, int32_t dst_dtype, int64_t n,
                               void* stream);
/* SolverPlan.denom (solver.py:100-102) as a float64 height x width array. */
ILS_API ils_status ils_denominator(double* out_dev, int32_t height, int32_t width, double lam, double c, void* stream);
/* SolverPlan.f_hat (solver.py:69-75): the full complex128 height x width fft2 of
 * a real plane from its fp64 half spectrum (rows of spec_pitch >= width/2+1). */
ILS_API ils_status ils_hermitian_full(const void* half_dev, int64_t spec_pitch, void* full_dev, int32_t height,
                                      int32_t width, void* stream);

/* ---- C5: one image slab-decomposed over nranks GPUs --------
 * Rank r owns rows [row0[r], row0[r+1]) for the row passes and spectrum
 * columns [col0[r], col0[r+1]) for the column passes.  Between them the
 * caller moves the half spectrum with two all-to-alls (NCCL on GPU):
 *   forward  (row -> col): rank r sends peer q a block [H_r][pitch[q]];
 *            it receives [H_q][pitch[r]] from every q, i.e. [H][pitch[r]];
 *   reverse  (col -> row): rank r sends peer q its rows plus q's two halo
 *            rows, [H_q + 2][pitch[r]] (periodic across ranks); it receives
 *            [H_r + 2][pitch[q]] from every q.
 * The kernels read and write those blocks directly (the pack/unpack of the
 * transpose is fused into the row pass's loads/stores and the column pass's
 * scatter).  ils_slab_get_layout returns row0/col0 (nranks+1 entries),
 * pitch (nranks) and counts[4][8] in complex elements: fwd send, fwd recv,
 * rev send, rev recv per peer.  f_ext is the rank's f rows plus the two
 * halo rows [H_r + 2][width]; u is [H_r][width]. */
ILS_API ils_status ils_slab_plan_create(ils_plan** out, int32_t height, int32_t width, const ils_params* params,
                                        int32_t dtype, int32_t device, int32_t nranks, int32_t rank);
ILS_API ils_status ils_slab_get_layout(const ils_plan* plan, int32_t* row0, int32_t* col0, int32_t* pitch,
                                       int64_t* counts);
/* mode 0: iteration-0 row pass (f_ext -> fwd send); 1: fused row pass
 * (rev recv -> fwd send), `iter` = index of the iterate it reads; 3: final
 * row pass (rev recv -> u). */
ILS_API ils_status ils_slab_row_pass(const ils_plan* plan, int32_t mode, const void* f_ext, const void* rev_recv,
                                     void* fwd_send, void* u, int32_t iter, void* stream, int32_t* status_dev);
/* Column solve pass on this rank's columns: fwd recv -> rev send. */
ILS_API ils_status ils_slab_col_pass(const ils_plan* plan, void* fwd_recv, void* rev_send, void* stream);

/* The whole C5 slab smooth in one call (SURVEY 8b's ils_smooth_dist): the row
 * and column slab passes above with the two transposes per iteration as NCCL
 * grouped send/recv (byte blocks in ils_slab_get_layout's order) on `stream`,
 * for `planes` consecutive planes of this rank (f_ext: [rows + 2][width]
 * per plane, f_ext_stride elements apart; u: [rows][width], u_stride apart).
 * nccl_comm is an ncclComm_t over the slab plan's nranks, rank = its rank
 * (ils_nccl_comm_create, or the caller's own).  NCCL is loaded at run time
 * (libnccl.so.2, or the path in ILS_NCCL_LIB).  workspace:
 * ils_dist_workspace_size bytes (the four all-to-all buffers).  Asynchronous;
 * bitwise the single-GPU ils_smooth result on this rank's rows. */
typedef struct {
  char internal[128]; /* ncclUniqueId */
} ils_nccl_id;
ILS_API ils_status ils_nccl_get_unique_id(ils_nccl_id* id);
ILS_API ils_status ils_nccl_comm_create(void** comm, int32_t nranks, const ils_nccl_id* id, int32_t rank,
                                        int32_t device);
ILS_API ils_status ils_nccl_comm_destroy(void* comm);
ILS_API ils_status ils_dist_workspace_size(const ils_plan* slab_plan, size_t* bytes);
ILS_API ils_status ils_smooth_dist(const ils_plan* slab_plan, const void* f_ext_dev, void* u_dev, int32_t planes,
                                   int64_t f_ext_stride, int64_t u_stride, void* workspace, void* nccl_comm,
                                   void* stream, int32_t* status_dev);

/* Introspection for tests and the bench. */
typedef struct {
  int32_t batch, height, width, dtype, packed;
  int32_t row_band, row_threads, row_grid, row_smem;
  int32_t col_cols, col_threads, col_grid, col_smem;
  int32_t row_passes, col_passes;
  int32_t row_group, col_group; /* threads per FFT line group */
  int32_t row_spec, col_spec;   /* compile-time FFT plan id, -1 = runtime plan */
  int32_t row_swz, col_swz;     /* 1 = XOR-swizzled shared-memory line layout */
  int32_t row_radix[16];
  int32_t col_radix[16];
  int64_t spec_pitch;        /* complex elements per spectrum row */
  int32_t launches_per_call; /* kernels one ils_smooth launches (no trace) */
  int32_t col2_spec;         /* two-stage column solve kernel id, -1 = k_col */
  int32_t col2_n1, col2_n2;  /* its split H = n1 * n2 */
  int32_t col2_cols;         /* spectrum columns per CTA */
  int32_t col3_spec;         /* three-stage column solve kernel id (takes precedence), -1 = none */
  int32_t col3_n1, col3_n2, col3_n3; /* its split H = n1 * n2 * n3 */
  int32_t col3_cols;         /* spectrum columns per CTA */
  int32_t row_roll_rows;     /* > 0: rolling-band first / fused row passes, rows per CTA chunk */
} ils_plan_info;
ILS_API ils_status ils_plan_get_info(const ils_plan* plan, ils_plan_info* info);

ILS_API const char* ils_last_error(void);
ILS_API int32_t ils_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* ILS_B200_H */
