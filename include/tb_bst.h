/*
 * tb_bst.h -- C ABI of the B200-native BST filtered-backprojection path.
 *
 * The reference (tomoblocks, pure Python) has no FFI; these entry points are
 * what its Python API binds through ctypes.  Each one
 * replaces a reference function, cited as pkg/src/tomoblocks/<file>:<line>:
 *
 *   tb_plan_create / tb_plan_destroy  <- BstPlan + FilterPlan      fourier_bp.py:69-267
 *   tb_fbp        (kernel "bst")      <- fbp                       fourier_bp.py:508-530
 *   tb_bst                            <- bst_backproject           fourier_bp.py:435-461
 *   tb_bst_scaled                     <- backproject stage         pipeline.py:511-518
 *   tb_ramp                           <- ramp_filter               fourier_bp.py:490-505
 *   tb_ss         (kernel "ss")       <- backproject_ss            projector.py:126-158
 *   tb_fbp_ss                         <- fbp(kernel="ss")          fourier_bp.py:525-527
 *   tb_forward                        <- forward_project           projector.py:94-123
 *   tb_normalize                      <- preprocess.normalize      preprocess.py:59-74
 *   tb_center_estimate / _apply       <- estimate/apply_center     preprocess.py:88-138
 *   tb_rings                          <- suppress_rings            preprocess.py:141-154
 *   tb_pre_params / tb_fbp_pre        <- center + rings + fbp      pipeline.py:461-518 (stages fused into K1)
 *   tb_fbp_counts                     <- normalize + fbp stages    pipeline.py:447-459, 486-518
 *   tb_fbp_frames                     <- read (layout 0) + fbp     volio.py:159-180, pipeline.py:486-518
 *
 * Conventions (grids.py): sinograms are angle-major float32 [B][A][n_t]
 * (A = n_theta, or 2*n_theta for full-turn input); images are float32
 * [B][n][n], row -> u2, col -> u1.  All data pointers are DEVICE pointers
 * on the plan's device; `stream` is a cudaStream_t (NULL = legacy default).
 * The caller owns input, output and workspace; no call allocates.  Calls are
 * asynchronous on `stream`; tb_read_status() synchronises and reports the
 * non-finite checks (reference: ValueError on non-finite input,
 * grids.py:130-131; FloatingPointError on non-finite output,
 * fourier_bp.py:459-460).  No C++ exception crosses this boundary: every
 * function returns a tb_status and tb_last_error() describes the last
 * failure on the calling thread.
 *
 * A plan is immutable after creation and may be used concurrently from
 * several host threads on different streams with distinct workspaces.
 */
#ifndef TB_BST_H
#define TB_BST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TB_ABI_VERSION 3

typedef enum {
  TB_OK = 0,
  TB_ERR_INVALID = 1,     /* bad argument / plan validation  (ValueError) */
  TB_ERR_UNSUPPORTED = 2, /* valid for the reference, not on this device   */
  TB_ERR_CUDA = 3,        /* CUDA runtime failure                          */
  TB_ERR_WORKSPACE = 4,   /* workspace too small                           */
  TB_ERR_NONFINITE_INPUT = 5,  /* (tb_read_status) input had NaN/Inf     */
  TB_ERR_NONFINITE_OUTPUT = 6  /* (tb_read_status) FloatingPointError    */
} tb_status;

typedef enum { TB_INTERP_BILINEAR = 0, TB_INTERP_NEAREST = 1 } tb_interp;
typedef enum { TB_FILTER_RAMP = 0, TB_FILTER_RAMP_APODIZED = 1 } tb_filter_kind;

/* Every BstPlan field (fourier_bp.py:77-85) plus the FilterPlan
 * (fourier_bp.py:256-257) and the angle-axis span (grids.py:78-79). */
typedef struct {
  int32_t n_t;            /* detector samples, >= 2                        */
  int32_t n_theta;        /* angles on [0, pi)                             */
  int32_t pad_factor;     /* >= 2                                          */
  int32_t radial_samples; /* 0 -> next_pow2(pad_factor * n_t)              */
  double kb_beta;         /* Kaiser-Bessel origin window                   */
  double kb_support;
  int32_t sigma_min_bins; /* >= 1                                          */
  int32_t interp;         /* tb_interp                                     */
  int32_t output_n;       /* 0 -> n_t                                      */
  int32_t full_turn;      /* input holds 2*n_theta angles on [0, 2 pi)     */
  int32_t filter_kind;    /* tb_filter_kind                                */
  double rolloff;         /* (0, 1]; used when filter_kind is apodized     */
  int32_t n_angles;       /* rows of the input sinogram; 0 -> n_theta (half
                             turn) or 2 n_theta (full turn).  Any other
                             count (an odd full turn) only serves the ramp,
                             slant-stack and forward paths, like the
                             reference's backproject_ss (projector.py:126-158);
                             its BST calls fail with TB_ERR_INVALID as the
                             reference's resample_polar does (fourier_bp.py:331-332) */
  int32_t flags;          /* TB_PLAN_* bits                                 */
} tb_plan_desc;

/* tb_plan_desc.flags: build no gridding tables (a plan that only serves
 * tb_ramp / tb_ss / tb_fbp_ss / tb_forward / preprocessing; its BST calls
 * fail with TB_ERR_INVALID). */
#define TB_PLAN_NO_GRID 1

typedef struct {
  int32_t n_t, n_theta, n_angles; /* n_angles = rows in the input sinogram  */
  int32_t radial_samples;         /* L                                      */
  int32_t ramp_samples;           /* npad = 2 * next_pow2(n_t)              */
  int32_t output_n;               /* n                                      */
  int32_t support_lo, support_hi; /* KB window index range (closed)         */
  double amplitude_scale;         /* BstPlan.amplitude_scale                */
} tb_plan_info;

typedef struct tb_plan tb_plan;

/* Workspace regions exposed for inspection by the parity tests
 * (byte offsets into the workspace; batch-major inside each region). */
typedef struct {
  size_t total;
  size_t polar;    /* float2 [B][rows][L/2]  K1 output (balanced, kernel-weighted) */
  size_t rowcoef;  /* float  [B][rows]       a_j (rect coefficient per row)        */
  size_t common;   /* float2 [B][L/2]        angle-independent row (K1b)           */
  size_t coefmean; /* float  [B]             coef.mean() (K1b)                     */
  size_t columns;  /* float2 [B][L/2+1][n]   K2 output                            */
  size_t filtered; /* float  [B][A][n_t]     ramp output (ss path / unfused path)  */
  size_t status;   /* int32  [2]             non-finite flags                      */
} tb_workspace_layout;

int tb_abi_version(void);
const char* tb_last_error(void);

int tb_plan_create(const tb_plan_desc* desc, int device, tb_plan** out);
int tb_plan_destroy(tb_plan* plan);
int tb_plan_get_info(const tb_plan* plan, tb_plan_info* info);

/* Bytes of workspace for `batch` slices per internal launch group. */
int tb_workspace_bytes(const tb_plan* plan, int batch, size_t* bytes);
int tb_workspace_get_layout(const tb_plan* plan, int batch, tb_workspace_layout* layout);

/* Filtered backprojection, kernel "bst": ramp -> BST -> x 1/(2 pi).
 * Processes n_slices slices in launch groups of `batch` slices, reusing the
 * workspace (sized with tb_workspace_bytes(plan, batch)). */
int tb_fbp(const tb_plan* plan, const float* sino, float* image, int n_slices,
           int batch, void* workspace, size_t workspace_bytes, void* stream);

/* tb_fbp with CUDA events around every kernel launch (measurement only):
 * synchronises `stream` and adds each stage's summed device time in ms to
 * stage_ms[5] = {ramp (unfused path), K1, K1b, K2, K3}. */
int tb_fbp_profiled(const tb_plan* plan, const float* sino, float* image, int n_slices,
                    int batch, void* workspace, size_t workspace_bytes, void* stream,
                    double* stage_ms);

/* fbp on transmission counts: the normalisation prologue
 * y = -ln(max(I - D, eps) / max(I0 - D, eps))   (preprocess.py:59-74,
 * pipeline.py:447-459) fused into the radial kernel's load, then as tb_fbp.
 * flat (I0) and dark (D) are device frames [A][n_t] shared by every slice. */
int tb_fbp_counts(const tb_plan* plan, const float* counts, const float* flat, const float* dark,
                  double eps, float* image, int n_slices, int batch, void* workspace,
                  size_t workspace_bytes, void* stream);

/* tb_fbp_counts for constant frames (the reference pipeline's i0 / dark
 * scalars, pipeline.py:447-451): no per-sample frame loads. */
int tb_fbp_counts_const(const tb_plan* plan, const float* counts, double i0, double dark,
                        double eps, float* image, int n_slices, int batch, void* workspace,
                        size_t workspace_bytes, void* stream);

/* fbp of a frame-major slab [A][n_slices][n_t] (a TOMOVOL1 layout-0 block as
 * read from disk, volio.py:159-180): the radial kernel reads rows at the
 * frame stride, so no transpose pass; output [n_slices][n][n]. */
int tb_fbp_frames(const tb_plan* plan, const float* frames, float* image, int n_slices, int batch,
                  void* workspace, size_t workspace_bytes, void* stream);

/* normalize alone (preprocess.normalize, preprocess.py:59-74): counts
 * [B][A][n_t] -> line integrals, same shape.  NaN counts stay NaN. */
int tb_normalize(const tb_plan* plan, const float* counts, const float* flat, const float* dark,
                 double eps, float* out, int n_slices, void* stream);

/* Rotation-centre estimate per slice (preprocess.estimate_center,
 * preprocess.py:88-118): beta_conf (device, [B][2] double) receives (beta in
 * detector bins, confidence); status (device, [B] int) 0 ok, 1 constant
 * sinogram, 2 implausible shift (the reference's CenteringError cases). */
int tb_center_estimate(const tb_plan* plan, const float* sino, int n_slices, double* beta_conf,
                       int* status, void* stream);

/* Undo a per-slice detector shift (preprocess.apply_center, :121-138) with
 * beta = beta_conf[2 q]; in and out [B][A][n_t] (may not alias). */
int tb_center_apply(const tb_plan* plan, const float* sino, const double* beta_conf, float* out,
                    int n_slices, void* stream);

/* Ring suppression (preprocess.suppress_rings, :141-154): subtract the
 * per-detector mean over angles minus its reflect-padded moving average of
 * odd `window` >= 3.  scratch: device [B][n_t] doubles.  May not alias. */
int tb_rings(const tb_plan* plan, const float* sino, float* out, int window, double* scratch,
             int n_slices, void* stream);

/* Fused centre / ring stages.  tb_pre_params: per slice the apply_center
 * shift (floor(beta), frac(beta)) as float pairs shift[n_slices][2], from
 * beta_conf[n_slices][2] (tb_center_estimate output or caller-filled; NULL =
 * beta 0), and with window > 0 (odd >= 3) the suppress_rings stripe profile
 * stripe[n_slices][n_t] of the centred sinogram (mean_scratch: n_slices * n_t
 * doubles).  tb_fbp_pre: tb_fbp whose radial kernel applies the shift and
 * subtracts the stripes as it loads each row (preprocess.py:119-154), with
 * stripe NULL for centring only; TB_ERR_UNSUPPORTED unless the plan fuses
 * the ramp filter into K1 (ramp_samples == radial_samples). */
int tb_pre_params(const tb_plan* plan, const float* sino, int n_slices, const double* beta_conf, int window,
                  double* mean_scratch, float* shift, float* stripe, void* stream);
int tb_fbp_pre(const tb_plan* plan, const float* sino, float* image, int n_slices, int batch, void* ws,
               size_t ws_bytes, const float* shift, const float* stripe, void* stream);

/* BST backprojection only (input already ramp-filtered; no 1/(2 pi)). */
int tb_bst(const tb_plan* plan, const float* sino, float* image, int n_slices,
           int batch, void* workspace, size_t workspace_bytes, void* stream);

/* tb_bst with the output multiplied by `scale` in the last kernel's epilogue
 * (the reference pipeline's backproject stage, bst_backproject x FBP_SCALE,
 * pipeline.py:511-518, without a separate pass over the images). */
int tb_bst_scaled(const tb_plan* plan, const float* sino, float* image, int n_slices,
                  int batch, void* workspace, size_t workspace_bytes, float scale, void* stream);

/* Ramp filter only: out has the input's shape [B][A][n_t]. */
int tb_ramp(const tb_plan* plan, const float* sino, float* out, int n_slices,
            void* stream);

/* Slant-stack backprojection of already-filtered rows onto the plan's n x n
 * grid, multiplied by `scale` (1 for backproject_ss). */
int tb_ss(const tb_plan* plan, const float* sino, float* image, int n_slices,
          float scale, void* stream);

/* Forward projector (projector.forward_project, projector.py:94-123): line
 * integrals of images [B][n][n] (n = plan output_n) on the plan's (t, theta)
 * grid -> sinograms [B][A][n_t]; step_length in (0, 1] pixel sizes, interp
 * tb_interp.  The adjoint partner of tb_ss. */
int tb_forward(const tb_plan* plan, const float* image, float* sino, int n_slices,
               double step_length, int interp, void* stream);

/* fbp(kernel="ss"): ramp -> slant stack -> x 1/(2 pi). */
int tb_fbp_ss(const tb_plan* plan, const float* sino, float* image, int n_slices,
              int batch, void* workspace, size_t workspace_bytes, void* stream);

/* Inspection of the K1 output: copies the polar half-spectrum of the last
 * launch group run with `batch` on this workspace (first lane) into `dst`
 * (device, [batch][rows][L/2] complex64 with rows = n_theta + 1 for
 * half-turn input, 2 n_theta full turn), asynchronously on `stream`. */
int tb_copy_polar(const tb_plan* plan, const void* workspace, int batch, void* dst, void* stream);

/* Reset / read the non-finite flags kept in the workspace.  tb_read_status
 * synchronises `stream` and returns TB_OK, TB_ERR_NONFINITE_INPUT or
 * TB_ERR_NONFINITE_OUTPUT. */
int tb_reset_status(const tb_plan* plan, void* workspace, void* stream);
int tb_read_status(const tb_plan* plan, const void* workspace, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TB_BST_H */
