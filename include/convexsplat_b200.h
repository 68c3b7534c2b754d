/*
 * convexsplat_b200 -- C ABI of the B200 (sm_100a) convex-splatting rasterizer.
 *
 * Drop-in for the hot path of the reference package `convexsplat` 0.1.0
 * (/root/reference/pkg/src/convexsplat).  Every entry point names the
 * reference interface it replaces.  The Python host side
 * (paper_2411_14974_b200/rasterizer.py) binds these with ctypes, exactly as
 * INTEGRATION.md shows for the reference package.
 *
 * Conventions
 *   - All pointers except the structs themselves are DEVICE pointers
 *     (cudaMalloc / torch CUDA tensors) unless a name says `host`.
 *   - The caller owns every buffer, including the workspace; the library
 *     never allocates, frees or synchronises (except cs_read_counters).
 *   - Calls are stream-ordered on `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream).  No global mutable state: calls are
 *     re-entrant given distinct workspaces.
 *   - Gradients are ACCUMULATED (+=) into caller-zeroed buffers so sums of
 *     per-view backwards follow GradientBuffer.add (backward.py:65-73).
 *   - Return codes: CS_OK, or a CS_ERR_* value (cs_error_string).
 */
#ifndef CONVEXSPLAT_B200_H
#define CONVEXSPLAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_ABI_VERSION 8

#if defined(__GNUC__)
#define CS_API __attribute__((visibility("default")))
#else
#define CS_API
#endif

enum cs_status {
    CS_OK = 0,
    CS_ERR_ARG = 1,           /* bad argument (null pointer, K out of range, bad sizes) */
    CS_ERR_CUDA = 2,          /* a kernel launch failed (cudaGetLastError) */
    CS_ERR_WORKSPACE = 3,     /* workspace smaller than cs_workspace_size() */
    CS_ERR_NONFINITE = 4,     /* a gradient row came out inf/NaN (cs_read_status) */
    CS_ERR_UNSUPPORTED = 5    /* tile size other than 16, sh_degree outside 0..3 */
};

/* Scaling of delta/sigma with depth: ScalingMode (field.py:17-23). */
enum cs_scaling { CS_SCALE_NONE = 0, CS_SCALE_SQRT = 1, CS_SCALE_DEPTH = 2, CS_SCALE_DEPTH2 = 3 };

/* Camera (model.py:135-172): x_cam = R p + t; pixel = (fx x/z + cx, fy y/z + cy);
 * orthographic drops the divide.  R is row-major. */
typedef struct cs_camera {
    double fx, fy, cx, cy;
    double R[9];
    double t[3];
    double z_near;
    int32_t width, height;
    int32_t ortho;
    int32_t reserved;
} cs_camera;

/* RenderSettings (rasterize.py:33-53) + Scene.background + ScalingMode. */
typedef struct cs_settings {
    double cutoff;            /* contribution_cutoff (default 2e-4) */
    double floor;             /* transmittance_floor (default 1e-4) */
    double background[3];     /* Scene.background */
    int32_t tile;             /* tile_size; 16 is the supported value */
    int32_t sh_degree;        /* 0..3 */
    int32_t scaling_mode;     /* enum cs_scaling */
    int32_t reserved;
} cs_settings;

/* Scene parameters in raw form, SoA float32 (SmoothConvex, model.py:57-126). */
typedef struct cs_params {
    int64_t n;                /* number of convexes */
    int32_t k;                /* points per convex, 3..16 (reference requires >= 4) */
    int32_t reserved;
    const float *points;      /* [n,k,3] */
    const float *raw_delta;   /* [n]  delta   = exp(raw)      */
    const float *raw_sigma;   /* [n]  sigma   = exp(raw)      */
    const float *raw_opacity; /* [n]  opacity = sigmoid(raw)  */
    const float *raw_mask;    /* [n]  mask    = sigmoid(raw)  */
    const float *sh;          /* [n,16,3] */
} cs_params;

/* RenderOutput (rasterize.py:68-74) + a depth map (sum of T*alpha*depth). */
typedef struct cs_frame {
    float *image;             /* [H,W,3] */
    float *final_T;           /* [H,W] */
    int32_t *count;           /* [H,W] */
    float *weight_sum;        /* [H,W] */
    float *depth;             /* [H,W] or NULL */
    uint8_t *visible;         /* [n] or NULL, written 0/1 */
} cs_frame;

/* GradientBuffer (backward.py:39-73); all [+=] accumulated. */
typedef struct cs_grads {
    float *d_points;          /* [n,k,3] */
    float *d_raw_delta;       /* [n] */
    float *d_raw_sigma;       /* [n] */
    float *d_raw_opacity;     /* [n] */
    float *d_raw_mask;        /* [n] */
    float *d_sh;              /* [n,16,3] */
} cs_grads;

/* Byte offsets of the named regions inside the caller's workspace. */
typedef struct cs_layout {
    size_t total_bytes;
    size_t counters;          /* uint32[32]: [0] n_visible [1] n_pairs [2] overflow;
                                 uint64[8] at word 16: work stats (forward evaluations,
                                 line evaluations, blends; backward evaluations, lines),
                                 counted only with CS_WORK_COUNTERS */
    size_t records;           /* float[n][rec_floats] per-convex blend record header */
    size_t lines;             /* double[n][max_k][4] per-convex hull lines (A, B, C, 0; log2 units) */
    size_t hull;              /* uint8[n][max_k]  hull cycle (indices into the K points) */
    size_t bbox;              /* int32[n][4]  x0,x1,y0,y1 half-open pixel rect */
    size_t depth_keys;        /* uint64[n]    f64 bits of the centre depth (~0 culled) */
    size_t order;             /* uint32[n]    convex ids sorted by (depth, id); first n_visible valid */
    size_t tiles_touched;     /* uint32[n] */
    size_t pair_offsets;      /* uint32[n+1]  exclusive scan of tiles_touched in depth order */
    size_t pair_tiles;        /* uint32[cap]  sorted tile id of each (tile, convex) pair */
    size_t pair_ids;          /* uint32[cap]  convex id of each pair (tile-major, depth order) */
    size_t tile_ranges;       /* uint32[tiles][2]  [start,end) into the pair arrays */
    size_t pixel_last;        /* int32[H*W]  pair index of the last blended candidate (-1 none) */
    size_t pixel_T;           /* float[H*W]  final transmittance (kept for the backward) */
    size_t pixel_clamp;       /* uint8[H*W]  bit c set iff channel c of C+T*bg lies in [0,1] */
    size_t grad_accum;        /* float[n][acc_floats] screen-space gradient accumulators */
    size_t scratch;           /* private sort/scan scratch */
    size_t scratch_bytes;
    int32_t rec_floats, acc_floats, max_k, tiles_x, tiles_y, reserved;
} cs_layout;

CS_API int cs_abi_version(void);
CS_API const char *cs_error_string(int code);

/* Workspace size/layout for a frame of this camera at n convexes of k points
 * and room for `pair_capacity` (tile, convex) pairs. Host-only, no CUDA. */
CS_API int cs_workspace_layout(const cs_camera *cam, const cs_settings *set, int64_t n, int32_t k,
                        int64_t pair_capacity, cs_layout *out);

/* Forward render.  Replaces rasterize.render (rasterize.py:156-209) including
 * prepare_view (rasterize.py:77-122) and bin_tiles (rasterize.py:134-144).
 * Stream-ordered; writes the frame and keeps, inside the workspace, what the
 * backward needs.  If the pairs overflow pair_capacity the frame is invalid
 * and counters[2] != 0: read counters[1] (the required pairs), grow the
 * workspace and call again. */
CS_API int cs_forward(const cs_camera *cam, const cs_settings *set, const cs_params *params,
               void *workspace, size_t workspace_bytes, int64_t pair_capacity,
               const cs_frame *frame, void *stream);

/* Backward.  Replaces backward.backward (backward.py:76-212) and
 * _accumulate_primitive_grads (backward.py:215-282).  Needs the workspace of
 * the cs_forward call for the same (camera, settings, params). */
CS_API int cs_backward(const cs_camera *cam, const cs_settings *set, const cs_params *params,
                void *workspace, size_t workspace_bytes, int64_t pair_capacity,
                const float *d_image /*[H,W,3]*/, const cs_grads *grads, void *stream);

/* Stage-wise forward for profiling and pipelining: stage 0 = preprocess
 * (prepare_view), 1 = depth order + tile binning (sort + bin_tiles), 2 =
 * blend.  cs_forward == stages 0..2.  Later stages need the earlier ones to
 * have run on the same workspace. */
CS_API int cs_forward_stages(const cs_camera *cam, const cs_settings *set, const cs_params *params,
                             void *workspace, size_t workspace_bytes, int64_t pair_capacity,
                             const cs_frame *frame, int32_t first_stage, int32_t last_stage, void *stream);

/* Stage-wise backward: stage 0 = backward blend (screen-space gradients),
 * 1 = per-convex chain to the raw parameters.  cs_backward == stages 0..1. */
CS_API int cs_backward_stages(const cs_camera *cam, const cs_settings *set, const cs_params *params,
                              void *workspace, size_t workspace_bytes, int64_t pair_capacity,
                              const float *d_image, const cs_grads *grads, int32_t first_stage,
                              int32_t last_stage, void *stream);

/* Stage-wise forward with flags.  CS_WORK_COUNTERS: the blend kernels also
 * count their work (evaluations, line evaluations, blends, warp
 * evaluations) into the workspace counters -- diagnostics for the roofline
 * accounting, ~7% slower blends, off in cs_forward / cs_forward_stages. */
#define CS_WORK_COUNTERS 2u
CS_API int cs_forward_ex(const cs_camera *cam, const cs_settings *set, const cs_params *params,
                         void *workspace, size_t workspace_bytes, int64_t pair_capacity,
                         const cs_frame *frame, uint32_t flags, int32_t first_stage, int32_t last_stage,
                         void *stream);

/* Convenience: copy counters[0..3] to host (synchronises `stream`). */
CS_API int cs_read_counters(const void *workspace, uint32_t *host_out4, void *stream);

/* Status of the last frame in this workspace (synchronises `stream`):
 * CS_ERR_NONFINITE if the last backward's chain stage produced an inf/NaN
 * gradient row (the values are still written, as the reference's NumPy
 * backward would return them; trainer.py:172-173 is where the reference
 * reacts to non-finite values), CS_ERR_WORKSPACE if the last forward's
 * pairs overflowed the capacity, else CS_OK. */
CS_API int cs_read_status(const void *workspace, void *stream);

/* Full per-view state of the prepared convexes, float64 (the drop-in
 * prepare_view's ProjectedConvex, projection.py:180-203, and ViewPrimitive,
 * rasterize.py:56-65).  Rows of convexes the view did not prepare are left
 * untouched; hull-line rows past the hull length are NaN. */
typedef struct cs_view_export {
    double *pixels;           /* [n,k,2]  projected points (projection.py:22-40) */
    double *point_depths;     /* [n,k]    camera-frame z of the points */
    double *normals;          /* [n,k,2]  hull-line unit normals (projection.py:116-128) */
    double *offsets;          /* [n,k]    hull-line offsets */
    double *delta_s, *sigma_s, *opacity, *scale;  /* [n] */
    double *view_dir;         /* [n,3]    unit camera-centre -> convex-centre */
    double *view_dist;        /* [n] */
    double *color;            /* [n,3]    eval_sh_color in float64 */
} cs_view_export;

/* Replaces the per-primitive outputs of rasterize.prepare_view
 * (rasterize.py:77-122) beyond the blend record: run after a forward (stage
 * 0 at least) on the same workspace. */
CS_API int cs_prepare_view_export(const cs_camera *cam, const cs_settings *set, const cs_params *params,
                                  const void *workspace, size_t workspace_bytes, int64_t pair_capacity,
                                  const cs_view_export *out, void *stream);

/* Blend decisions of a frame (diagnostics: the decision-forced parity check
 * of the float64 oracle, tests/).  Re-runs stage 2 of cs_forward on a
 * workspace whose stages 0..1 ran, with the same kernel the forward uses,
 * and also writes, for every pixel p (row-major), the pair indices (into
 * the sorted tile lists) of the candidates it blended, in blend order, to
 * positions[offsets[p] .. offsets[p] + frame->count[p]).  offsets [H*W]
 * int64 is the exclusive scan of the count of a previous cs_forward of the
 * same inputs (the blend is deterministic).  No reference counterpart: the
 * reference re-decides every blend in float64 (rasterize.py:194-195). */
CS_API int cs_forward_record(const cs_camera *cam, const cs_settings *set, const cs_params *params,
                             void *workspace, size_t workspace_bytes, int64_t pair_capacity,
                             const cs_frame *frame, const int64_t *offsets, int32_t *positions, void *stream);

/* Batched 2-D hull.  Replaces projection.graham_scan (projection.py:47-113)
 * on m point sets of up to npts (<= 32) float64 points: pts [m,npts,2],
 * counts [m] points used per set (NULL = npts); hull [m,npts] (-1 padded),
 * hull_n [m] (0 == None). */
CS_API int cs_graham_scan_batch(int32_t m, int32_t npts, const int32_t *counts, const double *pts,
                         int32_t *hull, int32_t *hull_n, void *stream);

/* ------------------------------------------------------------------------
 * Training-step kernels (the callers on either side of the hot path; SURVEY
 * section 8(f)): the image loss that produces d_image, the per-view
 * sigma-signal of the density control, and the Adam update.
 * ---------------------------------------------------------------------- */

/* Per-view densification signal (trainer.py:192-193), accumulated by the
 * backward's chain stage: sigma_signal += |this view's d_raw_sigma| * visible,
 * sigma_views += visible.  visible = that view's RenderOutput.visible. */
typedef struct cs_view_signal {
    float *sigma_signal;      /* [n] */
    float *sigma_views;       /* [n] */
    const uint8_t *visible;   /* [n] */
} cs_view_signal;

/* cs_backward + the per-view signal (signal may be NULL). */
CS_API int cs_backward_signal(const cs_camera *cam, const cs_settings *set, const cs_params *params,
                              void *workspace, size_t workspace_bytes, int64_t pair_capacity,
                              const float *d_image, const cs_grads *grads, const cs_view_signal *signal,
                              void *stream);

/* General backward: stages first..last (0 = backward blend, 1 = chain), an
 * optional per-view signal (NULL = none) and flags.  CS_GRADS_OVERWRITE:
 * the chain WRITES every row of the gradient buffers (rows of convexes this
 * view did not prepare get zeros) instead of accumulating into them -- the
 * result of GradientBuffer() + one view, without a zeroing pass or the read
 * half of the accumulation.  CS_WORK_COUNTERS: count the backward blend's
 * work (see cs_forward_ex).  cs_backward == flags 0, stages 0..1. */
#define CS_GRADS_OVERWRITE 1u
/* CS_ACCUM_ZEROED: the backward blend's screen-space accumulators were
 * already reset by cs_zero_accumulators, ordered before this call (stage 0
 * then skips its own reset). */
#define CS_ACCUM_ZEROED 4u
CS_API int cs_backward_ex(const cs_camera *cam, const cs_settings *set, const cs_params *params,
                          void *workspace, size_t workspace_bytes, int64_t pair_capacity,
                          const float *d_image, const cs_grads *grads, const cs_view_signal *signal,
                          uint32_t flags, int32_t first_stage, int32_t last_stage, void *stream);

/* Reset the backward blend's per-convex screen-space accumulators (the
 * first half of stage 0 of cs_backward_ex; no reference counterpart -- the
 * reference accumulates into fresh NumPy arrays, backward.py:125-131).  As
 * its own entry it can run on a second stream while the forward of the same
 * view renders; the backward then passes CS_ACCUM_ZEROED. */
CS_API int cs_zero_accumulators(const cs_camera *cam, const cs_settings *set, const cs_params *params,
                                void *workspace, size_t workspace_bytes, int64_t pair_capacity, void *stream);

/* The chain stage (stage 1) of cs_backward_ex over the convexes
 * [first, last) only: the gradient rows of a convex range are final as soon
 * as its launch completes, so a view-sharded step can all-reduce them
 * (bucketed by convex range) while the chain of the next range runs
 * (SURVEY 8(e)).  Needs stage 0 of the same backward first; flags:
 * CS_GRADS_OVERWRITE only. */
CS_API int cs_backward_chain_range(const cs_camera *cam, const cs_settings *set, const cs_params *params,
                                   void *workspace, size_t workspace_bytes, int64_t pair_capacity,
                                   const cs_grads *grads, const cs_view_signal *signal, uint32_t flags,
                                   int64_t first, int64_t last, void *stream);

/* Scratch bytes cs_image_loss needs for an H x W image. Host-only. */
CS_API int cs_image_loss_workspace(int32_t height, int32_t width, size_t *bytes);

/* Training loss.  Replaces losses.image_loss (losses.py:129-155) with
 * ssim_with_grad (losses.py:58-101): (1-lambda) L1 + lambda (1-SSIM)/2 +
 * beta mean(sigmoid(raw_mask)), 11x11 sigma-1.5 Gaussian on the valid region.
 * rendered/target [H,W,3]; d_image [H,W,3] is WRITTEN (d loss / d rendered);
 * d_raw_mask [n] is ACCUMULATED (+=) like trainer.py:176.  stats[9] (device,
 * written): [0] sum |rendered - target|, [1] sum over channels of sum of the
 * SSIM map, [2] sum sigmoid(raw_mask), [3] number of valid SSIM positions per
 * channel; then the values [4] total = (1-lambda) l1 + lambda dssim + beta
 * mask_term, [5] l1 = stats0/(3HW), [6] ssim = stats1/(3 stats3), [7] dssim =
 * (1 - ssim)/2, [8] mask_term = stats2/n. */
CS_API int cs_image_loss(int32_t height, int32_t width, const float *rendered, const float *target,
                         const float *raw_mask, int64_t n, double lambda_dssim, double beta_mask,
                         float *d_image, float *d_raw_mask, double *stats, void *workspace,
                         size_t workspace_bytes, void *stream);

/* One parameter tensor of the Adam update. */
typedef struct cs_adam_tensor {
    float *param;
    const float *grad;
    float *m;
    float *v;
    int64_t numel;
    double lr;
} cs_adam_tensor;

/* optim.Adam.step (optim.py:22-35) over `count` (<= 8) tensors, in place:
 * g = grad_scale * grad; m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
 * p -= lr (m / (1-b1^step)) / (sqrt(v / (1-b2^step)) + eps).
 * `tensors` is a HOST array; step is the 1-based step count. */
CS_API int cs_adam_step(int32_t count, const cs_adam_tensor *tensors, double beta1, double beta2, double eps,
                        int32_t step, double grad_scale, void *stream);

/* ------------------------------------------------------------------------
 * Scene-level operations on the SoA parameters.
 * ---------------------------------------------------------------------- */

/* Writable SoA scene arrays (same shapes as cs_params). */
typedef struct cs_scene_out {
    float *points;            /* [n,k,3] */
    float *raw_delta;         /* [n] */
    float *raw_sigma;         /* [n] */
    float *raw_opacity;       /* [n] */
    float *raw_mask;          /* [n] */
    float *sh;                /* [n,16,3] */
} cs_scene_out;

/* .3dcs checkpoint payload (sceneio.py:251-320): n rows of
 * points(3k) | raw_delta raw_sigma raw_opacity | sh(48) | raw_mask as
 * little-endian float32 (precision 32) or float16 (precision 16, round to
 * nearest even).  unpack: device rows -> SoA arrays; pack: SoA -> rows. */
CS_API int cs_checkpoint_unpack(int32_t precision, int64_t n, int32_t k, const void *rows,
                                const cs_scene_out *out, void *stream);
CS_API int cs_checkpoint_pack(int32_t precision, int64_t n, int32_t k, const cs_scene_out *scene, void *rows,
                              void *stream);

/* density.densify_and_prune settings (density.py:54-105, trainer.py:31-39). */
typedef struct cs_density_config {
    double sigma_threshold;       /* split when signal > threshold (sigma_loss_threshold) */
    double split_scale;           /* split_convex scale */
    double split_sigma_boost;
    double split_opacity_factor;
    double prune_opacity;         /* drop when opacity < prune_opacity */
    double size_limit;            /* drop when diameter > prune_size_fraction * scene_extent */
    int32_t allow_split;          /* iteration <= densify_stop */
    int32_t reserved;
} cs_density_config;

/* Pass 1: per convex, flags bit0 = survivor kept, bit1 = split; child_keep =
 * bitmask of the kept children (split_convex order); surv_count / child_count
 * = the numbers of rows each convex contributes (int64, for the scans). */
CS_API int cs_density_flags(const cs_params *params, const float *signal, const cs_density_config *cfg,
                            uint8_t *flags, uint32_t *child_keep, int64_t *surv_count, int64_t *child_count,
                            void *stream);

/* Pass 2 (after exclusive scans surv_pos / child_pos of the counts and the
 * kept-survivor total n_surv, a device scalar): writes the new scene rows in
 * the reference order -- kept survivors in index order, then the kept
 * children of each split parent -- and index_map (old index, -1 for a child). */
CS_API int cs_density_scatter(const cs_params *params, const cs_density_config *cfg, const uint8_t *flags,
                              const uint32_t *child_keep, const int64_t *surv_pos, const int64_t *child_pos,
                              const int64_t *n_surv, const cs_scene_out *out, int64_t *index_map, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CONVEXSPLAT_B200_H */
