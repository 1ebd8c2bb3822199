/*
 * mfa.h -- C ABI of the B200-native MFA-DVR hot path (libmfa.so).
 *
 * Method: Sun, Lenz, Yu, Peterka, "MFA-DVR: direct volume rendering of MFA
 * models" (arXiv 2204.11762).  "P:n" = line n of the paper text
 * (reference PAPER.md), "S:n" = line n of SPEC.md, "R-n" = a reading of the
 * paper recorded in DESIGN.md §2.  SURVEY.md §8(b) lists these entry points.
 *
 * Conventions shared by every call
 *  - Plain C types only; no C++ or CUDA types cross the boundary.  A stream
 *    argument is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Every call validates its arguments synchronously, before anything is
 *    enqueued, and returns a status.  On a non-OK status nothing was enqueued
 *    and mfa_last_error() returns a message naming the offending argument.
 *  - Work is asynchronous on the given stream; outputs are valid once the
 *    stream reaches the enqueued work.  Asynchronous CUDA faults surface as
 *    MFA_ERR_CUDA on a later call (or at the caller's synchronisation).
 *  - A model is bound to the CUDA device that was current at create time;
 *    calls made while another device is current return MFA_ERR_DEVICE.
 *  - A model is immutable after create: any number of threads and
 *    streams may call eval / render on it concurrently.  The caller
 *    guarantees no work is in flight when it calls mfa_model_destroy.
 *  - The library allocates nothing on the eval / render paths: outputs go to
 *    caller-owned device buffers.
 */
#ifndef MFA_H
#define MFA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mfa_model_t* mfa_model;
typedef void* mfa_stream;

typedef enum {
    MFA_OK = 0,
    MFA_ERR_INVALID_ARG = 1,  /* NULL pointer, bad size, inconsistent shapes */
    MFA_ERR_KNOTS = 2,        /* knot vector violates S:24-27 (length, order, clamping, multiplicity) */
    MFA_ERR_UNSUPPORTED = 3,  /* degree outside {1..5} or unequal per axis; a tiled render of more than
                                 64 views in one call; more than 256 renders of one model in flight
                                 on distinct streams */
    MFA_ERR_DOMAIN = 4,       /* non-finite control value */
    MFA_ERR_CUDA = 5,         /* a CUDA runtime error (message has the CUDA error string) */
    MFA_ERR_OOM = 6,          /* device allocation failed */
    MFA_ERR_DEVICE = 7        /* called with a different current device than the model's */
} mfa_status;

#define MFA_MAX_DEGREE 5

/* ------------------------------------------------------------------------
 * mfa_model_create -- ingest an MFA model.
 *
 * The model is the tensor-product B-spline of P:74 ("a tensor product of
 * nonuniform rational B-spline functions ... represented by a set of control
 * points and knots"), with all weights 1 (R-1) and size proportional to the
 * number of control points.
 *
 * degree[3]   polynomial degree per axis (u, v, w).  This build compiles
 *             degrees 1..5 and requires degree[0]==degree[1]==degree[2];
 *             otherwise MFA_ERR_UNSUPPORTED.
 * nctrl[3]    control-point counts n_u, n_v, n_w; each >= degree+1.
 * knots[3]    host pointers to fp64 knot vectors, length nctrl[d]+degree+1:
 *             nondecreasing, clamped (first and last degree+1 entries are 0
 *             and 1), interior multiplicity <= degree; copied.
 *             Else MFA_ERR_KNOTS with axis and index in the message.
 * ctrl        fp32 control values, u fastest: ctrl[(k*n_v + j)*n_u + i]
 *             (S:115 order); host pointer if ctrl_on_device == 0, else a
 *             device pointer on the current device; copied (the caller may
 *             free it when the call returns).  Non-finite -> MFA_ERR_DOMAIN.
 * stream      stream for the device-side ingest; the call synchronises it
 *             before returning.
 * out         receives the model handle (NULL on failure).
 *
 * Device memory: bricked row quads ~ 16 quad_f4(p) (1 + p/16)^2 n_u n_v n_w
 * bytes (quad_f4 = 2 for p <= 3: 32-byte row pairs, about 45 B per control
 * point at p = 3; 1 for p >= 4), or Bezier blocks (see
 * mfa_model_create_ex), plus per-axis span tables (< 1 MB); mfa_model_info
 * reports device_bytes / model_bytes.
 * ---------------------------------------------------------------------- */
mfa_status mfa_model_create(const int32_t degree[3], const int64_t nctrl[3],
                            const double* const knots[3], const float* ctrl,
                            int32_t ctrl_on_device, mfa_stream stream, mfa_model* out);

/*
 * mfa_model_create_ex -- as mfa_model_create, with options (NULL = defaults).
 * layout: MFA_LAYOUT_AUTO chooses Bezier blocks for degree <= 3 models with a
 *   non-uniform axis, or whose blocks take <= 64 MiB (they then stay in L2);
 *   falling back to quads if the blocks do not fit in device memory; else
 *   bricked row quads.  MFA_LAYOUT_QUADS / _BEZIER force
 *   one (Bezier needs degree <= 3: MFA_ERR_UNSUPPORTED otherwise).
 *   Bezier blocks: for every knot-span triple the (p+1)^3 Bernstein
 *   coefficients of the spline there (Bezier extraction; 256 B per triple for
 *   p = 3), so evaluation needs no per-span basis tables.  Device memory:
 *   4 (p+1)^2 * 4 * S_u S_v S_w bytes (C5: 16.7 GB).
 *   MFA_LAYOUT_BRICKS (degree <= 3, never chosen by AUTO): plain haloed
 *   bricks, one fp32 per control point in bricks of 16^3 knot spans plus the
 *   p halo points, rows padded to 16 bytes: <= 1.86 x the grid (C5: 1.85 x,
 *   473 MB) -- the compact option of P:133 / P:263 (model size proportional to
 *   the control points); the kernels read each neighbourhood row as two
 *   aligned 16-byte loads and shift it (slower than the Bezier blocks).
 *   MFA_LAYOUT_BEZIER_GROUPED (degree 3; what AUTO picks whenever it picks
 *   Bezier blocks at p = 3): the same blocks, 4 consecutive w-spans per
 *   1 KB group interleaved by 32-byte sector (line j of a group = sector j of
 *   its 4 blocks), so neighbouring rays that reload vertically adjacent blocks
 *   in one instruction share cache lines (render +6 % on C5).  Random-point
 *   mfa_eval_batch / mfa_eval_hessian on models far larger than L2 are faster
 *   on MFA_LAYOUT_BEZIER (C5: 10.4 vs 8.0 G points/s); results are identical.
 *   Device memory as MFA_LAYOUT_BEZIER with S_w rounded up to a multiple of 4.
 */
#define MFA_LAYOUT_AUTO 0
#define MFA_LAYOUT_QUADS 1
#define MFA_LAYOUT_BEZIER 2
#define MFA_LAYOUT_BRICKS 3
#define MFA_LAYOUT_BEZIER_GROUPED 4
typedef struct {
    int32_t layout;
} mfa_model_options;

mfa_status mfa_model_create_ex(const int32_t degree[3], const int64_t nctrl[3],
                               const double* const knots[3], const float* ctrl,
                               int32_t ctrl_on_device, const mfa_model_options* opt,
                               mfa_stream stream, mfa_model* out);

typedef struct {
    int32_t degree[3];
    int64_t nctrl[3];
    int32_t uniform[3];     /* 1 if the interior knots are exactly k/S */
    float v_min, v_max;     /* min / max control value (a TF domain default) */
    int64_t device_bytes;   /* device memory owned by the model */
    int32_t device;         /* CUDA ordinal the model lives on */
    int32_t layout;         /* MFA_LAYOUT_QUADS, _BEZIER, _BRICKS or _BEZIER_GROUPED */
    int64_t model_bytes;    /* the fp32 control grid as passed: 4 n_u n_v n_w (the model
                               size depends on the control-point count) */
    double create_ms;       /* wall time of mfa_model_create (validation, upload, relayout,
                               span tables, the closing stream synchronisation) */
} mfa_model_desc;

mfa_status mfa_model_info(mfa_model m, mfa_model_desc* out);

/* Frees the model's device memory.  NULL is accepted (no-op). */
mfa_status mfa_model_destroy(mfa_model m);

/* ------------------------------------------------------------------------
 * mfa_eval_batch -- queryValueMFA / queryGradientMFA for n points
 * (Algorithm 1 lines 6 and 9; "computing all derivatives along
 * the three dimensions at once").
 *
 * u, v, w     device fp32 arrays (SoA) of n parameter-space points in [0,1]^3.
 * value       device fp32 output, n entries (required).
 * du, dv, dw  device fp32 outputs: the PARAMETER-space partials dF/du, dF/dv,
 *             dF/dw (R-4).  All three NULL -> value only (no
 *             derivative work); otherwise all three must be non-NULL.
 * n_domain_errors  optional device counter (unsigned long long); incremented
 *             by the number of points outside [0,1]^3 or NaN.  Those points
 *             get NaN outputs (batched form of S:74's domain error, R-18).
 * n == 0 is valid and enqueues nothing.
 * For n >= 2^16 on a model larger than 64 MiB (one that does not stay in
 * L2; smaller models are gathered directly in input order, which is faster
 * for them) the call takes the binned path of mfa_eval_batch_ws with
 * STREAM-ORDERED scratch (cudaMallocAsync / cudaFreeAsync on `stream` from
 * the device's default memory pool, ~20 B per point; the pool's release
 * threshold is raised once to 8 GiB so the blocks stay cached between calls); if the
 * pool cannot serve it, the unbinned kernel runs instead (same outputs).
 * ---------------------------------------------------------------------- */
mfa_status mfa_eval_batch(mfa_model m, int64_t n, const float* u, const float* v, const float* w,
                          float* value, float* du, float* dv, float* dw,
                          unsigned long long* n_domain_errors, mfa_stream stream);

/*
 * mfa_eval_batch_ws -- mfa_eval_batch with a caller-owned device workspace of
 * at least mfa_eval_workspace_bytes(m, n) bytes (~20 B per point).  For
 * n >= 2^16 (and a model larger than 64 MiB) the points are first grouped by a coarse parameter-space bin
 * (~8^3 knot spans per bin; a counting sort into (u, v, w, index) records)
 * and evaluated in bin order, results written at their original indices:
 * neighbouring points then share control-point neighbourhoods in L1/L2
 * instead of each pulling ~16 separate lines from HBM.  Same outputs as
 * mfa_eval_batch (each point's arithmetic is unchanged); workspace == NULL runs
 * the unbinned kernel (one point per thread in input order).
 */
size_t mfa_eval_workspace_bytes(mfa_model m, int64_t n);
mfa_status mfa_eval_batch_ws(mfa_model m, int64_t n, const float* u, const float* v, const float* w,
                             float* value, float* du, float* dv, float* dw,
                             unsigned long long* n_domain_errors, void* workspace, size_t workspace_bytes,
                             mfa_stream stream);

/* ------------------------------------------------------------------------
 * mfa_eval_hessian -- value, gradient and the six second partials of the MFA
 * at n points ("Higher-order derivatives, up to the
 * polynomial degree, are also analytically available").
 *
 * u, v, w     device fp32 arrays (SoA) of n parameter-space points in [0,1]^3.
 * value       optional device fp32 [n].
 * grad        optional device fp32 [3][n]: dF/du, dF/dv, dF/dw (parameter space).
 * hess        device fp32 [6][n] (required): d2F/du2, d2F/dv2, d2F/dw2,
 *             d2F/dudv, d2F/dudw, d2F/dvdw (parameter space).
 * n_domain_errors, errors, n == 0: as mfa_eval_batch (NaN outputs for points
 * outside [0,1]^3).  Async on stream.  For n >= 2^16 the binned path runs with
 * stream-ordered scratch (~68 B per point), as mfa_eval_batch.
 * ---------------------------------------------------------------------- */
mfa_status mfa_eval_hessian(mfa_model m, int64_t n, const float* u, const float* v, const float* w,
                            float* value, float* grad, float* hess,
                            unsigned long long* n_domain_errors, mfa_stream stream);

/* mfa_eval_hessian with a caller-owned workspace of at least
 * mfa_hessian_workspace_bytes(m, n) bytes (~68 B per point): large batches are
 * spatially binned first (as mfa_eval_batch_ws); identical outputs. */
size_t mfa_hessian_workspace_bytes(mfa_model m, int64_t n);
mfa_status mfa_eval_hessian_ws(mfa_model m, int64_t n, const float* u, const float* v, const float* w,
                               float* value, float* grad, float* hess,
                               unsigned long long* n_domain_errors, void* workspace, size_t workspace_bytes,
                               mfa_stream stream);

/* ------------------------------------------------------------------------
 * mfa_render -- Algorithm 1 for every pixel of n_views views.
 *
 * Per pixel: a ray through the pixel centre (R-14 camera), clipped to
 * the box (l.2-3), samples at t_in + (k+1/2)*step (constant
 * distance; R-7), normalised to [0,1]^3 (l.5), value and
 * gradient queried (l.6, l.9), transfer function (l.7), Phong shading with a
 * headlight (l.10-11; R-11), front-to-back compositing (l.13) and early ray
 * termination when A > o_max (l.14-15; R-13).  Output is premultiplied RGBA
 * (C_r, C_g, C_b, A), background (0,0,0,0) (l.18; R-12).
 * ---------------------------------------------------------------------- */
typedef struct {
    double eye[3], look_at[3], up[3];
    double fov_y_deg;          /* > 0 perspective vertical field of view; 0 -> orthographic */
    double ortho_half_height;  /* half height of the orthographic viewport (world units) */
    int32_t width, height;     /* pixels; all views of one call share width and height */
} mfa_camera;

typedef struct {
    const float* rgba;         /* device, n_entries x {r,g,b,a}, non-premultiplied */
    int32_t n_entries;         /* 2 .. 1024 */
    float v_lo, v_hi;          /* value domain mapped onto the table (v_hi > v_lo) */
} mfa_tf;

typedef struct {
    double box_min[3], box_max[3];   /* world placement of the parameter cube */
    double step;                     /* sample distance, world units (> 0) */
    double o_max;                    /* ERT threshold O_Max (l.14); >= 1 disables ERT */
    int32_t shading;                 /* ShadingOn (l.8): 0 off (value only), 1 on (the gradient is
                                        queried for every sample, R-20), 2 on with the gradient and
                                        Phong skipped for samples whose TF opacity is 0 (NEXT-1's
                                        variant: they composite with weight 0, so the image and the
                                        sample count equal shading = 1's; degree <= 3 models, other
                                        layouts run shading = 1), 3 on with whole samples skipped
                                        (no block fetch, value, gradient or Phong) where the TF opacity
                                        is 0 over the value range of the sample's 2^3-span macro block
                                        (Bezier layout: the convex hull of its Bernstein coefficients;
                                        image and sample count again equal shading = 1's; other layouts
                                        run shading = 1) */
    double ka, kd, ks, shininess;    /* Phong constants */
    double grad_eps;                 /* |physical gradient| <= grad_eps -> ambient only (R-11) */
    int32_t out_fp16;                /* 0: fp32 RGBA (16 B/px); 1: fp16 RGBA (8 B/px) */
} mfa_render_params;

#define MFA_TILE 16

typedef struct {
    int64_t n_tiles;
    const int32_t* tiles;      /* device, n_tiles x {view, tile_x, tile_y}, 16x16-pixel tiles.
                                  Contract: 0 <= view < n_views (of this call, at most 64),
                                  0 <= tile_x < ceil(W/16), 0 <= tile_y < ceil(H/16); view < 0
                                  marks a padding entry.  Padding and any entry outside that
                                  range are skipped by the kernels (never read frames or store
                                  outside the image); listing a tile twice renders it twice. */
    int32_t scatter;           /* 0: rgba_out is the packed [n_tiles][16][16][4] buffer;
                                  1: each pixel is stored at its image position, rgba_out is
                                  [n_views][H][W][4] -- which may be another GPU's image mapped
                                  through CUDA IPC / peer access: the multi-GPU direct-store path
                                  (stores travel over NVLink as the tiles finish; no gather) */
} mfa_tiles;

/*
 * cams        HOST array of n_views cameras (copied into the launch).
 * tf, prm     host structs (tf->rgba is a device pointer).
 * tiles       NULL: render every pixel; rgba_out is [n_views][H][W][4].
 *             non-NULL: render only the listed 16x16 tiles; rgba_out is the
 *             packed buffer [n_tiles][16][16][4] (scatter = 0; pixels outside
 *             the image are left untouched) or the full image (scatter = 1).
 *             Used for screen-tile sharding across GPUs.
 * rgba_out    device buffer, fp32 or fp16 per prm->out_fp16.
 * samples_out optional device counter: += the number of composited samples
 *             (each sample up to and including the ERT sample).
 * Deterministic: a pixel's value does not depend on tiling, view batching or
 * launch configuration.  Each launch owns one of the model's 256 work-counter
 * slots until its completion event fires (launches on the same stream reuse
 * one slot in stream order); a launch that finds every slot held by an
 * unfinished launch on another stream fails with MFA_ERR_UNSUPPORTED and
 * enqueues nothing.
 * Stream capture: the call enqueues only a memset, the kernel and an event
 * record, so it can be captured into a CUDA graph (tests/test_gpu_parity.py
 * checks that a replay is bit-identical to the eager call).  A replayed
 * graph reuses the slot it was captured with: do not replay it concurrently
 * with other renders of the same model on other streams.
 */
mfa_status mfa_render(mfa_model m, int32_t n_views, const mfa_camera* cams, const mfa_tf* tf,
                      const mfa_render_params* prm, const mfa_tiles* tiles, void* rgba_out,
                      unsigned long long* samples_out, mfa_stream stream);

/*
 * mfa_render_host -- the same frame(s) as mfa_render (tiles == NULL), with
 * HOST buffers: tf_rgba_host (n_entries x 4 fp32) is copied in, and the image
 * [n_views][H][W][4] (fp32 or fp16 per prm->out_fp16) is written to
 * rgba_host, view by view, with the device->host copy of view v overlapping
 * the rendering of view v+1 (two device staging buffers, the caller's stream
 * and a copy stream).  The staging buffers, copy stream, events and the
 * device TF / counter are owned by the MODEL: created on the first call
 * (2 x one view of device memory), reused by later calls, freed by
 * mfa_model_destroy; host-buffer renders of one model are serialised (a
 * mutex).  rgba_host should be page-locked for the copies to overlap.
 * samples_host (optional) receives the composited-sample count.  Returns
 * after the image is on the host.
 */
mfa_status mfa_render_host(mfa_model m, int32_t n_views, const mfa_camera* cams,
                           const float* tf_rgba_host, int32_t tf_n_entries, float v_lo, float v_hi,
                           const mfa_render_params* prm, void* rgba_host,
                           unsigned long long* samples_host, mfa_stream stream);

/*
 * mfa_render_host_views -- mfa_render_host with one host destination per view
 * (rgba_host_views[v] receives view v, [H][W][4]); e.g. the views a rank of a
 * multi-GPU job renders, written straight into their slots of a host image
 * shared by all ranks.  Same ownership, overlap and errors as mfa_render_host.
 */
mfa_status mfa_render_host_views(mfa_model m, int32_t n_views, const mfa_camera* cams,
                                 const float* tf_rgba_host, int32_t tf_n_entries, float v_lo, float v_hi,
                                 const mfa_render_params* prm, void* const* rgba_host_views,
                                 unsigned long long* samples_host, mfa_stream stream);

/*
 * mfa_unpack_tiles -- scatter a packed tile buffer [n_tiles][16][16][4] (as
 * written by mfa_render with tiles) into images [n_views][H][W][4] (fp32).
 * in_fp16 selects the packed element type.  Device pointers.
 */
mfa_status mfa_unpack_tiles(const void* packed, int32_t in_fp16, const int32_t* tiles, int64_t n_tiles,
                            int32_t n_views, int32_t width, int32_t height, float* image_out,
                            mfa_stream stream);

/* ------------------------------------------------------------------------
 * Ground truth and image quality (§4.1.1 and
 * §4.2.1: "we generate the ground truth volume rendering image by computing
 * the value and gradient analytically from the synthetic functions for the
 * samples on rays.  Metrics of image quality include mean squared error
 * (MSE), peak signal-to-noise ratio (PSNR), and structural similarity index
 * (SSIM)").
 * ---------------------------------------------------------------------- */
#define MFA_FIELD_GAUSSIAN_BEAM 1   /* Eq. 1: prm = {V_min, V_max, mu, sigma, R} */
#define MFA_FIELD_MARSCHNER_LOBB 2  /* Eq. 2: prm = {f_M, alpha} */
#define MFA_SRC_MODEL 0
#define MFA_SRC_ANALYTIC 1

typedef struct {
    int32_t kind;        /* MFA_FIELD_* ; the function is defined on x, y, z in [-1,1] and
                            evaluated at x = 2u - 1 of the sample's parameter point u */
    int32_t value_src;   /* MFA_SRC_MODEL: value from the MFA query; MFA_SRC_ANALYTIC: from the field */
    int32_t grad_src;    /* the same for the gradient (the paper's gradient-only test takes the
                            analytic value and the MFA gradient) */
    double prm[6];
} mfa_field;

/*
 * mfa_render_field -- mfa_render with each sample's value and/or gradient
 * taken from the analytic field (fp64 evaluation) instead of the MFA query.
 * Rays, sample positions, TF, shading, compositing and ERT are exactly those
 * of mfa_render, so value_src = grad_src = MFA_SRC_ANALYTIC is the ground-truth
 * image of the same view, and value_src = ANALYTIC, grad_src = MODEL is the
 * gradient-accuracy image of P:209.  field == NULL or both sources MODEL is
 * mfa_render.  Same arguments, layout, ownership and errors as mfa_render;
 * an unknown field->kind returns MFA_ERR_INVALID_ARG.
 */
mfa_status mfa_render_field(mfa_model m, int32_t n_views, const mfa_camera* cams, const mfa_tf* tf,
                            const mfa_render_params* prm, const mfa_field* field, const mfa_tiles* tiles,
                            void* rgba_out, unsigned long long* samples_out, mfa_stream stream);

/*
 * mfa_render_ex -- mfa_render with the extensions, any combination of:
 *  field        as mfa_render_field (NULL: the MFA query only);
 *  n_lights     0: the headlight of mfa_render (R-11); 1..MFA_MAX_LIGHTS:
 *               directional lights ("multiple light sources can
 *               be added in the future").  light_dir: host fp64
 *               [n_lights][3] world-space directions TOWARDS each light
 *               (normalised here); light_intensity: host fp64 [n_lights].
 *               Phong per light l (R-30): c = clamp(rgb (k_a + k_d sum_l I_l
 *               max(0, N.L_l)) + k_s sum_l I_l [N.L_l > 0] max(0, R_l.V)^n),
 *               V = -d, R_l = 2 (N.L_l) N - L_l; zero gradient -> k_a rgb.
 *               One light L = -d, I = 1 reproduces the headlight.
 * ext == NULL is mfa_render.  Errors as mfa_render; bad lights ->
 * MFA_ERR_INVALID_ARG.  The extended kernels are separate instantiations:
 * mfa_render's hot path carries none of this.
 */
#define MFA_MAX_LIGHTS 8
typedef struct {
    const mfa_field* field;
    int32_t n_lights;
    const double* light_dir;
    const double* light_intensity;
    /* curvature transfer function (Kindlmann et al.'s curvature-based TF, named
       in P:100 as an application of the higher derivatives of P:78; R-31):
       curv_rgba: device fp32 [curv_n][curv_n][4], indexed [kappa_2][kappa_1]
       over [-curv_range, curv_range]^2 (bilinear, clamped); each sample's TF
       colour and opacity are multiplied by it.  kappa_1 >= kappa_2 are the
       principal curvatures (physical units) of the MFA's isosurface through
       the sample, from the MFA gradient and Hessian (n = -g/|g|); a sample with
       |g| <= grad_eps takes kappa = (0, 0).  curv_n = 0: off; else >= 2. */
    const float* curv_rgba;
    int32_t curv_n;
    double curv_range;
} mfa_render_ext;

mfa_status mfa_render_ex(mfa_model m, int32_t n_views, const mfa_camera* cams, const mfa_tf* tf,
                         const mfa_render_params* prm, const mfa_render_ext* ext, const mfa_tiles* tiles,
                         void* rgba_out, unsigned long long* samples_out, mfa_stream stream);

/*
 * mfa_image_quality -- MSE, PSNR and SSIM of image a against image b.
 *
 * img_a, img_b  device fp32 [height][width][4] premultiplied RGBA (mfa_render's
 *               output); alpha is ignored: the displayed colour is RGB over
 *               black, quantised to 8-bit levels q = floor(255 clamp(x,0,1) + 1/2).
 * err_map       optional device fp32 [height][width]: per-pixel Euclidean RGB
 *               error in 8-bit levels (the Fig. 6 error distribution).
 * workspace     device scratch of at least mfa_image_quality_workspace(width,
 *               height) bytes (caller-owned; nothing is allocated here).
 * out3          device fp64[3]: {MSE over pixels x 3 channels, PSNR = 10
 *               log10(255^2/MSE) (+inf if MSE == 0), mean SSIM}.  SSIM: luma
 *               0.299 R + 0.587 G + 0.114 B, 11x11 Gaussian window sigma 1.5,
 *               C1 = (0.01*255)^2, C2 = (0.03*255)^2, every window position
 *               inside the image (readings R-22, after SPEC S:469-516).
 * fp64 throughout; deterministic (fixed reduction order).  Async on stream.
 * width or height < 11: MFA_ERR_INVALID_ARG (and the workspace size is 0).
 */
size_t mfa_image_quality_workspace(int32_t width, int32_t height);
mfa_status mfa_image_quality(int32_t width, int32_t height, const float* img_a, const float* img_b,
                             float* err_map, void* workspace, size_t workspace_bytes, double* out3,
                             mfa_stream stream);

/* ------------------------------------------------------------------------
 * Encoder (PAPER.md P:74-76 and the Fig. 1 caption
 * "New control points and knots are added adaptively until all
 * evaluated points in each span of knots are within the allowable maximum
 * relative error of the original points ... knot spans that fall beyond the
 * tolerance are subdivided, and MFA is recomputed").
 *
 * Input: a structured grid, device fp32 values[m_w][m_v][m_u] (u fastest),
 * sample (i,j,k) at parameters (i/(m_u-1), j/(m_v-1), k/(m_w-1)) (R-27).
 * ---------------------------------------------------------------------- */

/*
 * mfa_fit_grid -- least-squares control values for given knots: the
 * minimiser of || (N_w (x) N_v (x) N_u) c - q ||_2 (computed separably, exact
 * for the tensor-product problem), fp64 arithmetic.
 * dims[3]     m_u, m_v, m_w (each in [2, 2^20]).
 * degree      1..5; nctrl[d] in [degree+1, dims[d]]; knots[d] host fp64 clamped
 *             knot vectors, length nctrl[d]+degree+1.
 * ctrl_out    device fp32 [n_w][n_v][n_u] (required); ctrl_out64 optional
 *             device fp64 copy.  A knot layout that leaves a basis function
 *             without samples makes the normal equations singular:
 *             MFA_ERR_INVALID_ARG naming the axis.  A non-finite input
 *             value: MFA_ERR_DOMAIN (checked before any fit).  Scratch is allocated
 *             internally (not a render-path call) from the device's default
 *             stream-ordered memory pool, whose release threshold is raised to
 *             8 GiB once per device so repeated fits / refinement rounds reuse
 *             it; returns after the stream is synchronised.
 */
mfa_status mfa_fit_grid(const int64_t dims[3], const float* values, int32_t degree, const int64_t nctrl[3],
                        const double* const knots[3], float* ctrl_out, double* ctrl_out64, mfa_stream stream);

typedef struct {
    int32_t degree;          /* 1..5, all axes */
    int64_t nctrl_init[3];   /* initial control counts (clamped uniform knots), >= degree+1 */
    double e_max;            /* allowable maximum relative error |f - q| / (max q - min q) */
    int32_t max_rounds;      /* refinement rounds after the first fit (0: fit once) */
    int64_t max_ctrl[3];     /* per-axis control-count caps (also capped at dims[d]) */
} mfa_encode_config;

typedef struct {
    int64_t nctrl[3];        /* control counts of the returned model */
    int32_t rounds;          /* fits performed */
    int32_t converged;       /* 1 if the max relative error <= e_max */
    double max_err, rms_err; /* relative errors of the returned fit at the input samples */
} mfa_encode_result;

/*
 * mfa_encode_grid -- the adaptive encoder: fit, evaluate at every sample,
 * per axis and knot span the max relative error over the samples in that
 * span; split every span above e_max holding >= 2(p+1) samples at its midpoint
 * (within the caps) and refit, until the max error <= e_max, max_rounds, or
 * nothing can be split (R-28).
 * knots_out[d]  host fp64, capacity max_ctrl[d]+degree+1: the final knots.
 * ctrl_out      device fp32, capacity prod(max_ctrl): the final control values
 *               [n_w][n_v][n_u] with n = res->nctrl.
 * round_log     optional host fp64 [(max_rounds+1)][5]: per fit n_u, n_v, n_w,
 *               max error, rms error.
 * Deterministic except for the rms summation order.  Synchronous.  A
 * non-finite input value: MFA_ERR_DOMAIN before the first fit.
 */
mfa_status mfa_encode_grid(const int64_t dims[3], const float* values, const mfa_encode_config* cfg,
                           double* const knots_out[3], float* ctrl_out, mfa_encode_result* res,
                           double* round_log, mfa_stream stream);

/*
 * mfa_enable_peer_access -- let kernels on the current device load / store
 * memory of peer_device (cudaDeviceEnablePeerAccess): the direct-store
 * multi-GPU path writes rank 0's image (mapped through CUDA IPC) from every
 * rank's render kernel over NVLink.  Same device or already enabled: MFA_OK;
 * no P2P path between the devices: MFA_ERR_DEVICE.
 */
mfa_status mfa_enable_peer_access(int32_t peer_device);

/*
 * mfa_ipc_open -- map another process's device allocation into the CURRENT
 * device's address space (cudaIpcOpenMemHandle with
 * cudaIpcMemLazyEnablePeerAccess), for the direct-store multi-GPU path: every
 * rank maps rank 0's image allocation on its own device, so its render kernel
 * stores into it over NVLink (or locally when both are the same device).
 * handle     host, the 64-byte cudaIpcMemHandle_t of the exporting process's
 *            allocation (e.g. torch's UntypedStorage._share_cuda_()[1]).
 * base_out   receives the device address of the allocation's first byte in
 *            this process (add the exporter's byte offset of the tensor).
 * The mapping stays until mfa_ipc_close(base).  NULL arguments:
 * MFA_ERR_INVALID_ARG; a handle this process cannot map (same process, no
 * P2P path, bad handle): MFA_ERR_CUDA with the CUDA error text.
 */
mfa_status mfa_ipc_open(const void* handle, void** base_out);

/* mfa_ipc_close -- unmap an allocation mapped by mfa_ipc_open. */
mfa_status mfa_ipc_close(void* base);

/*
 * mfa_ipc_alloc -- allocate `bytes` of device memory on the CURRENT device
 * (cudaMalloc: a whole allocation, so its IPC handle maps exactly this
 * buffer) and export it: *ptr_out = the device pointer, handle_out (64
 * bytes, caller-owned) = its cudaIpcMemHandle_t for mfa_ipc_open in another
 * process.  Used for the multi-GPU direct-store image (rank 0's image that
 * every rank's render kernel stores into over NVLink).  The caller owns the
 * buffer: mfa_ipc_free(ptr) after every mapping process has closed it.
 * Errors: MFA_ERR_INVALID_ARG (NULL outputs, bytes == 0), MFA_ERR_OOM,
 * MFA_ERR_CUDA (export failed).
 */
mfa_status mfa_ipc_alloc(size_t bytes, void** ptr_out, void* handle_out);
mfa_status mfa_ipc_free(void* ptr);

/* Thread-local message for the last non-OK status on this thread ("" if none). */
const char* mfa_last_error(void);

/* Library version string, e.g. "mfa-b200 0.1 sm_100a". */
const char* mfa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MFA_H */
