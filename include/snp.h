/*
 * snp.h -- C ABI of the B200 (sm_100a) forward splatting rasterizer for
 * splattable neural primitives (arXiv 2510.08491).
 *
 * Citation key: P:n = PAPER.md line n (section / equation named beside it),
 * S:n = SPEC.md line n, R<k> = reading k in DESIGN.md "Readings of the paper".
 *
 * The problem statement (Sec. 3.1 "Representation"): render the
 * radiance field given by primitives {P_i}; each P_i is an ellipsoid (centre mu,
 * scale s along its principal axes, rotation quaternion q) holding a density
 * field sigma(x) = f((x - mu)/||s||_inf) (Eq. 5), f a one-hidden-layer cosine
 * MLP of width N with frequency omega (Eq. 6), and a view-dependent colour from
 * spherical harmonics.  A pixel's colour is Eq. 4 alpha blending
 * of kappa = 1 - exp(-max(0, I)) (Eq. 9), I the closed-form line integral of
 * sigma over the ray's segment inside the ellipsoid (Eq. 7-8), over the
 * depth-sorted primitives the ray hits.
 *
 * Pipeline (each call asynchronous on the caller's CUDA stream):
 *   snp_create_scene  copy + validate primitives           (a1 ingest)
 *   snp_project       K1a project/cull + tile rect + depth key per (view,
 *                     primitive); K1b render records, forked onto the scene's
 *                     internal stream                      (a2)
 *   snp_bin_sort      K2 one-pass key duplication, K3 onesweep radix sort,
 *                     K4 tile ranges, tile order; joins K1b (a3-a5)
 *   snp_render        K5 per-pixel integral + blend, K6 exact fallback (a6)
 *   snp_destroy
 * Stages must run in this order; re-projecting invalidates later stages.  The
 * fork/join of K1b uses events, so a sequence of calls on one stream may be
 * captured into a CUDA graph (snp_bin_sort with sync_check = 0).
 *
 * Conventions: all arrays are fp32, row-major, structure-of-arrays over
 * primitives.  Quaternions are (w,x,y,z), normalised on read (R8); scales are
 * ellipsoid semi-axes in world units (R7).  Camera: pinhole, looks along +z,
 * x right, y down; R_wc is the world-from-camera rotation; the ray of pixel
 * (x, y) passes through the pixel centre (x + 0.5, y + 0.5) (R6).
 *
 * Errors: every call returns an snp_status.  Argument checks are synchronous
 * and launch nothing.  CUDA launch/async errors surface as SNP_ERR_CUDA from the
 * call that observes them.  snp_last_error() returns a thread-local message,
 * valid until the next snp_* call on that thread.  A scene handle is not
 * thread-safe; distinct handles are independent.
 */
#ifndef SNP_H
#define SNP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SNP_OK = 0,
    SNP_ERR_INVALID_ARGUMENT = 1,  /* null pointer, bad size, |q| = 0, s <= 0, non-finite value */
    SNP_ERR_OUT_OF_MEMORY = 2,
    SNP_ERR_CUDA = 3,
    SNP_ERR_UNSUPPORTED = 4,       /* e.g. n_hidden not in {4, 8, 16, 32} */
    SNP_ERR_BAD_STATE = 5,         /* stage called out of order */
    SNP_ERR_CAPACITY = 6           /* reserved (no-sync capacity overflow is reported by snp_get_stats) */
} snp_status;

typedef struct snp_scene_s *snp_scene;  /* opaque, owned by the library */

/* SNP_MEM_HOST_ASYNC (snp_render output only): host memory, written by a copy
 * enqueued on the call's stream without synchronising -- the buffer should be
 * pinned, and is valid once the caller has synchronised that stream. */
enum { SNP_MEM_HOST = 0, SNP_MEM_DEVICE = 1, SNP_MEM_HOST_ASYNC = 2 };

/* Colour of a primitive (snp_render_opts.colour_mode): its SH colour
 * c = max(0, sum_lm Y_lm(dir) sh_lm + 0.5) evaluated at
 *   SNP_COLOUR_PRIMITIVE: dir = normalize(mu - C), once per primitive and view (the 3DGS
 *                         convention; R14) -- the default and the measured mode;
 *   SNP_COLOUR_RAY:       dir = the pixel's own unit ray direction d, per (ray, hit). */
enum { SNP_COLOUR_PRIMITIVE = 0, SNP_COLOUR_RAY = 1 };

/* One primitive = 99 fp32 parameters for N = 8 ("99 parameters in total";
 * P:751 "41 parameters from its 8-neuron MLP"). */
typedef struct {
    int64_t n;               /* number of primitives, 0 <= n < 2^24 (0 renders background;
                                larger n: SNP_ERR_UNSUPPORTED) */
    int32_t n_hidden;        /* N_sigma: 4, 8 (the paper's), 16 or 32; w1 is [n][N][3],
                                b1 and w2 [n][N] */
    int32_t sh_degree;       /* 0..3; 3 = four bands, 16 coefficients */
    float omega;             /* frequency multiplier, 30 in the paper; > 0 */
    int32_t memory;          /* SNP_MEM_HOST or SNP_MEM_DEVICE (device of the scene) */
    const float *centers;    /* [n][3]    mu */
    const float *rotations;  /* [n][4]    q = (w,x,y,z), any nonzero norm */
    const float *scales;     /* [n][3]    s, ellipsoid semi-axes, > 0 */
    const float *w1;         /* [n][N][3] W1 of Eq. 6 */
    const float *b1;         /* [n][N]    b1 */
    const float *w2;         /* [n][N]    W2 */
    const float *b2;         /* [n]       b2 */
    const float *sh;         /* [n][16][3] SH coefficients, coefficient-major, RGB innermost */
} snp_scene_desc;

typedef struct {
    float R_wc[9];           /* world-from-camera rotation, row-major */
    float C_w[3];            /* camera centre = ray origin o */
    float fx, fy, cx, cy;    /* pinhole intrinsics in pixels, fx, fy > 0 */
    int32_t width, height;   /* image size, 1..32767 */
    float t_near, t_far;     /* ray segment [t_n, t_f] of Eq. 1 along the unit ray; 0 <= t_near < t_far */
} snp_camera;

typedef struct {
    float background[3];        /* added as T_final * bg (R16) */
    float transmittance_floor;  /* stop compositing once T < floor; 1e-4 */
    int32_t tile_row_begin;     /* image-stripe partition: only tile rows r = begin + k*stride */
    int32_t tile_row_stride;    /*   are binned/rendered; (0, 1) = whole image */
    int32_t out_memory;         /* snp_render output: SNP_MEM_DEVICE, SNP_MEM_HOST or SNP_MEM_HOST_ASYNC */
    int32_t sync_check;         /* snp_bin_sort: 1 = synchronise once to size the key buffer
                                   exactly (default); 0 = never synchronise (CUDA-graph safe):
                                   keys beyond an undersized buffer are dropped (the frame is
                                   then incomplete) and snp_get_stats reports
                                   capacity_overflow = 1; a call with 1 resizes */
    int32_t colour_mode;        /* snp_render: SNP_COLOUR_PRIMITIVE (0) or SNP_COLOUR_RAY */
} snp_render_opts;

typedef struct {
    uint64_t n_visible;        /* (view, primitive) pairs surviving K1 */
    uint64_t n_dup;            /* duplicated (tile, primitive) keys of the last bin_sort */
    uint64_t key_capacity;     /* current key buffer capacity */
    uint64_t tested_pairs;     /* (pixel, listed primitive) pairs visited by K5 */
    uint64_t candidate_pairs;  /* pairs passing the silhouette pre-test */
    uint64_t hit_pairs;        /* exact ray-ellipsoid hits */
    uint64_t composited;       /* kernels blended into pixels */
    uint64_t overflow_pixels;  /* pixels re-rendered by the exact fallback K6 */
    uint64_t capacity_overflow;/* 1 if the last no-sync bin_sort overflowed the key buffer */
    uint64_t backward_skipped; /* pixels the last snp_render_backward skipped (more than 16384
                                  hits on the ray: no gradient from them); 0 otherwise */
    uint64_t dead_keys;        /* keys of the last bin_sort that SNP_BIN_CONIC_TILES found
                                  outside the silhouette (sorted last, never rendered) */
} snp_stats;

/* Library version string. */
const char *snp_version(void);

/* Copies and validates the primitives: every q must have nonzero
 * norm, every s > 0, every value finite.  `device` is the CUDA device ordinal;
 * `cuda_stream` (cudaStream_t, may be NULL) orders the copies.  Structural
 * checks (NULL, n < 0, n_hidden, sh_degree, omega) run on the host and launch
 * nothing; the values are validated on the device after the copy (one
 * reduction kernel + one stream synchronisation) and a bad primitive returns
 * SNP_ERR_INVALID_ARGUMENT naming its index.  The caller may free its arrays on
 * return. */
snp_status snp_create_scene(const snp_scene_desc *desc, int device, void *cuda_stream, snp_scene *out);

/* Replaces the parameter values of an existing scene (same n; same validation
 * and memory rules as snp_create_scene) without reallocating.  Later stages must
 * be re-run (snp_project first). */
snp_status snp_update_scene(snp_scene s, const snp_scene_desc *desc, void *cuda_stream);

/* K1 for n_views cameras (all with the same width/height, 1 <= n_views <= 4096):
 * per (view, primitive): frustum cull, exact silhouette bbox -> 16x16 tile rect,
 * depth lower bound key, and the render record (camera-relative centre in
 * compensated hi/lo form, whitening matrix, SH colour, omega-scaled MLP).
 * `cams` is host memory, read before return. */
snp_status snp_project(snp_scene s, const snp_camera *cams, int32_t n_views, void *cuda_stream);

/* Temporal scenes (appendix "Dynamic scenes"; R24): time is
 * a fourth input of each primitive's network, so at a view's timestamp xi_t the phase of
 * hidden unit k is omega (W1_k . x^ + xi_t W_t,k + b1_k).  snp_set_temporal attaches the
 * temporal weights w_t [n][N] (host or device memory as `memory` says, copied; validated
 * finite, SNP_ERR_INVALID_ARGUMENT otherwise) -- NULL detaches them (static scene).
 * snp_project_at is snp_project with one timestamp per view (xi_t: host [n_views], read
 * before return; NULL = all 0).  The time-dependent colour model of the appendix is not
 * specified closely enough to implement: pass the colour at the view's time as SH. */
snp_status snp_set_temporal(snp_scene s, const float *w_t, int32_t memory, void *cuda_stream);
snp_status snp_project_at(snp_scene s, const snp_camera *cams, int32_t n_views, const float *xi_t,
                          void *cuda_stream);
/* Training temporal scenes: snp_render_backward also ADDS dL/dW_t into grad_w_t (device
 * [n][N], caller-owned and zeroed; NULL = not computed) while temporal weights are set. */
snp_status snp_set_temporal_grad(snp_scene s, float *grad_w_t);

/* K2-K4: keys (view | tile | depth) in primitive order, stable LSD radix sort,
 * per-(view, tile) ranges.  Uses opts->tile_row_begin/stride and sync_check. */
snp_status snp_bin_sort(snp_scene s, const snp_render_opts *opts, void *cuda_stream);

/* K5 (+K6): writes out_rgba[n_views][height][width][4] fp32 (R, G, B, opacity =
 * 1 - T).  out_rgba is device memory (or host memory when opts->out_memory is
 * SNP_MEM_HOST -- the call then synchronises -- or SNP_MEM_HOST_ASYNC -- the copy
 * is only enqueued).  Device output: pixels outside the stripe are left untouched;
 * host output: they are written as 0. */
snp_status snp_render(snp_scene s, const snp_render_opts *opts, float *out_rgba, void *cuda_stream);

/* Backward of snp_render: given
 * grad_rgba = dL/d(out_rgba) [n_views][height][width][4] (device), ADDS the gradients
 * of every primitive into grad_w1 [n][N][3], grad_b1 [n][N], grad_w2 [n][N], grad_b2 [n],
 * grad_sh [n][16][3] and -- when grad_centers is not NULL -- grad_centers [n][3],
 * grad_rotations [n][4], grad_scales [n][3] (device; the caller zeroes them; the three
 * geometry pointers are all NULL or all set).  The per-ray hit order and the T < floor
 * stop are piecewise constant and carry no gradient; the I <= 0 clamp of Eq. 9 has
 * gradient 0.  Call after snp_bin_sort of the same frame, with the same opts as the
 * snp_render it differentiates (background, transmittance_floor, colour_mode); the
 * whole image only (tile_row_begin = 0, tile_row_stride = 1), else SNP_ERR_UNSUPPORTED.
 * Every pixel is differentiated up to 16384 hits per ray (beyond 2048 through a
 * global-memory pass); pixels with more are skipped and counted in
 * snp_stats.backward_skipped (reset by every call). */
snp_status snp_render_backward(snp_scene s, const snp_render_opts *opts, const float *grad_rgba, float *grad_w1,
                               float *grad_b1, float *grad_w2, float *grad_b2, float *grad_sh, float *grad_centers,
                               float *grad_rotations, float *grad_scales, void *cuda_stream);
/* As snp_render_backward, given fwd_rgba = the out_rgba (device) of the snp_render of the
 * same binning and opts that the gradients refer to (NULL: rendered again internally).
 * The backward re-runs K5's traversal in gradient mode (each composited hit yields dL/dI
 * and dL/dc from fwd_rgba and its transmittance), then the per-hit parameter gradients;
 * pixels K5 hands to its fallbacks are differentiated by the per-pixel K7. */
snp_status snp_render_backward_ex(snp_scene s, const snp_render_opts *opts, const float *fwd_rgba,
                                  const float *grad_rgba, float *grad_w1, float *grad_b1, float *grad_w2,
                                  float *grad_b2, float *grad_sh, float *grad_centers, float *grad_rotations,
                                  float *grad_scales, void *cuda_stream);

/* Training step.  The paper trains with
 * 3DGS's loss plus a std(s) regulariser and Adam.
 * snp_loss_l1: L = sum |out_rgb - target_rgb| / (3 n_pixels) over device out_rgba
 *   [n_pixels][4] and target_rgb [n_pixels][3]; writes grad_rgba = dL/d(out_rgba) (alpha
 *   channel 0) and ADDS L to the device float *loss.
 * snp_loss_3dgs: 3DGS's loss L = (1 - lambda) L1 + lambda (1 - SSIM) ("the same loss
 *   function as 3DGS"; 3DGS uses lambda = 0.2), SSIM per channel over 11x11 Gaussian windows
 *   (sigma 1.5, zero padding), C1 = 0.01^2, C2 = 0.03^2, averaged over views, pixels and
 *   channels (R25); images [n_views][height][width] (out RGBA, target RGB, device);
 *   writes grad_rgba = dL/d(out_rgba) (alpha 0), ADDS L to *loss.  Scratch buffers belong to
 *   the scene handle s (48 floats per pixel). lambda outside [0, 1]: SNP_ERR_INVALID_ARGUMENT.
 * snp_scale_regularizer: R = weight * mean_i std(s_i) (population std of the semi-axes);
 *   ADDS dR/ds to grad_scales [n][3] and R to *loss (device).
 * snp_adam_step: one Adam step (bias-corrected) on every parameter array of the scene, in
 *   place: grads[8] and lr[8] follow snp_scene_desc's array order (centers, rotations,
 *   scales, w1, b1, w2, b2, sh); the semi-axes are stepped in log space (dL/dlog s =
 *   s dL/ds), so they stay positive; the moments live in the scene (zero at the first
 *   call); step >= 1 counts calls.  Later stages must be re-run (snp_project first). */
snp_status snp_loss_l1(const float *out_rgba, const float *target_rgb, int64_t n_pixels, float *grad_rgba, float *loss,
                       void *cuda_stream);
snp_status snp_loss_3dgs(snp_scene s, const float *out_rgba, const float *target_rgb, int32_t n_views, int32_t height,
                         int32_t width, float lambda_dssim, float *grad_rgba, float *loss, void *cuda_stream);
/* snp_loss_3dgs over n_views of a training step of step_views (>= n_views)
 * views: the means (loss and gradient) divide by step_views x height x width, and the
 * constant of (1 - SSIM) is taken in proportion, so that the parts of a step taken one
 * camera batch at a time add up to snp_loss_3dgs over the whole step.  step_views <
 * n_views: SNP_ERR_INVALID_ARGUMENT. */
snp_status snp_loss_3dgs_part(snp_scene s, const float *out_rgba, const float *target_rgb, int32_t n_views,
                              int32_t height, int32_t width, int32_t step_views, float lambda_dssim, float *grad_rgba,
                              float *loss, void *cuda_stream);
snp_status snp_scale_regularizer(snp_scene s, float weight, float *grad_scales, float *loss, void *cuda_stream);
snp_status snp_adam_step(snp_scene s, const float *const *grads, const float *lr, float beta1, float beta2, float eps,
                         int32_t step, void *cuda_stream);
/* Copies the scene's current parameters (e.g. after training steps) into dst[8]
 * (snp_scene_desc order and layouts; host or device memory as `memory` says).  Host
 * copies synchronise the stream. */
snp_status snp_get_params(snp_scene s, float *const *dst, int32_t memory, void *cuda_stream);

/* Convenience: snp_project + snp_bin_sort + snp_render. */
snp_status snp_render_views(snp_scene s, const snp_camera *cams, int32_t n_views,
                            const snp_render_opts *opts, float *out_rgba, void *cuda_stream);

snp_status snp_destroy(snp_scene s);

/* Thread-local text of the last error. */
const char *snp_last_error(void);

/* Parity/debug readback into HOST arrays (synchronises the stream; not on the
 * hot path).  Any pointer may be NULL.  rects [n_views*n][4] int32 tile rect
 * (tx0, ty0, tx1, ty1) or -1s when culled; depth_keys [n_views*n] (fp32 bits of
 * the depth lower bound); sorted_keys/sorted_ids up to `capacity` entries;
 * *n_dup receives the key count; tile_ranges [n_views*tiles][2] = [begin, end). */
snp_status snp_get_binning(snp_scene s, int32_t *rects, uint32_t *depth_keys, uint64_t *sorted_keys,
                           uint32_t *sorted_ids, int64_t capacity, int64_t *n_dup,
                           uint32_t *tile_ranges, void *cuda_stream);

/* Counters of the last project/bin_sort/render (synchronises the stream). */
snp_status snp_get_stats(snp_scene s, snp_stats *out, void *cuda_stream);

/* Debug readback of the raw device counters [0, n) (n <= 56; synchronises the
 * stream).  Slot 12 is the number of pixels the last render handed to the block-wide
 * K6 (more hits than K6w holds); slot 48 counts the grazing hits K5 evaluated with a
 * kappa error bound above 1.5e-5 (R23) since the last readback; slots 16..47
 * are only written by instrumented A/B builds (per-warp clock64 accounting).  The
 * call clears slots 16..48 after reading.  Not part of the hot path. */
snp_status snp_get_debug_counters(snp_scene s, uint64_t *out, int32_t n, void *cuda_stream);

/* Training: with `on`, every later snp_render / snp_render_views that covers one camera
 * batch (<= 32 views) and the whole image also records its composited hits (per hit: the
 * pixel, the primitive, the transmittance in front of it, its kappa and the colour
 * accumulated up to it; about 32 B per hit), and the next snp_render_backward_ex of the
 * same projection, colour mode and transmittance floor forms dL/dI and dL/dc from them
 * (Eq. 4, 9)
 * instead of traversing the frame again -- the same gradients.  A new snp_project or
 * snp_update_scene drops the record.  Off (0) by default. */
snp_status snp_set_record(snp_scene s, int32_t on);

/* Tight binning, from the next snp_project on:
 *   SNP_BIN_CONIC_TILES: K2 drops the keys of rect tiles whose pixel-centre rectangle the
 *     primitive's silhouette ellipse (the perspective image of the ellipsoid)
 *     does not reach -- such a tile holds no pixel whose ray hits the primitive, so the
 *     frame is unchanged; the keys are kept as dead keys sorted after all live ones
 *     (snp_stats.dead_keys);
 *   SNP_BIN_TILE_DEPTH: each key's depth is the larger of the primitive's bound and a
 *     per-tile bound (the support function of the ellipsoid along the tile's central ray),
 *     so K5 emits hits sooner (R19 holds with either bound).
 * 0 (the default) is the rect binning whose keys are bit-exact with the oracle's binning
 * definition.  Flags outside these two: SNP_ERR_INVALID_ARGUMENT. */
enum { SNP_BIN_CONIC_TILES = 1, SNP_BIN_TILE_DEPTH = 2 };
snp_status snp_set_binning(snp_scene s, int32_t flags);

/* Test hook: caps the per-pixel pending buffer of K5 at `k` entries (1..16) so
 * that the exact fallback K6 is exercised; 0 restores the default (16). */
snp_status snp_set_pending_limit(snp_scene s, int32_t k);

#ifdef __cplusplus
}
#endif
#endif /* SNP_H */
