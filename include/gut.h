/*
 * gut.h — C ABI of the B200-native 3DGUT forward rasterizer (ABI version 1).
 *
 * What it computes (PAPER.md = arXiv 2412.12507):
 *   render(gaussians, camera model, pose/shutter params) -> RGB, alpha, depth
 *   1. UT projection (Sec. 4.1, Eq. 6-10; Alg. 1-2):
 *      7 sigma points per Gaussian with weights from (alpha, beta, kappa),
 *      each projected exactly through the camera (pinhole, OpenCV rad-tan,
 *      Kannala-Brandt / equidistant fisheye, orthographic); rolling shutter
 *      gives every sigma point its own row-time extrinsic;
 *      then the 2D mean and covariance are re-estimated (Eq. 9-10).
 *   2. opacity-aware extent and tile binning with key duplication (Alg. 1
 *      lines 3-5), a (tile, depth) radix sort and
 *      per-tile ranges.
 *   3. per-pixel front-to-back compositing (Eq. 5) of each
 *      particle's 3D response at its maximum along the ray (Eq. 11,
 *      P:L192-200), SH colour, early transmittance termination.
 * Readings of silent points (quaternion order, thresholds, depth key, ...)
 * are DESIGN.md "Readings" R1..R27 and are shared with the test oracle.
 *
 * Conventions
 *   - All device work is enqueued asynchronously on the caller's stream;
 *     no call synchronises unless documented (stats != NULL, sync-capacity).
 *   - Every call returns gut_status; gut_last_error(ctx) names the offending
 *     field of the last non-OK status on that context.  No C++ exception,
 *     abort or exit crosses the ABI.
 *   - There is no CPU fallback: a device that is not sm_100 returns
 *     GUT_E_UNSUPPORTED from gut_context_create.
 *   - A context must not be used by two host threads at once (one context
 *     per thread / per rank).
 */
#ifndef GUT_H
#define GUT_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GUT_ABI_VERSION 1u

typedef struct gut_context gut_context; /* opaque: device, workspace, last error */
typedef struct gut_scene gut_scene;     /* opaque: packed device SoA copy of one Gaussian set */
typedef void *gut_stream;               /* a cudaStream_t (NULL = legacy default stream) */

typedef enum {
  GUT_OK = 0,
  GUT_E_INVALID_ARGUMENT = 1, /* bad struct_size, sizes, pointers, camera or options */
  GUT_E_UNSUPPORTED = 2,      /* device is not sm_100, or an unsupported combination */
  GUT_E_OUT_OF_MEMORY = 3,    /* device allocation failed */
  GUT_E_CAPACITY = 4,         /* key count exceeded the reserved capacity (graph mode) */
  GUT_E_CUDA = 5,             /* a CUDA runtime error; message in gut_last_error */
  GUT_E_INTERNAL = 6
} gut_status;

typedef enum { GUT_CAM_PINHOLE = 0, GUT_CAM_OPENCV = 1, GUT_CAM_FISHEYE = 2, GUT_CAM_ORTHO = 3 } gut_camera_model;

typedef enum {
  GUT_SHUTTER_GLOBAL = 0,
  GUT_SHUTTER_TOP_TO_BOTTOM = 1, /* shutter time of image row v is v/H        */
  GUT_SHUTTER_LEFT_TO_RIGHT = 2, /* u/W                                       */
  GUT_SHUTTER_BOTTOM_TO_TOP = 3, /* 1 - v/H                                   */
  GUT_SHUTTER_RIGHT_TO_LEFT = 4  /* 1 - u/W                                   */
} gut_shutter;

/* Camera (host struct, by value).  Doubles so the oracle and the GPU consume
 * identical values.  Camera axes are OpenCV (x right, y down, z forward).
 * Pixel (i,j) covers [i,i+1)x[j,j+1); its centre is (i+0.5, j+0.5) in the
 * same frame as (cx, cy).  The pose is camera->world: orientation quaternion
 * (w,x,y,z) and centre, at shutter time t=0 and t=1 (slerp / lerp in between,
 * reading R15).  GLOBAL shutter uses the t=0 pose only. */
typedef struct {
  uint32_t struct_size; /* = sizeof(gut_camera) */
  int32_t model;        /* gut_camera_model */
  int32_t width, height;
  double fx, fy, cx, cy; /* pixels (ORTHO: pixels per world unit) */
  double k[6];           /* OPENCV k1..k6 (k4..k6 rational denominator); FISHEYE k1..k4 */
  double p[2];           /* OPENCV p1, p2 */
  double fov_limit;      /* FISHEYE theta_max [rad] (required); OPENCV max normalised
                            undistorted radius r_lim (required if any k/p != 0) */
  int32_t shutter;       /* gut_shutter */
  int32_t pad0;
  double q_c2w[2][4];
  double c_w[2][3];
} gut_camera;

/* Gaussians (PAPER Sec. 3, Eq. 1-2: mu, q, s, sigma, SH of order <= 3).
 * count >= 0.  Arrays are read once by gut_scene_create (host pointers are
 * copied; device pointers are read on the given stream).  Parameters are
 * ACTIVATED (scale > 0, opacity in [0,1], reading R2).  Degenerate Gaussians
 * (non-finite, scale <= 0, zero quaternion, opacity <= alpha_min) are culled
 * and counted, not errors. */
typedef struct {
  uint32_t struct_size; /* = sizeof(gut_gaussians) */
  int32_t sh_degree;    /* 0..3 */
  int64_t count;
  int32_t on_device; /* 1: CUDA device pointers; 0: host pointers */
  int32_t pad0;
  const float *means;     /* [count][3] world units */
  const float *rotations; /* [count][4] (w,x,y,z), normalised inside (reading R1) */
  const float *scales;    /* [count][3] */
  const float *opacities; /* [count] */
  const float *sh;        /* [count][(sh_degree+1)^2][3] (3DGS layout) */
} gut_gaussians;

typedef struct {
  uint32_t struct_size;
  float ut_alpha, ut_beta, ut_kappa; /* 1, 2, 0; 3 + lambda > 0 required */
  float alpha_min;                   /* (float)(1/255): skip hits below (reading R20) */
  float alpha_max;                   /* 0.99: alpha clamp (reading R20) */
  float transmittance_min;           /* 1e-4: stop before T would drop below (R21) */
  float cov2d_dilation;              /* 0.3 px^2 added to Sigma' (reading R10) */
  float near_plane;                  /* 0.2 (z; distance for FISHEYE) (reading R9) */
  int32_t rs_max_iterations;         /* 8 secant steps per sigma point (R14) */
  float rs_tolerance_px;             /* 1e-4 px */
  int32_t tile_cull;                 /* 0 = AABB, 1 = ellipse-tile (default) */
  float background[3];               /* composited with the final T (R22) */
  int32_t timing;                    /* 1: record per-stage CUDA-event times (adds events) */
  int32_t kbuffer;                   /* hit order of the compositing (reading R28):
                                        0 = the tile's global depth order ("Ours", default);
                                        k in {1, 2, 4, 8, 16} = "Ours (sorted)": a per-ray MLAB
                                        k-buffer holding the k farthest pending hits by tau_max,
                                        the closest of k + 1 pending hits alpha-blended, the rest
                                        blended near to far at the end of the list (paper: k = 16).
                                        Other values: GUT_E_INVALID_ARGUMENT. */
  int32_t kernel_degree;             /* generalized Gaussian kernel of degree n (Supp. A, P:L458-462,
                                        reading R29): rho = exp(-lambda_n d^n / 2), lambda_n = 3^(2-n),
                                        d = Mahalanobis distance; 2 = the Gaussian (default); 1..8
                                        accepted, else GUT_E_INVALID_ARGUMENT.  Changes the extent
                                        level (Alg. 1) and the Eq. 11 response. */
} gut_options;

/* Outputs, HWC: rgb [H][W][3], alpha [H][W] (= 1 - T_final), depth [H][W]
 * (= sum alpha_i T_i tau_i, un-normalised, reading R23).  depth may be NULL.
 * on_device = 1: device pointers written on the stream.  on_device = 0: host
 * pointers (pinned recommended) filled by device->host copies enqueued on the
 * stream; valid once the stream has reached the end of the call. */
typedef struct {
  float *rgb;
  float *alpha;
  float *depth;
  int32_t on_device;
  int32_t pad0;
} gut_outputs;

typedef struct {
  int64_t n_input, n_visible, n_keys;
  int32_t n_tiles, max_tile_len;
  int64_t pairs_evaluated;   /* (pixel, list entry) evaluations in the blend */
  int64_t pairs_contributing;
  int64_t pixels_terminated;
  float ms_stage[7];         /* K1 project, K3 depth passes, K2 emit, K3 tile passes, K4 ranges,
                                K5 blend, total (timing = 1 only) */
  int32_t overflow;          /* 1 if the reserved key capacity was exceeded */
  int32_t pad0;
} gut_stats;

typedef enum {
  GUT_STAGE_PROJECT = 1, /* per Gaussian gut_proj_record [n_input] */
  GUT_STAGE_DEPTH_ORDER = 2, /* uint32 gid [n_visible], visible Gaussians by (depth, gid) */
  GUT_STAGE_SORTED = 3,  /* uint32 pairs (tile, gid) [n_keys], sorted by (tile, depth, gid) */
  GUT_STAGE_RANGES = 4,  /* uint32 pairs [start, end) [n_tiles] */
  GUT_STAGE_TILE_WORK = 5, /* uint32 pairs (list length, list entries the blend visited summed
                             over the tile's eight 8x4 pixel blocks, speculation and re-runs
                             included) [n_tiles] */
  GUT_STAGE_BLEND_TRACE = 6 /* uint32 x8 per blend work unit (segment slot, 8x4 pixel block):
                               (tile | segment << 16 | block << 29, SM id, start ns, end ns,
                               entries visited, pairs evaluated, pairs contributing, re-ran);
                               all zero for units that did not run; only with env
                               GUT_BLEND_TRACE=1 */,
  GUT_STAGE_COUNTERS = 7,   /* uint32[64]: the render's device counters (diagnostics; layout
                               internal, see csrc/launch.h CNT_*) */
  GUT_STAGE_RAYS = 8        /* per tile: float4 (a, b, snorm, beta) [256] of the pixel rays
                               relative to the tile anchor (PAPER L116 r(tau) = o + tau d; rays
                               kernel layout: pixel (x, y) of the tile at index
                               32 ((x >> 3) | ((y >> 2) << 1)) + 8 (y & 3) + (x & 7); snorm = 0
                               marks an invalid pixel), then float[4][8] per 8x8 block b
                               (x0 = 8 (b & 1), y0 = 8 (b >> 1)): {a00, ax, ay, rho_a, b00, bx,
                               by, rho_b}, the affine lattice a(x, y) = a00 + ax x + ay y of the
                               block's valid pixels (x, y = 0..7) with |residual| <= rho (rho =
                               +inf: none) that K5's candidate masks rely on.  [n_tiles] records
                               of 256 x 16 + 128 bytes */
} gut_stage;

typedef struct { /* GUT_STAGE_PROJECT record (K1 output, fp32) */
  float vx, vy, cxx, cxy, cyy, k2; /* Eq. 9-10 mean / covariance (+dilation), extent level */
  float depth;                     /* depth key (reading R13) */
  float rgb[3];                    /* SH colour (reading R18) */
  uint32_t tiles;                  /* tiles kept (0 = culled) */
  uint16_t rect[4];                /* tile x0, y0, x1, y1 (inclusive) */
} gut_proj_record;

uint32_t gut_abi_version(void);
void gut_options_default(gut_options *o);

/* Creates a context on CUDA device `cuda_device` (must be sm_100).  out != NULL. */
gut_status gut_context_create(int32_t cuda_device, gut_context **out);
void gut_context_destroy(gut_context *ctx);
/* Message for the last non-OK status on ctx (or a global message if ctx is NULL). */
const char *gut_last_error(const gut_context *ctx);

/* Capacity mode: pre-size the workspace for up to max_keys (Gaussian,tile)
 * keys, max_gaussians Gaussians and max_w x max_h images.  After this call
 * gut_render never synchronises; a frame whose key count exceeds max_keys is
 * truncated (its image is wrong) and the overflow is latched in a sticky
 * device word that the per-render reset does not clear.  It is reported --
 * and cleared -- as GUT_E_CAPACITY (plus gut_stats.overflow = 1) by the next
 * synchronising call on the context: gut_render with stats != NULL,
 * gut_timing_read or gut_check.  Without it, gut_render reads the key count
 * back (one stream sync per view) and grows the workspace. */
gut_status gut_workspace_reserve(gut_context *ctx, int64_t max_keys, int64_t max_gaussians,
                                 int32_t max_w, int32_t max_h);

/* Packs and validates a Gaussian set once (SoA, 16-byte aligned, on the
 * context's device).  Amortised over views.  The scene is owned by the
 * library until gut_scene_destroy. */
gut_status gut_scene_create(gut_context *ctx, const gut_gaussians *g, gut_stream s, gut_scene **out);
void gut_scene_destroy(gut_context *ctx, gut_scene *scene);

/* Renders one view.  stats (nullable): if non-NULL the call synchronises the
 * stream and fills it. */
gut_status gut_render(gut_context *ctx, const gut_scene *scene, const gut_camera *cam,
                      const gut_options *opt, const gut_outputs *out, gut_stream s, gut_stats *stats);

/* Gradients of a scalar loss with respect to the scene (device buffers, fp32,
 * written -- not accumulated -- by gut_render_backward). */
typedef struct {
  float *means;      /* [count][3] */
  float *rotations;  /* [count][4] w.r.t. the raw (unnormalised) input quaternion */
  float *scales;     /* [count][3] */
  float *opacities;  /* [count] */
  float *sh;         /* [count][(sh_degree+1)^2][3] */
  float *rgb;        /* nullable: [count][3] gradient of the view's SH colour */
  float *densify;    /* nullable: [count] densification statistic of this view, |dL/dmu| / (d / 2),
                        d = distance from mu to the camera centre at mu's shutter time (PAPER L218:
                        "3D positional gradients divided by half of the distance to the camera",
                        reading R32) */
} gut_gradients;

/* Backward pass (PAPER Supp. B, L494-513; reading R30) of the LAST gut_render
 * on this context, which must have been called with the same scene, camera
 * and options and device outputs: L = sum over pixels of grad_rgb . rgb +
 * grad_alpha alpha + grad_depth depth.  Gradients flow through the Eq. 5
 * compositing and the Eq. 11 3D response to mu, q, s, sigma and (through the
 * colour, view direction held constant) the SH coefficients; the UT
 * projection and the binning are not differentiated.
 * rgb/alpha/depth: the forward's device outputs ([H][W][3], [H][W], [H][W]);
 * grad_rgb [H][W][3] required, grad_alpha / grad_depth nullable (zero); depth
 * is required when grad_depth is given.  All pointers device memory on the
 * context's device; asynchronous on s.  Per-Gaussian sums accumulate in 32.32
 * fixed point (int64 atomics; resolution 2^-32 per term, range +-2^31): the
 * gradients are bitwise reproducible.  Supported: PINHOLE / OPENCV /
 * FISHEYE with any shutter and kernel_degree, kbuffer 0; otherwise
 * GUT_E_UNSUPPORTED.  It differentiates ctx's LAST render (its sorted lists
 * and workspace): a camera / options mismatch with that render gives
 * GUT_E_INVALID_ARGUMENT (after gut_render_batch the last render on ctx itself
 * is the last view of lane 0, not the batch's last view). */
gut_status gut_render_backward(gut_context *ctx, const gut_scene *scene, const gut_camera *cam,
                               const gut_options *opt, const float *rgb, const float *alpha,
                               const float *depth, const float *grad_rgb, const float *grad_alpha,
                               const float *grad_depth, const gut_gradients *grads, gut_stream s);

/* Projection quality (PAPER Supp. C, L522-588; reading R31), a measurement
 * tool: per Gaussian its 2D image (mean x, y in pixels; covariance xx, xy, yy)
 * as estimated by the UT (Eq. 6-10, no binning dilation), by EWA (Eq. 3:
 * linearisation at mu with a central-difference Jacobian, pose frozen at mu's
 * own shutter time -- RS-unaware) and by Monte Carlo with n_samples points
 * mu + R S z (z: counter-based N(0, I) from seed, gaussian, sample -- the
 * splitmix64 / Box-Muller spec of DESIGN.md R31), each projected with its own
 * rolling-shutter pose; kl_ut = KL(N_mc || N_ut), kl_ewa = KL(N_mc || N_ewa).
 * valid = 0 when a point fails to project.  out: device array [count];
 * asynchronous on s.  fp64. */
typedef struct {
  double ut[5], ewa[5], mc[5];
  double kl_ut, kl_ewa;
  int32_t valid, pad;
} gut_quality;
gut_status gut_projection_quality(gut_context *ctx, const gut_scene *scene, const gut_camera *cam,
                                  const gut_options *opt, int32_t n_samples, uint64_t seed, gut_quality *out,
                                  gut_stream s);

/* Renders n_views views (outs[i] for cams[i]).  With stats == NULL the views
 * are pipelined: up to gut_context_set_frames_in_flight() frames (default 4)
 * are in flight at once, view i on lane i mod F -- lane 0 is ctx on stream s,
 * lanes 1..F-1 are child contexts (own workspaces, reserved like ctx, created
 * on first use and owned by ctx) on their own streams, forked from and joined
 * back to s with events, so the call stays asynchronous on s and every output
 * is complete when s reaches the point after the call.  Pipelined frames run
 * the blend (K5) in a throughput schedule -- no speculative segments beyond
 * the successor grants, grants at most 4 segments ahead, a persistent grid of
 * 1.25 CTAs per SM so the next frames' projection and sorts share the SMs --
 * where gut_render runs it for latency (speculation window 2, every SM).  The
 * schedule decides only who computes what when: results are identical to
 * rendering the views one by one.  With stats != NULL the views are rendered
 * one at a time on s and stats[i] filled (synchronising). */
gut_status gut_render_batch(gut_context *ctx, const gut_scene *scene, const gut_camera *cams,
                            int32_t n_views, const gut_options *opt, const gut_outputs *outs,
                            gut_stream s, gut_stats *stats);

/* Frames in flight of gut_render_batch (1..8; 1 = one at a time on s). */
gut_status gut_context_set_frames_in_flight(gut_context *ctx, int32_t n);

/* Per-stage device times of every render issued with options.timing = 1 since
 * the last reset -- including those gut_render_batch ran on the context's
 * lanes: CUDA events recorded on the render's stream between the stages (with
 * frames in flight a lane's stage times include time shared with other
 * frames).  Synchronises.  ms_sum[7] receives the summed milliseconds per stage
 * (order of gut_stats.ms_stage), *n_renders the number of renders summed;
 * reset != 0 clears the accumulator. */
gut_status gut_timing_read(gut_context *ctx, double ms_sum[7], int32_t *n_renders, int32_t reset);

/* Synchronises `s` and reports whether any render issued on ctx since the
 * last synchronising call overflowed its reserved key capacity
 * (GUT_E_CAPACITY; the latch is cleared) -- GUT_OK otherwise. */
gut_status gut_check(gut_context *ctx, gut_stream s);

/* Tests only: copies an intermediate buffer of the LAST render on ctx to host
 * memory (synchronises).  *bytes_needed receives the size; if host_dst is
 * NULL or bytes is too small nothing is copied. */
gut_status gut_debug_copy_stage(gut_context *ctx, int32_t stage, void *host_dst, size_t bytes,
                                size_t *bytes_needed);

#ifdef __cplusplus
}
#endif
#endif
