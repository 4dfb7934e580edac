/*
 * gut_oracle.h — fp64 CPU ORACLE for the 3DGUT forward rasterizer.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or call this code.
 * The product path (include/gut.h, paper_2412_12507_b200/) never includes,
 * links or imports anything under oracle/, and this file includes nothing of
 * the product.  The two share only the seeded input generators (scenegen/).
 *
 * The oracle follows PAPER.md step by step:
 *   O1 Gaussian setup, UT weights, sigma points  PAPER L84-95 (Eq.1-2), L139-168 (Eq.6-8)
 *   O2 exact projection of each sigma point       PAPER L170 ; rolling shutter L34, L393
 *   O3 UT estimate, extent, tiles, depth, colour PAPER L170-178 (Eq.9-10), Alg.1
 *   O4 per-tile depth-ordered lists
 *   O5 pixel rays
 *   O6 front-to-back compositing, 3D max response PAPER L115-121 (Eq.5), L192-200 (Eq.11)
 *   O6' per-ray k-buffer / exact tau order        PAPER L205-212 (Sec. 4.3, "Ours (sorted)")
 *   generalized kernels of degree n              PAPER L454-462 (Supp. A)
 *   O7 backward of O6 (gradients)                PAPER L202, L494-513 (Supp. B), L218
 *   O8 projection quality (UT / EWA / MC, KL)     PAPER L98-102 (Eq. 3), L522-588 (Supp. C)
 * Readings of silent/ambiguous points are listed in DESIGN.md "Readings".
 */
#ifndef GUT_ORACLE_H
#define GUT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_PINHOLE = 0, ORC_OPENCV = 1, ORC_FISHEYE = 2, ORC_ORTHO = 3 };
enum { ORC_GLOBAL = 0, ORC_TOP_TO_BOTTOM = 1, ORC_LEFT_TO_RIGHT = 2,
       ORC_BOTTOM_TO_TOP = 3, ORC_RIGHT_TO_LEFT = 4 };

typedef struct {
  int32_t model, width, height, shutter;
  double fx, fy, cx, cy;
  double k[6];
  double p[2];
  double fov_limit;       /* FISHEYE theta_max [rad]; OPENCV r_lim (normalised); 0 = none */
  double q[2][4];         /* camera->world quaternion (w,x,y,z) at t=0, t=1 */
  double c[2][3];         /* camera centre (world) at t=0, t=1 */
} orc_camera;

typedef struct {
  double ut_alpha, ut_beta, ut_kappa;
  double alpha_min, alpha_max, t_min, dilation, near_plane;
  double bg[3];
  int32_t tile_cull;      /* 0 AABB, 1 ellipse-tile */
  int32_t kbuffer;        /* O6 hit order: 0 = the tile's global depth order ("Ours");
                             k >= 1 = per-ray MLAB k-buffer ("Ours (sorted)");
                             -1 = exact per-ray tau_max sort (the 3DGRT order) */
  int32_t kernel_degree;  /* Supp. A generalized Gaussian degree n (2 = Gaussian, Eq. 1) */
  int32_t pad;
} orc_options;

/* cull reasons (0 = visible) */
enum { ORC_OK = 0, ORC_CULL_PARAM = 1, ORC_CULL_OPACITY = 2, ORC_CULL_SIGMA = 3,
       ORC_CULL_COV = 4, ORC_CULL_OFFSCREEN = 5, ORC_CULL_NOTILE = 6 };

typedef struct {
  int32_t reason;          /* ORC_OK or a cull reason */
  int32_t tiles;           /* tiles kept (0 if culled) */
  int32_t rect[4];         /* tile x0,y0,x1,y1 (inclusive, clamped) */
  int32_t cull_ambig;      /* a validity quantity is within its margin */
  int32_t bin_ambig;       /* some candidate tile decision flips under +-1e-3 px */
  int32_t rs_iters;        /* max fixed-point iterations over the 7 points (RS) */
  int32_t rs_fail;         /* non-convergence */
  double vx, vy;           /* 2D mean v_mu (Eq. 9) */
  double cxx, cxy, cyy;    /* 2D covariance Sigma' (Eq. 10) + dilation */
  double k2;               /* 2 ln(sigma/alpha_min) */
  double hx, hy;           /* extent (AABB half sizes) */
  double depth;            /* ||x0 in camera frame|| at its own shutter time */
  double t0;               /* shutter time of the centre point */
  double rgb[3];           /* SH colour at d = normalize(mu - c(t0)) */
} orc_proj;

typedef struct {
  int32_t visited, contributed, terminated, invalid;
  double min_alpha_gap;    /* min |alpha - alpha_min| over visited entries */
  double min_term_gap;     /* min |T' - T_min| over blended/stopping entries */
  double min_order_gap;    /* min order margin of consecutive contributing entries: the relative
                              depth perturbation that could swap them under the (fp32 key, index)
                              order (gut_oracle.c order_margin) */
  int32_t amb_bin;         /* a binning-ambiguous pair could change this pixel */
  int32_t amb_cull;        /* a cull-ambiguous Gaussian could change this pixel */
  double min_tau_gap;      /* kbuffer != 0: min relative tau_max gap between two hits adjacent
                              in tau order (an fp32 tau could swap them) */
  int32_t alt_valid;       /* kbuffer != 0: exactly one such pair within the alt band -> alt_*
                              hold the pixel with the two hits' tau_max swapped (the other order) */
  int32_t alt_pad;
  double alt_rgb[3], alt_alpha, alt_depth;  /* (without the background term: C, 1 - T, D) */
} orc_pixdiag;

/* relative tau_max band of the alternative-order render (default 2e-6) */
void orc_set_alt_band(double band);

/* ---- O1 ---- */
int  orc_ut_weights(double a, double b, double k, double wmu[7], double wsig[7], double *lambda);
int  orc_quat_to_rot(const double q[4], double R[9]);
void orc_sigma_points(const double mu[3], const double R[9], const double s[3], double lambda,
                      double X[7][3]);
/* ---- O2 ---- */
void orc_pose_at(const orc_camera *cam, double t, double Rc2w[9], double c[3]);
int  orc_project_cam(const orc_camera *cam, const orc_options *o, const double xc[3], double uv[2],
                     double *margin);
int  orc_project_point(const orc_camera *cam, const orc_options *o, const double x[3], double uv[2],
                       double *t_out, int32_t *iters, double *margin);
/* ---- O3 ---- */
void orc_sh_basis(const double d[3], double Y[16]);
int  orc_tile_hits_ellipse(double vx, double vy, double cxx, double cxy, double cyy, double k2,
                           double x0, double y0, double x1, double y1);
void orc_preprocess(const float *means, const float *rots, const float *scales, const float *opac,
                    const float *sh, int32_t sh_degree, int64_t n, const orc_camera *cam,
                    const orc_options *o, orc_proj *out);
/* ---- O4 ---- (pairs: tile-major, then (depth, gid); returns K) */
int64_t orc_tile_lists(const orc_proj *proj, int64_t n, const orc_camera *cam, const orc_options *o,
                       const float *means, const float *scales, int32_t *tile_of, int32_t *gid_of,
                       int64_t cap, int32_t *ranges);
/* ---- O5 ---- */
int  orc_pixel_ray(const orc_camera *cam, double u, double v, double o[3], double d[3]);
/* ---- O6 ---- */
/* Per-ray re-ordering of one pixel's hit stream: hits in stream
 * order (tau_max, alpha, rgb), k = kbuffer option (>= 1 MLAB k-buffer, -1
 * exact tau sort, 0 stream order); Eq. 5 with the termination rule R21. */
/* Returns the number of stream hits consumed before termination (n if none). */
int32_t orc_kbuffer_blend(const double *tau, const double *alpha, const double *rgb, int32_t n, int32_t k,
                          double t_min, double C[3], double *T_out, double *D_out, int32_t *n_blended,
                          double *min_term_gap);
double orc_max_response(const double mu[3], const double R[9], const double s[3], const double o[3],
                        const double d[3], double *tau);
void orc_composite(const float *means, const float *rots, const float *scales, const float *opac,
                   const orc_proj *proj, const int32_t *gids, const int32_t *ranges,
                   const orc_camera *cam, const orc_options *o, const int32_t *tile_subset,
                   int32_t n_subset, float *rgb, float *alpha, float *depth, orc_pixdiag *diag);
/* full render: binned (brute = 0) or brute force over all valid Gaussians (brute = 1) */
int64_t orc_render(const float *means, const float *rots, const float *scales, const float *opac,
                   const float *sh, int32_t sh_degree, int64_t n, const orc_camera *cam,
                   const orc_options *o, int32_t brute, const int32_t *tile_subset, int32_t n_subset,
                   float *rgb, float *alpha, float *depth, orc_pixdiag *diag, orc_proj *proj_out,
                   int64_t *n_keys_out);
/* flag pixels that an ambiguous (Gaussian, tile) pair or a cull-ambiguous Gaussian could change */
void orc_mark_ambiguity(const float *means, const float *rots, const float *scales, const float *opac,
                        const orc_proj *proj, int64_t n, const orc_camera *cam, const orc_options *o,
                        double alpha_eps, const int32_t *tile_subset, int32_t n_subset,
                        orc_pixdiag *diag);
int  orc_threads(void);
/* ---- O8 (projection quality, Supp. C; reading R31) ---- */
void orc_normal3(uint64_t seed, int64_t gid, int32_t s, double z[3]);
double orc_kl2(const double g0[5], const double g1[5]);   /* KL(N0 || N1), g = (mx, my, cxx, cxy, cyy) */
typedef struct { double ut[5], ewa[5], mc[5], kl_ut, kl_ewa; int32_t valid, pad; } orc_quality;
void orc_projection_quality(const float *means, const float *rots, const float *scales, int64_t n,
                            const orc_camera *cam, const orc_options *o, int32_t n_mc, uint64_t seed,
                            orc_quality *out);
/* ---- O7 (backward, Supp. B; "Ours" order, any degree and shutter, reading R30) ----
 * upstream g_rgb [H][W][3], g_alpha [H][W], g_depth [H][W] (fp32);
 * outputs (fp64): d_means [n][3], d_rots [n][4], d_scales [n][3], d_opac [n],
 * d_sh [n][(d+1)^2][3], d_rgb [n][3] (gradient of the view's colour). Returns K. */
int64_t orc_backward(const float *means, const float *rots, const float *scales, const float *opac,
                     const float *sh, int32_t sh_degree, int64_t n, const orc_camera *cam,
                     const orc_options *o, const float *g_rgb, const float *g_alpha, const float *g_depth,
                     double *d_means, double *d_rots, double *d_scales, double *d_opac, double *d_sh,
                     double *d_rgb, double *loss);
/* Supp. A: lambda_n = 3^(2-n); response exp(-lambda_n (d^2)^(n/2) / 2) (reading R29) */
double orc_kernel_lambda(int32_t n);
double orc_kernel_response(double d2, int32_t n);

#ifdef __cplusplus
}
#endif
#endif
