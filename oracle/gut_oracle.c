/*
 * gut_oracle.c — fp64 CPU ORACLE for the 3DGUT forward rasterizer.
 *
 * TEST INFRASTRUCTURE ONLY (see gut_oracle.h): plain, slow, obviously correct.
 * Every function cites the PAPER.md passage (P:L<line>) it follows; readings of
 * silent or ambiguous points cite DESIGN.md "Readings" (R<n>) which restates
 * SURVEY.md §8(c).3.  No blocking, fusion or reordering beyond the paper's
 * definitions; a library primitive (qsort, libm) may serve as a step.
 *
 * Pins (tests/test_oracle_*.py, run with -m "not gpu") tie each step to
 * something other than this code: printed constants, closed forms, textbook
 * identities, brute force.  Parity status per function is in DESIGN.md.
 */
#include "gut_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TILE 16

static int finite3(const double v[3]) { return isfinite(v[0]) && isfinite(v[1]) && isfinite(v[2]); }
static double dot3(const double a[3], const double b[3]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static void cross3(const double a[3], const double b[3], double r[3]) {
  r[0] = a[1] * b[2] - a[2] * b[1];
  r[1] = a[2] * b[0] - a[0] * b[2];
  r[2] = a[0] * b[1] - a[1] * b[0];
}
/* r = M v for row-major 3x3 M */
static void mv3(const double M[9], const double v[3], double r[3]) {
  for (int i = 0; i < 3; ++i) r[i] = M[3 * i] * v[0] + M[3 * i + 1] * v[1] + M[3 * i + 2] * v[2];
}
/* r = M^T v */
static void mtv3(const double M[9], const double v[3], double r[3]) {
  for (int i = 0; i < 3; ++i) r[i] = M[i] * v[0] + M[3 + i] * v[1] + M[6 + i] * v[2];
}

/* Supp. A, reading R29: generalized Gaussian of degree n,
 * rho = exp(-(1/2) lambda_n d^n) with d^2 the Mahalanobis distance and
 * lambda_n = r^2 / r^n, r = 3 (the response at d = r equals the Gaussian's
 * exp(-r^2/2); n = 2 is the Gaussian, Eq. 1).  The printed formula omits the
 * 1/2, which contradicts "the same kernel response at a given distance r as
 * the reference Gaussian kernel"; we keep it (SPEC S:L59 reads the same). */
double orc_kernel_lambda(int32_t n) { return pow(3.0, 2.0 - (double)n); }

double orc_kernel_response(double d2, int32_t n) {
  if (n == 2) return exp(-0.5 * d2);
  return exp(-0.5 * orc_kernel_lambda(n) * pow(d2, 0.5 * (double)n));
}

int orc_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ======================================================================
 * O1 — Gaussian setup, UT weights, sigma points
 * ====================================================================== */

/* Eq. 7-8: lambda = alpha^2 (3 + kappa) - 3;
 * w0_mu = lambda/(3+lambda), w0_sig = w0_mu + (1 - alpha^2 + beta),
 * wi_mu = wi_sig = 1/(2(3+lambda)), i = 1..6.  Returns -1 if 3+lambda <= 0. */
int orc_ut_weights(double a, double b, double k, double wmu[7], double wsig[7], double *lambda) {
  double lam = a * a * (3.0 + k) - 3.0;
  if (!(3.0 + lam > 0.0)) return -1;
  wmu[0] = lam / (3.0 + lam);
  wsig[0] = wmu[0] + (1.0 - a * a + b);
  for (int i = 1; i < 7; ++i) wmu[i] = wsig[i] = 1.0 / (2.0 * (3.0 + lam));
  if (lambda) *lambda = lam;
  return 0;
}

/* Eq. 2: R from the quaternion q = (w,x,y,z), normalised first
 * (reading R1).  Row-major R.  Returns -1 for a zero / non-finite quaternion. */
int orc_quat_to_rot(const double q_in[4], double R[9]) {
  double n = sqrt(q_in[0] * q_in[0] + q_in[1] * q_in[1] + q_in[2] * q_in[2] + q_in[3] * q_in[3]);
  if (!(n > 0.0) || !isfinite(n)) return -1;
  double w = q_in[0] / n, x = q_in[1] / n, y = q_in[2] / n, z = q_in[3] / n;
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
  return 0;
}

/* Eq. 6: x0 = mu; x_i = mu + sqrt((3+lambda) Sigma)_[i];
 * x_{i+3} = mu - sqrt((3+lambda) Sigma)_[i]; the square root is "read off" the
 * factorisation Sigma = R S S^T R^T, i.e. the columns of R S (reading R3). */
void orc_sigma_points(const double mu[3], const double R[9], const double s[3], double lambda,
                      double X[7][3]) {
  double g = sqrt(3.0 + lambda);
  for (int a = 0; a < 3; ++a) X[0][a] = mu[a];
  for (int i = 0; i < 3; ++i) {
    for (int a = 0; a < 3; ++a) {
      double col = R[3 * a + i] * s[i]; /* (R S)[a][i] */
      X[1 + i][a] = mu[a] + g * col;
      X[4 + i][a] = mu[a] - g * col;
    }
  }
}

/* ======================================================================
 * O2 — exact projection of each sigma point, v = g(x)
 * ====================================================================== */

/* Pose at shutter time t (reading R15): camera->world orientation by slerp on
 * the shortest arc, camera centre by lerp.  Global shutter uses pose 0. */
void orc_pose_at(const orc_camera *cam, double t, double Rc2w[9], double c[3]) {
  double q0[4], q1[4], q[4];
  for (int i = 0; i < 4; ++i) { q0[i] = cam->q[0][i]; q1[i] = cam->q[1][i]; }
  if (cam->shutter == ORC_GLOBAL) t = 0.0;
  double n0 = sqrt(q0[0] * q0[0] + q0[1] * q0[1] + q0[2] * q0[2] + q0[3] * q0[3]);
  double n1 = sqrt(q1[0] * q1[0] + q1[1] * q1[1] + q1[2] * q1[2] + q1[3] * q1[3]);
  for (int i = 0; i < 4; ++i) { q0[i] /= n0; q1[i] /= n1; }
  double cs = q0[0] * q1[0] + q0[1] * q1[1] + q0[2] * q1[2] + q0[3] * q1[3];
  if (cs < 0) { cs = -cs; for (int i = 0; i < 4; ++i) q1[i] = -q1[i]; }
  if (cs > 1.0 - 1e-15) {
    for (int i = 0; i < 4; ++i) q[i] = (1 - t) * q0[i] + t * q1[i];
  } else {
    double om = acos(cs), so = sin(om);
    double a = sin((1 - t) * om) / so, b = sin(t * om) / so;
    for (int i = 0; i < 4; ++i) q[i] = a * q0[i] + b * q1[i];
  }
  orc_quat_to_rot(q, Rc2w);
  for (int i = 0; i < 3; ++i) c[i] = (1 - t) * cam->c[0][i] + t * cam->c[1][i];
}

static void opencv_distort(const orc_camera *c, double xn, double yn, double *xd, double *yd) {
  double r2 = xn * xn + yn * yn;
  double num = 1 + c->k[0] * r2 + c->k[1] * r2 * r2 + c->k[2] * r2 * r2 * r2;
  double den = 1 + c->k[3] * r2 + c->k[4] * r2 * r2 + c->k[5] * r2 * r2 * r2;
  double a = num / den;
  *xd = xn * a + 2 * c->p[0] * xn * yn + c->p[1] * (r2 + 2 * xn * xn);
  *yd = yn * a + c->p[0] * (r2 + 2 * yn * yn) + 2 * c->p[1] * xn * yn;
}

static double fisheye_theta_d(const orc_camera *c, double th) {
  double t2 = th * th;
  return th * (1 + c->k[0] * t2 + c->k[1] * t2 * t2 + c->k[2] * t2 * t2 * t2 + c->k[3] * t2 * t2 * t2 * t2);
}

/* Camera-frame projection per model (readings R7, R8, R9; SURVEY §8(c).2 O2
 * table).  Validity is part of the definition.  *margin = signed normalised
 * distance to the nearest validity bound (> 0 when valid). */
int orc_project_cam(const orc_camera *cam, const orc_options *o, const double x[3], double uv[2],
                    double *margin) {
  double m = 1e300;
  int valid = 1;
  switch (cam->model) {
    case ORC_PINHOLE: {
      double mz = (x[2] - o->near_plane) / fmax(1.0, fabs(x[2]));
      m = mz; valid = x[2] > o->near_plane;
      uv[0] = cam->fx * (x[0] / x[2]) + cam->cx;
      uv[1] = cam->fy * (x[1] / x[2]) + cam->cy;
      break;
    }
    case ORC_ORTHO: {
      m = (x[2] - o->near_plane) / fmax(1.0, fabs(x[2])); valid = x[2] > o->near_plane;
      uv[0] = cam->fx * x[0] + cam->cx;
      uv[1] = cam->fy * x[1] + cam->cy;
      break;
    }
    case ORC_OPENCV: {
      m = (x[2] - o->near_plane) / fmax(1.0, fabs(x[2])); valid = x[2] > o->near_plane;
      double xn = x[0] / x[2], yn = x[1] / x[2], r2 = xn * xn + yn * yn;
      if (cam->fov_limit > 0) {
        double rl2 = cam->fov_limit * cam->fov_limit;
        double mr = (rl2 - r2) / rl2;
        if (mr < m) m = mr;
        if (!(r2 <= rl2)) valid = 0;
      }
      double xd, yd;
      opencv_distort(cam, xn, yn, &xd, &yd);
      uv[0] = cam->fx * xd + cam->cx;
      uv[1] = cam->fy * yd + cam->cy;
      break;
    }
    case ORC_FISHEYE: {
      double nrm = sqrt(dot3(x, x));
      m = (nrm - o->near_plane) / fmax(1.0, nrm); valid = nrm > o->near_plane;
      double rho = sqrt(x[0] * x[0] + x[1] * x[1]);
      double th = atan2(rho, x[2]);
      double thmax = cam->fov_limit > 0 ? cam->fov_limit : M_PI;
      if (thmax - th < m) m = thmax - th;
      if (!(th <= thmax)) valid = 0;
      if (rho == 0.0) { uv[0] = cam->cx; uv[1] = cam->cy; }
      else {
        double td = fisheye_theta_d(cam, th);
        uv[0] = cam->fx * td * x[0] / rho + cam->cx;
        uv[1] = cam->fy * td * x[1] / rho + cam->cy;
      }
      break;
    }
    default: valid = 0; m = -1;
  }
  if (!isfinite(uv[0]) || !isfinite(uv[1])) valid = 0;
  if (margin) *margin = m;
  return valid;
}

/* shutter coordinate rho(u,v) in [0,1] (reading R16) */
static double shutter_coord(const orc_camera *cam, const double uv[2]) {
  double r;
  switch (cam->shutter) {
    case ORC_TOP_TO_BOTTOM: r = uv[1] / cam->height; break;
    case ORC_BOTTOM_TO_TOP: r = 1.0 - uv[1] / cam->height; break;
    case ORC_LEFT_TO_RIGHT: r = uv[0] / cam->width; break;
    case ORC_RIGHT_TO_LEFT: r = 1.0 - uv[0] / cam->width; break;
    default: return 0.0;
  }
  return r < 0 ? 0 : (r > 1 ? 1 : r);
}

static int project_world_at(const orc_camera *cam, const orc_options *o, const double x[3], double t,
                            double uv[2], double *margin, double xc_out[3]) {
  double R[9], c[3], d[3], xc[3];
  orc_pose_at(cam, t, R, c);
  for (int i = 0; i < 3; ++i) d[i] = x[i] - c[i];
  mtv3(R, d, xc); /* x_c = R_c2w^T (x - c(t)) */
  if (xc_out) for (int i = 0; i < 3; ++i) xc_out[i] = xc[i];
  return orc_project_cam(cam, o, xc, uv, margin);
}

/* g(x) with the sigma point's own extrinsic ("transforming each sigma
 * point with a different extrinsic matrix").  Reading R14: the
 * shutter time is the fixed point t* = clamp(rho(g(x; pose(t*))), 0, 1),
 * found by plain iteration from t0 = 0.5 until the pixel moves < 1e-9 px
 * (<= 200 iterations).  A point invalid at any iterate is invalid. */
int orc_project_point(const orc_camera *cam, const orc_options *o, const double x[3], double uv[2],
                      double *t_out, int32_t *iters, double *margin) {
  if (cam->shutter == ORC_GLOBAL) {
    if (t_out) *t_out = 0.0;
    if (iters) *iters = 0;
    return project_world_at(cam, o, x, 0.0, uv, margin, NULL);
  }
  double t = 0.5, cur[2];
  int valid = project_world_at(cam, o, x, t, cur, margin, NULL);
  int it = 0, converged = 0;
  while (valid && it < 200) {
    double tn = shutter_coord(cam, cur), nxt[2];
    valid = project_world_at(cam, o, x, tn, nxt, margin, NULL);
    double du = nxt[0] - cur[0], dv = nxt[1] - cur[1];
    cur[0] = nxt[0]; cur[1] = nxt[1]; t = tn; ++it;
    if (sqrt(du * du + dv * dv) < 1e-9) { converged = 1; break; }
  }
  uv[0] = cur[0]; uv[1] = cur[1];
  if (t_out) *t_out = t;
  if (iters) *iters = converged ? it : -it;
  return valid;
}

/* ======================================================================
 * O3 — UT estimate (Eq. 9-10), extent, tiles, depth key, colour
 * ====================================================================== */

/* 3DGS real SH basis, degree <= 3 (reading R19; SURVEY App. C constants). */
void orc_sh_basis(const double d[3], double Y[16]) {
  const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
  const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                        -1.0925484305920792, 0.5462742152960396};
  const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                        0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                        -0.5900435899266435};
  double x = d[0], y = d[1], z = d[2], xx = x * x, yy = y * y, zz = z * z;
  Y[0] = C0;
  Y[1] = -C1 * y; Y[2] = C1 * z; Y[3] = -C1 * x;
  Y[4] = C2[0] * x * y; Y[5] = C2[1] * y * z; Y[6] = C2[2] * (2 * zz - xx - yy);
  Y[7] = C2[3] * x * z; Y[8] = C2[4] * (xx - yy);
  Y[9] = C3[0] * y * (3 * xx - yy); Y[10] = C3[1] * x * y * z; Y[11] = C3[2] * y * (4 * zz - xx - yy);
  Y[12] = C3[3] * z * (2 * zz - 3 * xx - 3 * yy); Y[13] = C3[4] * x * (4 * zz - xx - yy);
  Y[14] = C3[5] * z * (xx - yy); Y[15] = C3[6] * x * (xx - 3 * yy);
}

/* Ellipse-tile test (reading R12; StopThePop culling): does the closed
 * square [x0,x1]x[y0,y1] intersect E = {v : (v-vmu)^T Sigma'^-1 (v-vmu) <= k2}?
 * If vmu is inside, yes; otherwise the minimum of the convex quadratic over
 * the square lies on its boundary: each edge is a clamped 1-D minimum. */
int orc_tile_hits_ellipse(double vx, double vy, double cxx, double cxy, double cyy, double k2,
                          double x0, double y0, double x1, double y1) {
  if (vx >= x0 && vx <= x1 && vy >= y0 && vy <= y1) return 1;
  double det = cxx * cyy - cxy * cxy;
  double A = cyy / det, B = -cxy / det, C = cxx / det; /* Sigma'^-1 = [[A,B],[B,C]] */
  double best = 1e300;
  double ys[2] = {y0, y1}, xs[2] = {x0, x1};
  for (int e = 0; e < 2; ++e) { /* horizontal edges y = ys[e] */
    double dy = ys[e] - vy, dx = -B * dy / A;
    if (dx < x0 - vx) dx = x0 - vx;
    if (dx > x1 - vx) dx = x1 - vx;
    double q = A * dx * dx + 2 * B * dx * dy + C * dy * dy;
    if (q < best) best = q;
  }
  for (int e = 0; e < 2; ++e) { /* vertical edges x = xs[e] */
    double dx = xs[e] - vx, dy = -B * dx / C;
    if (dy < y0 - vy) dy = y0 - vy;
    if (dy > y1 - vy) dy = y1 - vy;
    double q = A * dx * dx + 2 * B * dx * dy + C * dy * dy;
    if (q < best) best = q;
  }
  return best <= k2;
}

/* one tile decision with the square grown by `grow` px (negative = eroded) */
static int tile_test(const orc_proj *p, int tile_cull, int tx, int ty, double grow) {
  double x0 = TILE * tx - grow, x1 = TILE * tx + TILE + grow;
  double y0 = TILE * ty - grow, y1 = TILE * ty + TILE + grow;
  if (tile_cull == 0) { /* AABB: rectangle [vmu-h, vmu+h] overlaps the square */
    return (p->vx + p->hx >= x0) && (p->vx - p->hx <= x1) && (p->vy + p->hy >= y0) &&
           (p->vy - p->hy <= y1);
  }
  return orc_tile_hits_ellipse(p->vx, p->vy, p->cxx, p->cxy, p->cyy, p->k2, x0, y0, x1, y1);
}

/* the kept tiles of a Gaussian in row-major order (ty outer, tx inner);
 * Alg. 1: the rectangle r_i = ComputeRectangle(h_i, v_mu_i) gives the
 * candidate tiles tx in [floor((vx-hx)/16), floor((vx+hx)/16)] clamped to the
 * grid (reading R12); ellipse mode keeps those whose closed square meets E. */
static int kept_tiles(const orc_proj *p, int tile_cull, int tx_n, int *out) {
  int n = 0;
  for (int ty = p->rect[1]; ty <= p->rect[3]; ++ty)
    for (int tx = p->rect[0]; tx <= p->rect[2]; ++tx) {
      int keep = tile_cull == 0 ? 1 : tile_test(p, 1, tx, ty, 0.0);
      if (keep) { if (out) out[n] = ty * tx_n + tx; ++n; }
    }
  return n;
}

static void preprocess_one(const float *means, const float *rots, const float *scales,
                           const float *opac, const float *sh, int32_t deg, int64_t i,
                           const orc_camera *cam, const orc_options *o, orc_proj *p) {
  memset(p, 0, sizeof(*p));
  double mu[3] = {means[3 * i], means[3 * i + 1], means[3 * i + 2]};
  double q[4] = {rots[4 * i], rots[4 * i + 1], rots[4 * i + 2], rots[4 * i + 3]};
  double s[3] = {scales[3 * i], scales[3 * i + 1], scales[3 * i + 2]};
  double sig = opac[i];
  double R[9];
  /* O1.1-3: validity of the parameters (reading R2) */
  if (!finite3(mu) || !finite3(s) || !isfinite(sig) || orc_quat_to_rot(q, R) != 0 ||
      !(s[0] > 0 && s[1] > 0 && s[2] > 0)) { p->reason = ORC_CULL_PARAM; return; }
  if (!(sig > o->alpha_min)) { p->reason = ORC_CULL_OPACITY; return; }
  /* O1.5-6: weights (Eq. 7-8) and sigma points (Eq. 6) */
  double wmu[7], wsig[7], lam;
  if (orc_ut_weights(o->ut_alpha, o->ut_beta, o->ut_kappa, wmu, wsig, &lam) != 0) {
    p->reason = ORC_CULL_PARAM; return;
  }
  double X[7][3], V[7][2], T[7], minm = 1e300;
  orc_sigma_points(mu, R, s, lam, X);
  /* O2: project every sigma point exactly (Alg. 2 ProjectPoints) */
  int all_valid = 1;
  for (int k = 0; k < 7; ++k) {
    double m;
    int32_t it;
    int v = orc_project_point(cam, o, X[k], V[k], &T[k], &it, &m);
    if (m < minm) minm = m;
    if (it < 0) p->rs_fail = 1;
    if (abs(it) > p->rs_iters) p->rs_iters = abs(it);
    if (!v) all_valid = 0;
  }
  p->cull_ambig = fabs(minm) <= 1e-5;
  if (!all_valid) { p->reason = ORC_CULL_SIGMA; return; } /* reading R9 */
  /* O3.2: Eq. 9 and Eq. 10, then + dilation (reading R10) */
  double vx = 0, vy = 0;
  for (int k = 0; k < 7; ++k) { vx += wmu[k] * V[k][0]; vy += wmu[k] * V[k][1]; }
  double cxx = 0, cxy = 0, cyy = 0;
  for (int k = 0; k < 7; ++k) {
    double dx = V[k][0] - vx, dy = V[k][1] - vy;
    cxx += wsig[k] * dx * dx; cxy += wsig[k] * dx * dy; cyy += wsig[k] * dy * dy;
  }
  cxx += o->dilation; cyy += o->dilation;
  p->vx = vx; p->vy = vy; p->cxx = cxx; p->cxy = cxy; p->cyy = cyy;
  /* depth key (reading R13) and colour (reading R18) at the centre point's pose */
  double Rc[9], cc[3], dd[3], xc[3];
  p->t0 = T[0];
  orc_pose_at(cam, T[0], Rc, cc);
  for (int a = 0; a < 3; ++a) dd[a] = mu[a] - cc[a];
  mtv3(Rc, dd, xc);
  p->depth = sqrt(dot3(xc, xc));
  double nd = sqrt(dot3(dd, dd)), dir[3] = {dd[0] / nd, dd[1] / nd, dd[2] / nd}, Y[16];
  orc_sh_basis(dir, Y);
  int nc = (deg + 1) * (deg + 1);
  for (int ch = 0; ch < 3; ++ch) {
    double acc = 0;
    for (int b = 0; b < nc; ++b) acc += (double)sh[(i * nc + b) * 3 + ch] * Y[b];
    acc += 0.5;
    p->rgb[ch] = acc > 0 ? acc : 0;
  }
  double det = cxx * cyy - cxy * cxy;
  if (!(cxx > 0 && cyy > 0 && det > 0) || !isfinite(det)) { p->reason = ORC_CULL_COV; return; }
  /* O3.3-4: opacity-aware extent (Alg. 1 line 3; reading R11) */
  /* alpha >= alpha_min  <=>  omega^2 <= k2 (Alg. 1 l.3); degree n
   * kernel (Supp. A, reading R29): (1/2) lambda_n omega^n <= ln(sigma/alpha_min) */
  p->k2 = 2.0 * log(sig / o->alpha_min);
  if (o->kernel_degree != 2) p->k2 = pow(p->k2 / orc_kernel_lambda(o->kernel_degree), 2.0 / o->kernel_degree);
  p->hx = sqrt(p->k2 * cxx);
  p->hy = sqrt(p->k2 * cyy);
  /* O3.5: rectangle (Alg. 1 line 5) clamped to the tile grid */
  int tx_n = (cam->width + TILE - 1) / TILE, ty_n = (cam->height + TILE - 1) / TILE;
  int tx0 = (int)floor((vx - p->hx) / TILE), tx1 = (int)floor((vx + p->hx) / TILE);
  int ty0 = (int)floor((vy - p->hy) / TILE), ty1 = (int)floor((vy + p->hy) / TILE);
  /* ambiguity: candidates from the rectangle grown by 1e-3 px */
  {
    const double e = 1e-3;
    int ax0 = (int)floor((vx - p->hx - e) / TILE), ax1 = (int)floor((vx + p->hx + e) / TILE);
    int ay0 = (int)floor((vy - p->hy - e) / TILE), ay1 = (int)floor((vy + p->hy + e) / TILE);
    if (ax0 < 0) ax0 = 0;
    if (ay0 < 0) ay0 = 0;
    if (ax1 > tx_n - 1) ax1 = tx_n - 1;
    if (ay1 > ty_n - 1) ay1 = ty_n - 1;
    for (int ty = ay0; ty <= ay1 && !p->bin_ambig; ++ty)
      for (int tx = ax0; tx <= ax1; ++tx)
        if (tile_test(p, o->tile_cull, tx, ty, e) != tile_test(p, o->tile_cull, tx, ty, -e)) {
          p->bin_ambig = 1; break;
        }
  }
  if (tx0 < 0) tx0 = 0;
  if (ty0 < 0) ty0 = 0;
  if (tx1 > tx_n - 1) tx1 = tx_n - 1;
  if (ty1 > ty_n - 1) ty1 = ty_n - 1;
  p->rect[0] = tx0; p->rect[1] = ty0; p->rect[2] = tx1; p->rect[3] = ty1;
  if (tx0 > tx1 || ty0 > ty1) { p->reason = ORC_CULL_OFFSCREEN; return; }
  /* O3.6: tiles kept */
  p->tiles = kept_tiles(p, o->tile_cull, tx_n, NULL);
  if (p->tiles == 0) { p->reason = ORC_CULL_NOTILE; return; }
  p->reason = ORC_OK;
}

void orc_preprocess(const float *means, const float *rots, const float *scales, const float *opac,
                    const float *sh, int32_t sh_degree, int64_t n, const orc_camera *cam,
                    const orc_options *o, orc_proj *out) {
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < n; ++i)
    preprocess_one(means, rots, scales, opac, sh, sh_degree, i, cam, o, &out[i]);
}

/* ======================================================================
 * O4 — per-tile lists in global depth order ("3DGS sorts them
 * globally for each tile").  The sort key is the 3DGS key: the depth as a
 * 32-bit float, (float)depth, with ties by Gaussian index (readings R13,
 * R13'; SURVEY §8(a)-2 keys = tile << 32 | float bits of the depth).
 * ====================================================================== */
typedef struct { int32_t tile; int32_t gid; float depth; } orc_key;

static int key_cmp(const void *a, const void *b) {
  const orc_key *x = (const orc_key *)a, *y = (const orc_key *)b;
  if (x->tile != y->tile) return x->tile < y->tile ? -1 : 1;
  if (x->depth != y->depth) return x->depth < y->depth ? -1 : 1;
  return x->gid < y->gid ? -1 : (x->gid > y->gid);
}

/* Parity diagnostic for the order of two consecutive contributing entries
 * with fp64 depths di, dj: the smallest relative perturbation of the depths
 * that could change their order under the (fp32 key, index) rule.  Keys two
 * or more fp32 steps apart: the relative depth gap.  Equal or adjacent keys:
 * the distance of either depth to the nearest fp32 rounding boundary (a key
 * that stays the same keeps the index tie-break). */
static double rounding_margin(double d) {
  float f = (float)d;
  double lo = 0.5 * ((double)f + (double)nextafterf(f, 0.f));
  double hi = 0.5 * ((double)f + (double)nextafterf(f, INFINITY));
  return fmin(fabs(d - lo), fabs(hi - d)) / fabs(d);
}
static double order_margin(double di, double dj) {
  float ki = (float)di, kj = (float)dj, km = ki > kj ? ki : kj, kl = ki > kj ? kj : ki;
  if (nextafterf(kl, INFINITY) < km) return fabs(dj - di) / fmax(di, dj);
  return fmin(rounding_margin(di), rounding_margin(dj));
}

int64_t orc_tile_lists(const orc_proj *proj, int64_t n, const orc_camera *cam, const orc_options *o,
                       const float *means, const float *scales, int32_t *tile_of, int32_t *gid_of,
                       int64_t cap, int32_t *ranges) {
  (void)means; (void)scales;
  int tx_n = (cam->width + TILE - 1) / TILE, ty_n = (cam->height + TILE - 1) / TILE;
  int64_t K = 0;
  for (int64_t i = 0; i < n; ++i) if (proj[i].reason == ORC_OK) K += proj[i].tiles;
  if (K > cap || !tile_of) return K;
  orc_key *keys = (orc_key *)malloc(sizeof(orc_key) * (size_t)(K > 0 ? K : 1));
  int *buf = (int *)malloc(sizeof(int) * (size_t)tx_n * ty_n);
  int64_t w = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (proj[i].reason != ORC_OK) continue;
    int m = kept_tiles(&proj[i], o->tile_cull, tx_n, buf);
    for (int j = 0; j < m; ++j) { keys[w].tile = buf[j]; keys[w].gid = (int32_t)i; keys[w].depth = (float)proj[i].depth; ++w; }
  }
  qsort(keys, (size_t)K, sizeof(orc_key), key_cmp);
  for (int t = 0; t < tx_n * ty_n; ++t) { ranges[2 * t] = 0; ranges[2 * t + 1] = 0; }
  for (int64_t k = 0; k < K; ++k) {
    tile_of[k] = keys[k].tile; gid_of[k] = keys[k].gid;
    if (k == 0 || keys[k - 1].tile != keys[k].tile) ranges[2 * keys[k].tile] = (int32_t)k;
    ranges[2 * keys[k].tile + 1] = (int32_t)(k + 1);
  }
  free(keys); free(buf);
  return K;
}

/* ======================================================================
 * O5 — pixel rays r(tau) = o + tau d, ||d|| = 1
 * ====================================================================== */

static double pixel_time(const orc_camera *cam, double u, double v) { /* reading R17 */
  switch (cam->shutter) {
    case ORC_TOP_TO_BOTTOM: return v / cam->height;
    case ORC_BOTTOM_TO_TOP: return 1.0 - v / cam->height;
    case ORC_LEFT_TO_RIGHT: return u / cam->width;
    case ORC_RIGHT_TO_LEFT: return 1.0 - u / cam->width;
    default: return 0.0;
  }
}

int orc_pixel_ray(const orc_camera *cam, double u, double v, double o[3], double d[3]) {
  double oc[3] = {0, 0, 0}, dc[3];
  double xd = (u - cam->cx) / cam->fx, yd = (v - cam->cy) / cam->fy;
  int valid = 1;
  switch (cam->model) {
    case ORC_PINHOLE: dc[0] = xd; dc[1] = yd; dc[2] = 1; break;
    case ORC_ORTHO: oc[0] = xd; oc[1] = yd; dc[0] = 0; dc[1] = 0; dc[2] = 1; break;
    case ORC_OPENCV: {
      /* invert the distortion map by Newton (central-difference Jacobian),
       * start at (xd, yd), <= 50 iterations, residual < 1e-14 */
      double xn = xd, yn = yd;
      int ok = 0;
      for (int it = 0; it < 50; ++it) {
        double fx, fy;
        opencv_distort(cam, xn, yn, &fx, &fy);
        double rx = fx - xd, ry = fy - yd;
        if (sqrt(rx * rx + ry * ry) < 1e-14) { ok = 1; break; }
        const double h = 1e-7;
        double a1, b1, a2, b2, c1, d1, c2, d2;
        opencv_distort(cam, xn + h, yn, &a1, &b1);
        opencv_distort(cam, xn - h, yn, &a2, &b2);
        opencv_distort(cam, xn, yn + h, &c1, &d1);
        opencv_distort(cam, xn, yn - h, &c2, &d2);
        double J00 = (a1 - a2) / (2 * h), J10 = (b1 - b2) / (2 * h);
        double J01 = (c1 - c2) / (2 * h), J11 = (d1 - d2) / (2 * h);
        double det = J00 * J11 - J01 * J10;
        if (!(fabs(det) > 0)) break;
        xn -= (J11 * rx - J01 * ry) / det;
        yn -= (-J10 * rx + J00 * ry) / det;
      }
      if (!ok) valid = 0;
      if (cam->fov_limit > 0 && !(xn * xn + yn * yn <= cam->fov_limit * cam->fov_limit)) valid = 0;
      dc[0] = xn; dc[1] = yn; dc[2] = 1;
      break;
    }
    case ORC_FISHEYE: {
      double tdn = sqrt(xd * xd + yd * yd);
      double th = tdn;
      for (int it = 0; it < 50; ++it) { /* Newton on theta_d(theta) = tdn */
        double t2 = th * th;
        double f = fisheye_theta_d(cam, th) - tdn;
        double fp = 1 + 3 * cam->k[0] * t2 + 5 * cam->k[1] * t2 * t2 + 7 * cam->k[2] * t2 * t2 * t2 +
                    9 * cam->k[3] * t2 * t2 * t2 * t2;
        double step = f / fp;
        th -= step;
        if (fabs(step) < 1e-16) break;
      }
      double thmax = cam->fov_limit > 0 ? cam->fov_limit : M_PI;
      if (!(th <= thmax) || fabs(fisheye_theta_d(cam, th) - tdn) > 1e-12) valid = 0;
      if (tdn == 0.0) { dc[0] = 0; dc[1] = 0; dc[2] = 1; }
      else { dc[0] = sin(th) * xd / tdn; dc[1] = sin(th) * yd / tdn; dc[2] = cos(th); }
      break;
    }
    default: return 0;
  }
  double nd = sqrt(dot3(dc, dc));
  for (int a = 0; a < 3; ++a) dc[a] /= nd;
  double R[9], c[3];
  orc_pose_at(cam, pixel_time(cam, u, v), R, c);
  double ro[3];
  mv3(R, oc, ro);
  mv3(R, dc, d);
  for (int a = 0; a < 3; ++a) o[a] = c[a] + ro[a];
  return valid;
}

/* ======================================================================
 * O6 — 3D max response (Eq. 11) and front-to-back compositing (Eq. 5)
 * ====================================================================== */

/* Eq. 11: o_g = S^-1 R^T (o - mu), d_g = S^-1 R^T d,
 * tau_max = -o_g.d_g / d_g.d_g (a ray distance since ||d|| = 1); the response
 * at tau_max is exp(-omega^2/2) with omega^2 = ||o_g + tau_max d_g||^2
 * (Supp. B) = ||o_g x d_g||^2 / ||d_g||^2 (reading R25). Returns omega^2. */
double orc_max_response(const double mu[3], const double R[9], const double s[3], const double o[3],
                        const double d[3], double *tau) {
  double om[3] = {o[0] - mu[0], o[1] - mu[1], o[2] - mu[2]}, og[3], dg[3];
  mtv3(R, om, og);
  mtv3(R, d, dg);
  for (int a = 0; a < 3; ++a) { og[a] /= s[a]; dg[a] /= s[a]; }
  double dd = dot3(dg, dg), cr[3];
  cross3(og, dg, cr);
  if (tau) *tau = -dot3(og, dg) / dd;
  return dot3(cr, cr) / dd;
}

typedef struct { double mu[3], R[9], s[3], sig, rgb[3]; } orc_gauss;

static void load_gauss(const float *means, const float *rots, const float *scales, const float *opac,
                       const orc_proj *proj, int64_t i, orc_gauss *g) {
  double q[4] = {rots[4 * i], rots[4 * i + 1], rots[4 * i + 2], rots[4 * i + 3]};
  orc_quat_to_rot(q, g->R);
  for (int a = 0; a < 3; ++a) { g->mu[a] = means[3 * i + a]; g->s[a] = scales[3 * i + a]; }
  g->sig = opac[i];
  if (proj) for (int a = 0; a < 3; ++a) g->rgb[a] = proj[i].rgb[a];
}

/* ----------------------------------------------------------------------
 * O6' — per-ray hit order of "Ours (sorted)" (§4.3; reading R28).
 * "storing the per-ray k-farthest hit particles (typically using k = 16) in a
 * buffer.  The closest hits which cannot be stored in the buffer are
 * incrementally alpha-blended until the transmittance of the blended part
 * vanishes."  Hits (alpha >= alpha_min, tau_max > 0) arrive in the tile's
 * global depth order (O4).  While at most k hits are pending they are stored;
 * a further hit makes k + 1 pending hits and the closest of them (smallest
 * tau_max, ties: earlier in the stream) is alpha-blended -- so the buffer
 * always holds the k farthest pending hits.  At the end of the stream the
 * buffer is blended near to far.  Blending is Eq. 5 with the termination rule
 * R21 (a hit that would take T below T_min stops the ray unblended).
 * k = -1: every hit blended in exact tau_max order (the order 3DGRT's tracer
 * collects); k = 0: stream order (= O6, "Ours").
 * ---------------------------------------------------------------------- */
typedef struct { double tau, alpha, rgb[3]; int32_t pos; } orc_hit;

static int dbl_cmp(const void *a, const void *b) {
  double x = *(const double *)a, y = *(const double *)b;
  return x < y ? -1 : (x > y);
}

static int hit_cmp(const void *a, const void *b) {
  const orc_hit *x = (const orc_hit *)a, *y = (const orc_hit *)b;
  if (x->tau != y->tau) return x->tau < y->tau ? -1 : 1;
  return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

/* Eq. 5 step for one hit; returns 1 if the ray terminates (hit not blended) */
static int blend_hit(const orc_hit *h, double t_min, double C[3], double *T, double *D, double *min_term_gap) {
  double Tn = *T * (1.0 - h->alpha);
  double tg = fabs(Tn - t_min);
  if (min_term_gap && tg < *min_term_gap) *min_term_gap = tg;
  if (Tn < t_min) return 1;
  for (int c = 0; c < 3; ++c) C[c] += h->alpha * *T * h->rgb[c];
  *D += h->alpha * *T * h->tau;
  *T = Tn;
  return 0;
}

int32_t orc_kbuffer_blend(const double *tau, const double *alpha, const double *rgb, int32_t n, int32_t k,
                          double t_min, double C[3], double *T_out, double *D_out, int32_t *n_blended,
                          double *min_term_gap) {
  double T = 1.0, D = 0.0;
  int32_t nb = 0, consumed = n, dead = 0;
  C[0] = C[1] = C[2] = 0.0;
  orc_hit *buf = (orc_hit *)malloc(sizeof(orc_hit) * (size_t)(n > 0 ? n : 1));
  int32_t m = 0;
  for (int32_t i = 0; i < n && !dead; ++i) {
    orc_hit h = {tau[i], alpha[i], {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]}, i};
    if (k == 0) {                       /* stream order */
      dead = blend_hit(&h, t_min, C, &T, &D, min_term_gap);
      if (dead) consumed = i + 1; else ++nb;
      continue;
    }
    buf[m++] = h;
    if (k > 0 && m > k) {               /* k + 1 pending: blend the closest */
      int32_t j = 0;
      for (int32_t q = 1; q < m; ++q) if (hit_cmp(&buf[q], &buf[j]) < 0) j = q;
      orc_hit c = buf[j];
      buf[j] = buf[--m];
      dead = blend_hit(&c, t_min, C, &T, &D, min_term_gap);
      if (dead) consumed = i + 1; else ++nb;
    }
  }
  if (!dead && k != 0) {                /* end of stream: the pending hits near to far */
    qsort(buf, (size_t)m, sizeof(orc_hit), hit_cmp);
    for (int32_t j = 0; j < m; ++j) {
      if (blend_hit(&buf[j], t_min, C, &T, &D, min_term_gap)) break;
      ++nb;
    }
  }
  free(buf);
  *T_out = T;
  *D_out = D;
  if (n_blended) *n_blended = nb;
  return consumed;
}

static double g_alt_band = 2e-6;
void orc_set_alt_band(double band) { g_alt_band = band; }

/* one pixel of "Ours (sorted)": the hit stream of the tile list, then O6' */
static void composite_pixel_sorted(const orc_gauss *G, const int32_t *gids, int32_t a, int32_t b,
                                   const double *depth_of, const double o[3], const double d[3],
                                   const orc_options *opt, double C[3], double *T_out, double *Dp,
                                   orc_pixdiag *dg) {
  int32_t n = 0, cap = b > a ? b - a : 1;
  double *tau = (double *)malloc(sizeof(double) * (size_t)cap);
  double *al = (double *)malloc(sizeof(double) * (size_t)cap);
  double *rgb = (double *)malloc(sizeof(double) * 3 * (size_t)cap);
  double *dk = (double *)malloc(sizeof(double) * (size_t)cap);
  for (int32_t k = a; k < b; ++k) {
    const orc_gauss *g = &G[gids[k]];
    double t, w2 = orc_max_response(g->mu, g->R, g->s, o, d, &t);
    double x = g->sig * orc_kernel_response(w2, opt->kernel_degree);
    if (x > opt->alpha_max) x = opt->alpha_max;
    if (dg) {
      dg->visited++;
      double gap = fabs(x - opt->alpha_min);
      if (gap < dg->min_alpha_gap) dg->min_alpha_gap = gap;
    }
    if (x < opt->alpha_min) continue;
    if (!(t > 0.0)) continue;            /* reading R24 */
    tau[n] = t; al[n] = x;
    for (int c = 0; c < 3; ++c) rgb[3 * n + c] = g->rgb[c];
    dk[n] = depth_of ? depth_of[gids[k]] : 0;
    ++n;
  }
  int32_t nb = 0;
  double tg = 1e300;
  int32_t used = orc_kbuffer_blend(tau, al, rgb, n, opt->kbuffer, opt->t_min, C, T_out, Dp, &nb, &tg);
  if (dg) {
    dg->contributed = nb;
    dg->terminated = nb < n;   /* every hit is blended unless the ray terminates */
    if (tg < dg->min_term_gap) dg->min_term_gap = tg;
    /* order ambiguity over the hits that reached the buffer: stream (depth key)
     * neighbours and tau_max neighbours */
    for (int32_t i = 1; i < used; ++i) {
      double rg = order_margin(dk[i - 1], dk[i]);
      if (rg < dg->min_order_gap) dg->min_order_gap = rg;
    }
    /* tau-order neighbours among the consumed hits (indices sorted by tau) */
    int32_t *ix = (int32_t *)malloc(sizeof(int32_t) * (size_t)(used > 0 ? used : 1));
    for (int32_t i = 0; i < used; ++i) ix[i] = i;
    for (int32_t i = 1; i < used; ++i) {  /* insertion sort by tau (short streams) */
      int32_t v = ix[i], j = i - 1;
      while (j >= 0 && tau[ix[j]] > tau[v]) { ix[j + 1] = ix[j]; --j; }
      ix[j + 1] = v;
    }
    int32_t npair = 0, pa = -1, pb = -1;
    for (int32_t i = 1; i < used; ++i) {
      double ta = tau[ix[i]], tb = tau[ix[i - 1]];
      double rg = fabs(ta - tb) / fmax(fabs(ta), fabs(tb));
      if (rg < dg->min_tau_gap) dg->min_tau_gap = rg;
      if (rg <= g_alt_band) { ++npair; pa = ix[i - 1]; pb = ix[i]; }
    }
    free(ix);
    /* one near-tie: the same stream with the two hits' tau_max exchanged is the
     * other order an fp32 tau could produce; the test accepts either render */
    if (npair == 1) {
      double t2 = tau[pa];
      tau[pa] = tau[pb];
      tau[pb] = t2;
      double Ca[3], Ta, Da, tga = 1e300;
      int32_t nba = 0;
      orc_kbuffer_blend(tau, al, rgb, n, opt->kbuffer, opt->t_min, Ca, &Ta, &Da, &nba, &tga);
      dg->alt_valid = 1;
      for (int c = 0; c < 3; ++c) dg->alt_rgb[c] = Ca[c];
      dg->alt_alpha = 1.0 - Ta;
      dg->alt_depth = Da;
    }
  }
  free(tau); free(al); free(rgb); free(dk);
}

/* one pixel: Eq. 5 front to back with alpha_i = sigma_i rho_i(o + tau_max d)
 * (P:L121), alpha clamp / skip / termination per readings R20-R21 */
static void composite_pixel(const orc_gauss *G, const int32_t *gids, int32_t a, int32_t b,
                            const double *depth_of, const double o[3], const double d[3],
                            const orc_options *opt, double C[3], double *T_out, double *Dp,
                            orc_pixdiag *dg) {
  if (opt->kbuffer != 0) { composite_pixel_sorted(G, gids, a, b, depth_of, o, d, opt, C, T_out, Dp, dg); return; }
  double T = 1.0;
  C[0] = C[1] = C[2] = 0; *Dp = 0;
  double prev_depth = -1;
  for (int32_t k = a; k < b; ++k) {
    const orc_gauss *g = &G[gids[k]];
    double tau, w2 = orc_max_response(g->mu, g->R, g->s, o, d, &tau);
    double al = g->sig * orc_kernel_response(w2, opt->kernel_degree);
    if (al > opt->alpha_max) al = opt->alpha_max;
    if (dg) {
      dg->visited++;
      double gap = fabs(al - opt->alpha_min);
      if (gap < dg->min_alpha_gap) dg->min_alpha_gap = gap;
    }
    if (al < opt->alpha_min) continue;
    /* reading R24: only hits in front of the ray origin, tau_max > 0
     * ("alpha_i = sigma_i rho_i(o + tau d) for any tau in R+") */
    if (!(tau > 0.0)) continue;
    double Tn = T * (1.0 - al);
    if (dg) {
      double tg = fabs(Tn - opt->t_min);
      if (tg < dg->min_term_gap) dg->min_term_gap = tg;
      double dep = depth_of ? depth_of[gids[k]] : 0;
      if (prev_depth >= 0 && depth_of) {
        double rg = order_margin(prev_depth, dep);
        if (rg < dg->min_order_gap) dg->min_order_gap = rg;
      }
      prev_depth = dep;
    }
    if (Tn < opt->t_min) { if (dg) dg->terminated = 1; break; }
    for (int c = 0; c < 3; ++c) C[c] += al * T * g->rgb[c];
    *Dp += al * T * tau;
    T = Tn;
    if (dg) dg->contributed++;
  }
  *T_out = T;
}

void orc_composite(const float *means, const float *rots, const float *scales, const float *opac,
                   const orc_proj *proj, const int32_t *gids, const int32_t *ranges,
                   const orc_camera *cam, const orc_options *o, const int32_t *tile_subset,
                   int32_t n_subset, float *rgb, float *alpha, float *depth, orc_pixdiag *diag) {
  int tx_n = (cam->width + TILE - 1) / TILE, ty_n = (cam->height + TILE - 1) / TILE;
  int n_tiles = tile_subset ? n_subset : tx_n * ty_n;
  /* per-Gaussian constants for the Gaussians referenced by the lists */
  int64_t maxg = -1;
  for (int t = 0; t < tx_n * ty_n; ++t)
    for (int32_t k = ranges[2 * t]; k < ranges[2 * t + 1]; ++k) if (gids[k] > maxg) maxg = gids[k];
  int64_t ng = maxg + 1;
  orc_gauss *G = (orc_gauss *)malloc(sizeof(orc_gauss) * (size_t)(ng > 0 ? ng : 1));
  double *dep = (double *)malloc(sizeof(double) * (size_t)(ng > 0 ? ng : 1));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < ng; ++i) { load_gauss(means, rots, scales, opac, proj, i, &G[i]); dep[i] = proj[i].depth; }
#pragma omp parallel for schedule(dynamic, 1)
  for (int ti = 0; ti < n_tiles; ++ti) {
    int t = tile_subset ? tile_subset[ti] : ti;
    int tx = t % tx_n, ty = t / tx_n;
    for (int py = ty * TILE; py < ty * TILE + TILE && py < cam->height; ++py)
      for (int px = tx * TILE; px < tx * TILE + TILE && px < cam->width; ++px) {
        int64_t pix = (int64_t)py * cam->width + px;
        orc_pixdiag dg;
        memset(&dg, 0, sizeof(dg));
        dg.min_alpha_gap = dg.min_term_gap = dg.min_order_gap = dg.min_tau_gap = 1e300;
        double ro[3], rd[3], C[3], T, Dp;
        if (!orc_pixel_ray(cam, px + 0.5, py + 0.5, ro, rd)) {
          /* invalid pixel: RGB = bg, alpha = 0, depth = 0 (O5) */
          for (int c = 0; c < 3; ++c) rgb[3 * pix + c] = (float)o->bg[c];
          alpha[pix] = 0; depth[pix] = 0; dg.invalid = 1;
        } else {
          composite_pixel(G, gids, ranges[2 * t], ranges[2 * t + 1], dep, ro, rd, o, C, &T, &Dp, &dg);
          for (int c = 0; c < 3; ++c) rgb[3 * pix + c] = (float)(C[c] + T * o->bg[c]);
          alpha[pix] = (float)(1.0 - T);
          depth[pix] = (float)Dp;
        }
        if (diag) diag[pix] = dg;
      }
  }
  free(G); free(dep);
}

/* order of the brute-force list: ((float)depth, index) as O4 */
typedef struct { float depth; int32_t gid; } orc_dk;
static int dk_cmp(const void *a, const void *b) {
  const orc_dk *x = (const orc_dk *)a, *y = (const orc_dk *)b;
  if (x->depth != y->depth) return x->depth < y->depth ? -1 : 1;
  return x->gid < y->gid ? -1 : (x->gid > y->gid);
}

int64_t orc_render(const float *means, const float *rots, const float *scales, const float *opac,
                   const float *sh, int32_t sh_degree, int64_t n, const orc_camera *cam,
                   const orc_options *o, int32_t brute, const int32_t *tile_subset, int32_t n_subset,
                   float *rgb, float *alpha, float *depth, orc_pixdiag *diag, orc_proj *proj_out,
                   int64_t *n_keys_out) {
  int tx_n = (cam->width + TILE - 1) / TILE, ty_n = (cam->height + TILE - 1) / TILE, nt = tx_n * ty_n;
  orc_proj *proj = proj_out ? proj_out : (orc_proj *)malloc(sizeof(orc_proj) * (size_t)(n > 0 ? n : 1));
  orc_preprocess(means, rots, scales, opac, sh, sh_degree, n, cam, o, proj);
  int32_t *ranges = (int32_t *)calloc((size_t)nt * 2, sizeof(int32_t));
  int32_t *gids = NULL, *tiles = NULL;
  int64_t K = 0;
  if (!brute) {
    K = orc_tile_lists(proj, n, cam, o, means, scales, NULL, NULL, 0, NULL);
    tiles = (int32_t *)malloc(sizeof(int32_t) * (size_t)(K > 0 ? K : 1));
    gids = (int32_t *)malloc(sizeof(int32_t) * (size_t)(K > 0 ? K : 1));
    orc_tile_lists(proj, n, cam, o, means, scales, tiles, gids, K, ranges);
  } else {
    /* brute force (SURVEY §8(c).2 mode B): every Gaussian valid through O1-O3
     * (ignoring rectangles and tiles), sorted by ((float)depth, index), at every pixel */
    orc_dk *l = (orc_dk *)malloc(sizeof(orc_dk) * (size_t)(n > 0 ? n : 1));
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i) {
      int r = proj[i].reason;
      if (r == ORC_OK || r == ORC_CULL_OFFSCREEN || r == ORC_CULL_NOTILE) { l[m].depth = (float)proj[i].depth; l[m].gid = (int32_t)i; ++m; }
    }
    qsort(l, (size_t)m, sizeof(orc_dk), dk_cmp);
    gids = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    for (int64_t k = 0; k < m; ++k) gids[k] = l[k].gid;
    for (int t = 0; t < nt; ++t) { ranges[2 * t] = 0; ranges[2 * t + 1] = (int32_t)m; }
    free(l);
    K = m;
  }
  orc_composite(means, rots, scales, opac, proj, gids, ranges, cam, o, tile_subset, n_subset, rgb,
                alpha, depth, diag);
  if (n_keys_out) *n_keys_out = K;
  free(ranges); free(gids); free(tiles);
  if (!proj_out) free(proj);
  return K;
}

/* Pixels that a binning-ambiguous (Gaussian, tile) pair or a cull-ambiguous
 * Gaussian could change: the Gaussian's alpha at the pixel
 * is >= alpha_min - alpha_eps. */
void orc_mark_ambiguity(const float *means, const float *rots, const float *scales, const float *opac,
                        const orc_proj *proj, int64_t n, const orc_camera *cam, const orc_options *o,
                        double alpha_eps, const int32_t *tile_subset, int32_t n_subset, orc_pixdiag *diag) {
  int tx_n = (cam->width + TILE - 1) / TILE, ty_n = (cam->height + TILE - 1) / TILE;
  const double e = 1e-3;
  char *in_sub = (char *)malloc((size_t)tx_n * ty_n);
  memset(in_sub, tile_subset ? 0 : 1, (size_t)tx_n * ty_n);
  if (tile_subset) for (int k = 0; k < n_subset; ++k) in_sub[tile_subset[k]] = 1;
  for (int64_t i = 0; i < n; ++i) {
    const orc_proj *p = &proj[i];
    int is_bin = p->bin_ambig && (p->reason == ORC_OK || p->reason == ORC_CULL_OFFSCREEN || p->reason == ORC_CULL_NOTILE);
    int is_cull = p->cull_ambig && p->reason != ORC_CULL_PARAM && p->reason != ORC_CULL_OPACITY;
    if (!is_bin && !is_cull) continue;
    orc_gauss g;
    load_gauss(means, rots, scales, opac, NULL, i, &g);
    int ax0 = 0, ax1 = tx_n - 1, ay0 = 0, ay1 = ty_n - 1;
    if (!is_cull) {
      ax0 = (int)floor((p->vx - p->hx - e) / TILE); ax1 = (int)floor((p->vx + p->hx + e) / TILE);
      ay0 = (int)floor((p->vy - p->hy - e) / TILE); ay1 = (int)floor((p->vy + p->hy + e) / TILE);
      if (ax0 < 0) ax0 = 0;
      if (ay0 < 0) ay0 = 0;
      if (ax1 > tx_n - 1) ax1 = tx_n - 1;
      if (ay1 > ty_n - 1) ay1 = ty_n - 1;
    }
    for (int ty = ay0; ty <= ay1; ++ty)
      for (int tx = ax0; tx <= ax1; ++tx) {
        if (!in_sub[ty * tx_n + tx]) continue;
        if (!is_cull && tile_test(p, o->tile_cull, tx, ty, e) == tile_test(p, o->tile_cull, tx, ty, -e)) continue;
#pragma omp parallel for schedule(static)
        for (int py = ty * TILE; py < ty * TILE + TILE; ++py) {
          if (py >= cam->height) continue;
          for (int px = tx * TILE; px < tx * TILE + TILE && px < cam->width; ++px) {
            double ro[3], rd[3], tau;
            if (!orc_pixel_ray(cam, px + 0.5, py + 0.5, ro, rd)) continue;
            double w2 = orc_max_response(g.mu, g.R, g.s, ro, rd, &tau);
            double al = g.sig * orc_kernel_response(w2, o->kernel_degree);
            if (al >= o->alpha_min - alpha_eps) {
              if (is_cull) diag[(int64_t)py * cam->width + px].amb_cull = 1;
              else diag[(int64_t)py * cam->width + px].amb_bin = 1;
            }
          }
        }
      }
  }
  free(in_sub);
}

/* ======================================================================
 * O7 — backward pass of the compositing and the 3D response (Supp. B,
 * P:L494-513; "avoids propagating gradients through the projection", P:L202:
 * the UT / binning is not differentiated, reading R30).  Scalar loss
 * L = sum_px g_rgb . rgb + g_alpha alpha + g_depth depth with the given
 * per-pixel upstream gradients; "Ours" order (kbuffer = 0); any kernel degree
 * (Supp. A) and camera incl. rolling shutter (the pixel rays of O5).
 * Plain fp64 chain rule, written out per hit:
 *   Eq. 5: w_i = alpha_i T_i, C = sum w_i c_i, D = sum w_i tau_i, T_f = prod(1 - alpha_i)
 *   dL/dc_i = w_i g_rgb;  dL/dtau_i = w_i g_depth
 *   dL/dalpha_i = T_i (c_i.g_rgb + tau_i g_depth) - S_i / (1 - alpha_i),
 *     S_i = sum_{j>i} w_j (c_j.g_rgb + tau_j g_depth) + T_f (bg.g_rgb - g_alpha)
 *   alpha = min(alpha_max, sigma rho), rho = exp(-omega^2/2)  (clamped: no gradient)
 *   Eq. 11 with o_g = M (o - mu), d_g = M d, M = S^-1 R^T, x_g = o_g + tau d_g:
 *     d omega^2 / d o_g = 2 x_g,  d omega^2 / d d_g = 2 tau x_g,
 *     d tau / d o_g = -d_g / |d_g|^2,  d tau / d d_g = -(x_g + tau d_g) / |d_g|^2
 *   dL/dmu = -M^T dL/do_g;  dL/dM = dL/do_g (o - mu)^T + dL/dd_g d^T
 *   M_ij = R_ji / s_i: dL/ds_i = -(1/s_i) sum_j dL/dM_ij M_ij, dL/dR_ji = dL/dM_ij / s_i
 *   R(q^), q^ = q/|q| (Eq. 2): dL/dq = (I - q^ q^T) dL/dq^ / |q|
 *   colour c = max(0, sum_k sh_k Y_k(dir) + 1/2) at the forward's direction
 *   (reading R18, held constant): dL/dsh_k = dL/dc Y_k where c > 0.
 * ====================================================================== */
typedef struct { int32_t gid; double al, rho, T, tau, g, w2; int clamped; } orc_bhit;

int64_t orc_backward(const float *means, const float *rots, const float *scales, const float *opac,
                     const float *sh, int32_t sh_degree, int64_t n, const orc_camera *cam,
                     const orc_options *o, const float *g_rgb, const float *g_alpha, const float *g_depth,
                     double *d_means, double *d_rots, double *d_scales, double *d_opac, double *d_sh,
                     double *d_rgb, double *loss) {
  int tx_n = (cam->width + TILE - 1) / TILE, ty_n = (cam->height + TILE - 1) / TILE, nt = tx_n * ty_n;
  int nc = (sh_degree + 1) * (sh_degree + 1);
  orc_proj *proj = (orc_proj *)malloc(sizeof(orc_proj) * (size_t)(n > 0 ? n : 1));
  orc_preprocess(means, rots, scales, opac, sh, sh_degree, n, cam, o, proj);
  int32_t *ranges = (int32_t *)calloc((size_t)nt * 2, sizeof(int32_t));
  int64_t K = orc_tile_lists(proj, n, cam, o, means, scales, NULL, NULL, 0, NULL);
  int32_t *tiles = (int32_t *)malloc(sizeof(int32_t) * (size_t)(K > 0 ? K : 1));
  int32_t *gids = (int32_t *)malloc(sizeof(int32_t) * (size_t)(K > 0 ? K : 1));
  orc_tile_lists(proj, n, cam, o, means, scales, tiles, gids, K, ranges);
  orc_gauss *G = (orc_gauss *)malloc(sizeof(orc_gauss) * (size_t)(n > 0 ? n : 1));
  double *gM = (double *)calloc((size_t)(n > 0 ? n : 1) * 9, sizeof(double));
  for (int64_t i = 0; i < n; ++i) load_gauss(means, rots, scales, opac, proj, i, &G[i]);
  memset(d_means, 0, sizeof(double) * 3 * (size_t)n); memset(d_rots, 0, sizeof(double) * 4 * (size_t)n);
  memset(d_scales, 0, sizeof(double) * 3 * (size_t)n); memset(d_opac, 0, sizeof(double) * (size_t)n);
  memset(d_sh, 0, sizeof(double) * 3 * (size_t)nc * (size_t)n); memset(d_rgb, 0, sizeof(double) * 3 * (size_t)n);
  orc_bhit *hits = (orc_bhit *)malloc(sizeof(orc_bhit) * (size_t)(K > 0 ? K : 1));
  double Lsum = 0.0;  /* the forward loss in fp64 (finite-difference pins) */
  for (int t = 0; t < nt; ++t) {
    int tx = t % tx_n, ty = t / tx_n;
    for (int py = ty * TILE; py < ty * TILE + TILE && py < cam->height; ++py)
      for (int px = tx * TILE; px < tx * TILE + TILE && px < cam->width; ++px) {
        int64_t pix = (int64_t)py * cam->width + px;
        const double gc[3] = {g_rgb[3 * pix], g_rgb[3 * pix + 1], g_rgb[3 * pix + 2]};
        const double ga = g_alpha[pix], gdp = g_depth[pix];
        /* a pixel with zero upstream gradient adds exactly nothing to L or to any
         * gradient: skipped (sampled full-size checks zero all but a few tiles) */
        if (gc[0] == 0.0 && gc[1] == 0.0 && gc[2] == 0.0 && ga == 0.0 && gdp == 0.0) continue;
        double ro[3], rd[3];
        if (!orc_pixel_ray(cam, px + 0.5, py + 0.5, ro, rd)) continue;
        /* forward walk (= O6, kbuffer 0) recording the blended hits */
        double T = 1.0;
        int m = 0;
        for (int32_t k = ranges[2 * t]; k < ranges[2 * t + 1]; ++k) {
          const orc_gauss *g = &G[gids[k]];
          double tau, w2 = orc_max_response(g->mu, g->R, g->s, ro, rd, &tau);
          double rho = orc_kernel_response(w2, o->kernel_degree), al = g->sig * rho;
          int clamped = al > o->alpha_max;
          if (clamped) al = o->alpha_max;
          if (al < o->alpha_min || !(tau > 0.0)) continue;
          double Tn = T * (1.0 - al);
          if (Tn < o->t_min) break;
          orc_bhit h = {gids[k], al, rho, T, tau, 0.0, w2, clamped};
          h.g = g->rgb[0] * gc[0] + g->rgb[1] * gc[1] + g->rgb[2] * gc[2] + tau * gdp;
          hits[m++] = h;
          T = Tn;
        }
        double S = T * (o->bg[0] * gc[0] + o->bg[1] * gc[1] + o->bg[2] * gc[2] - ga);
        for (int q = 0; q < m; ++q) S += hits[q].al * hits[q].T * hits[q].g;
        Lsum += S + ga;  /* = rgb.g_rgb + depth g_depth + alpha g_alpha (alpha = 1 - T_f) */
        /* backward, front to back with the running suffix S_i */
        for (int q = 0; q < m; ++q) {
          const orc_bhit *h = &hits[q];
          const orc_gauss *g = &G[h->gid];
          const double w = h->al * h->T;
          S -= w * h->g;                               /* S_i = sum over j > i (+ T_f term) */
          const double dal = h->T * h->g - S / (1.0 - h->al);
          for (int c = 0; c < 3; ++c) d_rgb[3 * h->gid + c] += w * gc[c];
          const double dtau = w * gdp;
          double dw2 = 0.0;
          if (!h->clamped) {
            d_opac[h->gid] += h->rho * dal;
            /* d rho / d omega^2 = -(1/2) lambda_n (n/2) (omega^2)^(n/2 - 1) rho (Supp. A; n = 2: -rho/2) */
            const int32_t nd = o->kernel_degree;
            const double drho = nd == 2 ? -0.5 * h->rho
                                        : -0.5 * orc_kernel_lambda(nd) * 0.5 * nd * pow(h->w2, 0.5 * nd - 1.0) * h->rho;
            dw2 = g->sig * drho * dal;
          }
          /* Eq. 11 chain */
          double om[3] = {ro[0] - g->mu[0], ro[1] - g->mu[1], ro[2] - g->mu[2]}, og[3], dg[3];
          mtv3(g->R, om, og);
          mtv3(g->R, rd, dg);
          for (int a = 0; a < 3; ++a) { og[a] /= g->s[a]; dg[a] /= g->s[a]; }
          const double dd = dot3(dg, dg), tau = -dot3(og, dg) / dd;
          double xg[3], go[3], gd[3];
          for (int a = 0; a < 3; ++a) xg[a] = og[a] + tau * dg[a];
          for (int a = 0; a < 3; ++a) {
            go[a] = dw2 * 2.0 * xg[a] - dtau * dg[a] / dd;
            gd[a] = dw2 * 2.0 * tau * xg[a] - dtau * (xg[a] + tau * dg[a]) / dd;
          }
          /* M = S^-1 R^T: M_ij = R_ji / s_i;  dL/dmu = -M^T go */
          for (int j = 0; j < 3; ++j) {
            double acc = 0;
            for (int i = 0; i < 3; ++i) acc += (g->R[3 * j + i] / g->s[i]) * go[i];
            d_means[3 * h->gid + j] -= acc;
          }
          for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) gM[9 * (size_t)h->gid + 3 * i + j] += go[i] * om[j] + gd[i] * rd[j];
        }
      }
  }
  /* per Gaussian: M -> (s, R) -> q; colour -> SH */
  for (int64_t i = 0; i < n; ++i) {
    const orc_gauss *g = &G[i];
    const double *gm = &gM[9 * (size_t)i];
    double gR[9];  /* dL/dR_ji = dL/dM_ij / s_i */
    for (int a = 0; a < 3; ++a) {
      double acc = 0;
      for (int j = 0; j < 3; ++j) acc += gm[3 * a + j] * (g->R[3 * j + a] / g->s[a]);
      d_scales[3 * i + a] = -acc / g->s[a];
      for (int j = 0; j < 3; ++j) gR[3 * j + a] = gm[3 * a + j] / g->s[a];
    }
    double qn = sqrt((double)rots[4 * i] * rots[4 * i] + (double)rots[4 * i + 1] * rots[4 * i + 1] +
                     (double)rots[4 * i + 2] * rots[4 * i + 2] + (double)rots[4 * i + 3] * rots[4 * i + 3]);
    if (qn > 0) {
      double w = rots[4 * i] / qn, x = rots[4 * i + 1] / qn, y = rots[4 * i + 2] / qn, z = rots[4 * i + 3] / qn;
      const double dRw[9] = {0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0};
      const double dRx[9] = {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x};
      const double dRy[9] = {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y};
      const double dRz[9] = {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0};
      double gq[4] = {0, 0, 0, 0};
      for (int k = 0; k < 9; ++k) { gq[0] += gR[k] * dRw[k]; gq[1] += gR[k] * dRx[k]; gq[2] += gR[k] * dRy[k]; gq[3] += gR[k] * dRz[k]; }
      const double qh[4] = {w, x, y, z}, pr = gq[0] * w + gq[1] * x + gq[2] * y + gq[3] * z;
      for (int k = 0; k < 4; ++k) d_rots[4 * i + k] = (gq[k] - qh[k] * pr) / qn;
    }
    /* SH: the forward's direction (reading R18) and clamp */
    if (proj[i].reason != ORC_OK) continue;
    double Rc[9], cc[3], dd[3], Y[16];
    orc_pose_at(cam, proj[i].t0, Rc, cc);
    for (int a = 0; a < 3; ++a) dd[a] = g->mu[a] - cc[a];
    double nd = sqrt(dot3(dd, dd)), dir[3] = {dd[0] / nd, dd[1] / nd, dd[2] / nd};
    orc_sh_basis(dir, Y);
    for (int ch = 0; ch < 3; ++ch) {
      if (!(proj[i].rgb[ch] > 0)) continue;
      for (int b = 0; b < nc; ++b) d_sh[(i * nc + b) * 3 + ch] = d_rgb[3 * i + ch] * Y[b];
    }
  }
  free(hits); free(gM); free(G); free(gids); free(tiles); free(ranges); free(proj);
  if (loss) *loss = Lsum;
  return K;
}

/* ======================================================================
 * O8 — projection quality (Supp. C): for one Gaussian, its 2D
 * image as estimated by (a) the UT (Eq. 6-10, O3 without the binning
 * dilation), (b) EWA, the first-order linearisation at mu (Eq. 3):
 * mean g(mu), covariance J Sigma J^T with J the central-difference Jacobian of
 * the camera projection at mu's camera-frame point under the pose frozen at
 * mu's own shutter time (RS-unaware, as the paper's EWA baseline), and
 * (c) Monte Carlo: n samples x = mu + R S z, z ~ N(0, I3) from the shared
 * counter-based generator below, each projected exactly (O2, RS-aware); sample
 * mean and covariance (1/n).  KL(N_mc || N_ut) and KL(N_mc || N_ewa) in closed
 * form (reading R31).  valid = 0 if any point fails to project.
 * ====================================================================== */
/* counter-based N(0,1) triple (shared spec with the GPU, implemented twice):
 * splitmix64 finaliser of (seed, gaussian, sample, k); 53-bit uniforms in
 * (0,1); Box-Muller in fp64 (z0, z1 from (u0, u1); z2 from (u2, u3)). */
static uint64_t orc_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
void orc_normal3(uint64_t seed, int64_t gid, int32_t s, double z[3]) {
  double u[4];
  for (int k = 0; k < 4; ++k) {
    uint64_t h = orc_mix64(seed ^ orc_mix64(((uint64_t)gid << 24) ^ ((uint64_t)s << 2) ^ (uint64_t)k));
    u[k] = ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  }
  const double two_pi = 6.283185307179586476925286766559;
  double r0 = sqrt(-2.0 * log(u[0])), r1 = sqrt(-2.0 * log(u[2]));
  z[0] = r0 * cos(two_pi * u[1]);
  z[1] = r0 * sin(two_pi * u[1]);
  z[2] = r1 * cos(two_pi * u[3]);
}

/* KL(N0 || N1) for 2D Gaussians g = (mx, my, cxx, cxy, cyy) */
double orc_kl2(const double g0[5], const double g1[5]) {
  double d1 = g1[2] * g1[4] - g1[3] * g1[3], d0 = g0[2] * g0[4] - g0[3] * g0[3];
  double i00 = g1[4] / d1, i01 = -g1[3] / d1, i11 = g1[2] / d1;
  double tr = i00 * g0[2] + 2.0 * i01 * g0[3] + i11 * g0[4];
  double dx = g1[0] - g0[0], dy = g1[1] - g0[1];
  double q = i00 * dx * dx + 2.0 * i01 * dx * dy + i11 * dy * dy;
  return 0.5 * (tr + q - 2.0 + log(d1 / d0));
}

void orc_projection_quality(const float *means, const float *rots, const float *scales, int64_t n,
                            const orc_camera *cam, const orc_options *o, int32_t n_mc, uint64_t seed,
                            orc_quality *out) {
  double wmu[7], wsig[7], lam;
  orc_ut_weights(o->ut_alpha, o->ut_beta, o->ut_kappa, wmu, wsig, &lam);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < n; ++i) {
    orc_quality *q = &out[i];
    memset(q, 0, sizeof(*q));
    double mu[3] = {means[3 * i], means[3 * i + 1], means[3 * i + 2]}, R[9];
    double s[3] = {scales[3 * i], scales[3 * i + 1], scales[3 * i + 2]};
    double qq[4] = {rots[4 * i], rots[4 * i + 1], rots[4 * i + 2], rots[4 * i + 3]};
    if (orc_quat_to_rot(qq, R) != 0 || !(s[0] > 0 && s[1] > 0 && s[2] > 0)) continue;
    int ok = 1;
    /* (a) UT */
    double X[7][3], uv[7][2], t0 = 0;
    orc_sigma_points(mu, R, s, lam, X);
    for (int k = 0; k < 7 && ok; ++k) ok = orc_project_point(cam, o, X[k], uv[k], k == 0 ? &t0 : NULL, NULL, NULL);
    if (!ok) continue;
    double mx = 0, my = 0, cxx = 0, cxy = 0, cyy = 0;
    for (int k = 0; k < 7; ++k) { mx += wmu[k] * uv[k][0]; my += wmu[k] * uv[k][1]; }
    for (int k = 0; k < 7; ++k) {
      double dx = uv[k][0] - mx, dy = uv[k][1] - my;
      cxx += wsig[k] * dx * dx; cxy += wsig[k] * dx * dy; cyy += wsig[k] * dy * dy;
    }
    q->ut[0] = mx; q->ut[1] = my; q->ut[2] = cxx; q->ut[3] = cxy; q->ut[4] = cyy;
    /* (b) EWA at the pose frozen at t0 */
    double Rc[9], cc[3], d[3], xc[3], g0[2], J[2][3];
    orc_pose_at(cam, t0, Rc, cc);
    for (int a = 0; a < 3; ++a) d[a] = mu[a] - cc[a];
    mtv3(Rc, d, xc);
    ok = orc_project_cam(cam, o, xc, g0, NULL);
    const double h = 1e-6 * sqrt(dot3(xc, xc));
    for (int a = 0; a < 3 && ok; ++a) {
      double xp[3] = {xc[0], xc[1], xc[2]}, xm[3] = {xc[0], xc[1], xc[2]}, up[2], um[2];
      xp[a] += h; xm[a] -= h;
      ok = orc_project_cam(cam, o, xp, up, NULL) && orc_project_cam(cam, o, xm, um, NULL);
      J[0][a] = (up[0] - um[0]) / (2 * h);
      J[1][a] = (up[1] - um[1]) / (2 * h);
    }
    if (!ok) continue;
    /* Sigma_cam = Rc^T R S^2 R^T Rc */
    double RS[9], A[9], Sc[9];
    for (int r = 0; r < 3; ++r) for (int c2 = 0; c2 < 3; ++c2) RS[3 * r + c2] = R[3 * r + c2] * s[c2];
    for (int r = 0; r < 3; ++r) for (int c2 = 0; c2 < 3; ++c2) {
      double acc = 0; for (int k = 0; k < 3; ++k) acc += Rc[3 * k + r] * RS[3 * k + c2]; A[3 * r + c2] = acc;  /* Rc^T R S */
    }
    for (int r = 0; r < 3; ++r) for (int c2 = 0; c2 < 3; ++c2) {
      double acc = 0; for (int k = 0; k < 3; ++k) acc += A[3 * r + k] * A[3 * c2 + k]; Sc[3 * r + c2] = acc;
    }
    double JS[2][3];
    for (int r = 0; r < 2; ++r) for (int c2 = 0; c2 < 3; ++c2) {
      double acc = 0; for (int k = 0; k < 3; ++k) acc += J[r][k] * Sc[3 * k + c2]; JS[r][c2] = acc;
    }
    q->ewa[0] = g0[0]; q->ewa[1] = g0[1];
    q->ewa[2] = JS[0][0] * J[0][0] + JS[0][1] * J[0][1] + JS[0][2] * J[0][2];
    q->ewa[3] = JS[0][0] * J[1][0] + JS[0][1] * J[1][1] + JS[0][2] * J[1][2];
    q->ewa[4] = JS[1][0] * J[1][0] + JS[1][1] * J[1][1] + JS[1][2] * J[1][2];
    /* (c) Monte Carlo (sums relative to the UT mean) */
    double s1x = 0, s1y = 0, sxx = 0, sxy = 0, syy = 0;
    for (int32_t smp = 0; smp < n_mc && ok; ++smp) {
      double z[3], x[3], u2[2];
      orc_normal3(seed, i, smp, z);
      for (int a = 0; a < 3; ++a) x[a] = mu[a] + RS[3 * a] * z[0] + RS[3 * a + 1] * z[1] + RS[3 * a + 2] * z[2];
      ok = orc_project_point(cam, o, x, u2, NULL, NULL, NULL);
      double dx = u2[0] - mx, dy = u2[1] - my;
      s1x += dx; s1y += dy; sxx += dx * dx; sxy += dx * dy; syy += dy * dy;
    }
    if (!ok || n_mc < 2) continue;
    double ax = s1x / n_mc, ay = s1y / n_mc;
    q->mc[0] = mx + ax; q->mc[1] = my + ay;
    q->mc[2] = sxx / n_mc - ax * ax; q->mc[3] = sxy / n_mc - ax * ay; q->mc[4] = syy / n_mc - ay * ay;
    q->kl_ut = orc_kl2(q->mc, q->ut);
    q->kl_ewa = orc_kl2(q->mc, q->ewa);
    q->valid = 1;
  }
}
