// k1_project.cu — K1: per-Gaussian Unscented-Transform projection (sm_100a).
//
// PAPER.md Sec. 4.1 (L135-178), Alg. 1 Rasterize + Alg. 2 Estimate2DGaussian
// (L627-667): lambda, sigma points (Eq. 6), weights (Eq. 7-8), exact
// projection of every sigma point g(x) (L170) — with its own row-time pose
// under rolling shutter (L34, L393) — then the 2D mean / covariance (Eq. 9-10),
// the opacity-aware extent (Alg. 1 l.3), the rectangle (l.5), the tile count
// (StopThePop-style ellipse culling, L216), the depth key and the SH colour.
//
// One thread per Gaussian; SoA float4 loads (3 x 16 B for every Gaussian, the
// SH block only for survivors).  fp32 arithmetic except the camera-frame
// centre R0^T (mu - c0), which is formed in fp64 so that sigma-point pixels
// carry only the error of their small offsets.  Block-aggregated atomics
// produce the visible count, the key total K and the four 8-bit digit
// histograms of the depth keys consumed by the onesweep passes (K3).
#include "launch.h"

namespace gut {

// atan2(y, x) for y >= 0: octant reduction + odd minimax polynomial for atan
// on [0, 1] (fitted here; max abs error 9e-8 in fp32, ~ CUDA's atan2f, at a
// third of its instructions).  Only the fisheye projection (theta) uses it.
__device__ __forceinline__ float atan2_pos(float y, float x) {
  const float ax = fabsf(x);
  const float mx = fmaxf(y, ax), mn = fminf(y, ax);
  const float a = mx > 0.f ? mn * rs_rcp(mx) : 0.f;
  const float u = a * a;
  float p = 0.0024561970494687557f;
  p = fmaf(p, u, -0.014399108476936817f);
  p = fmaf(p, u, 0.039777275174856186f);
  p = fmaf(p, u, -0.07234489917755127f);
  p = fmaf(p, u, 0.10498751699924469f);
  p = fmaf(p, u, -0.141611710190773f);
  p = fmaf(p, u, 0.19985897839069366f);
  p = fmaf(p, u, -0.33332595229148865f);
  p = fmaf(p, u, 0.9999998807907104f);
  float t = p * a;
  if (y > ax) t = 1.5707963267948966f - t;
  if (x < 0.f) t = 3.141592653589793f - t;
  return t;
}

// MODEL: the camera model as a compile-time constant (-1: read from c at run
// time).  MUFU reciprocal / square root (relative error ~2^-22, like the
// other fp32 roundings here far inside the 1e-3 px binning band).
template <int MODEL = -1>
__device__ __forceinline__ bool project_cam_f(const DevCam &c, f3 x, float &du, float &dv) {
  // returns pixel offsets from the principal point (du, dv); validity first
  switch (MODEL >= 0 ? MODEL : c.model) {
    case CAM_PINHOLE: {
      if (!(x.z > c.near_plane)) return false;
      const float rz = rs_rcp(x.z);
      du = c.fxf * (x.x * rz);
      dv = c.fyf * (x.y * rz);
      return true;
    }
    case CAM_ORTHO: {
      if (!(x.z > c.near_plane)) return false;
      du = c.fxf * x.x;
      dv = c.fyf * x.y;
      return true;
    }
    case CAM_OPENCV: {
      if (!(x.z > c.near_plane)) return false;
      const float rz = rs_rcp(x.z);
      float xn = x.x * rz, yn = x.y * rz, r2 = xn * xn + yn * yn;
      if (c.fovf > 0.f && !(r2 <= c.fovf * c.fovf)) return false;
      float num = 1.f + r2 * (c.kf[0] + r2 * (c.kf[1] + r2 * c.kf[2]));
      float den = 1.f + r2 * (c.kf[3] + r2 * (c.kf[4] + r2 * c.kf[5]));
      float a = num * rs_rcp(den);
      float xd = xn * a + 2.f * c.pf[0] * xn * yn + c.pf[1] * (r2 + 2.f * xn * xn);
      float yd = yn * a + c.pf[0] * (r2 + 2.f * yn * yn) + 2.f * c.pf[1] * xn * yn;
      du = c.fxf * xd;
      dv = c.fyf * yd;
      return true;
    }
    case CAM_FISHEYE: {
      const float rho2 = x.x * x.x + x.y * x.y;
      // |x| > near, squared (near * |near| keeps a negative near always true)
      if (!(rho2 + x.z * x.z > c.near_plane * fabsf(c.near_plane))) return false;
      const float rho = rs_sqrt(rho2);
      const float th = atan2_pos(rho, x.z);
      if (!(th <= c.fovf)) return false;
      if (rho == 0.f) { du = 0.f; dv = 0.f; return true; }
      float t2 = th * th;
      float td = th * (1.f + t2 * (c.kf[0] + t2 * (c.kf[1] + t2 * (c.kf[2] + t2 * c.kf[3]))));
      float s = td * rs_rcp(rho);
      du = c.fxf * (s * x.x);
      dv = c.fyf * (s * x.y);
      return true;
    }
  }
  return false;
}

__device__ __forceinline__ float shutter_coord(const DevCam &c, float du, float dv) {
  float r;
  switch (c.shutter) {
    case SH_T2B: r = (dv + c.cyf) * c.inv_hf; break;
    case SH_B2T: r = 1.f - (dv + c.cyf) * c.inv_hf; break;
    case SH_L2R: r = (du + c.cxf) * c.inv_wf; break;
    case SH_R2L: r = 1.f - (du + c.cxf) * c.inv_wf; break;
    default: return 0.f;
  }
  return fminf(fmaxf(r, 0.f), 1.f);
}

// camera-frame point at shutter time t: x_c(t) = R(t)^T (x - c(t)) with
// R(t) = R0 Exp(t phi), c(t) = c0 + t dc  =>  Exp(t phi)^T (y - t w),
// y = R0^T (x - c0), w = R0^T dc.
__device__ __forceinline__ f3 cam_point_at(const DevCam &c, f3 y, f3 w, float t) {
  float Rt[9];
  rodrigues(mk(c.phi_axisf[0], c.phi_axisf[1], c.phi_axisf[2]), t * c.phi_anglef, Rt);
  return mtv(Rt, y - t * w);
}

// g(x) with the sigma point's own extrinsic (reading R14): the shutter time is
// the fixed point t* = clamp(rho(g(x; pose(t*)))), solved by secant steps from
// (0.5, rho(g(x; pose(0.5)))) until the pixel moves < rs_tol_px.
// (one out-of-line copy: the seven inlined secant loops of a Gaussian overflow
// the instruction cache -- ncu: 40% "no instruction" stalls in rolling shutter)
template <int MODEL>
__device__ __noinline__ bool project_sigma_rs(const DevCam &c, f3 y, f3 w, float &du, float &dv, float &t_out);
// RS: the rolling-shutter instantiation of K1 (project_kernel<DEG, true>); the
// global-shutter one never contains the shutter solve
template <bool RS, int MODEL>
__device__ __forceinline__ bool project_sigma(const DevCam &c, f3 y, f3 w, float &du, float &dv,
                                              float &t_out) {
  if (!RS || c.shutter == SH_GLOBAL) {
    t_out = 0.f;
    return project_cam_f<MODEL>(c, y, du, dv);
  }
  return project_sigma_rs<MODEL>(c, y, w, du, dv, t_out);
}
template <int MODEL>
__device__ __noinline__ bool project_sigma_rs(const DevCam &c, f3 y, f3 w, float &du, float &dv, float &t_out) {
  float t0 = 0.5f, u0, v0;
  if (!project_cam_f<MODEL>(c, cam_point_at(c, y, w, t0), u0, v0)) return false;
  float f0 = shutter_coord(c, u0, v0) - t0;
  float t1 = t0 + f0, u1, v1;
  if (!project_cam_f<MODEL>(c, cam_point_at(c, y, w, t1), u1, v1)) return false;
  float f1 = shutter_coord(c, u1, v1) - t1;
  // stop when the pixel moved less than the tolerance -- or than fp32 can
  // resolve at this pixel position (4 ulps), beyond which steps are noise -- or
  // when the time no longer changes
  const float tol2 = c.rs_tol_px * c.rs_tol_px;
  for (int it = 0; it < c.rs_max_iter; ++it) {
    const float ddu = u1 - u0, ddv = v1 - v0, ulp4 = 4.8e-7f * (fabsf(u1) + fabsf(v1));
    if (ddu * ddu + ddv * ddv < fmaxf(tol2, ulp4 * ulp4) || t1 == t0) break;
    float den = f1 - f0;
    float t2 = fabsf(den) > 1e-12f ? t1 - f1 * (t1 - t0) * __frcp_rn(den) : t1 + f1;
    t2 = fminf(fmaxf(t2, 0.f), 1.f);
    t0 = t1; u0 = u1; v0 = v1; f0 = f1; t1 = t2;
    if (!project_cam_f<MODEL>(c, cam_point_at(c, y, w, t1), u1, v1)) return false;
    f1 = shutter_coord(c, u1, v1) - t1;
  }
  du = u1; dv = v1; t_out = t1;
  return true;
}

// ---- fp64 twin of the projection for Gaussians whose sigma points land far
// from the principal point: fp32 pixel coordinates carry ~eps*|v| absolute
// error, which above ~2048 px would exceed half the 1e-3 px binning band.
__device__ bool project_cam_d(const DevCam &c, d3 x, double &du, double &dv) {
  switch (c.model) {
    case CAM_PINHOLE:
      if (!(x.z > (double)c.near_plane)) return false;
      du = c.fx * (x.x / x.z); dv = c.fy * (x.y / x.z);
      return true;
    case CAM_ORTHO:
      if (!(x.z > (double)c.near_plane)) return false;
      du = c.fx * x.x; dv = c.fy * x.y;
      return true;
    case CAM_OPENCV: {
      if (!(x.z > (double)c.near_plane)) return false;
      double xn = x.x / x.z, yn = x.y / x.z, r2 = xn * xn + yn * yn;
      if (c.fov > 0 && !(r2 <= c.fov * c.fov)) return false;
      double num = 1 + r2 * (c.k[0] + r2 * (c.k[1] + r2 * c.k[2]));
      double den = 1 + r2 * (c.k[3] + r2 * (c.k[4] + r2 * c.k[5]));
      double a = num / den;
      double xd = xn * a + 2 * c.p[0] * xn * yn + c.p[1] * (r2 + 2 * xn * xn);
      double yd = yn * a + c.p[0] * (r2 + 2 * yn * yn) + 2 * c.p[1] * xn * yn;
      du = c.fx * xd; dv = c.fy * yd;
      return true;
    }
    case CAM_FISHEYE: {
      double nrm = sqrt(x.x * x.x + x.y * x.y + x.z * x.z);
      if (!(nrm > (double)c.near_plane)) return false;
      double rho = sqrt(x.x * x.x + x.y * x.y);
      double th = atan2(rho, x.z);
      if (!(th <= (double)c.fovf)) return false;  // same threshold value as the fp32 path
      if (rho == 0) { du = 0; dv = 0; return true; }
      double t2 = th * th;
      double td = th * (1 + t2 * (c.k[0] + t2 * (c.k[1] + t2 * (c.k[2] + t2 * c.k[3]))));
      du = c.fx * (td * x.x / rho); dv = c.fy * (td * x.y / rho);
      return true;
    }
  }
  return false;
}

__device__ __forceinline__ double shutter_coord_d(const DevCam &c, double du, double dv) {
  double r;
  switch (c.shutter) {
    case SH_T2B: r = (dv + c.cy) / c.height; break;
    case SH_B2T: r = 1.0 - (dv + c.cy) / c.height; break;
    case SH_L2R: r = (du + c.cx) / c.width; break;
    case SH_R2L: r = 1.0 - (du + c.cx) / c.width; break;
    default: return 0.0;
  }
  return fmin(fmax(r, 0.0), 1.0);
}

__device__ bool project_sigma_d(const DevCam &c, d3 y, d3 w, double &du, double &dv, double &t_out) {
  t_out = 0.0;
  if (c.shutter == SH_GLOBAL) return project_cam_d(c, y, du, dv);
  const d3 ax = mkd(c.phi_axis[0], c.phi_axis[1], c.phi_axis[2]);
  auto at = [&](double t) {
    double Rt[9];
    rodrigues_d(ax, t * c.phi_angle, Rt);
    return mtv(Rt, y - t * w);
  };
  double t0 = 0.5, u0, v0;
  if (!project_cam_d(c, at(t0), u0, v0)) return false;
  double f0 = shutter_coord_d(c, u0, v0) - t0;
  double t1 = t0 + f0, u1, v1;
  if (!project_cam_d(c, at(t1), u1, v1)) return false;
  double f1 = shutter_coord_d(c, u1, v1) - t1;
  for (int it = 0; it < c.rs_max_iter; ++it) {
    if (hypot(u1 - u0, v1 - v0) < (double)c.rs_tol_px) break;
    double den = f1 - f0;
    double t2 = fabs(den) > 1e-15 ? t1 - f1 * (t1 - t0) / den : t1 + f1;
    t2 = fmin(fmax(t2, 0.0), 1.0);
    t0 = t1; u0 = u1; v0 = v1; f0 = f1; t1 = t2;
    if (!project_cam_d(c, at(t1), u1, v1)) return false;
    f1 = shutter_coord_d(c, u1, v1) - t1;
  }
  du = u1; dv = v1; t_out = t1;
  return true;
}

// 3DGS real SH basis up to degree DEG (reading R19), colour = max(sum + 0.5, 0)
template <int DEG>
__device__ __forceinline__ f3 sh_colour(const float4 *sh, int64_t n, int64_t i, f3 d) {
  constexpr int NC = (DEG + 1) * (DEG + 1);
  constexpr int CH = (3 * NC + 3) / 4;
  float f[CH * 4];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    float4 v = __ldg(&sh[(int64_t)c * n + i]);
    f[4 * c] = v.x; f[4 * c + 1] = v.y; f[4 * c + 2] = v.z; f[4 * c + 3] = v.w;
  }
  float Y[16];
  float x = d.x, y = d.y, z = d.z, xx = x * x, yy = y * y, zz = z * z;
  Y[0] = 0.28209479177387814f;
  if (DEG >= 1) { Y[1] = -0.4886025119029199f * y; Y[2] = 0.4886025119029199f * z; Y[3] = -0.4886025119029199f * x; }
  if (DEG >= 2) {
    Y[4] = 1.0925484305920792f * x * y; Y[5] = -1.0925484305920792f * y * z;
    Y[6] = 0.31539156525252005f * (2.f * zz - xx - yy); Y[7] = -1.0925484305920792f * x * z;
    Y[8] = 0.5462742152960396f * (xx - yy);
  }
  if (DEG >= 3) {
    Y[9] = -0.5900435899266435f * y * (3.f * xx - yy); Y[10] = 2.890611442640554f * x * y * z;
    Y[11] = -0.4570457994644658f * y * (4.f * zz - xx - yy);
    Y[12] = 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
    Y[13] = -0.4570457994644658f * x * (4.f * zz - xx - yy); Y[14] = 1.445305721320277f * z * (xx - yy);
    Y[15] = -0.5900435899266435f * x * (xx - 3.f * yy);
  }
  float r = 0.5f, g = 0.5f, b = 0.5f;
#pragma unroll
  for (int k = 0; k < NC; ++k) { r += Y[k] * f[3 * k]; g += Y[k] * f[3 * k + 1]; b += Y[k] * f[3 * k + 2]; }
  return mk(fmaxf(r, 0.f), fmaxf(g, 0.f), fmaxf(b, 0.f));
}

// ---- shared tail of both K1 kernels: depth key, SH colour, blend payload,
// packed ellipse record.  Returns the depth key.
template <int DEG>
__device__ __forceinline__ uint32_t finish_gaussian(const DevCam &c, const SceneDev &s, int64_t i, float4 po,
                                                    float4 sc, const float *R, double t0, float4 e0,
                                                    float4 e1, float4 *__restrict__ ell,
                                                    float4 *__restrict__ payload) {
  // depth key (reading R13): camera-frame distance of mu at its own time t0,
  // |R(t0)^T (mu - c(t0))| = |mu - c(t0)| (fp64, then the fp32 key)
  const d3 dw = mkd(po.x, po.y, po.z) - mkd(c.c0[0], c.c0[1], c.c0[2]) -
                (c.shutter == SH_GLOBAL ? mkd(0, 0, 0) : t0 * mkd(c.dc[0], c.dc[1], c.dc[2]));
  const double nd2 = dot(dw, dw);
  const float depth = (float)sqrt(nd2);
  // colour (reading R18): SH at d = normalize(mu - c(t0)) (the difference in
  // fp64, the normalisation in fp32: ~1e-7 relative in the direction)
  const f3 dwf = tof(dw);
  const f3 rgb = sh_colour<DEG>(s.sh, s.n, i, rsqrtf(dot(dwf, dwf)) * dwf);
  ell[2 * i] = e0;
  ell[2 * i + 1] = e1;
  // blend payload (80 B): w0 = c(0) - mu in fp64 (K5 forms the cancelling
  // o_g x d_g = cof(M) (w x d) from it, see k5_blend.cu), k^2 = 2 ln(sigma /
  // alpha_min) (the ellipse record's value; K5 derives log2 sigma from it),
  // M = diag(1/s) R^T (Eq. 11 o_g = M (o - mu)), rgb
  const float is0 = rs_rcp(sc.x), is1 = rs_rcp(sc.y), is2 = rs_rcp(sc.z);  // (MUFU, ~2^-22 relative)
  const d3 w0 = mkd(c.c0[0], c.c0[1], c.c0[2]) - mkd(po.x, po.y, po.z);
  const unsigned long long wz = (unsigned long long)__double_as_longlong(w0.z);
  float4 *pl = payload + (size_t)GUT_PAYLOAD_F4 * i;
  reinterpret_cast<double2 *>(pl)[0] = make_double2(w0.x, w0.y);
  pl[1] = make_float4(__int_as_float((int)(uint32_t)wz), __int_as_float((int)(uint32_t)(wz >> 32)), fabsf(e1.y),
                      R[0] * is0);
  pl[2] = make_float4(R[3] * is0, R[6] * is0, R[1] * is1, R[4] * is1);
  pl[3] = make_float4(R[7] * is1, R[2] * is2, R[5] * is2, R[8] * is2);
  pl[4] = make_float4(rgb.x, rgb.y, rgb.z, c.kdeg != 2 ? log2f(po.w) : 0.f);  // log2 sigma: K5's alpha for degree != 2
  return __float_as_uint(depth);
}

// Opacity-aware extent level (Alg. 1 l.3): alpha >= alpha_min <=>
// omega^2 <= k2, k2 = 2 ln(sigma / alpha_min) (via log1p: accurate when sigma is
// near alpha_min); generalized kernel of degree n (Supp. A, reading R29):
// (1/2) lambda_n omega^n <= ln(sigma / alpha_min) -> k2 = (k2_2 / lambda_n)^(2/n)
__device__ __forceinline__ float extent_level(const DevCam &c, float sigma) {
  const float k2 = 2.f * log1pf((sigma - c.alpha_min) / c.alpha_min);
  return c.kdeg == 2 ? k2 : powf(k2 / c.klam, 2.f / (float)c.kdeg);
}

__device__ __forceinline__ bool load_gaussian(const DevCam &c, const SceneDev &s, int64_t i, float4 &po, float4 &sc,
                                              float *R) {
  po = __ldg(&s.pos_opa[i]);
  const float4 ro = __ldg(&s.rot[i]);
  sc = __ldg(&s.scale[i]);
  const float qn2 = ro.x * ro.x + ro.y * ro.y + ro.z * ro.z + ro.w * ro.w;
  const bool ok = isfinite(po.x) && isfinite(po.y) && isfinite(po.z) && isfinite(qn2) && qn2 > 0.f &&
                  sc.x > 0.f && sc.y > 0.f && sc.z > 0.f && isfinite(sc.x) && isfinite(sc.y) &&
                  isfinite(sc.z) && po.w > c.alpha_min && isfinite(po.w);
  if (!ok) return false;
  // O1: R(q) from the normalised quaternion (w,x,y,z), Eq. 2
  const float inv = 1.f / sqrtf(qn2);
  const float w = ro.x * inv, x = ro.y * inv, y = ro.z * inv, z = ro.w * inv;
  R[0] = 1.f - 2.f * (y * y + z * z); R[1] = 2.f * (x * y - w * z); R[2] = 2.f * (x * z + w * y);
  R[3] = 2.f * (x * y + w * z); R[4] = 1.f - 2.f * (x * x + z * z); R[5] = 2.f * (y * z - w * x);
  R[6] = 2.f * (x * z - w * y); R[7] = 2.f * (y * z + w * x); R[8] = 1.f - 2.f * (x * x + y * y);
  return true;
}

__device__ __forceinline__ uint32_t pack_rect(int x, int y) { return (uint32_t)x | ((uint32_t)y << 16); }

// block-aggregated visible count, key total and depth-digit histograms
__device__ __forceinline__ void k1_block_totals(uint32_t my_tiles, uint32_t key, uint32_t (*s_hist)[256],
                                                unsigned long long *s_k, uint32_t *s_nv, uint32_t *counters) {
  if (my_tiles) {
    atomicAdd(&s_hist[0][key & 255u], 1u);
    atomicAdd(&s_hist[1][(key >> 8) & 255u], 1u);
    atomicAdd(&s_hist[2][(key >> 16) & 255u], 1u);
    atomicAdd(&s_hist[3][key >> 24], 1u);
  }
  unsigned long long kk = my_tiles;
  uint32_t nv = my_tiles ? 1u : 0u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kk += __shfl_xor_sync(0xffffffffu, kk, o);
    nv += __shfl_xor_sync(0xffffffffu, nv, o);
  }
  if ((threadIdx.x & 31) == 0) { s_k[threadIdx.x >> 5] = kk; s_nv[threadIdx.x >> 5] = nv; }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long K = 0;
    uint32_t V = 0;
    for (int w = 0; w < 8; ++w) { K += s_k[w]; V += s_nv[w]; }
    if (V) {
      atomicAdd(&counters[CNT_NVIS], V);
      atomicAdd(reinterpret_cast<unsigned long long *>(&counters[CNT_K]), K);
    }
  }
  for (int j = threadIdx.x; j < 1024; j += 256) {
    const uint32_t v = (&s_hist[0][0])[j];
    if (v) atomicAdd(&counters[CNT_HIST_DEPTH + j], v);
  }
}

// ---- K1 main (fp32): one thread per Gaussian
template <int DEG, bool LIST, int MODEL>
#ifndef GUT_K1_CTAS
#define GUT_K1_CTAS 4  // 64 registers: 32 warps per SM (measured best)
#endif
__global__ __launch_bounds__(256, GUT_K1_CTAS) void project_kernel(DevCam c, SceneDev s, uint32_t *__restrict__ dkey,
                                                         uint32_t *__restrict__ tiles, float4 *__restrict__ ell,
                                                         float4 *__restrict__ payload, uint32_t *counters,
                                                         uint32_t *__restrict__ deferred,
                                                         const uint32_t *__restrict__ list) {
  __shared__ uint32_t s_hist[4][256];
  __shared__ unsigned long long s_k[8];
  __shared__ uint32_t s_nv[8];
  // LIST: the Gaussians the pre-filter kept (counters[CNT_K1LIST] of them)
  const int64_t n_items = LIST ? (int64_t)counters[CNT_K1LIST] : s.n;
  if (LIST && (int64_t)blockIdx.x * 256 >= n_items) return;  // (whole block past the list: uniform)
  for (int j = threadIdx.x; j < 1024; j += 256) (&s_hist[0][0])[j] = 0;
  __syncthreads();
  const int64_t idx = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t i = LIST ? (idx < n_items ? (int64_t)list[idx] : s.n) : idx;
  uint32_t my_code = 0, key = GUT_CULLED_KEY;  // my_code: tile code (gut_internal.cuh)
  if (i < s.n) {
    float4 po, sc;
    float R[9];
    bool ok = load_gaussian(c, s, i, po, sc, R);
    bool wide = false;
    float du[7], dv[7], tt[7];
    d3 y0d = mkd(0, 0, 0);
    if (ok) {
      // camera-frame centre in fp64, sigma offsets gamma s_j R[:,j] rotated in fp32 (Eq. 6)
      y0d = mtv(c.R0, mkd(po.x, po.y, po.z) - mkd(c.c0[0], c.c0[1], c.c0[2]));
      const f3 y0 = tof(y0d);
      const f3 wv = mtv(c.R0f, mk(c.dcf[0], c.dcf[1], c.dcf[2]));
      const float sj[3] = {sc.x, sc.y, sc.z};
      ok = project_sigma<LIST, MODEL>(c, y0, wv, du[0], dv[0], tt[0]);
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const f3 L = (c.gamma * sj[j]) * mk(R[j], R[3 + j], R[6 + j]);
        const f3 Lc = mtv(c.R0f, L);
        ok = ok && project_sigma<LIST, MODEL>(c, y0 + Lc, wv, du[1 + j], dv[1 + j], tt[1 + j]);
        ok = ok && project_sigma<LIST, MODEL>(c, y0 - Lc, wv, du[4 + j], dv[4 + j], tt[4 + j]);
      }
    }
    float vx = 0, vy = 0, cxx = 0, cxy = 0, cyy = 0, k2 = 0;
    if (ok) {
      float mag = 0.f;
#pragma unroll
      for (int k = 0; k < 7; ++k) mag = fmaxf(mag, fmaxf(fabsf(du[k]), fabsf(dv[k])));
      if (mag > 2048.f) {  // far sigma points: redo this Gaussian in fp64 (project_wide_kernel)
        wide = true;
        ok = false;
      }
    }
    if (ok) {
      // Eq. 9-10, then + dilation (reading R10)
      vx = c.wmu0 * du[0] + c.wmui * (((du[1] + du[4]) + (du[2] + du[5])) + (du[3] + du[6]));
      vy = c.wmu0 * dv[0] + c.wmui * (((dv[1] + dv[4]) + (dv[2] + dv[5])) + (dv[3] + dv[6]));
      const float ex = du[0] - vx, ey = dv[0] - vy;
      cxx = c.wsig0 * ex * ex; cxy = c.wsig0 * ex * ey; cyy = c.wsig0 * ey * ey;
      float sxx = 0, sxy = 0, syy = 0;
#pragma unroll
      for (int k = 1; k < 7; ++k) {
        const float ax = du[k] - vx, ay = dv[k] - vy;
        sxx += ax * ax; sxy += ax * ay; syy += ay * ay;
      }
      cxx += c.wsigi * sxx + c.dilation;
      cxy += c.wsigi * sxy;
      cyy += c.wsigi * syy + c.dilation;
      const float det = cxx * cyy - cxy * cxy;
      ok = cxx > 0.f && cyy > 0.f && det > 0.f && isfinite(det);
      // opacity-aware extent level (Alg. 1 l.3, reading R11)
      // k2 = 2 ln(sigma/alpha_min) via log1p: accurate when sigma is near alpha_min
      k2 = extent_level(c, po.w);
      ok = ok && k2 > 0.f;
    }
    Ell e;
    if (ok) {
      const float hx = sqrtf(k2 * cxx), hy = sqrtf(k2 * cyy);
      e.vx = vx + c.cxf; e.vy = vy + c.cyf;
      e.cxx = cxx; e.cxy = cxy; e.cyy = cyy; e.k2 = k2;
      const float fx0 = floorf(fminf(fmaxf((e.vx - hx) * (1.f / GUT_TILE), -1e6f), 1e6f));
      const float fx1 = floorf(fminf(fmaxf((e.vx + hx) * (1.f / GUT_TILE), -1e6f), 1e6f));
      const float fy0 = floorf(fminf(fmaxf((e.vy - hy) * (1.f / GUT_TILE), -1e6f), 1e6f));
      const float fy1 = floorf(fminf(fmaxf((e.vy + hy) * (1.f / GUT_TILE), -1e6f), 1e6f));
      e.x0 = max((int)fx0, 0); e.x1 = min((int)fx1, c.tiles_x - 1);
      e.y0 = max((int)fy0, 0); e.y1 = min((int)fy1, c.tiles_y - 1);
      ok = e.x0 <= e.x1 && e.y0 <= e.y1;
      if (ok) {
        my_code = ell_tile_code(e, c.tile_cull);
        ok = my_code != 0;
      }
    }
    if (ok) {
      key = finish_gaussian<DEG>(c, s, i, po, sc, R, (double)tt[0],
                                 make_float4(e.vx, e.vy, e.cxx, e.cxy),
                                 make_float4(e.cyy, e.k2, __uint_as_float(pack_rect(e.x0, e.y0)),
                                             __uint_as_float(pack_rect(e.x1, e.y1))),
                                 ell, payload);
    } else {
      my_code = 0;
      key = GUT_CULLED_KEY;
    }
    dkey[i] = key;
    tiles[i] = my_code;
    if (wide) deferred[atomicAdd(&counters[CNT_NDEFER], 1u)] = (uint32_t)i;
  }
  k1_block_totals(code_count(my_code), key, s_hist, s_k, s_nv, counters);
}

// ---- K1 wide (fp64 UT + fp64 ellipse) for the deferred Gaussians.  The packed
// record stores -k2 as a flag; K2 then reads the fp64 ellipse from ell64.
template <int DEG>
__global__ __launch_bounds__(256) void project_wide_kernel(DevCam c, SceneDev s, uint32_t *__restrict__ dkey,
                                                           uint32_t *__restrict__ tiles, float4 *__restrict__ ell,
                                                           double2 *__restrict__ ell64,
                                                           float4 *__restrict__ payload, uint32_t *counters,
                                                           const uint32_t *__restrict__ deferred) {
  __shared__ uint32_t s_hist[4][256];
  __shared__ unsigned long long s_k[8];
  __shared__ uint32_t s_nv[8];
  const uint32_t nd = counters[CNT_NDEFER];
  for (uint32_t base = blockIdx.x * 256; base < nd; base += gridDim.x * 256) {
    __syncthreads();
    for (int j = threadIdx.x; j < 1024; j += 256) (&s_hist[0][0])[j] = 0;
    __syncthreads();
    uint32_t my_code = 0, key = GUT_CULLED_KEY;  // my_code: tile code (gut_internal.cuh)
    const uint32_t q = base + threadIdx.x;
    if (q < nd) {
      const int64_t i = deferred[q];
      float4 po, sc;
      float R[9];
      bool ok = load_gaussian(c, s, i, po, sc, R);
      const d3 y0d = mtv(c.R0, mkd(po.x, po.y, po.z) - mkd(c.c0[0], c.c0[1], c.c0[2]));
      const d3 w = mtv(c.R0, mkd(c.dc[0], c.dc[1], c.dc[2]));
      const double sj[3] = {sc.x, sc.y, sc.z};
      double du[7], dv[7], t0 = 0, tdummy;
      ok = ok && project_sigma_d(c, y0d, w, du[0], dv[0], t0);
      for (int j = 0; j < 3 && ok; ++j) {
        const d3 Lc = mtv(c.R0, ((double)c.gamma * sj[j]) * mkd(R[j], R[3 + j], R[6 + j]));
        ok = ok && project_sigma_d(c, y0d + Lc, w, du[1 + j], dv[1 + j], tdummy);
        ok = ok && project_sigma_d(c, y0d - Lc, w, du[4 + j], dv[4 + j], tdummy);
      }
      EllD e;
      if (ok) {
        double mx = (double)c.wmu0 * du[0], my = (double)c.wmu0 * dv[0];
        for (int k = 1; k < 7; ++k) { mx += (double)c.wmui * du[k]; my += (double)c.wmui * dv[k]; }
        double sxx = 0, sxy = 0, syy = 0;
        for (int k = 0; k < 7; ++k) {
          const double wk = k == 0 ? (double)c.wsig0 : (double)c.wsigi;
          const double ax = du[k] - mx, ay = dv[k] - my;
          sxx += wk * ax * ax; sxy += wk * ax * ay; syy += wk * ay * ay;
        }
        e.cxx = sxx + c.dilation; e.cxy = sxy; e.cyy = syy + c.dilation;
        const double det = e.cxx * e.cyy - e.cxy * e.cxy;
        const float k2f = extent_level(c, po.w);  // same value as the fp32 path / K5
        e.k2 = k2f;
        ok = e.cxx > 0 && e.cyy > 0 && det > 0 && isfinite(det) && k2f > 0.f;
        if (ok) {
          e.vx = mx + c.cx; e.vy = my + c.cy;
          const double hx = sqrt(e.k2 * e.cxx), hy = sqrt(e.k2 * e.cyy);
          const double fx0 = floor(fmin(fmax((e.vx - hx) / GUT_TILE, -1e9), 1e9));
          const double fx1 = floor(fmin(fmax((e.vx + hx) / GUT_TILE, -1e9), 1e9));
          const double fy0 = floor(fmin(fmax((e.vy - hy) / GUT_TILE, -1e9), 1e9));
          const double fy1 = floor(fmin(fmax((e.vy + hy) / GUT_TILE, -1e9), 1e9));
          e.x0 = (int)fmax(fx0, 0.0); e.x1 = (int)fmin(fx1, (double)(c.tiles_x - 1));
          e.y0 = (int)fmax(fy0, 0.0); e.y1 = (int)fmin(fy1, (double)(c.tiles_y - 1));
          ok = e.x0 <= e.x1 && e.y0 <= e.y1;
          if (ok) {
            my_code = ell_tile_code(e, c.tile_cull);
            ok = my_code != 0;
          }
        }
      }
      if (ok) {
        ell64[3 * i] = make_double2(e.vx, e.vy);
        ell64[3 * i + 1] = make_double2(e.cxx, e.cxy);
        ell64[3 * i + 2] = make_double2(e.cyy, e.k2);
        key = finish_gaussian<DEG>(c, s, i, po, sc, R, t0,
                                   make_float4((float)e.vx, (float)e.vy, (float)e.cxx, (float)e.cxy),
                                   make_float4((float)e.cyy, -(float)e.k2, __uint_as_float(pack_rect(e.x0, e.y0)),
                                               __uint_as_float(pack_rect(e.x1, e.y1))),
                                   ell, payload);
      } else {
        my_code = 0;
        key = GUT_CULLED_KEY;
      }
      dkey[i] = key;
      tiles[i] = my_code;
    }
    k1_block_totals(code_count(my_code), key, s_hist, s_k, s_nv, counters);
  }
}

__global__ void pack_scene_kernel(const float *__restrict__ means, const float *__restrict__ rots,
                                  const float *__restrict__ scales, const float *__restrict__ opac,
                                  const float *__restrict__ sh, SceneDev s) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= s.n) return;
  s.pos_opa[i] = make_float4(means[3 * i], means[3 * i + 1], means[3 * i + 2], opac[i]);
  s.rot[i] = make_float4(rots[4 * i], rots[4 * i + 1], rots[4 * i + 2], rots[4 * i + 3]);
  s.scale[i] = make_float4(scales[3 * i], scales[3 * i + 1], scales[3 * i + 2], 0.f);
  int nf = 3 * (s.sh_degree + 1) * (s.sh_degree + 1);
  const float *src = sh + (int64_t)nf * i;
  for (int c = 0; c < s.sh_chunks; ++c) {
    float v[4];
    for (int j = 0; j < 4; ++j) v[j] = (4 * c + j < nf) ? src[4 * c + j] : 0.f;
    s.sh[(int64_t)c * s.n + i] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

void launch_pack_scene(const float *means, const float *rots, const float *scales, const float *opac,
                       const float *sh, SceneDev s, cudaStream_t st) {
  if (s.n == 0) return;
  int64_t blocks = (s.n + 255) / 256;
  pack_scene_kernel<<<(unsigned)blocks, 256, 0, st>>>(means, rots, scales, opac, sh, s);
}


// Rolling shutter: a cheap, conservative pre-filter so that the expensive
// per-sigma-point shutter-time solves run on dense warps (street scenes cull
// ~3/4 of the Gaussians per camera; without it warps average ~7 active lanes).
// A Gaussian is dropped only if its CENTRE sigma point is invalid at every
// shutter time t in [0, 1] -- and then the full K1 culls it too (reading R9:
// any invalid sigma point culls).  Over t the camera-frame centre stays in the
// ball |x_c(t) - y| <= |dc| + |phi| |y| around y = R0^T (mu - c0); the tests
// below hold for every point of that ball (plus an fp32 slack): behind the near
// plane; OpenCV outside the validity radius r_lim; fisheye beyond theta_max or
// inside the near sphere.  Culled Gaussians get K1's culled outputs; the rest
// are appended to a list (warp-aggregated) for project_kernel.
__global__ __launch_bounds__(256) void project_prefilter_kernel(DevCam c, SceneDev s, uint32_t *__restrict__ dkey,
                                                                uint32_t *__restrict__ tiles, uint32_t *counters,
                                                                uint32_t *__restrict__ list) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  bool keep = false;
  if (i < s.n) {
    const float4 po = __ldg(&s.pos_opa[i]);
    keep = true;
    if (isfinite(po.x) && isfinite(po.y) && isfinite(po.z)) {
      const f3 y = mtv(c.R0f, mk((float)((double)po.x - c.c0[0]), (float)((double)po.y - c.c0[1]),
                                 (float)((double)po.z - c.c0[2])));
      const float ny = sqrtf(dot(y, y));
      const float dcn = sqrtf(c.dcf[0] * c.dcf[0] + c.dcf[1] * c.dcf[1] + c.dcf[2] * c.dcf[2]);
      const float dl = dcn + fabsf(c.phi_anglef) * ny + 1e-4f * ny + 1e-4f;  // ball radius + fp32 slack
      const float rho = sqrtf(y.x * y.x + y.y * y.y);
      if (c.model == CAM_PINHOLE || c.model == CAM_OPENCV) {
        if (y.z + dl < c.near_plane) keep = false;
        else if (c.model == CAM_OPENCV && c.fovf > 0.f && rho - dl > 0.f && rho - dl > c.fovf * (y.z + dl))
          keep = false;
      } else if (c.model == CAM_FISHEYE) {
        if (ny + dl < c.near_plane) keep = false;
        else if (ny > 2.f * dl) {
          // angle of y to the axis minus the ball's angular radius (asin(dl/|y|) <= 2 dl/|y| here)
          const float th = atan2f(rho, y.z) - 2.f * dl / ny;
          if (th > c.fovf + 1e-5f) keep = false;
        }
      }
    }
    if (!keep) {
      dkey[i] = GUT_CULLED_KEY;
      tiles[i] = 0u;
    }
  }
  const uint32_t bal = __ballot_sync(0xffffffffu, keep);
  const int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == 0 && bal) base = atomicAdd(&counters[CNT_K1LIST], (uint32_t)__popc(bal));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (keep) list[base + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)i;
}

// one SH degree: K1 instantiated per camera model and shutter (the rolling-
// shutter one over the pre-filter's compacted list)
template <int DEG>
static void launch_k1_deg(const DevCam &cam, const SceneDev &s, uint32_t *dkey, uint32_t *tiles, float4 *ell,
                          double2 *ell64, float4 *payload, uint32_t *counters, uint32_t *deferred, uint32_t *list,
                          unsigned blocks, unsigned wblocks, cudaStream_t st) {
  if (list) {  // rolling shutter (compacted list); ortho never takes the pre-filter path
    switch (cam.model) {
      case CAM_PINHOLE:
        project_kernel<DEG, true, CAM_PINHOLE><<<blocks, 256, 0, st>>>(cam, s, dkey, tiles, ell, payload, counters, deferred, list);
        break;
      case CAM_OPENCV:
        project_kernel<DEG, true, CAM_OPENCV><<<blocks, 256, 0, st>>>(cam, s, dkey, tiles, ell, payload, counters, deferred, list);
        break;
      default:
        project_kernel<DEG, true, CAM_FISHEYE><<<blocks, 256, 0, st>>>(cam, s, dkey, tiles, ell, payload, counters, deferred, list);
        break;
    }
  } else {
    switch (cam.model) {
      case CAM_PINHOLE:
        project_kernel<DEG, false, CAM_PINHOLE><<<blocks, 256, 0, st>>>(cam, s, dkey, tiles, ell, payload, counters, deferred, list);
        break;
      case CAM_OPENCV:
        project_kernel<DEG, false, CAM_OPENCV><<<blocks, 256, 0, st>>>(cam, s, dkey, tiles, ell, payload, counters, deferred, list);
        break;
      case CAM_FISHEYE:
        project_kernel<DEG, false, CAM_FISHEYE><<<blocks, 256, 0, st>>>(cam, s, dkey, tiles, ell, payload, counters, deferred, list);
        break;
      default:
        project_kernel<DEG, false, CAM_ORTHO><<<blocks, 256, 0, st>>>(cam, s, dkey, tiles, ell, payload, counters, deferred, list);
        break;
    }
  }
  project_wide_kernel<DEG><<<wblocks, 256, 0, st>>>(cam, s, dkey, tiles, ell, ell64, payload, counters, deferred);
}

void launch_project(const DevCam &cam, const SceneDev &s, uint32_t *dkey, uint32_t *tiles, float4 *ell,
                    double2 *ell64, float4 *payload, uint32_t *counters, uint32_t *deferred, uint32_t *list,
                    cudaStream_t st) {
  if (s.n == 0) return;
  const unsigned blocks = (unsigned)((s.n + 255) / 256);
  const unsigned wblocks = 148 * 4;  // grid-stride over the deferred Gaussians (count known on the device only)
  // (global shutter: measured slower on every config -- the per-Gaussian work is small)
  if (cam.shutter != SH_GLOBAL && cam.model != CAM_ORTHO) {
    project_prefilter_kernel<<<blocks, 256, 0, st>>>(cam, s, dkey, tiles, counters, list);
  } else {
    list = nullptr;
  }
  switch (s.sh_degree) {
    case 0: launch_k1_deg<0>(cam, s, dkey, tiles, ell, ell64, payload, counters, deferred, list, blocks, wblocks, st); break;
    case 1: launch_k1_deg<1>(cam, s, dkey, tiles, ell, ell64, payload, counters, deferred, list, blocks, wblocks, st); break;
    case 2: launch_k1_deg<2>(cam, s, dkey, tiles, ell, ell64, payload, counters, deferred, list, blocks, wblocks, st); break;
    default: launch_k1_deg<3>(cam, s, dkey, tiles, ell, ell64, payload, counters, deferred, list, blocks, wblocks, st); break;
  }
}

}  // namespace gut

namespace gut {

// ---------------------------------------------------------------- Supp. C
// Projection quality (reading R31): per Gaussian the 2D image
// estimated by the UT (Eq. 6-10 without the binning dilation), by EWA (first-
// order linearisation at mu, Eq. 3: central-difference Jacobian of the camera
// projection, pose frozen at mu's own shutter time -- RS-unaware) and by Monte
// Carlo (n samples mu + R S z, z from the shared counter-based generator, each
// projected with its own RS-aware pose), and KL(MC || UT), KL(MC || EWA).
// One warp per Gaussian, fp64 (a measurement tool, not the render path).
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// N(0,1) triple of (seed, gaussian, sample): splitmix64 -> 53-bit uniforms ->
// Box-Muller (the spec the oracle implements independently, orc_normal3)
__device__ __forceinline__ d3 normal3(unsigned long long seed, long long gid, int s) {
  double u[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const unsigned long long h =
        mix64(seed ^ mix64(((unsigned long long)gid << 24) ^ ((unsigned long long)s << 2) ^ (unsigned long long)k));
    u[k] = ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  }
  const double tp = 6.283185307179586476925286766559;
  const double r0 = sqrt(-2.0 * log(u[0])), r1 = sqrt(-2.0 * log(u[2]));
  double s1, c1, s3, c3;
  sincos(tp * u[1], &s1, &c1);
  sincos(tp * u[3], &s3, &c3);
  return mkd(r0 * c1, r0 * s1, r1 * c3);
}

__device__ __forceinline__ double kl2(const double *g0, const double *g1) {
  const double d1 = g1[2] * g1[4] - g1[3] * g1[3], d0 = g0[2] * g0[4] - g0[3] * g0[3];
  const double i00 = g1[4] / d1, i01 = -g1[3] / d1, i11 = g1[2] / d1;
  const double tr = i00 * g0[2] + 2.0 * i01 * g0[3] + i11 * g0[4];
  const double dx = g1[0] - g0[0], dy = g1[1] - g0[1];
  return 0.5 * (tr + i00 * dx * dx + 2.0 * i01 * dx * dy + i11 * dy * dy - 2.0 + log(d1 / d0));
}

__global__ __launch_bounds__(256) void quality_kernel(DevCam c, SceneDev s, int n_mc, unsigned long long seed,
                                                      QualityRec *__restrict__ out) {
  const long long i = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= s.n) return;
  const float4 po = s.pos_opa[i], ro = s.rot[i], sc = s.scale[i];
  const double qn = sqrt((double)ro.x * ro.x + (double)ro.y * ro.y + (double)ro.z * ro.z + (double)ro.w * ro.w);
  const double w_ = ro.x / qn, x_ = ro.y / qn, y_ = ro.z / qn, z_ = ro.w / qn;
  const double R[9] = {1 - 2 * (y_ * y_ + z_ * z_), 2 * (x_ * y_ - w_ * z_), 2 * (x_ * z_ + w_ * y_),
                       2 * (x_ * y_ + w_ * z_), 1 - 2 * (x_ * x_ + z_ * z_), 2 * (y_ * z_ - w_ * x_),
                       2 * (x_ * z_ - w_ * y_), 2 * (y_ * z_ + w_ * x_), 1 - 2 * (x_ * x_ + y_ * y_)};
  const double sv[3] = {sc.x, sc.y, sc.z};
  const d3 mu = mkd(po.x, po.y, po.z), c0 = mkd(c.c0[0], c.c0[1], c.c0[2]);
  const d3 w = mtv(c.R0, mkd(c.dc[0], c.dc[1], c.dc[2]));
  bool ok = qn > 0 && sv[0] > 0 && sv[1] > 0 && sv[2] > 0;
  QualityRec q;
  memset(&q, 0, sizeof(q));
  double mx = 0, my = 0, t0 = 0;
  if (lane == 0 && ok) {
    // (a) UT: sigma points mu +- gamma s_j R[:, j]
    const d3 y0 = mtv(c.R0, mu - c0);
    double du[7], dv[7], tt;
    ok = project_sigma_d(c, y0, w, du[0], dv[0], t0);
    for (int j = 0; j < 3 && ok; ++j) {
      const d3 L = mtv(c.R0, ((double)c.gamma * sv[j]) * mkd(R[j], R[3 + j], R[6 + j]));
      ok = ok && project_sigma_d(c, y0 + L, w, du[1 + j], dv[1 + j], tt);
      ok = ok && project_sigma_d(c, y0 - L, w, du[4 + j], dv[4 + j], tt);
    }
    if (ok) {
      mx = (double)c.wmu0 * du[0]; my = (double)c.wmu0 * dv[0];
      for (int k = 1; k < 7; ++k) { mx += (double)c.wmui * du[k]; my += (double)c.wmui * dv[k]; }
      double sxx = 0, sxy = 0, syy = 0;
      for (int k = 0; k < 7; ++k) {
        const double wk = k == 0 ? (double)c.wsig0 : (double)c.wsigi;
        const double ax = du[k] - mx, ay = dv[k] - my;
        sxx += wk * ax * ax; sxy += wk * ax * ay; syy += wk * ay * ay;
      }
      q.ut[0] = mx + c.cx; q.ut[1] = my + c.cy; q.ut[2] = sxx; q.ut[3] = sxy; q.ut[4] = syy;
      // (b) EWA at the pose frozen at t0: p = R_t^T (y - t0 w)
      double Rt[9];
      rodrigues_d(mkd(c.phi_axis[0], c.phi_axis[1], c.phi_axis[2]), t0 * c.phi_angle, Rt);
      const d3 p0 = mtv(Rt, y0 - t0 * w);
      double g0u, g0v, J[2][3];
      ok = project_cam_d(c, p0, g0u, g0v);
      const double h = 1e-6 * sqrt(dot(p0, p0));
      for (int a = 0; a < 3 && ok; ++a) {
        d3 e = mkd(a == 0, a == 1, a == 2);
        double up, vp, um, vm;
        ok = project_cam_d(c, p0 + h * e, up, vp) && project_cam_d(c, p0 - h * e, um, vm);
        J[0][a] = (up - um) / (2 * h);
        J[1][a] = (vp - vm) / (2 * h);
      }
      if (ok) {
        // Sigma_cam = A A^T, A = R_t^T R0^T R S
        double A[9];
        for (int col = 0; col < 3; ++col) {
          const d3 v = mtv(Rt, mtv(c.R0, sv[col] * mkd(R[col], R[3 + col], R[6 + col])));
          A[col] = v.x; A[3 + col] = v.y; A[6 + col] = v.z;
        }
        double JA[2][3];
        for (int r = 0; r < 2; ++r)
          for (int col = 0; col < 3; ++col) JA[r][col] = J[r][0] * A[col] + J[r][1] * A[3 + col] + J[r][2] * A[6 + col];
        q.ewa[0] = g0u + c.cx; q.ewa[1] = g0v + c.cy;
        q.ewa[2] = JA[0][0] * JA[0][0] + JA[0][1] * JA[0][1] + JA[0][2] * JA[0][2];
        q.ewa[3] = JA[0][0] * JA[1][0] + JA[0][1] * JA[1][1] + JA[0][2] * JA[1][2];
        q.ewa[4] = JA[1][0] * JA[1][0] + JA[1][1] * JA[1][1] + JA[1][2] * JA[1][2];
      }
    }
  }
  ok = __shfl_sync(0xffffffffu, ok, 0);
  mx = __shfl_sync(0xffffffffu, mx, 0);
  my = __shfl_sync(0xffffffffu, my, 0);
  // (c) Monte Carlo: sums relative to the UT mean
  double s1x = 0, s1y = 0, sxx = 0, sxy = 0, syy = 0;
  bool mok = ok;
  for (int smp = lane; smp < n_mc && ok; smp += 32) {
    const d3 z = normal3(seed, i, smp);
    const d3 x = mu + mkd(R[0] * sv[0] * z.x + R[1] * sv[1] * z.y + R[2] * sv[2] * z.z,
                          R[3] * sv[0] * z.x + R[4] * sv[1] * z.y + R[5] * sv[2] * z.z,
                          R[6] * sv[0] * z.x + R[7] * sv[1] * z.y + R[8] * sv[2] * z.z);
    double du, dv, tt;
    mok = mok && project_sigma_d(c, mtv(c.R0, x - c0), w, du, dv, tt);
    const double dx = du - mx, dy = dv - my;
    s1x += dx; s1y += dy; sxx += dx * dx; sxy += dx * dy; syy += dy * dy;
  }
  ok = __all_sync(0xffffffffu, mok) && ok;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1x += __shfl_xor_sync(0xffffffffu, s1x, o); s1y += __shfl_xor_sync(0xffffffffu, s1y, o);
    sxx += __shfl_xor_sync(0xffffffffu, sxx, o); sxy += __shfl_xor_sync(0xffffffffu, sxy, o);
    syy += __shfl_xor_sync(0xffffffffu, syy, o);
  }
  if (lane == 0) {
    if (ok && n_mc >= 2) {
      const double ax = s1x / n_mc, ay = s1y / n_mc;
      q.mc[0] = mx + ax + c.cx; q.mc[1] = my + ay + c.cy;
      q.mc[2] = sxx / n_mc - ax * ax; q.mc[3] = sxy / n_mc - ax * ay; q.mc[4] = syy / n_mc - ay * ay;
      q.kl_ut = kl2(q.mc, q.ut);
      q.kl_ewa = kl2(q.mc, q.ewa);
      q.valid = 1;
    } else {
      memset(&q, 0, sizeof(q));
    }
    out[i] = q;
  }
}

void launch_quality(const DevCam &cam, const SceneDev &s, int n_mc, unsigned long long seed, QualityRec *out,
                    cudaStream_t st) {
  if (s.n > 0) quality_kernel<<<(unsigned)((s.n * 32 + 255) / 256), 256, 0, st>>>(cam, s, n_mc, seed, out);
}

}  // namespace gut

namespace gut {

// Shutter time t0 of each Gaussian's centre (the fixed point K1 solves for
// sigma point 0, reading R14; fp64 secant as the wide kernel): the view
// direction of its SH colour is normalize(mu - c(t0)) (reading R18).  Used by
// the backward's SH gradients under rolling shutter.
__global__ __launch_bounds__(256) void centre_time_kernel(DevCam c, SceneDev s, float *__restrict__ t0) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= s.n) return;
  const float4 po = s.pos_opa[i];
  const d3 y0 = mtv(c.R0, mkd(po.x, po.y, po.z) - mkd(c.c0[0], c.c0[1], c.c0[2]));
  const d3 w = mtv(c.R0, mkd(c.dc[0], c.dc[1], c.dc[2]));
  double du, dv, t = 0.0;
  if (!project_sigma_d(c, y0, w, du, dv, t)) t = 0.0;
  t0[i] = (float)t;
}

void launch_centre_times(const DevCam &cam, const SceneDev &s, float *t0, cudaStream_t st) {
  if (s.n > 0) centre_time_kernel<<<(unsigned)((s.n + 255) / 256), 256, 0, st>>>(cam, s, t0);
}

}  // namespace gut
