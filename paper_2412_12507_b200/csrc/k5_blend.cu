// k5_blend.cu — K5: per-pixel front-to-back compositing with the 3D
// max-response (the paper's "Render"), sm_100a.
//
// PAPER Eq. 5 (L115-121): c = sum_i c_i alpha_i prod_{j<i}(1 - alpha_j),
// alpha_i = sigma_i rho_i(o + tau d); Eq. 11 (L195-200): tau_max =
// -o_g.d_g / d_g.d_g with o_g = S^-1 R^T (o - mu), d_g = S^-1 R^T d, and the
// response at tau_max is exp(-omega^2/2), omega^2 = ||o_g x d_g||^2/||d_g||^2
// (Supp. B, L506).  Order = the tile's global depth order (L208).
//
// One CTA per 16x16 tile, one pixel per thread, warps on 8x4 pixel blocks.
// Precision design: the cross product o_g x d_g
// cancels catastrophically in fp32 for small, distant Gaussians, so every
// pixel ray is written relative to a per-tile anchor ray (D, O) as
//   d' = D + a T1 + b T2  (central cameras; a, b = tangent-plane offsets),
//   o  = O + a T1 + b T2  (orthographic),   o = O + beta dc  (rolling shutter),
// and per (tile, entry) the large, cancelling part c0 = o_g x (M D) is formed
// in fp64 while staging the entry into shared memory.  What remains per
// (pixel, entry) pair is fp32 and small:
//   n = c0 + a P + b Q [+ beta (h + a PU + b QV)],  e = e0 + a U + b V
//   omega^2 = |n|^2 / |e|^2,   reject before MUFU if |n|^2 > k^2 |e|^2
// with k^2 = 2 ln(sigma / alpha_min) (alpha >= alpha_min <=> omega^2 <= k^2).
#include "launch.h"

namespace gut {

__device__ __forceinline__ d3 normalize_d(d3 v) {
  double n = sqrt(dot(v, v));
  return (1.0 / n) * v;
}

__device__ __forceinline__ double pixel_time(const DevCam &c, double u, double v) {
  switch (c.shutter) {
    case SH_T2B: return v / c.height;
    case SH_B2T: return 1.0 - v / c.height;
    case SH_L2R: return u / c.width;
    case SH_R2L: return 1.0 - u / c.width;
    default: return 0.0;
  }
}

// inverse camera in fp64: camera-frame unit direction (and ortho origin offset)
__device__ bool unproject(const DevCam &c, double u, double v, d3 &dcam, d3 &ocam) {
  const double xd = (u - c.cx) / c.fx, yd = (v - c.cy) / c.fy;
  ocam = mkd(0, 0, 0);
  switch (c.model) {
    case CAM_PINHOLE: dcam = normalize_d(mkd(xd, yd, 1.0)); return true;
    case CAM_ORTHO: ocam = mkd(xd, yd, 0.0); dcam = mkd(0, 0, 1); return true;
    case CAM_OPENCV: {
      // Newton with the analytic Jacobian of the rad-tan distortion map
      double x = xd, y = yd;
      bool conv = false;
      for (int it = 0; it < 30; ++it) {
        double r2 = x * x + y * y;
        double num = 1 + r2 * (c.k[0] + r2 * (c.k[1] + r2 * c.k[2]));
        double den = 1 + r2 * (c.k[3] + r2 * (c.k[4] + r2 * c.k[5]));
        double dnum = c.k[0] + r2 * (2 * c.k[1] + 3 * c.k[2] * r2);
        double dden = c.k[3] + r2 * (2 * c.k[4] + 3 * c.k[5] * r2);
        double a = num / den, ap = (dnum * den - num * dden) / (den * den);
        double fx = x * a + 2 * c.p[0] * x * y + c.p[1] * (r2 + 2 * x * x) - xd;
        double fy = y * a + c.p[0] * (r2 + 2 * y * y) + 2 * c.p[1] * x * y - yd;
        if (fabs(fx) + fabs(fy) < 1e-14) { conv = true; break; }
        double j00 = a + 2 * x * x * ap + 2 * c.p[0] * y + 6 * c.p[1] * x;
        double j01 = 2 * x * y * ap + 2 * c.p[0] * x + 2 * c.p[1] * y;
        double j11 = a + 2 * y * y * ap + 6 * c.p[0] * y + 2 * c.p[1] * x;
        double det = j00 * j11 - j01 * j01;
        if (!(fabs(det) > 0)) break;
        x -= (j11 * fx - j01 * fy) / det;
        y -= (-j01 * fx + j00 * fy) / det;
      }
      if (!conv) return false;
      if (c.fov > 0 && !(x * x + y * y <= c.fov * c.fov)) return false;
      dcam = normalize_d(mkd(x, y, 1.0));
      return true;
    }
    case CAM_FISHEYE: {
      const double td = sqrt(xd * xd + yd * yd);
      double th = td;
      if (c.k[0] != 0 || c.k[1] != 0 || c.k[2] != 0 || c.k[3] != 0) {
        for (int it = 0; it < 30; ++it) {
          double t2 = th * th;
          double f = th * (1 + t2 * (c.k[0] + t2 * (c.k[1] + t2 * (c.k[2] + t2 * c.k[3])))) - td;
          double fp = 1 + t2 * (3 * c.k[0] + t2 * (5 * c.k[1] + t2 * (7 * c.k[2] + t2 * 9 * c.k[3])));
          double st = f / fp;
          th -= st;
          if (fabs(st) < 1e-15) break;
        }
        double t2 = th * th;
        if (fabs(th * (1 + t2 * (c.k[0] + t2 * (c.k[1] + t2 * (c.k[2] + t2 * c.k[3])))) - td) > 1e-12) return false;
      }
      if (!(th <= c.fov)) return false;
      if (td == 0.0) { dcam = mkd(0, 0, 1); return true; }
      double s, co;
      sincos(th, &s, &co);
      dcam = mkd(s * xd / td, s * yd / td, co);
      return true;
    }
  }
  return false;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int MODE>  // 0: central global shutter, 1: orthographic, 2: central rolling shutter
__global__ __launch_bounds__(GUT_BLEND_THREADS) void blend_kernel(
    DevCam c, const uint2 *__restrict__ ranges, const uint32_t *__restrict__ gids,
    const float4 *__restrict__ payload, float *__restrict__ out_rgb, float *__restrict__ out_alpha,
    float *__restrict__ out_depth, uint32_t *counters, uint2 *__restrict__ tile_work) {
  constexpr int NF = MODE == 2 ? 10 : 7;
  __shared__ float4 s_f[NF][GUT_BLEND_THREADS];
  __shared__ double s_red[8][4];
  __shared__ double s_anchor[13];  // D(3) O(3) T1(3) T2(3) t_anchor
  __shared__ int s_nvalid;

  const int tile = blockIdx.x;
  const int tx = tile % c.tiles_x, ty = tile / c.tiles_x;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int px = tx * GUT_TILE + (w & 1) * 8 + (lane & 7);
  const int py = ty * GUT_TILE + (w >> 1) * 4 + (lane >> 3);
  const bool inside = px < c.width && py < c.height;
  const double u = px + 0.5, v = py + 0.5;

  // ---- per-pixel ray in fp64 (PAPER L116 r(tau) = o + tau d; reading R17 time)
  d3 dcam = mkd(0, 0, 1), ocam = mkd(0, 0, 0);
  bool valid = inside && unproject(c, u, v, dcam, ocam);
  const double tp = pixel_time(c, u, v);
  d3 dw = mkd(0, 0, 0);
  if (valid) {
    if (MODE == 2) {
      double Rt[9], Rw[9];
      rodrigues_d(mkd(c.phi_axis[0], c.phi_axis[1], c.phi_axis[2]), tp * c.phi_angle, Rt);
      matmul3(c.R0, Rt, Rw);
      dw = mv(Rw, dcam);
    } else if (MODE == 0) {
      dw = mv(c.R0, dcam);
    }
  }
  // ---- tile anchor: mean valid direction (central) / mean valid origin (ortho)
  d3 red = MODE == 1 ? ocam : dw;
  if (!valid) red = mkd(0, 0, 0);
  double rx = warp_sum(red.x), ry = warp_sum(red.y), rz = warp_sum(red.z);
  double rn = warp_sum(valid ? 1.0 : 0.0);
  if (lane == 0) { s_red[w][0] = rx; s_red[w][1] = ry; s_red[w][2] = rz; s_red[w][3] = rn; }
  __syncthreads();
  if (threadIdx.x == 0) {
    d3 s = mkd(0, 0, 0);
    double cnt = 0;
    for (int k = 0; k < 8; ++k) { s = s + mkd(s_red[k][0], s_red[k][1], s_red[k][2]); cnt += s_red[k][3]; }
    s_nvalid = (int)cnt;
    d3 D, O, T1, T2;
    double ta = 0;
    if (MODE == 1) {
      d3 m = (cnt > 0 ? 1.0 / cnt : 0.0) * s;
      O = mkd(c.c0[0], c.c0[1], c.c0[2]) + mv(c.R0, m);
      D = mv(c.R0, mkd(0, 0, 1));
      T1 = mv(c.R0, mkd(1, 0, 0));
      T2 = mv(c.R0, mkd(0, 1, 0));
      s_anchor[12] = 0;
      // store the mean camera-frame offset in T-slots' spare: reuse s_red
      s_red[0][0] = m.x; s_red[0][1] = m.y;
    } else {
      D = cnt > 0 ? normalize_d(s) : mkd(0, 0, 1);
      d3 h = fabs(D.x) < 0.6 ? mkd(1, 0, 0) : (fabs(D.y) < 0.6 ? mkd(0, 1, 0) : mkd(0, 0, 1));
      T1 = normalize_d(h - dot(h, D) * D);
      T2 = cross(D, T1);
      if (MODE == 2) {
        double uc = fmin(fmax(tx * GUT_TILE + 8.0, 0.5), c.width - 0.5);
        double vc = fmin(fmax(ty * GUT_TILE + 8.0, 0.5), c.height - 0.5);
        ta = pixel_time(c, uc, vc);
      }
      O = mkd(c.c0[0] + ta * c.dc[0], c.c0[1] + ta * c.dc[1], c.c0[2] + ta * c.dc[2]);
    }
    s_anchor[0] = D.x; s_anchor[1] = D.y; s_anchor[2] = D.z;
    s_anchor[3] = O.x; s_anchor[4] = O.y; s_anchor[5] = O.z;
    s_anchor[6] = T1.x; s_anchor[7] = T1.y; s_anchor[8] = T1.z;
    s_anchor[9] = T2.x; s_anchor[10] = T2.y; s_anchor[11] = T2.z;
    s_anchor[12] = ta;
  }
  __syncthreads();
  const d3 D = mkd(s_anchor[0], s_anchor[1], s_anchor[2]);
  const d3 O = mkd(s_anchor[3], s_anchor[4], s_anchor[5]);
  const d3 T1 = mkd(s_anchor[6], s_anchor[7], s_anchor[8]);
  const d3 T2 = mkd(s_anchor[9], s_anchor[10], s_anchor[11]);
  const f3 T1f = tof(T1), T2f = tof(T2);
  float a = 0.f, b = 0.f, beta = 0.f, snorm = 1.f;
  if (valid) {
    if (MODE == 1) {
      a = (float)(ocam.x - s_red[0][0]);
      b = (float)(ocam.y - s_red[0][1]);
    } else {
      double den = dot(dw, D);
      a = (float)(dot(dw, T1) / den);
      b = (float)(dot(dw, T2) / den);
      snorm = (float)(1.0 / den);
      if (!(den > 0)) valid = false;
      if (MODE == 2) beta = (float)(tp - s_anchor[12]);
    }
  }

  // ---- compositing state
  float T = 1.f, Cr = 0.f, Cg = 0.f, Cb = 0.f, Dp = 0.f;
  bool done = !valid;
  uint32_t n_eval = 0, n_contrib = 0, n_term = 0, processed = 0;
  const uint2 rg = ranges[tile];
  const uint32_t start = rg.x, end = rg.y > rg.x ? rg.y : rg.x;
  if (threadIdx.x == 0 && end > start) atomicMax(&counters[CNT_MAXLEN], end - start);
  const f3 dcw = mk((float)c.dc[0], (float)c.dc[1], (float)c.dc[2]);

  for (uint32_t b0 = start; b0 < end; b0 += GUT_BLEND_THREADS) {
    const uint32_t cnt = min((uint32_t)GUT_BLEND_THREADS, end - b0);
    __syncthreads();
    if (threadIdx.x < cnt) {
      // ---- stage one list entry: fp64 for the cancelling part, fp32 for the rest
      const uint32_t g = __ldg(&gids[b0 + threadIdx.x]);
      const float4 p0 = __ldg(&payload[4 * g]), p1 = __ldg(&payload[4 * g + 1]);
      const float4 p2 = __ldg(&payload[4 * g + 2]), p3 = __ldg(&payload[4 * g + 3]);
      const float M[9] = {p1.x, p1.y, p1.z, p1.w, p2.x, p2.y, p2.z, p2.w, p3.x};
      const double Md[9] = {p1.x, p1.y, p1.z, p1.w, p2.x, p2.y, p2.z, p2.w, p3.x};
      const d3 og = mv(Md, O - mkd(p0.x, p0.y, p0.z));
      const d3 e0d = mv(Md, D);
      const d3 c0 = cross(og, e0d);
      const double g0 = dot(og, e0d);
      const f3 ogf = tof(og), e0 = tof(e0d);
      f3 U = mv(M, T1f), V = mv(M, T2f), P, Q;
      float gu, gv;
      if (MODE == 1) {
        P = cross(U, e0); Q = cross(V, e0); gu = dot(U, e0); gv = dot(V, e0);
        U = mk(0, 0, 0); V = mk(0, 0, 0);
      } else {
        P = cross(ogf, U); Q = cross(ogf, V); gu = dot(ogf, U); gv = dot(ogf, V);
      }
      const float k2 = 2.f * logf(p0.w / c.alpha_min);
      const float l2s = log2f(p0.w);
      const int t = threadIdx.x;
      s_f[0][t] = make_float4((float)c0.x, (float)c0.y, (float)c0.z, k2);
      s_f[1][t] = make_float4(P.x, P.y, P.z, Q.x);
      s_f[2][t] = make_float4(Q.y, Q.z, e0.x, e0.y);
      s_f[3][t] = make_float4(e0.z, U.x, U.y, U.z);
      s_f[4][t] = make_float4(V.x, V.y, V.z, l2s);
      s_f[5][t] = make_float4((float)g0, gu, gv, 0.f);
      s_f[6][t] = make_float4(p3.y, p3.z, p3.w, 0.f);
      if (MODE == 2) {
        const f3 m = mv(M, dcw);
        const f3 h = cross(m, e0), PU = cross(m, U), QV = cross(m, V);
        s_f[NF - 3][t] = make_float4(h.x, h.y, h.z, dot(m, e0));
        s_f[NF - 2][t] = make_float4(PU.x, PU.y, PU.z, dot(m, U));
        s_f[NF - 1][t] = make_float4(QV.x, QV.y, QV.z, dot(m, V));
      }
    }
    __syncthreads();
    for (uint32_t k = 0; k < cnt; ++k) {
      if (done) break;
      ++n_eval;
      const float4 f0 = s_f[0][k], f1 = s_f[1][k], f2 = s_f[2][k], f3v = s_f[3][k], f4 = s_f[4][k];
      float nx = fmaf(a, f1.x, fmaf(b, f1.w, f0.x));
      float ny = fmaf(a, f1.y, fmaf(b, f2.x, f0.y));
      float nz = fmaf(a, f1.z, fmaf(b, f2.y, f0.z));
      if (MODE == 2) {
        const float4 h = s_f[NF - 3][k], pu = s_f[NF - 2][k], qv = s_f[NF - 1][k];
        nx = fmaf(beta, fmaf(a, pu.x, fmaf(b, qv.x, h.x)), nx);
        ny = fmaf(beta, fmaf(a, pu.y, fmaf(b, qv.y, h.y)), ny);
        nz = fmaf(beta, fmaf(a, pu.z, fmaf(b, qv.z, h.z)), nz);
      }
      const float ex = fmaf(a, f3v.y, fmaf(b, f4.x, f2.z));
      const float ey = fmaf(a, f3v.z, fmaf(b, f4.y, f2.w));
      const float ez = fmaf(a, f3v.w, fmaf(b, f4.z, f3v.x));
      const float N = fmaf(nx, nx, fmaf(ny, ny, nz * nz));
      const float Dd = fmaf(ex, ex, fmaf(ey, ey, ez * ez));
      if (N > f0.w * Dd) continue;  // omega^2 > k^2  <=>  alpha < alpha_min
      const float rD = __frcp_rn(Dd);
      const float w2 = N * rD;
      const float al = fminf(c.alpha_max, exp2f(fmaf(-0.72134752044448170f, w2, f4.w)));
      if (!(al >= c.alpha_min)) continue;
      const float4 f5 = s_f[5][k];
      float gg = fmaf(a, f5.y, fmaf(b, f5.z, f5.x));
      if (MODE == 2) {
        const float4 h = s_f[NF - 3][k], pu = s_f[NF - 2][k], qv = s_f[NF - 1][k];
        gg = fmaf(beta, fmaf(a, pu.w, fmaf(b, qv.w, h.w)), gg);
      }
      const float tau = -gg * rD * snorm;
      if (!(tau > 0.f)) continue;  // reading R24
      const float Tn = T * (1.f - al);
      if (Tn < c.t_min) { done = true; n_term = 1; break; }
      const float4 f6 = s_f[6][k];
      const float wgt = al * T;
      Cr = fmaf(wgt, f6.x, Cr);
      Cg = fmaf(wgt, f6.y, Cg);
      Cb = fmaf(wgt, f6.z, Cb);
      Dp = fmaf(wgt, tau, Dp);
      T = Tn;
      ++n_contrib;
    }
    processed = b0 - start + cnt;
    if (__syncthreads_count(done) == GUT_BLEND_THREADS) break;
  }

  if (inside) {
    const size_t pix = (size_t)py * c.width + px;
    if (valid) {
      out_rgb[3 * pix] = Cr + T * c.bg[0];
      out_rgb[3 * pix + 1] = Cg + T * c.bg[1];
      out_rgb[3 * pix + 2] = Cb + T * c.bg[2];
      out_alpha[pix] = 1.f - T;
      if (out_depth) out_depth[pix] = Dp;
    } else {
      out_rgb[3 * pix] = c.bg[0];
      out_rgb[3 * pix + 1] = c.bg[1];
      out_rgb[3 * pix + 2] = c.bg[2];
      out_alpha[pix] = 0.f;
      if (out_depth) out_depth[pix] = 0.f;
    }
  }
  // statistics
  if (threadIdx.x == 0) tile_work[tile] = make_uint2(end - start, processed);
  unsigned long long e1 = warp_sum((unsigned long long)n_eval);
  unsigned long long e2 = warp_sum((unsigned long long)n_contrib);
  unsigned long long e3 = warp_sum((unsigned long long)n_term);
  if (lane == 0 && (e1 | e2 | e3)) {
    atomicAdd(reinterpret_cast<unsigned long long *>(&counters[CNT_PAIRS_EVAL]), e1);
    atomicAdd(reinterpret_cast<unsigned long long *>(&counters[CNT_PAIRS_CONTRIB]), e2);
    atomicAdd(reinterpret_cast<unsigned long long *>(&counters[CNT_TERMINATED]), e3);
  }
}

void launch_blend(const DevCam &cam, const uint2 *ranges, const uint32_t *gids, const float4 *payload,
                  float *rgb, float *alpha, float *depth, uint32_t *counters, uint2 *tile_work, cudaStream_t st) {
  const unsigned blocks = (unsigned)cam.n_tiles;
  if (cam.model == CAM_ORTHO)
    blend_kernel<1><<<blocks, GUT_BLEND_THREADS, 0, st>>>(cam, ranges, gids, payload, rgb, alpha, depth, counters, tile_work);
  else if (cam.shutter != SH_GLOBAL)
    blend_kernel<2><<<blocks, GUT_BLEND_THREADS, 0, st>>>(cam, ranges, gids, payload, rgb, alpha, depth, counters, tile_work);
  else
    blend_kernel<0><<<blocks, GUT_BLEND_THREADS, 0, st>>>(cam, ranges, gids, payload, rgb, alpha, depth, counters, tile_work);
}

}  // namespace gut
