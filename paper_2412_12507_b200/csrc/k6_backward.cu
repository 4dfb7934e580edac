// k6_backward.cu — K6: backward pass of the compositing and the 3D response
// (PAPER Supp. B, L494-513; reading R30: the UT / binning is not
// differentiated; the colour's view direction is held constant).
//
// Scalar loss L = sum_px g_rgb.rgb + g_alpha alpha + g_depth depth.  Per pixel,
// front to back over the tile's list (the forward's order and hit rules):
//   w_i = alpha_i T_i,  g_i = c_i.g_rgb + tau_i g_depth,
//   dL/dalpha_i = T_i g_i - S_i / (1 - alpha_i),  S_i = G - sum_{j<=i} w_j g_j,
//   G = rgb.g_rgb + depth g_depth - T_f g_alpha  (from the forward's outputs),
//   dL/dc_i = w_i g_rgb,  dL/dtau_i = w_i g_depth,
//   alpha = min(alpha_max, sigma exp(-omega^2/2)).
// Eq. 11 in canonical space with the pixel ray d' = D + a T1 + b T2 (tile
// anchor, as in K5; tau_world = tau' |d'|), o_g = M (o - mu), d_g = M d',
// n = o_g x d_g (the cofactor form, accurate), x_g = (d_g x n) / |d_g|^2:
//   dL/do_g = 2 dL/domega^2 x_g - (dL/dtau' / |d_g|^2) d_g
//   dL/dM   = dL/do_g (M^-1 x_g)^T - (dL/dtau' / |d_g|^2) x_g d'^T
//   dL/dmu  = -M^T dL/do_g
// (o - mu = M^-1 x_g - tau' d' removes the cancelling (o - mu) term).  Per
// list entry the 32 lanes' contributions are summed with warp shuffles and
// added to per-Gaussian fp32 accumulators with atomics (summation order not
// fixed: results reproducible to fp32 rounding, not bitwise).  A per-Gaussian
// kernel then maps dL/dM -> (s, R) -> q and dL/dc -> SH.
#include "launch.h"

namespace gut {

namespace {

template <int MODE> struct BwNF { static constexpr int v = 10; };  // float4 per staged entry
template <> struct BwNF<2> { static constexpr int v = 13; };              // + rolling-shutter terms

__device__ __forceinline__ float ex2f_(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <class T>
__device__ __forceinline__ T wsum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Butterfly reduce-scatter: value q of the result (q = lane >> 1) summed over
// the warp.  Step with offset o keeps the half of the values selected by the
// lane's bit o and adds the partner's copy of that half.
__device__ __forceinline__ float reduce16(const float (&v)[16], int lane) {
  float x8[8], x4[4], x2[2];
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float keep = b4 ? v[8 + k] : v[k], send = b4 ? v[k] : v[8 + k];
    x8[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float keep = b3 ? x8[4 + k] : x8[k], send = b3 ? x8[k] : x8[4 + k];
    x4[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float keep = b2 ? x4[2 + k] : x4[k], send = b2 ? x4[k] : x4[2 + k];
    x2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  const float keep = b1 ? x2[1] : x2[0], send = b1 ? x2[0] : x2[1];
  const float x1 = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  return x1 + __shfl_xor_sync(0xffffffffu, x1, 1);
}

}  // namespace

// One CTA per tile, 8 warps = the tile's 8x4 pixel blocks (one pixel per lane,
// rays_kernel's layout); every warp walks the whole list in chunks of 32.
template <int MODE>
#ifndef GUT_K6_MINB
#define GUT_K6_MINB 1  // min resident CTAs per SM for the register budget (tuning switch)
#endif
__global__ __launch_bounds__(256, GUT_K6_MINB) void backward_kernel(DevCam c, BwdBufs B) {
  constexpr int BW_NF = BwNF<MODE>::v;
  extern __shared__ float4 s_dyn[];
  // CTAs take the tiles in decreasing list length (the plan's queue 1 with one
  // unit per tile): the longest lists start first, no long tail
  const int tile = (int)(B.order[blockIdx.x] & 0xFFFFFFu), w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr unsigned FULL = 0xffffffffu;
  float4 *tbl = s_dyn + w * 32 * BW_NF;
  int px, py;
  px = (tile % c.tiles_x) * GUT_TILE + (w & 1) * 8 + (lane & 7);
  py = (tile / c.tiles_x) * GUT_TILE + (w >> 1) * 4 + (lane >> 3);
  const bool inside = px < c.width && py < c.height;
  const float4 pl = B.pix[(size_t)tile * GUT_TILE_PX + w * 32 + lane];
  const float a = pl.x, b = pl.y, snorm = pl.z, beta = pl.w;  // beta: rolling shutter t_pixel - t_anchor
  bool done = !(inside && snorm > 0.f);
  // per-pixel upstream gradients and the forward's outputs
  float gr = 0.f, gg = 0.f, gb = 0.f, gA = 0.f, gD = 0.f, Gtot = 0.f;
  if (!done) {
    const size_t p = (size_t)py * c.width + px;
    gr = B.g_rgb[3 * p]; gg = B.g_rgb[3 * p + 1]; gb = B.g_rgb[3 * p + 2];
    gA = B.g_alpha ? B.g_alpha[p] : 0.f;
    gD = B.g_depth ? B.g_depth[p] : 0.f;
    const float Tf = 1.f - B.alpha[p];
    Gtot = B.rgb[3 * p] * gr + B.rgb[3 * p + 1] * gg + B.rgb[3 * p + 2] * gb + (B.depth ? B.depth[p] * gD : 0.f) -
           Tf * gA;
  }
  // tile anchor -> world (MODE 2: the anchors are world-frame, origin O = c(t_anchor))
  const TileAnchor &A = B.anchors[tile];
  d3 D, T1, T2, dO = mkd(0, 0, 0);
  if (MODE == 2) {
    D = mkd(A.D[0], A.D[1], A.D[2]); T1 = mkd(A.T1[0], A.T1[1], A.T1[2]); T2 = mkd(A.T2[0], A.T2[1], A.T2[2]);
    dO = mkd(A.O[0] - c.c0[0], A.O[1] - c.c0[1], A.O[2] - c.c0[2]);
  } else {
    D = mv(c.R0, mkd(A.D[0], A.D[1], A.D[2]));
    T1 = mv(c.R0, mkd(A.T1[0], A.T1[1], A.T1[2]));
    T2 = mv(c.R0, mkd(A.T2[0], A.T2[1], A.T2[2]));
  }
  const f3 dcw = mk((float)c.dc[0], (float)c.dc[1], (float)c.dc[2]);
  // kernel degree n (Supp. A): log2 alpha = log2 sigma - lambda_n (omega^2)^(n/2) / (2 ln 2)
  const bool gen = c.kdeg != 2;
  const float kgl = -0.72134752044448170f * c.klam, khn = 0.5f * (float)c.kdeg;
  const f3 Df = tof(D), T1f = tof(T1), T2f = tof(T2);
  const f3 dpw = Df + a * T1f + b * T2f;  // d' (world, |d'| = snorm)
  // the warp's pixel box in (a, b) for the conservative entry cull (as K5)
  float amin = done ? 3e38f : a, amax = done ? -3e38f : a, bmin = done ? 3e38f : b, bmax = done ? -3e38f : b;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    amin = fminf(amin, __shfl_xor_sync(FULL, amin, o));
    amax = fmaxf(amax, __shfl_xor_sync(FULL, amax, o));
    bmin = fminf(bmin, __shfl_xor_sync(FULL, bmin, o));
    bmax = fmaxf(bmax, __shfl_xor_sync(FULL, bmax, o));
  }
  if (amin > amax) { amin = amax = bmin = bmax = 0.f; }
  const float ac = 0.5f * (amin + amax), bc = 0.5f * (bmin + bmax);
  const float ra = 0.5f * (amax - amin) + 1e-7f * (fabsf(amin) + fabsf(amax));
  const float rb = 0.5f * (bmax - bmin) + 1e-7f * (fabsf(bmin) + fabsf(bmax));
  const uint2 rg = B.ranges[tile];
  const uint32_t start = rg.y > rg.x ? rg.x : 0u, end = rg.y > rg.x ? rg.y : 0u;
  const float l2amin = log2f(c.alpha_min);
  float T = 1.f, Gpre = 0.f;
  for (uint32_t b0 = start; b0 < end; b0 += 32) {
    if (__all_sync(FULL, done)) break;
    const uint32_t kk = b0 + lane;
    __syncwarp();
    bool maybe = false;
    if (kk < end) {
      const uint32_t gid = B.gids[kk];
      const float4 *src = B.payload + (size_t)GUT_PAYLOAD_F4 * gid;
      const double2 wxy = *reinterpret_cast<const double2 *>(src);
      const float4 p1 = src[1], p2 = src[2], p3 = src[3], p4 = src[4];
      const d3 wv = mkd(wxy.x, wxy.y, __hiloint2double(__float_as_int(p1.y), __float_as_int(p1.x))) + dO;
      const f3 x = tof(cross(wv, D));
      const float M[9] = {p1.w, p2.x, p2.y, p2.z, p2.w, p3.x, p3.y, p3.z, p3.w};
      const float rn0 = fmaf(M[0], M[0], fmaf(M[1], M[1], M[2] * M[2]));
      const float rn1 = fmaf(M[3], M[3], fmaf(M[4], M[4], M[5] * M[5]));
      const float rn2 = fmaf(M[6], M[6], fmaf(M[7], M[7], M[8] * M[8]));
      // (MUFU rsqrt / rcp as K5's staging: the same c0 and hit decisions)
      float r012 = rn0 * rn1 * rn2, rq;
      asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rq) : "f"(r012));
      const float dM = r012 * rq;
      const float irn0 = rs_rcp(rn0), irn1 = rs_rcp(rn1), irn2 = rs_rcp(rn2);
      const f3 Mx = mv(M, x);
      const f3 c0 = mk(Mx.x * (dM * irn0), Mx.y * (dM * irn1), Mx.z * (dM * irn2));
      const f3 ogf = mv(M, tof(wv)), e0 = mv(M, Df), U = mv(M, T1f), V = mv(M, T2f);
      const f3 P = cross(ogf, U), Q = cross(ogf, V);
      const float k2 = p1.z;
      const float l2s = c.kdeg == 2 ? fmaf(k2, 0.72134752044448170f, l2amin) : p4.w;
      float4 *t = tbl + lane * BW_NF;
      t[0] = make_float4(c0.x, c0.y, c0.z, k2);
      t[1] = make_float4(P.x, P.y, P.z, Q.x);
      t[2] = make_float4(Q.y, Q.z, e0.x, e0.y);
      t[3] = make_float4(e0.z, U.x, U.y, U.z);
      t[4] = make_float4(V.x, V.y, V.z, l2s);
      t[5] = make_float4(dot(ogf, e0), dot(ogf, U), dot(ogf, V), __uint_as_float(gid));
      t[6] = make_float4(p4.x, p4.y, p4.z, 0.f);
      // M^-1 = R S: (M^-1)_jk = M_kj / |M_k|^2
      t[7] = make_float4(M[0] * irn0, M[3] * irn1, M[6] * irn2, M[1] * irn0);
      t[8] = make_float4(M[4] * irn1, M[7] * irn2, M[2] * irn0, M[5] * irn1);
      t[9] = make_float4(M[8] * irn2, 0.f, 0.f, 0.f);
      if (MODE == 2) {  // o_g(beta) = o_g + beta m, m = M dc: n += beta (h + a PU + b QV), g += beta (m.d_g)
        const f3 m = mv(M, dcw);
        const f3 h = cross(m, e0), PU = cross(m, U), QV = cross(m, V);
        t[10] = make_float4(h.x, h.y, h.z, dot(m, e0));
        t[11] = make_float4(PU.x, PU.y, PU.z, dot(m, U));
        t[12] = make_float4(QV.x, QV.y, QV.z, dot(m, V));
      }
      // conservative cull against the warp's pixel box (triangle inequality,
      // 1e-3 margin): omega^2 > k^2 on the whole box -> no pixel can hit
      const f3 n0 = c0 + ac * P + bc * Q, e0c = e0 + ac * U + bc * V;
      // (MUFU square roots: 2^-22 relative, inside the 1e-3 margin)
      const float lo = rs_sqrt(dot(n0, n0)) - (ra * rs_sqrt(dot(P, P)) + rb * rs_sqrt(dot(Q, Q)));
      const float hi = rs_sqrt(dot(e0c, e0c)) + (ra * rs_sqrt(dot(U, U)) + rb * rs_sqrt(dot(V, V)));
      maybe = MODE == 2 || !(lo > 0.f && lo * lo > 1.001f * k2 * (hi * hi));  // (RS: every entry kept, as K5)
    }
    uint32_t msk = __ballot_sync(FULL, maybe);
    __syncwarp();
    while (msk) {
      const int j = __ffs(msk) - 1;
      msk &= msk - 1;
      const float4 *t = tbl + j * BW_NF;
      const float4 f0 = t[0], f1 = t[1], f2 = t[2], f3v = t[3], f4 = t[4];
      float nx = fmaf(a, f1.x, fmaf(b, f1.w, f0.x));
      float ny = fmaf(a, f1.y, fmaf(b, f2.x, f0.y));
      float nz = fmaf(a, f1.z, fmaf(b, f2.y, f0.z));
      float gb2 = 0.f;
      if (MODE == 2) {
        const float4 h = t[10], pu = t[11], qv = t[12];
        nx = fmaf(beta, fmaf(a, pu.x, fmaf(b, qv.x, h.x)), nx);
        ny = fmaf(beta, fmaf(a, pu.y, fmaf(b, qv.y, h.y)), ny);
        nz = fmaf(beta, fmaf(a, pu.z, fmaf(b, qv.z, h.z)), nz);
        gb2 = beta * fmaf(a, pu.w, fmaf(b, qv.w, h.w));
      }
      const float ex = fmaf(a, f3v.y, fmaf(b, f4.x, f2.z));
      const float ey = fmaf(a, f3v.z, fmaf(b, f4.y, f2.w));
      const float ez = fmaf(a, f3v.w, fmaf(b, f4.z, f3v.x));
      const float N = fmaf(nx, nx, fmaf(ny, ny, nz * nz));
      const float Dd = fmaf(ex, ex, fmaf(ey, ey, ez * ez));
      bool ok = !done && N <= f0.w * Dd;
      if (!__any_sync(FULL, ok)) continue;
      const float4 f5 = t[5], cc = t[6];
      const float rD = rs_rcp(Dd);  // (MUFU, as K5)
      const float w2 = N * rD;
      float pw = w2;  // (omega^2)^(n/2)
      if (gen) pw = ex2f_(khn * __log2f(w2));
      const float raw = ex2f_(gen ? fmaf(kgl, pw, f4.w) : fmaf(-0.72134752044448170f, w2, f4.w));
      const float al = fminf(c.alpha_max, raw);
      const float gdot = fmaf(a, f5.y, fmaf(b, f5.z, f5.x)) + gb2;
      const float taup = -gdot * rD, tau = taup * snorm;
      ok = ok && al >= c.alpha_min && tau > 0.f;
      float v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = 0.f;
      if (ok) {
        const float Tn = T * (1.f - al);
        if (Tn < c.t_min) {
          done = true;
          ok = false;
        } else {
          const float wgt = al * T;
          const float gi = cc.x * gr + cc.y * gg + cc.z * gb + tau * gD;
          Gpre = fmaf(wgt, gi, Gpre);
          const float dal = T * gi - (Gtot - Gpre) * rs_rcp(1.f - al);
          const bool clamped = raw > c.alpha_max;
          // d alpha / d omega^2 = -(1/2) lambda_n (n/2) (omega^2)^(n/2 - 1) alpha (n = 2: -alpha/2)
          const float dadw = gen ? (w2 > 0.f ? -0.5f * c.klam * khn * pw / w2 * raw : 0.f) : -0.5f * raw;
          const float dw2 = clamped ? 0.f : dadw * dal;
          const float dtp = wgt * gD * snorm;  // dL/dtau'
          // x_g = (d_g x n) / |d_g|^2
          const float xgx = (ey * nz - ez * ny) * rD, xgy = (ez * nx - ex * nz) * rD, xgz = (ex * ny - ey * nx) * rD;
          const float cg = dtp * rD;
          const float gox = 2.f * dw2 * xgx - cg * ex, goy = 2.f * dw2 * xgy - cg * ey, goz = 2.f * dw2 * xgz - cg * ez;
          const float4 m0 = t[7], m1 = t[8], m2 = t[9];
          // y = M^-1 x_g
          const float yx = m0.x * xgx + m0.y * xgy + m0.z * xgz;
          const float yy = m0.w * xgx + m1.x * xgy + m1.y * xgz;
          const float yz = m1.z * xgx + m1.w * xgy + m2.x * xgz;
          v[0] = gox; v[1] = goy; v[2] = goz;
          const float gx3[3] = {gox, goy, goz}, xg3[3] = {xgx, xgy, xgz}, y3[3] = {yx, yy, yz};
          const float d3v[3] = {dpw.x, dpw.y, dpw.z};
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int s = 0; s < 3; ++s) v[3 + 3 * r + s] = gx3[r] * y3[s] - cg * xg3[r] * d3v[s];
          v[12] = clamped ? 0.f : raw * ex2f_(-f4.w) * dal;  // rho = raw / sigma
          v[13] = wgt * gr; v[14] = wgt * gg; v[15] = wgt * gb;
          T = Tn;
        }
      }
      if (!__any_sync(FULL, ok)) continue;
      // reduce-scatter of the 16 values over the 32 lanes (16 + 1 shuffles
      // instead of 80): afterwards lanes 2q and 2q + 1 hold the sum of value q
      // and the 16 even lanes issue one atomic each (one instruction)
      {
        const float s = reduce16(v, lane);
        // 32.32 fixed point (cvt saturates beyond +-2^31): deterministic sums
        if ((lane & 1) == 0)
          atomicAdd(reinterpret_cast<unsigned long long *>(B.acc + (size_t)16 * __float_as_uint(f5.w) + (lane >> 1)),
                    (unsigned long long)__float2ll_rn(s * (float)GUT_BWD_FIX));
      }
    }
  }
}

// Per Gaussian: dL/dmu = -M^T sum dL/do_g; dL/ds, dL/dq from dL/dM; dL/dsigma;
// SH from the colour gradient at the forward's direction (clamped channels: 0).
__global__ __launch_bounds__(256) void backward_finish_kernel(DevCam c, SceneDev s, BwdBufs B) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= s.n) return;
  const int nc = (s.sh_degree + 1) * (s.sh_degree + 1);
  float *gm = B.d_means + 3 * i, *gq = B.d_rots + 4 * i, *gs = B.d_scales + 3 * i, *gsh = B.d_sh + 3 * nc * i;
  const bool vis = B.tiles[i] != 0;
  float acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = vis ? (float)((double)B.acc[16 * i + q] * (1.0 / GUT_BWD_FIX)) : 0.f;
  const float4 po = s.pos_opa[i], ro = s.rot[i], sc = s.scale[i];
  const float qn = sqrtf(ro.x * ro.x + ro.y * ro.y + ro.z * ro.z + ro.w * ro.w);
  const float qw = ro.x / qn, qx = ro.y / qn, qy = ro.z / qn, qz = ro.w / qn;
  const float R[9] = {1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qw * qz), 2 * (qx * qz + qw * qy),
                      2 * (qx * qy + qw * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qw * qx),
                      2 * (qx * qz - qw * qy), 2 * (qy * qz + qw * qx), 1 - 2 * (qx * qx + qy * qy)};
  const float sv[3] = {sc.x, sc.y, sc.z};
  float gR[9];
  for (int j = 0; j < 3; ++j) {  // dL/dmu_j = -sum_i M_ij go_i, M_ij = R_ji / s_i
    float m = 0.f;
    for (int r = 0; r < 3; ++r) m += (R[3 * j + r] / sv[r]) * acc[r];
    gm[j] = vis ? -m : 0.f;
  }
  const double tc = B.t0 ? (double)B.t0[i] : 0.0;
  const d3 dw = mkd(po.x, po.y, po.z) - mkd(c.c0[0] + tc * c.dc[0], c.c0[1] + tc * c.dc[1], c.c0[2] + tc * c.dc[2]);
  if (B.densify) {  // PAPER L218 (reading R32): |dL/dmu| / (distance / 2)
    const float gn = sqrtf(gm[0] * gm[0] + gm[1] * gm[1] + gm[2] * gm[2]);
    B.densify[i] = gn / (0.5f * (float)sqrt(dot(dw, dw)));
  }
  for (int r = 0; r < 3; ++r) {
    float t = 0.f;
    for (int j = 0; j < 3; ++j) {
      const float G = acc[3 + 3 * r + j];
      t += G * (R[3 * j + r] / sv[r]);
      gR[3 * j + r] = G / sv[r];
    }
    gs[r] = vis ? -t / sv[r] : 0.f;
  }
  const float dRw[9] = {0, -2 * qz, 2 * qy, 2 * qz, 0, -2 * qx, -2 * qy, 2 * qx, 0};
  const float dRx[9] = {0, 2 * qy, 2 * qz, 2 * qy, -4 * qx, -2 * qw, 2 * qz, 2 * qw, -4 * qx};
  const float dRy[9] = {-4 * qy, 2 * qx, 2 * qw, 2 * qx, 0, 2 * qz, -2 * qw, 2 * qz, -4 * qy};
  const float dRz[9] = {-4 * qz, -2 * qw, 2 * qx, 2 * qw, -4 * qz, 2 * qy, 2 * qx, 2 * qy, 0};
  float g4[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k = 0; k < 9; ++k) {
    g4[0] += gR[k] * dRw[k]; g4[1] += gR[k] * dRx[k]; g4[2] += gR[k] * dRy[k]; g4[3] += gR[k] * dRz[k];
  }
  const float qh[4] = {qw, qx, qy, qz};
  const float pr = g4[0] * qw + g4[1] * qx + g4[2] * qy + g4[3] * qz;
  for (int k = 0; k < 4; ++k) gq[k] = vis ? (g4[k] - qh[k] * pr) / qn : 0.f;
  B.d_opac[i] = acc[12];
  if (B.d_rgb) { B.d_rgb[3 * i] = acc[13]; B.d_rgb[3 * i + 1] = acc[14]; B.d_rgb[3 * i + 2] = acc[15]; }
  // SH (the forward's direction normalize(mu - c(t0)), t0 = mu's shutter time)
  const float4 col = vis ? B.payload[(size_t)GUT_PAYLOAD_F4 * i + 4] : make_float4(0.f, 0.f, 0.f, 0.f);
  const f3 d = tof((1.0 / sqrt(dot(dw, dw))) * dw);
  const float x = d.x, y = d.y, z = d.z, xx = x * x, yy = y * y, zz = z * z;
  float Y[16];
  Y[0] = 0.28209479177387814f;
  Y[1] = -0.4886025119029199f * y; Y[2] = 0.4886025119029199f * z; Y[3] = -0.4886025119029199f * x;
  Y[4] = 1.0925484305920792f * x * y; Y[5] = -1.0925484305920792f * y * z;
  Y[6] = 0.31539156525252005f * (2.f * zz - xx - yy); Y[7] = -1.0925484305920792f * x * z;
  Y[8] = 0.5462742152960396f * (xx - yy);
  Y[9] = -0.5900435899266435f * y * (3.f * xx - yy); Y[10] = 2.890611442640554f * x * y * z;
  Y[11] = -0.4570457994644658f * y * (4.f * zz - xx - yy);
  Y[12] = 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
  Y[13] = -0.4570457994644658f * x * (4.f * zz - xx - yy); Y[14] = 1.445305721320277f * z * (xx - yy);
  Y[15] = -0.5900435899266435f * x * (xx - 3.f * yy);
  const float gc[3] = {col.x > 0.f ? acc[13] : 0.f, col.y > 0.f ? acc[14] : 0.f, col.z > 0.f ? acc[15] : 0.f};
  for (int k = 0; k < nc; ++k)
    for (int ch = 0; ch < 3; ++ch) gsh[3 * k + ch] = gc[ch] * Y[k];
}

void launch_backward(const DevCam &cam, const SceneDev &s, const BwdBufs &b, cudaStream_t st) {
  if (b.t0) launch_centre_times(cam, s, const_cast<float *>(b.t0), st);
  cudaMemsetAsync(b.acc, 0, (size_t)16 * s.n * sizeof(long long), st);
  // queue-1 order of the tiles, longest list first (plan kernels, one unit per tile)
  cudaMemsetAsync(b.counters + CNT_PLAN_HIST, 0, 1024 * sizeof(uint32_t), st);
  launch_plan(b.ranges, cam.n_tiles, 1 << 30, 1, b.seg_base, b.order, b.counters, st, 1);
  if (cam.n_tiles > 0) {
    if (cam.shutter != SH_GLOBAL) {
      constexpr size_t smem = sizeof(float4) * 8 * 32 * BwNF<2>::v;
      static std::once_flag once[GUT_MAX_DEVICES];  // (a per-device attribute)
      int dev = 0;
      cudaGetDevice(&dev);
      std::call_once(once[min(dev, GUT_MAX_DEVICES - 1)], [] {
        cudaFuncSetAttribute(backward_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      });
      backward_kernel<2><<<cam.n_tiles, 256, smem, st>>>(cam, b);
    } else {
      backward_kernel<0><<<cam.n_tiles, 256, sizeof(float4) * 8 * 32 * BwNF<0>::v, st>>>(cam, b);
    }
  }
  if (s.n > 0) backward_finish_kernel<<<(unsigned)((s.n + 255) / 256), 256, 0, st>>>(cam, s, b);
}

}  // namespace gut
