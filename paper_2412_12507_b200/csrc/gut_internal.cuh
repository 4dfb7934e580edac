// gut_internal.cuh — device-side types and helpers shared by the sm_100a kernels.
// Product code: never includes anything under oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define GUT_TILE 16
#define GUT_TILE_PX (GUT_TILE * GUT_TILE)  // pixels per tile (ray LUT, look-back status, partials)
#define GUT_BLEND_NP 2  // K5 pixels per lane
#define GUT_BLEND_WARPS (GUT_TILE_PX / (32 * GUT_BLEND_NP))  // K5 work units per tile (8x8 pixel blocks)
#define GUT_KBUF_UNITS (GUT_TILE_PX / 32)  // K5 k-buffer variant: work units per tile (8x4 blocks, 1 pixel per lane)
#ifndef GUT_BLEND_CTA
#define GUT_BLEND_CTA 256  // K5 threads per CTA (independent warps; sized for the register budget)
#endif
#ifndef GUT_BLEND_CTAS
#define GUT_BLEND_CTAS 2  // K5 resident CTAs per SM (register budget 65536 / (256 x 2) = 128)
#endif
#define GUT_PAYLOAD_F4 5  // K1 -> K5 blend payload per Gaussian, in float4 (k1_project.cu finish_gaussian)
#ifndef GUT_SORT_THREADS
#define GUT_SORT_THREADS 512
#endif
#ifndef GUT_SORT_ITEMS
#define GUT_SORT_ITEMS 8
#endif
#define GUT_SORT_PART (GUT_SORT_THREADS * GUT_SORT_ITEMS)  // 4096 keys per onesweep partition
#define GUT_EMIT_THREADS 256
#define GUT_EMIT_ITEMS 4
#define GUT_EMIT_PART (GUT_EMIT_THREADS * GUT_EMIT_ITEMS)  // 1024 Gaussians per emit partition
#define GUT_CULLED_KEY 0xFFFFFFFFu

namespace gut {

enum { CAM_PINHOLE = 0, CAM_OPENCV = 1, CAM_FISHEYE = 2, CAM_ORTHO = 3 };
enum { SH_GLOBAL = 0, SH_T2B = 1, SH_L2R = 2, SH_B2T = 3, SH_R2L = 4 };

// Per-view camera + options, passed by value as a kernel parameter.
struct DevCam {
  int model, width, height, shutter;
  int tiles_x, tiles_y, n_tiles, tile_cull;
  // intrinsics (fp64 master copy; fp32 copies for K1)
  double fx, fy, cx, cy, k[6], p[2], fov;
  float fxf, fyf, cxf, cyf, kf[6], pf[2], fovf;
  float inv_wf, inv_hf;  // 1 / width, 1 / height (rolling-shutter row time)
  // pose: R0 = camera->world at t=0 (row-major), c0 = centre at t=0,
  // dc = c1 - c0, phi = axis-angle (body frame) of R0^T R1 (slerp = R0 Exp(t phi))
  double R0[9], c0[3], dc[3], phi_axis[3], phi_angle;
  float R0f[9], dcf[3], phi_axisf[3], phi_anglef;
  // UT weights (Eq. 7-8) and thresholds
  float gamma;        // sqrt(3 + lambda)
  float wmu0, wmui, wsig0, wsigi;
  float alpha_min, alpha_max, t_min, dilation, near_plane;
  float rs_tol_px;
  int rs_max_iter;
  float bg[3];
  int kbuf;  // 0 = "Ours" (tile order); 1..16 = "Ours (sorted)" per-ray k-buffer size
  int kdeg;     // Supp. A generalized Gaussian degree n (2 = Gaussian)
  float klam;   // lambda_n = 3^(2 - n)
};

// ---------------------------------------------------------------- small math
struct f3 { float x, y, z; };
struct d3 { double x, y, z; };

__host__ __device__ __forceinline__ f3 mk(float x, float y, float z) { return {x, y, z}; }
__host__ __device__ __forceinline__ d3 mkd(double x, double y, double z) { return {x, y, z}; }
__host__ __device__ __forceinline__ f3 operator+(f3 a, f3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__host__ __device__ __forceinline__ f3 operator-(f3 a, f3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__host__ __device__ __forceinline__ f3 operator*(float s, f3 a) { return {s * a.x, s * a.y, s * a.z}; }
__host__ __device__ __forceinline__ float dot(f3 a, f3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__host__ __device__ __forceinline__ f3 cross(f3 a, f3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__host__ __device__ __forceinline__ d3 operator+(d3 a, d3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__host__ __device__ __forceinline__ d3 operator-(d3 a, d3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__host__ __device__ __forceinline__ d3 operator*(double s, d3 a) { return {s * a.x, s * a.y, s * a.z}; }
__host__ __device__ __forceinline__ double dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__host__ __device__ __forceinline__ d3 cross(d3 a, d3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__host__ __device__ __forceinline__ f3 tof(d3 a) { return {(float)a.x, (float)a.y, (float)a.z}; }
__host__ __device__ __forceinline__ d3 tod(f3 a) { return {(double)a.x, (double)a.y, (double)a.z}; }
// row-major 3x3 times vector / transposed times vector
template <class M, class V>
__host__ __device__ __forceinline__ V mv(const M *m, V v) {
  return {m[0] * v.x + m[1] * v.y + m[2] * v.z, m[3] * v.x + m[4] * v.y + m[5] * v.z,
          m[6] * v.x + m[7] * v.y + m[8] * v.z};
}
template <class M, class V>
__host__ __device__ __forceinline__ V mtv(const M *m, V v) {
  return {m[0] * v.x + m[3] * v.y + m[6] * v.z, m[1] * v.x + m[4] * v.y + m[7] * v.z,
          m[2] * v.x + m[5] * v.y + m[8] * v.z};
}

// Rodrigues: R = I + sin(a) [u]x + (1 - cos(a)) [u]x^2, row-major (fp32)
// (rolling-shutter rotations are tiny: |angle| ~ readout x angular rate; the
// Taylor branch is exact to the precision and avoids the sincos range reduction)
__device__ __forceinline__ void rodrigues(f3 u, float ang, float R[9]) {
  float s, c, t;
  if (fabsf(ang) < 0.03f) {
    const float a2 = ang * ang;
    s = ang * (1.f - a2 * (1.f / 6.f) * (1.f - a2 * 0.05f));
    t = 0.5f * a2 * (1.f - a2 * (1.f / 12.f));  // 1 - cos without cancellation
    c = 1.f - t;
  } else {
    sincosf(ang, &s, &c);
    t = 1.f - c;
  }
  R[0] = c + t * u.x * u.x;       R[1] = t * u.x * u.y - s * u.z; R[2] = t * u.x * u.z + s * u.y;
  R[3] = t * u.x * u.y + s * u.z; R[4] = c + t * u.y * u.y;       R[5] = t * u.y * u.z - s * u.x;
  R[6] = t * u.x * u.z - s * u.y; R[7] = t * u.y * u.z + s * u.x; R[8] = c + t * u.z * u.z;
}
__device__ __forceinline__ void rodrigues_d(d3 u, double ang, double R[9]) {
  double s, c, t;
  if (fabs(ang) < 0.01) {
    const double a2 = ang * ang;
    s = ang * (1.0 - a2 / 6.0 * (1.0 - a2 / 20.0 * (1.0 - a2 / 42.0)));
    t = 0.5 * a2 * (1.0 - a2 / 12.0 * (1.0 - a2 / 30.0 * (1.0 - a2 / 56.0)));
    c = 1.0 - t;
  } else {
    sincos(ang, &s, &c);
    t = 1.0 - c;
  }
  R[0] = c + t * u.x * u.x;       R[1] = t * u.x * u.y - s * u.z; R[2] = t * u.x * u.z + s * u.y;
  R[3] = t * u.x * u.y + s * u.z; R[4] = c + t * u.y * u.y;       R[5] = t * u.y * u.z - s * u.x;
  R[6] = t * u.x * u.z - s * u.y; R[7] = t * u.y * u.z + s * u.x; R[8] = c + t * u.z * u.z;
}
template <class T>
__host__ __device__ __forceinline__ void matmul3(const T *A, const T *B, T *C) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) C[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
}

// ----------------------------------------------------------- tile row spans
// Ellipse-tile test in closed form per tile row (StopThePop-style culling,
// PAPER L216): E = {v : (v - vmu)^T Sigma'^-1 (v - vmu) <= k2}.  The band
// y in [16 ty, 16 ty + 16] cuts E in a convex set whose x-extent is either the
// ellipse's extreme point (if it lies in the band) or the chord at the band
// edge nearest to it.  Tiles whose closed x-range meets that extent are kept.
// K1 (counting) and K2 (emission) call this same function, so counts and
// emitted keys agree bit for bit.
// Precision: fp32 for ordinary Gaussians; "wide" Gaussians (sigma points more
// than 2048 px from the principal point, e.g. edge-on splats grazing the near
// plane) run the UT and this test in fp64 (EllT<double>), because fp32 pixel
// coordinates there have an ulp above the 1e-3 px binning band.
template <class Real>
struct EllT {
  Real vx, vy, cxx, cxy, cyy, k2;
  int x0, y0, x1, y1;  // clamped tile rectangle
};
using Ell = EllT<float>;
using EllD = EllT<double>;

// fp32: MUFU square root / reciprocal (relative error ~2^-22, far inside the
// 1e-3 px binning band; K1 and K2 share them, so counts still match keys)
__device__ __forceinline__ float rs_sqrt(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ double rs_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float rs_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ double rs_rcp(double x) { return 1.0 / x; }

// Row-invariant part of the per-tile-row x-extent of the ellipse (computed
// once per Gaussian; K1's counts / masks and K2's key emission both go
// through row_span_setup + row_span_at, so they agree bit for bit).
template <class Real> struct RowSpan {
  Real hy, hx, ystar, slope, cond, icyy;
};
template <class Real>
__device__ __forceinline__ RowSpan<Real> row_span_setup(const EllT<Real> &e) {
  RowSpan<Real> r;
  r.hy = rs_sqrt(e.k2 * e.cyy);
  const Real icxx = rs_rcp(e.cxx);
  r.icyy = rs_rcp(e.cyy);
  r.hx = rs_sqrt(e.k2 * e.cxx);
  r.ystar = e.cxy * rs_sqrt(e.k2 * icxx);  // dy of the rightmost point (leftmost at -ystar)
  r.slope = e.cxy * r.icyy;
  r.cond = fmax(e.cxx - e.cxy * r.slope, (Real)0);  // det / cyy
  return r;
}
template <class Real>
__device__ __forceinline__ void row_span_at(const EllT<Real> &e, const RowSpan<Real> &r, int ty, int tile_cull,
                                            int &lo, int &hi) {
  if (tile_cull == 0) { lo = e.x0; hi = e.x1; return; }
  const Real zero = 0, itile = (Real)(1.0 / GUT_TILE);
  Real a = fmax((Real)(GUT_TILE * ty) - e.vy, -r.hy);
  Real b = fmin((Real)(GUT_TILE * ty + GUT_TILE) - e.vy, r.hy);
  if (a > b) { lo = 1; hi = 0; return; }
  Real xr, xl;
  if (r.ystar >= a && r.ystar <= b) xr = r.hx;
  else {
    Real yy = r.ystar < a ? a : b;
    xr = r.slope * yy + rs_sqrt(fmax(r.cond * (e.k2 - yy * yy * r.icyy), zero));
  }
  if (-r.ystar >= a && -r.ystar <= b) xl = -r.hx;
  else {
    Real yy = -r.ystar < a ? a : b;
    xl = r.slope * yy - rs_sqrt(fmax(r.cond * (e.k2 - yy * yy * r.icyy), zero));
  }
  Real XL = e.vx + xl, XR = e.vx + xr;
  XL = fmin(fmax(XL, (Real)-1e7), (Real)1e7);
  XR = fmin(fmax(XR, (Real)-1e7), (Real)1e7);
  int l = (int)ceil(XL * itile) - 1;
  int h = (int)floor(XR * itile);
  lo = max(l, e.x0);
  hi = min(h, e.x1);
}
template <class Real>
__device__ __forceinline__ void row_span(const EllT<Real> &e, int ty, int tile_cull, int &lo, int &hi) {
  row_span_at(e, row_span_setup(e), ty, tile_cull, lo, hi);
}

template <class Real>
__device__ __forceinline__ int ell_tile_count(const EllT<Real> &e, int tile_cull) {
  if (tile_cull == 0) return (e.x1 - e.x0 + 1) * (e.y1 - e.y0 + 1);
  const RowSpan<Real> rs = row_span_setup(e);
  int n = 0;
  for (int ty = e.y0; ty <= e.y1; ++ty) {
    int lo, hi;
    row_span_at(e, rs, ty, tile_cull, lo, hi);
    n += max(hi - lo + 1, 0);
  }
  return n;
}

// K1 -> K2 tile code per Gaussian: 0 = culled; bits 31, 30 clear: tile
// rectangle of at most 3x3 tiles, bits 0-8 = hit mask (row-major over the
// rectangle), bits 9-19 = x0, bits 20-29 = y0; bit 30 set: at most 4x4 tiles
// (x0, y0 < 128), bits 0-15 = hit mask, bits 16-22 = x0, bits 23-29 = y0;
// bit 31 set: bits 0-30 = tile count (K2 walks the rows of the ellipse record).  Counts and masks come from the same
// row_span() calls, so K2 emits exactly the counted keys.
template <class Real>
__device__ __forceinline__ uint32_t ell_tile_code(const EllT<Real> &e, int tile_cull) {
  const int w = e.x1 - e.x0 + 1, h = e.y1 - e.y0 + 1;
  if (w <= 3 && h <= 3 && e.x0 < 2048 && e.y0 < 1024) {
    const RowSpan<Real> rs = row_span_setup(e);
    uint32_t mask = 0;
    for (int r = 0; r < h; ++r) {
      int lo, hi;
      row_span_at(e, rs, e.y0 + r, tile_cull, lo, hi);
      for (int x = lo; x <= hi; ++x) mask |= 1u << (3 * r + (x - e.x0));
    }
    return mask ? (mask | ((uint32_t)e.x0 << 9) | ((uint32_t)e.y0 << 20)) : 0u;
  }
  if (w <= 4 && h <= 4 && e.x0 < 128 && e.y0 < 128) {  // 4x4 hit mask (bit 30)
    const RowSpan<Real> rs = row_span_setup(e);
    uint32_t mask = 0;
    for (int r = 0; r < h; ++r) {
      int lo, hi;
      row_span_at(e, rs, e.y0 + r, tile_cull, lo, hi);
      for (int x = lo; x <= hi; ++x) mask |= 1u << (4 * r + (x - e.x0));
    }
    return mask ? (0x40000000u | mask | ((uint32_t)e.x0 << 16) | ((uint32_t)e.y0 << 23)) : 0u;
  }
  const int n = ell_tile_count(e, tile_cull);
  return n > 0 ? (0x80000000u | (uint32_t)min(n, 0x7FFFFFFF)) : 0u;
}
__device__ __forceinline__ uint32_t code_count(uint32_t code) {
  return (code >> 31) ? (code & 0x7FFFFFFFu)
                      : (uint32_t)__popc(code & ((code >> 30) ? 0xFFFFu : 0x1FFu));
}

__device__ __forceinline__ Ell load_ell(const float4 *ell, uint32_t g) {
  float4 a = ell[2 * g], b = ell[2 * g + 1];
  Ell e;
  e.vx = a.x; e.vy = a.y; e.cxx = a.z; e.cxy = a.w; e.cyy = b.x; e.k2 = b.y;
  uint32_t r0 = __float_as_uint(b.z), r1 = __float_as_uint(b.w);
  e.x0 = (int)(r0 & 0xFFFF); e.y0 = (int)(r0 >> 16); e.x1 = (int)(r1 & 0xFFFF); e.y1 = (int)(r1 >> 16);
  return e;
}

// ------------------------------------------------------ decoupled look-back
// 64-bit status words: [63:32] epoch, [31:30] flag (1 = aggregate, 2 = inclusive),
// [29:0] count.  A word from an older epoch reads as "not ready", so the
// status arrays never need clearing between passes / renders.
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long mk_status(uint32_t epoch, uint32_t flag, uint32_t cnt) {
  return ((unsigned long long)epoch << 32) | ((unsigned long long)flag << 30) | (cnt & 0x3FFFFFFFu);
}
// Split form (k3_sort.cu): publish the partition's aggregate as soon as it is
// known, then walk back later with a wider window of predecessors in flight.
// A wave of CTAs publishes aggregates at about the same time, so a partition
// j places into a wave sums ~j aggregates before it meets an inclusive word:
// the window width sets the number of L2 round trips of that walk.
__device__ __forceinline__ void lookback_publish(unsigned long long *status, int stride, int part, int col,
                                                 uint32_t mine, uint32_t epoch) {
  st_relaxed(&status[(size_t)part * stride + col], mk_status(epoch, part == 0 ? 2 : 1, mine));
}
template <int WIN>
__device__ __forceinline__ uint32_t lookback_walk(unsigned long long *status, int stride, int part, int col,
                                                  uint32_t mine, uint32_t epoch) {
  if (part == 0) return 0;
  uint32_t sum = 0;
  int j = part - 1;
  while (true) {
    unsigned long long w[WIN];
#pragma unroll
    for (int q = 0; q < WIN; ++q) w[q] = j - q >= 0 ? ld_relaxed(&status[(size_t)(j - q) * stride + col]) : 0ull;
    int used = 0;
    bool fin = false;
#pragma unroll
    for (int q = 0; q < WIN; ++q) {
      if (used != q || j - q < 0) break;
      const unsigned long long s = w[q];
      const uint32_t flag = (uint32_t)(s >> 30) & 3u;
      if ((uint32_t)(s >> 32) != epoch || flag == 0) break;  // not ready yet: reload from here
      sum += (uint32_t)s & 0x3FFFFFFFu;
      ++used;
      if (flag == 2) { fin = true; break; }
    }
    if (fin) break;
    j -= used;
  }
  st_relaxed(&status[(size_t)part * stride + col], mk_status(epoch, 2, sum + mine));
  return sum;
}


}  // namespace gut
