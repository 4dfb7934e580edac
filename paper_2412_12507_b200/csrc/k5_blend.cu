// k5_blend.cu — K5: per-pixel front-to-back compositing with the 3D
// max-response (the paper's "Render"), sm_100a.
//
// PAPER Eq. 5 (L115-121): c = sum_i c_i alpha_i prod_{j<i}(1 - alpha_j),
// alpha_i = sigma_i rho_i(o + tau d); Eq. 11 (L195-200): tau_max =
// -o_g.d_g / d_g.d_g with o_g = S^-1 R^T (o - mu), d_g = S^-1 R^T d, and the
// response at tau_max is exp(-omega^2/2), omega^2 = ||o_g x d_g||^2/||d_g||^2
// (Supp. B, L506).  Order = the tile's global depth order (L208).
//
// Precision: o_g x d_g cancels catastrophically
// in fp32 for small, distant Gaussians, so every pixel ray is written relative
// to a per-tile anchor ray (D, O) as
//   d' = D + a T1 + b T2  (central cameras; a, b = tangent-plane offsets),
//   o  = O + a T1 + b T2  (orthographic),   o = O + beta dc  (rolling shutter),
// and per (tile, entry) the large, cancelling part c0 = o_g x (M D) is formed
// in fp64 while the entry is staged into shared memory.  Per (pixel, entry):
//   n = c0 + a P + b Q [+ beta (h + a PU + b QV)],  e = e0 + a U + b V
//   omega^2 = |n|^2 / |e|^2,   reject before MUFU if |n|^2 > k^2 |e|^2
// with k^2 = 2 ln(sigma / alpha_min) (alpha >= alpha_min <=> omega^2 <= k^2).
//
// Load balance: tile lists are split into segments of `seg` entries; every
// (tile, segment) is one CTA, all running concurrently.  Front-to-back
// blending is associative ((C1,T1) over (C2,T2) = (C1 + T1 C2, T1 T2)) except
// for the termination rule, so each segment first runs speculatively from
// T = 1 (exact for segment 0), publishes its per-pixel transmittance product
// P_s and resolves the product of its predecessors T_pre by decoupled
// look-back.  If the pixel survives the segment (no local termination and
// T_pre P_s >= T_min) no entry of the segment can have terminated it in the
// sequential loop (T is monotone) and its exact contribution is T_pre times
// the speculative sums; otherwise the segment is re-run from T_pre with the
// termination rule (each pixel re-runs at most the one segment where it
// terminates).  Products travel as fixed-point -log2 sums so prefixes are
// bitwise deterministic.  The last segment CTA of a tile (atomic counter)
// sums the partial results in segment order (deterministic) and writes the
// pixels.
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

// (warp block w, lane) -> pixel of a 16x16 tile: 8x4 pixel blocks (coherent ballots)
__device__ __forceinline__ void tile_pixel(int tile, int tiles_x, int w, int lane, int &px, int &py) {
  px = (tile % tiles_x) * GUT_TILE + (w & 1) * 8 + (lane & 7);
  py = (tile / tiles_x) * GUT_TILE + (w >> 1) * 4 + (lane >> 3);
}

// ---------------------------------------------------------------- rays (a5)
// Per tile: fp64 rays of its pixels, anchor = mean valid direction (central)
// or mean valid origin (orthographic); per pixel the fp32 offsets (a, b), the
// distance factor snorm = |d'| (0 marks an invalid pixel) and, for rolling
// shutter, beta = t_pixel - t_anchor.  MODE 0/1: camera frame (depends on the
// intrinsics only, cached by the host); MODE 2: world frame (per view).
template <int MODE>
__global__ __launch_bounds__(GUT_TILE_PX) void rays_kernel(DevCam c, float4 *__restrict__ pix,
                                                                 TileAnchor *__restrict__ anchors) {
  __shared__ double s_red[8][4];
  __shared__ double s_a[13];
  const int tile = blockIdx.x;
  const int tx = tile % c.tiles_x, ty = tile / c.tiles_x;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int px, py;
  tile_pixel(tile, c.tiles_x, w, lane, px, py);
  const bool inside = px < c.width && py < c.height;
  const double u = px + 0.5, v = py + 0.5;
  d3 dcam = mkd(0, 0, 1), ocam = mkd(0, 0, 0);
  bool valid = inside && unproject(c, u, v, dcam, ocam);
  const double tp = pixel_time(c, u, v);
  d3 dw = dcam;
  if (MODE == 2 && valid) {
    double Rt[9], Rw[9];
    rodrigues_d(mkd(c.phi_axis[0], c.phi_axis[1], c.phi_axis[2]), tp * c.phi_angle, Rt);
    matmul3(c.R0, Rt, Rw);
    dw = mv(Rw, dcam);
  }
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
    d3 D, O, T1, T2;
    double ta = 0;
    if (MODE == 1) {
      O = (cnt > 0 ? 1.0 / cnt : 0.0) * s;  // mean camera-frame origin offset
      D = mkd(0, 0, 1); T1 = mkd(1, 0, 0); T2 = mkd(0, 1, 0);
    } else {
      D = cnt > 0 ? normalize_d(s) : mkd(0, 0, 1);
      d3 h = fabs(D.x) < 0.6 ? mkd(1, 0, 0) : (fabs(D.y) < 0.6 ? mkd(0, 1, 0) : mkd(0, 0, 1));
      T1 = normalize_d(h - dot(h, D) * D);
      T2 = cross(D, T1);
      O = mkd(c.c0[0], c.c0[1], c.c0[2]);
      if (MODE == 2) {
        double uc = fmin(fmax(tx * GUT_TILE + 8.0, 0.5), c.width - 0.5);
        double vc = fmin(fmax(ty * GUT_TILE + 8.0, 0.5), c.height - 0.5);
        ta = pixel_time(c, uc, vc);
        O = mkd(c.c0[0] + ta * c.dc[0], c.c0[1] + ta * c.dc[1], c.c0[2] + ta * c.dc[2]);
      }
    }
    double vals[13] = {D.x, D.y, D.z, T1.x, T1.y, T1.z, T2.x, T2.y, T2.z, O.x, O.y, O.z, ta};
    for (int k = 0; k < 13; ++k) s_a[k] = vals[k];
    TileAnchor A;
    for (int k = 0; k < 3; ++k) { A.D[k] = vals[k]; A.T1[k] = vals[3 + k]; A.T2[k] = vals[6 + k]; A.O[k] = vals[9 + k]; }
    A.ta = ta; A.pad[0] = A.pad[1] = A.pad[2] = 0;
    anchors[tile] = A;
  }
  __syncthreads();
  float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
  if (valid) {
    const d3 D = mkd(s_a[0], s_a[1], s_a[2]), T1 = mkd(s_a[3], s_a[4], s_a[5]), T2 = mkd(s_a[6], s_a[7], s_a[8]);
    if (MODE == 1) {
      out = make_float4((float)(ocam.x - s_a[9]), (float)(ocam.y - s_a[10]), 1.f, 0.f);
    } else {
      const double den = dot(dw, D);
      if (den > 0) {
        out.x = (float)(dot(dw, T1) / den);
        out.y = (float)(dot(dw, T2) / den);
        out.z = (float)(1.0 / den);
        out.w = MODE == 2 ? (float)(tp - s_a[12]) : 0.f;
      }
    }
  }
  pix[(size_t)tile * GUT_TILE_PX + threadIdx.x] = out;
  // Per 8x8 block (MODE 0/1): least-squares affine lattice of the fp32 offsets
  // of its valid pixels, and the largest residual against the fp32-rounded
  // coefficients.  K5's candidate masks bound a Gaussian's footprint on this
  // lattice and widen it by the residual (blend: entry_mask).
  __shared__ float2 s_ab[GUT_TILE_PX];
  s_ab[threadIdx.x] = make_float2(out.x, out.z > 0.f ? out.y : __int_as_float(0x7fc00000));  // NaN b: invalid
  __syncthreads();
  if (threadIdx.x < 4) {
    const int B = threadIdx.x;
    float *fit = anchors[tile].fit[B];
    auto idx = [&](int cx, int ry) {
      const int y = (B >> 1) * 8 + ry;
      return (((B & 1) | ((y >> 2) << 1)) << 5) + (ry & 3) * 8 + cx;
    };
    double n = 0, sx = 0, sy = 0, sxx = 0, sxy = 0, syy = 0, sa = 0, sxa = 0, sya = 0, sb = 0, sxb = 0, syb = 0;
    for (int ry = 0; ry < 8; ++ry)
      for (int cx = 0; cx < 8; ++cx) {
        const float2 v = s_ab[idx(cx, ry)];
        if (MODE == 2 || v.y != v.y) continue;
        const double x = cx, y = ry, a = v.x, b = v.y;
        n += 1; sx += x; sy += y; sxx += x * x; sxy += x * y; syy += y * y;
        sa += a; sxa += x * a; sya += y * a; sb += b; sxb += x * b; syb += y * b;
      }
    // normal equations [n sx sy; sx sxx sxy; sy sxy syy] c = rhs (Cramer)
    const double c00 = sxx * syy - sxy * sxy, c01 = sy * sxy - sx * syy, c02 = sx * sxy - sy * sxx;
    const double det = n * c00 + sx * c01 + sy * c02;
    double ca[3] = {0, 0, 0}, cb[3] = {0, 0, 0};
    bool ok = n > 0;
    if (n >= 3 && det > 1e-6 * n * n * n) {
      const double c11 = n * syy - sy * sy, c12 = sx * sy - n * sxy, c22 = n * sxx - sx * sx;
      ca[0] = (c00 * sa + c01 * sxa + c02 * sya) / det;
      ca[1] = (c01 * sa + c11 * sxa + c12 * sya) / det;
      ca[2] = (c02 * sa + c12 * sxa + c22 * sya) / det;
      cb[0] = (c00 * sb + c01 * sxb + c02 * syb) / det;
      cb[1] = (c01 * sb + c11 * sxb + c12 * syb) / det;
      cb[2] = (c02 * sb + c12 * sxb + c22 * syb) / det;
    } else if (ok) {  // collinear / too few valid pixels: a constant lattice (loose, still conservative)
      ca[0] = sa / n;
      cb[0] = sb / n;
    }
    float fa[3], fb[3];
    for (int q = 0; q < 3; ++q) { fa[q] = (float)ca[q]; fb[q] = (float)cb[q]; }
    double ra = 0, rb = 0;
    for (int ry = 0; ry < 8; ++ry)
      for (int cx = 0; cx < 8; ++cx) {
        const float2 v = s_ab[idx(cx, ry)];
        if (!ok || v.y != v.y) continue;
        ra = fmax(ra, fabs((double)v.x - ((double)fa[0] + (double)fa[1] * cx + (double)fa[2] * ry)));
        rb = fmax(rb, fabs((double)v.y - ((double)fb[0] + (double)fb[1] * cx + (double)fb[2] * ry)));
      }
    const float inf = __int_as_float(0x7f800000);
    const bool use = ok && MODE != 2 && isfinite(ra) && isfinite(rb);
    fit[0] = fa[0]; fit[1] = fa[1]; fit[2] = fa[2]; fit[3] = use ? __double2float_ru(ra * (1 + 1e-6)) : inf;
    fit[4] = fb[0]; fit[5] = fb[1]; fit[6] = fb[2]; fit[7] = use ? __double2float_ru(rb * (1 + 1e-6)) : inf;
  }
}

void launch_rays(const DevCam &cam, float4 *pix, TileAnchor *anchors, cudaStream_t st) {
  const unsigned blocks = (unsigned)cam.n_tiles;
  if (cam.model == CAM_ORTHO) rays_kernel<1><<<blocks, GUT_TILE_PX, 0, st>>>(cam, pix, anchors);
  else if (cam.shutter != SH_GLOBAL) rays_kernel<2><<<blocks, GUT_TILE_PX, 0, st>>>(cam, pix, anchors);
  else rays_kernel<0><<<blocks, GUT_TILE_PX, 0, st>>>(cam, pix, anchors);
}

// ---------------------------------------------------------------- plan
// Per tile: S_t = max(1, ceil(len / seg)) segments; slots are numbered
// tile-major (seg_base[t] + s).  The unit of work is one warp's 8x4 pixel
// block of a tile (unit u = 8 t + w) over one segment: warps never wait for
// each other.  Per unit, min(S_t, window) segments are granted up front
// (queue 1, tiles in decreasing list length = longest chains first); a
// completing segment s with pixels still alive grants further segments
// (queue 2, served first).  The segment index is assigned when a warp takes a
// unit from a queue (next_s[u]++), so a unit's segments start in order and
// the look-back only ever waits on segments that are already running.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *s_w, uint32_t &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t y = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += z;
    }
    s_w[lane] = y;
  }
  __syncthreads();
  const uint32_t r = (w > 0 ? s_w[w - 1] : 0) + x - v;
  total = s_w[31];
  __syncthreads();
  return r;
}

// queue-1 order bucket: decreasing list length (log scale, 1024 buckets)
__device__ __forceinline__ uint32_t len_bucket(uint32_t len) {
  const uint32_t key = len == 0 ? 0u : min(1023u, (uint32_t)(log2f((float)len) * 60.f) + 1u);
  return 1023u - key;
}

// Three small kernels: (a) per tile S_t into seg_base and the bucket
// histogram of the initial grants (warp-aggregated atomics), (b) one CTA
// scans both in place (8 contiguous tiles per thread), (c) per tile its
// position in its bucket (warp-aggregated atomics) and the queue-1 entries.
// The per-unit counters are zeroed by the host (memset) before the blend.
__device__ __forceinline__ void tile_plan(const uint2 *ranges, int t, int seg, int window, int upt, uint32_t &S,
                                          uint32_t &g, uint32_t &bk) {
  const uint2 r = ranges[t];
  const uint32_t len = r.y > r.x ? r.y - r.x : 0;
  S = len == 0 ? 1 : (len + seg - 1) / seg;
  g = min(S, (uint32_t)window) * (uint32_t)upt;
  bk = len_bucket(len);
}

__global__ __launch_bounds__(256) void plan_count_kernel(const uint2 *__restrict__ ranges, int n_tiles, int seg,
                                                         int window, int upt, uint32_t *__restrict__ seg_base,
                                                         uint32_t *counters) {
  const int t = blockIdx.x * 256 + threadIdx.x;
  uint32_t S = 0, g = 0, bk = 0xFFFFFFFFu;
  if (t < n_tiles) {
    tile_plan(ranges, t, seg, window, upt, S, g, bk);
    seg_base[t] = S;
  }
  const uint32_t peers = __match_any_sync(0xffffffffu, bk);
  const uint32_t gsum = __reduce_add_sync(peers, g);
  if (t < n_tiles && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&counters[CNT_PLAN_HIST + bk], gsum);
}

__global__ __launch_bounds__(1024) void plan_scan_kernel(int n_tiles, uint32_t *__restrict__ seg_base,
                                                         uint32_t *counters) {
  __shared__ uint32_t s_w[32];
  const int tid = threadIdx.x;
  uint32_t run = 0;
  for (int base = 0; base < n_tiles; base += 1024 * 8) {
    const int t0 = base + tid * 8;
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = t0 + k < n_tiles ? seg_base[t0 + k] : 0u;
      sum += v[k];
    }
    uint32_t total;
    uint32_t off = run + block_excl_scan(sum, s_w, total);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (t0 + k < n_tiles) seg_base[t0 + k] = off;
      off += v[k];
    }
    run += total;
  }
  uint32_t n_init;
  const uint32_t h = counters[CNT_PLAN_HIST + tid];
  const uint32_t boff = block_excl_scan(h, s_w, n_init);
  counters[CNT_PLAN_HIST + tid] = boff;
  if (tid == 0) {
    counters[CNT_NITEMS] = run;
    counters[CNT_Q_NINIT] = n_init;
  }
}

__global__ __launch_bounds__(256) void plan_fill_kernel(const uint2 *__restrict__ ranges, int n_tiles, int seg,
                                                        int window, int upt, uint32_t *__restrict__ q1,
                                                        uint32_t *counters) {
  const int t = blockIdx.x * 256 + threadIdx.x, lane = threadIdx.x & 31;
  uint32_t S = 0, g = 0, bk = 0xFFFFFFFFu;
  if (t < n_tiles) tile_plan(ranges, t, seg, window, upt, S, g, bk);
  const uint32_t peers = __match_any_sync(0xffffffffu, bk);
  const int leader = __ffs(peers) - 1;
  // exclusive prefix of g among this lane's peers (g is the same for equal buckets
  // unless S < window; sum explicitly)
  uint32_t pre = 0, gsum = 0;
  for (uint32_t m = peers; m; m &= m - 1) {
    const int l = __ffs(m) - 1;
    const uint32_t gl = __shfl_sync(peers, g, l);
    gsum += gl;
    if (l < lane) pre += gl;
  }
  uint32_t pos = 0;
  if (t < n_tiles && lane == leader) pos = atomicAdd(&counters[CNT_PLAN_HIST + bk], gsum);
  pos = __shfl_sync(peers, pos, leader) + pre;
  // entry = unit | segment << 24 (a unit's first segments in order)
  const uint32_t u = (uint32_t)upt;
  for (uint32_t k = 0; k < g; ++k) q1[pos + k] = (u * (uint32_t)t + k % u) | ((k / u) << 24);
}

void launch_plan(const uint2 *ranges, int n_tiles, int seg, int window, uint32_t *seg_base, uint32_t *q1,
                 uint32_t *counters, cudaStream_t st, int upt) {
  const unsigned blocks = (unsigned)((n_tiles + 255) / 256);
  plan_count_kernel<<<blocks, 256, 0, st>>>(ranges, n_tiles, seg, window, upt, seg_base, counters);
  plan_scan_kernel<<<1, 1024, 0, st>>>(n_tiles, seg_base, counters);
  plan_fill_kernel<<<blocks, 256, 0, st>>>(ranges, n_tiles, seg, window, upt, q1, counters);
}

// ---------------------------------------------------------------- blend
// Transmittance products travel between segments as fixed-point -log2 sums
// (integer addition is associative, so prefixes are bitwise deterministic
// whatever the look-back walk): L = round(-log2(P) 2^32), saturated at 2^36
// (T = 2^-16 < T_min: "dead").  Status word: [63:62] flag (1 aggregate,
// 2 inclusive), [61:40] epoch, [39:0] L.
#define GUT_L_ONE 4294967296.0
#define GUT_L_DEAD (16ull << 32)

// (MUFU lg2 / ex2: absolute error ~2^-22 in log2 T, i.e. ~2e-7 relative in
// the transmittance; the fixed-point sums themselves stay exact integers)
__device__ __forceinline__ unsigned long long l_of(float P) {
  if (!(P > 0.f)) return GUT_L_DEAD;
  float lg;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(P));
  const float l = -lg * 4294967296.f;
  return l >= (float)GUT_L_DEAD ? GUT_L_DEAD : (l <= 0.f ? 0ull : (unsigned long long)__float2ull_rn(l));
}
__device__ __forceinline__ float t_of(unsigned long long L) {
  if (L >= GUT_L_DEAD) return 0.f;
  float t;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(-(float)L * 2.3283064365386963e-10f));
  return t;
}
__device__ __forceinline__ unsigned long long st_word(uint32_t flag, uint32_t epoch, unsigned long long L) {
  return ((unsigned long long)flag << 62) | ((unsigned long long)(epoch & 0x3FFFFFu) << 40) | L;
}

// Upper bound of the pixel's prefix transmittance before segment s, as a
// fixed-point -log2 sum: the published products of some of its predecessors
// (aggregates back to the first inclusive word, at most 4).  Any subset of
// the prefix factors bounds the prefix from above, so words not yet published
// are simply skipped (0 = no information).
__device__ __forceinline__ unsigned long long pred_L(const unsigned long long *stat, int s, uint32_t epoch) {
  unsigned long long L = 0;
  const int jmax = min(s, 4);
  for (int j = 1; j <= jmax; ++j) {
    const unsigned long long wv = ld_relaxed(stat - (size_t)j * GUT_TILE_PX);
    const uint32_t flag = (uint32_t)(wv >> 62);
    if (flag == 0 || (uint32_t)((wv >> 40) & 0x3FFFFFu) != (epoch & 0x3FFFFFu)) continue;
    L += wv & ((1ull << 40) - 1);
    if (L >= GUT_L_DEAD) return GUT_L_DEAD;
    if (flag == 2) break;
  }
  return L;
}
__device__ __forceinline__ bool pred_dead(const unsigned long long *stat, int s, uint32_t epoch) {
  return pred_L(stat, s, epoch) >= GUT_L_DEAD;
}

// Redo checkpoints of a speculative pass: the lane's pixel state after every
// `seg / GUT_CK` entries, recorded while the pixel is live, so a re-run from
// the exact prefix T_pre resumes at the last checkpoint the exact sequence
// certainly reached (T_pre T_c >= T_min) instead of at the segment start.
#ifndef GUT_POLL_CHUNKS
#define GUT_POLL_CHUNKS 2u  // speculative pass: chunks between predecessor polls (power of 2; tuning switch)
#endif
#ifndef GUT_CK
#define GUT_CK 80  // checkpoints per speculative segment: with 2560-entry segments one per 32-entry chunk (8 / 16 / 32: K5 +6% / +3% / +1%; tuning switch)
#endif
template <int NP> struct Checkpoints {
  float4 C[GUT_CK][NP];
  float T[GUT_CK][NP];
  int n[NP];
  float4 keepC[NP];  // (between the two passes: the non-re-running pixels' results)
  bool keepTerm[NP];
};

// Per-warp table of staged list entries (32 per chunk).  MODE 0/1: the
// quadratic forms of F = |n|^2 - k^2 |e|^2 and D = |e|^2 in the lane's pixel
// offset (da, db) from the warp box centre; MODE 2 (rolling shutter, beta
// varies per row): the raw anchored vectors.
template <int MODE> struct WarpTbl { static constexpr int NF = 6; };

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// log2 of alpha / ... : log2 sigma - omega^2 / (2 ln 2) (Gaussian, Eq. 11 response);
// degree n: log2 sigma - lambda_n (omega^2)^(n/2) / (2 ln 2) (MUFU lg2 / ex2)
__device__ __forceinline__ float kernel_arg(bool gen, float kgl, float khn, float w2, float l2s) {
  if (!gen) return fmaf(-0.72134752044448170f, w2, l2s);
  float lw, p;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lw) : "f"(w2));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p) : "f"(khn * lw));
  return fmaf(kgl, p, l2s);
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <> struct WarpTbl<2> { static constexpr int NF = 11; };

// The NP pixels of one lane (GUT_BLEND_NP): ray offsets in, running blend state out.
template <int NP> struct LanePx {
  float a[NP], b[NP], beta[NP], snorm[NP];
  float Cr[NP], Cg[NP], Cb[NP], Dp[NP], T[NP];
  bool done[NP], term[NP];
};

// "Ours (sorted)" (reading R28): the lane's per-ray MLAB
// k-buffer -- the KB farthest pending hits (tau_max, alpha, Gaussian id),
// ascending in tau; empty slots hold tau = -inf and sit at the bottom.
template <int KB> struct KBuf {
  float t[KB > 0 ? KB : 1], a[KB > 0 ? KB : 1];
  uint32_t g[KB > 0 ? KB : 1];
};

// Eq. 5 step of one hit leaving the k-buffer (termination rule R21); the
// colour is gathered from the K1 payload (rgb in the fifth float4).
template <int NP>
__device__ __forceinline__ void kb_blend(LanePx<NP> &L, int k, float tau, float al, uint32_t gid,
                                         const float4 *__restrict__ payload, float t_min, uint32_t &n_contrib) {
  const float Tn = L.T[k] * (1.f - al);
  if (Tn < t_min) {
    L.done[k] = true;
    L.term[k] = true;
    return;
  }
  const float4 cc = __ldg(&payload[(size_t)GUT_PAYLOAD_F4 * gid + 4]);
  const float wgt = al * L.T[k];
  L.Cr[k] = fmaf(wgt, cc.x, L.Cr[k]);
  L.Cg[k] = fmaf(wgt, cc.y, L.Cg[k]);
  L.Cb[k] = fmaf(wgt, cc.z, L.Cb[k]);
  L.Dp[k] = fmaf(wgt, tau, L.Dp[k]);
  L.T[k] = Tn;
  ++n_contrib;
}

// A hit enters the k-buffer: of the KB + 1 pending hits the closest leaves
// (register insertion chain, static indices only) and is blended.
template <int KB, int NP>
__device__ __forceinline__ void kb_insert(KBuf<KB> &kb, LanePx<NP> &L, int k, float tau, float al, uint32_t gid,
                                          const float4 *__restrict__ payload, float t_min, uint32_t &n_contrib) {
  const bool sw = tau < kb.t[0];
  const float pt = sw ? tau : kb.t[0], pa = sw ? al : kb.a[0];
  const uint32_t pg = sw ? gid : kb.g[0];
  float mt = sw ? kb.t[0] : tau, ma = sw ? kb.a[0] : al;
  uint32_t mg = sw ? kb.g[0] : gid;
#pragma unroll
  for (int i = 1; i < KB; ++i) {
    const bool lo = mt < kb.t[i];
    const float ti = kb.t[i], ai = kb.a[i];
    const uint32_t gi = kb.g[i];
    kb.t[i - 1] = lo ? mt : ti; kb.a[i - 1] = lo ? ma : ai; kb.g[i - 1] = lo ? mg : gi;
    mt = lo ? ti : mt; ma = lo ? ai : ma; mg = lo ? gi : mg;
  }
  kb.t[KB - 1] = mt; kb.a[KB - 1] = ma; kb.g[KB - 1] = mg;
  if (pt > -INFINITY) kb_blend<NP>(L, k, pt, pa, pg, payload, t_min, n_contrib);
}

// One pass of ONE WARP over the segment [s0, s1): no CTA barriers.  Each chunk
// of 32 entries is staged by the 32 lanes (one entry each: fp64 for the
// cancelling part), culled against the warp's pixel box in registers, and the
// surviving entries are evaluated by every lane, for each of its NP pixels, in
// list order.  The warp leaves the list as soon as all its pixels have
// terminated.  Termination rule (reading R21): stop before an entry would take
// T below T_min.  The caller sets L.a/b/beta/snorm, L.T (start), L.done
// (= inactive) and L.term = false; the colour sums start at 0 here.
// Per-warp constants of the current unit (the tile anchor D, dO = O - c(0) in
// fp64, D / T1 / T2 in fp32, the pixel box) live in shared memory rather than
// registers: the staging reloads them once per 32-entry chunk (broadcast),
// which frees ~25 registers in the evaluation loops.
#define GUT_WC_F4 9  // float4 per warp
#ifndef GUT_K5_HALF_SKIP
#define GUT_K5_HALF_SKIP 1  // per-pixel-row-half warp-uniform skip of the evaluation (tuning switch)
#endif
__device__ __forceinline__ float4 *warp_consts(int nf) {
  extern __shared__ float4 s_dyn[];
  return s_dyn + (GUT_BLEND_CTA / 32) * 2 * 32 * GUT_PAYLOAD_F4 + (GUT_BLEND_CTA / 32) * 32 * nf +
         (threadIdx.x >> 5) * GUT_WC_F4;
}
template <int MODE>
constexpr size_t blend_smem_bytes() {
  return sizeof(float4) * ((GUT_BLEND_CTA / 32) * 2 * 32 * GUT_PAYLOAD_F4 + (GUT_BLEND_CTA / 32) * 32 * WarpTbl<MODE>::NF +
                           (GUT_BLEND_CTA / 32) * GUT_WC_F4);
}
__device__ __forceinline__ void store_warp_consts(float4 *wc, const d3 &D, const d3 &dO, const f3 &T1f, const f3 &T2f,
                                                  float ac, float bc, float ra, float rb, float tc, float rt,
                                                  const float *fit) {
  if ((threadIdx.x & 31) == 0) {
    wc[7] = make_float4(fit[0], fit[1], fit[2], fit[3]);
    wc[8] = make_float4(fit[4], fit[5], fit[6], fit[7]);
    double2 *wd = reinterpret_cast<double2 *>(wc);
    wd[0] = make_double2(D.x, D.y);
    wd[1] = make_double2(D.z, dO.x);
    wd[2] = make_double2(dO.y, dO.z);
    wc[3] = make_float4((float)D.x, (float)D.y, (float)D.z, T1f.x);
    wc[4] = make_float4(T1f.y, T1f.z, T2f.x, T2f.y);
    wc[5] = make_float4(T2f.z, ac, bc, ra);
    wc[6] = make_float4(rb, tc, rt, 0.f);
  }
  __syncwarp();
}
__device__ __forceinline__ double2 lds_d2(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// Candidate mask of one staged entry over the warp's 8x8 pixel block (bit
// 8 ry + cx; word 0 = rows 0-3, word 1 = rows 4-7): a superset of the pixels
// whose hit test F(da, db) <= 0 can pass.  The pixels' offsets lie on the
// block's affine lattice p -> w0 + J p (rays_kernel fit, residual rho), so
// F(true) <= 0 implies G(p) = F(w0 + J p) <= Em, Em = the lattice error
// |grad F| rho + |Hess F| rho^2 over the box plus a rounding margin 1e-4 mag
// (the hit test's own fp32 error is ~1e-7 mag).  {G <= Em} is an ellipse when
// the Hessian is positive definite (well conditioned: det > 1e-3 Hxx Hyy);
// the mask is its bounding box on the lattice, widened by 1% + 1e-3 px for
// the fp32 solve.  Any other case keeps every pixel.
__device__ __forceinline__ uint2 entry_mask(float F0, float Fa, float Fb, float Faa, float Fab, float Fbb, float as,
                                            float bs, float A, float Bm, float mag, float4 fa, float4 fb) {
  const float u0 = fa.x - as, v0 = fb.x - bs;
  const float ax = fa.y, ay = fa.z, bx = fb.y, by = fb.z, rha = fa.w, rhb = fb.w;
  const float A2 = A + rha, B2 = Bm + rhb;
  const float aFaa = fabsf(Faa), aFab = fabsf(Fab), aFbb = fabsf(Fbb);
  const float Em = fmaf(fmaf(2.f * aFaa, A2, fmaf(aFab, B2, fabsf(Fa))), rha,
                        fmaf(fmaf(2.f * aFbb, B2, fmaf(aFab, A2, fabsf(Fb))), rhb,
                             fmaf(fmaf(aFaa, rha, aFab * rhb), rha, aFbb * rhb * rhb))) +
                   1e-4f * mag;
  const float Fu = fmaf(2.f * Faa, u0, fmaf(Fab, v0, Fa)), Fv = fmaf(2.f * Fbb, v0, fmaf(Fab, u0, Fb));
  const float G0 = fmaf(u0, fmaf(Faa, u0, fmaf(Fab, v0, Fa)), fmaf(v0, fmaf(Fbb, v0, Fb), F0));
  const float gx = fmaf(ax, Fu, bx * Fv), gy = fmaf(ay, Fu, by * Fv);
  const float hx0 = fmaf(2.f * Faa, ax, Fab * bx), hx1 = fmaf(Fab, ax, 2.f * Fbb * bx);
  const float hy0 = fmaf(2.f * Faa, ay, Fab * by), hy1 = fmaf(Fab, ay, 2.f * Fbb * by);
  const float Hxx = fmaf(ax, hx0, bx * hx1), Hxy = fmaf(ay, hx0, by * hx1), Hyy = fmaf(ay, hy0, by * hy1);
  const float det = fmaf(Hxx, Hyy, -Hxy * Hxy);
  uint2 m = make_uint2(~0u, ~0u);
  if (Hxx > 0.f && Hyy > 0.f && det > 1e-3f * Hxx * Hyy && Em < 1e30f) {
    const float id = rcp_approx(det);  // (MUFU: 2^-22 relative, inside the 1% widening)
    const float nx = fmaf(Hyy, gx, -Hxy * gy), ny = fmaf(Hxx, gy, -Hxy * gx);
    const float px = -nx * id, py = -ny * id;  // minimiser p* = -H^-1 g
    const float gp = fmaf(gx, px, gy * py);    // g . p* = -g^T H^-1 g
    const float R = Em + 1e-2f * fabsf(gp) - fmaf(0.5f, gp, G0);  // Em - min G (+ margin)
    if (!(R >= 0.f)) {
      if (R < 0.f) m = make_uint2(0u, 0u);
    } else if (R < 1e30f) {
      const float r2 = 2.f * R * id;
      const float hx = fmaf(1.01f, sqrt_approx(r2 * Hyy), fmaf(1e-2f * id, fabsf(Hyy * gx) + fabsf(Hxy * gy), 1e-3f));
      const float hy = fmaf(1.01f, sqrt_approx(r2 * Hxx), fmaf(1e-2f * id, fabsf(Hxx * gy) + fabsf(Hxy * gx), 1e-3f));
      // pixel index bounds on the lattice (cvt saturates out-of-range values)
      const int xl = max(__float2int_ru(px - hx), 0), xh = min(__float2int_rd(px + hx), 7);
      const int yl = max(__float2int_ru(py - hy), 0), yh = min(__float2int_rd(py + hy), 7);
      // columns xl..xh of rows yl..yh (empty when a range is: the shifts
      // then give a zero or wrapped-to-zero difference)
      const uint32_t col = (xh >= xl) ? (2u << xh) - (1u << xl) : 0u;
      const unsigned long long rows = (yh >= yl) ? (2ull << (8 * yh + 7)) - (1ull << (8 * yl)) : 0ull;
      const uint32_t rep = col * 0x01010101u;
      m = make_uint2(rep & (uint32_t)rows, rep & (uint32_t)(rows >> 32));
    }
  }
  return m;
}

#ifndef GUT_K5_MASKS
#define GUT_K5_MASKS 1  // candidate masks on/off (tuning switch)
#endif
#ifndef GUT_K5_MASK_MIN
#define GUT_K5_MASK_MIN 2   // entries a chunk's masks must drop to stay on (tuning switch)
#endif
#ifndef GUT_K5_MASK_SKIP
#define GUT_K5_MASK_SKIP 3  // chunks without masks after a chunk below GUT_K5_MASK_MIN
#endif
template <int MODE, int NP, int KB = 0>
__device__ __forceinline__ void warp_pass(const DevCam &c, const BlendBufs &B, uint32_t s0, uint32_t s1,
                                          LanePx<NP> &L, uint32_t &n_eval, uint32_t &n_contrib,
                                          uint32_t &processed, const unsigned long long *poll_stat, int poll_s,
                                          Checkpoints<NP> *ck, uint32_t ck_step, const uint32_t *act,
                                          KBuf<KB> *kb = nullptr, int half = 0) {
  constexpr int NF = WarpTbl<MODE>::NF;
  constexpr unsigned FULL = 0xffffffffu;
  // dynamic shared memory: [raw payload double buffer: 8 warps x 2 x 32 x 5]
  // [per-warp entry table: 8 warps x 32 x NF]
  extern __shared__ float4 s_dyn[];
  constexpr int PF = GUT_PAYLOAD_F4;
  constexpr int RAW = (GUT_BLEND_CTA / 32) * 2 * 32 * PF;
  float4 *__restrict__ wt = s_dyn + RAW + (threadIdx.x >> 5) * 32 * NF;
  const uint32_t wt_s = (uint32_t)__cvta_generic_to_shared(wt);
  const int lane = threadIdx.x & 31;
  const float alpha_min = c.alpha_min, alpha_max = c.alpha_max, t_min = c.t_min;
  const float l2amin = log2f(alpha_min);
  // kernel degree n (Supp. A): log2 alpha = log2 sigma - lambda_n omega^n / (2 ln 2)
  const bool gen = c.kdeg != 2;
  const float kgl = -0.72134752044448170f * c.klam, khn = 0.5f * (float)c.kdeg;
  const f3 dcw = mk((float)c.dc[0], (float)c.dc[1], (float)c.dc[2]);
  // raw payload of the warp's current / next chunk (cp.async double buffer)
  float4 *__restrict__ raw = s_dyn + (threadIdx.x >> 5) * 2 * 32 * PF;
  // the unit's anchor and box (store_warp_consts): dO = O - c(0) (payload w0 = c(0) - mu)
  const uint32_t wc_s = (uint32_t)__cvta_generic_to_shared(warp_consts(NF));
  bool all_done = true;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    all_done = all_done && L.done[k];
    if (ck) ck->n[k] = 0;
  }
  processed = 0;
  // per-pixel start positions (a re-run resumes each pixel at its own
  // checkpoint): pixels starting later are dormant until the walk reaches
  // them, and the walk jumps over stretches where no pixel is active
  bool pend[NP];
  uint32_t actp[NP], start = 0xFFFFFFFFu;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    actp[k] = act ? act[k] : s0;
    pend[k] = !L.done[k] && actp[k] > s0;
    if (!L.done[k]) start = min(start, actp[k]);
    if (pend[k]) L.done[k] = true;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) start = min(start, __shfl_xor_sync(FULL, start, o));
  bool anyp = false;
#pragma unroll
  for (int k = 0; k < NP; ++k) anyp = anyp || pend[k];
  const bool wpend = __any_sync(FULL, anyp);  // (only a re-run has dormant pixels)
  uint32_t ck_next = s0 + ck_step;           // next checkpoint position (speculative pass)
  int ck_idx = 0;
  if (start >= s1) {
#pragma unroll
    for (int k = 0; k < NP; ++k) if (pend[k]) L.done[k] = false;  // (nothing left to walk: unchanged state)
    return;
  }
  // gathers run one chunk ahead (cp.async), Gaussian ids two chunks ahead
  uint32_t gnext = 0;
  int buf = 0;
  auto prime = [&](uint32_t p) {
    gnext = p + lane < s1 ? __ldg(&B.gids[p + lane]) : 0u;
    if (p + lane < s1) {
      float4 *dst = raw + lane * PF;
      for (int q = 0; q < PF; ++q) cp_async16(dst + q, &B.payload[(size_t)PF * gnext + q]);
    }
    cp_async_commit();
    gnext = p + 32 + lane < s1 ? __ldg(&B.gids[p + 32 + lane]) : 0u;
  };
  prime(start);
  int mk_skip = 0;  // chunks left without candidate masks (warp-uniform)
  for (uint32_t b0 = start; b0 < s1; b0 += 32, buf ^= 1) {
    bool anypend = false;
    if (wpend) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        if (pend[k] && actp[k] <= b0) { pend[k] = false; L.done[k] = false; }
        anypend = anypend || pend[k];
      }
    }
    // speculative pass of a later segment: every GUT_POLL_CHUNKS chunks, stop pixels whose
    // exact sequence has certainly terminated by now: T_spec times the bound of
    // the published prefix below T_min (Ls := dead, exact; a re-run resolves it)
    if (poll_stat && ((b0 - s0) & (GUT_POLL_CHUNKS * 32u - 1u)) == (((GUT_POLL_CHUNKS * 32u) / 2u) & ~31u)) {
#pragma unroll
      for (int k = 0; k < NP; ++k)
        if (!L.done[k]) {
          const unsigned long long Lb = pred_L(poll_stat + 64 * k, poll_s, __ldg(B.epoch) + GUT_EPOCH_BLEND);
          // (MUFU ex2: a pixel stopped here by a rounding error is re-run exactly
          // from T_pre like any pixel that terminates in the segment)
          if (Lb >= GUT_L_DEAD || L.T[k] * ex2_approx(-(float)Lb * 2.3283064365386963e-10f) < t_min)
            L.done[k] = L.term[k] = true;
        }
    }
    if (ck && b0 == ck_next && ck_idx < GUT_CK) {  // (the speculative pass walks from s0 in steps of 32: no jumps)
      ck_next += ck_step;
#pragma unroll
      for (int k = 0; k < NP; ++k)
        if (!L.done[k]) {
          ck->C[ck_idx][k] = make_float4(L.Cr[k], L.Cg[k], L.Cb[k], L.Dp[k]);
          ck->T[ck_idx][k] = L.T[k];
          ck->n[k] = ck_idx + 1;
        }
      ++ck_idx;
    }
    all_done = true;
#pragma unroll
    for (int k = 0; k < NP; ++k) all_done = all_done && L.done[k];
    if (__all_sync(FULL, all_done)) {
      if (!__any_sync(FULL, anypend)) break;
      // no active pixel: jump to the next resume position and restart the gathers
      uint32_t nxt = 0xFFFFFFFFu;
#pragma unroll
      for (int k = 0; k < NP; ++k) if (pend[k]) nxt = min(nxt, actp[k]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nxt = min(nxt, __shfl_xor_sync(FULL, nxt, o));
      cp_async_wait<0>();
      __syncwarp();
      prime(nxt);
      b0 = nxt - 32;  // (the loop increment lands on nxt with buf = 0)
      buf = 1;
      continue;
    }
    if (b0 + 32 < s1) {  // prefetch the next chunk
      if (b0 + 32 + lane < s1) {
        float4 *dst = raw + ((buf ^ 1) * 32 + lane) * PF;
        for (int q = 0; q < PF; ++q) cp_async16(dst + q, &B.payload[(size_t)PF * gnext + q]);
      }
      cp_async_commit();
      gnext = b0 + 64 + lane < s1 ? __ldg(&B.gids[b0 + 64 + lane]) : 0u;
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    processed = min(b0 + 32, s1) - s0;
    const uint32_t kk = b0 + (uint32_t)lane;
    bool maybe = false;
    uint2 cmask = make_uint2(0u, 0u);  // candidate pixels of the lane's entry (MODE 0/1)
    if (kk < s1) {
      // ---- stage entry kk.  The cancelling part c0 = o_g x d_g (o_g = M w,
      // d_g = M D, w = O - mu) uses (M a) x (M b) = cof(M) (a x b) with
      // cof(M) = det(M) M^-T = diag(s_i^2 det M) M for M = diag(1/s) R^T:
      // only w x D is formed in fp64 (the small vector), the rest in fp32.
      const float4 *src = raw + (buf * 32 + lane) * PF;
      const double2 wxy = *reinterpret_cast<const double2 *>(src);
      const double2 q0 = lds_d2(wc_s), q1 = lds_d2(wc_s + 16), q2 = lds_d2(wc_s + 32);
      const float4 q3 = lds128(wc_s + 48), q4 = lds128(wc_s + 64), q5 = lds128(wc_s + 80), q6 = lds128(wc_s + 96);
      const d3 D = mkd(q0.x, q0.y, q1.x), dO = mkd(q1.y, q2.x, q2.y);
      const f3 Df = mk(q3.x, q3.y, q3.z), T1f = mk(q3.w, q4.x, q4.y), T2f = mk(q4.z, q4.w, q5.x);
      const float ac = q5.y, bc = q5.z, ra = q5.w, rb = q6.x, tc = q6.y, rt = q6.z;
      const float4 p1 = src[1], p2 = src[2], p3 = src[3], p4 = src[4];
      const d3 w = mkd(wxy.x, wxy.y, __hiloint2double(__float_as_int(p1.y), __float_as_int(p1.x))) + dO;
      const f3 x = tof(cross(w, D));
      const float M[9] = {p1.w, p2.x, p2.y, p2.z, p2.w, p3.x, p3.y, p3.z, p3.w};
      // row norms |M_i|^2 = 1/s_i^2; lambda_i = s_i^2 det M = sqrt(n0 n1 n2) / n_i
      const float rn0 = fmaf(M[0], M[0], fmaf(M[1], M[1], M[2] * M[2]));
      const float rn1 = fmaf(M[3], M[3], fmaf(M[4], M[4], M[5] * M[5]));
      const float rn2 = fmaf(M[6], M[6], fmaf(M[7], M[7], M[8] * M[8]));
      // (MUFU rsqrt / rcp: relative error ~2^-22 in the row scales, harmless)
      const float r012 = rn0 * rn1 * rn2, dM = r012 * rsqrt_approx(r012);
      const f3 Mx = mv(M, x);
      const f3 c0 = mk(Mx.x * (dM * rcp_approx(rn0)), Mx.y * (dM * rcp_approx(rn1)), Mx.z * (dM * rcp_approx(rn2)));
      const f3 ogf = mv(M, tof(w)), e0 = mv(M, Df);
      const float g0 = dot(ogf, e0);
      f3 U = mv(M, T1f), V = mv(M, T2f), P, Q;
      float gu, gv;
      if (MODE == 1) {
        P = cross(U, e0); Q = cross(V, e0); gu = dot(U, e0); gv = dot(V, e0);
        U = mk(0, 0, 0); V = mk(0, 0, 0);
      } else {
        P = cross(ogf, U); Q = cross(ogf, V); gu = dot(ogf, U); gv = dot(ogf, V);
      }
      // k^2 = 2 ln(sigma/alpha_min) (K1, via log1p); log2 sigma = k^2 / (2 ln 2) + log2 alpha_min
      const float k2 = p1.z;
      const float l2s = c.kdeg == 2 ? fmaf(k2, 0.72134752044448170f, l2amin) : p4.w;  // (p4.w = log2 sigma from K1)
      // ---- conservative cull against the warp's pixel box (a in ac +- ra,
      // b in bc +- rb): |n| >= |n(ac,bc)| - ra|P| - rb|Q|, |e| <= |e(ac,bc)| +
      // ra|U| + rb|V| (triangle inequality); omega^2 > k^2 on the whole box if
      // (|n0| - dn)^2 > k^2 (|e0| + de)^2 (1e-3 margin for fp32 rounding).
      // Rolling shutter: every entry is kept.
      const f3 n0 = c0 + ac * P + bc * Q;
      const f3 e0c = e0 + ac * U + bc * V;
      f3 mdc = mk(0, 0, 0), h = mk(0, 0, 0), PU = mk(0, 0, 0), QV = mk(0, 0, 0);
      if (MODE == 2) {
        // rolling shutter: n = c0 + aP + bQ + beta (h + a PU + b QV) with beta
        // (pixel time - anchor time) in tc +- rt over the warp's rows.  Around
        // the box centre n = n_c + da (P + tc PU) + db (Q + tc QV) + dt (h + ac PU
        // + bc QV) + da dt PU + db dt QV, so |n| >= |n_c| - (ra |P + tc PU| + rb |Q
        // + tc QV| + rt |h + ac PU + bc QV| + ra rt |PU| + rb rt |QV|) (triangle
        // inequality); e does not depend on beta.  Same 1e-3 margin as below.
        mdc = mv(M, dcw);
        h = cross(mdc, e0); PU = cross(mdc, U); QV = cross(mdc, V);
        const f3 Pt = P + tc * PU, Qt = Q + tc * QV, Ht = h + ac * PU + bc * QV;
        const f3 nc = n0 + tc * Ht;
        const float lo = sqrt_approx(dot(nc, nc)) -
                         (ra * sqrt_approx(dot(Pt, Pt)) + rb * sqrt_approx(dot(Qt, Qt)) + rt * sqrt_approx(dot(Ht, Ht)) +
                          rt * (ra * sqrt_approx(dot(PU, PU)) + rb * sqrt_approx(dot(QV, QV))));
        const float hi = sqrt_approx(dot(e0c, e0c)) + (ra * sqrt_approx(dot(U, U)) + rb * sqrt_approx(dot(V, V)));
        maybe = !(lo > 0.f && lo * lo > 1.001f * k2 * (hi * hi));
      } else {
        // (MUFU square roots: 2^-22 relative, inside the 1e-3 margin below)
        const float lo = sqrt_approx(dot(n0, n0)) - (ra * sqrt_approx(dot(P, P)) + rb * sqrt_approx(dot(Q, Q)));
        const float hi = sqrt_approx(dot(e0c, e0c)) + (ra * sqrt_approx(dot(U, U)) + rb * sqrt_approx(dot(V, V)));
        maybe = !(lo > 0.f && lo * lo > 1.001f * k2 * (hi * hi));
      }
      if (maybe) {
        float4 *t = wt + lane * NF;
        if (MODE == 2) {
          const f3 m = mdc;
          t[0] = make_float4(c0.x, c0.y, c0.z, k2);
          t[1] = make_float4(P.x, P.y, P.z, Q.x);
          t[2] = make_float4(Q.y, Q.z, e0.x, e0.y);
          t[3] = make_float4(e0.z, U.x, U.y, U.z);
          t[4] = make_float4(V.x, V.y, V.z, l2s);
          t[5] = make_float4(g0, gu, gv, 0.f);
          t[6] = make_float4(p4.x, p4.y, p4.z, KB > 0 ? __uint_as_float(__ldg(&B.gids[kk])) : 0.f);
          t[7] = make_float4(h.x, h.y, h.z, dot(m, e0));
          t[8] = make_float4(PU.x, PU.y, PU.z, dot(m, U));
          t[9] = make_float4(QV.x, QV.y, QV.z, dot(m, V));
        } else {
          // Quadratic forms of F = |n|^2 - k^2 |e|^2 and D = |e|^2 in the pixel
          // offset (da, db) from an expansion point (a*, b*): the box point
          // nearest the Gaussian (minimiser of |n|^2, clamped to the box), so
          // the coefficients' rounding stays relative to the values at the
          // pixels (expanding about the box centre would cost eps * omega_c^2
          // for Gaussians far smaller than the box).
          const float pp = dot(P, P), pq = dot(P, Q), qq = dot(Q, Q);
          const float np = dot(n0, P), nq = dot(n0, Q);
          const float det = fmaf(pp, qq, -pq * pq);
          float xa = 0.f, xb = 0.f;
          if (det > 1e-30f * pp * qq && det > 0.f) {
            const float id = rcp_approx(det);  // (expansion point only)
            xa = (pq * nq - qq * np) * id;
            xb = (pq * np - pp * nq) * id;
          }
          const float as = ac + fminf(fmaxf(xa, -ra), ra), bs = bc + fminf(fmaxf(xb, -rb), rb);
          const f3 ns = c0 + as * P + bs * Q;
          const f3 es = e0 + as * U + bs * V;
          const float N0 = dot(ns, ns), Na = 2.f * dot(ns, P), Nb = 2.f * dot(ns, Q);
          const float Nab = 2.f * pq;
          const float D0 = dot(es, es), Da = 2.f * dot(es, U), Db = 2.f * dot(es, V);
          const float Daa = dot(U, U), Dab = 2.f * dot(U, V), Dbb = dot(V, V);
          const float gs = g0 + as * gu + bs * gv;
          const float F0 = fmaf(-k2, D0, N0), Fa = fmaf(-k2, Da, Na), Fb = fmaf(-k2, Db, Nb);
          const float Faa = fmaf(-k2, Daa, pp), Fab = fmaf(-k2, Dab, Nab), Fbb = fmaf(-k2, Dbb, qq);
          // second, tighter cull: a lower bound of the quadratic F over the box
          // (offsets da in [la, ha], db in [lb, hb] from (a*, b*)) as the sum of
          // the exact 1-D minima of the a- and b-parts and the worst cross term;
          // margin 1e-4 of the terms' magnitude for fp32 rounding
          const float la = ac - ra - as, ha = ac + ra - as, lb = bc - rb - bs, hb = bc + rb - bs;
          const float A = fmaxf(-la, ha), Bm = fmaxf(-lb, hb);
          // (approximate 1-D minimisers: the quadratic is evaluated at them, an
          // offset delta raises the value by Faa delta^2 only -- far inside the margin)
          const float xa_ = Faa > 0.f ? fminf(fmaxf(-0.5f * Fa * rcp_approx(Faa), la), ha) : (Fa > 0.f ? la : ha);
          const float xb_ = Fbb > 0.f ? fminf(fmaxf(-0.5f * Fb * rcp_approx(Fbb), lb), hb) : (Fb > 0.f ? lb : hb);
          const float ma = fminf(xa_ * fmaf(Faa, xa_, Fa), fminf(la * fmaf(Faa, la, Fa), ha * fmaf(Faa, ha, Fa)));
          const float mb = fminf(xb_ * fmaf(Fbb, xb_, Fb), fminf(lb * fmaf(Fbb, lb, Fb), hb * fmaf(Fbb, hb, Fb)));
          const float mab = fabsf(Fab) * A * Bm;
          const float mag = fabsf(F0) + fabsf(Fa) * A + fabsf(Fb) * Bm + (fabsf(Faa) * A + fabsf(Fab) * Bm) * A +
                            fabsf(Fbb) * Bm * Bm;
          maybe = !(F0 + ma + mb - mab > 1e-4f * mag);
          if (maybe) {
            t[0] = make_float4(F0, Fa, Fb, Faa);
            t[1] = make_float4(Fab, Fbb, as, bs);
            t[2] = make_float4(D0, Da, Db, Daa);
            t[3] = make_float4(Dab, Dbb, gs, gu);
            t[4] = make_float4(gv, k2, l2s, 0.f);
            t[5] = make_float4(p4.x, p4.y, p4.z, KB > 0 ? __uint_as_float(__ldg(&B.gids[kk])) : 0.f);
            if (GUT_K5_MASKS && mk_skip == 0) {
              uint2 em = entry_mask(F0, Fa, Fb, Faa, Fab, Fbb, as, bs, A, Bm, mag, lds128(wc_s + 112),
                                    lds128(wc_s + 128));
              if (NP == 1) em = make_uint2(half ? em.y : em.x, 0u);
              cmask = em;
            } else {
              cmask = make_uint2(~0u, NP > 1 ? ~0u : 0u);
            }
          }
        }
      }
    }
    uint32_t m = __ballot_sync(FULL, maybe);
    {  // statistics: pairs (live pixel, entry surviving the warp-box cull) of this chunk
      uint32_t live = 0;
#pragma unroll
      for (int k = 0; k < NP; ++k) live += L.done[k] ? 0u : 1u;
      n_eval += live * (uint32_t)__popc(m);
    }
    if (MODE != 2) {
      // only entries with a candidate pixel that is still live are evaluated
      const uint32_t live0 = __ballot_sync(FULL, !L.done[0]);
      const uint32_t live1 = NP > 1 ? __ballot_sync(FULL, !L.done[NP > 1 ? 1 : 0]) : 0u;
      const uint32_t mb = m;
      m = __ballot_sync(FULL, maybe && ((cmask.x & live0) | (cmask.y & live1)) != 0u);
      // adaptive: the masks cost ~150 warp-instructions a chunk and save ~30 per
      // entry they drop; where a chunk drops fewer than GUT_K5_MASK_MIN entries
      // (large footprints), the next GUT_K5_MASK_SKIP chunks go without
      if (mk_skip > 0) --mk_skip;
      else if (__popc(mb) - __popc(m) < GUT_K5_MASK_MIN) mk_skip = GUT_K5_MASK_SKIP;
    }
    __syncwarp();
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t ta = wt_s + (uint32_t)j * (NF * 16);
      if (MODE == 2) {
        const float4 f0 = lds128(ta), f1 = lds128(ta + 16), f2 = lds128(ta + 32), f3v = lds128(ta + 48),
                     f4 = lds128(ta + 64), f5 = lds128(ta + 80);
        const float4 h = lds128(ta + 112), pu = lds128(ta + 128), qv = lds128(ta + 144);
        float N[NP], Dd[NP];
        bool hit[NP], any = false;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const float a = L.a[k], b = L.b[k], beta = L.beta[k];
          float nx = fmaf(a, f1.x, fmaf(b, f1.w, f0.x));
          float ny = fmaf(a, f1.y, fmaf(b, f2.x, f0.y));
          float nz = fmaf(a, f1.z, fmaf(b, f2.y, f0.z));
          nx = fmaf(beta, fmaf(a, pu.x, fmaf(b, qv.x, h.x)), nx);
          ny = fmaf(beta, fmaf(a, pu.y, fmaf(b, qv.y, h.y)), ny);
          nz = fmaf(beta, fmaf(a, pu.z, fmaf(b, qv.z, h.z)), nz);
          const float ex = fmaf(a, f3v.y, fmaf(b, f4.x, f2.z));
          const float ey = fmaf(a, f3v.z, fmaf(b, f4.y, f2.w));
          const float ez = fmaf(a, f3v.w, fmaf(b, f4.z, f3v.x));
          N[k] = fmaf(nx, nx, fmaf(ny, ny, nz * nz));
          Dd[k] = fmaf(ex, ex, fmaf(ey, ey, ez * ez));
          // omega^2 <= k^2  <=>  alpha >= alpha_min
          hit[k] = !L.done[k] && N[k] <= f0.w * Dd[k];
          any = any || hit[k];
        }
        if (!__any_sync(FULL, any)) continue;
        const float4 cc = lds128(ta + 96);
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const float a = L.a[k], b = L.b[k], beta = L.beta[k];
          const float rD = rcp_approx(Dd[k]);
          const float w2 = N[k] * rD;
          float gg = fmaf(a, f5.y, fmaf(b, f5.z, f5.x));
          gg = fmaf(beta, fmaf(a, pu.w, fmaf(b, qv.w, h.w)), gg);
          // MUFU ex2 / rcp (rel. error < 2^-21): alpha = sigma exp(-omega^2 / 2)
          const float al = fminf(alpha_max, ex2_approx(kernel_arg(gen, kgl, khn, w2, f4.w)));
          const float tau = -gg * rD * L.snorm[k];
          const float Tn = L.T[k] * (1.f - al);
          const bool ok = hit[k] && al >= alpha_min && tau > 0.f;  // reading R24: tau > 0
          if (KB > 0) {  // "Ours (sorted)": the hit enters the per-ray k-buffer
            if (ok) kb_insert<KB, NP>(*kb, L, k, tau, al, __float_as_uint(cc.w), B.payload, t_min, n_contrib);
            continue;
          }
          const bool dead = ok && Tn < t_min;
          if (dead) { L.done[k] = true; L.term[k] = true; }
          if (ok && !dead) {
            const float wgt = al * L.T[k];
            L.Cr[k] = fmaf(wgt, cc.x, L.Cr[k]);
            L.Cg[k] = fmaf(wgt, cc.y, L.Cg[k]);
            L.Cb[k] = fmaf(wgt, cc.z, L.Cb[k]);
            L.Dp[k] = fmaf(wgt, tau, L.Dp[k]);
            ++n_contrib;
            L.T[k] = Tn;
          }
        }
      } else {
        // the entry's candidate pixels (mask words, warp-uniform); lanes
        // predicated, the body skipped (warp-uniform branch) when no candidate
        // pixel of the warp is inside the footprint
        const float4 f0 = lds128(ta), f1 = lds128(ta + 16);
        float F[NP], da[NP], db[NP];
        bool hit[NP], any = false;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          da[k] = L.a[k] - f1.z;
          db[k] = L.b[k] - f1.w;
          // F = N - k^2 D <= 0  <=>  omega^2 <= k^2  <=>  alpha >= alpha_min
          F[k] = fmaf(da[k], fmaf(f0.w, da[k], fmaf(f1.x, db[k], f0.y)), fmaf(db[k], fmaf(f1.y, db[k], f0.z), f0.x));
          hit[k] = !L.done[k] && F[k] <= 0.f;
          any = any || hit[k];
        }
        if (!__any_sync(FULL, any)) continue;
        const float4 f2 = lds128(ta + 32), f3v = lds128(ta + 48), f4 = lds128(ta + 64), cc = lds128(ta + 80);
#pragma unroll
        for (int k = 0; k < NP; ++k) {
#if GUT_K5_HALF_SKIP
          // the entry covers only one of the warp's two 8x4 halves: skip the other
          if (NP > 1 && !__any_sync(FULL, hit[k])) continue;
#endif
          const float Dd = fmaf(da[k], fmaf(f2.w, da[k], fmaf(f3v.x, db[k], f2.y)),
                                fmaf(db[k], fmaf(f3v.y, db[k], f2.z), f2.x));
          const float rD = rcp_approx(Dd);
          const float w2 = fmaxf(fmaf(f4.y, Dd, F[k]), 0.f) * rD;
          const float gg = fmaf(da[k], f3v.w, fmaf(db[k], f4.x, f3v.z));
          // MUFU ex2 / rcp (rel. error < 2^-21): alpha = sigma exp(-omega^2 / 2)
          const float al = fminf(alpha_max, ex2_approx(kernel_arg(gen, kgl, khn, w2, f4.z)));
          const float tau = -gg * rD * L.snorm[k];
          const float Tn = L.T[k] * (1.f - al);
          const bool ok = hit[k] && al >= alpha_min && tau > 0.f;  // reading R24: tau > 0
          if (KB > 0) {  // "Ours (sorted)": the hit enters the per-ray k-buffer
            if (ok) kb_insert<KB, NP>(*kb, L, k, tau, al, __float_as_uint(cc.w), B.payload, t_min, n_contrib);
            continue;
          }
          const bool dead = ok && Tn < t_min;
          if (dead) { L.done[k] = true; L.term[k] = true; }
          if (ok && !dead) {
            const float wgt = al * L.T[k];
            L.Cr[k] = fmaf(wgt, cc.x, L.Cr[k]);
            L.Cg[k] = fmaf(wgt, cc.y, L.Cg[k]);
            L.Cb[k] = fmaf(wgt, cc.z, L.Cb[k]);
            L.Dp[k] = fmaf(wgt, tau, L.Dp[k]);
            ++n_contrib;
            L.T[k] = Tn;
          }
        }
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();  // a warp leaving early must not leave copies in flight
  __syncwarp();
}

#ifndef GUT_BLEND_WAIT_NS
#define GUT_BLEND_WAIT_NS 2048  // longest back-off of a warp waiting for a granted segment (tuning switch)
#endif
// Work queue (lane 0 of a warp).  Queue 2 (granted successors of running
// chains) is served before queue 1 (initial grants).  Both hand out tickets
// with one atomicAdd (no CAS retry storms among thousands of warps); a warp
// holding a queue-2 ticket whose slot is not yet written waits on that slot
// alone (backoff), and leaves once every unit has been written.  The segment
// index is assigned here, in hand-out order per unit.
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t *p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ bool fetch_work(const BlendBufs &B, uint32_t n_init, int &unit, int &s) {
  uint32_t *cnt = B.counters;
  const uint32_t n_units = (uint32_t)B.n_tiles * GUT_BLEND_WARPS;
  for (;;) {
    const uint32_t hd1 = ld_volatile_u32(&cnt[CNT_Q_HEAD1]);
    const uint32_t h2 = ld_volatile_u32(&cnt[CNT_Q_HEAD2]), a2 = ld_volatile_u32(&cnt[CNT_Q_ALLOC2]);
    const bool q1_empty = hd1 >= n_init;
    // nothing left to hand out and enough warps already waiting for future
    // grants: leave (a warp never leaves holding a ticket, so every granted
    // slot keeps a consumer; idle warps would only burn issue slots)
    if (q1_empty && h2 >= a2 + GUT_BLEND_MAX_WAITERS) return false;
    if (q1_empty || h2 < a2) {
      const uint32_t t2 = atomicAdd(&cnt[CNT_Q_HEAD2], 1u);
      uint32_t u1;
      for (int k = 0; (u1 = ld_volatile_u32(&B.q2[t2])) == 0; ++k) {
        if ((k & 3) == 3 && ld_volatile_u32(&cnt[CNT_Q_FINISHED]) >= n_units) return false;
        __nanosleep(k < 2 ? 128 : (k < 6 ? 512 : GUT_BLEND_WAIT_NS));
      }
      B.q2[t2] = 0;  // slot reusable by the next render
      unit = (int)(u1 - 1);
      // granted successors follow the unit's first min(S, window) segments
      const uint2 rg = B.ranges[unit / GUT_BLEND_WARPS];
      const uint32_t len = rg.y > rg.x ? rg.y - rg.x : 0u;
      const uint32_t S = len == 0 ? 1u : (len + B.seg - 1) / B.seg;
      s = (int)(min(S, (uint32_t)B.window) + atomicAdd(&B.next_s[unit], 1u));
      return true;
    }
    const uint32_t h1 = atomicAdd(&cnt[CNT_Q_HEAD1], 1u);
    if (h1 < n_init) {
      const uint32_t e = B.q1[h1];  // unit | segment << 24 (plan_fill_kernel)
      unit = (int)(e & 0xFFFFFFu);
      s = (int)(e >> 24);
      atomicAdd(&B.q1_taken[unit], 1u);  // (successor grants wait for this: see the grant below)
      return true;
    }
  }
}

// Persistent CTAs (as many as fit), each warp looping independently over
// work units (tile, 8x8 pixel block, segment) taken from the queues; a lane
// owns NP = 2 pixels of the block (rows r and r + 4).  Per unit: the pixels,
// the speculative pass, the look-back, the redo, then either the pixel write
// (single-segment tile) or the partials, the successor grants and, in the
// warp completing the unit's last granted segment, the in-order combine.  No
// CTA-wide barriers: a warp whose pixels finish early moves on.
template <int MODE>
__global__ __launch_bounds__(GUT_BLEND_CTA, GUT_BLEND_CTAS) void blend_kernel(DevCam c, BlendBufs B) {
  constexpr int NT = GUT_TILE_PX, NP = GUT_BLEND_NP;
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  uint32_t n_eval_acc = 0, n_contrib_acc = 0, n_term_acc = 0;
  const uint32_t n_init = B.counters[CNT_Q_NINIT];
  const uint32_t epoch = __ldg(B.epoch) + GUT_EPOCH_BLEND;  // (device epoch: graph-replayable)

  for (;;) {
    int unit = -1, s = 0;
    if (lane == 0 && !fetch_work(B, n_init, unit, s)) unit = -1;
    unit = __shfl_sync(FULL, unit, 0);
    s = __shfl_sync(FULL, s, 0);
    if (unit < 0) break;
    const int tile = unit / GUT_BLEND_WARPS, w = unit % GUT_BLEND_WARPS;
    unsigned long long t_begin = 0;
    if (B.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));

    const uint2 rg = B.ranges[tile];  // empty tile: (UINT_MAX, 0)
    const uint32_t start = rg.y > rg.x ? rg.x : 0u, end = rg.y > rg.x ? rg.y : 0u, len = end - start;
    const int S = len == 0 ? 1 : (int)((len + B.seg - 1) / B.seg);
    const uint32_t s0 = start + (uint32_t)s * B.seg, s1 = min(s0 + (uint32_t)B.seg, end);
    const uint32_t slot = B.seg_base[tile] + (uint32_t)s;
    // pixel k of the lane = lane of the 8x4 LUT block w8 (rays_kernel layout)
    const int pidx0 = (((w & 1) | ((w >> 1) << 2)) << 5) + lane;  // + 64 k
    LanePx<NP> L;
    bool valid[NP], inside[NP];
    int px[NP], py[NP];
    float amin = 3e38f, amax = -3e38f, bmin = 3e38f, bmax = -3e38f, tmin = 3e38f, tmax = -3e38f;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      tile_pixel(tile, c.tiles_x, ((w & 1) | (((w >> 1) * 2 + k) << 1)), lane, px[k], py[k]);
      inside[k] = px[k] < c.width && py[k] < c.height;
      const float4 pl = B.pix[(size_t)tile * NT + pidx0 + 64 * k];
      L.a[k] = pl.x; L.b[k] = pl.y; L.snorm[k] = pl.z; L.beta[k] = pl.w;
      valid[k] = inside[k] && pl.z > 0.f;
      if (valid[k]) {
        amin = fminf(amin, pl.x); amax = fmaxf(amax, pl.x);
        bmin = fminf(bmin, pl.y); bmax = fmaxf(bmax, pl.y);
        tmin = fminf(tmin, pl.w); tmax = fmaxf(tmax, pl.w);
      }
    }
    // ---- the tile anchor in the world frame (fp64)
    const TileAnchor &A = B.anchors[tile];
    d3 D, T1, T2, O;
    if (MODE == 2) {
      D = mkd(A.D[0], A.D[1], A.D[2]); T1 = mkd(A.T1[0], A.T1[1], A.T1[2]);
      T2 = mkd(A.T2[0], A.T2[1], A.T2[2]); O = mkd(A.O[0], A.O[1], A.O[2]);
    } else {
      D = mv(c.R0, mkd(A.D[0], A.D[1], A.D[2]));
      T1 = mv(c.R0, mkd(A.T1[0], A.T1[1], A.T1[2]));
      T2 = mv(c.R0, mkd(A.T2[0], A.T2[1], A.T2[2]));
      O = mkd(c.c0[0], c.c0[1], c.c0[2]);
      if (MODE == 1) O = O + mv(c.R0, mkd(A.O[0], A.O[1], A.O[2]));
    }
    const f3 T1f = tof(T1), T2f = tof(T2);
    // warp pixel box in (a, b) for the conservative warp cull
    float ac, bc, ra, rb, tc = 0.f, rt = 0.f;
    {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        amin = fminf(amin, __shfl_xor_sync(FULL, amin, o));
        amax = fmaxf(amax, __shfl_xor_sync(FULL, amax, o));
        bmin = fminf(bmin, __shfl_xor_sync(FULL, bmin, o));
        bmax = fmaxf(bmax, __shfl_xor_sync(FULL, bmax, o));
        if (MODE == 2) {
          tmin = fminf(tmin, __shfl_xor_sync(FULL, tmin, o));
          tmax = fmaxf(tmax, __shfl_xor_sync(FULL, tmax, o));
        }
      }
      if (amin > amax) { amin = amax = 0.f; bmin = bmax = 0.f; tmin = tmax = 0.f; }  // no valid pixel: the warp is idle
      if (MODE == 2) {  // pixel-time offsets of the warp's rows (rolling shutter)
        tc = 0.5f * (tmin + tmax);
        rt = 0.5f * (tmax - tmin) + 1e-7f * (fabsf(tmin) + fabsf(tmax));
      }
      ac = 0.5f * (amin + amax);
      bc = 0.5f * (bmin + bmax);
      ra = 0.5f * (amax - amin) + 1e-7f * (fabsf(amin) + fabsf(amax));
      rb = 0.5f * (bmax - bmin) + 1e-7f * (fabsf(bmin) + fabsf(bmax));
    }
    if (s == 0 && w == 0 && lane == 0 && len > 0) atomicMax(&B.counters[CNT_MAXLEN], len);
    unsigned long long *stat = B.status + (size_t)slot * NT + pidx0;  // pixel k: + 64 k

    // ---- predecessor peek (pixels already known dead are skipped: same result),
    // then the speculative pass: transmittance from 1 (exact for segment 0)
    bool run[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      run[k] = valid[k] && !(s > 0 && pred_dead(stat + 64 * k, s, epoch));
      L.done[k] = !run[k];
      L.term[k] = false;
      L.T[k] = 1.f;
      L.Cr[k] = L.Cg[k] = L.Cb[k] = L.Dp[k] = 0.f;
    }
    uint32_t n_eval = 0, n_contrib = 0, processed = 0;
    Checkpoints<NP> ck;
    // (rounded up to whole chunks: at most GUT_CK checkpoints per segment)
    const uint32_t ck_step = max(32u, ((uint32_t)B.seg / GUT_CK + 31u) & ~31u);
    store_warp_consts(warp_consts(WarpTbl<MODE>::NF), D, O - mkd(c.c0[0], c.c0[1], c.c0[2]), T1f, T2f, ac, bc, ra,
                      rb, tc, rt, A.fit[w]);
    unsigned long long t_spec = 0, t_lb = 0;  // (trace only: end of the speculative pass / of the look-back)
    float T_pre[NP], T_end[NP];
    bool alive_in[NP], redo[NP], any_redo = false, wredo = false;
    uint32_t act[NP];
    uint32_t e2 = 0, c2 = 0, p2 = 0;
    // pass 0: the speculative pass; pass 1 (only if a pixel needs it): the exact
    // re-run of the pixels that terminate inside this segment.  ONE inlined copy
    // of warp_pass serves both passes (half the blend kernel's code).
    for (int pass = 0; pass < 2; ++pass) {
      warp_pass<MODE, NP>(c, B, s0, s1, L, pass ? e2 : n_eval, pass ? c2 : n_contrib, pass ? p2 : processed,
                          pass == 0 && s > 0 ? stat : nullptr, s, pass == 0 && s > 0 ? &ck : nullptr, ck_step,
                          pass ? act : nullptr);
      if (pass == 1) break;
      if (B.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_spec));
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const unsigned long long Ls = (L.term[k] || (valid[k] && !run[k])) ? GUT_L_DEAD : l_of(L.T[k]);
        T_pre[k] = 1.f;
        alive_in[k] = valid[k];
        if (S > 1 && valid[k]) {
          unsigned long long *st = stat + 64 * k;
          unsigned long long Lpre = 0;
          if (s == 0) {
            st_relaxed(st, st_word(2, epoch, Ls));
          } else {
            st_relaxed(st, st_word(1, epoch, Ls));
            // decoupled look-back over this pixel's earlier segments (integer sums)
            for (int j = s - 1;; --j) {
              const unsigned long long wv = ld_relaxed(st - (size_t)(s - j) * NT);
              const uint32_t flag = (uint32_t)(wv >> 62);
              if (flag == 0 || (uint32_t)((wv >> 40) & 0x3FFFFFu) != (epoch & 0x3FFFFFu)) {
                __nanosleep(256);  // predecessor still running: yield issue slots to the SM's other warps
                ++j;
                continue;
              }
              Lpre += wv & ((1ull << 40) - 1);
              if (Lpre >= GUT_L_DEAD) { Lpre = GUT_L_DEAD; break; }
              if (flag == 2) break;
            }
            const unsigned long long Lin = Lpre + Ls >= GUT_L_DEAD ? GUT_L_DEAD : Lpre + Ls;
            st_relaxed(st, st_word(2, epoch, Lin));
          }
          T_pre[k] = t_of(Lpre);
          alive_in[k] = T_pre[k] >= c.t_min;
        }
        // ---- exact result: scale the speculative sums, or redo the segment from T_pre
        redo[k] = alive_in[k] && s > 0 && (L.term[k] || T_pre[k] * L.T[k] < c.t_min);
        any_redo = any_redo || redo[k];
        T_end[k] = L.T[k];
        if (s > 0 && alive_in[k] && !redo[k]) {
          L.Cr[k] *= T_pre[k]; L.Cg[k] *= T_pre[k]; L.Cb[k] *= T_pre[k]; L.Dp[k] *= T_pre[k];
          T_end[k] = T_pre[k] * L.T[k];
        }
      }
      if (B.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_lb));
      wredo = __any_sync(FULL, any_redo);
      if (!wredo) break;
      // each re-running pixel resumes at the latest checkpoint its exact
      // sequence certainly reached (T_pre T_c >= T_min), or at the segment start;
      // the other pixels' results wait in the checkpoint record meanwhile
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        ck.keepC[k] = make_float4(L.Cr[k], L.Cg[k], L.Cb[k], L.Dp[k]);
        ck.keepTerm[k] = L.term[k];
        L.done[k] = !redo[k];
        L.term[k] = false;
        int ck_k = -1;
        if (redo[k])
          for (int q = ck.n[k] - 1; q >= 0; --q)
            if (T_pre[k] * ck.T[q][k] >= c.t_min) { ck_k = q; break; }
        act[k] = ck_k >= 0 ? s0 + (uint32_t)(ck_k + 1) * ck_step : s0;
        if (ck_k >= 0) {
          const float4 cc = ck.C[ck_k][k];
          L.Cr[k] = T_pre[k] * cc.x; L.Cg[k] = T_pre[k] * cc.y; L.Cb[k] = T_pre[k] * cc.z; L.Dp[k] = T_pre[k] * cc.w;
          L.T[k] = T_pre[k] * ck.T[ck_k][k];
        } else {
          L.Cr[k] = L.Cg[k] = L.Cb[k] = L.Dp[k] = 0.f;
          L.T[k] = T_pre[k];
        }
      }
    }
    if (wredo) {
#pragma unroll
      for (int k = 0; k < NP; ++k)
        if (redo[k]) {
          T_end[k] = L.T[k];
        } else {
          const float4 kc = ck.keepC[k];
          L.Cr[k] = kc.x; L.Cg[k] = kc.y; L.Cb[k] = kc.z; L.Dp[k] = kc.w;
          L.term[k] = ck.keepTerm[k];
        }
      processed += p2;
    }
    n_eval_acc += n_eval;
    n_contrib_acc += n_contrib;
#pragma unroll
    for (int k = 0; k < NP; ++k) n_term_acc += (alive_in[k] && L.term[k]) ? 1u : 0u;
    if (lane == 0) {
      atomicAdd(&B.tile_work[tile].y, processed);
      if (s == 0 && w == 0) B.tile_work[tile].x = len;
    }
    if (B.trace) {
      uint32_t na = 0;  // pixels still alive when the segment starts (exact prefix)
#pragma unroll
      for (int k = 0; k < NP; ++k) na += alive_in[k] ? 1u : 0u;
      const uint32_t n_alive = warp_sum(na);
      const uint32_t e1 = warp_sum(n_eval), e2 = warp_sum(n_contrib);
      if (lane == 0) {
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        // (16-ns units from t_begin: end of the speculative pass | end of the look-back << 16)
        const uint32_t smid = (uint32_t)min((t_spec - t_begin) >> 4, 65535ull) |
                              ((uint32_t)min((t_lb - t_begin) >> 4, 65535ull) << 16);
        const size_t ti = 2 * ((size_t)slot * GUT_BLEND_WARPS + w);
        B.trace[ti] = make_uint4((uint32_t)tile | ((uint32_t)s << 16) | ((uint32_t)w << 29), smid,
                                 (uint32_t)t_begin, (uint32_t)t_end);
        B.trace[ti + 1] = make_uint4(processed, e1, e2, (wredo ? 1u : 0u) | (n_alive << 1));
      }
    }

    // ---- outputs: single segment -> pixels; else partials, successor grants,
    // and the in-order combine by the warp completing the unit's last granted segment
    float Tf[NP];
    bool write = true;
#pragma unroll
    for (int k = 0; k < NP; ++k) Tf[k] = T_end[k];
    if (S > 1) {
      float tmax = 0.f;
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const size_t j = (size_t)slot * NT + pidx0 + 64 * k;
        B.part_c[j] = alive_in[k] ? make_float4(L.Cr[k], L.Cg[k], L.Cb[k], L.Dp[k]) : make_float4(0.f, 0.f, 0.f, 0.f);
        B.part_t[j] = alive_in[k] ? T_end[k] : -1.f;
        const bool alive_out = alive_in[k] && !L.term[k] && T_end[k] >= c.t_min;
        if (alive_out) tmax = fmaxf(tmax, T_end[k]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(FULL, tmax, o));

      __syncwarp();  // the lanes' partials are ordered before lane 0's release below
      uint32_t nseg = 0;
      const uint32_t g0 = (uint32_t)min(S, B.window);
      if (lane == 0) {
        // Successors (queue 2, segments >= g0) are granted only once all of the
        // unit's initial queue-1 segments have been taken by running warps: a
        // successor's look-back then never waits on a segment still sitting in
        // queue 1 (which, with queue 2 served first, could starve when few warps
        // are resident, e.g. next to another frame's kernels).  A completion
        // that sees an initial segment not yet taken skips granting: that
        // segment's own completion sees every initial segment taken and grants.
        if (tmax > 0.f && ld_volatile_u32(&B.q1_taken[unit]) >= g0) {
          // grant segments up to s + max(window, the depth the slowest pixel of
          // the block still needs at its decay so far) (queue 2)
          int ahead = B.window;
          const float n_done = (float)((uint32_t)(s + 1) * (uint32_t)B.seg);
          const float decay = -__logf(tmax);  // over n_done entries
          if (decay < 1e-3f * n_done / (float)B.seg) {
            ahead = S;
          } else {
            const float rem = n_done * __logf(tmax / c.t_min) / decay;
            ahead = max(ahead, (int)fminf(rem / (float)B.seg + 1.f, (float)S));
          }
          if (B.grant_cap > 0) ahead = min(ahead, B.grant_cap);  // (frames in flight: less speculation)
          // granted = g0 + extra (g0 = the up-front grants, extra zeroed per render)
          const uint32_t target = (uint32_t)min(S, s + 1 + ahead) - g0;
          uint32_t g = ld_volatile_u32(&B.granted[unit]);
          while (g < target) {
            const uint32_t prev = atomicCAS(&B.granted[unit], g, target);
            if (prev == g) {
              const uint32_t n = target - g, pos = atomicAdd(&B.counters[CNT_Q_ALLOC2], n);
              for (uint32_t k = 0; k < n; ++k) atomicExch(&B.q2[pos + k], (uint32_t)unit + 1u);
              break;
            }
            g = prev;
          }
        }
        // completion count with acq_rel: releases this segment's partials and
        // grants, acquires those of every segment counted before it
        const uint32_t d = atom_add_acq_rel(&B.unit_done[unit], 1u) + 1u;
        const uint32_t g = g0 + ld_acquire_u32(&B.granted[unit]);
        nseg = d == g ? g : 0u;
      }
      nseg = __shfl_sync(FULL, nseg, 0);
      write = nseg != 0;
      if (write) {
        __syncwarp();  // lane 0's acquire orders the other lanes' loads (L2 reads, __ldcg)
        const uint32_t first = B.seg_base[tile];
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          float Cr = 0.f, Cg = 0.f, Cb = 0.f, Dp = 0.f, T = 1.f;
#pragma unroll 8
          for (uint32_t q = 0; q < nseg; ++q) {  // (unrolled: loads in flight, sums in order)
            const size_t jj = (size_t)(first + q) * NT + pidx0 + 64 * k;
            const float4 pc = __ldcg(&B.part_c[jj]);
            const float pt = __ldcg(&B.part_t[jj]);
            Cr += pc.x; Cg += pc.y; Cb += pc.z; Dp += pc.w;
            if (pt >= 0.f) T = pt;
          }
          L.Cr[k] = Cr; L.Cg[k] = Cg; L.Cb[k] = Cb; L.Dp[k] = Dp; Tf[k] = T;
        }
      }
    }
    if (write) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        if (!inside[k]) continue;
        const size_t p = (size_t)py[k] * c.width + px[k];
        if (valid[k]) {
          B.rgb[3 * p] = L.Cr[k] + Tf[k] * c.bg[0];
          B.rgb[3 * p + 1] = L.Cg[k] + Tf[k] * c.bg[1];
          B.rgb[3 * p + 2] = L.Cb[k] + Tf[k] * c.bg[2];
          B.alpha[p] = 1.f - Tf[k];
          if (B.depth) B.depth[p] = L.Dp[k];
        } else {
          B.rgb[3 * p] = c.bg[0];
          B.rgb[3 * p + 1] = c.bg[1];
          B.rgb[3 * p + 2] = c.bg[2];
          B.alpha[p] = 0.f;
          if (B.depth) B.depth[p] = 0.f;
        }
      }
      if (lane == 0) atomicAdd(&B.counters[CNT_Q_FINISHED], 1u);  // termination count only (no data)
    }
  }
  // ---- statistics (once per warp)
  {
    const unsigned long long e1 = warp_sum((unsigned long long)n_eval_acc);
    const unsigned long long e2 = warp_sum((unsigned long long)n_contrib_acc);
    const unsigned long long e3 = warp_sum((unsigned long long)n_term_acc);
    if (lane == 0 && (e1 | e2 | e3)) {
      atomicAdd(reinterpret_cast<unsigned long long *>(&B.counters[CNT_PAIRS_EVAL]), e1);
      atomicAdd(reinterpret_cast<unsigned long long *>(&B.counters[CNT_PAIRS_CONTRIB]), e2);
      atomicAdd(reinterpret_cast<unsigned long long *>(&B.counters[CNT_TERMINATED]), e3);
    }
  }
}

template <int MODE>
static void blend_launch(const DevCam &cam, const BlendBufs &b, cudaStream_t st) {
  constexpr size_t smem = blend_smem_bytes<MODE>();
  // per device, thread-safe (a process may drive several devices): the
  // dynamic shared-memory attribute is a per-device setting
  static std::once_flag once[GUT_MAX_DEVICES];
  static int grids[GUT_MAX_DEVICES];
  int dev = 0;
  cudaGetDevice(&dev);
  dev = min(dev, GUT_MAX_DEVICES - 1);
  static int smss[GUT_MAX_DEVICES];
  std::call_once(once[dev], [&] {
    cudaFuncSetAttribute(blend_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, blend_kernel<MODE>, GUT_BLEND_CTA, smem);
    grids[dev] = max(1, sms) * max(1, per);
    smss[dev] = max(1, sms);
    // tuning knob: a smaller persistent grid leaves SMs to the next frame's kernels
    if (const char *e = getenv("GUT_BLEND_GRID")) grids[dev] = max(1, min(grids[dev], atoi(e)));
  });
  // frames in flight (b.grid_x4 > 0): 1.25 CTAs per SM measured best for
  // throughput (bench frame, 4 in flight: 880 vs 842 frames/s, e2e 859 vs
  // 838; one frame alone would take 1.55 instead of 1.29 ms)
  const int grid = b.grid_x4 > 0 ? max(1, min(grids[dev], smss[dev] * b.grid_x4 / 4)) : grids[dev];
  blend_kernel<MODE><<<grid, GUT_BLEND_CTA, smem, st>>>(cam, b);
}

void launch_blend(const DevCam &cam, const BlendBufs &b, cudaStream_t st) {
  if (cam.model == CAM_ORTHO) blend_launch<1>(cam, b, st);
  else if (cam.shutter != SH_GLOBAL) blend_launch<2>(cam, b, st);
  else blend_launch<0>(cam, b, st);
}

// ---------------------------------------------------------------- "Ours (sorted)"
// PAPER L205-212 (reading R28): per-ray MLAB k-buffer of KB hits.  The buffer
// carries state along the whole list, so a ray's list cannot be split into
// independently composited segments: the unit of work is one warp on one 8x4
// pixel block (one pixel per lane, the buffer in registers) over its tile's
// whole list, taken from queue 1 (tiles in decreasing list length).  The
// staging, the two-stage warp cull and the per-pixel Eq. 11 evaluation are
// those of the global-order kernel; an evaluated hit (alpha >= alpha_min,
// tau_max > 0) enters the buffer and the closest of the KB + 1 pending hits
// is blended; at the end of the list the buffer is blended near to far.
template <int MODE, int KB>
__global__ __launch_bounds__(GUT_BLEND_CTA, GUT_BLEND_CTAS) void blend_kbuf_kernel(DevCam c, BlendBufs B) {
  constexpr int NT = GUT_TILE_PX;
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  uint32_t n_eval_acc = 0, n_contrib_acc = 0, n_term_acc = 0;
  const uint32_t n_init = B.counters[CNT_Q_NINIT];
  for (;;) {
    uint32_t h = 0;
    if (lane == 0) h = atomicAdd(&B.counters[CNT_Q_HEAD1], 1u);
    h = __shfl_sync(FULL, h, 0);
    if (h >= n_init) break;
    const int unit = (int)(B.q1[h] & 0xFFFFFFu);
    const int tile = unit / GUT_KBUF_UNITS, w = unit % GUT_KBUF_UNITS;
    const uint2 rg = B.ranges[tile];
    const uint32_t start = rg.y > rg.x ? rg.x : 0u, end = rg.y > rg.x ? rg.y : 0u;
    int px, py;
    tile_pixel(tile, c.tiles_x, w, lane, px, py);  // = rays_kernel's thread w * 32 + lane
    const bool inside = px < c.width && py < c.height;
    const float4 pl = B.pix[(size_t)tile * NT + w * 32 + lane];
    LanePx<1> L;
    L.a[0] = pl.x; L.b[0] = pl.y; L.snorm[0] = pl.z; L.beta[0] = pl.w;
    const bool valid = inside && pl.z > 0.f;
    float amin = valid ? pl.x : 3e38f, amax = valid ? pl.x : -3e38f;
    float bmin = valid ? pl.y : 3e38f, bmax = valid ? pl.y : -3e38f;
    float tmin = valid ? pl.w : 3e38f, tmax = valid ? pl.w : -3e38f;
    const TileAnchor &A = B.anchors[tile];
    d3 D, T1, T2, O;
    if (MODE == 2) {
      D = mkd(A.D[0], A.D[1], A.D[2]); T1 = mkd(A.T1[0], A.T1[1], A.T1[2]);
      T2 = mkd(A.T2[0], A.T2[1], A.T2[2]); O = mkd(A.O[0], A.O[1], A.O[2]);
    } else {
      D = mv(c.R0, mkd(A.D[0], A.D[1], A.D[2]));
      T1 = mv(c.R0, mkd(A.T1[0], A.T1[1], A.T1[2]));
      T2 = mv(c.R0, mkd(A.T2[0], A.T2[1], A.T2[2]));
      O = mkd(c.c0[0], c.c0[1], c.c0[2]);
      if (MODE == 1) O = O + mv(c.R0, mkd(A.O[0], A.O[1], A.O[2]));
    }
    const f3 T1f = tof(T1), T2f = tof(T2);
    float ac, bc, ra, rb, tc = 0.f, rt = 0.f;
    {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        amin = fminf(amin, __shfl_xor_sync(FULL, amin, o));
        amax = fmaxf(amax, __shfl_xor_sync(FULL, amax, o));
        bmin = fminf(bmin, __shfl_xor_sync(FULL, bmin, o));
        bmax = fmaxf(bmax, __shfl_xor_sync(FULL, bmax, o));
        if (MODE == 2) {
          tmin = fminf(tmin, __shfl_xor_sync(FULL, tmin, o));
          tmax = fmaxf(tmax, __shfl_xor_sync(FULL, tmax, o));
        }
      }
      if (amin > amax) { amin = amax = 0.f; bmin = bmax = 0.f; tmin = tmax = 0.f; }
      if (MODE == 2) {
        tc = 0.5f * (tmin + tmax);
        rt = 0.5f * (tmax - tmin) + 1e-7f * (fabsf(tmin) + fabsf(tmax));
      }
      ac = 0.5f * (amin + amax);
      bc = 0.5f * (bmin + bmax);
      ra = 0.5f * (amax - amin) + 1e-7f * (fabsf(amin) + fabsf(amax));
      rb = 0.5f * (bmax - bmin) + 1e-7f * (fabsf(bmin) + fabsf(bmax));
    }
    if (w == 0 && lane == 0 && end > start) atomicMax(&B.counters[CNT_MAXLEN], end - start);
    L.done[0] = !valid;
    L.term[0] = false;
    L.T[0] = 1.f;
    L.Cr[0] = L.Cg[0] = L.Cb[0] = L.Dp[0] = 0.f;
    KBuf<KB> kb;
#pragma unroll
    for (int i = 0; i < KB; ++i) { kb.t[i] = -INFINITY; kb.a[i] = 0.f; kb.g[i] = 0u; }
    uint32_t n_eval = 0, n_contrib = 0, processed = 0;
    // (the 8x4 block w is half (w >> 1) & 1 of the 8x8 fit block (w & 1) | ((w >> 2) << 1))
    store_warp_consts(warp_consts(WarpTbl<MODE>::NF), D, O - mkd(c.c0[0], c.c0[1], c.c0[2]), T1f, T2f, ac, bc, ra,
                      rb, tc, rt, A.fit[(w & 1) | ((w >> 2) << 1)]);
    warp_pass<MODE, 1, KB>(c, B, start, end, L, n_eval, n_contrib, processed,
                           nullptr, 0, nullptr, 0, nullptr, &kb, (w >> 1) & 1);
    // end of the list: the pending hits near to far (colours gathered up front)
    if (!L.done[0]) {
      float4 cc[KB];
#pragma unroll
      for (int i = 0; i < KB; ++i)
        cc[i] = kb.t[i] > -INFINITY ? __ldg(&B.payload[(size_t)GUT_PAYLOAD_F4 * kb.g[i] + 4])
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int i = 0; i < KB; ++i) {
        if (L.done[0] || !(kb.t[i] > -INFINITY)) continue;
        const float Tn = L.T[0] * (1.f - kb.a[i]);
        if (Tn < c.t_min) { L.done[0] = L.term[0] = true; continue; }
        const float wgt = kb.a[i] * L.T[0];
        L.Cr[0] = fmaf(wgt, cc[i].x, L.Cr[0]);
        L.Cg[0] = fmaf(wgt, cc[i].y, L.Cg[0]);
        L.Cb[0] = fmaf(wgt, cc[i].z, L.Cb[0]);
        L.Dp[0] = fmaf(wgt, kb.t[i], L.Dp[0]);
        L.T[0] = Tn;
        ++n_contrib;
      }
    }
    n_eval_acc += n_eval;
    n_contrib_acc += n_contrib;
    n_term_acc += (valid && L.term[0]) ? 1u : 0u;
    if (lane == 0) {
      atomicAdd(&B.tile_work[tile].y, processed);
      if (w == 0) B.tile_work[tile].x = end - start;
    }
    if (inside) {
      const size_t p = (size_t)py * c.width + px;
      const float Tf = valid ? L.T[0] : 1.f;
      B.rgb[3 * p] = (valid ? L.Cr[0] : 0.f) + Tf * c.bg[0];
      B.rgb[3 * p + 1] = (valid ? L.Cg[0] : 0.f) + Tf * c.bg[1];
      B.rgb[3 * p + 2] = (valid ? L.Cb[0] : 0.f) + Tf * c.bg[2];
      B.alpha[p] = 1.f - Tf;
      if (B.depth) B.depth[p] = valid ? L.Dp[0] : 0.f;
    }
  }
  const unsigned long long e1 = warp_sum((unsigned long long)n_eval_acc);
  const unsigned long long e2 = warp_sum((unsigned long long)n_contrib_acc);
  const unsigned long long e3 = warp_sum((unsigned long long)n_term_acc);
  if (lane == 0 && (e1 | e2 | e3)) {
    atomicAdd(reinterpret_cast<unsigned long long *>(&B.counters[CNT_PAIRS_EVAL]), e1);
    atomicAdd(reinterpret_cast<unsigned long long *>(&B.counters[CNT_PAIRS_CONTRIB]), e2);
    atomicAdd(reinterpret_cast<unsigned long long *>(&B.counters[CNT_TERMINATED]), e3);
  }
}

template <int MODE, int KB>
static void blend_kbuf_launch(const DevCam &cam, const BlendBufs &b, cudaStream_t st) {
  constexpr size_t smem = blend_smem_bytes<MODE>();
  // per device, thread-safe (a process may drive several devices): the
  // dynamic shared-memory attribute is a per-device setting
  static std::once_flag once[GUT_MAX_DEVICES];
  static int grids[GUT_MAX_DEVICES], smss[GUT_MAX_DEVICES];
  int dev = 0;
  cudaGetDevice(&dev);
  dev = min(dev, GUT_MAX_DEVICES - 1);
  std::call_once(once[dev], [&] {
    cudaFuncSetAttribute(blend_kbuf_kernel<MODE, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, blend_kbuf_kernel<MODE, KB>, GUT_BLEND_CTA, smem);
    grids[dev] = max(1, sms) * max(1, per);
    smss[dev] = max(1, sms);
  });
  // frames in flight: the smaller persistent grid, as blend_launch
  const int grid = b.grid_x4 > 0 ? max(1, min(grids[dev], smss[dev] * b.grid_x4 / 4)) : grids[dev];
  blend_kbuf_kernel<MODE, KB><<<grid, GUT_BLEND_CTA, smem, st>>>(cam, b);
}

template <int KB>
static void blend_kbuf_modes(const DevCam &cam, const BlendBufs &b, cudaStream_t st) {
  if (cam.model == CAM_ORTHO) blend_kbuf_launch<1, KB>(cam, b, st);
  else if (cam.shutter != SH_GLOBAL) blend_kbuf_launch<2, KB>(cam, b, st);
  else blend_kbuf_launch<0, KB>(cam, b, st);
}

void launch_blend_kbuf(const DevCam &cam, const BlendBufs &b, cudaStream_t st) {
  switch (cam.kbuf) {
    case 1: blend_kbuf_modes<1>(cam, b, st); break;
    case 2: blend_kbuf_modes<2>(cam, b, st); break;
    case 4: blend_kbuf_modes<4>(cam, b, st); break;
    case 8: blend_kbuf_modes<8>(cam, b, st); break;
    case 16: blend_kbuf_modes<16>(cam, b, st); break;
    default: break;  // validated by the ABI
  }
}

}  // namespace gut
