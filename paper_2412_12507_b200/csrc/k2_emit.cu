// k2_emit.cu — K2 (scan + key emission, the paper's "Duplicate") and K4
// (tile ranges), sm_100a.
//
// K2 walks the visible Gaussians in depth order (output of the depth passes
// of K3).  A CTA owns 1024 consecutive Gaussians: it scans their tile counts,
// gets its global key offset by decoupled look-back, then emits its keys with
// one OUTPUT slot per thread (slot -> Gaussian by binary search in the local
// scan, -> tile by walking the Gaussian's tile-row spans), so the writes of
// (tile id, Gaussian id) are coalesced and large Gaussians do not serialise a
// thread.  Row spans come from row_span(), the same function K1 counted with,
// so counts and emitted keys agree bit for bit.  Because emission follows
// depth order and the tile passes are stable, equal-tile keys stay ordered by
// (depth, index) — the tie rule of PAPER L208 / DESIGN.md R13.
// K2 also builds the two 8-bit digit histograms of the tile ids.
//
// K4 marks [start, end) of every tile in the sorted key array (Alg. 1's
// tiles, "same tiling ... as 3DGS").
#include "launch.h"

namespace gut {

__global__ __launch_bounds__(GUT_EMIT_THREADS) void emit_kernel(
    const uint32_t *__restrict__ order, const uint32_t *n_vis_p, const uint32_t *__restrict__ tiles,
    const float4 *__restrict__ ell, const double2 *__restrict__ ell64, int tiles_x, int tile_cull,
    uint32_t *__restrict__ out_tile,
    uint32_t *__restrict__ out_gid, uint32_t cap_k, uint32_t *counters, unsigned long long *status,
    uint32_t epoch) {
  __shared__ uint32_t s_incl[GUT_EMIT_PART];
  __shared__ uint32_t s_gid[GUT_EMIT_PART];
  __shared__ float4 s_e0[GUT_EMIT_PART];  // vx, vy, cxx, cxy
  __shared__ float4 s_e1[GUT_EMIT_PART];  // cyy, k2, rect0, rect1
  __shared__ uint32_t s_hist[2][256];
  __shared__ uint32_t s_tmp[16];
  __shared__ uint32_t s_part, s_prefix;

  const uint32_t n = *n_vis_p;
  if (threadIdx.x == 0) s_part = atomicAdd(&counters[CNT_TICKETS + 4], 1u);
  for (int j = threadIdx.x; j < 512; j += GUT_EMIT_THREADS) (&s_hist[0][0])[j] = 0;
  __syncthreads();
  const uint32_t part = s_part;
  const uint32_t base = part * GUT_EMIT_PART;
  if (base >= n) return;

  // load 4 consecutive Gaussians per thread, thread-local inclusive scan
  uint32_t c[GUT_EMIT_ITEMS], acc = 0;
#pragma unroll
  for (int j = 0; j < GUT_EMIT_ITEMS; ++j) {
    uint32_t li = threadIdx.x * GUT_EMIT_ITEMS + j, gi = base + li;
    uint32_t g = 0, cnt = 0;
    if (gi < n) {
      g = __ldg(&order[gi]);
      cnt = __ldg(&tiles[g]);
      s_e0[li] = __ldg(&ell[2 * g]);
      s_e1[li] = __ldg(&ell[2 * g + 1]);
    }
    s_gid[li] = g;
    acc += cnt;
    c[j] = acc;
  }
  // block exclusive scan of per-thread sums
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = acc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_tmp[w] = x;
  __syncthreads();
  uint32_t wpre = 0, total = 0;
  for (int ww = 0; ww < GUT_EMIT_THREADS / 32; ++ww) {
    if (ww < w) wpre += s_tmp[ww];
    total += s_tmp[ww];
  }
  const uint32_t texcl = wpre + x - acc;
#pragma unroll
  for (int j = 0; j < GUT_EMIT_ITEMS; ++j) s_incl[threadIdx.x * GUT_EMIT_ITEMS + j] = texcl + c[j];
  if (threadIdx.x == 0) s_prefix = lookback(status, 1, (int)part, 0, total, epoch);
  __syncthreads();
  const uint32_t prefix = s_prefix;

  // one output slot per thread per round
  for (uint32_t e = threadIdx.x; e < total; e += GUT_EMIT_THREADS) {
    // Gaussian owning slot e: first li with s_incl[li] > e
    int lo = 0, hi = GUT_EMIT_PART - 1;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (s_incl[mid] > e) hi = mid; else lo = mid + 1;
    }
    uint32_t j = e - (lo > 0 ? s_incl[lo - 1] : 0u);
    float4 a = s_e0[lo], b = s_e1[lo];
    Ell el;
    el.vx = a.x; el.vy = a.y; el.cxx = a.z; el.cxy = a.w; el.cyy = b.x; el.k2 = b.y;
    uint32_t r0 = __float_as_uint(b.z), r1 = __float_as_uint(b.w);
    el.x0 = (int)(r0 & 0xFFFF); el.y0 = (int)(r0 >> 16); el.x1 = (int)(r1 & 0xFFFF); el.y1 = (int)(r1 >> 16);
    uint32_t tile = 0;
    if (el.k2 >= 0.f) {
      for (int ty = el.y0; ty <= el.y1; ++ty) {
        int l, h;
        row_span(el, ty, tile_cull, l, h);
        uint32_t cnt = (uint32_t)max(h - l + 1, 0);
        if (j < cnt) { tile = (uint32_t)(ty * tiles_x + l + (int)j); break; }
        j -= cnt;
      }
    } else {  // "wide" Gaussian: fp64 ellipse written by the fp64 K1 kernel
      const uint32_t g = s_gid[lo];
      const double2 q0 = ell64[3 * g], q1 = ell64[3 * g + 1], q2 = ell64[3 * g + 2];
      EllD ed;
      ed.vx = q0.x; ed.vy = q0.y; ed.cxx = q1.x; ed.cxy = q1.y; ed.cyy = q2.x; ed.k2 = q2.y;
      ed.x0 = el.x0; ed.y0 = el.y0; ed.x1 = el.x1; ed.y1 = el.y1;
      for (int ty = ed.y0; ty <= ed.y1; ++ty) {
        int l, h;
        row_span(ed, ty, tile_cull, l, h);
        uint32_t cnt = (uint32_t)max(h - l + 1, 0);
        if (j < cnt) { tile = (uint32_t)(ty * tiles_x + l + (int)j); break; }
        j -= cnt;
      }
    }
    uint32_t pos = prefix + e;
    if (pos < cap_k) {
      out_tile[pos] = tile;
      out_gid[pos] = s_gid[lo];
      atomicAdd(&s_hist[0][tile & 255u], 1u);
      atomicAdd(&s_hist[1][(tile >> 8) & 255u], 1u);
    } else {
      counters[CNT_OVERFLOW] = 1u;
    }
  }
  __syncthreads();
  for (int jj = threadIdx.x; jj < 512; jj += GUT_EMIT_THREADS) {
    uint32_t v = (&s_hist[0][0])[jj];
    if (v) atomicAdd(&counters[CNT_HIST_TILE + jj], v);
  }
}

__global__ void ranges_kernel(const uint32_t *__restrict__ tile_sorted, const uint32_t *counters, uint32_t cap_k,
                              uint2 *__restrict__ ranges) {
  const unsigned long long Kfull = *reinterpret_cast<const unsigned long long *>(&counters[CNT_K]);
  const uint32_t K = (uint32_t)min(Kfull, (unsigned long long)cap_k);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) {
    uint32_t t = tile_sorted[k];
    if (k == 0 || tile_sorted[k - 1] != t) ranges[t].x = k;
    if (k == K - 1 || tile_sorted[k + 1] != t) ranges[t].y = k + 1;
  }
}

void launch_emit(const uint32_t *order, const uint32_t *n_vis, uint32_t n_upper, const uint32_t *tiles,
                 const float4 *ell, const double2 *ell64, int tiles_x, int tile_cull, uint32_t *out_tile,
                 uint32_t *out_gid,
                 uint32_t cap_k, uint32_t *counters, unsigned long long *status, uint32_t epoch,
                 cudaStream_t st) {
  if (n_upper == 0) return;
  unsigned blocks = (n_upper + GUT_EMIT_PART - 1) / GUT_EMIT_PART;
  emit_kernel<<<blocks, GUT_EMIT_THREADS, 0, st>>>(order, n_vis, tiles, ell, ell64, tiles_x, tile_cull, out_tile, out_gid,
                                                   cap_k, counters, status, epoch);
}

void launch_ranges(const uint32_t *tile_sorted, const uint32_t *counters, uint32_t cap_k, uint2 *ranges,
                   cudaStream_t st) {
  ranges_kernel<<<148 * 8, 256, 0, st>>>(tile_sorted, counters, cap_k, ranges);
}

}  // namespace gut
