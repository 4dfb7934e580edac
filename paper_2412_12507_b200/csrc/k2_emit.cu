// k2_emit.cu — K2 (scan + key emission, the paper's "Duplicate"), sm_100a.
// (K4, the tile ranges, is fused into the final tile pass: k3_sort.cu.)
//
// K2 walks the visible Gaussians in depth order (output of the depth passes
// of K3) in partitions of 1024: per-partition key totals and their scan give
// every partition its first key slot; the emission then reads one 4-byte tile
// code per Gaussian (K1, gut_internal.cuh ell_tile_code): small Gaussians
// (tile rectangle <= 3x3) emit straight from the hit mask, big ones are
// expanded row by row by a warp with row_span(), the function K1 counted
// with, so counts and emitted keys agree bit for bit.  Because emission
// follows depth order and the tile passes are stable, equal-tile keys stay
// ordered by (depth, index) — the tie rule of PAPER L208 / DESIGN.md R13.
// K2 also builds the two 8-bit digit histograms of the tile ids.
#include "launch.h"

namespace gut {

// block-wide exclusive scan of two values at once (256 threads)
__device__ __forceinline__ void block_scan2(uint32_t x, uint32_t y, uint32_t *s_tmp, uint32_t &ex, uint32_t &ey,
                                            uint32_t &tx, uint32_t &ty) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t a = x, b = y;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t pa = __shfl_up_sync(0xffffffffu, a, o), pb = __shfl_up_sync(0xffffffffu, b, o);
    if (lane >= o) { a += pa; b += pb; }
  }
  if (lane == 31) { s_tmp[w] = a; s_tmp[8 + w] = b; }
  __syncthreads();
  uint32_t wa = 0, wb = 0;
  tx = ty = 0;
#pragma unroll
  for (int ww = 0; ww < GUT_EMIT_THREADS / 32; ++ww) {
    const uint32_t va = s_tmp[ww], vb = s_tmp[8 + ww];
    if (ww < w) { wa += va; wb += vb; }
    tx += va; ty += vb;
  }
  ex = wa + a - x;
  ey = wb + b - y;
  __syncthreads();  // s_tmp reusable
}

// keys staged in shared memory per CTA (written out as one coalesced run);
// a partition with more keys writes them straight to global memory
#ifndef GUT_EMIT_STAGE
#define GUT_EMIT_STAGE 4096
#endif

// A CTA owns GUT_EMIT_PART consecutive Gaussians (depth order); its first
// key slot comes from emit_count_kernel + emit_scan_kernel (per-partition key
// totals, scanned), so no CTA waits on another.  K2 reads only the 4-byte
// tile code per Gaussian (gut_internal.cuh ell_tile_code): a Gaussian whose
// tile rectangle is at most 3x3 emits its keys straight from the hit mask;
// the others ("big", a few percent, clustered at the front of the depth
// order) go to a global list that emit_big_kernel expands over the whole GPU.
__device__ __forceinline__ void emit_key(uint32_t pos, uint32_t tile, uint32_t g, uint32_t cap_k, uint32_t *out_tile,
                                         uint32_t *out_gid, uint32_t (*s_hist)[256], uint32_t *counters) {
  if (pos < cap_k) {
    out_tile[pos] = tile;
    out_gid[pos] = g;
    atomicAdd(&s_hist[0][tile & 255u], 1u);
    atomicAdd(&s_hist[1][(tile >> 8) & 255u], 1u);
  } else {
    counters[CNT_OVERFLOW] = 1u;
    counters[CNT_STICKY_OVERFLOW] = 1u;  // latched until the host reads it (gut_check)
  }
}

__global__ __launch_bounds__(GUT_EMIT_THREADS) void emit_kernel(
    const uint32_t *__restrict__ order, const uint32_t *n_vis_p, const uint32_t *__restrict__ tiles,
    const float4 *__restrict__ ell, const double2 *__restrict__ ell64, int tiles_x, int tile_cull,
    uint32_t *__restrict__ out_tile, uint32_t *__restrict__ out_gid, uint32_t cap_k, uint32_t *counters,
    const uint32_t *__restrict__ part_off, uint2 *__restrict__ big_list, const uint32_t *__restrict__ codes) {
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ uint32_t s_hist[2][256];
  __shared__ uint32_t s_tmp[16];
  __shared__ uint32_t s_kt[GUT_EMIT_STAGE], s_kg[GUT_EMIT_STAGE];  // staged (tile, gid) keys of the CTA

  const uint32_t n = *n_vis_p;
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t base = blockIdx.x * GUT_EMIT_PART;
  if (base >= n) return;
  const uint32_t prefix = __ldg(&part_off[blockIdx.x]);
  for (int j = tid; j < 512; j += GUT_EMIT_THREADS) (&s_hist[0][0])[j] = 0;

  // ---- codes and counts (4 consecutive Gaussians per thread), block scan
  uint32_t g[GUT_EMIT_ITEMS], code[GUT_EMIT_ITEMS], sc = 0;
#pragma unroll
  for (int j = 0; j < GUT_EMIT_ITEMS; ++j) {
    const uint32_t gi = base + tid * GUT_EMIT_ITEMS + j;
    g[j] = 0;
    code[j] = 0;
    if (gi < n) {
      g[j] = __ldg(&order[gi]);
      code[j] = codes ? __ldg(&codes[gi]) : __ldg(&tiles[g[j]]);
    }
    sc += code_count(code[j]);
  }
  uint32_t ex, ey, total, ty_;
  block_scan2(sc, 0u, s_tmp, ex, ey, total, ty_);  // (its barriers also order the s_hist reset)

  // ---- small Gaussians: keys from the mask, row-major (staged in shared
  // memory when the CTA's keys fit, then written out as one coalesced run)
  const bool staged = total <= GUT_EMIT_STAGE;
  uint32_t pos = prefix + ex, lpos = ex;
  bool big[GUT_EMIT_ITEMS];
  uint32_t bpos[GUT_EMIT_ITEMS];
#pragma unroll
  for (int j = 0; j < GUT_EMIT_ITEMS; ++j) {
    big[j] = (code[j] >> 31) != 0u;
    bpos[j] = pos;
    if (!big[j] && code[j]) {
      const bool m4 = (code[j] >> 30) & 1u;  // 4x4 mask format
      const uint32_t x0 = m4 ? (code[j] >> 16) & 0x7Fu : (code[j] >> 9) & 0x7FFu;
      const uint32_t y0 = m4 ? (code[j] >> 23) & 0x7Fu : (code[j] >> 20) & 0x3FFu;
      const uint32_t cw = m4 ? 4u : 3u;
      for (uint32_t m = code[j] & (m4 ? 0xFFFFu : 0x1FFu); m; m &= m - 1) {
        const uint32_t b = (uint32_t)(__ffs(m) - 1);
        // row = b / cw without an integer division (cw = 3: b < 9, (11 b) >> 5 = b / 3)
        const uint32_t row = m4 ? b >> 2 : (b * 11u) >> 5;
        const uint32_t tile = (y0 + row) * (uint32_t)tiles_x + x0 + (b - row * cw);
        if (staged) {
          s_kt[lpos] = tile;
          s_kg[lpos] = g[j];
        } else {
          emit_key(pos, tile, g[j], cap_k, out_tile, out_gid, s_hist, counters);
        }
        ++pos;
        ++lpos;
      }
    } else {
      const uint32_t cnt = code_count(code[j]);
      if (staged)  // a big Gaussian's slots (emit_big_kernel writes them): not counted here
        for (uint32_t q = 0; q < cnt; ++q) s_kt[lpos + q] = 0xFFFFFFFFu;
      pos += cnt;
      lpos += cnt;
    }
  }
  // ---- big Gaussians: appended to a global list (depth order clusters them in
  // the first partitions) and expanded by emit_big_kernel over the whole GPU
#pragma unroll
  for (int j = 0; j < GUT_EMIT_ITEMS; ++j) {
    const uint32_t bm = __ballot_sync(FULL, big[j]);
    if (!bm) continue;
    uint32_t slot = 0;
    if (lane == __ffs(bm) - 1) slot = atomicAdd(&counters[CNT_NBIG], (uint32_t)__popc(bm));
    slot = __shfl_sync(FULL, slot, __ffs(bm) - 1) + (uint32_t)__popc(bm & ((1u << lane) - 1u));
    if (big[j]) big_list[slot] = make_uint2(g[j], bpos[j]);
  }
  __syncthreads();
  if (staged) {  // the CTA's run [prefix, prefix + total): a big Gaussian's slots hold
                 // a sentinel here, overwritten by emit_big_kernel (launched after)
    const uint32_t lim = prefix < cap_k ? min(total, cap_k - prefix) : 0u;
    // (the tile-digit histograms count only the keys written: a truncated
    // list must not see more keys than it holds)
    for (uint32_t q = tid; q < lim; q += GUT_EMIT_THREADS) {
      const uint32_t t = s_kt[q];
      out_tile[prefix + q] = t;
      out_gid[prefix + q] = s_kg[q];
      if (t != 0xFFFFFFFFu) {
        atomicAdd(&s_hist[0][t & 255u], 1u);
        atomicAdd(&s_hist[1][(t >> 8) & 255u], 1u);
      }
    }
    if (lim < total && tid == 0) {
      counters[CNT_OVERFLOW] = 1u;
      counters[CNT_STICKY_OVERFLOW] = 1u;  // latched until the host reads it (gut_check)
    }
    __syncthreads();  // (the histogram atomics above before the flush)
  }
  for (int jj = tid; jj < 512; jj += GUT_EMIT_THREADS) {
    const uint32_t v = (&s_hist[0][0])[jj];
    if (v) atomicAdd(&counters[CNT_HIST_TILE + jj], v);
  }
}

// big Gaussians (tile rectangle > 3x3): one warp each, grid-stride over the
// list, a lane per tile row (row_span), a warp scan places the rows, the keys
// are written by consecutive lanes
__global__ __launch_bounds__(GUT_EMIT_THREADS) void emit_big_kernel(
    const uint2 *__restrict__ big_list, const float4 *__restrict__ ell, const double2 *__restrict__ ell64,
    int tiles_x, int tile_cull, uint32_t *__restrict__ out_tile, uint32_t *__restrict__ out_gid, uint32_t cap_k,
    uint32_t *counters) {
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ uint32_t s_hist[2][256];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int j = tid; j < 512; j += GUT_EMIT_THREADS) (&s_hist[0][0])[j] = 0;
  __syncthreads();
  const uint32_t nbig = counters[CNT_NBIG];
  const uint32_t wstride = gridDim.x * (GUT_EMIT_THREADS / 32);
  for (uint32_t bi = blockIdx.x * (GUT_EMIT_THREADS / 32) + (uint32_t)(tid >> 5); bi < nbig; bi += wstride) {
    const uint2 bg = big_list[bi];
    const uint32_t gg = bg.x;
    uint32_t kpos = bg.y;
    const float4 a = __ldg(&ell[2 * gg]), b = __ldg(&ell[2 * gg + 1]);
    const uint32_t r0w = __float_as_uint(b.z), r1w = __float_as_uint(b.w);
    const int x0 = (int)(r0w & 0xFFFF), y0 = (int)(r0w >> 16), x1 = (int)(r1w & 0xFFFF), y1 = (int)(r1w >> 16);
    const bool wide = b.y < 0.f;
    Ell el;
    EllD ed;
    if (!wide) {
      el.vx = a.x; el.vy = a.y; el.cxx = a.z; el.cxy = a.w; el.cyy = b.x; el.k2 = b.y;
      el.x0 = x0; el.y0 = y0; el.x1 = x1; el.y1 = y1;
    } else {  // "wide" Gaussian: fp64 ellipse written by the fp64 K1 kernel
      const double2 q0 = ell64[3 * gg], q1 = ell64[3 * gg + 1], q2 = ell64[3 * gg + 2];
      ed.vx = q0.x; ed.vy = q0.y; ed.cxx = q1.x; ed.cxy = q1.y; ed.cyy = q2.x; ed.k2 = q2.y;
      ed.x0 = x0; ed.y0 = y0; ed.x1 = x1; ed.y1 = y1;
    }
    for (int rb = y0; rb <= y1; rb += 32) {
      const int ty = rb + lane;
      int l = 0, h = -1;
      if (ty <= y1) {
        if (!wide) row_span(el, ty, tile_cull, l, h);
        else row_span(ed, ty, tile_cull, l, h);
      }
      const uint32_t cnt = (uint32_t)max(h - l + 1, 0);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t tot = __shfl_sync(FULL, incl, 31);
      for (uint32_t e0 = 0; e0 < tot; e0 += 32) {  // warp-uniform trip count (full-mask shuffles)
        const uint32_t e = e0 + (uint32_t)lane;
        int lo = 0;  // first row (lane) with incl > e
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const uint32_t v = __shfl_sync(FULL, incl, lo + step - 1);
          if (v <= e) lo += step;
        }
        const uint32_t ex_lo = __shfl_sync(FULL, incl - cnt, lo);
        const int l_lo = __shfl_sync(FULL, l, lo);
        if (e < tot) {
          const uint32_t tile = (uint32_t)(rb + lo) * (uint32_t)tiles_x + (uint32_t)l_lo + (e - ex_lo);
          emit_key(kpos + e, tile, gg, cap_k, out_tile, out_gid, s_hist, counters);
        }
      }
      kpos += tot;
    }
  }
  __syncthreads();
  for (int jj = tid; jj < 512; jj += GUT_EMIT_THREADS) {
    const uint32_t v = (&s_hist[0][0])[jj];
    if (v) atomicAdd(&counters[CNT_HIST_TILE + jj], v);
  }
}

// per-partition key totals (the emit's partition prefixes after the scan)
__global__ __launch_bounds__(GUT_EMIT_THREADS) void emit_count_kernel(const uint32_t *__restrict__ order,
                                                                      const uint32_t *n_vis_p,
                                                                      const uint32_t *__restrict__ tiles,
                                                                      uint32_t *__restrict__ part_off) {
  __shared__ uint32_t s_w[GUT_EMIT_THREADS / 32];
  const uint32_t n = *n_vis_p, base = blockIdx.x * GUT_EMIT_PART;
  if (base >= n) return;
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < GUT_EMIT_ITEMS; ++j) {
    const uint32_t gi = base + j * GUT_EMIT_THREADS + threadIdx.x;
    if (gi < n) sum += code_count(__ldg(&tiles[__ldg(&order[gi])]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < GUT_EMIT_THREADS / 32; ++w) t += s_w[w];
    part_off[blockIdx.x] = t;
  }
}

// exclusive scan of the partition totals in place (one CTA; partitions past
// n_vis hold stale values but are never read)
__global__ __launch_bounds__(1024) void emit_scan_kernel(const uint32_t *n_vis_p, uint32_t *__restrict__ part_off) {
  __shared__ uint32_t s_w[32];
  const uint32_t n = *n_vis_p, np = (n + GUT_EMIT_PART - 1) / GUT_EMIT_PART;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t run = 0;
  for (uint32_t b0 = 0; b0 < np; b0 += 1024) {
    const uint32_t i = b0 + threadIdx.x;
    const uint32_t v = i < np ? part_off[i] : 0u;
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
    const uint32_t ex = run + (w > 0 ? s_w[w - 1] : 0u) + x - v;
    if (i < np) part_off[i] = ex;
    run += s_w[31];
    __syncthreads();
  }
}

void launch_emit(const uint32_t *order, const uint32_t *n_vis, uint32_t n_upper, const uint32_t *tiles,
                 const float4 *ell, const double2 *ell64, int tiles_x, int tile_cull, uint32_t *out_tile,
                 uint32_t *out_gid, uint32_t cap_k, uint32_t *counters, uint32_t *part_off, uint2 *big_list,
                 cudaStream_t st, const uint32_t *codes) {
  if (n_upper == 0) return;
  unsigned blocks = (n_upper + GUT_EMIT_PART - 1) / GUT_EMIT_PART;
  if (!codes) emit_count_kernel<<<blocks, GUT_EMIT_THREADS, 0, st>>>(order, n_vis, tiles, part_off);
  emit_scan_kernel<<<1, 1024, 0, st>>>(n_vis, part_off);
  emit_kernel<<<blocks, GUT_EMIT_THREADS, 0, st>>>(order, n_vis, tiles, ell, ell64, tiles_x, tile_cull, out_tile, out_gid,
                                                   cap_k, counters, part_off, big_list, codes);
  emit_big_kernel<<<148 * 4, GUT_EMIT_THREADS, 0, st>>>(big_list, ell, ell64, tiles_x, tile_cull, out_tile, out_gid,
                                                        cap_k, counters);
}

}  // namespace gut
