// k3_sort.cu — K3: hand-written onesweep LSD radix-sort pass (sm_100a).
//
// The (tile_id, depth) order of PAPER L208 ("3DGS sorts them globally for each
// tile") is produced as an LSD radix sort in two levels:
//   level 1: 4 passes over the 32-bit depth key of the N_vis visible Gaussians
//            (value = Gaussian index; the first pass also drops culled ones);
//   level 2: after depth-ordered emission (K2), 1-2 passes over the tile id.
// Stable LSD passes give exactly the (tile, depth, index) order of one 64-bit
// key sort while moving 3-5x fewer bytes.
//
// One pass = one kernel: a CTA claims a 4096-key partition by ticket (forward
// progress for the look-back), ranks its keys per 8-bit digit with warp
// match-any (stable: items are ranked in sequence order), publishes its digit
// histogram and resolves its global digit offsets by decoupled look-back
// (epoch-tagged status words), then reorders through shared memory so the
// global writes are digit runs (coalesced).  Placement comes only from scans:
// deterministic, no atomics choose positions.
#include "launch.h"

namespace gut {

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// exclusive scans over the 256 digits of two values at once: threads 0..255
// (warps 0-7) hold digit values, every thread of the CTA calls (barriers)
__device__ __forceinline__ void digit_scan2(uint32_t a, uint32_t b, uint32_t *s_tmp, uint32_t &ea, uint32_t &eb,
                                            uint32_t &tb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = a, y = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t px = __shfl_up_sync(0xffffffffu, x, o), py = __shfl_up_sync(0xffffffffu, y, o);
    if (lane >= o) { x += px; y += py; }
  }
  if (lane == 31 && w < 8) { s_tmp[w] = x; s_tmp[8 + w] = y; }
  __syncthreads();
  uint32_t wa = 0, wb = 0;
  tb = 0;
#pragma unroll
  for (int ww = 0; ww < 8; ++ww) {
    const uint32_t va = s_tmp[ww], vb = s_tmp[8 + ww];
    if (ww < w) { wa += va; wb += vb; }
    tb += vb;
  }
  ea = wa + x - a;
  eb = wb + y - b;
  __syncthreads();
}

#ifndef GUT_SORT_WIN
#define GUT_SORT_WIN 8  // look-back predecessors loaded per round trip (16, 32 measured slower)
#endif
#ifndef GUT_SORT_BALLOT
#define GUT_SORT_BALLOT 1  // digit peers by 9 ballots (measured faster than match.any)
#endif
template <bool FIRST>
__global__ __launch_bounds__(GUT_SORT_THREADS) void onesweep_kernel(
    const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in, uint32_t *__restrict__ keys_out,
    uint32_t *__restrict__ vals_out, const uint32_t *n_dev, uint32_t n_host, int shift,
    const uint32_t *__restrict__ hist, unsigned long long *status, uint32_t *ticket,
    const uint32_t *__restrict__ epoch_base, uint32_t epoch_off, uint2 *__restrict__ ranges,
    const uint32_t *__restrict__ codes_src, uint32_t *__restrict__ codes_out, uint32_t *__restrict__ part_tot) {
  constexpr int W = GUT_SORT_THREADS / 32;
  static_assert(GUT_SORT_THREADS >= 256, "one thread per digit");
  __shared__ uint32_t s_keys[GUT_SORT_PART];
  __shared__ uint32_t s_vals[GUT_SORT_PART];
  __shared__ uint16_t s_wcnt[W][256];  // per-warp digit counts, then exclusive over warps (< 4096)
  __shared__ uint32_t s_goff[256];
  __shared__ uint32_t s_loff[256];
  __shared__ uint32_t s_tmp[16];
  __shared__ uint32_t s_part;

  const uint32_t n = n_dev ? min(*n_dev, n_host) : n_host;
  const uint32_t epoch = __ldg(epoch_base) + epoch_off;  // (device epoch: graph-replayable)
  if (threadIdx.x == 0) s_part = atomicAdd(ticket, 1u);
  for (int j = threadIdx.x; j < W * 256; j += GUT_SORT_THREADS) (&s_wcnt[0][0])[j] = 0;
  __syncthreads();
  const uint32_t part = s_part;
  const uint32_t base = part * GUT_SORT_PART;
  if (base >= n) return;

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  uint32_t key[GUT_SORT_ITEMS], val[GUT_SORT_ITEMS], rank[GUT_SORT_ITEMS];
  // warp w owns the contiguous sub-range [base + w*32*ITEMS, base + (w+1)*32*ITEMS)
#pragma unroll
  for (int j = 0; j < GUT_SORT_ITEMS; ++j) {
    uint32_t idx = base + w * (32 * GUT_SORT_ITEMS) + j * 32 + lane;
    bool in = idx < n;
    key[j] = in ? __ldg(&keys_in[idx]) : GUT_CULLED_KEY;
    if (FIRST) val[j] = idx;
    else val[j] = in ? __ldg(&vals_in[idx]) : 0u;
    if (!FIRST && !in) key[j] = 0xFFFFFFFFu;
    rank[j] = (in && (!FIRST || key[j] != GUT_CULLED_KEY)) ? 1u : 0u;  // validity until ranked
  }
  // stable per-warp ranking, rounds in sequence order.  First pass: culled
  // keys are interspersed, so validity is a 9th digit bit (9 ballots).  Later
  // passes: the only invalid items are the tail past n -- the highest lanes
  // of the last rounds of the last warps, after every valid item in sequence
  // order -- so they rank as digit 255 behind the valid ones (8 ballots), are
  // not written, and are taken off digit 255's partition total below.
  constexpr int NB = FIRST ? 9 : 8;
#pragma unroll
  for (int j = 0; j < GUT_SORT_ITEMS; ++j) {
    const bool valid = rank[j] != 0;
    const uint32_t d = valid ? (key[j] >> shift) & 255u : (FIRST ? 256u : 255u);
#if GUT_SORT_BALLOT
    // peers = lanes with the same digit: per bit one predicate (bit test),
    // one ballot and one predicated AND (4 instructions; the compiler's own
    // form of "bit ? bal : ~bal" takes 6)
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < NB; ++b)
      asm("{\n\t.reg .pred p;\n\t.reg .b32 t, bal;\n\t"
          "and.b32 t, %1, %2;\n\tsetp.ne.u32 p, t, 0;\n\t"
          "vote.sync.ballot.b32 bal, p, 0xffffffff;\n\t"
          "@p and.b32 %0, %0, bal;\n\t"
          "@!p lop3.b32 %0, %0, bal, 0, 0x30;\n\t}"
          : "+r"(peers)
          : "r"(d), "r"(1u << b));
#else
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
#endif
    const uint32_t before = __popc(peers & lt);
    const bool counted = FIRST ? valid : true;
    uint32_t prev = counted ? s_wcnt[w][d & 255u] : 0u;
    __syncwarp();
    if (counted && before == 0) s_wcnt[w][d & 255u] = (uint16_t)(prev + __popc(peers));
    __syncwarp();
    rank[j] = valid ? (prev + before) : 0xFFFFFFFFu;
  }
  __syncthreads();
  // per digit (threads 0..255): exclusive over warps, partition total; the
  // aggregate is published at once (the look-back walk comes after the
  // shared-memory scatter, with the keys out of registers)
  uint32_t tot = 0, hv = 0;
  if (threadIdx.x < 256) {
    const uint32_t dgt = threadIdx.x;
#pragma unroll
    for (int ww = 0; ww < W; ++ww) {
      const uint32_t c = s_wcnt[ww][dgt];
      s_wcnt[ww][dgt] = (uint16_t)tot;
      tot += c;
    }
    if (!FIRST && dgt == 255u && base + GUT_SORT_PART > n) tot -= base + GUT_SORT_PART - n;  // the tail items
    lookback_publish(status, 256, (int)part, (int)dgt, tot, epoch);
    hv = __ldg(&hist[dgt]);
  }
  // global digit start (exclusive scan of the pass histogram) and local digit start
  uint32_t hex, lex, ltotal;
  digit_scan2(hv, tot, s_tmp, hex, lex, ltotal);
  if (threadIdx.x < 256) s_loff[threadIdx.x] = lex;
  __syncthreads();
  // scatter into shared memory in digit order
#pragma unroll
  for (int j = 0; j < GUT_SORT_ITEMS; ++j) {
    if (rank[j] != 0xFFFFFFFFu) {
      const uint32_t d = (key[j] >> shift) & 255u;
      const uint32_t pos = s_loff[d] + s_wcnt[w][d] + rank[j];
      s_keys[pos] = key[j];
      s_vals[pos] = val[j];
    }
  }
  // decoupled look-back (window of GUT_SORT_WIN predecessors per round trip)
  if (threadIdx.x < 256)
    s_goff[threadIdx.x] = hex + lookback_walk<GUT_SORT_WIN>(status, 256, (int)part, (int)threadIdx.x, tot, epoch);
  __syncthreads();
  // coalesced write-out of the digit runs
  for (uint32_t p = threadIdx.x; p < ltotal; p += GUT_SORT_THREADS) {
    const uint32_t k = s_keys[p];
    const uint32_t d = (k >> shift) & 255u;
    const uint32_t o = s_goff[d] + (p - s_loff[d]);
    if (keys_out) keys_out[o] = k;
    const uint32_t v = s_vals[p];
    vals_out[o] = v;
    if (codes_out) {
      // final depth pass (K2's inputs): the tile code of the Gaussian at depth
      // position o, and the key total of each GUT_EMIT_PART-position partition
      // (one atomic per run of equal partitions in the warp)
      const uint32_t cd = __ldg(&codes_src[v]);
      codes_out[o] = cd;
      const uint32_t pp = o / GUT_EMIT_PART, am = __activemask();
      const uint32_t peers = __match_any_sync(am, pp);
      const uint32_t sum = __reduce_add_sync(peers, code_count(cd));
      if ((threadIdx.x & 31) == __ffs(peers) - 1 && sum) atomicAdd(&part_tot[pp], sum);
    }
    if (ranges) {
      // K4 fused into the final tile pass: a tile's keys are contiguous in this
      // CTA's run (the input is ordered by the lower digits) and in the output,
      // so the min / max over CTAs of their first / last positions is its range
      if (p == 0 || s_keys[p - 1] != k) atomicMin(&ranges[k].x, o);
      if (p + 1 == ltotal || s_keys[p + 1] != k) atomicMax(&ranges[k].y, o + 1);
    }
  }
}

void launch_sort_pass(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                      uint32_t *vals_out, const uint32_t *n_dev, uint32_t n_host, int shift,
                      const uint32_t *hist, unsigned long long *status, uint32_t *ticket,
                      const uint32_t *epoch_base, uint32_t epoch_off, bool first, cudaStream_t st, uint2 *ranges,
                      const uint32_t *codes_src, uint32_t *codes_out, uint32_t *part_tot) {
  if (n_host == 0) return;
  unsigned blocks = (n_host + GUT_SORT_PART - 1) / GUT_SORT_PART;
  if (first)
    onesweep_kernel<true><<<blocks, GUT_SORT_THREADS, 0, st>>>(keys_in, vals_in, keys_out, vals_out, n_dev,
                                                               n_host, shift, hist, status, ticket, epoch_base,
                                                               epoch_off, ranges, codes_src, codes_out, part_tot);
  else
    onesweep_kernel<false><<<blocks, GUT_SORT_THREADS, 0, st>>>(keys_in, vals_in, keys_out, vals_out, n_dev,
                                                                n_host, shift, hist, status, ticket, epoch_base,
                                                                epoch_off, ranges, codes_src, codes_out, part_tot);
}

// Start of a render (one launch): block 0 advances the device epoch base by
// GUT_EPOCHS_PER_RENDER (clearing the blend status words when the blend's
// 22-bit epoch field wraps, every 2^19 renders), every thread empties one
// tile range (start UINT_MAX, end 0) for the final tile pass to fill (K4).
__global__ void frame_init_kernel(uint32_t *counters, unsigned long long *bstatus, size_t n, uint2 *ranges,
                                  int n_tiles, uint32_t *zero, int n_zero) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n_tiles) ranges[t] = make_uint2(0xFFFFFFFFu, 0u);
  if (t < n_zero) zero[t] = 0u;
  if (blockIdx.x != 0) return;
  __shared__ uint32_t s_wrap;
  if (threadIdx.x == 0) {
    const uint32_t old = counters[CNT_EPOCH], nb = old + GUT_EPOCHS_PER_RENDER;
    s_wrap = ((old + GUT_EPOCH_BLEND) >> 22) != ((nb + GUT_EPOCH_BLEND) >> 22);
    counters[CNT_EPOCH] = nb;
  }
  __syncthreads();
  if (s_wrap)
    for (size_t j = threadIdx.x; j < n; j += blockDim.x) bstatus[j] = 0ull;
}

void launch_frame_init(uint32_t *counters, unsigned long long *bstatus, size_t n_bstatus, uint2 *ranges,
                       int n_tiles, uint32_t *zero, int n_zero, cudaStream_t st) {
  const unsigned blocks = (unsigned)max(1, (max(n_tiles, n_zero) + 255) / 256);
  frame_init_kernel<<<blocks, 256, 0, st>>>(counters, bstatus, n_bstatus, ranges, n_tiles, zero, n_zero);
}

}  // namespace gut
