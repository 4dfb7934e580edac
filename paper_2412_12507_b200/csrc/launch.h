// launch.h — host-side launchers of the sm_100a kernels (internal to libgut).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "gut_internal.cuh"

namespace gut {

constexpr int GUT_MAX_DEVICES = 64;  // per-device launch setup slots

// Packed scene (device SoA).  pos_opa = (mu, sigma), rot = (w,x,y,z) raw,
// scale = (s, 0), sh = float4 chunk c of Gaussian i at sh[c * n + i].
struct SceneDev {
  int64_t n;
  int sh_degree, sh_chunks;
  float4 *pos_opa, *rot, *scale, *sh;
};

// Counters block (uint32 words), zeroed at the start of every render.
enum : int {
  CNT_NVIS = 0,
  CNT_K = 2,          // u64
  CNT_TICKETS = 4,    // 12 tickets
  CNT_OVERFLOW = 16,
  CNT_PAIRS_EVAL = 18,     // u64
  CNT_PAIRS_CONTRIB = 20,  // u64
  CNT_TERMINATED = 22,     // u64
  CNT_MAXLEN = 24,
  CNT_NITEMS = 26,         // blend segment slots (sum over tiles of S_t)
  CNT_NPRE = 27,           // transmittance-prefix work items
  CNT_NDEFER = 28,         // Gaussians deferred to the fp64 K1 kernel
  CNT_Q_NINIT = 32,        // blend work queue: initial grants (queue 1 length)
  CNT_Q_HEAD1 = 33,        //   next queue-1 entry
  CNT_Q_HEAD2 = 34,        //   next queue-2 (granted successor) entry
  CNT_Q_ALLOC2 = 35,       //   queue-2 entries allocated
  CNT_Q_FINISHED = 36,     //   units (8 per tile) whose pixels are written
  CNT_NBIG = 37,           // K2: Gaussians in the big list (tile rectangle > 3x3)
  CNT_K1LIST = 38,         // K1 (rolling shutter): Gaussians kept by the pre-filter
  CNT_HIST_DEPTH = 64,     // 4 x 256
  CNT_HIST_TILE = 64 + 1024,  // 2 x 256
  CNT_PLAN_HIST = 64 + 1024 + 512,  // 1024 blend queue-1 buckets
  CNT_WORDS = 64 + 1024 + 512 + 1024,
  // sticky words after the per-render memset range: set by the kernels, read
  // and cleared only by the host at a synchronising call (gut_check & co.)
  CNT_STICKY_OVERFLOW = CNT_WORDS,
  // look-back epoch base of the current render, advanced on the device at the
  // start of every render (frame_init_kernel): a render is replayable as a CUDA graph
  CNT_EPOCH = CNT_WORDS + 1,
  CNT_ALLOC = CNT_WORDS + 4
};

void launch_pack_scene(const float *means, const float *rots, const float *scales, const float *opac,
                       const float *sh, SceneDev s, cudaStream_t st);

// K1 (fp32) followed by the fp64 kernel for the deferred "wide" Gaussians;
// ell64 [3 x double2 per Gaussian] holds their fp64 ellipse (record k2 < 0)
// list: N uint32 scratch (rolling shutter: the Gaussians kept by the pre-filter)
void launch_project(const DevCam &cam, const SceneDev &s, uint32_t *dkey, uint32_t *tiles, float4 *ell,
                    double2 *ell64, float4 *payload, uint32_t *counters, uint32_t *deferred, uint32_t *list,
                    cudaStream_t st);

// one onesweep LSD pass over 8-bit digit `shift`; first = keys only, value = index,
// items equal to GUT_CULLED_KEY dropped.  n_dev: device count (nullable, then n_host).
void launch_sort_pass(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                      uint32_t *vals_out, const uint32_t *n_dev, uint32_t n_host, int shift,
                      const uint32_t *hist, unsigned long long *status, uint32_t *ticket,
                      const uint32_t *epoch_base, uint32_t epoch_off, bool first, cudaStream_t st,
                      uint2 *ranges = nullptr, const uint32_t *codes_src = nullptr, uint32_t *codes_out = nullptr,
                      uint32_t *part_tot = nullptr);
// (final depth pass: codes_out[o] = codes_src[value] -- the K1 tile code in depth order -- and
// part_tot[o / GUT_EMIT_PART] += its key count; part_tot zeroed by launch_frame_init)
// Epochs per render: sort passes use base + 0..6 (depth 0-3, tile 4 and 6), the blend base + GUT_EPOCH_BLEND.
#define GUT_EPOCHS_PER_RENDER 8u
#define GUT_EPOCH_BLEND 7u
// Start of a render: advances the device epoch base by GUT_EPOCHS_PER_RENDER
// (when the blend's 22-bit epoch field wraps it clears the blend status words,
// n_bstatus, so a stale word can never alias the current render) and empties
// the tile ranges that the final tile pass fills (K4).
void launch_frame_init(uint32_t *counters, unsigned long long *bstatus, size_t n_bstatus, uint2 *ranges,
                       int n_tiles, uint32_t *zero, int n_zero, cudaStream_t st);
// (K4 is fused into the final tile pass: ranges != nullptr there; launch_frame_init empties them)

// K2: per-partition key totals, their scan, then the emission (part_off:
// one uint32 per GUT_EMIT_PART Gaussians of the upper bound n_upper)
// (codes != nullptr: the tile codes in depth order with part_off already holding the
// partition totals -- the final depth pass wrote both -- so only the scan and the emission run)
void launch_emit(const uint32_t *order, const uint32_t *n_vis, uint32_t n_upper, const uint32_t *tiles,
                 const float4 *ell, const double2 *ell64, int tiles_x, int tile_cull, uint32_t *out_tile,
                 uint32_t *out_gid, uint32_t cap_k, uint32_t *counters, uint32_t *part_off, uint2 *big_list,
                 cudaStream_t st, const uint32_t *codes = nullptr);



// Per-tile ray anchor (fp64).  Global shutter: camera frame, a function of the
// intrinsics only (cached).  Rolling shutter: world frame, per view.
struct TileAnchor {
  double D[3], T1[3], T2[3], O[3], ta, pad[3];
  // per 8x8 pixel block B (x0 = 8 (B & 1), y0 = 8 (B >> 1)): the pixels' fp32
  // offsets as an affine lattice a(x, y) = a00 + ax x + ay y (+ |residual| <=
  // rho_a), same for b, x, y = 0..7 within the block -- {a00, ax, ay, rho_a,
  // b00, bx, by, rho_b}; rho = +inf: no usable fit (K5 masks then keep every pixel)
  float fit[4][8];
};

// per-pixel (a, b, snorm, beta) relative to the tile anchor + per-tile anchors
void launch_rays(const DevCam &cam, float4 *pix, TileAnchor *anchors, cudaStream_t st);

// blend work plan (see k5_blend.cu): segment slots (seg_base) and queue 1 =
// the first min(S_t, window) segment grants of every unit, longest tiles
// first.  The per-unit counters (extra grants, next segment, completed) are
// zeroed by the host before the blend.
// upt = work units per tile (GUT_BLEND_WARPS 8x8 blocks; GUT_KBUF_UNITS 8x4 blocks for the k-buffer)
void launch_plan(const uint2 *ranges, int n_tiles, int seg, int window, uint32_t *seg_base, uint32_t *q1,
                 uint32_t *counters, cudaStream_t st, int upt = GUT_BLEND_WARPS);

struct BlendBufs {
  const uint2 *ranges;
  const uint32_t *gids;
  const float4 *payload;
  const float4 *pix;
  const TileAnchor *anchors;
  const uint32_t *seg_base;     // per tile: first (tile, segment) slot, tile-major
  uint32_t *granted;            // per unit (8 tile + warp block): grants beyond the first min(S, window)
  uint32_t *next_s;             // per unit: next segment index to hand out
  uint32_t *unit_done;          // per unit: segments completed
  uint32_t *q1_taken;           // per unit: queue-1 (initial) segments taken by a warp
  const uint32_t *q1;           // queue 1: unit ids (initial grants, longest tiles first)
  uint32_t *q2;                 // queue 2: unit id + 1 per granted successor (0 = empty slot)
  unsigned long long *status;   // per (slot, pixel) look-back word (flag | epoch | -log2 T)
  float4 *part_c;    // per (slot, pixel) partial colour + depth
  float *part_t;     // per (slot, pixel) transmittance at segment end (-1 inactive)
  uint2 *tile_work;
  uint4 *trace;  // optional (GUT_BLEND_TRACE=1): per (slot, warp block) 2 x uint4 (see GUT_STAGE_BLEND_TRACE)
  int seg, window, n_tiles;
  const uint32_t *epoch;  // device epoch base (CNT_EPOCH); the blend uses base + GUT_EPOCH_BLEND
  float *rgb, *alpha, *depth;
  uint32_t *counters;
  // persistent blend grid in quarter-CTAs per SM (0: as many as fit).  Frames
  // in flight (gut_render_batch lanes) use GUT_BATCH_BLEND_X4: the next
  // frames' K1-K3 then run beside this frame's K5 (throughput over latency)
  int grid_x4;
  int grant_cap;  // successor grants at most this many segments ahead (0: as the decay predicts)
};
#define GUT_BATCH_BLEND_X4 5  // 1.25 CTAs per SM

// queue-2 slots beyond the grants: one ticket per resident blend warp (>= 148 SMs x 64 warps)
#define GUT_BLEND_Q2_SLACK (1u << 16)
// blend warps allowed to wait for future grants once queue 1 is drained
#ifndef GUT_BLEND_MAX_WAITERS
#define GUT_BLEND_MAX_WAITERS 768u
#endif

void launch_blend(const DevCam &cam, const BlendBufs &b, cudaStream_t st);
// "Ours (sorted)": per-ray MLAB k-buffer of cam.kbuf hits (1, 2, 4, 8, 16), queue 1
// planned with GUT_KBUF_UNITS units per tile and one segment per tile
void launch_blend_kbuf(const DevCam &cam, const BlendBufs &b, cudaStream_t st);

// K6: backward of the last render (k6_backward.cu)
struct BwdBufs {
  const uint2 *ranges;
  const uint32_t *gids;         // the forward's sorted Gaussian ids
  const float4 *payload;        // K1 payload of the forward
  const float4 *pix;
  const TileAnchor *anchors;
  const uint32_t *tiles;        // K1 tile code (0 = culled)
  const float *rgb, *alpha, *depth;          // forward outputs (device)
  const float *g_rgb, *g_alpha, *g_depth;    // upstream gradients (device; alpha / depth nullable)
  // per Gaussian 16 accumulators in 32.32 fixed point (int64, two's
  // complement): integer additions commute, so the gradients are bitwise
  // reproducible whatever order the atomics land in
  long long *acc;
  uint32_t *order;              // tiles, longest list first (plan queue 1, n_tiles entries)
  uint32_t *seg_base;           // plan scratch (n_tiles)
  uint32_t *counters;           // the context's counters block (plan histogram)
  const float *t0;              // per Gaussian centre shutter time (nullptr: global shutter)
  float *d_means, *d_rots, *d_scales, *d_opac, *d_sh, *d_rgb;  // outputs (d_rgb nullable)
  float *densify;               // nullable: |dL/dmu| / (distance / 2)
};
#define GUT_BWD_FIX 4294967296.0  // fixed-point scale of the K6 accumulators (2^32)
void launch_backward(const DevCam &cam, const SceneDev &s, const BwdBufs &b, cudaStream_t st);
// per Gaussian the shutter time of its centre (k1_project.cu; SH direction under rolling shutter)
void launch_centre_times(const DevCam &cam, const SceneDev &s, float *t0, cudaStream_t st);

// Supp. C projection quality (k1_project.cu); layout = gut_quality (include/gut.h)
struct QualityRec {
  double ut[5], ewa[5], mc[5], kl_ut, kl_ewa;
  int32_t valid, pad;
};
void launch_quality(const DevCam &cam, const SceneDev &s, int n_mc, unsigned long long seed, QualityRec *out,
                    cudaStream_t st);

}  // namespace gut
