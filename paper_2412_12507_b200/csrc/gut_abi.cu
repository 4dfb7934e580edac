// gut_abi.cu — host side of the C ABI declared in include/gut.h.
//
// Validates arguments, owns the device workspace (grown on demand or reserved
// up front), builds the per-view kernel parameters and enqueues K1..K5 on the
// caller's stream.  No arithmetic of the method runs here: every step of the
// path is a kernel (k1_project.cu, k3_sort.cu, k2_emit.cu, k5_blend.cu).  The
// only host-side numbers are the per-view camera constants (pose at t = 0,
// the slerp axis-angle, UT weights from alpha/beta/kappa).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <array>
#include <string>
#include <vector>

#include "../../include/gut.h"
#include "launch.h"

using namespace gut;

struct gut_scene {
  SceneDev d;
  int device;
};

struct gut_context {
  int device = 0;
  std::string err;
  // workspace
  size_t cap_n = 0, cap_k = 0, cap_tiles = 0, cap_pix = 0;
  uint32_t *dkey = nullptr, *tiles = nullptr;
  float4 *ell = nullptr, *payload = nullptr;
  double2 *ell64 = nullptr;
  uint32_t *deferred = nullptr, *k1_list = nullptr;
  uint2 *big_list = nullptr;  // K2: (Gaussian, first key slot) of the big Gaussians
  uint32_t *sa_k = nullptr, *sa_v = nullptr, *sb_k = nullptr, *sb_v = nullptr;
  uint32_t *ka = nullptr, *va = nullptr, *kb = nullptr, *vb = nullptr;
  uint2 *ranges = nullptr, *tile_work = nullptr;
  uint4 *trace = nullptr;  // K5 per-work-item trace (env GUT_BLEND_TRACE=1, diagnostics only)
  size_t cap_trace = 0, last_items = 0;
  bool trace_on = false;
  float *img = nullptr;     // host-output staging (RGB, alpha, depth); two slots for the batch's copy stream
  float *img_slot[2] = {nullptr, nullptr};
  int img_next = 0;
  cudaStream_t copy_stream = nullptr;                  // gut_render_batch: device->host copies off the render stream
  cudaEvent_t ev_rendered[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr}, ev_copy_tail = nullptr;
  unsigned long long *st_depth = nullptr, *st_emit = nullptr, *st_tile = nullptr;
  uint32_t *counters = nullptr, *h_counters = nullptr;
  // K5: ray LUT (cached per intrinsics for global shutter), blend work plan
  float4 *pix = nullptr;
  TileAnchor *anchors = nullptr;
  uint32_t *seg_base = nullptr, *unit_ctr = nullptr;  // unit_ctr: 4 x n_units (extra grants, next_s, done, q1 taken)
  uint32_t *q1 = nullptr, *q2 = nullptr;  // blend work queues (k5_blend.cu)
  unsigned long long *bstatus = nullptr;
  float *part_t = nullptr;
  float4 *part_c = nullptr;
  size_t cap_items = 0;
  bool lut_valid = false;
  double lut_key[20] = {};
  // K5 segment length and speculation window: one frame at a time (latency:
  // speculation shortens the densest tiles' critical path) and frames in flight
  // (throughput: the other frames fill the GPU, so no speculation beyond the
  // grants and a smaller persistent grid; DESIGN.md §5 "Scheduling")
  // (one segment length for both: the split-list composition's rounding
  // depends on it, and a batch must return exactly what single renders do)
  int blend_seg = 2560, blend_window = 2;
  int blend_seg_rs = 2048;  // rolling-shutter frames (Waymo-shaped: 0.847 vs 0.889 ms at 2560)
  int blend_window_batch = 1, batch_x4 = GUT_BATCH_BLEND_X4, batch_grant_cap = 4;
  bool reserved = false;
  std::vector<std::array<cudaEvent_t, 7>> tsets;  // per-render stage events (timing = 1)
  size_t tnext = 0;
  // last render (for gut_debug_copy_stage)
  int64_t last_n = 0;
  int last_tiles = 0;
  const uint32_t *last_order = nullptr, *last_keys = nullptr, *last_vals = nullptr;
  DevCam last_cam;                    // (gut_render_backward: must match)
  const gut_scene *last_scene = nullptr;
  long long *gacc = nullptr;          // K6 fixed-point accumulators (16 per Gaussian)
  float *gt0 = nullptr;               // K6 centre shutter times (1 per Gaussian)
  size_t cap_gacc = 0;
  // gut_render_batch: frames in flight -- lane 0 is this context on the
  // caller's stream, lanes 1.. are child contexts (own workspaces) on their
  // own streams, joined back to the caller's stream with events
  int frames_in_flight = 4;
  int64_t res_keys = 0, res_n = 0;
  int32_t res_w = 0, res_h = 0;
  std::vector<gut_context *> lanes;
  std::vector<cudaStream_t> lane_streams;
  std::vector<cudaEvent_t> lane_events;
  cudaEvent_t fork_event = nullptr;
};

static thread_local std::string g_err;

static gut_status fail(gut_context *ctx, gut_status s, const std::string &msg) {
  if (ctx) ctx->err = msg; else g_err = msg;
  return s;
}

#define CUDA_TRY(ctx, call)                                                                        \
  do {                                                                                             \
    cudaError_t e__ = (call);                                                                      \
    if (e__ != cudaSuccess) {                                                                      \
      return fail(ctx, e__ == cudaErrorMemoryAllocation ? GUT_E_OUT_OF_MEMORY : GUT_E_CUDA,        \
                  std::string(#call) + ": " + cudaGetErrorString(e__));                            \
    }                                                                                              \
  } while (0)

template <class T>
static cudaError_t regrow(T *&p, size_t &cap_field_unused, size_t count) {
  (void)cap_field_unused;
  if (p) cudaFree(p);
  p = nullptr;
  return cudaMalloc((void **)&p, count * sizeof(T) + 16);
}

static gut_status ensure_n(gut_context *ctx, size_t n) {
  if (n <= ctx->cap_n) return GUT_OK;
  size_t c = n + n / 8 + 1024, dummy = 0;
  CUDA_TRY(ctx, regrow(ctx->dkey, dummy, c));
  CUDA_TRY(ctx, regrow(ctx->tiles, dummy, c));
  CUDA_TRY(ctx, regrow(ctx->ell, dummy, 2 * c));
  CUDA_TRY(ctx, regrow(ctx->ell64, dummy, 3 * c));
  CUDA_TRY(ctx, regrow(ctx->deferred, dummy, c));
  CUDA_TRY(ctx, regrow(ctx->k1_list, dummy, c));
  CUDA_TRY(ctx, regrow(ctx->big_list, dummy, c));
  CUDA_TRY(ctx, regrow(ctx->payload, dummy, (size_t)GUT_PAYLOAD_F4 * c));
  CUDA_TRY(ctx, regrow(ctx->sa_k, dummy, c));
  CUDA_TRY(ctx, regrow(ctx->sa_v, dummy, c));
  CUDA_TRY(ctx, regrow(ctx->sb_k, dummy, c));
  CUDA_TRY(ctx, regrow(ctx->sb_v, dummy, c));
  size_t parts = (c + GUT_SORT_PART - 1) / GUT_SORT_PART + 1;
  CUDA_TRY(ctx, regrow(ctx->st_depth, dummy, parts * 256));
  CUDA_TRY(ctx, cudaMemset(ctx->st_depth, 0, parts * 256 * sizeof(unsigned long long)));
  size_t eparts = (c + GUT_EMIT_PART - 1) / GUT_EMIT_PART + 1;
  CUDA_TRY(ctx, regrow(ctx->st_emit, dummy, eparts));
  CUDA_TRY(ctx, cudaMemset(ctx->st_emit, 0, eparts * sizeof(unsigned long long)));
  ctx->cap_n = c;
  return GUT_OK;
}

static gut_status ensure_k(gut_context *ctx, size_t k) {
  if (k <= ctx->cap_k && ctx->ka) return GUT_OK;
  size_t c = k + k / 4 + 4096, dummy = 0;
  if (c >= (size_t)0x3FFFFFFF) return fail(ctx, GUT_E_CAPACITY, "key count exceeds 2^30");
  CUDA_TRY(ctx, regrow(ctx->ka, dummy, c));
  CUDA_TRY(ctx, regrow(ctx->va, dummy, c));
  CUDA_TRY(ctx, regrow(ctx->kb, dummy, c));
  CUDA_TRY(ctx, regrow(ctx->vb, dummy, c));
  size_t parts = (c + GUT_SORT_PART - 1) / GUT_SORT_PART + 1;
  CUDA_TRY(ctx, regrow(ctx->st_tile, dummy, parts * 256));
  CUDA_TRY(ctx, cudaMemset(ctx->st_tile, 0, parts * 256 * sizeof(unsigned long long)));
  ctx->cap_k = c;
  return GUT_OK;
}

static gut_status ensure_tiles(gut_context *ctx, size_t t) {
  if (t <= ctx->cap_tiles) return GUT_OK;
  size_t dummy = 0;
  CUDA_TRY(ctx, regrow(ctx->ranges, dummy, t));
  CUDA_TRY(ctx, regrow(ctx->tile_work, dummy, t));
  CUDA_TRY(ctx, regrow(ctx->pix, dummy, t * GUT_TILE_PX));
  CUDA_TRY(ctx, regrow(ctx->anchors, dummy, t));
  CUDA_TRY(ctx, regrow(ctx->seg_base, dummy, t));
  CUDA_TRY(ctx, regrow(ctx->unit_ctr, dummy, 4 * t * GUT_BLEND_WARPS));
  ctx->lut_valid = false;
  ctx->cap_tiles = t;
  return GUT_OK;
}

// blend work items: at most n_tiles + K / seg + 1 (tile, segment) pairs
static gut_status ensure_items(gut_context *ctx, size_t items) {
  if (items <= ctx->cap_items) return GUT_OK;
  size_t c = items + items / 8 + 64, dummy = 0;
  CUDA_TRY(ctx, regrow(ctx->bstatus, dummy, c * GUT_TILE_PX));
  CUDA_TRY(ctx, cudaMemset(ctx->bstatus, 0, c * GUT_TILE_PX * sizeof(unsigned long long)));
  CUDA_TRY(ctx, regrow(ctx->part_c, dummy, c * GUT_TILE_PX));
  CUDA_TRY(ctx, regrow(ctx->part_t, dummy, c * GUT_TILE_PX));
  CUDA_TRY(ctx, regrow(ctx->q1, dummy, c * GUT_BLEND_WARPS));
  // queue 2: every grant plus one outstanding ticket per resident warp; the
  // consumers re-zero the slots they take (tickets past the last grant find 0)
  const size_t q2n = c * GUT_BLEND_WARPS + GUT_BLEND_Q2_SLACK;
  CUDA_TRY(ctx, regrow(ctx->q2, dummy, q2n));
  CUDA_TRY(ctx, cudaMemset(ctx->q2, 0, q2n * sizeof(uint32_t)));
  ctx->cap_items = c;
  return GUT_OK;
}

static gut_status ensure_pix(gut_context *ctx, size_t p) {
  if (p <= ctx->cap_pix) return GUT_OK;
  size_t dummy = 0;
  CUDA_TRY(ctx, cudaDeviceSynchronize());  // (a copy may still read the old slots)
  CUDA_TRY(ctx, regrow(ctx->img, dummy, 10 * p));
  ctx->img_slot[0] = ctx->img;
  ctx->img_slot[1] = ctx->img + 5 * p;
  ctx->cap_pix = p;
  return GUT_OK;
}

// ------------------------------------------------------------- validation
static bool quat_ok(const double q[4]) {
  double n = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
  return std::isfinite(n) && n > 0;
}

static gut_status build_cam(gut_context *ctx, const gut_camera *cam, const gut_options *o, DevCam &c) {
  if (!cam) return fail(ctx, GUT_E_INVALID_ARGUMENT, "camera: NULL");
  if (cam->struct_size != sizeof(gut_camera)) return fail(ctx, GUT_E_INVALID_ARGUMENT, "camera.struct_size");
  if (cam->model < 0 || cam->model > 3) return fail(ctx, GUT_E_INVALID_ARGUMENT, "camera.model");
  if (cam->width <= 0 || cam->height <= 0) return fail(ctx, GUT_E_INVALID_ARGUMENT, "camera.width/height");
  if (!(cam->fx > 0) || !(cam->fy > 0) || !std::isfinite(cam->fx) || !std::isfinite(cam->fy))
    return fail(ctx, GUT_E_INVALID_ARGUMENT, "camera.fx/fy");
  if (!std::isfinite(cam->cx) || !std::isfinite(cam->cy)) return fail(ctx, GUT_E_INVALID_ARGUMENT, "camera.cx/cy");
  if (cam->shutter < 0 || cam->shutter > 4) return fail(ctx, GUT_E_INVALID_ARGUMENT, "camera.shutter");
  if (!quat_ok(cam->q_c2w[0]) || !quat_ok(cam->q_c2w[1])) return fail(ctx, GUT_E_INVALID_ARGUMENT, "camera.q_c2w");
  bool distorted = false;
  for (int i = 0; i < 6; ++i) distorted |= cam->k[i] != 0;
  distorted |= cam->p[0] != 0 || cam->p[1] != 0;
  if (cam->model == GUT_CAM_FISHEYE && !(cam->fov_limit > 0 && cam->fov_limit <= M_PI))
    return fail(ctx, GUT_E_INVALID_ARGUMENT, "camera.fov_limit (FISHEYE needs theta_max in (0, pi])");
  if (cam->model == GUT_CAM_OPENCV && distorted && !(cam->fov_limit > 0))
    return fail(ctx, GUT_E_INVALID_ARGUMENT, "camera.fov_limit (distorted OPENCV needs r_lim > 0)");
  if (cam->model == GUT_CAM_ORTHO && cam->shutter != GUT_SHUTTER_GLOBAL)
    return fail(ctx, GUT_E_UNSUPPORTED, "camera: rolling shutter with ORTHO is not supported");
  if (!o) return fail(ctx, GUT_E_INVALID_ARGUMENT, "options: NULL");
  if (o->struct_size != sizeof(gut_options)) return fail(ctx, GUT_E_INVALID_ARGUMENT, "options.struct_size");
  double a = o->ut_alpha, be = o->ut_beta, ka = o->ut_kappa;
  double lam = a * a * (3.0 + ka) - 3.0;
  if (!(3.0 + lam > 0)) return fail(ctx, GUT_E_INVALID_ARGUMENT, "options.ut_alpha/ut_kappa: 3 + lambda <= 0");
  if (!(o->alpha_min > 0 && o->alpha_min < 1)) return fail(ctx, GUT_E_INVALID_ARGUMENT, "options.alpha_min");
  if (!(o->alpha_max > o->alpha_min && o->alpha_max <= 1)) return fail(ctx, GUT_E_INVALID_ARGUMENT, "options.alpha_max");
  if (!(o->transmittance_min >= 0 && o->transmittance_min < 1))
    return fail(ctx, GUT_E_INVALID_ARGUMENT, "options.transmittance_min");
  if (!(o->cov2d_dilation >= 0) || !(o->near_plane >= 0)) return fail(ctx, GUT_E_INVALID_ARGUMENT, "options.cov2d_dilation/near_plane");
  if (o->rs_max_iterations < 0 || !(o->rs_tolerance_px >= 0)) return fail(ctx, GUT_E_INVALID_ARGUMENT, "options.rs_*");
  if (o->tile_cull != 0 && o->tile_cull != 1) return fail(ctx, GUT_E_INVALID_ARGUMENT, "options.tile_cull");
  if (!(o->kbuffer == 0 || o->kbuffer == 1 || o->kbuffer == 2 || o->kbuffer == 4 || o->kbuffer == 8 || o->kbuffer == 16))
    return fail(ctx, GUT_E_INVALID_ARGUMENT, "options.kbuffer (0, 1, 2, 4, 8 or 16)");
  if (o->kernel_degree < 1 || o->kernel_degree > 8)
    return fail(ctx, GUT_E_INVALID_ARGUMENT, "options.kernel_degree (1..8)");

  memset(&c, 0, sizeof(c));
  c.model = cam->model; c.width = cam->width; c.height = cam->height; c.shutter = cam->shutter;
  c.tiles_x = (cam->width + GUT_TILE - 1) / GUT_TILE;
  c.tiles_y = (cam->height + GUT_TILE - 1) / GUT_TILE;
  if ((int64_t)c.tiles_x * c.tiles_y > 65536) return fail(ctx, GUT_E_UNSUPPORTED, "camera: more than 65536 tiles");
  c.n_tiles = c.tiles_x * c.tiles_y;
  c.tile_cull = o->tile_cull;
  c.kbuf = o->kbuffer;
  c.kdeg = o->kernel_degree;
  c.klam = (float)pow(3.0, 2.0 - (double)o->kernel_degree);  // Supp. A: lambda_n = r^2 / r^n, r = 3
  c.fx = cam->fx; c.fy = cam->fy; c.cx = cam->cx; c.cy = cam->cy;
  for (int i = 0; i < 6; ++i) { c.k[i] = cam->k[i]; c.kf[i] = (float)cam->k[i]; }
  c.p[0] = cam->p[0]; c.p[1] = cam->p[1];
  c.fov = cam->model == GUT_CAM_FISHEYE ? cam->fov_limit : (cam->fov_limit > 0 ? cam->fov_limit : 0);
  c.fxf = (float)c.fx; c.fyf = (float)c.fy; c.cxf = (float)c.cx; c.cyf = (float)c.cy;
  c.inv_wf = 1.f / (float)c.width; c.inv_hf = 1.f / (float)c.height;
  c.pf[0] = (float)c.p[0]; c.pf[1] = (float)c.p[1]; c.fovf = (float)c.fov;
  // pose: R0 from the normalised t=0 quaternion; slerp axis-angle of q0^-1 q1
  double q0[4], q1[4];
  double n0 = sqrt(cam->q_c2w[0][0] * cam->q_c2w[0][0] + cam->q_c2w[0][1] * cam->q_c2w[0][1] +
                   cam->q_c2w[0][2] * cam->q_c2w[0][2] + cam->q_c2w[0][3] * cam->q_c2w[0][3]);
  double n1 = sqrt(cam->q_c2w[1][0] * cam->q_c2w[1][0] + cam->q_c2w[1][1] * cam->q_c2w[1][1] +
                   cam->q_c2w[1][2] * cam->q_c2w[1][2] + cam->q_c2w[1][3] * cam->q_c2w[1][3]);
  for (int i = 0; i < 4; ++i) { q0[i] = cam->q_c2w[0][i] / n0; q1[i] = cam->q_c2w[1][i] / n1; }
  {
    double w = q0[0], x = q0[1], y = q0[2], z = q0[3];
    double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                   2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                   2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    for (int i = 0; i < 9; ++i) { c.R0[i] = R[i]; c.R0f[i] = (float)R[i]; }
  }
  for (int i = 0; i < 3; ++i) c.c0[i] = cam->c_w[0][i];
  c.phi_axis[0] = 1; c.phi_axisf[0] = 1;
  if (cam->shutter != GUT_SHUTTER_GLOBAL) {
    for (int i = 0; i < 3; ++i) { c.dc[i] = cam->c_w[1][i] - cam->c_w[0][i]; c.dcf[i] = (float)c.dc[i]; }
    double d = q0[0] * q1[0] + q0[1] * q1[1] + q0[2] * q1[2] + q0[3] * q1[3];
    if (d < 0) for (int i = 0; i < 4; ++i) q1[i] = -q1[i];
    // q_rel = conj(q0) * q1
    double aw = q0[0], ax = -q0[1], ay = -q0[2], az = -q0[3];
    double bw = q1[0], bx = q1[1], by = q1[2], bz = q1[3];
    double rw = aw * bw - ax * bx - ay * by - az * bz;
    double rx = aw * bx + ax * bw + ay * bz - az * by;
    double ry = aw * by - ax * bz + ay * bw + az * bx;
    double rz = aw * bz + ax * by - ay * bx + az * bw;
    double vn = sqrt(rx * rx + ry * ry + rz * rz);
    c.phi_angle = 2.0 * atan2(vn, rw);
    if (vn > 0) { c.phi_axis[0] = rx / vn; c.phi_axis[1] = ry / vn; c.phi_axis[2] = rz / vn; }
    for (int i = 0; i < 3; ++i) c.phi_axisf[i] = (float)c.phi_axis[i];
    c.phi_anglef = (float)c.phi_angle;
  }
  // UT weights (Eq. 7-8)
  c.gamma = (float)sqrt(3.0 + lam);
  c.wmu0 = (float)(lam / (3.0 + lam));
  c.wmui = (float)(1.0 / (2.0 * (3.0 + lam)));
  c.wsig0 = (float)(lam / (3.0 + lam) + (1.0 - a * a + be));
  c.wsigi = c.wmui;
  c.alpha_min = o->alpha_min; c.alpha_max = o->alpha_max; c.t_min = o->transmittance_min;
  c.dilation = o->cov2d_dilation; c.near_plane = o->near_plane;
  c.rs_tol_px = o->rs_tolerance_px; c.rs_max_iter = o->rs_max_iterations;
  for (int i = 0; i < 3; ++i) c.bg[i] = o->background[i];
  return GUT_OK;
}

// ------------------------------------------------------------------- ABI
extern "C" {

uint32_t gut_abi_version(void) { return GUT_ABI_VERSION; }

void gut_options_default(gut_options *o) {
  if (!o) return;
  memset(o, 0, sizeof(*o));
  o->struct_size = sizeof(gut_options);
  o->ut_alpha = 1.0f; o->ut_beta = 2.0f; o->ut_kappa = 0.0f;
  o->alpha_min = (float)(1.0 / 255.0);
  o->alpha_max = 0.99f;
  o->transmittance_min = 1e-4f;
  o->cov2d_dilation = 0.3f;
  o->near_plane = 0.2f;
  o->rs_max_iterations = 8;
  o->rs_tolerance_px = 1e-4f;
  o->tile_cull = 1;
  o->kernel_degree = 2;
}

gut_status gut_context_create(int32_t dev, gut_context **out) {
  if (!out) return fail(nullptr, GUT_E_INVALID_ARGUMENT, "out: NULL");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(nullptr, GUT_E_UNSUPPORTED, "no CUDA device (there is no CPU fallback)");
  if (dev < 0 || dev >= ndev) return fail(nullptr, GUT_E_INVALID_ARGUMENT, "cuda_device out of range");
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return fail(nullptr, GUT_E_CUDA, "cudaGetDeviceProperties");
  if (p.major != 10 || p.minor != 0)
    return fail(nullptr, GUT_E_UNSUPPORTED, "device is not sm_100 (B200); libgut is built for sm_100a only");
  if (cudaSetDevice(dev) != cudaSuccess) return fail(nullptr, GUT_E_CUDA, "cudaSetDevice");
  gut_context *ctx = new (std::nothrow) gut_context();
  if (!ctx) return fail(nullptr, GUT_E_OUT_OF_MEMORY, "context");
  ctx->device = dev;
  if (const char *e = getenv("GUT_BLEND_TRACE")) ctx->trace_on = atoi(e) != 0;
  if (const char *e = getenv("GUT_BLEND_SEG")) {  // tuning knob: list entries per blend work item
    int v = atoi(e);
    if (v >= 256 && v % 256 == 0) ctx->blend_seg = ctx->blend_seg_rs = v;
  }
  if (const char *e = getenv("GUT_BLEND_WINDOW")) {  // tuning knob: speculative segments in flight per tile
    int v = atoi(e);
    if (v >= 1 && v <= 255) ctx->blend_window = v;  // (queue-1 entries carry the segment in 8 bits)
  }
  // frames in flight (gut_render_batch lanes): the window and the lanes'
  // persistent blend grid in quarter-CTAs per SM
  if (const char *e = getenv("GUT_BLEND_WINDOW_BATCH")) {
    int v = atoi(e);
    if (v >= 1 && v <= 255) ctx->blend_window_batch = v;
  }
  if (const char *e = getenv("GUT_BATCH_GRANT_CAP")) ctx->batch_grant_cap = std::max(0, atoi(e));
  if (const char *e = getenv("GUT_BATCH_BLEND_X4")) {
    int v = atoi(e);
    if (v >= 1 && v <= 64) ctx->batch_x4 = v;
  }
  if (cudaMalloc((void **)&ctx->counters, CNT_ALLOC * sizeof(uint32_t)) != cudaSuccess ||
      cudaMallocHost((void **)&ctx->h_counters, CNT_ALLOC * sizeof(uint32_t)) != cudaSuccess ||
      cudaMemset(ctx->counters, 0, CNT_ALLOC * sizeof(uint32_t)) != cudaSuccess) {
    delete ctx;
    return fail(nullptr, GUT_E_OUT_OF_MEMORY, "counters");
  }
  *out = ctx;
  return GUT_OK;
}

void gut_context_destroy(gut_context *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (gut_context *l : ctx->lanes) gut_context_destroy(l);
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
    for (int i = 0; i < 2; ++i) { cudaEventDestroy(ctx->ev_rendered[i]); cudaEventDestroy(ctx->ev_copied[i]); }
    cudaEventDestroy(ctx->ev_copy_tail);
  }
  for (cudaStream_t st : ctx->lane_streams) cudaStreamDestroy(st);
  for (cudaEvent_t e : ctx->lane_events) cudaEventDestroy(e);
  if (ctx->fork_event) cudaEventDestroy(ctx->fork_event);
  cudaSetDevice(ctx->device);
  void *ps[] = {ctx->dkey, ctx->tiles, ctx->ell, ctx->ell64, ctx->deferred, ctx->k1_list, ctx->big_list, ctx->payload, ctx->sa_k, ctx->sa_v,
                ctx->sb_k, ctx->sb_v,
                ctx->ka, ctx->va, ctx->kb, ctx->vb, ctx->ranges, ctx->tile_work, ctx->img, ctx->st_depth,
                ctx->st_emit, ctx->st_tile, ctx->counters, ctx->pix, ctx->anchors, ctx->seg_base, ctx->unit_ctr, ctx->q1, ctx->q2,
                ctx->bstatus, ctx->part_c, ctx->part_t, ctx->trace, ctx->gacc, ctx->gt0};
  for (void *p : ps) if (p) cudaFree(p);
  if (ctx->h_counters) cudaFreeHost(ctx->h_counters);
  for (auto &set : ctx->tsets)
    for (auto &e : set) cudaEventDestroy(e);
  delete ctx;
}

const char *gut_last_error(const gut_context *ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

gut_status gut_workspace_reserve(gut_context *ctx, int64_t max_keys, int64_t max_gaussians, int32_t max_w,
                                 int32_t max_h) {
  if (!ctx) return fail(nullptr, GUT_E_INVALID_ARGUMENT, "ctx: NULL");
  if (max_keys <= 0 || max_gaussians < 0 || max_w <= 0 || max_h <= 0)
    return fail(ctx, GUT_E_INVALID_ARGUMENT, "gut_workspace_reserve: sizes");
  cudaSetDevice(ctx->device);
  gut_status s;
  if ((s = ensure_n(ctx, (size_t)max_gaussians)) != GUT_OK) return s;
  if ((s = ensure_k(ctx, (size_t)max_keys)) != GUT_OK) return s;
  size_t tiles = (size_t)((max_w + 15) / 16) * ((max_h + 15) / 16);
  if ((s = ensure_tiles(ctx, tiles)) != GUT_OK) return s;
  if ((s = ensure_pix(ctx, (size_t)max_w * max_h)) != GUT_OK) return s;
  // blend work items of either compositing order (segments of "Ours", 8x4
  // units of the k-buffer) so that a reserved render never allocates
  const size_t items = std::max(tiles + (size_t)max_keys / (size_t)std::min(ctx->blend_seg, ctx->blend_seg_rs) + 2,
                                2 * tiles + 2);
  if ((s = ensure_items(ctx, items)) != GUT_OK) return s;
  ctx->reserved = true;
  ctx->res_keys = max_keys; ctx->res_n = max_gaussians; ctx->res_w = max_w; ctx->res_h = max_h;
  for (gut_context *l : ctx->lanes)  // batch lanes follow the reservation
    if ((s = gut_workspace_reserve(l, max_keys, max_gaussians, max_w, max_h)) != GUT_OK)
      return fail(ctx, s, std::string("batch lane: ") + l->err);
  return GUT_OK;
}

gut_status gut_context_set_frames_in_flight(gut_context *ctx, int32_t n) {
  if (!ctx) return fail(nullptr, GUT_E_INVALID_ARGUMENT, "ctx: NULL");
  if (n < 1 || n > 8) return fail(ctx, GUT_E_INVALID_ARGUMENT, "frames_in_flight must be in [1, 8]");
  ctx->frames_in_flight = n;
  return GUT_OK;
}

gut_status gut_scene_create(gut_context *ctx, const gut_gaussians *g, gut_stream stream, gut_scene **out) {
  if (!ctx || !g || !out) return fail(ctx, GUT_E_INVALID_ARGUMENT, "gut_scene_create: NULL argument");
  *out = nullptr;
  if (g->struct_size != sizeof(gut_gaussians)) return fail(ctx, GUT_E_INVALID_ARGUMENT, "gaussians.struct_size");
  if (g->count < 0 || g->count > 0x3FFFFFFF) return fail(ctx, GUT_E_INVALID_ARGUMENT, "gaussians.count");
  if (g->sh_degree < 0 || g->sh_degree > 3) return fail(ctx, GUT_E_INVALID_ARGUMENT, "gaussians.sh_degree");
  if (g->count > 0 && (!g->means || !g->rotations || !g->scales || !g->opacities || !g->sh))
    return fail(ctx, GUT_E_INVALID_ARGUMENT, "gaussians: NULL array");
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  gut_scene *sc = new (std::nothrow) gut_scene();
  if (!sc) return fail(ctx, GUT_E_OUT_OF_MEMORY, "scene");
  sc->device = ctx->device;
  SceneDev &d = sc->d;
  d.n = g->count;
  d.sh_degree = g->sh_degree;
  const int nf = 3 * (g->sh_degree + 1) * (g->sh_degree + 1);
  d.sh_chunks = (nf + 3) / 4;
  size_t n = (size_t)(g->count > 0 ? g->count : 1);
  if (cudaMalloc((void **)&d.pos_opa, n * 16) != cudaSuccess || cudaMalloc((void **)&d.rot, n * 16) != cudaSuccess ||
      cudaMalloc((void **)&d.scale, n * 16) != cudaSuccess ||
      cudaMalloc((void **)&d.sh, n * 16 * d.sh_chunks) != cudaSuccess) {
    gut_scene_destroy(ctx, sc);
    return fail(ctx, GUT_E_OUT_OF_MEMORY, "scene arrays");
  }
  if (g->count > 0) {
    const float *m = g->means, *r = g->rotations, *s = g->scales, *o = g->opacities, *h = g->sh;
    float *raw = nullptr;
    if (!g->on_device) {
      size_t tot = n * (3 + 4 + 3 + 1 + nf);
      if (cudaMalloc((void **)&raw, tot * sizeof(float)) != cudaSuccess) {
        gut_scene_destroy(ctx, sc);
        return fail(ctx, GUT_E_OUT_OF_MEMORY, "scene staging");
      }
      float *p = raw;
      const float *src[5] = {g->means, g->rotations, g->scales, g->opacities, g->sh};
      size_t cnt[5] = {3, 4, 3, 1, (size_t)nf};
      const float **dst[5] = {&m, &r, &s, &o, &h};
      for (int k = 0; k < 5; ++k) {
        cudaMemcpyAsync(p, src[k], n * cnt[k] * sizeof(float), cudaMemcpyHostToDevice, st);
        *dst[k] = p;
        p += n * cnt[k];
      }
    }
    launch_pack_scene(m, r, s, o, h, d, st);
    if (raw) {
      cudaStreamSynchronize(st);
      cudaFree(raw);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      gut_scene_destroy(ctx, sc);
      return fail(ctx, GUT_E_CUDA, std::string("scene pack: ") + cudaGetErrorString(e));
    }
  }
  *out = sc;
  return GUT_OK;
}

void gut_scene_destroy(gut_context *ctx, gut_scene *sc) {
  (void)ctx;
  if (!sc) return;
  cudaSetDevice(sc->device);
  if (sc->d.pos_opa) cudaFree(sc->d.pos_opa);
  if (sc->d.rot) cudaFree(sc->d.rot);
  if (sc->d.scale) cudaFree(sc->d.scale);
  if (sc->d.sh) cudaFree(sc->d.sh);
  delete sc;
}


// Reads and clears the sticky overflow word (CNT_STICKY_OVERFLOW, outside the
// per-render memset) after the work queued on `st` -- i.e. every render issued
// on this context before the call -- has finished.  Synchronises st.
static gut_status take_sticky(gut_context *ctx, cudaStream_t st, bool &overflow) {
  overflow = false;
  uint32_t *w = ctx->counters + CNT_STICKY_OVERFLOW;
  CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_counters + CNT_STICKY_OVERFLOW, w, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemsetAsync(w, 0, sizeof(uint32_t), st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  overflow = ctx->h_counters[CNT_STICKY_OVERFLOW] != 0;
  for (size_t i = 0; i < ctx->lanes.size(); ++i) {  // batch lanes (their renders were joined to st)
    bool o = false;
    gut_status r = take_sticky(ctx->lanes[i], ctx->lane_streams[i], o);
    if (r != GUT_OK) return fail(ctx, r, ctx->lanes[i]->err);
    overflow = overflow || o;
  }
  return GUT_OK;
}

// copy_st (gut_render_batch, host outputs): the device->host copies run on the
// context's copy stream from one of two staging slots, so the next render on
// st does not wait for them (it only waits until the slot it reuses is copied)
static gut_status render_one(gut_context *ctx, const gut_scene *scene, const gut_camera *cam, const gut_options *opt,
                             const gut_outputs *out, cudaStream_t st, gut_stats *stats, bool use_copy_stream = false) {
  if (!ctx) return fail(nullptr, GUT_E_INVALID_ARGUMENT, "ctx: NULL");
  if (!scene) return fail(ctx, GUT_E_INVALID_ARGUMENT, "scene: NULL");
  if (!out || !out->rgb || !out->alpha) return fail(ctx, GUT_E_INVALID_ARGUMENT, "outputs.rgb/alpha: NULL");
  if (scene->device != ctx->device) return fail(ctx, GUT_E_INVALID_ARGUMENT, "scene belongs to another device");
  DevCam dc;
  gut_status s = build_cam(ctx, cam, opt, dc);
  if (s != GUT_OK) return s;
  cudaSetDevice(ctx->device);
  const int64_t N = scene->d.n;
  const size_t npix = (size_t)dc.width * dc.height;
  if ((s = ensure_n(ctx, (size_t)N)) != GUT_OK) return s;
  if ((s = ensure_tiles(ctx, (size_t)dc.n_tiles)) != GUT_OK) return s;
  if (!out->on_device && (s = ensure_pix(ctx, npix)) != GUT_OK) return s;
  if (!ctx->ka && (s = ensure_k(ctx, (size_t)N * 4 + 1024)) != GUT_OK) return s;
  const bool timing = opt->timing != 0;
  cudaEvent_t *ev = nullptr;
  if (timing) {
    if (ctx->tnext == ctx->tsets.size()) {
      std::array<cudaEvent_t, 7> set;
      for (auto &e : set) CUDA_TRY(ctx, cudaEventCreate(&e));
      ctx->tsets.push_back(set);
    }
    ev = ctx->tsets[ctx->tnext++].data();
    cudaEventRecord(ev[0], st);
  }

  uint32_t *cnt = ctx->counters;
  CUDA_TRY(ctx, cudaMemsetAsync(cnt, 0, CNT_WORDS * sizeof(uint32_t), st));
  // look-back epochs of this render (device-side, so a captured render replays correctly)
  uint32_t *part_tot = reinterpret_cast<uint32_t *>(ctx->st_emit);  // K2 partition key totals (final depth pass)
  launch_frame_init(cnt, ctx->bstatus, ctx->cap_items * GUT_TILE_PX, ctx->ranges, dc.n_tiles, part_tot,
                    (int)((N + GUT_EMIT_PART - 1) / GUT_EMIT_PART), st);
  // K1: UT projection
  launch_project(dc, scene->d, ctx->dkey, ctx->tiles, ctx->ell, ctx->ell64, ctx->payload, cnt, ctx->deferred,
                 ctx->k1_list, st);
  if (timing) cudaEventRecord(ev[1], st);
  // K3 level 1: depth sort of the visible Gaussians (4 LSD passes, first one compacts)
  const uint32_t n32 = (uint32_t)N;
  const uint32_t *hd = cnt + CNT_HIST_DEPTH;
  launch_sort_pass(ctx->dkey, nullptr, ctx->sa_k, ctx->sa_v, nullptr, n32, 0, hd, ctx->st_depth,
                   cnt + CNT_TICKETS + 0, cnt + CNT_EPOCH, 0u, true, st);
  launch_sort_pass(ctx->sa_k, ctx->sa_v, ctx->sb_k, ctx->sb_v, cnt + CNT_NVIS, n32, 8, hd + 256, ctx->st_depth,
                   cnt + CNT_TICKETS + 1, cnt + CNT_EPOCH, 1u, false, st);
  launch_sort_pass(ctx->sb_k, ctx->sb_v, ctx->sa_k, ctx->sa_v, cnt + CNT_NVIS, n32, 16, hd + 512, ctx->st_depth,
                   cnt + CNT_TICKETS + 2, cnt + CNT_EPOCH, 2u, false, st);
  launch_sort_pass(ctx->sa_k, ctx->sa_v, nullptr, ctx->sb_v, cnt + CNT_NVIS, n32, 24, hd + 768, ctx->st_depth,
                   cnt + CNT_TICKETS + 3, cnt + CNT_EPOCH, 3u, false, st, nullptr, ctx->tiles, ctx->sb_k, part_tot);
  const uint32_t *order = ctx->sb_v;
  if (timing) cudaEventRecord(ev[2], st);
  // key count: capacity mode keeps the stream asynchronous; otherwise read K back
  size_t n_keys_host;
  if (ctx->reserved) {
    n_keys_host = ctx->cap_k;
  } else {
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_counters, cnt, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    unsigned long long K;
    memcpy(&K, &ctx->h_counters[CNT_K], 8);
    if ((s = ensure_k(ctx, (size_t)K)) != GUT_OK) return s;
    n_keys_host = (size_t)K;
  }
  // K2: depth-ordered scan + emission of (tile, gid) keys
  launch_emit(order, cnt + CNT_NVIS, n32, ctx->tiles, ctx->ell, ctx->ell64, dc.tiles_x, dc.tile_cull, ctx->ka, ctx->va,
              (uint32_t)ctx->cap_k, cnt, part_tot, ctx->big_list, st, ctx->sb_k);
  if (timing) cudaEventRecord(ev[3], st);
  // K3 level 2: stable tile passes
  const uint32_t *ht = cnt + CNT_HIST_TILE;
  const uint32_t *kdev = cnt + CNT_K;  // low word of the u64 key count (K < 2^30)
  const uint32_t nk = (uint32_t)n_keys_host;
  const uint32_t *fk, *fv;
  // (K4 ranges fused into the final tile pass)
  const bool two = dc.n_tiles > 256;
  launch_sort_pass(ctx->ka, ctx->va, ctx->kb, ctx->vb, kdev, nk, 0, ht, ctx->st_tile, cnt + CNT_TICKETS + 5,
                   cnt + CNT_EPOCH, 4u, false, st, two ? nullptr : ctx->ranges);
  fk = ctx->kb; fv = ctx->vb;
  if (two) {
    launch_sort_pass(ctx->kb, ctx->vb, ctx->ka, ctx->va, kdev, nk, 8, ht + 256, ctx->st_tile,
                     cnt + CNT_TICKETS + 6, cnt + CNT_EPOCH, 6u, false, st, ctx->ranges);
    fk = ctx->ka; fv = ctx->va;
  }
  if (timing) cudaEventRecord(ev[4], st);
  if (timing) cudaEventRecord(ev[5], st);  // K4: fused (stage time ~0)
  float *rgb = out->rgb, *alpha = out->alpha, *depth = out->depth;
  int slot = 0;
  if (!out->on_device) {
    if (use_copy_stream) {
      slot = ctx->img_next;
      ctx->img_next ^= 1;
      if (!ctx->copy_stream) {
        CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
          CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_rendered[i], cudaEventDisableTiming));
          CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_copied[i], cudaEventDisableTiming));
          CUDA_TRY(ctx, cudaEventRecord(ctx->ev_copied[i], ctx->copy_stream));
        }
        CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_copy_tail, cudaEventDisableTiming));
      }
      // the blend below writes the slot: wait until its previous copy has read it
      CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->ev_copied[slot], 0));
    } else if (ctx->copy_stream) {  // (slot 0 may still be read by an earlier batch's copy)
      CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->ev_copied[0], 0));
    }
    float *img = ctx->img_slot[slot];
    rgb = img;
    alpha = img + 3 * npix;
    depth = out->depth ? img + 4 * npix : nullptr;
  }
  // a5: pixel rays relative to per-tile anchors — a function of the intrinsics
  // only for global shutter (built once per intrinsics), per view for RS
  {
    double key[20] = {(double)dc.model, (double)dc.width, (double)dc.height, dc.fx, dc.fy, dc.cx, dc.cy,
                      dc.k[0], dc.k[1], dc.k[2], dc.k[3], dc.k[4], dc.k[5], dc.p[0], dc.p[1], dc.fov,
                      (double)dc.shutter, 0, 0, 0};
    const bool cacheable = dc.shutter == GUT_SHUTTER_GLOBAL;
    if (!cacheable || !ctx->lut_valid || memcmp(key, ctx->lut_key, sizeof(key)) != 0) {
      launch_rays(dc, ctx->pix, ctx->anchors, st);
      memcpy(ctx->lut_key, key, sizeof(key));
      ctx->lut_valid = cacheable;
    }
  }
  const int bseg = dc.shutter != SH_GLOBAL ? ctx->blend_seg_rs : ctx->blend_seg;
  const int bwin = use_copy_stream ? ctx->blend_window_batch : ctx->blend_window;
  // (k-buffer: one item per tile but twice the units per tile -> q1 needs 2 x n_tiles x GUT_BLEND_WARPS)
  const size_t max_items = dc.kbuf > 0 ? 2 * (size_t)dc.n_tiles + 2
                                       : (size_t)dc.n_tiles + ctx->cap_k / (size_t)bseg + 2;
  if ((s = ensure_items(ctx, max_items)) != GUT_OK) return s;
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->tile_work, 0, (size_t)dc.n_tiles * sizeof(uint2), st));
  const size_t n_units = (size_t)dc.n_tiles * GUT_BLEND_WARPS;
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->unit_ctr, 0, 4 * n_units * sizeof(uint32_t), st));
  if (dc.kbuf > 0)  // one segment per tile (the buffer state runs along the whole list), 8x4 units
    launch_plan(ctx->ranges, dc.n_tiles, 1 << 30, 1, ctx->seg_base, ctx->q1, cnt, st, GUT_KBUF_UNITS);
  else
    launch_plan(ctx->ranges, dc.n_tiles, bseg, bwin, ctx->seg_base, ctx->q1, cnt, st);
  BlendBufs bb;
  bb.ranges = ctx->ranges; bb.gids = fv; bb.payload = ctx->payload; bb.pix = ctx->pix; bb.anchors = ctx->anchors;
  bb.seg_base = ctx->seg_base; bb.granted = ctx->unit_ctr; bb.next_s = ctx->unit_ctr + n_units; bb.unit_done = ctx->unit_ctr + 2 * n_units;
  bb.q1_taken = ctx->unit_ctr + 3 * n_units;
  bb.q1 = ctx->q1; bb.q2 = ctx->q2;
  bb.status = ctx->bstatus;
  bb.part_c = ctx->part_c; bb.part_t = ctx->part_t;
  bb.tile_work = ctx->tile_work; bb.seg = bseg; bb.window = bwin; bb.n_tiles = dc.n_tiles;
  bb.trace = nullptr;
  if (ctx->trace_on) {
    if (ctx->cap_trace < max_items) {
      size_t dummy = 0;
      CUDA_TRY(ctx, regrow(ctx->trace, dummy, 2 * GUT_BLEND_WARPS * max_items));
      ctx->cap_trace = max_items;
    }
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->trace, 0, 2 * GUT_BLEND_WARPS * max_items * sizeof(uint4), st));
    bb.trace = ctx->trace;
    ctx->last_items = max_items;
  }
  bb.epoch = cnt + CNT_EPOCH;
  bb.rgb = rgb; bb.alpha = alpha; bb.depth = depth; bb.counters = cnt;
  bb.grid_x4 = use_copy_stream ? ctx->batch_x4 : 0;  // (frames in flight: a smaller persistent blend grid)
  bb.grant_cap = use_copy_stream ? ctx->batch_grant_cap : 0;
  if (dc.kbuf > 0) launch_blend_kbuf(dc, bb, st);
  else launch_blend(dc, bb, st);
  if (timing) cudaEventRecord(ev[6], st);
  {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ctx, GUT_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  }
  if (!out->on_device) {
    cudaStream_t cs = st;
    if (use_copy_stream) {
      CUDA_TRY(ctx, cudaEventRecord(ctx->ev_rendered[slot], st));
      CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_rendered[slot], 0));
      cs = ctx->copy_stream;
    }
    CUDA_TRY(ctx, cudaMemcpyAsync(out->rgb, rgb, 3 * npix * sizeof(float), cudaMemcpyDeviceToHost, cs));
    CUDA_TRY(ctx, cudaMemcpyAsync(out->alpha, alpha, npix * sizeof(float), cudaMemcpyDeviceToHost, cs));
    if (out->depth)
      CUDA_TRY(ctx, cudaMemcpyAsync(out->depth, depth, npix * sizeof(float), cudaMemcpyDeviceToHost, cs));
    if (use_copy_stream) CUDA_TRY(ctx, cudaEventRecord(ctx->ev_copied[slot], cs));
  }
  ctx->last_n = N;
  ctx->last_tiles = dc.n_tiles;
  ctx->last_order = order;
  ctx->last_cam = dc;
  ctx->last_scene = scene;
  ctx->last_keys = fk;
  ctx->last_vals = fv;
  if (stats) {
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_counters, cnt, 32 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    const uint32_t *h = ctx->h_counters;
    memset(stats, 0, sizeof(*stats));
    unsigned long long K, pe, pc, pt;
    memcpy(&K, &h[CNT_K], 8);
    memcpy(&pe, &h[CNT_PAIRS_EVAL], 8);
    memcpy(&pc, &h[CNT_PAIRS_CONTRIB], 8);
    memcpy(&pt, &h[CNT_TERMINATED], 8);
    stats->n_input = N;
    stats->n_visible = h[CNT_NVIS];
    stats->n_keys = (int64_t)K;
    stats->n_tiles = dc.n_tiles;
    stats->max_tile_len = (int32_t)h[CNT_MAXLEN];
    stats->pairs_evaluated = (int64_t)pe;
    stats->pairs_contributing = (int64_t)pc;
    stats->pixels_terminated = (int64_t)pt;
    bool sticky = false;  // a truncated earlier render (stats = NULL) is reported here too
    if ((s = take_sticky(ctx, st, sticky)) != GUT_OK) return s;
    stats->overflow = (h[CNT_OVERFLOW] != 0 || K > ctx->cap_k || sticky) ? 1 : 0;
    if (timing) {
      for (int i = 0; i < 6; ++i) cudaEventElapsedTime(&stats->ms_stage[i], ev[i], ev[i + 1]);
      cudaEventElapsedTime(&stats->ms_stage[6], ev[0], ev[6]);
    }
    if (stats->overflow) return fail(ctx, GUT_E_CAPACITY, "key capacity exceeded (gut_workspace_reserve)");
  }
  return GUT_OK;
}

gut_status gut_render(gut_context *ctx, const gut_scene *scene, const gut_camera *cam, const gut_options *opt,
                      const gut_outputs *out, gut_stream s, gut_stats *stats) {
  return render_one(ctx, scene, cam, opt, out, (cudaStream_t)s, stats);
}

gut_status gut_render_backward(gut_context *ctx, const gut_scene *scene, const gut_camera *cam,
                               const gut_options *opt, const float *rgb, const float *alpha, const float *depth,
                               const float *grad_rgb, const float *grad_alpha, const float *grad_depth,
                               const gut_gradients *grads, gut_stream s) {
  if (!ctx) return fail(nullptr, GUT_E_INVALID_ARGUMENT, "ctx: NULL");
  if (!scene || !grads) return fail(ctx, GUT_E_INVALID_ARGUMENT, "scene / grads: NULL");
  if (!rgb || !alpha || !grad_rgb) return fail(ctx, GUT_E_INVALID_ARGUMENT, "rgb / alpha / grad_rgb: NULL");
  if (grad_depth && !depth) return fail(ctx, GUT_E_INVALID_ARGUMENT, "grad_depth needs the forward depth");
  if (scene->d.n > 0 && (!grads->means || !grads->rotations || !grads->scales || !grads->opacities || !grads->sh))
    return fail(ctx, GUT_E_INVALID_ARGUMENT, "grads: NULL buffer");
  DevCam dc;
  gut_status st_ = build_cam(ctx, cam, opt, dc);
  if (st_ != GUT_OK) return st_;
  if (dc.model == CAM_ORTHO || dc.kbuf != 0)
    return fail(ctx, GUT_E_UNSUPPORTED, "backward: PINHOLE/OPENCV/FISHEYE (any shutter, any degree), kbuffer 0 only");
  if (ctx->last_scene != scene || memcmp(&ctx->last_cam, &dc, sizeof(DevCam)) != 0)
    return fail(ctx, GUT_E_INVALID_ARGUMENT, "backward: scene / camera / options differ from the last render");
  cudaSetDevice(ctx->device);
  const int64_t N = scene->d.n;
  if (ctx->cap_gacc < (size_t)N) {
    if (ctx->gacc) cudaFree(ctx->gacc);
    if (ctx->gt0) cudaFree(ctx->gt0);
    ctx->gacc = nullptr;
    ctx->gt0 = nullptr;
    CUDA_TRY(ctx, cudaMalloc(&ctx->gacc, (size_t)16 * (N > 0 ? N : 1) * sizeof(long long)));
    CUDA_TRY(ctx, cudaMalloc(&ctx->gt0, (size_t)(N > 0 ? N : 1) * sizeof(float)));
    ctx->cap_gacc = (size_t)N;
  }
  BwdBufs b;
  b.ranges = ctx->ranges; b.gids = ctx->last_vals; b.payload = ctx->payload; b.pix = ctx->pix;
  b.anchors = ctx->anchors; b.tiles = ctx->tiles;
  b.rgb = rgb; b.alpha = alpha; b.depth = depth; b.g_rgb = grad_rgb; b.g_alpha = grad_alpha; b.g_depth = grad_depth;
  b.acc = ctx->gacc;
  b.order = ctx->q1; b.seg_base = ctx->seg_base; b.counters = ctx->counters;  // (forward plan scratch, reused)
  b.t0 = dc.shutter != GUT_SHUTTER_GLOBAL ? ctx->gt0 : nullptr;
  b.d_means = grads->means; b.d_rots = grads->rotations; b.d_scales = grads->scales; b.d_opac = grads->opacities;
  b.d_sh = grads->sh; b.d_rgb = grads->rgb; b.densify = grads->densify;
  launch_backward(dc, scene->d, b, (cudaStream_t)s);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, GUT_E_CUDA, std::string("backward launch: ") + cudaGetErrorString(e));
  return GUT_OK;
}

gut_status gut_projection_quality(gut_context *ctx, const gut_scene *scene, const gut_camera *cam,
                                  const gut_options *opt, int32_t n_samples, uint64_t seed, gut_quality *out,
                                  gut_stream s) {
  static_assert(sizeof(gut_quality) == sizeof(QualityRec), "gut_quality layout");
  if (!ctx) return fail(nullptr, GUT_E_INVALID_ARGUMENT, "ctx: NULL");
  if (!scene || !out) return fail(ctx, GUT_E_INVALID_ARGUMENT, "scene / out: NULL");
  if (n_samples < 2) return fail(ctx, GUT_E_INVALID_ARGUMENT, "n_samples < 2");
  DevCam dc;
  gut_status st_ = build_cam(ctx, cam, opt, dc);
  if (st_ != GUT_OK) return st_;
  cudaSetDevice(ctx->device);
  launch_quality(dc, scene->d, n_samples, (unsigned long long)seed, reinterpret_cast<QualityRec *>(out),
                 (cudaStream_t)s);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, GUT_E_CUDA, std::string("quality launch: ") + cudaGetErrorString(e));
  return GUT_OK;
}

// Child contexts and streams of the batch lanes (created once, reserved like ctx).
static gut_status ensure_lanes(gut_context *ctx, int n) {
  while ((int)ctx->lanes.size() < n - 1) {
    gut_context *l = nullptr;
    gut_status r = gut_context_create(ctx->device, &l);
    if (r != GUT_OK) return fail(ctx, r, "batch lane context");
    l->blend_seg = ctx->blend_seg;
    l->blend_seg_rs = ctx->blend_seg_rs;
    l->blend_window = ctx->blend_window;
    l->blend_window_batch = ctx->blend_window_batch;
    l->batch_x4 = ctx->batch_x4;
    l->batch_grant_cap = ctx->batch_grant_cap;
    l->frames_in_flight = 1;
    if (ctx->reserved && (r = gut_workspace_reserve(l, ctx->res_keys, ctx->res_n, ctx->res_w, ctx->res_h)) != GUT_OK) {
      gut_context_destroy(l);
      return fail(ctx, r, "batch lane workspace");
    }
    cudaStream_t st;
    cudaEvent_t ev;
    CUDA_TRY(ctx, cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CUDA_TRY(ctx, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    ctx->lanes.push_back(l);
    ctx->lane_streams.push_back(st);
    ctx->lane_events.push_back(ev);
  }
  if (!ctx->fork_event) CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->fork_event, cudaEventDisableTiming));
  return GUT_OK;
}

gut_status gut_render_batch(gut_context *ctx, const gut_scene *scene, const gut_camera *cams, int32_t n_views,
                            const gut_options *opt, const gut_outputs *outs, gut_stream s, gut_stats *stats) {
  if (!ctx) return fail(nullptr, GUT_E_INVALID_ARGUMENT, "ctx: NULL");
  if (n_views < 0 || (n_views > 0 && (!cams || !outs))) return fail(ctx, GUT_E_INVALID_ARGUMENT, "batch arguments");
  cudaStream_t st = (cudaStream_t)s;
  const int L = std::min(ctx->frames_in_flight, (int)n_views);
  if (stats || L <= 1) {  // one frame at a time (stats synchronise per view anyway)
    for (int32_t v = 0; v < n_views; ++v) {
      gut_status r = render_one(ctx, scene, &cams[v], opt, &outs[v], st, stats ? &stats[v] : nullptr);
      if (r != GUT_OK) return r;
    }
    return GUT_OK;
  }
  cudaSetDevice(ctx->device);
  gut_status r = ensure_lanes(ctx, L);
  if (r != GUT_OK) return r;
  // fork: the lanes start after the work already queued on the caller's stream
  CUDA_TRY(ctx, cudaEventRecord(ctx->fork_event, st));
  for (int i = 0; i < L - 1; ++i) CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->lane_streams[i], ctx->fork_event, 0));
  // views round-robin over the lanes: frame v + 1's first kernels overlap frame v's tail
  for (int32_t v = 0; v < n_views && r == GUT_OK; ++v) {
    const int l = v % L;
    gut_context *c = l == 0 ? ctx : ctx->lanes[l - 1];
    r = render_one(c, scene, &cams[v], opt, &outs[v], l == 0 ? st : ctx->lane_streams[l - 1], nullptr, true);
    if (r != GUT_OK && c != ctx) fail(ctx, r, c->err);
  }
  // join: the caller's stream waits for every lane and every lane's host
  // copies (also after an error)
  for (int i = 0; i < L - 1; ++i) {
    CUDA_TRY(ctx, cudaEventRecord(ctx->lane_events[i], ctx->lane_streams[i]));
    CUDA_TRY(ctx, cudaStreamWaitEvent(st, ctx->lane_events[i], 0));
  }
  for (int i = 0; i < L; ++i) {
    gut_context *c = i == 0 ? ctx : ctx->lanes[i - 1];
    if (c->copy_stream) {
      CUDA_TRY(ctx, cudaEventRecord(c->ev_copy_tail, c->copy_stream));
      CUDA_TRY(ctx, cudaStreamWaitEvent(st, c->ev_copy_tail, 0));
    }
  }
  return r;
}

gut_status gut_timing_read(gut_context *ctx, double ms_sum[7], int32_t *n_renders, int32_t reset) {
  if (!ctx || !ms_sum) return fail(ctx, GUT_E_INVALID_ARGUMENT, "gut_timing_read: NULL argument");
  cudaSetDevice(ctx->device);
  for (int i = 0; i < 7; ++i) ms_sum[i] = 0;
  int32_t n = 0;
  // this context's renders and its batch lanes' (gut_render_batch)
  for (size_t li = 0; li <= ctx->lanes.size(); ++li) {
    gut_context *c = li == 0 ? ctx : ctx->lanes[li - 1];
    for (size_t r = 0; r < c->tnext; ++r) {
      auto &e = c->tsets[r];
      CUDA_TRY(ctx, cudaEventSynchronize(e[6]));
      float t;
      for (int i = 0; i < 6; ++i) {
        CUDA_TRY(ctx, cudaEventElapsedTime(&t, e[i], e[i + 1]));
        ms_sum[i] += t;
      }
      CUDA_TRY(ctx, cudaEventElapsedTime(&t, e[0], e[6]));
      ms_sum[6] += t;
    }
    n += (int32_t)c->tnext;
    if (reset) c->tnext = 0;
  }
  if (n_renders) *n_renders = n;
  CUDA_TRY(ctx, cudaDeviceSynchronize());  // (renders without timing events too)
  bool sticky = false;
  gut_status s = take_sticky(ctx, (cudaStream_t)0, sticky);
  if (s != GUT_OK) return s;
  if (sticky) return fail(ctx, GUT_E_CAPACITY, "key capacity exceeded by an earlier render (gut_workspace_reserve)");
  return GUT_OK;
}

gut_status gut_check(gut_context *ctx, gut_stream stream) {
  if (!ctx) return fail(nullptr, GUT_E_INVALID_ARGUMENT, "ctx: NULL");
  cudaSetDevice(ctx->device);
  bool sticky = false;
  gut_status s = take_sticky(ctx, (cudaStream_t)stream, sticky);
  if (s != GUT_OK) return s;
  if (sticky) return fail(ctx, GUT_E_CAPACITY, "key capacity exceeded by an earlier render (gut_workspace_reserve)");
  return GUT_OK;
}

gut_status gut_debug_copy_stage(gut_context *ctx, int32_t stage, void *host_dst, size_t bytes, size_t *bytes_needed) {
  if (!ctx) return fail(nullptr, GUT_E_INVALID_ARGUMENT, "ctx: NULL");
  cudaSetDevice(ctx->device);
  CUDA_TRY(ctx, cudaDeviceSynchronize());
  uint32_t h[8];
  CUDA_TRY(ctx, cudaMemcpy(h, ctx->counters, sizeof(h), cudaMemcpyDeviceToHost));
  unsigned long long K;
  memcpy(&K, &h[CNT_K], 8);
  if (K > ctx->cap_k) K = ctx->cap_k;
  const size_t N = (size_t)ctx->last_n, nv = h[CNT_NVIS];
  size_t need = 0;
  switch (stage) {
    case GUT_STAGE_PROJECT: need = N * sizeof(gut_proj_record); break;
    case GUT_STAGE_DEPTH_ORDER: need = nv * sizeof(uint32_t); break;
    case GUT_STAGE_SORTED: need = (size_t)K * 2 * sizeof(uint32_t); break;
    case GUT_STAGE_RANGES:
    case GUT_STAGE_TILE_WORK: need = (size_t)ctx->last_tiles * 2 * sizeof(uint32_t); break;
    case GUT_STAGE_BLEND_TRACE: need = ctx->trace ? 2 * GUT_BLEND_WARPS * ctx->last_items * sizeof(uint4) : 0; break;
    case GUT_STAGE_COUNTERS: need = 64 * sizeof(uint32_t); break;
    case GUT_STAGE_RAYS: need = (size_t)ctx->last_tiles * (GUT_TILE_PX * sizeof(float4) + 4 * 8 * sizeof(float)); break;
    default: return fail(ctx, GUT_E_INVALID_ARGUMENT, "stage");
  }
  if (bytes_needed) *bytes_needed = need;
  if (!host_dst || bytes < need) return GUT_OK;
  if (stage == GUT_STAGE_PROJECT) {
    uint32_t *tl = new uint32_t[N + 1], *dk = new uint32_t[N + 1];
    float4 *el = new float4[2 * N + 1], *pl = new float4[GUT_PAYLOAD_F4 * N + 1];
    cudaMemcpy(tl, ctx->tiles, N * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(dk, ctx->dkey, N * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(el, ctx->ell, N * 32, cudaMemcpyDeviceToHost);
    cudaMemcpy(pl, ctx->payload, N * GUT_PAYLOAD_F4 * sizeof(float4), cudaMemcpyDeviceToHost);
    gut_proj_record *r = (gut_proj_record *)host_dst;
    for (size_t i = 0; i < N; ++i) {
      memset(&r[i], 0, sizeof(r[i]));
      // tile code (gut_internal.cuh ell_tile_code) -> tile count
      r[i].tiles = (tl[i] >> 31) ? (tl[i] & 0x7FFFFFFFu)
                                 : (uint32_t)__builtin_popcount(tl[i] & ((tl[i] >> 30) ? 0xFFFFu : 0x1FFu));
      if (!tl[i]) continue;
      float4 a = el[2 * i], b = el[2 * i + 1], p4 = pl[GUT_PAYLOAD_F4 * i + 4];
      r[i].vx = a.x; r[i].vy = a.y; r[i].cxx = a.z; r[i].cxy = a.w; r[i].cyy = b.x; r[i].k2 = fabsf(b.y);
      memcpy(&r[i].depth, &dk[i], 4);
      r[i].rgb[0] = p4.x; r[i].rgb[1] = p4.y; r[i].rgb[2] = p4.z;
      uint32_t r0, r1;
      memcpy(&r0, &b.z, 4);
      memcpy(&r1, &b.w, 4);
      r[i].rect[0] = (uint16_t)(r0 & 0xFFFF); r[i].rect[1] = (uint16_t)(r0 >> 16);
      r[i].rect[2] = (uint16_t)(r1 & 0xFFFF); r[i].rect[3] = (uint16_t)(r1 >> 16);
    }
    delete[] tl; delete[] dk; delete[] el; delete[] pl;
  } else if (stage == GUT_STAGE_DEPTH_ORDER) {
    CUDA_TRY(ctx, cudaMemcpy(host_dst, ctx->last_order, need, cudaMemcpyDeviceToHost));
  } else if (stage == GUT_STAGE_SORTED) {
    uint32_t *t = new uint32_t[K + 1], *g = new uint32_t[K + 1];
    cudaMemcpy(t, ctx->last_keys, K * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(g, ctx->last_vals, K * 4, cudaMemcpyDeviceToHost);
    uint32_t *o = (uint32_t *)host_dst;
    for (size_t k = 0; k < K; ++k) { o[2 * k] = t[k]; o[2 * k + 1] = g[k]; }
    delete[] t; delete[] g;
  } else if (stage == GUT_STAGE_RANGES) {
    CUDA_TRY(ctx, cudaMemcpy(host_dst, ctx->ranges, need, cudaMemcpyDeviceToHost));
    uint32_t *r = (uint32_t *)host_dst;  // empty tiles: (UINT_MAX, 0) on the device -> (0, 0)
    for (size_t t = 0; t < need / 8; ++t)
      if (r[2 * t + 1] <= r[2 * t]) r[2 * t] = r[2 * t + 1] = 0;
  } else if (stage == GUT_STAGE_COUNTERS) {
    CUDA_TRY(ctx, cudaMemcpy(host_dst, ctx->counters, need, cudaMemcpyDeviceToHost));
  } else if (stage == GUT_STAGE_BLEND_TRACE) {
    CUDA_TRY(ctx, cudaMemcpy(host_dst, ctx->trace, need, cudaMemcpyDeviceToHost));
  } else if (stage == GUT_STAGE_RAYS) {
    const size_t nt = (size_t)ctx->last_tiles;
    float4 *px = new float4[nt * GUT_TILE_PX + 1];
    TileAnchor *an = new TileAnchor[nt + 1];
    cudaMemcpy(px, ctx->pix, nt * GUT_TILE_PX * sizeof(float4), cudaMemcpyDeviceToHost);
    cudaMemcpy(an, ctx->anchors, nt * sizeof(TileAnchor), cudaMemcpyDeviceToHost);
    char *o = (char *)host_dst;
    for (size_t t = 0; t < nt; ++t) {
      memcpy(o, px + t * GUT_TILE_PX, GUT_TILE_PX * sizeof(float4));
      memcpy(o + GUT_TILE_PX * sizeof(float4), an[t].fit, sizeof(an[t].fit));
      o += GUT_TILE_PX * sizeof(float4) + sizeof(an[t].fit);
    }
    delete[] px; delete[] an;
  } else {
    CUDA_TRY(ctx, cudaMemcpy(host_dst, ctx->tile_work, need, cudaMemcpyDeviceToHost));
  }
  return GUT_OK;
}

}  // extern "C"
