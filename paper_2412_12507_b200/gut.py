"""Thin Python binding of libgut (include/gut.h): argument marshalling only.

Every step of the render runs in the sm_100a kernels behind the C ABI; this
module only converts Python values into the ABI structs and passes pointers.
PyTorch is used for device memory and streams.  There is no CPU fallback: if
libgut.so is missing or the device is not a B200, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GUT_LIB") or os.path.join(_HERE, "libgut.so")  # GUT_LIB: tuning experiments only

GUT_OK = 0
STATUS = {0: "GUT_OK", 1: "GUT_E_INVALID_ARGUMENT", 2: "GUT_E_UNSUPPORTED", 3: "GUT_E_OUT_OF_MEMORY",
          4: "GUT_E_CAPACITY", 5: "GUT_E_CUDA", 6: "GUT_E_INTERNAL"}
MODELS = {"pinhole": 0, "opencv": 1, "fisheye": 2, "ortho": 3}
SHUTTERS = {"global": 0, "top_to_bottom": 1, "left_to_right": 2, "bottom_to_top": 3, "right_to_left": 4}
STAGE_PROJECT, STAGE_DEPTH_ORDER, STAGE_SORTED, STAGE_RANGES, STAGE_TILE_WORK = 1, 2, 3, 4, 5
STAGE_BLEND_TRACE, STAGE_COUNTERS, STAGE_RAYS = 6, 7, 8


class gut_camera(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("model", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("k", C.c_double * 6), ("p", C.c_double * 2), ("fov_limit", C.c_double),
                ("shutter", C.c_int32), ("pad0", C.c_int32), ("q_c2w", (C.c_double * 4) * 2),
                ("c_w", (C.c_double * 3) * 2)]


class gut_gaussians(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("sh_degree", C.c_int32), ("count", C.c_int64),
                ("on_device", C.c_int32), ("pad0", C.c_int32), ("means", C.c_void_p), ("rotations", C.c_void_p),
                ("scales", C.c_void_p), ("opacities", C.c_void_p), ("sh", C.c_void_p)]


class gut_options(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("ut_alpha", C.c_float), ("ut_beta", C.c_float),
                ("ut_kappa", C.c_float), ("alpha_min", C.c_float), ("alpha_max", C.c_float),
                ("transmittance_min", C.c_float), ("cov2d_dilation", C.c_float), ("near_plane", C.c_float),
                ("rs_max_iterations", C.c_int32), ("rs_tolerance_px", C.c_float), ("tile_cull", C.c_int32),
                ("background", C.c_float * 3), ("timing", C.c_int32), ("kbuffer", C.c_int32),
                ("kernel_degree", C.c_int32)]


class gut_outputs(C.Structure):
    _fields_ = [("rgb", C.c_void_p), ("alpha", C.c_void_p), ("depth", C.c_void_p), ("on_device", C.c_int32),
                ("pad0", C.c_int32)]


class gut_stats(C.Structure):
    _fields_ = [("n_input", C.c_int64), ("n_visible", C.c_int64), ("n_keys", C.c_int64), ("n_tiles", C.c_int32),
                ("max_tile_len", C.c_int32), ("pairs_evaluated", C.c_int64), ("pairs_contributing", C.c_int64),
                ("pixels_terminated", C.c_int64), ("ms_stage", C.c_float * 7), ("overflow", C.c_int32),
                ("pad0", C.c_int32)]

    def as_dict(self):
        return {k: (list(getattr(self, k)) if k == "ms_stage" else getattr(self, k))
                for k, _ in self._fields_ if k != "pad0"}


class gut_proj_record(C.Structure):
    _fields_ = [("vx", C.c_float), ("vy", C.c_float), ("cxx", C.c_float), ("cxy", C.c_float), ("cyy", C.c_float),
                ("k2", C.c_float), ("depth", C.c_float), ("rgb", C.c_float * 3), ("tiles", C.c_uint32),
                ("rect", C.c_uint16 * 4)]


class gut_gradients(C.Structure):
    _fields_ = [("means", C.c_void_p), ("rotations", C.c_void_p), ("scales", C.c_void_p), ("opacities", C.c_void_p),
                ("sh", C.c_void_p), ("rgb", C.c_void_p), ("densify", C.c_void_p)]


EXPORTS = ["gut_abi_version", "gut_options_default", "gut_context_create", "gut_context_destroy",
           "gut_last_error", "gut_workspace_reserve", "gut_scene_create", "gut_scene_destroy", "gut_render",
           "gut_render_batch", "gut_render_backward", "gut_projection_quality", "gut_timing_read",
           "gut_debug_copy_stage"]
STAGE_NAMES = ["K1_project", "K3_sort_depth", "K2_emit", "K3_sort_tile", "K4_ranges", "K5_blend", "total"]

_lib = None


class GutError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def lib():
    """Loads libgut.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2412_12507_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.gut_abi_version.restype = C.c_uint32
        L.gut_options_default.argtypes = [C.POINTER(gut_options)]
        L.gut_context_create.argtypes = [i32, C.POINTER(vp)]
        L.gut_context_destroy.argtypes = [vp]
        L.gut_last_error.argtypes = [vp]
        L.gut_last_error.restype = C.c_char_p
        L.gut_workspace_reserve.argtypes = [vp, i64, i64, i32, i32]
        L.gut_scene_create.argtypes = [vp, C.POINTER(gut_gaussians), vp, C.POINTER(vp)]
        L.gut_scene_destroy.argtypes = [vp, vp]
        L.gut_render.argtypes = [vp, vp, C.POINTER(gut_camera), C.POINTER(gut_options), C.POINTER(gut_outputs), vp,
                                 C.POINTER(gut_stats)]
        L.gut_render_batch.argtypes = [vp, vp, C.POINTER(gut_camera), i32, C.POINTER(gut_options),
                                       C.POINTER(gut_outputs), vp, C.POINTER(gut_stats)]
        L.gut_debug_copy_stage.argtypes = [vp, i32, vp, C.c_size_t, C.POINTER(C.c_size_t)]
        L.gut_render_backward.argtypes = [vp, vp, C.POINTER(gut_camera), C.POINTER(gut_options), vp, vp, vp, vp, vp,
                                          vp, C.POINTER(gut_gradients), vp]
        L.gut_projection_quality.argtypes = [vp, vp, C.POINTER(gut_camera), C.POINTER(gut_options), i32, C.c_uint64,
                                             vp, vp]
        L.gut_timing_read.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_int32), i32]
        L.gut_check.argtypes = [vp, vp]
        L.gut_context_set_frames_in_flight.argtypes = [vp, i32]
        for name in ("gut_context_create", "gut_workspace_reserve", "gut_scene_create", "gut_render",
                     "gut_render_batch", "gut_render_backward", "gut_projection_quality", "gut_timing_read",
                     "gut_debug_copy_stage", "gut_check", "gut_context_set_frames_in_flight"):
            getattr(L, name).restype = C.c_int
        L.gut_options_default.restype = None
        L.gut_context_destroy.restype = None
        L.gut_scene_destroy.restype = None
        _lib = L
    return _lib


def _check(status, ctx=None):
    if status != GUT_OK:
        msg = lib().gut_last_error(ctx)
        raise GutError(status, msg.decode() if msg else "")


# ------------------------------------------------------------- marshalling
def make_camera(cam) -> gut_camera:
    """Any object with the scenegen.Camera attributes -> gut_camera."""
    c = gut_camera()
    c.struct_size = C.sizeof(gut_camera)
    c.model = MODELS[cam.model]
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    for i in range(6):
        c.k[i] = float(cam.k[i])
    c.p[0], c.p[1] = float(cam.p[0]), float(cam.p[1])
    c.fov_limit = float(cam.fov_limit)
    c.shutter = SHUTTERS[cam.shutter]
    for t in range(2):
        for i in range(4):
            c.q_c2w[t][i] = float(cam.q_c2w[t][i])
        for i in range(3):
            c.c_w[t][i] = float(cam.c_w[t][i])
    return c


def make_options(opt=None, timing: bool = False) -> gut_options:
    o = gut_options()
    lib().gut_options_default(C.byref(o))
    if opt is not None:
        o.ut_alpha, o.ut_beta, o.ut_kappa = opt.ut_alpha, opt.ut_beta, opt.ut_kappa
        o.alpha_min, o.alpha_max = opt.alpha_min, opt.alpha_max
        o.transmittance_min, o.cov2d_dilation = opt.transmittance_min, opt.cov2d_dilation
        o.near_plane, o.rs_max_iterations = opt.near_plane, int(opt.rs_max_iterations)
        o.rs_tolerance_px, o.tile_cull = opt.rs_tolerance_px, int(opt.tile_cull)
        for i in range(3):
            o.background[i] = opt.background[i]
        o.kbuffer = int(getattr(opt, "kbuffer", 0))
        o.kernel_degree = int(getattr(opt, "kernel_degree", 2))
    o.timing = int(timing)
    return o


# ------------------------------------------------------------- same-name calls
def gut_abi_version() -> int:
    return int(lib().gut_abi_version())


def gut_context_create(device: int = 0):
    h = C.c_void_p()
    _check(lib().gut_context_create(device, C.byref(h)))
    return h


def gut_context_destroy(ctx):
    lib().gut_context_destroy(ctx)


def gut_workspace_reserve(ctx, max_keys: int, max_gaussians: int, max_w: int, max_h: int):
    _check(lib().gut_workspace_reserve(ctx, int(max_keys), int(max_gaussians), int(max_w), int(max_h)), ctx)


def gut_scene_create(ctx, means, rotations, scales, opacities, sh, sh_degree: int, stream=None):
    """Arrays are torch CUDA tensors (on_device) or numpy float32 arrays (host)."""
    nc = (int(sh_degree) + 1) ** 2
    if int(sh.shape[0]) != int(means.shape[0]) or (sh.ndim == 3 and (sh.shape[1] != nc or sh.shape[2] != 3)) \
            or (sh.ndim == 2 and sh.shape[1] != 3 * nc) or sh.ndim not in (2, 3):
        raise ValueError(f"sh must be [N, {nc}, 3] (or [N, {3 * nc}]) for sh_degree {sh_degree}, "
                         f"got {tuple(sh.shape)}")
    g = gut_gaussians()
    g.struct_size = C.sizeof(gut_gaussians)
    g.sh_degree = int(sh_degree)
    g.count = int(means.shape[0])
    import numpy as np
    if isinstance(means, np.ndarray):
        arrs = [np.ascontiguousarray(a, np.float32) for a in (means, rotations, scales, opacities, sh)]
        g.on_device = 0
        ptrs = [a.ctypes.data for a in arrs]
        keep = arrs
    else:
        arrs = [a.contiguous().float() for a in (means, rotations, scales, opacities, sh)]
        g.on_device = 1
        ptrs = [a.data_ptr() for a in arrs]
        keep = arrs
    g.means, g.rotations, g.scales, g.opacities, g.sh = ptrs
    h = C.c_void_p()
    _check(lib().gut_scene_create(ctx, C.byref(g), _stream_ptr(stream), C.byref(h)), ctx)
    del keep
    return h


def gut_scene_destroy(ctx, scene):
    lib().gut_scene_destroy(ctx, scene)


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        except Exception:
            pass
        return None
    return C.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)


def gut_render(ctx, scene, cam: gut_camera, opt: gut_options, out: gut_outputs, stream=None, stats=True):
    st = gut_stats() if stats else None
    _check(lib().gut_render(ctx, scene, C.byref(cam), C.byref(opt), C.byref(out), _stream_ptr(stream),
                            C.byref(st) if st is not None else None), ctx)
    return st


def gut_render_backward(ctx, scene, cam: gut_camera, opt: gut_options, rgb, alpha, depth, grad_rgb, grad_alpha,
                        grad_depth, grads: gut_gradients, stream=None):
    """Backward of the last gut_render (device pointers as ints or None)."""
    _check(lib().gut_render_backward(ctx, scene, C.byref(cam), C.byref(opt), rgb, alpha, depth, grad_rgb, grad_alpha,
                                     grad_depth, C.byref(grads), _stream_ptr(stream)), ctx)


QUALITY_FIELDS = ("ut", "ewa", "mc", "kl_ut", "kl_ewa", "valid")


def gut_projection_quality(ctx, scene, cam: gut_camera, opt: gut_options, n_samples: int, seed: int, out_ptr,
                           stream=None):
    """Supp. C: per-Gaussian UT / EWA / Monte-Carlo 2D Gaussians and KL into a
    device buffer of count x 144 bytes (gut_quality records)."""
    _check(lib().gut_projection_quality(ctx, scene, C.byref(cam), C.byref(opt), int(n_samples), int(seed), out_ptr,
                                        _stream_ptr(stream)), ctx)


def gut_render_batch(ctx, scene, cams: Sequence[gut_camera], opt: gut_options, outs: Sequence[gut_outputs],
                     stream=None, stats=False):
    n = len(cams)
    carr = (gut_camera * n)(*cams)
    oarr = (gut_outputs * n)(*outs)
    st = (gut_stats * n)() if stats else None
    _check(lib().gut_render_batch(ctx, scene, carr, n, C.byref(opt), oarr, _stream_ptr(stream), st), ctx)
    return st


def gut_context_set_frames_in_flight(ctx, n: int):
    _check(lib().gut_context_set_frames_in_flight(ctx, int(n)), ctx)


def gut_timing_read(ctx, reset: bool = True):
    """Summed per-stage milliseconds of the timing=1 renders since the last reset."""
    ms = (C.c_double * 7)()
    n = C.c_int32(0)
    _check(lib().gut_timing_read(ctx, ms, C.byref(n), int(reset)), ctx)
    return dict(zip(STAGE_NAMES, list(ms))), int(n.value)


def gut_check(ctx, stream=None):
    """Synchronises `stream`; raises GutError(GUT_E_CAPACITY) if a render since
    the last synchronising call overflowed its reserved key capacity."""
    _check(lib().gut_check(ctx, _stream_ptr(stream)), ctx)


def gut_debug_copy_stage(ctx, stage: int):
    import numpy as np
    need = C.c_size_t(0)
    _check(lib().gut_debug_copy_stage(ctx, stage, None, 0, C.byref(need)), ctx)
    buf = (C.c_ubyte * max(int(need.value), 1))()
    _check(lib().gut_debug_copy_stage(ctx, stage, buf, need.value, C.byref(need)), ctx)
    raw = bytes(buf)[: need.value]
    if stage == STAGE_PROJECT:
        dt = np.dtype([("vx", "<f4"), ("vy", "<f4"), ("cxx", "<f4"), ("cxy", "<f4"), ("cyy", "<f4"), ("k2", "<f4"),
                       ("depth", "<f4"), ("rgb", "<f4", 3), ("tiles", "<u4"), ("rect", "<u2", 4)])
        assert dt.itemsize == C.sizeof(gut_proj_record)
        return np.frombuffer(raw, dt).copy()
    if stage == STAGE_RAYS:  # per tile: float4 [256] ray offsets, then float [4][8] block lattices
        rec = np.frombuffer(raw, np.float32).reshape(-1, 256 * 4 + 32)
        return rec[:, :1024].reshape(-1, 256, 4).copy(), rec[:, 1024:].reshape(-1, 4, 8).copy()
    arr = np.frombuffer(raw, np.uint32).copy()
    if stage in (STAGE_SORTED, STAGE_RANGES, STAGE_TILE_WORK):
        arr = arr.reshape(-1, 2)
    elif stage == STAGE_BLEND_TRACE:
        arr = arr.reshape(-1, 8)
    return arr


# ------------------------------------------------------------- convenience
class Renderer:
    """Context + resident scene.  render() returns torch tensors (device)."""

    def __init__(self, scene, device: int = 0, reserve_keys: Optional[int] = None, max_wh=(1920, 1280)):
        import torch
        self.torch = torch
        self.device = device
        self.ctx = gut_context_create(device)
        if reserve_keys:
            gut_workspace_reserve(self.ctx, reserve_keys, scene.count, max_wh[0], max_wh[1])
        self.scene = gut_scene_create(self.ctx, scene.means, scene.rotations, scene.scales, scene.opacities,
                                      scene.sh, scene.sh_degree)
        self.n, self.nc = scene.count, (scene.sh_degree + 1) ** 2
        torch.cuda.synchronize(device)

    def render(self, cam, opt=None, timing=False, stats=True, out=None):
        torch = self.torch
        H, W = cam.height, cam.width
        if out is None:
            dev = torch.device("cuda", self.device)
            out = (torch.empty((H, W, 3), device=dev), torch.empty((H, W), device=dev),
                   torch.empty((H, W), device=dev))
        o = gut_outputs(out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr() if out[2] is not None else None, 1, 0)
        st = gut_render(self.ctx, self.scene, make_camera(cam), make_options(opt, timing), o, stats=stats)
        return out[0], out[1], out[2], st

    def backward(self, cam, opt, out, grad_rgb, grad_alpha=None, grad_depth=None, sh_shape=None):
        """Gradients (torch tensors on the device) of sum(grad_rgb rgb + grad_alpha
        alpha + grad_depth depth) for the last render(cam, opt) whose outputs
        are `out` = (rgb, alpha, depth)."""
        torch = self.torch
        n = self.n
        dev = torch.device("cuda", self.device)
        g = {k: torch.empty(sz, device=dev) for k, sz in (("means", (n, 3)), ("rotations", (n, 4)), ("scales", (n, 3)),
                                                           ("opacities", (n,)), ("sh", (n, self.nc, 3)),
                                                           ("rgb", (n, 3)), ("densify", (n,)))}
        gg = gut_gradients(*(g[k].data_ptr() for k in ("means", "rotations", "scales", "opacities", "sh", "rgb",
                                                         "densify")))
        p = lambda t: None if t is None else t.contiguous().data_ptr()  # noqa: E731
        gut_render_backward(self.ctx, self.scene, make_camera(cam), make_options(opt), p(out[0]), p(out[1]),
                            p(out[2]) if grad_depth is not None else p(out[2]), p(grad_rgb), p(grad_alpha),
                            p(grad_depth), gg)
        return g

    def projection_quality(self, cam, opt=None, n_samples=500, seed=0):
        """numpy structured array (ut, ewa, mc [5], kl_ut, kl_ewa, valid) per Gaussian."""
        import numpy as np
        torch = self.torch
        buf = torch.empty((self.n, 18), dtype=torch.float64, device=torch.device("cuda", self.device))
        gut_projection_quality(self.ctx, self.scene, make_camera(cam), make_options(opt), n_samples, seed,
                               buf.data_ptr())
        torch.cuda.synchronize(self.device)
        dt = np.dtype([("ut", "<f8", 5), ("ewa", "<f8", 5), ("mc", "<f8", 5), ("kl_ut", "<f8"), ("kl_ewa", "<f8"),
                       ("valid", "<i4"), ("pad", "<i4")])
        return buf.cpu().numpy().view(dt).reshape(-1)

    def stage(self, stage):
        return gut_debug_copy_stage(self.ctx, stage)

    def close(self):
        if self.ctx:
            gut_scene_destroy(self.ctx, self.scene)
            gut_context_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
