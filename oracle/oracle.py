"""ctypes wrapper of the fp64 C oracle (oracle/gut_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py — never by the product package
paper_2412_12507_b200/.  It shares no code with the CUDA path; both consume the
seeded inputs of scenegen/ only.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "gut_oracle.c")]

MODELS = {"pinhole": 0, "opencv": 1, "fisheye": 2, "ortho": 3}
SHUTTERS = {"global": 0, "top_to_bottom": 1, "left_to_right": 2, "bottom_to_top": 3, "right_to_left": 4}
REASONS = {0: "ok", 1: "param", 2: "opacity", 3: "sigma", 4: "cov", 5: "offscreen", 6: "notile"}


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc (-O2, no fast-math, no FP contraction
    so the fp64 results are reproducible), OpenMP over Gaussians / tiles."""
    hdr = os.path.join(_HERE, "gut_oracle.h")
    if not force and os.path.exists(_LIB_PATH):
        newest = max(os.path.getmtime(p) for p in _SRC + [hdr])
        if os.path.getmtime(_LIB_PATH) >= newest:
            return _LIB_PATH
    cmd = ["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-fno-fast-math", "-ffp-contract=off",
           "-fopenmp", "-fPIC", "-shared", "-o", _LIB_PATH] + _SRC + ["-lm"]
    subprocess.check_call(cmd)
    return _LIB_PATH


class OrcCamera(C.Structure):
    _fields_ = [("model", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("shutter", C.c_int32), ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double),
                ("cy", C.c_double), ("k", C.c_double * 6), ("p", C.c_double * 2),
                ("fov_limit", C.c_double), ("q", (C.c_double * 4) * 2), ("c", (C.c_double * 3) * 2)]


class OrcOptions(C.Structure):
    _fields_ = [("ut_alpha", C.c_double), ("ut_beta", C.c_double), ("ut_kappa", C.c_double),
                ("alpha_min", C.c_double), ("alpha_max", C.c_double), ("t_min", C.c_double),
                ("dilation", C.c_double), ("near_plane", C.c_double), ("bg", C.c_double * 3),
                ("tile_cull", C.c_int32), ("kbuffer", C.c_int32),
                ("kernel_degree", C.c_int32), ("pad", C.c_int32)]


class OrcProj(C.Structure):
    _fields_ = [("reason", C.c_int32), ("tiles", C.c_int32), ("rect", C.c_int32 * 4),
                ("cull_ambig", C.c_int32), ("bin_ambig", C.c_int32), ("rs_iters", C.c_int32),
                ("rs_fail", C.c_int32), ("vx", C.c_double), ("vy", C.c_double), ("cxx", C.c_double),
                ("cxy", C.c_double), ("cyy", C.c_double), ("k2", C.c_double), ("hx", C.c_double),
                ("hy", C.c_double), ("depth", C.c_double), ("t0", C.c_double), ("rgb", C.c_double * 3)]


class OrcPixDiag(C.Structure):
    _fields_ = [("visited", C.c_int32), ("contributed", C.c_int32), ("terminated", C.c_int32),
                ("invalid", C.c_int32), ("min_alpha_gap", C.c_double), ("min_term_gap", C.c_double),
                ("min_order_gap", C.c_double), ("amb_bin", C.c_int32), ("amb_cull", C.c_int32),
                ("min_tau_gap", C.c_double), ("alt_valid", C.c_int32), ("alt_pad", C.c_int32),
                ("alt_rgb", C.c_double * 3), ("alt_alpha", C.c_double), ("alt_depth", C.c_double)]


PROJ_DTYPE = np.dtype([("reason", "<i4"), ("tiles", "<i4"), ("rect", "<i4", 4), ("cull_ambig", "<i4"),
                       ("bin_ambig", "<i4"), ("rs_iters", "<i4"), ("rs_fail", "<i4"), ("vx", "<f8"),
                       ("vy", "<f8"), ("cxx", "<f8"), ("cxy", "<f8"), ("cyy", "<f8"), ("k2", "<f8"),
                       ("hx", "<f8"), ("hy", "<f8"), ("depth", "<f8"), ("t0", "<f8"), ("rgb", "<f8", 3)])
DIAG_DTYPE = np.dtype([("visited", "<i4"), ("contributed", "<i4"), ("terminated", "<i4"),
                       ("invalid", "<i4"), ("min_alpha_gap", "<f8"), ("min_term_gap", "<f8"),
                       ("min_order_gap", "<f8"), ("amb_bin", "<i4"), ("amb_cull", "<i4"),
                       ("min_tau_gap", "<f8"), ("alt_valid", "<i4"), ("alt_pad", "<i4"),
                       ("alt_rgb", "<f8", 3), ("alt_alpha", "<f8"), ("alt_depth", "<f8")])
assert PROJ_DTYPE.itemsize == C.sizeof(OrcProj)
assert DIAG_DTYPE.itemsize == C.sizeof(OrcPixDiag)

_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        dp, ip, fp = C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_float)
        L.orc_ut_weights.argtypes = [C.c_double, C.c_double, C.c_double, dp, dp, dp]
        L.orc_quat_to_rot.argtypes = [dp, dp]
        L.orc_sigma_points.argtypes = [dp, dp, dp, C.c_double, dp]
        L.orc_pose_at.argtypes = [C.POINTER(OrcCamera), C.c_double, dp, dp]
        L.orc_project_cam.argtypes = [C.POINTER(OrcCamera), C.POINTER(OrcOptions), dp, dp, dp]
        L.orc_project_point.argtypes = [C.POINTER(OrcCamera), C.POINTER(OrcOptions), dp, dp, dp, ip, dp]
        L.orc_sh_basis.argtypes = [dp, dp]
        L.orc_tile_hits_ellipse.argtypes = [C.c_double] * 10
        L.orc_preprocess.argtypes = [fp, fp, fp, fp, fp, C.c_int32, C.c_int64, C.POINTER(OrcCamera),
                                     C.POINTER(OrcOptions), C.c_void_p]
        L.orc_tile_lists.argtypes = [C.c_void_p, C.c_int64, C.POINTER(OrcCamera), C.POINTER(OrcOptions),
                                     fp, fp, ip, ip, C.c_int64, ip]
        L.orc_tile_lists.restype = C.c_int64
        L.orc_pixel_ray.argtypes = [C.POINTER(OrcCamera), C.c_double, C.c_double, dp, dp]
        L.orc_max_response.argtypes = [dp, dp, dp, dp, dp, dp]
        L.orc_max_response.restype = C.c_double
        L.orc_composite.argtypes = [fp, fp, fp, fp, C.c_void_p, ip, ip, C.POINTER(OrcCamera),
                                    C.POINTER(OrcOptions), ip, C.c_int32, fp, fp, fp, C.c_void_p]
        L.orc_render.argtypes = [fp, fp, fp, fp, fp, C.c_int32, C.c_int64, C.POINTER(OrcCamera),
                                 C.POINTER(OrcOptions), C.c_int32, ip, C.c_int32, fp, fp, fp,
                                 C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
        L.orc_render.restype = C.c_int64
        L.orc_mark_ambiguity.argtypes = [fp, fp, fp, fp, C.c_void_p, C.c_int64, C.POINTER(OrcCamera),
                                         C.POINTER(OrcOptions), C.c_double, ip, C.c_int32, C.c_void_p]
        L.orc_threads.restype = C.c_int
        L.orc_kbuffer_blend.argtypes = [dp, dp, dp, C.c_int32, C.c_int32, C.c_double, dp, dp, dp, ip, dp]
        L.orc_kbuffer_blend.restype = C.c_int32
        L.orc_set_alt_band.argtypes = [C.c_double]
        L.orc_set_alt_band.restype = None
        L.orc_backward.argtypes = [fp, fp, fp, fp, fp, C.c_int32, C.c_int64, C.POINTER(OrcCamera),
                                   C.POINTER(OrcOptions), fp, fp, fp, dp, dp, dp, dp, dp, dp, dp]
        L.orc_backward.restype = C.c_int64
        L.orc_normal3.argtypes = [C.c_uint64, C.c_int64, C.c_int32, dp]
        L.orc_kl2.argtypes = [dp, dp]
        L.orc_kl2.restype = C.c_double
        L.orc_projection_quality.argtypes = [fp, fp, fp, C.c_int64, C.POINTER(OrcCamera), C.POINTER(OrcOptions),
                                             C.c_int32, C.c_uint64, C.c_void_p]
        L.orc_kernel_lambda.argtypes = [C.c_int32]
        L.orc_kernel_lambda.restype = C.c_double
        L.orc_kernel_response.argtypes = [C.c_double, C.c_int32]
        L.orc_kernel_response.restype = C.c_double
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def camera(cam) -> OrcCamera:
    c = OrcCamera()
    c.model = MODELS[cam.model]
    c.width, c.height = int(cam.width), int(cam.height)
    c.shutter = SHUTTERS[cam.shutter]
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    for i in range(6):
        c.k[i] = cam.k[i]
    c.p[0], c.p[1] = cam.p
    c.fov_limit = cam.fov_limit
    for t in range(2):
        for i in range(4):
            c.q[t][i] = cam.q_c2w[t][i]
        for i in range(3):
            c.c[t][i] = cam.c_w[t][i]
    return c


def options(opt) -> OrcOptions:
    o = OrcOptions()
    o.ut_alpha, o.ut_beta, o.ut_kappa = opt.ut_alpha, opt.ut_beta, opt.ut_kappa
    o.alpha_min, o.alpha_max, o.t_min = opt.alpha_min, opt.alpha_max, opt.transmittance_min
    o.dilation, o.near_plane = opt.cov2d_dilation, opt.near_plane
    for i in range(3):
        o.bg[i] = opt.background[i]
    o.tile_cull = int(opt.tile_cull)
    o.kbuffer = int(getattr(opt, "kbuffer", 0))
    o.kernel_degree = int(getattr(opt, "kernel_degree", 2))
    return o


# ---------------------------------------------------------------- O1
def ut_weights(a=1.0, b=2.0, k=0.0):
    wm, ws, lam = np.zeros(7), np.zeros(7), np.zeros(1)
    rc = lib().orc_ut_weights(a, b, k, _dp(wm), _dp(ws), _dp(lam))
    if rc != 0:
        raise ValueError("3 + lambda <= 0")
    return wm, ws, float(lam[0])


def quat_to_rot(q):
    q = np.ascontiguousarray(q, np.float64)
    R = np.zeros(9)
    if lib().orc_quat_to_rot(_dp(q), _dp(R)) != 0:
        raise ValueError("zero quaternion")
    return R.reshape(3, 3)


def sigma_points(mu, R, s, lam):
    mu = np.ascontiguousarray(mu, np.float64)
    R = np.ascontiguousarray(R, np.float64).reshape(9)
    s = np.ascontiguousarray(s, np.float64)
    X = np.zeros((7, 3))
    lib().orc_sigma_points(_dp(mu), _dp(R), _dp(s), float(lam), _dp(X))
    return X


# ---------------------------------------------------------------- O2
def pose_at(cam, t):
    R, c = np.zeros(9), np.zeros(3)
    oc = camera(cam)
    lib().orc_pose_at(C.byref(oc), float(t), _dp(R), _dp(c))
    return R.reshape(3, 3), c


def project_cam(cam, opt, xc):
    xc = np.ascontiguousarray(xc, np.float64)
    uv, m = np.zeros(2), np.zeros(1)
    oc, oo = camera(cam), options(opt)
    v = lib().orc_project_cam(C.byref(oc), C.byref(oo), _dp(xc), _dp(uv), _dp(m))
    return bool(v), uv, float(m[0])


def project_point(cam, opt, x):
    x = np.ascontiguousarray(x, np.float64)
    uv, t, m = np.zeros(2), np.zeros(1), np.zeros(1)
    it = np.zeros(1, np.int32)
    oc, oo = camera(cam), options(opt)
    v = lib().orc_project_point(C.byref(oc), C.byref(oo), _dp(x), _dp(uv), _dp(t), _ip(it), _dp(m))
    return bool(v), uv, float(t[0]), int(it[0])


# ---------------------------------------------------------------- O3
def sh_basis(d):
    d = np.ascontiguousarray(d, np.float64)
    Y = np.zeros(16)
    lib().orc_sh_basis(_dp(d), _dp(Y))
    return Y


def tile_hits_ellipse(vx, vy, cxx, cxy, cyy, k2, x0, y0, x1, y1):
    return bool(lib().orc_tile_hits_ellipse(vx, vy, cxx, cxy, cyy, k2, x0, y0, x1, y1))


def _scene_arrays(scene):
    m = np.ascontiguousarray(scene.means, np.float32)
    r = np.ascontiguousarray(scene.rotations, np.float32)
    s = np.ascontiguousarray(scene.scales, np.float32)
    o = np.ascontiguousarray(scene.opacities, np.float32)
    sh = np.ascontiguousarray(scene.sh, np.float32)
    return m, r, s, o, sh


def preprocess(scene, cam, opt):
    m, r, s, o, sh = _scene_arrays(scene)
    out = np.zeros(scene.count, PROJ_DTYPE)
    oc, oo = camera(cam), options(opt)
    lib().orc_preprocess(_fp(m), _fp(r), _fp(s), _fp(o), _fp(sh), scene.sh_degree, scene.count,
                         C.byref(oc), C.byref(oo), out.ctypes.data)
    return out


# ---------------------------------------------------------------- O4
def tile_lists(proj, cam, opt):
    oc, oo = camera(cam), options(opt)
    proj = np.ascontiguousarray(proj)
    n = proj.shape[0]
    K = lib().orc_tile_lists(proj.ctypes.data, n, C.byref(oc), C.byref(oo), None, None, None, None, 0, None)
    tx, ty = cam.tiles
    tiles = np.zeros(max(K, 1), np.int32)
    gids = np.zeros(max(K, 1), np.int32)
    ranges = np.zeros((tx * ty, 2), np.int32)
    lib().orc_tile_lists(proj.ctypes.data, n, C.byref(oc), C.byref(oo), None, None, _ip(tiles), _ip(gids),
                         K, _ip(ranges))
    return tiles[:K], gids[:K], ranges


# ---------------------------------------------------------------- O5 / O6
def pixel_ray(cam, u, v):
    o, d = np.zeros(3), np.zeros(3)
    oc = camera(cam)
    valid = lib().orc_pixel_ray(C.byref(oc), float(u), float(v), _dp(o), _dp(d))
    return bool(valid), o, d


def max_response(mu, R, s, o, d):
    mu, o, d = (np.ascontiguousarray(a, np.float64) for a in (mu, o, d))
    R = np.ascontiguousarray(R, np.float64).reshape(9)
    s = np.ascontiguousarray(s, np.float64)
    tau = np.zeros(1)
    w2 = lib().orc_max_response(_dp(mu), _dp(R), _dp(s), _dp(o), _dp(d), _dp(tau))
    return float(w2), float(tau[0])


def kernel_response(d2, n):
    """Supp. A generalized Gaussian response at Mahalanobis^2 distance d2."""
    return float(lib().orc_kernel_response(float(d2), int(n)))


def kernel_lambda(n):
    return float(lib().orc_kernel_lambda(int(n)))


def kbuffer_blend(tau, alpha, rgb, k, t_min):
    """O6' on one hit stream: returns (C[3], T, D, n_blended,
    n_consumed).  k >= 1 MLAB k-buffer, -1 exact tau sort, 0 stream order."""
    tau = np.ascontiguousarray(tau, np.float64)
    alpha = np.ascontiguousarray(alpha, np.float64)
    rgb = np.ascontiguousarray(rgb, np.float64).reshape(-1)
    n = tau.size
    Cc, T, D, tg = np.zeros(3), np.zeros(1), np.zeros(1), np.full(1, 1e300)
    nb = C.c_int32(0)
    used = lib().orc_kbuffer_blend(_dp(tau), _dp(alpha), _dp(rgb), n, int(k), float(t_min), _dp(Cc), _dp(T),
                                   _dp(D), C.byref(nb), _dp(tg))
    return Cc, float(T[0]), float(D[0]), int(nb.value), int(used)


def composite(scene, proj, gids, ranges, cam, opt, tile_subset=None):
    """O6 over externally supplied sorted lists (e.g. the GPU's own lists)."""
    m, r, s, o, _ = _scene_arrays(scene)
    H, W = cam.height, cam.width
    rgb = np.zeros((H, W, 3), np.float32)
    alpha = np.zeros((H, W), np.float32)
    depth = np.zeros((H, W), np.float32)
    diag = np.zeros(H * W, DIAG_DTYPE)
    gids = np.ascontiguousarray(gids, np.int32)
    if gids.size == 0:
        gids = np.zeros(1, np.int32)
    ranges = np.ascontiguousarray(ranges, np.int32)
    sub = None if tile_subset is None else np.ascontiguousarray(tile_subset, np.int32)
    oc, oo = camera(cam), options(opt)
    lib().orc_composite(_fp(m), _fp(r), _fp(s), _fp(o), np.ascontiguousarray(proj).ctypes.data, _ip(gids),
                        _ip(ranges), C.byref(oc), C.byref(oo), None if sub is None else _ip(sub),
                        0 if sub is None else sub.size, _fp(rgb), _fp(alpha), _fp(depth), diag.ctypes.data)
    return rgb, alpha, depth, diag.reshape(H, W)


def render(scene, cam, opt, brute=False, tile_subset=None, ambiguity=True, alpha_eps=1e-5):
    """Full oracle render (O1..O6).  Returns dict with rgb [H,W,3], alpha, depth,
    per-pixel diagnostics, per-Gaussian projection records and K."""
    m, r, s, o, sh = _scene_arrays(scene)
    H, W = cam.height, cam.width
    rgb = np.zeros((H, W, 3), np.float32)
    alpha = np.zeros((H, W), np.float32)
    depth = np.zeros((H, W), np.float32)
    diag = np.zeros(H * W, DIAG_DTYPE)
    proj = np.zeros(scene.count, PROJ_DTYPE)
    sub = None if tile_subset is None else np.ascontiguousarray(tile_subset, np.int32)
    K = C.c_int64(0)
    oc, oo = camera(cam), options(opt)
    lib().orc_render(_fp(m), _fp(r), _fp(s), _fp(o), _fp(sh), scene.sh_degree, scene.count, C.byref(oc),
                     C.byref(oo), int(brute), None if sub is None else _ip(sub),
                     0 if sub is None else sub.size, _fp(rgb), _fp(alpha), _fp(depth), diag.ctypes.data,
                     proj.ctypes.data, C.byref(K))
    if ambiguity:
        lib().orc_mark_ambiguity(_fp(m), _fp(r), _fp(s), _fp(o), proj.ctypes.data, scene.count, C.byref(oc),
                                 C.byref(oo), float(alpha_eps), None if sub is None else _ip(sub),
                                 0 if sub is None else sub.size, diag.ctypes.data)
    return dict(rgb=rgb, alpha=alpha, depth=depth, diag=diag.reshape(H, W), proj=proj, n_keys=int(K.value))


def backward(scene, cam, opt, g_rgb, g_alpha, g_depth):
    """O7: gradients of L = sum(g_rgb rgb + g_alpha alpha + g_depth depth) with
    respect to the scene parameters (fp64 dict)."""
    m, r, s, o, sh = _scene_arrays(scene)
    n, nc = scene.count, (scene.sh_degree + 1) ** 2
    out = {k: np.zeros(sz) for k, sz in (("means", (n, 3)), ("rotations", (n, 4)), ("scales", (n, 3)),
                                          ("opacities", (n,)), ("sh", (n, nc, 3)), ("rgb", (n, 3)))}
    gr = np.ascontiguousarray(g_rgb, np.float32)
    ga = np.ascontiguousarray(g_alpha, np.float32)
    gd = np.ascontiguousarray(g_depth, np.float32)
    oc, oo = camera(cam), options(opt)
    loss = np.zeros(1)
    lib().orc_backward(_fp(m), _fp(r), _fp(s), _fp(o), _fp(sh), scene.sh_degree, n, C.byref(oc), C.byref(oo),
                       _fp(gr), _fp(ga), _fp(gd), _dp(out["means"]), _dp(out["rotations"]), _dp(out["scales"]),
                       _dp(out["opacities"]), _dp(out["sh"]), _dp(out["rgb"]), _dp(loss))
    out["loss"] = float(loss[0])
    return out


QUALITY_DTYPE = np.dtype([("ut", "<f8", 5), ("ewa", "<f8", 5), ("mc", "<f8", 5), ("kl_ut", "<f8"),
                          ("kl_ewa", "<f8"), ("valid", "<i4"), ("pad", "<i4")])


def normal3(seed, gid, s):
    z = np.zeros(3)
    lib().orc_normal3(int(seed), int(gid), int(s), _dp(z))
    return z


def kl2(g0, g1):
    return float(lib().orc_kl2(_dp(np.ascontiguousarray(g0, np.float64)), _dp(np.ascontiguousarray(g1, np.float64))))


def projection_quality(scene, cam, opt, n_mc=500, seed=0):
    """O8 (Supp. C): per Gaussian UT / EWA / Monte-Carlo 2D Gaussians and KL."""
    m, r, s, _, _ = _scene_arrays(scene)
    out = np.zeros(scene.count, QUALITY_DTYPE)
    oc, oo = camera(cam), options(opt)
    lib().orc_projection_quality(_fp(m), _fp(r), _fp(s), scene.count, C.byref(oc), C.byref(oo), int(n_mc), int(seed),
                                 out.ctypes.data)
    return out


def threads() -> int:
    return int(lib().orc_threads())
