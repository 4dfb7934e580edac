"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module is the ONLY code both sides of the parity check consume.  It holds
no arithmetic of the method (no projection, no UT, no binning, no compositing):
it draws Gaussians and camera poses from a fixed recipe and returns plain numpy
arrays / plain-value dataclasses.  The recipe is SURVEY.md §8(d).2 (the paper
fixes only resolutions, camera models and one Gaussian count: PAPER.md L297,
L304, L306, L359, L619).  Every draw uses numpy PCG64(seed) in a fixed order, so
a (config, seed) pair always yields bit-identical inputs.

Conventions:
  * quaternions are (w, x, y, z); scales are activated (> 0); opacities in [0, 1]
  * SH coefficients are [N][(deg+1)^2][3]  (3DGS layout)
  * camera pose = camera->world rotation quaternion + camera centre, at t=0 and
    t=1 (equal for a global shutter); camera axes are OpenCV (x right, y down,
    z forward)
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Tuple

import numpy as np

CAMERA_MODELS = ("pinhole", "opencv", "fisheye", "ortho")
SHUTTERS = ("global", "top_to_bottom", "left_to_right", "bottom_to_top", "right_to_left")

#: (float)(1/255): the alpha_min threshold is DEFINED as this fp32 value on both
#: sides of the parity check; never recompute it in fp64.
ALPHA_MIN_F32 = float(np.float32(1.0 / 255.0))


@dataclasses.dataclass
class Camera:
    model: str
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    k: Tuple[float, ...] = (0.0,) * 6          # OPENCV k1..k6 ; FISHEYE k1..k4
    p: Tuple[float, float] = (0.0, 0.0)        # OPENCV p1, p2
    fov_limit: float = 0.0                     # FISHEYE theta_max [rad]; OPENCV r_lim
    shutter: str = "global"
    q_c2w: Tuple[Tuple[float, ...], Tuple[float, ...]] = ((1.0, 0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0))
    c_w: Tuple[Tuple[float, ...], Tuple[float, ...]] = ((0.0, 0.0, 0.0), (0.0, 0.0, 0.0))

    def __post_init__(self):
        assert self.model in CAMERA_MODELS, self.model
        assert self.shutter in SHUTTERS, self.shutter
        self.k = tuple(float(v) for v in (list(self.k) + [0.0] * 6)[:6])
        self.p = tuple(float(v) for v in self.p)
        self.q_c2w = tuple(tuple(float(v) for v in q) for q in self.q_c2w)
        self.c_w = tuple(tuple(float(v) for v in c) for c in self.c_w)

    @property
    def tiles(self) -> Tuple[int, int]:
        return ((self.width + 15) // 16, (self.height + 15) // 16)


@dataclasses.dataclass
class RenderOptions:
    """Plain values shared by oracle and GPU.  Thresholds are
    the exact fp32 values that cross the ABI."""
    ut_alpha: float = 1.0
    ut_beta: float = 2.0
    ut_kappa: float = 0.0
    alpha_min: float = ALPHA_MIN_F32
    alpha_max: float = float(np.float32(0.99))
    transmittance_min: float = float(np.float32(1e-4))
    cov2d_dilation: float = float(np.float32(0.3))
    near_plane: float = float(np.float32(0.2))
    rs_max_iterations: int = 8
    rs_tolerance_px: float = float(np.float32(1e-4))
    tile_cull: int = 1             # 0 = AABB, 1 = ellipse-tile (StopThePop-style)
    kbuffer: int = 0               # 0 = "Ours" (tile depth order); k >= 1 = "Ours (sorted)" MLAB k-buffer
    kernel_degree: int = 2         # Supp. A generalized Gaussian degree n (2 = Gaussian)
    background: Tuple[float, float, float] = (0.0, 0.0, 0.0)


@dataclasses.dataclass
class Scene:
    means: np.ndarray       # [N,3] f32
    rotations: np.ndarray   # [N,4] f32 (w,x,y,z), not necessarily normalised
    scales: np.ndarray      # [N,3] f32 activated
    opacities: np.ndarray   # [N]   f32 activated
    sh: np.ndarray          # [N,(d+1)^2,3] f32
    sh_degree: int

    @property
    def count(self) -> int:
        return int(self.means.shape[0])

    def subset(self, idx) -> "Scene":
        return Scene(self.means[idx].copy(), self.rotations[idx].copy(), self.scales[idx].copy(),
                     self.opacities[idx].copy(), self.sh[idx].copy(), self.sh_degree)


# ----------------------------------------------------------------------------
# pose helpers (input construction only)
# ----------------------------------------------------------------------------

def _mat_to_quat(R: np.ndarray) -> Tuple[float, float, float, float]:
    """Rotation matrix -> unit quaternion (w,x,y,z) (Shepperd's method)."""
    R = np.asarray(R, dtype=np.float64)
    tr = R[0, 0] + R[1, 1] + R[2, 2]
    if tr > 0:
        s = math.sqrt(tr + 1.0) * 2
        w, x, y, z = 0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s
    elif R[0, 0] > R[1, 1] and R[0, 0] > R[2, 2]:
        s = math.sqrt(1.0 + R[0, 0] - R[1, 1] - R[2, 2]) * 2
        w, x, y, z = (R[2, 1] - R[1, 2]) / s, 0.25 * s, (R[0, 1] + R[1, 0]) / s, (R[0, 2] + R[2, 0]) / s
    elif R[1, 1] > R[2, 2]:
        s = math.sqrt(1.0 + R[1, 1] - R[0, 0] - R[2, 2]) * 2
        w, x, y, z = (R[0, 2] - R[2, 0]) / s, (R[0, 1] + R[1, 0]) / s, 0.25 * s, (R[1, 2] + R[2, 1]) / s
    else:
        s = math.sqrt(1.0 + R[2, 2] - R[0, 0] - R[1, 1]) * 2
        w, x, y, z = (R[1, 0] - R[0, 1]) / s, (R[0, 2] + R[2, 0]) / s, (R[1, 2] + R[2, 1]) / s, 0.25 * s
    q = np.array([w, x, y, z])
    q /= np.linalg.norm(q)
    if q[0] < 0:
        q = -q
    return tuple(float(v) for v in q)


def look_at_c2w(eye, target, up=(0.0, 0.0, 1.0)) -> np.ndarray:
    """Camera->world rotation (columns = camera x,y,z axes in world) for an
    OpenCV camera at `eye` looking at `target` (x right, y down, z forward)."""
    eye = np.asarray(eye, np.float64)
    z = np.asarray(target, np.float64) - eye
    z /= np.linalg.norm(z)
    x = np.cross(z, np.asarray(up, np.float64))
    if np.linalg.norm(x) < 1e-9:
        x = np.cross(z, np.array([0.0, 1.0, 0.0]))
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    return np.stack([x, y, z], axis=1)


def _rot_axis(axis, ang) -> np.ndarray:
    a = np.asarray(axis, np.float64)
    a = a / np.linalg.norm(a)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + math.sin(ang) * K + (1 - math.cos(ang)) * (K @ K)


def make_camera(model, width, height, f, cx, cy, eye, target, up=(0, 0, 1), **kw) -> Camera:
    q = _mat_to_quat(look_at_c2w(eye, target, up))
    return Camera(model=model, width=width, height=height, fx=f, fy=f, cx=cx, cy=cy,
                  q_c2w=(q, q), c_w=(tuple(eye), tuple(eye)), **kw)


# ----------------------------------------------------------------------------
# attribute sampler (SURVEY §8(d).2 "Common attribute sampler")
# ----------------------------------------------------------------------------

def sample_attrs(n: int, rng: np.random.Generator, s_med: float, sh_degree: int):
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    b = s_med * np.exp(rng.normal(0.0, 0.6, n))
    s = np.stack([b, b * rng.uniform(0.4, 1.0, n), b * rng.uniform(0.05, 0.4, n)], axis=1)
    hi = rng.uniform(0.0, 1.0, n) < 0.55
    sig = np.where(hi, rng.uniform(0.85, 0.995, n), rng.uniform(0.02, 0.85, n))
    nc = (sh_degree + 1) ** 2
    sh = np.zeros((n, nc, 3))
    sh[:, 0, :] = rng.uniform(-1.5, 1.5, (n, 3))
    for l in range(1, sh_degree + 1):
        lo, hi_ = l * l, (l + 1) * (l + 1)
        sh[:, lo:hi_, :] = rng.normal(0.0, 0.1 / l, (n, hi_ - lo, 3))
    return q, s, sig, sh


def _pack(means, q, s, sig, sh, deg) -> Scene:
    return Scene(np.ascontiguousarray(means, np.float32), np.ascontiguousarray(q, np.float32),
                 np.ascontiguousarray(s, np.float32), np.ascontiguousarray(sig, np.float32),
                 np.ascontiguousarray(sh, np.float32), deg)


# ----------------------------------------------------------------------------
# tiny scenes (config 0) and the per-code-path variants
# ----------------------------------------------------------------------------

TINY_VARIANTS = ("pinhole", "ortho", "opencv", "fisheye", "rs")


def tiny(seed: int = 0, variant: str = "pinhole", n: int = 64, size: int = 64,
         sh_degree: int = 0) -> Tuple[Scene, Camera]:
    """BASELINE.json configs[0]: 64 random Gaussians, SH deg 0, pinhole 64x64.
    Positions are drawn in the camera frame (camera at the origin, identity
    pose), SURVEY §8(d).2 'tiny' row."""
    assert variant in TINY_VARIANTS
    rng = np.random.Generator(np.random.PCG64(seed))
    if variant == "fisheye":
        # directions on the cap theta <= 100 deg, distance U(2,6)
        u = rng.uniform(math.cos(math.radians(100.0)), 1.0, n)
        ph = rng.uniform(0, 2 * math.pi, n)
        r = rng.uniform(2.0, 6.0, n)
        st = np.sqrt(1 - u * u)
        means = np.stack([r * st * np.cos(ph), r * st * np.sin(ph), r * u], 1)
    else:
        means = np.stack([rng.uniform(-1.2, 1.2, n), rng.uniform(-1.2, 1.2, n),
                          rng.uniform(2.0, 6.0, n)], 1)
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    s = np.exp(rng.uniform(math.log(0.03), math.log(0.3), (n, 3)))
    sig = rng.uniform(0.05, 0.99, n)
    nc = (sh_degree + 1) ** 2
    sh = np.zeros((n, nc, 3))
    sh[:, 0, :] = rng.uniform(-1.5, 1.5, (n, 3))
    for l in range(1, sh_degree + 1):
        lo, hi_ = l * l, (l + 1) * (l + 1)
        sh[:, lo:hi_, :] = rng.normal(0.0, 0.1 / l, (n, hi_ - lo, 3))
    scene = _pack(means, q, s, sig, sh, sh_degree)
    ident = ((1.0, 0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0))
    zero = ((0.0, 0.0, 0.0), (0.0, 0.0, 0.0))
    h = size / 2.0
    if variant == "pinhole":
        cam = Camera("pinhole", size, size, size, size, h, h, q_c2w=ident, c_w=zero)
    elif variant == "ortho":
        cam = Camera("ortho", size, size, size / 2.0, size / 2.0, h, h, q_c2w=ident, c_w=zero)
    elif variant == "opencv":
        cam = Camera("opencv", size, size, size, size, h, h, k=(-0.2, 0.05, 0, 0, 0, 0),
                     p=(1e-3, -1e-3), fov_limit=1.0, q_c2w=ident, c_w=zero)
    elif variant == "fisheye":
        cam = Camera("fisheye", size, size, size * 20.0 / 64.0, size * 20.0 / 64.0, h, h,
                     fov_limit=math.radians(110.0), q_c2w=ident, c_w=zero)
    else:  # rolling shutter pinhole: 0.35 translation along x, 2 deg yaw (Supp. C)
        q1 = _mat_to_quat(_rot_axis((0, 1, 0), math.radians(2.0)))
        cam = Camera("pinhole", size, size, size, size, h, h, shutter="top_to_bottom",
                     q_c2w=((1.0, 0.0, 0.0, 0.0), q1), c_w=((0.0, 0.0, 0.0), (0.35, 0.0, 0.0)))
    return scene, cam


# ----------------------------------------------------------------------------
# large configs (BASELINE.json configs[1..4])
# ----------------------------------------------------------------------------

def _garden_positions(n: int, rng: np.random.Generator):
    """'unbounded garden', z-up: 40% on 6 ellipsoid surfaces, 30% ground disk,
    30% background shell.  Returns positions and a per-point scale multiplier."""
    n_obj = int(round(0.4 * n))
    n_gnd = int(round(0.3 * n))
    n_bg = n - n_obj - n_gnd
    centres = rng.uniform(-0.6, 0.6, (6, 3)) * np.array([1.0, 1.0, 0.5]) + np.array([0, 0, 0.4])
    radii = rng.uniform(0.2, 0.8, (6, 3))
    which = rng.integers(0, 6, n_obj)
    d = rng.standard_normal((n_obj, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    p_obj = centres[which] + d * radii[which] * (1.0 + rng.normal(0, 0.01, (n_obj, 1)))
    # ground disk r<=6, density ~ 1/(1+r): inverse CDF of p(r) ~ r/(1+r) on [0,6]
    # (sampled by rejection to keep the recipe obvious)
    rs = np.empty(0)
    while rs.size < n_gnd:
        cand = rng.uniform(0, 6, 2 * n_gnd)
        keep = rng.uniform(0, 1, 2 * n_gnd) < (1.0 / (1.0 + cand))
        rs = np.concatenate([rs, cand[keep]])
    rs = rs[:n_gnd]
    ph = rng.uniform(0, 2 * math.pi, n_gnd)
    p_gnd = np.stack([rs * np.cos(ph), rs * np.sin(ph), np.zeros(n_gnd)], 1)
    rb = rng.uniform(8.0, 30.0, n_bg)
    d = rng.standard_normal((n_bg, 3))
    d[:, 2] = np.abs(d[:, 2])
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    p_bg = d * rb[:, None]
    pos = np.concatenate([p_obj, p_gnd, p_bg])
    mult = np.concatenate([np.ones(n_obj + n_gnd), rb / 4.0])
    return pos, mult


def _room_positions(n: int, rng: np.random.Generator):
    """ScanNet++-shaped: 7x5x2.8 m room, 65% on the 6 faces, 35% on 12 boxes."""
    L, Wd, H = 7.0, 5.0, 2.8
    n_face = int(round(0.65 * n))
    n_box = n - n_face
    areas = np.array([L * Wd, L * Wd, L * H, L * H, Wd * H, Wd * H])
    f = rng.choice(6, n_face, p=areas / areas.sum())
    u, v = rng.uniform(0, 1, n_face), rng.uniform(0, 1, n_face)
    p = np.zeros((n_face, 3))
    p[f == 0] = np.stack([u * L, v * Wd, np.zeros(n_face)], 1)[f == 0]
    p[f == 1] = np.stack([u * L, v * Wd, np.full(n_face, H)], 1)[f == 1]
    p[f == 2] = np.stack([u * L, np.zeros(n_face), v * H], 1)[f == 2]
    p[f == 3] = np.stack([u * L, np.full(n_face, Wd), v * H], 1)[f == 3]
    p[f == 4] = np.stack([np.zeros(n_face), u * Wd, v * H], 1)[f == 4]
    p[f == 5] = np.stack([np.full(n_face, L), u * Wd, v * H], 1)[f == 5]
    bmin = np.stack([rng.uniform(0.2, L - 1.7, 12), rng.uniform(0.2, Wd - 1.7, 12), np.zeros(12)], 1)
    bsz = rng.uniform(0.3, 1.5, (12, 3))
    which = rng.integers(0, 12, n_box)
    uvw = rng.uniform(0, 1, (n_box, 3))
    face_axis = rng.integers(0, 3, n_box)
    side = rng.integers(0, 2, n_box).astype(np.float64)
    uvw[np.arange(n_box), face_axis] = side
    pb = bmin[which] + uvw * bsz[which]
    return np.concatenate([p, pb]), np.ones(n)


def _street_positions(n: int, rng: np.random.Generator):
    """Waymo-shaped street corridor along +x."""
    n_road = int(round(0.30 * n)); n_fac = int(round(0.35 * n))
    n_cl = int(round(0.20 * n)); n_car = int(round(0.10 * n))
    n_sky = n - n_road - n_fac - n_cl - n_car
    road = np.stack([rng.uniform(-100, 100, n_road), rng.uniform(-8, 8, n_road), np.zeros(n_road)], 1)
    side = np.where(rng.uniform(0, 1, n_fac) < 0.5, -12.0, 12.0)
    hgt = rng.uniform(6, 20, n_fac)
    fac = np.stack([rng.uniform(-100, 100, n_fac), side, rng.uniform(0, 1, n_fac) * hgt], 1)
    cc = np.stack([rng.uniform(-100, 100, 64), np.where(rng.uniform(0, 1, 64) < 0.5, -10.0, 10.0),
                   rng.uniform(0.3, 2.0, 64)], 1)
    cl = cc[rng.integers(0, 64, n_cl)] + rng.normal(0, 0.6, (n_cl, 3))
    cars = np.stack([rng.uniform(-90, 90, 40), rng.choice([-5.0, -2.0, 2.0, 5.0], 40), np.zeros(40)], 1)
    csz = np.array([4.5, 1.8, 1.5])
    which = rng.integers(0, 40, n_car)
    uvw = rng.uniform(0, 1, (n_car, 3))
    ax = rng.integers(0, 3, n_car)
    uvw[np.arange(n_car), ax] = rng.integers(0, 2, n_car)
    car = cars[which] + (uvw - np.array([0.5, 0.5, 0.0])) * csz
    d = rng.standard_normal((n_sky, 3))
    d[:, 2] = np.abs(d[:, 2])
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    sky = d * 150.0
    pos = np.concatenate([road, fac, cl, car, sky])
    mult = np.concatenate([np.ones(n - n_sky), np.full(n_sky, 20.0)])
    return pos, mult


CONFIGS = {
    # name: (N, sh_degree, s_med, scene seed, view seed, structure)
    "tiny": (64, 0, None, 0, None, "tiny"),
    "mipnerf360": (1_000_000, 3, 0.012, 360, 361, "garden"),
    "scannetpp": (500_000, 3, 0.015, 2023, 2024, "room"),
    "waymo": (2_000_000, 3, 0.05, 2020, 2021, "street"),
    "multiview": (3_000_000, 3, 0.007, 12507, 12508, "garden"),
}


def make_scene(config: str, n: int = None) -> Scene:
    """The synthetic scene of a BASELINE.json config (optionally with a smaller
    N for parity tests; the recipe is otherwise unchanged)."""
    N, deg, s_med, seed, _, structure = CONFIGS[config]
    if config == "tiny":
        return tiny(seed)[0]
    n = N if n is None else int(n)
    rng = np.random.Generator(np.random.PCG64(seed))
    if structure == "garden":
        pos, mult = _garden_positions(n, rng)
    elif structure == "room":
        pos, mult = _room_positions(n, rng)
    else:
        pos, mult = _street_positions(n, rng)
    q, s, sig, sh = sample_attrs(n, rng, s_med, deg)
    s = s * mult[:, None]
    return _pack(pos, q, s, sig, sh, deg)


def make_views(config: str, count: int = None) -> List[Camera]:
    """The camera set of a BASELINE.json config."""
    _, _, _, _, vseed, _ = CONFIGS[config]
    rng = np.random.Generator(np.random.PCG64(vseed))
    cams: List[Camera] = []
    if config == "mipnerf360":
        nv = 16 if count is None else count
        for i in range(nv):
            a = 2 * math.pi * i / 16.0
            eye = (4.0 * math.cos(a), 4.0 * math.sin(a), 1.3)
            cams.append(make_camera("pinhole", 1297, 840, 1150.0, 648.5, 420.0, eye, (0, 0, 0.3)))
    elif config == "scannetpp":
        nv = 16 if count is None else count
        for i in range(nv):
            eye = np.array([rng.uniform(0.8, 7.0 - 0.8), rng.uniform(0.8, 5.0 - 0.8), 1.4])
            yaw = rng.uniform(0, 2 * math.pi)
            pitch = math.radians(rng.uniform(-20.0, 10.0))
            fwd = np.array([math.cos(yaw) * math.cos(pitch), math.sin(yaw) * math.cos(pitch), math.sin(pitch)])
            cams.append(make_camera("fisheye", 1752, 1168, 790.0, 876.0, 584.0, eye, eye + fwd,
                                    fov_limit=math.radians(85.0)))
    elif config == "waymo":
        nf = 16 if count is None else count
        readout, speed, yaw_rate = 0.033, 10.0, 0.1
        for i in range(nf):
            x0 = -40.0 + 5.0 * i
            for yaw_deg in (0.0, 45.0, -45.0):
                yaw = math.radians(yaw_deg)
                fwd = np.array([math.cos(yaw), math.sin(yaw), 0.0])
                e0 = np.array([x0, 0.0, 2.0])
                R0 = look_at_c2w(e0, e0 + fwd)
                # ego motion during the readout: translation along the heading (+x), yaw about world z
                e1 = e0 + np.array([speed * readout, 0.0, 0.0])
                R1 = _rot_axis((0, 0, 1), yaw_rate * readout) @ R0
                cams.append(Camera("opencv", 1920, 1280, 2060.0, 2060.0, 960.0, 640.0,
                                   k=(-0.12, 0.03, 0, 0, 0, 0), p=(5e-4, -3e-4), fov_limit=0.9,
                                   shutter="top_to_bottom",
                                   q_c2w=(_mat_to_quat(R0), _mat_to_quat(R1)),
                                   c_w=(tuple(e0), tuple(e1))))
    elif config == "multiview":
        nv = 256 if count is None else count
        golden = (math.sqrt(5.0) - 1.0) / 2.0
        for i in range(nv):
            r = rng.uniform(3.5, 5.0)
            el = math.radians(rng.uniform(-5.0, 40.0))
            az = 2 * math.pi * ((i * golden) % 1.0)
            c = np.array([0.0, 0.0, 0.5])
            eye = c + r * np.array([math.cos(el) * math.cos(az), math.cos(el) * math.sin(az), math.sin(el)])
            cams.append(make_camera("fisheye", 1920, 1080, 620.0, 960.0, 540.0, eye, (0.0, 0.0, 0.0),
                                    fov_limit=math.radians(105.0)))
    elif config == "tiny":
        cams.append(tiny(0)[1])
    else:
        raise KeyError(config)
    return cams


def scaled_camera(cam: Camera, factor: float) -> Camera:
    """Same pose and model at a reduced resolution (parity cases the oracle
    finishes in seconds).  Intrinsics scale with the image."""
    w = max(16, int(round(cam.width * factor)))
    h = max(16, int(round(cam.height * factor)))
    sx, sy = w / cam.width, h / cam.height
    return dataclasses.replace(cam, width=w, height=h, fx=cam.fx * sx, fy=cam.fy * sy,
                               cx=cam.cx * sx, cy=cam.cy * sy)
