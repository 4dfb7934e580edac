"""torch.autograd binding of the C ABI: forward = gut_render, backward =
gut_render_backward (PAPER Supp. B; reading R30).  Argument marshalling only:
the render and its gradients run in libgut's kernels; PyTorch supplies the
device memory and the autograd graph around them (activations, losses,
optimisers are the caller's).

    r = RenderFunction.context(device=0)
    rgb, alpha, depth = render(r, means, rotations, scales, opacities, sh, sh_degree, cam, opt)
    loss = (rgb - target).abs().mean(); loss.backward()     # grads on the five tensors
"""
from __future__ import annotations

import torch

from . import gut


class _Ctx:
    """A libgut context reused across steps (the scene is re-packed per call).

    gut_render_backward differentiates the context's LAST render (its lists and
    workspace), so each backward must belong to the most recent forward on
    this context: `seq` counts forwards and backward() checks it (render
    several views before one backward with one _Ctx per outstanding view)."""

    def __init__(self, device: int = 0):
        self.device = device
        self.ctx = gut.gut_context_create(device)
        self.scene = None
        self.seq = 0

    def close(self):
        if self.ctx:
            if self.scene:
                gut.gut_scene_destroy(self.ctx, self.scene)
            gut.gut_context_destroy(self.ctx)
            self.ctx = None


class RenderFunction(torch.autograd.Function):
    @staticmethod
    def context(device: int = 0) -> _Ctx:
        return _Ctx(device)

    @staticmethod
    def forward(ctx, gctx: _Ctx, cam, opt, sh_degree: int, means, rotations, scales, opacities, sh):
        # progressive SH (the 3DGS schedule): sh may store more coefficients than
        # the active degree uses; only the first (d+1)^2 are packed and get gradients
        nc = (sh_degree + 1) ** 2
        if sh.dim() != 3 or sh.shape[2] != 3 or sh.shape[1] < nc:
            raise ValueError(f"sh must be [N, >= {nc}, 3] for sh_degree {sh_degree}, got {tuple(sh.shape)}")
        if gctx.scene:
            gut.gut_scene_destroy(gctx.ctx, gctx.scene)
        gctx.scene = gut.gut_scene_create(gctx.ctx, means.detach(), rotations.detach(), scales.detach(),
                                          opacities.detach(), sh.detach()[:, :nc].contiguous(), sh_degree)
        gctx.seq += 1
        ctx.seq = gctx.seq
        dev = means.device
        H, W = cam.height, cam.width
        rgb = torch.empty((H, W, 3), device=dev)
        alpha = torch.empty((H, W), device=dev)
        depth = torch.empty((H, W), device=dev)
        gcam, gopt = gut.make_camera(cam), gut.make_options(opt)
        out = gut.gut_outputs(rgb.data_ptr(), alpha.data_ptr(), depth.data_ptr(), 1, 0)
        gut.gut_render(gctx.ctx, gctx.scene, gcam, gopt, out, stats=False)
        ctx.gctx, ctx.gcam, ctx.gopt = gctx, gcam, gopt
        ctx.n, ctx.nc, ctx.nc_stored = means.shape[0], nc, sh.shape[1]
        ctx.save_for_backward(rgb, alpha, depth)
        return rgb, alpha, depth

    @staticmethod
    def backward(ctx, g_rgb, g_alpha, g_depth):
        if ctx.seq != ctx.gctx.seq:
            raise RuntimeError("gut backward: this render is no longer the context's last render "
                               "(one backward per forward, in order; use one context per outstanding view)")
        rgb, alpha, depth = ctx.saved_tensors
        dev = rgb.device
        n, nc = ctx.n, ctx.nc
        g = {k: torch.empty(sz, device=dev) for k, sz in (("means", (n, 3)), ("rotations", (n, 4)),
                                                           ("scales", (n, 3)), ("opacities", (n,)),
                                                           ("sh", (n, nc, 3)))}
        grads = gut.gut_gradients(*(g[k].data_ptr() for k in ("means", "rotations", "scales", "opacities", "sh")),
                                  None, None)
        p = lambda t: None if t is None else t.contiguous().data_ptr()  # noqa: E731
        g_rgb = g_rgb if g_rgb is not None else torch.zeros_like(rgb)
        gut.gut_render_backward(ctx.gctx.ctx, ctx.gctx.scene, ctx.gcam, ctx.gopt, rgb.data_ptr(), alpha.data_ptr(),
                                depth.data_ptr(), p(g_rgb), p(g_alpha), p(g_depth), grads)
        g_sh = g["sh"]
        if ctx.nc_stored > nc:  # coefficients above the active degree: zero gradient
            g_sh = torch.cat([g_sh, torch.zeros((n, ctx.nc_stored - nc, 3), device=dev)], dim=1)
        return (None, None, None, None, g["means"], g["rotations"], g["scales"], g["opacities"], g_sh)


def render(gctx: _Ctx, means, rotations, scales, opacities, sh, sh_degree: int, cam, opt=None):
    """Differentiable render (rgb [H,W,3], alpha [H,W], depth [H,W]) of activated
    Gaussian parameters (scales > 0, opacities in [0, 1]) on gctx's device."""
    return RenderFunction.apply(gctx, cam, opt, sh_degree, means, rotations, scales, opacities, sh)
