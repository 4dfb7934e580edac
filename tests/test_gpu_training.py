"""A training loop through the C ABI (PAPER Sec. 4.4 / Supp. B workload):
paper_2412_12507_b200.autograd wraps gut_render / gut_render_backward as a
torch.autograd.Function; Adam fits a perturbed copy of a tiny scene to the
target image rendered from the original.  The photometric loss must drop."""
import numpy as np
import pytest

import scenegen as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_12507_b200 import build
    build.build()


@pytest.mark.parametrize("variant", ["pinhole", "fisheye", "rs"])
def test_fit_tiny_scene(variant):
    import torch
    from paper_2412_12507_b200 import autograd as A
    scene, cam = S.tiny(11, variant, n=64, sh_degree=1)
    dev = torch.device("cuda", 0)
    T = lambda a: torch.tensor(np.asarray(a, np.float32), device=dev)  # noqa: E731
    g = A.RenderFunction.context(0)
    with torch.no_grad():
        target, _, _ = A.render(g, T(scene.means), T(scene.rotations), T(scene.scales), T(scene.opacities),
                                T(scene.sh), 1, cam)
        target = target.clone()
    rng = np.random.default_rng(0)
    means = T(scene.means + rng.normal(0, 0.03, scene.means.shape)).requires_grad_()
    quats = T(scene.rotations).requires_grad_()
    log_s = T(np.log(scene.scales) + rng.normal(0, 0.2, scene.scales.shape)).requires_grad_()
    logit_o = T(np.log(scene.opacities / (1 - scene.opacities)) * 0 + 0.0).requires_grad_()
    sh = T(scene.sh + rng.normal(0, 0.3, scene.sh.shape)).requires_grad_()
    opt = torch.optim.Adam([{"params": [means], "lr": 2e-3}, {"params": [quats], "lr": 1e-2},
                            {"params": [log_s], "lr": 1e-2}, {"params": [logit_o], "lr": 5e-2},
                            {"params": [sh], "lr": 2e-2}])
    losses = []
    for it in range(200):
        opt.zero_grad()
        rgb, alpha, depth = A.render(g, means, quats, torch.exp(log_s), torch.sigmoid(logit_o), sh, 1, cam)
        loss = (rgb - target).abs().mean()
        loss.backward()
        opt.step()
        losses.append(float(loss.detach()))
    g.close()
    print(f"{variant}: L1 {losses[0]:.4f} -> {losses[-1]:.4f}")
    assert np.isfinite(losses).all()
    assert losses[-1] < 0.35 * losses[0], (losses[0], losses[-1])
