"""GPU parity of the generalized Gaussian kernels of degree n (PAPER Supp. A,
L454-462, reading R29) through the C ABI: every stage against the fp64
oracle (K1 extent level, binning, K5 response), for "Ours" and "Ours (sorted)"."""
import numpy as np
import pytest

import scenegen as S
from test_gpu_parity import _full_parity
from test_gpu_kbuffer import _full as _full_kbuf

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_12507_b200 import build
    build.build()


@pytest.mark.parametrize("n", [3, 4, 5, 8])  # the degrees of Table 4
@pytest.mark.parametrize("variant", S.TINY_VARIANTS)
def test_tiny_degree(variant, n):
    scene, cam = S.tiny(2, variant, n=96)
    _full_parity(scene, cam, S.RenderOptions(kernel_degree=n), label=f"{variant} n={n}")


@pytest.mark.parametrize("n", [4, 8])
def test_tiny_degree_kbuffer(n):
    scene, cam = S.tiny(4, "fisheye", n=128)
    _full_kbuf(scene, cam, S.RenderOptions(kernel_degree=n, kbuffer=16), label=f"fisheye n={n} k=16")


@pytest.mark.parametrize("config,n,factor,view", [("multiview", 100_000, 0.2, 5), ("waymo", 80_000, 0.15, 1)])
def test_reduced_config_degree4(config, n, factor, view):
    scene = S.make_scene(config, n=n)
    cam = S.scaled_camera(S.make_views(config)[view], factor)
    g, o, _ = _full_parity(scene, cam, S.RenderOptions(kernel_degree=4), max_excluded=0.02,
                           label=f"{config} n={n} degree 4")
    # the degree changes every extent (k2_4 = 3 sqrt(k2_2)): the key count moves
    g2, _, _ = _full_parity(scene, cam, S.RenderOptions(), max_excluded=0.02, label=f"{config} degree 2")
    assert g["stats"]["n_keys"] != g2["stats"]["n_keys"]


def test_invalid_degree():
    from paper_2412_12507_b200 import gut
    scene, cam = S.tiny(0)
    r = gut.Renderer(scene)
    with pytest.raises(gut.GutError) as e:
        r.render(cam, S.RenderOptions(kernel_degree=0))
    assert e.value.status == 1 and "kernel_degree" in str(e.value)
    r.close()
