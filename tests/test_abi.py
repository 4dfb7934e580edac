"""CPU checks of the boundary: libgut.so builds for sm_100a, loads, exports
every symbol include/gut.h declares, struct layouts agree with the binding,
and without a GPU the library refuses to run (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "gut.h")


@pytest.fixture(scope="module")
def libgut():
    from paper_2412_12507_b200 import build
    build.build()
    from paper_2412_12507_b200 import gut
    return gut


def declared_functions():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^[\w \*]*?\b(gut_[a-z_]+)\s*\(", src, re.M)))


def test_exports_every_declared_symbol(libgut):
    names = declared_functions()
    assert len(names) >= 11, names
    out = subprocess.run(["nm", "-D", "--defined-only", libgut.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (gut_[a-z_]+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    L = libgut.lib()
    for n in names:
        assert getattr(L, n) is not None


def test_struct_layouts_match_header(libgut, tmp_path):
    prog = tmp_path / "sz.c"
    prog.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "gut.h"\n'
                    'int main(){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(gut_camera), sizeof(gut_options),'
                    'sizeof(gut_stats), sizeof(gut_proj_record), sizeof(gut_gaussians), sizeof(gut_outputs),'
                    'offsetof(gut_camera, q_c2w), sizeof(gut_gradients), sizeof(gut_quality),'
                    'offsetof(gut_options, kbuffer), offsetof(gut_options, kernel_degree));}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I" + os.path.join(ROOT, "include"), str(prog), "-o", str(exe)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    g = libgut
    want = [C.sizeof(g.gut_camera), C.sizeof(g.gut_options), C.sizeof(g.gut_stats), C.sizeof(g.gut_proj_record),
            C.sizeof(g.gut_gaussians), C.sizeof(g.gut_outputs), g.gut_camera.q_c2w.offset, C.sizeof(g.gut_gradients),
            144, g.gut_options.kbuffer.offset, g.gut_options.kernel_degree.offset]
    assert got == want


def test_sm100a_only(libgut):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libgut.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, out


def test_abi_version_and_defaults(libgut):
    assert libgut.gut_abi_version() == 1
    o = libgut.make_options()
    assert (o.ut_alpha, o.ut_beta, o.ut_kappa) == (1.0, 2.0, 0.0)
    assert o.alpha_min == pytest.approx(1 / 255) and o.tile_cull == 1


def test_no_cpu_fallback(libgut):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(libgut.GutError) as e:
        libgut.gut_context_create(0)
    assert e.value.status in (2, 5)
