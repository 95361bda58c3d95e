"""The C-ABI library loads and exports every entry point include/snp.h declares;
argument validation runs before any CUDA call (so it is testable without a GPU)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def snp():
    from paper_2510_08491_b200 import build as B
    B.build()
    from paper_2510_08491_b200 import snp as S
    return S


def test_exports_match_header(snp):
    hdr = open(os.path.join(ROOT, "include", "snp.h")).read()
    declared = set(re.findall(r"\b(snp_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(snp.EXPORTS), declared ^ set(snp.EXPORTS)
    L = snp.lib()
    for name in declared:
        assert hasattr(L, name), name
    out = os.popen(f"nm -D --defined-only {snp.LIB_PATH}").read()
    for name in declared:
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_version_and_no_torch_in_signatures(snp):
    assert b"sm_100a" in snp.lib().snp_version()
    hdr = open(os.path.join(ROOT, "include", "snp.h")).read()
    assert "torch" not in hdr.replace("PyTorch", "").lower() or "at::" not in hdr


def _desc(snp, scene, **over):
    arrs = [np.ascontiguousarray(getattr(scene, f), np.float32) for f in snp.FIELDS]
    d = snp.SceneDesc(scene.n, 8, 3, 30.0, snp.SNP_MEM_HOST, *[a.ctypes.data for a in arrs])
    for k, v in over.items():
        setattr(d, k, v)
    return d, arrs


def test_argument_validation_without_gpu(snp):
    L = snp.lib()
    h = C.c_void_p()
    assert L.snp_create_scene(None, 0, None, C.byref(h)) == 1
    sc = synth.make_scene(0, 16)
    for n_hidden in (0, 6, 12, 64):                                             # widths 4/8/16/32 only
        d, keep = _desc(snp, sc, n_hidden=n_hidden)
        assert L.snp_create_scene(C.byref(d), 0, None, C.byref(h)) == 4      # UNSUPPORTED
    d, keep = _desc(snp, sc, sh_degree=4)
    assert L.snp_create_scene(C.byref(d), 0, None, C.byref(h)) == 1
    d, keep = _desc(snp, sc, n=-1)
    assert L.snp_create_scene(C.byref(d), 0, None, C.byref(h)) == 1
    # stage calls on a NULL handle
    assert L.snp_project(None, None, 1, None) == 1
    assert L.snp_bin_sort(None, None, None) == 1
    assert L.snp_render(None, None, None, None) == 1
    assert L.snp_project_at(None, None, 1, None, None) == 1
    assert L.snp_set_temporal(None, None, 0, None) == 1
    assert L.snp_render_backward(None, None, None, None, None, None, None, None, None, None, None, None) == 1
    assert L.snp_render_backward_ex(None, None, None, None, None, None, None, None, None, None, None, None,
                                    None) == 1
    assert L.snp_scale_regularizer(None, 0.0, None, None, None) == 1
    assert L.snp_adam_step(None, None, None, 0.9, 0.999, 1e-8, 1, None) == 1
    assert L.snp_get_params(None, None, 0, None) == 1
    # the loss needs no scene: its argument checks come first
    assert L.snp_loss_l1(None, None, -1, None, None, None) == 1
    assert L.snp_loss_l1(None, None, 5, None, None, None) == 1
    assert L.snp_destroy(None) == 0


def test_product_fails_loudly_without_library(snp, monkeypatch, tmp_path):
    monkeypatch.setattr(snp, "_lib", None)
    monkeypatch.setattr(snp, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        snp.lib()


def test_product_does_not_import_oracle():
    import ast
    pkg = os.path.join(ROOT, "paper_2510_08491_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dp, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, (ast.Import, ast.ImportFrom)):
                        names = [a.name for a in node.names] + [getattr(node, "module", "") or ""]
                        assert not any(n.split(".")[0] in ("oracle", "synth") for n in names), (f, names)
            if f.endswith((".cu", ".cuh", ".h")):
                for line in open(os.path.join(dp, f)):
                    assert not (line.startswith("#include") and "oracle" in line), (f, line)
