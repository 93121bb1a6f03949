"""The C-ABI library loads and exports every entry point include/glr_b200.h
declares; host-only geometry queries answer without a GPU (CPU tests)."""

import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "glr_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(glr_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    names = declared_functions()
    for must in ["glr_sobel", "glr_edge_stack", "glr_corner_response", "glr_corners",
                 "glr_select_anchors", "glr_heat_map", "glr_topk", "glr_gather", "glr_wnnm",
                 "glr_wnnm_scatter", "glr_scatter_count", "glr_normalize", "glr_gap_masksum",
                 "glr_gap_fourier", "glr_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2301_03047_b200 import _native as N
    lib = N.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in N.SIGNATURES, f"{name} missing from the ctypes binding"


def test_host_queries_without_gpu():
    from paper_2301_03047_b200 import _native as N
    assert N.query("glr_version") == 1
    # expansion factor: pixel stride e*4C must be a multiple of 16 bytes
    for c, p in [(24, 8), (16, 8), (8, 8), (2, 8), (1, 8), (1, 12), (3, 4), (1, 3)]:
        e = N.query("glr_heat_expand_factor", c, p)
        assert e >= 1 and (4 * c * e) % 16 == 0
    assert N.query("glr_heat_expand_factor", 24, 8) == 1
    assert N.query("glr_heat_stride", 1024, 1024, 8) % 8 == 0
    assert N.query("glr_heat_stride", 256, 256, 8) == 249 * 249 + 7
    assert N.query("glr_corner_workspace", 64, 64, 3) > 64 * 64 * 3 * 8
    assert N.query("glr_nms_workspace", 64, 64) > 0


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2301_03047_b200 as G
    from paper_2301_03047_b200._native import NativeUnavailable
    with pytest.raises(NativeUnavailable):
        G.sobel_gradients(np.zeros((8, 8, 1)))
    with pytest.raises(NativeUnavailable):
        G.wnnm_prox(np.eye(4), G.WnnmParams(noise_sigma=0.1))
