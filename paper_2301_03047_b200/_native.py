"""ctypes binding of libglr_b200.so (include/glr_b200.h).

The product path has no CPU fallback: importing a compute entry point
without the built library, or calling it without a CUDA device, raises
``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libglr_b200.so"

GLR_OK = 0
GLR_ERR_INVALID = 1
GLR_ERR_BOUNDS = 2
GLR_ERR_NONFINITE = 3
GLR_ERR_CUDA = 4
GLR_ERR_UNSUPPORTED = 5
GLR_ERR_WORKSPACE = 6


class NativeUnavailable(RuntimeError):
    """The CUDA extension is missing or no CUDA device is visible."""


class GlrCudaError(RuntimeError):
    """A CUDA launch or runtime call inside libglr_b200 failed."""


vp = C.c_void_p
i32 = C.c_int
i64 = C.c_int64
f64 = C.c_double
sz = C.c_size_t

# name -> (restype, argtypes); mirrors include/glr_b200.h
SIGNATURES: dict[str, tuple] = {
    "glr_last_error": (C.c_char_p, []),
    "glr_version": (i32, []),
    "glr_device_info": (i32, [vp, vp, vp]),
    "glr_eig_work": (i32, [vp, i32]),
    "glr_sobel": (i32, [vp, i32, i32, i32, vp, vp, vp]),
    "glr_edge_stack": (i32, [vp, vp, i32, i32, i32, f64, i32, i32, vp, vp, vp, vp]),
    "glr_stack_from_maps": (i32, [vp, i32, i32, i32, i32, vp, vp]),
    "glr_corner_workspace": (sz, [i32, i32, i32]),
    "glr_corner_response": (i32, [vp, i32, i32, i32, vp, vp, vp]),
    "glr_corner_response_grad": (i32, [vp, vp, i32, i32, i32, vp, vp, vp]),
    "glr_nms_workspace": (sz, [i32, i32]),
    "glr_corners": (i32, [vp, i32, i32, i32, i32, f64, vp, vp, vp, sz, vp]),
    "glr_anchor_workspace": (sz, [i32, i32]),
    "glr_select_anchors": (i32, [vp, vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp]),
    "glr_heat_expand_factor": (i32, [i32, i32]),
    "glr_heat_workspace": (sz, [i32, i32, i32]),
    "glr_heat_map": (i32, [vp, i32, i32, i32, i32, i32, vp, i32, vp, vp, vp, sz, vp]),
    "glr_topk_workspace": (sz, [i32, i32, i32]),
    "glr_heat_topk_workspace": (sz, [i32, i32, i32, i32]),
    "glr_heat_topk": (i32, [vp, i32, i32, i32, i32, i32, vp, i32, i32, i32, i32, vp, vp, vp, vp, sz,
                            vp]),
    "glr_topk": (i32, [vp, i32, vp, i32, i32, i32, vp, i32, i32, vp, vp, vp, sz, vp]),
    "glr_gather": (i32, [vp, i32, i32, i32, i32, vp, i32, i32, vp, vp]),
    "glr_block_match": (i32, [vp, i32, i32, i32, i32, vp, i32, i32, i32, i32, vp, vp, vp]),
    "glr_rerank_pixel": (i32, [vp, i32, i32, i32, i32, vp, i32, i32, vp]),
    "glr_tv_workspace": (sz, [i32, i32, i32]),
    "glr_xcorr_valid": (i32, [vp, i32, i32, i32, vp, i32, i32, vp, vp]),
    "glr_tv_denoise": (i32, [vp, i32, i32, i32, f64, i32, vp, vp, sz, vp]),
    "glr_wnnm_workspace": (sz, [i32, i32]),
    "glr_wnnm": (i32, [vp, i32, i32, i32, f64, f64, f64, f64, vp, vp, vp, sz, vp]),
    "glr_wnnm_scatter": (i32, [vp, i32, i32, i32, i32, vp, i32, vp, i32, f64, f64, f64, i32, vp,
                               vp, i32, vp, vp, sz, vp]),
    "glr_vcache_remap": (i32, [vp, i32, i32, vp, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, i32,
                               vp]),
    "glr_scatter_count": (i32, [vp, i32, vp, i32, i32, i32, i32, vp, vp]),
    "glr_scatter_add_f64": (i32, [vp, vp, i32, i32, i32, i32, i32, i32, vp, vp, vp]),
    "glr_scatter_fixed": (i32, [vp, vp, i32, i32, i32, i32, i32, i32, i32, vp, vp]),
    "glr_heat_stride": (i64, [i32, i32, i32]),
    "glr_normalize": (i32, [vp, vp, vp, i32, i32, i32, i32, vp, vp]),
    "glr_masksum_forward": (i32, [vp, vp, i32, i32, i32, vp, vp]),
    "glr_masksum_adjoint": (i32, [vp, vp, i32, i32, i32, vp, vp]),
    "glr_gap_workspace": (sz, [i32, i32]),
    "glr_gap_masksum": (i32, [vp, vp, i32, vp, vp, vp, vp, i32, i32, i32, f64, f64, f64, vp, vp,
                              vp, vp]),
    "glr_fft_workspace": (sz, [i32, i32]),
    "glr_fourier_forward": (i32, [vp, vp, i32, i32, i32, vp, vp, vp]),
    "glr_fourier_adjoint": (i32, [vp, vp, i32, i32, i32, vp, vp, vp]),
    "glr_gap_fourier": (i32, [vp, vp, i32, vp, vp, vp, i32, i32, i32, i32, f64, f64, f64, vp, vp,
                              vp, vp]),
    "glr_lincomb": (i32, [vp, f64, vp, f64, vp, f64, i64, i32, f64, f64, vp, vp]),
    "glr_interp_msfa": (i32, [vp, vp, i32, i32, i32, C.POINTER(C.c_double), i32, vp, vp, vp]),
    "glr_interp_cacti": (i32, [vp, vp, i32, i32, i32, vp, vp]),
    "glr_sq_err": (i32, [vp, vp, i32, f64, vp, vp, vp]),
    "glr_ssim_workspace": (sz, [i32, i32, i32]),
    "glr_ssim": (i32, [vp, vp, i32, i32, i32, f64, i32, C.POINTER(C.c_double), i32, vp, vp, vp]),
}

_lib = None


def lib_path() -> Path:
    return _LIB_PATH


def load(require_gpu: bool = False):
    """Load the shared library (once). ``require_gpu`` also checks for a CUDA
    device, which every compute entry point needs."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise NativeUnavailable(
                f"{_LIB_PATH.name} is not built; run `python -c \"import __graft_entry__ as g; "
                f"g.build()\"` (no CPU fallback exists)")
        lib = C.CDLL(str(_LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_gpu:
        import torch
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device visible: the GLR B200 path has no CPU fallback")
    return _lib


def last_error() -> str:
    return load().glr_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    """Map a C status code onto the reference's exception types."""
    if status == GLR_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if status in (GLR_ERR_INVALID, GLR_ERR_BOUNDS, GLR_ERR_NONFINITE):
        raise ValueError(msg)
    if status == GLR_ERR_CUDA:
        raise GlrCudaError(msg)
    raise RuntimeError(f"glr status {status}: {msg}")


# Own kernels launched per successful call (fixed by each entry point's body;
# the CUB radix-sort kernels inside glr_corners are not counted). Used for the
# bench's gpu_launches claim.
KERNELS_PER_CALL = {
    "glr_sobel": 1, "glr_stack_from_maps": 1, "glr_corner_response": 6, "glr_corner_response_grad": 5, "glr_corners": 3,
    "glr_select_anchors": 1, "glr_heat_map": 2, "glr_topk": 1, "glr_gather": 1, "glr_wnnm": 3,
    "glr_wnnm_scatter": 3, "glr_scatter_count": 1, "glr_scatter_fixed": 1,
    "glr_scatter_add_f64": 1, "glr_normalize": 1, "glr_masksum_forward": 1,
    "glr_masksum_adjoint": 1, "glr_gap_masksum": 2, "glr_fourier_forward": 4,
    "glr_fourier_adjoint": 4, "glr_gap_fourier": 11, "glr_sq_err": 2, "glr_vcache_remap": 3,
    "glr_lincomb": 1, "glr_interp_msfa": 3, "glr_interp_cacti": 1, "glr_heat_topk": 6, "glr_ssim": 3,
    "glr_block_match": 1, "glr_rerank_pixel": 1, "glr_xcorr_valid": 1,
}
launch_count = 0


def call(name: str, *args) -> int:
    global launch_count
    lib = load(require_gpu=True)
    st = getattr(lib, name)(*args)
    check(st, name)
    if name == "glr_edge_stack":  # relative max pass + maps and/or stack
        launch_count += int(bool(args[6])) + int(args[8] is not None) + int(args[9] is not None)
    elif name == "glr_tv_denoise":  # one launch per dual step + the output
        launch_count += (int(args[5]) + 1) if args[4] > 0 else 0
    else:
        launch_count += KERNELS_PER_CALL.get(name, 0)
    return st


def query(name: str, *args):
    """Host-only size / geometry queries (no device needed)."""
    return getattr(load(), name)(*args)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
