"""ctypes binding to libshorb200.so (the C ABI in include/shorb200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, every device operation raises.  Device buffers are torch
CUDA tensors (allocation, streams and torch.distributed are the only things
torch provides); the C ABI sees plain pointers and the current stream.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libshorb200.so"

SHB_OK, SHB_EINVAL, SHB_ECUDA, SHB_ENOMEM, SHB_ERANGE, SHB_EIO = 0, 1, 2, 3, 4, 5
FP64, FP32 = 0, 1

# every symbol include/shorb200.h declares, with its ctypes signature
_u64, _u32, _i32, _f64, _vp = (ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int,
                               ctypes.c_double, ctypes.c_void_p)
_P64 = ctypes.POINTER(ctypes.c_uint64)
_PF64 = ctypes.POINTER(ctypes.c_double)
SIGNATURES = {
    "shb_abi_version": ([], _i32),
    "shb_last_error": ([], ctypes.c_char_p),
    "shb_device_info": ([_i32, ctypes.POINTER(ctypes.c_int), ctypes.c_char_p, _i32], _i32),
    "shb_kernel_launches": ([], _u64),
    "shb_fp64_peak": ([_f64, _PF64, _vp], _i32),
    "shb_fp64_dmma_peak": ([_f64, _PF64, _vp], _i32),
    "shb_modexp": ([_vp, _u64, _u64, _u64, _u64, _vp], _i32),
    "shb_class_counts": ([_vp, _u64, _vp, _u64, _vp], _i32),
    "shb_compact_eq": ([_vp, _u64, _u32, _u64, _vp, _u64, _P64, _vp], _i32),
    "shb_support_progression": ([_vp, _u64, _P64, _P64, _P64, _vp], _i32),
    "shb_state_progression": ([_vp, _u64, _P64, _P64, _P64, _vp], _i32),
    "shb_gather_progression": ([_vp, _u64, _u64, _u64, _vp, _vp], _i32),
    "shb_progression_is_uniform": ([_vp, _u64, ctypes.POINTER(ctypes.c_int), _PF64, _PF64, _vp], _i32),
    "shb_progression_kind": ([_vp, _u64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), _PF64, _PF64,
                              _vp], _i32),
    "shb_fill_progression": ([_vp, _u64, _u64, _u64, _u64, _f64, _f64, _vp, _vp], _i32),
    "shb_dft": ([_vp, _u64, _u64, _u64, _u64, _u64, _u64, _u32, _f64, _i32, _vp, _vp, _vp, _vp], _i32),
    "shb_dft_engine": ([ctypes.c_int, ctypes.c_int, _u64, _i32, _u32, ctypes.POINTER(ctypes.c_int)], ctypes.c_char_p),
    "shb_dft_real": ([_vp, _u64, _u64, _u64, _u64, _u64, _u64, _u32, _f64, _i32, _vp, _vp, _vp, _vp], _i32),
    "shb_dft_uniform": ([_f64, _f64, _u64, _u64, _u64, _u64, _u64, _u64, _u32, _f64, _i32, _vp, _vp, _vp, _vp],
                        _i32),
    "shb_dft_num_blocks": ([_u64, _i32], _u64),
    "shb_apply_hadamard": ([_vp, _u64, _i32, _vp], _i32),
    "shb_apply_controlled_phase": ([_vp, _u64, _i32, _i32, _f64, _f64, _vp], _i32),
    "shb_bit_reverse_permute": ([_vp, _vp, _u64, _vp], _i32),
    "shb_probabilities": ([_vp, _u64, _vp, _vp], _i32),
    "shb_sum": ([_vp, _u64, _PF64, _vp], _i32),
    "shb_cumsum_total": ([_vp, _u64, _PF64, _vp], _i32),
    "shb_cumsum_search": ([_vp, _u64, _f64, _P64, _vp], _i32),
    "shb_cumsum_total_from": ([_vp, _u64, _f64, _PF64, _vp], _i32),
    "shb_cumsum_search_from": ([_vp, _u64, _f64, _f64, _P64, _vp], _i32),
    "shb_sample_index": ([_vp, _u64, _f64, _P64, _PF64, _vp], _i32),
    "shb_cumsum_tiles": ([_u64], _u64),
    "shb_cumsum_record_bytes": ([], _u64),
    "shb_cumsum_records": ([_vp, _u64, _f64, _vp, _vp], _i32),
    "shb_cumsum_walk": ([_vp, _u64, _vp, _f64, _vp, _PF64, _vp], _i32),
    "shb_cumsum_find": ([_vp, _u64, _vp, _f64, _f64, _P64, _vp], _i32),
    "shb_dense_dft_host": ([_vp, _u64, _u32, _i32, _vp], _i32),
    "shb_partial_row_sums_host": ([_vp, _vp, _vp, _u64, _u64, _u64, _u64, _u64], _i32),
    "shb_init": ([_i32, ctypes.POINTER(_vp)], _i32),
    "shb_init_devices": ([_vp, _i32, ctypes.POINTER(_vp)], _i32),
    "shb_free": ([_vp], None),
    "shb_ctx_state": ([_vp, ctypes.POINTER(ctypes.c_int), _P64, _P64, ctypes.POINTER(ctypes.c_int)], _i32),
    "shb_ctx_modexp": ([_vp, _u64, _u64, _u32], _i32),
    "shb_ctx_class_counts": ([_vp, _vp, _u64], _i32),
    "shb_collapse": ([_vp, _u32, _P64, _PF64], _i32),
    "shb_measure": ([_vp, _f64, ctypes.POINTER(ctypes.c_uint32), _P64, _PF64], _i32),
    "shb_ctx_dft": ([_vp, _i32, _u32], _i32),
    "shb_norm": ([_vp, _PF64], _i32),
    "shb_sample": ([_vp, _f64, _P64], _i32),
    "shb_copy_spectrum": ([_vp, _u64, _u64, _vp], _i32),
    "shb_copy_support": ([_vp, _vp, _u64, _P64], _i32),
    "shb_copy_residues": ([_vp, _u64, _u64, _vp], _i32),
    "shb_dump_state": ([_vp, ctypes.c_char_p], _i32),
    "shb_host_measure_class": ([_vp, _u64, _u64, _f64, ctypes.POINTER(ctypes.c_uint32), _P64, _PF64], _i32),
    "shb_host_seqsum_const": ([_f64, _u64], _f64),
    "shb_host_pairwise_sum_const": ([_f64, _u64], _f64),
}

_lib = None


def load(path: Path | None = None) -> ctypes.CDLL:
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise ImportError(
            f"{p} is missing: build it with `python -m paper_1801_01434_b200.build` "
            "(the B200 path has no CPU fallback)")
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.shb_abi_version() != 1:
        raise ImportError("libshorb200.so ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == SHB_OK:
        return
    msg = (load().shb_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc in (SHB_EINVAL, SHB_ERANGE):
        raise ValueError(text)
    if rc == SHB_ENOMEM:
        raise MemoryError(text)
    if rc == SHB_EIO:
        raise OSError(text)
    raise RuntimeError(text)


# ------------------------------------------------------------------ torch glue

def torch():
    import torch as _t
    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the B200 path has no CPU fallback")
    load()
    return t


def stream_ptr() -> int:
    t = torch()
    return t.cuda.current_stream().cuda_stream


def ptr(tensor) -> int:
    return 0 if tensor is None else int(tensor.data_ptr())


def host_seqsum_const(w: float, count: int) -> float:
    return float(load().shb_host_seqsum_const(float(w), int(count)))


def host_pairwise_sum_const(w: float, count: int) -> float:
    return float(load().shb_host_pairwise_sum_const(float(w), int(count)))


def as_c_double_ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)
