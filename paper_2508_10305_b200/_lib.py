"""ctypes binding of the in-tree CUDA library ``_gpzb.so`` (include/gpzb.h).

There is no fallback: if the library is missing this module raises
ImportError, and every compress / decompress call needs a CUDA device.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GPZB_LIB") or os.path.join(_HERE, "_gpzb.so")  # GPZB_LIB: A/B builds

OK, DOMAIN, WIDTH, CORRUPT, UNSUPPORTED, INVALID, NEED_SIDE = 0, 1, 2, 3, 4, 5, 6
F32, F64 = 0, 1
GLOBAL_HEADER_SIZE = 46
MAX_BLOCK_SIZE = 1 << 24   # K2b / K4b above 1024 particles per block (include/gpzb.h)
CTA_BLOCK_SIZE = 1024      # the largest block one CTA holds (the fast kernels)


class Result(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32),
        ("reason", ctypes.c_int32),
        ("block", ctypes.c_int64),
        ("axis", ctypes.c_int32),
        ("nonfinite_mask", ctypes.c_uint32),
        ("out_len", ctypes.c_uint64),
        ("eb_abs", ctypes.c_double),
        ("decode_block", ctypes.c_int64),
        ("decode_reason", ctypes.c_int32),
        ("decode_axis", ctypes.c_int32),
        ("count_block", ctypes.c_int64),
        ("table_flags", ctypes.c_uint32),
        ("pad_", ctypes.c_uint32),
        ("side_bytes", ctypes.c_uint64),
        ("reserved", ctypes.c_uint64 * 5),
    ]


class Header(ctypes.Structure):
    _fields_ = [
        ("dims", ctypes.c_uint32),
        ("precision", ctypes.c_uint32),
        ("preserve_order", ctypes.c_uint32),
        ("eb_mode", ctypes.c_uint32),
        ("eb", ctypes.c_double),
        ("eb_abs", ctypes.c_double),
        ("block_size", ctypes.c_uint32),
        ("version", ctypes.c_uint32),
        ("particle_count", ctypes.c_uint64),
        ("block_count", ctypes.c_uint64),
        ("table_end", ctypes.c_uint64),
        ("payload_len", ctypes.c_uint64),
    ]


# name -> (restype, argtypes); the exported surface of include/gpzb.h
_VP, _U64, _I32, _U32, _D = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_double
_RES = ctypes.POINTER(Result)
_HDR = ctypes.POINTER(Header)
SIGNATURES = {
    "gpzb_compress_bound": (_I32, [_U64, _I32, _I32, _U32, _U32, _I32, ctypes.POINTER(_U64)]),
    "gpzb_compress_workspace": (_I32, [_U64, _I32, _I32, _U32, ctypes.POINTER(_U64)]),
    "gpzb_decompress_workspace": (_I32, [_HDR, ctypes.POINTER(_U64)]),
    "gpzb_workspace_reset_async": (_I32, [_VP, _U64, _U64, _U32, _VP]),
    "gpzb_range_async": (_I32, [ctypes.POINTER(_VP), _I32, _I32, _U64, _U32, _VP, _U64, _VP]),
    "gpzb_range_words": (_I32, [_VP, _U64, ctypes.POINTER(_VP)]),
    "gpzb_encode_plan_async": (_I32, [ctypes.POINTER(_VP), _I32, _I32, _U64, _D, _I32, _U32, _U32, _I32, _VP,
                                      _U64, _VP]),
    "gpzb_encode_async": (_I32, [ctypes.POINTER(_VP), _I32, _I32, _U64, _D, _I32, _U32, _U32, _I32, _VP, _U64,
                                 _VP, _U64, _VP, _U64, _U64, _U64, _U64, _I32, _VP]),
    "gpzb_emit_async": (_I32, [ctypes.POINTER(_VP), _I32, _I32, _U64, _D, _I32, _U32, _I32, _VP, _U64, _VP, _VP,
                               _U64, _U64, _U64, _U64, _I32, _VP]),
    "gpzb_compress_result": (_I32, [_VP, _U64, _U64, _U32, _VP, _RES]),
    "gpzb_compress": (_I32, [ctypes.POINTER(_VP), _I32, _I32, _U64, _D, _I32, _U32, _U32, _I32, _VP, _U64, _VP,
                             _U64, _VP, _RES]),
    "gpzb_block_geometry": (_I32, [ctypes.POINTER(_VP), _I32, _I32, _U64, _U32, _U32, _D, _VP, _VP, _VP, _VP, _VP,
                                   _U64, _VP, _RES]),
    "gpzb_quantize": (_I32, [ctypes.POINTER(_VP), _I32, _I32, _U64, _U32, _U32, _D, _VP, _VP, _VP, _VP, _U64, _VP,
                             _RES]),
    "gpzb_encode_payloads": (_I32, [ctypes.POINTER(_VP), _I32, _I32, _U64, _U32, _U32, _I32, _D, _VP, _U64, _VP,
                                    _VP, _U64, _VP, _RES]),
    "gpzb_scan_workspace": (_I32, [_U64, ctypes.POINTER(_U64)]),
    "gpzb_scan_sizes": (_I32, [_VP, _U64, _VP, _VP, _U64, _VP]),
    "gpzb_parse_header": (_I32, [ctypes.c_char_p, _U64, _U64, _HDR, _RES]),
    "gpzb_block_counts_async": (_I32, [_VP, _U64, _HDR, _VP, _VP]),
    "gpzb_decompress": (_I32, [_VP, _U64, _HDR, ctypes.POINTER(_VP), _U64, _VP, _VP, _U64, _VP, _RES]),
    "gpzb_decompress_async": (_I32, [_VP, _U64, _HDR, ctypes.POINTER(_VP), _U64, _VP, _VP, _U64, _VP]),
    "gpzb_decompress_range_async": (_I32, [_VP, _U64, _HDR, ctypes.POINTER(_VP), _U64, _VP, _VP, _U64, _U64, _U64,
                                           _I32, _VP]),
    "gpzb_decompress_result": (_I32, [_VP, _U64, _HDR, _VP, _RES]),
    "gpzb_pair_workspace": (_I32, [_U64, _I32, ctypes.POINTER(_U64)]),
    "gpzb_pair_blocks": (_I32, [ctypes.POINTER(_VP), ctypes.POINTER(_VP), _I32, _I32, _I32, _U64, _D, _U32, _U32,
                                _VP, _VP, _VP, _U64, _VP, _RES]),
    "gpzb_pair_stats": (_I32, [ctypes.POINTER(_VP), ctypes.POINTER(_VP), _I32, _I32, _I32, _U64, _VP, _VP, _D,
                               _VP, _U64, _VP, _U64, _VP, ctypes.POINTER(_D), ctypes.POINTER(_U64)]),
    "gpzb_reason_message": (ctypes.c_char_p, [_I32]),
    "gpzb_version": (ctypes.c_char_p, []),
    "gpzb_kernel_launches": (_U64, []),
    "gpzb_encode_path_counts": (_I32, [_VP, _U64, _U64, _U32, _I32, _I32, _VP, ctypes.POINTER(_U64)]),
}


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"CUDA library {path} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()


def reason_message(code: int) -> str:
    return lib.gpzb_reason_message(int(code)).decode()


def ptr_array(ptrs):
    return (ctypes.c_void_p * max(1, len(ptrs)))(*ptrs)
