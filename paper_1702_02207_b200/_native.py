"""ctypes binding of ``libosc_b200.so`` (declared in ``include/osc_b200.h``).

This is the binding a maintainer would add to the reference package (see
INTEGRATION.md).  There is no CPU fallback: if the library or a CUDA device is
missing, every entry point raises :class:`NativeUnavailableError`.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# OSC_LIB: load another build of the same library (compiler-option sweeps in
# scripts/; the product default is the in-tree build).
LIB_PATH = os.environ.get("OSC_LIB") or os.path.join(HERE, "libosc_b200.so")

OSC_OK, OSC_NONFINITE, OSC_INVALID, OSC_CUDA_ERROR = 0, 1, 2, 3
ABI_VERSION = 11
OSC_FMA = 1
OSC_TRUSTED = 2
OSC_TILES_INTERIOR = 4
OSC_TILES_EDGES = 8

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_dbl = ctypes.c_double

# name -> (restype, argtypes); mirrors include/osc_b200.h one to one.
SIGNATURES = {
    "osc_abi_version": (ctypes.c_int, []),
    "osc_last_error": (ctypes.c_char_p, []),
    "osc_validate_parameters": (ctypes.c_int, [_vp, _vp, _i64, ctypes.POINTER(ctypes.c_int64),
                                               _vp]),
    "osc_last_invalid_parameter": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int),
                                                  ctypes.POINTER(ctypes.c_int64)]),
    "osc_rk4_batch2": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _dbl, _i64, _i64, _vp, _vp,
                                      _vp, _vp, ctypes.c_uint32, _vp]),
    "osc_analytic_batch2": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "osc_compare_batch2": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _vp]),
    "osc_rk4_batch2_compare": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _dbl, _i64, _i64, _vp,
                                              _vp, _vp, _vp, ctypes.c_uint32, _vp]),
    "osc_rk4_chains": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _dbl, _i64, _i64, _vp,
                                      _vp, _vp, _vp, _i64, ctypes.c_uint32, _vp]),
    "osc_rk4_chain_advance": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64,
                                             _dbl, _i64, _i64, _vp, _vp, _vp, _vp,
                                             ctypes.c_uint32, _vp]),
    "osc_rk4_chain_advance_div2": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64,
                                                  _i64, _dbl, _i64, _i64, _vp, _vp, _vp, _vp,
                                                  _vp, ctypes.c_uint32, _vp]),
    "osc_edge_sync_status": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_uint64), _vp]),
    "osc_rk4_shard_run": (ctypes.c_int, [_vp, _dbl, _i64, _i64, _i64, ctypes.c_uint32, _vp]),
    "osc_rk4_shard_run_nccl": (ctypes.c_int, [_vp, _vp, ctypes.c_int, ctypes.c_int, _dbl, _i64,
                                              _i64, _i64, ctypes.c_uint32, _vp]),
    "osc_stream_write_u64": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64]),
    "osc_stream_wait_u64": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64]),
    "osc_chain_plan": (ctypes.c_int, [_i64, _i64, _i64, _i64, _vp]),
    "osc_rk4_chain_sharded": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int), _vp,
                                             _vp, _vp, _vp, _i64, _dbl, _i64, _i64, _vp,
                                             ctypes.c_uint32]),
    "osc_rowscale": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp]),
    "osc_rk4_dense": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _dbl, _i64, _vp, _vp]),
    "osc_equation_engine": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _dbl, _i64, _i64, _vp,
                                           _vp, _vp, _vp, _vp]),
    "osc_device_alloc": (ctypes.c_int, [ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]),
    "osc_device_free": (ctypes.c_int, [_vp]),
    "osc_ipc_export": (ctypes.c_int, [_vp, ctypes.c_char_p]),
    "osc_ipc_import": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "osc_ipc_close": (ctypes.c_int, [_vp]),
    "osc_ipc_event_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_char_p]),
    "osc_ipc_event_open": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "osc_event_record": (ctypes.c_int, [_vp, _vp]),
    "osc_stream_wait_event": (ctypes.c_int, [_vp, _vp]),
    "osc_event_destroy": (ctypes.c_int, [_vp]),
    "osc_derivative": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, ctypes.c_int, _vp]),
    "osc_energy": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, ctypes.c_int, _vp]),
    "osc_check_division": (ctypes.c_int, [_i64, ctypes.c_uint64, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_uint64), _vp]),
    "osc_div2_classify": (ctypes.c_int, [_vp, _i64, _vp, _vp]),
    "osc_div2c_table": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp]),
    "osc_bench_fp64": (ctypes.c_int, [_i64, ctypes.c_int, _vp, ctypes.POINTER(ctypes.c_int64),
                                       _vp]),
    "osc_rk4_batch2_host": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _dbl, _i64, _i64, _vp,
                                           _vp, _vp]),
    "osc_rk4_chains_host": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _dbl, _i64, _i64,
                                           _vp, _vp, _vp]),
    "osc_derivative_host": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, ctypes.c_int]),
    "osc_energy_host": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, ctypes.c_int]),
}


class Peer(ctypes.Structure):
    """osc_peer_t: a neighbour's next-input buffers for the fused exchange."""

    _fields_ = [("x", ctypes.c_void_p), ("v", ctypes.c_void_p), ("offset", ctypes.c_int64),
                ("count", ctypes.c_int64)]


class EdgeSync(ctypes.Structure):
    """osc_edge_sync_t: device-side ordering of a shard's edge tiles with its
    neighbours (ready: the neighbours' counters facing us; counters: ours)."""

    _fields_ = [("ready", ctypes.c_void_p * 2), ("counters", ctypes.c_void_p),
                ("period", ctypes.c_uint64), ("timeout_ns", ctypes.c_int64)]


class Shard(ctypes.Structure):
    """osc_shard_t: one shard of the multi-process fused exchange."""

    _fields_ = [("m", ctypes.c_void_p), ("C", ctypes.c_void_p),
                ("x", ctypes.c_void_p * 2), ("v", ctypes.c_void_p * 2),
                ("nx", (ctypes.c_void_p * 2) * 2), ("nv", (ctypes.c_void_p * 2) * 2),
                ("n", ctypes.c_int64), ("own_lo", ctypes.c_int64), ("own_hi", ctypes.c_int64),
                ("offset", ctypes.c_int64 * 2), ("ghost", ctypes.c_int64),
                ("first_bad", ctypes.c_void_p), ("sync", EdgeSync), ("div2", ctypes.c_void_p)]


class NativeUnavailableError(RuntimeError):
    """The sm_100a library or a CUDA device is missing; there is no fallback."""


_LIB = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the library and bind every exported symbol (no device needed)."""
    global _LIB
    if _LIB is not None and path == LIB_PATH:
        return _LIB
    if not os.path.exists(path):
        raise NativeUnavailableError(
            f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.osc_abi_version() != ABI_VERSION:
        raise NativeUnavailableError("libosc_b200.so ABI version mismatch")
    if path == LIB_PATH:
        _LIB = lib
    return lib


_DEVICE_OK = False


def lib() -> ctypes.CDLL:
    """The library, after checking (once) that a CUDA device is present."""
    global _DEVICE_OK
    if not _DEVICE_OK:
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailableError("no CUDA device: the B200 path has no CPU fallback")
        _DEVICE_OK = True
    return load()


def last_error() -> str:
    return (load().osc_last_error() or b"").decode(errors="replace")


def last_invalid_parameter():
    """(which, flat index) of the offending parameter of this thread's last
    OSC_INVALID -- which = 0 masses, 1 springs -- or None."""
    which, index = ctypes.c_int(-1), ctypes.c_int64(-1)
    if load().osc_last_invalid_parameter(ctypes.byref(which), ctypes.byref(index)):
        return which.value, index.value
    return None
