"""Peer memory between the processes of a multi-GPU run (one process per GPU).

Thin wrappers over the C ABI's ``osc_device_alloc`` / ``osc_ipc_*`` /
``osc_event_*``: raw device allocations (so an exported pointer is an
allocation base), their CUDA IPC handles, mapped neighbour buffers (NVLink
peer access between GPUs) and interprocess events.  Used by
``sharded.ShardedChain(transport="peer")``; lifetimes are explicit (``close``)
so that no process unmaps or frees while a neighbour can still touch memory.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native


def _check(rc, what):
    if rc != _native.OSC_OK:
        raise RuntimeError(f"{what}: {_native.last_error()}")


class _CudaArray:
    """__cuda_array_interface__ view of a raw float64 device vector."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class DeviceVector:
    """A float64 device vector in its own cudaMalloc allocation, exportable by IPC."""

    def __init__(self, n: int, device: torch.device):
        lib = _native.lib()
        p = ctypes.c_void_p()
        _check(lib.osc_device_alloc(8 * max(n, 1), ctypes.byref(p)), "osc_device_alloc")
        self.ptr = p.value
        self.n = n
        self.tensor = torch.as_tensor(_CudaArray(self.ptr, n), device=device)

    def handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _check(_native.lib().osc_ipc_export(ctypes.c_void_p(self.ptr), buf), "osc_ipc_export")
        return buf.raw

    def free(self):
        if self.ptr:
            self.tensor = None
            _check(_native.lib().osc_device_free(ctypes.c_void_p(self.ptr)), "osc_device_free")
            self.ptr = 0


def import_buffer(handle: bytes) -> int:
    """Map a neighbour's exported allocation; returns the device pointer."""
    p = ctypes.c_void_p()
    _check(_native.lib().osc_ipc_import(handle, ctypes.byref(p)), "osc_ipc_import")
    return p.value


def close_buffer(ptr: int):
    _check(_native.lib().osc_ipc_close(ctypes.c_void_p(ptr)), "osc_ipc_close")


class IpcEvent:
    """An interprocess CUDA event (created here or opened from a handle)."""

    def __init__(self, handle: bytes | None = None):
        lib = _native.lib()
        ev = ctypes.c_void_p()
        if handle is None:
            buf = ctypes.create_string_buffer(64)
            _check(lib.osc_ipc_event_create(ctypes.byref(ev), buf), "osc_ipc_event_create")
            self.handle = buf.raw
        else:
            _check(lib.osc_ipc_event_open(handle, ctypes.byref(ev)), "osc_ipc_event_open")
            self.handle = handle
        self.ev = ev.value

    def record(self, stream: torch.cuda.Stream):
        _check(_native.lib().osc_event_record(ctypes.c_void_p(self.ev),
                                              ctypes.c_void_p(stream.cuda_stream)),
               "osc_event_record")

    def wait(self, stream: torch.cuda.Stream):
        _check(_native.lib().osc_stream_wait_event(ctypes.c_void_p(stream.cuda_stream),
                                                   ctypes.c_void_p(self.ev)),
               "osc_stream_wait_event")

    def destroy(self):
        if self.ev:
            _check(_native.lib().osc_event_destroy(ctypes.c_void_p(self.ev)), "osc_event_destroy")
            self.ev = 0


def edge_sync_status(counters_ptr: int, stream: torch.cuda.Stream):
    """The timeout record of an edge-sync counter block after ``stream``'s
    work is done: None, or (period, side, value seen) of the wait that
    expired (osc_edge_sync_status)."""
    rec = (ctypes.c_uint64 * 4)()
    rc = _native.lib().osc_edge_sync_status(ctypes.c_void_p(counters_ptr), rec,
                                            ctypes.c_void_p(stream.cuda_stream))
    if rc == _native.OSC_OK:
        return None
    if rec[0] == 0:
        _check(rc, "osc_edge_sync_status")
    return int(rec[1]), int(rec[2]), int(rec[3])


def stream_write_u64(stream: torch.cuda.Stream, ptr: int, value: int):
    """Store value at ptr once all prior work of stream is done (fenced)."""
    _check(_native.lib().osc_stream_write_u64(ctypes.c_void_p(stream.cuda_stream),
                                              ctypes.c_void_p(ptr), int(value)),
           "osc_stream_write_u64")


def stream_wait_u64(stream: torch.cuda.Stream, ptr: int, value: int):
    """Hold later work of stream until *ptr >= value (GPU front-end wait)."""
    _check(_native.lib().osc_stream_wait_u64(ctypes.c_void_p(stream.cuda_stream),
                                             ctypes.c_void_p(ptr), int(value)),
           "osc_stream_wait_u64")
