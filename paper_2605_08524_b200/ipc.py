"""Peer-memory regions for the K5/K6 transport (``fcpb_ipc_*`` in ``include/fcpb.h``).

A region is device memory allocated by ``libfcpb.so`` together with its CUDA IPC handle.
``exchange`` all-gathers the handles over the process group (any backend: gloo works, the
handles are 64 bytes) and opens every peer's region, so each rank can read its peers'
buffers with copy-engine memcpys -- across the GPUs of one NVSwitch box, and equally between
processes that share one GPU (which is how the multi-rank executor is tested on a one-GPU
box).  Views are torch tensors over the raw pointers (``__cuda_array_interface__``, no copy).
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import native

_HANDLE_BYTES = 64


class _CudaArray:
    """Minimal ``__cuda_array_interface__`` exporter; keeps its region alive."""

    def __init__(self, ptr: int, shape, typestr: str, owner):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 2}
        self._owner = owner


_TYPESTR = {torch.float32: "<f4", torch.int32: "<i4", torch.uint8: "|u1", torch.int16: "<i2"}


class Region:
    """A device buffer (own or a peer's, opened through IPC)."""

    def __init__(self, ptr: int, nbytes: int, device: torch.device, owned: bool, opened: bool):
        self.ptr, self.nbytes, self.device = ptr, nbytes, device
        self._owned, self._opened = owned, opened

    def tensor(self, dtype, shape, byte_offset: int = 0) -> torch.Tensor:
        """A torch view of the region (bf16 is exported as int16 and reinterpreted)."""
        numel = 1
        for d in shape:
            numel *= d
        esz = torch.empty((), dtype=dtype).element_size()
        if byte_offset + numel * esz > self.nbytes:
            raise ValueError("view exceeds the region")
        base = dtype if dtype in _TYPESTR else {2: torch.int16, 4: torch.int32, 1: torch.uint8}[esz]
        arr = _CudaArray(self.ptr + byte_offset, shape, _TYPESTR[base], self)
        with torch.cuda.device(self.device):
            t = torch.as_tensor(arr, device=self.device)
        return t if base is dtype else t.view(dtype)

    def close(self):
        lib = native.load()
        if self._opened and self.ptr:
            native.check(lib.fcpb_ipc_close(self.device.index, ctypes.c_void_p(self.ptr)))
        elif self._owned and self.ptr:
            native.check(lib.fcpb_ipc_free(self.device.index, ctypes.c_void_p(self.ptr)))
        self.ptr = 0


class IpcRegion(Region):
    """This rank's region: allocated zero-filled, with an IPC handle for the peers."""

    def __init__(self, nbytes: int, device):
        device = torch.device(device)
        lib = native.load()
        ptr = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(_HANDLE_BYTES)
        native.check(lib.fcpb_ipc_alloc(device.index, max(int(nbytes), 1), ctypes.byref(ptr), handle))
        super().__init__(ptr.value, int(nbytes), device, owned=True, opened=False)
        self.handle = handle.raw

    def exchange(self, group=None) -> list[Region]:
        """All-gather the handles and open every peer's region; entry ``rank`` is this
        region itself.  Collective over ``group``."""
        group = group or dist.group.WORLD
        world, me = dist.get_world_size(group), dist.get_rank(group)
        got = [None] * world
        dist.all_gather_object(got, (self.handle, self.nbytes), group=group)
        lib = native.load()
        out: list[Region] = []
        for r, (h, nb) in enumerate(got):
            if r == me:
                out.append(self)
                continue
            ptr = ctypes.c_void_p()
            native.check(lib.fcpb_ipc_open(self.device.index, h, ctypes.byref(ptr)))
            out.append(Region(ptr.value, nb, self.device, owned=False, opened=True))
        return out
