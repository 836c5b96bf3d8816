"""ctypes binding of ``libfcpb.so`` (the C ABI declared in ``include/fcpb.h``).

This is the only way the package reaches the GPU kernels.  There is no CPU
or PyTorch fallback: if the library is missing, or the device is not sm_100,
every entry point raises ``NativeError``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import NativeError, ParameterError

# FCPB_LIB: A/B experiments against another build of the same ABI (scripts/); default in-tree.
_LIB_PATH = os.environ.get("FCPB_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfcpb.so")

c_i32, c_i64, c_f32, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p


class FwdArgs(ctypes.Structure):
    _fields_ = [("num_q_heads", c_i32), ("num_kv_heads", c_i32), ("head_dim", c_i32),
                ("softmax_scale", c_f32),
                ("q", c_vp), ("q_tokens", c_i64),
                ("k", c_vp), ("v", c_vp), ("kv_tokens", c_i64),
                ("k_recv", c_vp), ("v_recv", c_vp), ("kv_recv_tokens", c_i64),
                ("o", c_vp), ("lse", c_vp),
                ("o_partial", c_vp), ("lse_partial", c_vp), ("partial_rows", c_i64),
                ("segments", c_vp), ("num_segments", c_i32),
                ("kv_refs", c_vp), ("num_kv_refs", c_i32),
                ("items", c_vp), ("num_items", c_i32),
                ("num_ctas", c_i32), ("head_major", c_i32), ("hm_lead", c_i32), ("sched_counter", c_vp)]


class MergeArgs(ctypes.Structure):
    _fields_ = [("num_q_heads", c_i32), ("head_dim", c_i32),
                ("o_partial", c_vp), ("lse_partial", c_vp),
                ("groups", c_vp), ("num_groups", c_i32),
                ("part_rows", c_vp), ("merged_tokens", c_i64),
                ("o", c_vp), ("lse", c_vp)]


class BwdArgs(ctypes.Structure):
    _fields_ = [("num_q_heads", c_i32), ("num_kv_heads", c_i32), ("head_dim", c_i32),
                ("softmax_scale", c_f32),
                ("q", c_vp), ("dout", c_vp),
                ("lse2_t", c_vp), ("delta_t", c_vp), ("t_pad", c_i64), ("q_tokens", c_i64),
                ("k", c_vp), ("v", c_vp), ("kv_tokens", c_i64),
                ("k_recv", c_vp), ("v_recv", c_vp), ("kv_recv_tokens", c_i64),
                ("dq_accum", c_vp), ("dk_accum", c_vp), ("dv_accum", c_vp),
                ("dk_recv_accum", c_vp), ("dv_recv_accum", c_vp), ("dk_out", c_vp), ("dv_out", c_vp),
                ("ds_out", c_vp), ("pair_base", c_vp),
                ("kvsegs", c_vp), ("num_kvsegs", c_i32),
                ("qrefs", c_vp), ("num_qrefs", c_i32),
                ("items", c_vp), ("num_items", c_i32),
                ("num_ctas", c_i32), ("head_major", c_i32), ("hm_lead", c_i32), ("sched_counter", c_vp)]


class DqArgs(ctypes.Structure):
    _fields_ = [("num_q_heads", c_i32), ("num_kv_heads", c_i32), ("head_dim", c_i32),
                ("softmax_scale", c_f32),
                ("q", c_vp), ("dout", c_vp),
                ("lse2_t", c_vp), ("delta_t", c_vp), ("t_pad", c_i64), ("q_tokens", c_i64),
                ("k", c_vp), ("v", c_vp), ("kv_tokens", c_i64),
                ("k_recv", c_vp), ("v_recv", c_vp), ("kv_recv_tokens", c_i64),
                ("dq", c_vp),
                ("segments", c_vp), ("num_segments", c_i32),
                ("kv_refs", c_vp), ("num_kv_refs", c_i32),
                ("items", c_vp), ("num_items", c_i32),
                ("num_ctas", c_i32), ("head_major", c_i32), ("hm_lead", c_i32), ("sched_counter", c_vp)]


class DqDsArgs(ctypes.Structure):
    _fields_ = [("num_q_heads", c_i32), ("num_kv_heads", c_i32), ("head_dim", c_i32),
                ("softmax_scale", c_f32),
                ("ds", c_vp), ("ds_tiles", c_i64),
                ("k", c_vp), ("kv_tokens", c_i64),
                ("k_recv", c_vp), ("kv_recv_tokens", c_i64),
                ("dq", c_vp),
                ("segments", c_vp), ("num_segments", c_i32),
                ("kv_refs", c_vp), ("num_kv_refs", c_i32),
                ("items", c_vp), ("num_items", c_i32),
                ("pair_ids", c_vp), ("pair_off", c_vp),
                ("num_ctas", c_i32), ("head_major", c_i32), ("hm_lead", c_i32), ("sched_counter", c_vp)]


EXPORTS = ("fcpb_attn_fwd", "fcpb_attn_bwd", "fcpb_attn_bwd_dq", "fcpb_attn_bwd_dq_ds",
           "fcpb_lse_merge", "fcpb_bwd_preprocess",
           "fcpb_f32_to_bf16", "fcpb_dkv_reduce", "fcpb_dkv_finalize", "fcpb_stream_signal", "fcpb_stream_wait",
           "fcpb_last_error", "fcpb_version", "fcpb_device_supported",
           "fcpb_bwd_preprocess_bytes", "fcpb_fwd_partial_bytes", "fcpb_ds_tile_bytes",
           "fcpb_debug_counters", "fcpb_ipc_alloc", "fcpb_ipc_open", "fcpb_ipc_close", "fcpb_ipc_free",
           "fcpb_copy_2d", "fcpb_gather_copy", "fcpb_gather_copy_based", "fcpb_gather_seg_bytes")
_SIZE_T = ("fcpb_bwd_preprocess_bytes", "fcpb_fwd_partial_bytes", "fcpb_ds_tile_bytes")
_I64 = ("fcpb_gather_seg_bytes",)

_lib = None


def load(path: str | None = None):
    """Load (once) and type the shared library; raises NativeError if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or _LIB_PATH
    if not os.path.exists(p):
        raise NativeError(f"{p} not built: run `make` (or __graft_entry__.build())")
    lib = ctypes.CDLL(p)
    lib.fcpb_attn_fwd.argtypes = [ctypes.POINTER(FwdArgs), c_vp]
    lib.fcpb_attn_bwd.argtypes = [ctypes.POINTER(BwdArgs), c_vp]
    lib.fcpb_attn_bwd_dq.argtypes = [ctypes.POINTER(DqArgs), c_vp]
    lib.fcpb_attn_bwd_dq_ds.argtypes = [ctypes.POINTER(DqDsArgs), c_vp]
    lib.fcpb_lse_merge.argtypes = [ctypes.POINTER(MergeArgs), c_vp]
    lib.fcpb_bwd_preprocess.argtypes = [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_i32,
                                         c_i32, c_vp]
    lib.fcpb_f32_to_bf16.argtypes = [c_vp, c_vp, c_i64, c_vp]
    lib.fcpb_dkv_reduce.argtypes = [c_vp, c_vp, c_vp, c_i64, c_i64, c_vp]
    lib.fcpb_dkv_finalize.argtypes = [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp]
    lib.fcpb_stream_signal.argtypes = [c_vp, ctypes.c_uint32, c_vp]
    lib.fcpb_stream_wait.argtypes = [c_vp, ctypes.c_uint32, c_vp]
    lib.fcpb_last_error.restype = ctypes.c_char_p
    lib.fcpb_device_supported.argtypes = [ctypes.c_int]
    lib.fcpb_bwd_preprocess_bytes.argtypes = [c_i64, c_i32]
    lib.fcpb_fwd_partial_bytes.argtypes = [c_i64, c_i32, c_i32]
    lib.fcpb_ds_tile_bytes.argtypes = [c_i64, c_i32]
    lib.fcpb_ipc_alloc.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.POINTER(c_vp), ctypes.c_char_p]
    lib.fcpb_ipc_open.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(c_vp)]
    lib.fcpb_ipc_close.argtypes = [ctypes.c_int, c_vp]
    lib.fcpb_ipc_free.argtypes = [ctypes.c_int, c_vp]
    lib.fcpb_copy_2d.argtypes = [c_vp, ctypes.c_size_t, c_vp, ctypes.c_size_t, ctypes.c_size_t,
                                 ctypes.c_size_t, c_vp]
    lib.fcpb_debug_counters.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int, ctypes.c_int]
    lib.fcpb_gather_copy.argtypes = [c_vp, c_i32, c_i32, c_vp]
    lib.fcpb_gather_copy_based.argtypes = [c_vp, c_i32, ctypes.POINTER(ctypes.c_uint64), c_i32, c_i32, c_vp]
    lib.fcpb_gather_seg_bytes.argtypes = []
    for name in EXPORTS:
        getattr(lib, name).restype = (ctypes.c_char_p if name == "fcpb_last_error" else
                                      ctypes.c_size_t if name in _SIZE_T else
                                      ctypes.c_int64 if name in _I64 else ctypes.c_int)
    if path is None:
        _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = load().fcpb_last_error().decode(errors="replace")
    if rc == -1:
        raise ParameterError(msg)
    raise NativeError(f"libfcpb status {rc}: {msg}")


def ptr(t) -> int:
    """Device pointer of a torch tensor, or 0 for None."""
    return 0 if t is None else t.data_ptr()


def stream_handle(stream) -> int:
    return stream.cuda_stream if stream is not None else 0


def copy_2d(dst: int, dpitch: int, src: int, spitch: int, width: int, height: int, stream) -> None:
    """Device-to-device 2-D copy on `stream` (one copy-engine operation)."""
    check(load().fcpb_copy_2d(dst, dpitch, src, spitch, width, height, stream_handle(stream)))


def gather_copy(segs, num_ctas: int, stream) -> None:
    """K5 pull kernel: segs is a device int64 tensor [n, 3] of (dst, src, bytes) ranges
    (``fcpb_gather_copy``), copied by SM loads on `num_ctas` CTAs, ordered on `stream`."""
    if str(segs.dtype) != "torch.int64" or segs.dim() != 2 or segs.shape[1] != 3 or not segs.is_cuda:
        raise ParameterError("gather_copy: segs must be a CUDA int64 tensor [n, 3]")
    check(load().fcpb_gather_copy(segs.data_ptr(), segs.shape[0], num_ctas, stream_handle(stream)))


def gather_copy_based(segs, bases, num_ctas: int, stream) -> None:
    """K5 pull kernel over base-relative segments (``fcpb_gather_copy_based``): segs is a
    device int64 tensor [n, 3] of ((base << 56) | offset, (base << 56) | offset, bytes), bases a
    list of at most 32 addresses passed by value."""
    if str(segs.dtype) != "torch.int64" or segs.dim() != 2 or segs.shape[1] != 3 or not segs.is_cuda:
        raise ParameterError("gather_copy_based: segs must be a CUDA int64 tensor [n, 3]")
    if len(bases) > 32:
        raise ParameterError("gather_copy_based: at most 32 bases")
    arr = (ctypes.c_uint64 * max(len(bases), 1))(*bases)
    check(load().fcpb_gather_copy_based(segs.data_ptr(), segs.shape[0], arr, len(bases), num_ctas,
                                        stream_handle(stream)))


def gather_seg_bytes() -> int:
    """Largest byte range one fcpb_gather_copy segment may cover."""
    return int(load().fcpb_gather_seg_bytes())


def stream_signal(flag_addr: int, value: int, stream) -> None:
    """Write `value` to a (peer-mapped) 32-bit flag after the stream's prior work."""
    check(load().fcpb_stream_signal(flag_addr, value & 0xFFFFFFFF, stream_handle(stream)))


def stream_wait(flag_addr: int, value: int, stream) -> None:
    """Later work on `stream` waits until the local 32-bit flag reaches `value`."""
    check(load().fcpb_stream_wait(flag_addr, value & 0xFFFFFFFF, stream_handle(stream)))


def fwd_rescale_events(reset: bool = True) -> int:
    """Test hook (synchronous): warp-level lazy O-rescale events of the forward kernel since
    the last reset (``fcpb_debug_counters``)."""
    out = (ctypes.c_uint64 * 1)()
    check(load().fcpb_debug_counters(out, 1, 1 if reset else 0))
    return int(out[0])
