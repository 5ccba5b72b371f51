"""ctypes binding of libpd_b200.so (include/pd_b200.h).

The product path has no CPU fallback: if the library is missing or cannot be
loaded, every call raises. Return codes map onto the reference's exception
types (PD_ERR_INVALID -> ValidationError, PD_ERR_TIMEOUT/DEADLOCK ->
SimulationError, PD_ERR_CUDA -> NativeError).
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_double, c_float, c_int, c_int32, c_int64, c_void_p
from pathlib import Path

from .errors import NativeError, SimulationError, ValidationError

# PD_LIB: an alternative in-tree build of the same library (A/B measurements of compile-time variants)
LIB_PATH = Path(os.environ.get("PD_LIB") or Path(__file__).resolve().parent / "libpd_b200.so")

PD_F32, PD_BF16 = 0, 1
EPI_STORE, EPI_LOSS, EPI_MASK, EPI_SGD, EPI_GRADF32, EPI_GELU, EPI_GELU_BWD, EPI_RESID = range(8)
ITEM_WIDTH = 20
(IT_OP, IT_STAGE, IT_MB, IT_WORKER, IT_VERSION, IT_WSLOT, IT_WNEW, IT_ACT, IT_XSLOT, IT_GSLOT, IT_OUT,
 IT_BLOCK, IT_DEP, IT_WAR, IT_RWAIT, IT_AWAIT, IT_DST, IT_SRC, IT_ROUND) = range(19)

# Symbols include/pd_b200.h declares; tests check every one is exported.
EXPORTED = (
    "pd_abi_version", "pd_last_error", "pd_device_sm_count", "pd_gemm", "pd_bias_sgd", "pd_sgd_update", "pd_cast", "pd_allreduce_sgd", "pd_bias_grad",
    "pd_flag_signal", "pd_flag_wait", "pd_copy", "pd_ipc_get_handle", "pd_ipc_open", "pd_ipc_close",
    "pd_enable_peer_access", "pd_rt_create", "pd_rt_add_stage", "pd_rt_add_view", "pd_rt_load_program", "pd_rt_run",
    "pd_rt_records", "pd_rt_set_records", "pd_gemm_pick", "pd_rt_set_serial", "pd_rt_set_graph", "pd_rt_layer_timing", "pd_rt_layer_stats", "pd_rt_kernel_timing", "pd_rt_kernel_stats", "pd_rt_launch_count", "pd_rt_destroy",
    "pd_conv3x3", "pd_splitk_plan", "pd_maxpool2", "pd_maxpool2_bwd", "pd_im2col3", "pd_reduce_sgd",
    "pd_colsum_blocks", "pd_bias_grad_tall", "pd_softmax_ce", "pd_memcpy_async", "pd_layer_scratch_floats",
    "pd_layer_save_bytes", "pd_layer_work_bytes", "pd_attention_fwd", "pd_attention_bwd", "pd_layernorm_fwd",
    "pd_layernorm_bwd_blocks", "pd_layernorm_bwd", "pd_embedding_fwd", "pd_embedding_bwd", "pd_softmax_ce_vocab",
)
PD_CONV_FWD, PD_CONV_DGRAD, PD_CONV_WGRAD, PD_GEMM_WGRAD_SPLITK = range(4)
# device pass records (pd_rt_set_records)
REC_WIDTH = 8
REC_T0, REC_T1, REC_VER0, REC_VER1, REC_BYTES, REC_COMMIT = range(6)


class Epilogue(Structure):
    _fields_ = [
        ("kind", c_int), ("out", c_void_p), ("ldo", c_int64), ("bias", c_void_p), ("relu", c_int),
        ("mask", c_void_p), ("ldm", c_int64), ("target", c_void_p), ("ldt", c_int64), ("scale", c_float),
        ("loss", c_void_p), ("master", c_void_p), ("ldw", c_int64), ("lr", c_float), ("aux", c_void_p),
    ]


PD_LAYER_LINEAR, PD_LAYER_CONV3, PD_LAYER_EMBED, PD_LAYER_BLOCK, PD_LAYER_HEAD = range(5)
PD_LOSS_MSE, PD_LOSS_CE = 0, 1


class LayerDesc(Structure):
    _fields_ = [
        ("kind", c_int), ("relu", c_int), ("pool", c_int), ("im2col", c_int), ("h", c_int), ("w", c_int),
        ("c_in", c_int), ("c_out", c_int), ("argmax", POINTER(c_void_p)), ("cols", POINTER(c_void_p)),
        ("ffn", c_int), ("vocab", c_int), ("save", POINTER(c_void_p)), ("work", c_void_p),
    ]


class StageDesc(Structure):
    _fields_ = [
        ("worker", c_int), ("stage", c_int), ("replica", c_int), ("rep", c_int), ("first_worker", c_int),
        ("n_layers", c_int), ("dims", POINTER(c_int64)), ("batch", c_int), ("dtype", c_int),
        ("is_first", c_int), ("is_last", c_int), ("relu_last", c_int), ("ring_depth", c_int), ("init_slot", c_int),
        ("act_depth", c_int), ("in_depth", c_int), ("grad_depth", c_int), ("n_data_blocks", c_int),
        ("remote_prev", c_int), ("remote_next", c_int), ("lr", c_float),
        ("w_master", POINTER(c_void_p)), ("b_master", POINTER(c_void_p)), ("w_ring", POINTER(c_void_p)),
        ("b_ring", POINTER(c_void_p)), ("act", POINTER(c_void_p)), ("act_in", POINTER(c_void_p)),
        ("grad_in", POINTER(c_void_p)), ("dz_last", POINTER(c_void_p)),
        ("target", POINTER(c_void_p)), ("loss", c_void_p), ("tmp", c_void_p * 2),
        ("act_ready", c_void_p), ("act_ack", c_void_p), ("grad_ready", c_void_p), ("grad_ack", c_void_p),
        ("red_grad", POINTER(c_void_p)), ("red_bgrad", POINTER(c_void_p)), ("red_ready", c_void_p),
        ("red_done", c_void_p), ("err_word", c_void_p),
        ("layers", POINTER(LayerDesc)), ("loss_kind", c_int), ("logits", c_void_p), ("part", c_void_p),
        ("sync", c_void_p), ("fused_bias", c_int), ("bpart", POINTER(c_void_p)), ("grad_bpart", POINTER(c_void_p)),
        ("dz_bpart", POINTER(c_void_p)), ("red_lready", c_void_p), ("red_lupd", c_void_p),
    ]


class WorkerView(Structure):
    _fields_ = [
        ("worker", c_int), ("remote", c_int), ("in_depth", c_int), ("grad_depth", c_int), ("n_layers", c_int),
        ("act_in", POINTER(c_void_p)), ("grad_in", POINTER(c_void_p)),
        ("act_ready", c_void_p), ("act_ack", c_void_p), ("grad_ready", c_void_p), ("grad_ack", c_void_p),
        ("red_grad", POINTER(c_void_p)), ("red_bgrad", POINTER(c_void_p)), ("red_ready", c_void_p),
        ("red_done", c_void_p), ("fused_bias", c_int), ("grad_bpart", POINTER(c_void_p)),
        ("w_master", POINTER(c_void_p)), ("b_master", POINTER(c_void_p)), ("red_lready", c_void_p),
        ("red_lupd", c_void_p),
    ]


class Record(Structure):
    _fields_ = [("item", c_int32), ("pad", c_int32), ("t_start_ms", c_double), ("t_end_ms", c_double)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libpd_b200.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)"
            )
        L = ctypes.CDLL(str(LIB_PATH))
        L.pd_last_error.restype = ctypes.c_char_p
        L.pd_gemm.argtypes = [c_int, c_void_p, c_int, c_int64, c_void_p, c_int, c_int64, c_int, c_int, c_int,
                              POINTER(Epilogue), c_void_p]
        L.pd_bias_sgd.argtypes = [c_int, c_void_p, c_int, c_int, c_int64, c_void_p, c_void_p, c_float, c_void_p]
        L.pd_sgd_update.argtypes = [c_int, c_void_p, c_void_p, c_void_p, c_int64, c_float, c_void_p]
        L.pd_cast.argtypes = [c_int, c_void_p, c_void_p, c_int64, c_void_p]
        L.pd_flag_signal.argtypes = [c_void_p, c_int, c_void_p]
        L.pd_copy.argtypes = [c_void_p, c_void_p, c_int64, c_void_p]
        L.pd_flag_wait.argtypes = [c_void_p, c_int, c_void_p, c_void_p]
        L.pd_ipc_get_handle.argtypes = [c_void_p, c_void_p, POINTER(c_int64)]
        L.pd_ipc_open.argtypes = [c_void_p, POINTER(c_void_p)]
        L.pd_ipc_close.argtypes = [c_void_p]
        L.pd_rt_create.argtypes = [c_int, POINTER(c_void_p)]
        L.pd_rt_add_stage.argtypes = [c_void_p, POINTER(StageDesc)]
        L.pd_rt_add_view.argtypes = [c_void_p, POINTER(WorkerView)]
        L.pd_allreduce_sgd.argtypes = [c_int, POINTER(c_void_p), c_int, c_void_p, c_void_p, c_int64, c_float, c_void_p]
        L.pd_bias_grad.argtypes = [c_int, c_void_p, c_int, c_int, c_int64, c_void_p, c_void_p]
        L.pd_rt_load_program.argtypes = [c_void_p, POINTER(c_int32), c_int]
        L.pd_rt_run.argtypes = [c_void_p, c_void_p, c_int]
        L.pd_rt_records.argtypes = [c_void_p, POINTER(Record), c_int, POINTER(c_int)]
        L.pd_rt_set_records.argtypes = [c_void_p, c_void_p, c_int, c_void_p]
        L.pd_gemm_pick.argtypes = [c_int, c_int, c_int, c_int, c_int, c_int, POINTER(c_int), POINTER(c_int)]
        L.pd_rt_destroy.argtypes = [c_void_p]
        L.pd_rt_kernel_timing.argtypes = [c_void_p, c_int]
        L.pd_rt_set_serial.argtypes = [c_void_p, c_int]
        L.pd_rt_set_graph.argtypes = [c_void_p, c_int]
        L.pd_rt_layer_timing.argtypes = [c_void_p, c_void_p, c_int]
        L.pd_rt_layer_stats.argtypes = [c_void_p, c_int, c_int, POINTER(c_double)]
        L.pd_rt_kernel_stats.argtypes = [c_void_p, c_int, POINTER(c_double), c_int]
        L.pd_rt_launch_count.argtypes = [c_void_p, POINTER(c_int64)]
        L.pd_device_sm_count.argtypes = [c_int, POINTER(c_int)]
        L.pd_conv3x3.argtypes = [c_int, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, POINTER(Epilogue),
                                 c_void_p]
        L.pd_splitk_plan.argtypes = [c_int, c_int, c_int, POINTER(c_int)]
        L.pd_maxpool2.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p]
        L.pd_maxpool2_bwd.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p]
        L.pd_im2col3.argtypes = [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p]
        L.pd_reduce_sgd.argtypes = [c_int, c_void_p, c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_float,
                                    c_void_p]
        L.pd_colsum_blocks.argtypes = [c_int64, c_int]
        L.pd_bias_grad_tall.argtypes = [c_void_p, c_int64, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_float,
                                        c_void_p]
        L.pd_softmax_ce.argtypes = [c_void_p, c_int64, c_void_p, c_int, c_int, c_void_p, c_int64, c_void_p, c_void_p]
        L.pd_memcpy_async.argtypes = [c_void_p, c_void_p, c_int64, c_void_p]
        L.pd_layer_scratch_floats.argtypes = [POINTER(LayerDesc), c_int]
        L.pd_layer_scratch_floats.restype = c_int64
        for fn in ("pd_layer_save_bytes", "pd_layer_work_bytes"):
            getattr(L, fn).argtypes = [POINTER(LayerDesc), c_int]
            getattr(L, fn).restype = c_int64
        L.pd_attention_fwd.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p]
        L.pd_attention_bwd.argtypes = [c_void_p] * 7 + [c_int, c_int, c_int, c_void_p]
        L.pd_layernorm_fwd.argtypes = [c_void_p] * 5 + [c_int64, c_int, c_void_p]
        L.pd_layernorm_bwd_blocks.argtypes = [c_int64]
        L.pd_layernorm_bwd.argtypes = [c_void_p] * 8 + [c_int64, c_int, c_void_p]
        L.pd_embedding_fwd.argtypes = [c_void_p] * 4 + [c_int64, c_int, c_int, c_void_p]
        L.pd_embedding_bwd.argtypes = [c_void_p] * 4 + [c_int64, c_int, c_int, c_void_p]
        L.pd_softmax_ce_vocab.argtypes = [c_void_p, c_int64, c_void_p, c_int64, c_int, c_int, c_void_p, c_int64,
                                          c_void_p, c_void_p]
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = lib().pd_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == 1:
        raise ValidationError(text)
    if rc in (3, 4):
        raise SimulationError(text)
    raise NativeError(text)


def ptr(t) -> int:
    """Raw device address of a torch tensor (or 0 for None)."""
    return 0 if t is None else int(t.data_ptr())


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def dtype_code(torch_dtype) -> int:
    import torch

    if torch_dtype == torch.float32:
        return PD_F32
    if torch_dtype == torch.bfloat16:
        return PD_BF16
    raise ValidationError(f"unsupported dtype {torch_dtype}")


def gemm(A, a_mn: bool, B, b_mn: bool, M: int, N: int, K: int, *, kind: int = EPI_STORE, out=None, ldo=None,
         bias=None, relu=False, mask=None, ldm=None, target=None, ldt=None, scale=1.0, loss=None, master=None,
         ldw=None, lr=0.0, aux=None, stream=None) -> None:
    """C[M,N] = sum_k A(m,k) B(n,k) + fused epilogue, on torch tensors (row-major, contiguous rows).
    aux: EPI_GELU's pre-activation output (ld = ldo)."""
    lda = A.stride(0)
    ldb = B.stride(0)
    ep = Epilogue(kind=kind, out=ptr(out), ldo=ldo if ldo is not None else (out.stride(0) if out is not None else 0),
                  bias=ptr(bias), relu=int(bool(relu)), mask=ptr(mask),
                  ldm=ldm if ldm is not None else (mask.stride(0) if mask is not None else 0),
                  target=ptr(target), ldt=ldt if ldt is not None else (target.stride(0) if target is not None else 0),
                  scale=scale, loss=ptr(loss), master=ptr(master),
                  ldw=ldw if ldw is not None else (master.stride(0) if master is not None else 0), lr=lr,
                  aux=ptr(aux))
    check(lib().pd_gemm(dtype_code(A.dtype), ptr(A), int(a_mn), lda, ptr(B), int(b_mn), ldb, M, N, K,
                        ctypes.byref(ep), stream_ptr(stream)), "pd_gemm")


def gemm_pick(M: int, N: int, K: int, a_mn: bool, b_mn: bool, kind: int) -> tuple[int, int]:
    """(CTA group, tile width) the tcgen05 dispatch picks for this problem (gemm.cu choose_cfg)."""
    cg, bn = c_int(0), c_int(0)
    check(lib().pd_gemm_pick(M, N, K, int(a_mn), int(b_mn), kind, ctypes.byref(cg), ctypes.byref(bn)), "pd_gemm_pick")
    return int(cg.value), int(bn.value)


def bias_sgd(dz, rows: int, cols: int, b_master, b_out, lr: float, stream=None) -> None:
    check(lib().pd_bias_sgd(dtype_code(dz.dtype), ptr(dz), rows, cols, dz.stride(0), ptr(b_master), ptr(b_out),
                            lr, stream_ptr(stream)), "pd_bias_sgd")


def sgd_update(master, grad, out, lr: float, stream=None) -> None:
    check(lib().pd_sgd_update(dtype_code(out.dtype), ptr(master), ptr(grad), ptr(out), master.numel(), lr,
                              stream_ptr(stream)), "pd_sgd_update")


def ipc_export(t) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of t's allocation, byte offset of t inside it)."""
    h = (ctypes.c_char * 64)()
    off = ctypes.c_int64(0)
    check(lib().pd_ipc_get_handle(ptr(t), h, ctypes.byref(off)), "pd_ipc_get_handle")
    return bytes(h), int(off.value)


_ipc_bases: dict = {}


def ipc_import(handle: bytes, offset: int) -> int:
    """Device address in this process of an exported (handle, offset); allocations opened once."""
    base = _ipc_bases.get(handle)
    if base is None:
        out = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(handle, 64)
        check(lib().pd_ipc_open(buf, ctypes.byref(out)), "pd_ipc_open")
        base = _ipc_bases[handle] = int(out.value)
    return base + offset


def _epi(kind, out=None, ldo=0, bias=None, relu=False, mask=None, ldm=0, loss=None, master=None, ldw=0, lr=0.0):
    return Epilogue(kind=kind, out=ptr(out), ldo=ldo, bias=ptr(bias), relu=int(bool(relu)), mask=ptr(mask), ldm=ldm,
                    target=0, ldt=0, scale=1.0, loss=ptr(loss), master=ptr(master), ldw=ldw, lr=lr)


def splitk_plan(M: int, N: int, K: int) -> int:
    s = c_int(0)
    check(lib().pd_splitk_plan(M, N, K, ctypes.byref(s)), "pd_splitk_plan")
    return int(s.value)


def conv3x3(pass_: int, act, other, n: int, h: int, w: int, c_in: int, c_out: int, *, out, bias=None,
            relu=False, mask=None, stream=None) -> None:
    """One implicit-GEMM 3x3 convolution pass (include/pd_b200.h PD_CONV_*) on torch tensors."""
    if pass_ == PD_CONV_FWD:
        ep = _epi(EPI_STORE, out, c_out, bias=bias, relu=relu)
    elif pass_ == PD_CONV_DGRAD:
        ep = _epi(EPI_MASK, out, c_in, mask=mask, ldm=c_in)
    else:
        ep = _epi(EPI_GRADF32, out, c_out)
    check(lib().pd_conv3x3(pass_, ptr(act), ptr(other), n, h, w, c_in, c_out, ctypes.byref(ep),
                           stream_ptr(stream)), "pd_conv3x3")
