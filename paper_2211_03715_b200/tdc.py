"""Thin ctypes binding of the libtdc.so C-ABI (include/tdc.h).

Argument marshalling only: every step of the TKD layer runs in the CUDA
kernels behind the ABI.  There is no CPU fallback -- if the library is
missing, importing this module raises.  Function names mirror the C names.
torch is used only to hand over device pointers and streams.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TDC_LIB") or os.path.join(HERE, "libtdc.so")

TDC_OK, TDC_ERR_INVALID_ARGUMENT, TDC_ERR_UNSUPPORTED, TDC_ERR_CUDA, \
    TDC_ERR_OUT_OF_MEMORY, TDC_ERR_INTERNAL = range(6)
TDC_LAYOUT_NCHW, TDC_LAYOUT_NHWC = 0, 1
TDC_MATH_FP32, TDC_MATH_3XTF32, TDC_MATH_TF32, TDC_MATH_3XBF16 = 0, 1, 2, 3
MATH_NAMES = {"fp32": TDC_MATH_FP32, "3xtf32": TDC_MATH_3XTF32, "tf32": TDC_MATH_TF32,
              "3xbf16": TDC_MATH_3XBF16}

# Every symbol include/tdc.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "tdc_version", "tdc_status_string", "tdc_last_error", "tdc_conv_output_shape",
    "tdc_conv_plan", "tdc_conv_plan_query", "tdc_conv_forward", "tdc_conv_forward_host",
    "tdc_conv_plan_destroy", "tdc_conv_forward_ex", "tdc_model_create", "tdc_model_forward",
    "tdc_model_output_shape", "tdc_model_destroy", "tdc_conv_plan_ex", "tdc_conv_forward_host_many",
]
TDC_OP_CONV, TDC_OP_TKD, TDC_OP_MAXPOOL, TDC_OP_AVGPOOL, TDC_OP_FC = range(5)


class tdc_conv_desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "batch", "c_in", "height", "width", "c_out", "rank_in", "rank_out", "kernel",
        "stride", "pad", "layout", "math")]


class tdc_plan_info(ctypes.Structure):
    _fields_ = [("h_out", ctypes.c_int32), ("w_out", ctypes.c_int32),
                ("variant", ctypes.c_int32), ("variant_name", ctypes.c_char * 48),
                ("launches_per_forward", ctypes.c_int32), ("concurrent_forward", ctypes.c_int32),
                ("tile_h", ctypes.c_int32), ("tile_w", ctypes.c_int32),
                ("threads_per_cta", ctypes.c_int32), ("smem_bytes_per_cta", ctypes.c_int32),
                ("ctas_per_image", ctypes.c_int64), ("workspace_bytes", ctypes.c_int64),
                ("weight_bytes", ctypes.c_int64)] + [(n, ctypes.c_int32) for n in (
                    "bn_stage1", "bn_core", "bn_stage3", "ksplit_stage1", "ksplit_core", "ksplit_stage3",
                    "core3", "gsplit_stage1", "gsplit_core", "gsplit_stage3")]


HINT_FIELDS = ("core3", "bn_stage1", "bn_core", "bn_stage3", "ksplit_stage1", "ksplit_core", "ksplit_stage3",
               "gsplit_stage1", "gsplit_core", "gsplit_stage3", "fused_layer")


class tdc_plan_hints(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in HINT_FIELDS]


class tdc_model_op(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "kind", "src", "res", "c_in", "c_out", "height", "width", "kernel", "stride", "pad",
        "rank_in", "rank_out", "relu")] + [
        (n, ctypes.POINTER(ctypes.c_float)) for n in ("w", "u_in", "u_out", "bias", "bn")]


class TdcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"tdc status {status}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    fp = ctypes.POINTER(ctypes.c_float)
    vp = ctypes.c_void_p
    i32 = ctypes.c_int32
    desc_p = ctypes.POINTER(tdc_conv_desc)
    lib.tdc_version.restype = ctypes.c_char_p
    lib.tdc_status_string.restype = ctypes.c_char_p
    lib.tdc_status_string.argtypes = [ctypes.c_int]
    lib.tdc_last_error.restype = ctypes.c_char_p
    lib.tdc_conv_output_shape.argtypes = [desc_p, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    lib.tdc_conv_plan.argtypes = [desc_p, fp, fp, fp, fp, i32, ctypes.POINTER(vp)]
    lib.tdc_conv_plan_query.argtypes = [vp, ctypes.POINTER(tdc_plan_info)]
    lib.tdc_conv_forward.argtypes = [vp, vp, vp, i32, vp]
    lib.tdc_conv_forward_host.argtypes = [vp, vp, vp, i32, vp]
    lib.tdc_conv_forward_host_many.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                               ctypes.POINTER(i32), i32, vp]
    lib.tdc_conv_plan_destroy.argtypes = [vp]
    lib.tdc_conv_forward_ex.argtypes = [vp, vp, vp, i32, vp, i32, vp]
    lib.tdc_conv_plan_ex.argtypes = [desc_p, fp, fp, fp, fp, ctypes.POINTER(tdc_plan_hints), i32,
                                     ctypes.POINTER(vp)]
    lib.tdc_model_create.argtypes = [ctypes.POINTER(tdc_model_op), i32, i32, i32, ctypes.POINTER(vp)]
    lib.tdc_model_forward.argtypes = [vp, vp, i32, vp, vp]
    lib.tdc_model_output_shape.argtypes = [vp, i32, ctypes.POINTER(i32), ctypes.POINTER(i32),
                                           ctypes.POINTER(i32)]
    lib.tdc_model_destroy.argtypes = [vp]
    for name in EXPORTED:
        getattr(lib, name).restype = getattr(lib, name).restype or ctypes.c_int
    return lib


_lib = _load()
lib = _lib


def _check(status: int):
    if status != TDC_OK:
        raise TdcError(status, _lib.tdc_last_error().decode())


def tdc_version() -> str:
    return _lib.tdc_version().decode()


def tdc_status_string(status: int) -> str:
    return _lib.tdc_status_string(status).decode()


def tdc_last_error() -> str:
    return _lib.tdc_last_error().decode()


def make_desc(B, C, H, W, N, D1, D2, K=3, stride=1, pad=1, layout=TDC_LAYOUT_NHWC,
              math=TDC_MATH_FP32) -> tdc_conv_desc:
    return tdc_conv_desc(B, C, H, W, N, D1, D2, K, stride, pad, layout, math)


def tdc_conv_output_shape(desc: tdc_conv_desc):
    h, w = ctypes.c_int32(), ctypes.c_int32()
    _check(_lib.tdc_conv_output_shape(ctypes.byref(desc), ctypes.byref(h), ctypes.byref(w)))
    return h.value, w.value


def _fptr(a):
    """Host fp32 numpy array -> float*; None -> NULL."""
    if a is None:
        return None
    import numpy as np
    if not (isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags.c_contiguous):
        raise TypeError("weights must be C-contiguous float32 numpy arrays")
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def tdc_conv_plan(desc: tdc_conv_desc, core, u_in, u_out, bias=None, device: int = 0):
    h = ctypes.c_void_p()
    _check(_lib.tdc_conv_plan(ctypes.byref(desc), _fptr(core), _fptr(u_in), _fptr(u_out),
                              _fptr(bias), device, ctypes.byref(h)))
    return h


def make_hints(**kw) -> tdc_plan_hints:
    """Planner overrides; unspecified fields = the planner's own choice."""
    h = tdc_plan_hints(core3=-1, fused_layer=-1)
    for k, v in kw.items():
        if k not in HINT_FIELDS:
            raise KeyError(k)
        setattr(h, k, int(v))
    return h


def tdc_conv_plan_ex(desc: tdc_conv_desc, core, u_in, u_out, bias=None, hints=None, device: int = 0):
    h = ctypes.c_void_p()
    _check(_lib.tdc_conv_plan_ex(ctypes.byref(desc), _fptr(core), _fptr(u_in), _fptr(u_out), _fptr(bias),
                                 ctypes.byref(hints) if hints is not None else None, device, ctypes.byref(h)))
    return h


def tdc_conv_plan_query(plan) -> tdc_plan_info:
    info = tdc_plan_info()
    _check(_lib.tdc_conv_plan_query(plan, ctypes.byref(info)))
    return info


def tdc_conv_forward(plan, x_ptr: int, y_ptr: int, batch: int, stream: int = 0) -> None:
    _check(_lib.tdc_conv_forward(plan, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr),
                                 batch, ctypes.c_void_p(stream)))


def tdc_conv_forward_host(plan, x_host_ptr: int, y_host_ptr: int, batch: int,
                          stream: int = 0) -> None:
    _check(_lib.tdc_conv_forward_host(plan, ctypes.c_void_p(x_host_ptr),
                                      ctypes.c_void_p(y_host_ptr), batch,
                                      ctypes.c_void_p(stream)))


def tdc_conv_forward_host_many(plans, x_host_ptrs, y_host_ptrs, batches, stream: int = 0) -> None:
    n = len(plans)
    vp = ctypes.c_void_p
    _check(_lib.tdc_conv_forward_host_many((vp * n)(*plans), (vp * n)(*x_host_ptrs), (vp * n)(*y_host_ptrs),
                                           (ctypes.c_int32 * n)(*batches), n, vp(stream)))


def forward_host_many(plans, xs, ys, stream=None) -> None:
    """n end-to-end forwards (ConvPlan objects, pinned host tensors) as one pipeline."""
    sh = ConvPlan._stream_handle(stream)
    tdc_conv_forward_host_many([p._h for p in plans], [x.data_ptr() for x in xs], [y.data_ptr() for y in ys],
                               [int(x.shape[0]) for x in xs], sh)


def tdc_conv_plan_destroy(plan) -> None:
    _check(_lib.tdc_conv_plan_destroy(plan))


@dataclass
class PlanInfo:
    h_out: int
    w_out: int
    variant: int
    variant_name: str
    launches_per_forward: int
    concurrent_forward: int
    tile_h: int
    tile_w: int
    threads_per_cta: int
    smem_bytes_per_cta: int
    ctas_per_image: int
    workspace_bytes: int
    weight_bytes: int
    bn_stage1: int = 0
    bn_core: int = 0
    bn_stage3: int = 0
    ksplit_stage1: int = 0
    ksplit_core: int = 0
    ksplit_stage3: int = 0
    core3: int = 0
    gsplit_stage1: int = 1
    gsplit_core: int = 1
    gsplit_stage3: int = 1


class ConvPlan:
    """RAII wrapper: a planned TKD layer on one device.

    ``forward(x, y, stream)`` takes torch CUDA tensors (device memory only) and
    enqueues the kernels on ``stream`` (a torch.cuda.Stream or raw handle)."""

    def __init__(self, shape, weights: dict, layout: int = TDC_LAYOUT_NHWC,
                 math: int = TDC_MATH_FP32, device: int = 0, hints: dict | None = None):
        self.shape = shape
        self.desc = make_desc(shape.B, shape.C, shape.H, shape.W, shape.N, shape.D1,
                              shape.D2, shape.K, shape.stride, shape.pad, layout, math)
        self.layout = layout
        self.device = device
        self._h = tdc_conv_plan_ex(self.desc, weights["core"], weights["u_in"], weights["u_out"],
                                   weights.get("bias"), make_hints(**hints) if hints else None, device)

    def info(self) -> PlanInfo:
        i = tdc_conv_plan_query(self._h)
        return PlanInfo(i.h_out, i.w_out, i.variant, i.variant_name.decode(),
                        i.launches_per_forward, i.concurrent_forward, i.tile_h, i.tile_w,
                        i.threads_per_cta, i.smem_bytes_per_cta, i.ctas_per_image,
                        i.workspace_bytes, i.weight_bytes, i.bn_stage1, i.bn_core, i.bn_stage3,
                        i.ksplit_stage1, i.ksplit_core, i.ksplit_stage3, i.core3,
                        i.gsplit_stage1, i.gsplit_core, i.gsplit_stage3)

    @staticmethod
    def _stream_handle(stream) -> int:
        if stream is None:
            import torch
            return torch.cuda.current_stream().cuda_stream
        return int(getattr(stream, "cuda_stream", stream))

    def forward(self, x, y, batch: int | None = None, stream=None) -> None:
        for t, name in ((x, "x"), (y, "y")):
            if not (t.is_cuda and t.is_contiguous() and str(t.dtype) == "torch.float32"):
                raise TypeError(f"{name} must be a contiguous float32 CUDA tensor")
        b = int(x.shape[0]) if batch is None else batch
        tdc_conv_forward(self._h, x.data_ptr(), y.data_ptr(), b, self._stream_handle(stream))

    def forward_host(self, x_host, y_host, batch: int | None = None, stream=None) -> None:
        b = int(x_host.shape[0]) if batch is None else batch
        tdc_conv_forward_host(self._h, x_host.data_ptr(), y_host.data_ptr(), b,
                              self._stream_handle(stream))

    def close(self):
        if getattr(self, "_h", None):
            tdc_conv_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tdc_conv_forward_ex(plan, x_ptr: int, y_ptr: int, batch: int, res_ptr: int = 0, relu: int = 0,
                        stream: int = 0) -> None:
    _check(_lib.tdc_conv_forward_ex(plan, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr), batch,
                                    ctypes.c_void_p(res_ptr or None), relu, ctypes.c_void_p(stream)))


class Model:
    """RAII wrapper of tdc_model_*: an op list (dicts as built by ``synth.models``) planned
    on one device for batches up to ``max_batch``; ``forward(x, out)`` takes NHWC fp32
    CUDA tensors."""

    def __init__(self, ops: list, max_batch: int, device: int = 0):
        import numpy as np
        self._keep = []
        arr = (tdc_model_op * len(ops))()
        for i, o in enumerate(ops):
            a = arr[i]
            for k in ("kind", "src", "res", "c_in", "c_out", "height", "width", "kernel", "stride", "pad",
                      "relu"):
                setattr(a, k, int(o[k]))
            a.rank_in, a.rank_out = int(o.get("rank_in", 0)), int(o.get("rank_out", 0))
            for k in ("w", "u_in", "u_out", "bias", "bn"):
                v = o.get(k)
                if v is not None:
                    v = np.ascontiguousarray(v, dtype=np.float32)
                    self._keep.append(v)
                setattr(a, k, _fptr(v))
        self.ops = ops
        self._h = ctypes.c_void_p()
        _check(_lib.tdc_model_create(arr, len(ops), max_batch, device, ctypes.byref(self._h)))
        self.max_batch = max_batch
        self._keep = None

    def output_shape(self, op: int = -1):
        h, w, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(_lib.tdc_model_output_shape(self._h, op, ctypes.byref(h), ctypes.byref(w), ctypes.byref(c)))
        return h.value, w.value, c.value

    def forward(self, x, out, batch: int | None = None, stream=None) -> None:
        for t, name in ((x, "x"), (out, "out")):
            if not (t.is_cuda and t.is_contiguous() and str(t.dtype) == "torch.float32"):
                raise TypeError(f"{name} must be a contiguous float32 CUDA tensor")
        b = int(x.shape[0]) if batch is None else batch
        _check(_lib.tdc_model_forward(self._h, ctypes.c_void_p(x.data_ptr()), b, ctypes.c_void_p(out.data_ptr()),
                                      ctypes.c_void_p(ConvPlan._stream_handle(stream))))

    def close(self):
        if getattr(self, "_h", None):
            _lib.tdc_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
