"""fp64 CPU oracle for the TKD convolution layer (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2211_03715_b200``) never does; the two share no code.

This module is argument marshalling around ``liboracle.so`` (built from
``tdc_oracle.c`` by :func:`build`): fp32 test tensors are widened exactly to
fp64 and passed to the C loops.  Parity status per function is listed in
``tdc_oracle.h`` and DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tdc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no FMA contraction, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "tdc_oracle.h"))):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call([
            "gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
            "-shared", "-fPIC", "-o", tmp, _SRC,
        ])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        i = ctypes.c_int
        lib.tdc_oracle_out_dim.argtypes = [i, i, i, i]
        lib.tdc_oracle_conv7.argtypes = [dp, i, i, i, i, dp, i, i, i, i, i, dp]
        lib.tdc_oracle_reconstruct.argtypes = [dp, dp, dp, i, i, i, i, i, dp]
        lib.tdc_oracle_tkd_stages.argtypes = [dp, i, i, i, i, dp, i, i, i, dp, dp, i,
                                              dp, i, i, dp, dp, dp]
        lib.tdc_oracle_tkd_point.argtypes = [dp, i, i, i, i, dp, i, i, i, dp, dp, i,
                                             dp, i, i, i, i, i, i, dp]
        lib.tdc_oracle_set_threads.argtypes = [i]
        lib.tdc_oracle_max_threads.restype = i
        _lib = lib
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def set_threads(n: int) -> None:
    _load().tdc_oracle_set_threads(int(n))


def max_threads() -> int:
    return int(_load().tdc_oracle_max_threads())


def out_dim(h: int, k: int, stride: int, pad: int) -> int:
    return int(_load().tdc_oracle_out_dim(h, k, stride, pad))


def conv7(x, w, stride: int = 1, pad: int = 0) -> np.ndarray:
    """Seven-loop cross-correlation. x: B,C,H,W; w: N,C,R,S -> B,N,H',W'."""
    x = _f64(x)
    w = _f64(w)
    B, C, H, W = x.shape
    N, C2, R, S = w.shape
    if C2 != C:
        raise ValueError("channel mismatch")
    Ho, Wo = out_dim(H, R, stride, pad), out_dim(W, S, stride, pad)
    if Ho < 1 or Wo < 1:
        raise ValueError("empty output")
    y = np.empty((B, N, Ho, Wo), dtype=np.float64)
    rc = _load().tdc_oracle_conv7(_ptr(x), B, C, H, W, _ptr(w), N, R, S, stride, pad, _ptr(y))
    if rc:
        raise ValueError(f"tdc_oracle_conv7 rc={rc}")
    return y


def reconstruct(core, u_in, u_out) -> np.ndarray:
    """Eq. tkd2: W_rec[n,c,r,t] = sum_{a,q} U_out[n,q] core[q,a,r,t] U_in[c,a]."""
    core, u_in, u_out = _f64(core), _f64(u_in), _f64(u_out)
    D2, D1, K, K2 = core.shape
    C, N = u_in.shape[0], u_out.shape[0]
    if K != K2 or u_in.shape[1] != D1 or u_out.shape[1] != D2:
        raise ValueError("shape mismatch")
    w = np.empty((N, C, K, K), dtype=np.float64)
    rc = _load().tdc_oracle_reconstruct(_ptr(core), _ptr(u_in), _ptr(u_out), C, N, D1, D2, K, _ptr(w))
    if rc:
        raise ValueError(f"tdc_oracle_reconstruct rc={rc}")
    return w


def _dims(x, core, u_in, u_out):
    B, C, H, W = x.shape
    D2, D1, K, K2 = core.shape
    N = u_out.shape[0]
    if K != K2 or u_in.shape != (C, D1) or u_out.shape != (N, D2):
        raise ValueError("shape mismatch")
    return B, C, H, W, D1, D2, K, N


def tkd_stages(x, core, u_in, u_out, bias=None, stride: int = 1, pad: int = 0,
               return_intermediates: bool = False):
    """Three-stage TKD layer in fp64 (NCHW).  Returns y (and x1, z if asked)."""
    x, core, u_in, u_out = _f64(x), _f64(core), _f64(u_in), _f64(u_out)
    bias = None if bias is None else _f64(bias)
    B, C, H, W, D1, D2, K, N = _dims(x, core, u_in, u_out)
    Ho, Wo = out_dim(H, K, stride, pad), out_dim(W, K, stride, pad)
    if Ho < 1 or Wo < 1:
        raise ValueError("empty output")
    y = np.empty((B, N, Ho, Wo), dtype=np.float64)
    x1 = np.empty((B, D1, H, W), dtype=np.float64) if return_intermediates else None
    z = np.empty((B, D2, Ho, Wo), dtype=np.float64) if return_intermediates else None
    rc = _load().tdc_oracle_tkd_stages(_ptr(x), B, C, H, W, _ptr(core), D1, D2, K,
                                       _ptr(u_in), _ptr(u_out), N, _ptr(bias), stride, pad,
                                       _ptr(x1), _ptr(z), _ptr(y))
    if rc:
        raise ValueError(f"tdc_oracle_tkd_stages rc={rc}")
    return (y, x1, z) if return_intermediates else y


def tkd_points(x, core, u_in, u_out, points, bias=None, stride: int = 1, pad: int = 0):
    """y[b,n,i,j] for each (b,n,i,j) in ``points``, evaluated one by one."""
    x, core, u_in, u_out = _f64(x), _f64(core), _f64(u_in), _f64(u_out)
    bias = None if bias is None else _f64(bias)
    B, C, H, W, D1, D2, K, N = _dims(x, core, u_in, u_out)
    lib = _load()
    out = np.empty(len(points), dtype=np.float64)
    v = ctypes.c_double()
    for k, (b, n, i, j) in enumerate(points):
        rc = lib.tdc_oracle_tkd_point(_ptr(x), B, C, H, W, _ptr(core), D1, D2, K,
                                      _ptr(u_in), _ptr(u_out), N, _ptr(bias), stride, pad,
                                      int(b), int(n), int(i), int(j), ctypes.byref(v))
        if rc:
            raise ValueError(f"tdc_oracle_tkd_point rc={rc} at {(b, n, i, j)}")
        out[k] = v.value
    return out


def tkd_full(x, core, u_in, u_out, bias=None, stride: int = 1, pad: int = 0):
    """Plain definition: conv7 with the reconstructed kernel."""
    y = conv7(x, reconstruct(core, u_in, u_out), stride, pad)
    if bias is not None:
        y = y + _f64(bias)[None, :, None, None]
    return y
