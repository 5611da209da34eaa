"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracle.

* ``liboracle.so``  : oracle/oracle.c, the C restatement of the reference's
  naive oracles / blocked layouts / generator / norms (each function cites
  the reference file:line it follows).
* ``_ref/libdconv_ref.so`` : the unmodified reference core compiled from
  /root/reference/proj sources by oracle/Makefile (``make ref``), driven
  through oracle/ref_driver.cpp. Optional (absent on a box where it was not
  built); used to pin the restatement bitwise and as the CPU baseline.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
reference arm may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_F64P = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class Spec(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("N", "C", "K", "H", "W", "R", "S", "stride", "pad_h", "pad_w", "vlen")]


def _build(target: str = "liboracle.so") -> None:
    subprocess.run(["make", "-s", target], cwd=_HERE, check=True)


def _load():
    path = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        _build()
    lib = C.CDLL(path)
    lib.orc_validate.argtypes = [C.POINTER(Spec)]
    lib.orc_output_shape.argtypes = [C.POINTER(Spec), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.orc_make_spec.argtypes = [C.c_int] * 11 + [C.POINTER(Spec)]
    lib.orc_pass_flops.argtypes = [C.POINTER(Spec)]
    lib.orc_pass_flops.restype = C.c_int64
    lib.orc_splitmix_next.argtypes = [C.POINTER(C.c_uint64)]
    lib.orc_splitmix_next.restype = C.c_uint64
    lib.orc_random_f32.argtypes = [C.c_uint64, _F32P, C.c_int64]
    lib.orc_uniform.argtypes = [C.c_uint64, C.c_float, C.c_float, _F32P, C.c_int64]
    lib.orc_he_normal.argtypes = [C.c_uint64, C.c_float, _F32P, C.c_int64]
    for f in ("orc_conv_forward", "orc_conv_backward", "orc_conv_update"):
        getattr(lib, f).argtypes = [C.POINTER(Spec), _F32P, _F32P, _F32P, C.c_int]
    for f in ("orc_conv_forward_f64", "orc_conv_backward_f64", "orc_conv_update_f64"):
        getattr(lib, f).argtypes = [C.POINTER(Spec), _F64P, _F64P, _F64P]
    lib.orc_act_elems.argtypes = [C.c_int] * 7
    lib.orc_act_elems.restype = C.c_int64
    lib.orc_wt_elems.argtypes = [C.c_int] * 5
    lib.orc_wt_elems.restype = C.c_int64
    lib.orc_to_blocked_act.argtypes = [_F32P] + [C.c_int] * 7 + [_F32P]
    lib.orc_from_blocked_act.argtypes = [_F32P] + [C.c_int] * 7 + [_F32P]
    lib.orc_to_blocked_wt.argtypes = [_F32P] + [C.c_int] * 5 + [_F32P]
    lib.orc_from_blocked_wt.argtypes = [_F32P] + [C.c_int] * 5 + [_F32P]
    lib.orc_transform_weight_stride1.argtypes = [_F32P] + [C.c_int] * 5 + [_F32P]
    lib.orc_error_norms_f32.argtypes = [_F32P, _F32P, C.c_int64, _F64P]
    lib.orc_apply_op_canonical.argtypes = [_F32P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _F32P]
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def spec(N, C_, K, H, W, R, S, stride, pad_h=-1, pad_w=-1, vlen=16) -> Spec:
    """make_layer_spec (layer_spec.cpp:20-43); pad < 0 = "same" default."""
    s = Spec()
    st = lib().orc_make_spec(N, C_, K, H, W, R, S, stride, pad_h, pad_w, vlen, C.byref(s))
    if st:
        raise ValueError(("NonIntegralShape", "InvalidLayerSpec")[st - 1])
    return s


def output_shape(s: Spec):
    P, Q = C.c_int(), C.c_int()
    st = lib().orc_output_shape(C.byref(s), C.byref(P), C.byref(Q))
    if st:
        raise ValueError(("NonIntegralShape", "InvalidLayerSpec")[st - 1])
    return P.value, Q.value


def pass_flops(s: Spec) -> int:
    return lib().orc_pass_flops(C.byref(s))


def random_f32(seed: int, shape) -> np.ndarray:
    """harness.cpp:274-278 random_f32 with Rng(seed): uniform in [-0.5, 0.5]."""
    out = np.empty(int(np.prod(shape)), np.float32)
    lib().orc_random_f32(seed, out, out.size)
    return out.reshape(shape)


def uniform(seed: int, shape, lo=-1.0, hi=1.0) -> np.ndarray:
    out = np.empty(int(np.prod(shape)), np.float32)
    lib().orc_uniform(seed, lo, hi, out, out.size)
    return out.reshape(shape)


def he_normal(seed: int, shape, fan_in: int) -> np.ndarray:
    out = np.empty(int(np.prod(shape)), np.float32)
    lib().orc_he_normal(seed, float(np.sqrt(2.0 / fan_in)), out, out.size)
    return out.reshape(shape)


def conv_forward(s: Spec, inp, wt, threads=None) -> np.ndarray:
    P, Q = output_shape(s)
    out = np.empty((s.N, s.K, P, Q), np.float32)
    lib().orc_conv_forward(C.byref(s), np.ascontiguousarray(inp, np.float32), np.ascontiguousarray(wt, np.float32),
                           out, threads or os.cpu_count())
    return out


def conv_backward(s: Spec, grad_out, wt, threads=None) -> np.ndarray:
    out = np.empty((s.N, s.C, s.H, s.W), np.float32)
    lib().orc_conv_backward(C.byref(s), np.ascontiguousarray(grad_out, np.float32),
                            np.ascontiguousarray(wt, np.float32), out, threads or os.cpu_count())
    return out


def conv_update(s: Spec, inp, grad_out, threads=None) -> np.ndarray:
    out = np.empty((s.K, s.C, s.R, s.S), np.float32)
    lib().orc_conv_update(C.byref(s), np.ascontiguousarray(inp, np.float32),
                          np.ascontiguousarray(grad_out, np.float32), out, threads or os.cpu_count())
    return out


def conv_forward_f64(s, inp, wt):
    P, Q = output_shape(s)
    out = np.empty((s.N, s.K, P, Q), np.float64)
    lib().orc_conv_forward_f64(C.byref(s), np.ascontiguousarray(inp, np.float64), np.ascontiguousarray(wt, np.float64),
                               out)
    return out


def conv_backward_f64(s, grad_out, wt):
    out = np.empty((s.N, s.C, s.H, s.W), np.float64)
    lib().orc_conv_backward_f64(C.byref(s), np.ascontiguousarray(grad_out, np.float64),
                                np.ascontiguousarray(wt, np.float64), out)
    return out


def conv_update_f64(s, inp, grad_out):
    out = np.empty((s.K, s.C, s.R, s.S), np.float64)
    lib().orc_conv_update_f64(C.byref(s), np.ascontiguousarray(inp, np.float64),
                              np.ascontiguousarray(grad_out, np.float64), out)
    return out


def to_blocked_act(nchw, vlen=16, halo_h=0, halo_w=0) -> np.ndarray:
    n, c, h, w = nchw.shape
    out = np.empty(lib().orc_act_elems(n, c, h, w, vlen, halo_h, halo_w), np.float32)
    lib().orc_to_blocked_act(np.ascontiguousarray(nchw, np.float32), n, c, h, w, vlen, halo_h, halo_w, out)
    return out


def from_blocked_act(blk, n, c, h, w, vlen=16, halo_h=0, halo_w=0) -> np.ndarray:
    out = np.empty((n, c, h, w), np.float32)
    lib().orc_from_blocked_act(np.ascontiguousarray(blk, np.float32), n, c, h, w, vlen, halo_h, halo_w, out)
    return out


def to_blocked_wt(kcrs, vlen=16) -> np.ndarray:
    k, c, r, s = kcrs.shape
    out = np.empty(lib().orc_wt_elems(k, c, r, s, vlen), np.float32)
    lib().orc_to_blocked_wt(np.ascontiguousarray(kcrs, np.float32), k, c, r, s, vlen, out)
    return out


def from_blocked_wt(blk, k, c, r, s, vlen=16) -> np.ndarray:
    out = np.empty((k, c, r, s), np.float32)
    lib().orc_from_blocked_wt(np.ascontiguousarray(blk, np.float32), k, c, r, s, vlen, out)
    return out


def transform_weight_stride1(blk, k, c, r, s, vlen=16) -> np.ndarray:
    out = np.empty(lib().orc_wt_elems(c, k, r, s, vlen), np.float32)
    lib().orc_transform_weight_stride1(np.ascontiguousarray(blk, np.float32), k, c, r, s, vlen, out)
    return out


def error_norms(ref, got) -> dict:
    """norms.cpp:7-25 plus the BASELINE gate e = max|d| / rms(ref)."""
    ref = np.ascontiguousarray(ref, np.float32).ravel()
    got = np.ascontiguousarray(got, np.float32).ravel()
    out = np.zeros(4, np.float64)
    lib().orc_error_norms_f32(ref, got, ref.size, out)
    rms = float(np.sqrt(np.mean(ref.astype(np.float64) ** 2))) if ref.size else 0.0
    return {"linf_abs": out[0], "l2_abs": out[1], "linf_rel": out[2], "l2_rel": out[3],
            "max_over_rms": out[0] / rms if rms > 0 else out[0]}


def apply_op_canonical(out, kind, bias=None):
    n, k, p, q = out.shape
    b = np.ascontiguousarray(bias if bias is not None else np.zeros(k), np.float32)
    o = np.ascontiguousarray(out, np.float32).copy()
    lib().orc_apply_op_canonical(o, n, k, p, q, kind, b)
    return o


# ------------------------------------------------------------- the reference itself
# Two builds of the unmodified reference core (oracle/Makefile):
#   _ref/libdconv_ref.so        -O3 -march=x86-64-v3 -ffp-contract=off: bitwise pins;
#   _ref/libdconv_ref_native.so the reference's own Release flags (-O3 -march=native,
#                               default FP contraction): the timed CPU baseline.
_ref = {}
_NATIVE_FLAGS = ("avx512f", "avx512bw", "avx512vl", "avx512dq", "avx512_fp16", "amx_tile")


def _host_flags():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def ref_available(native: bool = False) -> bool:
    return os.path.exists(_ref_path(native))


def _ref_path(native: bool) -> str:
    return os.path.join(_HERE, "_ref", "libdconv_ref_native.so" if native else "libdconv_ref.so")


def native_usable() -> bool:
    """the -march=native (sapphirerapids) build runs on this host"""
    return ref_available(True) and all(f in _host_flags() for f in _NATIVE_FLAGS)


def ref_build_info(native: bool) -> str:
    p = os.path.join(_HERE, "_ref", "COMPILER_NATIVE" if native else "COMPILER")
    try:
        with open(p) as f:
            return " ".join(f.read().split())
    except OSError:
        return "unknown"


def ref(native: bool = False):
    """The reference core (oracle/_ref/libdconv_ref[_native].so), or None."""
    if native not in _ref:
        path = _ref_path(native)
        if not os.path.exists(path):
            return None
        r = C.CDLL(path)
        ip = C.POINTER(C.c_int)
        r.ref_last_error.restype = C.c_char_p
        r.ref_pass_flops.argtypes = [ip]
        r.ref_pass_flops.restype = C.c_int64
        for f in ("ref_conv_forward_naive", "ref_conv_backward_naive", "ref_conv_update_naive"):
            getattr(r, f).argtypes = [ip, _F32P, _F32P, _F32P]
        r.ref_random_f32.argtypes = [C.c_uint64, _F32P, C.c_int64]
        r.ref_to_blocked_act.argtypes = [_F32P] + [C.c_int] * 7 + [_F32P]
        r.ref_to_blocked_wt.argtypes = [_F32P] + [C.c_int] * 5 + [_F32P]
        r.ref_transform_weight_stride1.argtypes = [_F32P] + [C.c_int] * 5 + [_F32P]
        r.ref_direct_pass.argtypes = [ip, C.c_int, C.c_int, C.c_int, _F32P, _F32P, _F32P,
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _ref[native] = r
    return _ref[native]


def spec_array(s: Spec):
    return (C.c_int * 11)(s.N, s.C, s.K, s.H, s.W, s.R, s.S, s.stride, s.pad_h, s.pad_w, s.vlen)


def ref_direct_pass(s: Spec, pass_: int, threads: int, iters: int, a, b, native: bool = False):
    """Time the reference direct engine (pass 0 F / 1 B / 2 U). Returns (out, best_ms, avg_ms)."""
    r = ref(native)
    P, Q = output_shape(s)
    shape = [(s.N, s.K, P, Q), (s.N, s.C, s.H, s.W), (s.K, s.C, s.R, s.S)][pass_]
    out = np.empty(shape, np.float32)
    best, avg = C.c_double(), C.c_double()
    st = r.ref_direct_pass(spec_array(s), pass_, threads, iters, np.ascontiguousarray(a, np.float32),
                           np.ascontiguousarray(b, np.float32), out, C.byref(best), C.byref(avg))
    if st:
        raise RuntimeError(r.ref_last_error().decode())
    return out, best.value, avg.value
