"""ctypes binding of libnw.so (include/nw.h): argument marshalling only.

Every computation happens in the library's CUDA kernels; this module converts
torch tensors to device pointers and status codes to exceptions.  There is no
fallback: if libnw.so is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnw.so")

# enums (mirror include/nw.h)
NW_OK, NW_ERR_INVALID, NW_ERR_UNSUPPORTED, NW_ERR_NOMEM, NW_ERR_CUDA, NW_ERR_WORKSPACE, NW_ERR_STATE = range(7)
MATH_FP32_SIMT, MATH_BF16X3, MATH_BF16 = 0, 1, 2
DTYPE_F32, DTYPE_BF16 = 0, 1
(ATTR_MATH, ATTR_DTYPE, ATTR_TRANSPOSED, ATTR_OUTPUT_PADDING, ATTR_OUTER_TAPS, ATTR_PAD,
 ATTR_PRELU, ATTR_DEPTHWISE) = range(8)
(TABLE_BT, TABLE_G, TABLE_AT, TABLE_GATHER, TABLE_SCATTER, TABLE_ORIGINS, TABLE_PHASE_TAPS,
 TABLE_DIMS) = range(8)

EXPORTS = [
    "nw_plan", "nw_plan_set", "nw_plan_set_prelu", "nw_plan_finalize", "nw_plan_destroy", "nw_plan_info",
    "nw_plan_tables", "nw_output_size", "nw_workspace_size", "nw_workspace_size_ola",
    "nw_workspace_size_direct", "nw_transform_filter", "nw_conv_forward", "nw_conv_ola", "nw_conv_direct",
    "nw_count_mults", "nw_launch_count", "nw_status_str", "nw_workspace_size_host", "nw_conv_forward_host",
    "nw_profile_begin", "nw_profile_end", "nw_decompose",
]


class PlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "K", "stride", "transposed", "pad", "output_padding", "m_outer", "r_outer", "m_inner",
        "points_axis", "points", "window", "tile_out", "n_phase", "Kp", "cin", "cout", "cin_e",
        "cout_e", "cin_pad", "cout_pad", "math", "dtype")] + [("filter_bytes", ctypes.c_size_t),
                                                              ("m_rows", ctypes.c_int),
                                                              ("single_kernel", ctypes.c_int)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class NWError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_str(status)} ({status})")


_lib: Optional[ctypes.CDLL] = None


def load() -> ctypes.CDLL:
    """Load libnw.so (built in-tree by paper_2102_13272_b200.build); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2102_13272_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, LL, SZ, VP = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_size_t, ctypes.c_void_p
    st = ctypes.c_int
    sig = {
        "nw_plan": (st, [I, I, I, I, I, I, ctypes.POINTER(P)]),
        "nw_plan_set": (st, [P, I, LL]),
        "nw_plan_set_prelu": (st, [P, VP]),
        "nw_plan_finalize": (st, [P]),
        "nw_plan_destroy": (st, [P]),
        "nw_plan_info": (st, [P, ctypes.POINTER(PlanInfo)]),
        "nw_plan_tables": (st, [P, I, ctypes.POINTER(LL), SZ, ctypes.POINTER(SZ)]),
        "nw_output_size": (st, [P, I, I, ctypes.POINTER(I), ctypes.POINTER(I)]),
        "nw_workspace_size": (st, [P, I, I, I, ctypes.POINTER(SZ)]),
        "nw_workspace_size_ola": (st, [P, I, I, I, ctypes.POINTER(SZ)]),
        "nw_workspace_size_direct": (st, [P, I, I, I, ctypes.POINTER(SZ)]),
        "nw_transform_filter": (st, [P, VP, VP, VP]),
        "nw_conv_forward": (st, [P, VP, VP, VP, I, I, I, VP, SZ, VP]),
        "nw_conv_ola": (st, [P, VP, VP, VP, I, I, I, VP, SZ, VP]),
        "nw_conv_direct": (st, [P, VP, VP, VP, I, I, I, VP, SZ, VP]),
        "nw_count_mults": (st, [P, I, I, I, ctypes.POINTER(ctypes.c_ulonglong)]),
        "nw_launch_count": (ctypes.c_ulonglong, []),
        "nw_status_str": (ctypes.c_char_p, [I]),
        "nw_workspace_size_host": (st, [P, I, I, I, ctypes.POINTER(SZ)]),
        "nw_conv_forward_host": (st, [P, VP, VP, VP, I, I, I, VP, SZ, VP]),
        "nw_profile_begin": (st, []),
        "nw_profile_end": (st, [ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_ulonglong),
                                ctypes.POINTER(ctypes.c_double), SZ, ctypes.POINTER(SZ)]),
        "nw_decompose": (st, [I, I, I, I, ctypes.c_char_p, SZ, ctypes.POINTER(SZ), ctypes.POINTER(I)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    _lib = lib
    return lib


def status_str(s: int) -> str:
    return load().nw_status_str(s).decode()


def _chk(s: int, what: str) -> None:
    if s != NW_OK:
        raise NWError(s, what)


def _ptr(t) -> int:
    """Device pointer of a torch tensor (or an int / None)."""
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Plan:
    """Owns one nw_plan_t.  Attributes are set before the first use (finalize)."""

    def __init__(self, K: int, stride: int, m_outer: int, m_inner: int, Cin: int, Cout: int, *,
                 math: int = MATH_BF16X3, dtype: int = DTYPE_F32, transposed: bool = False,
                 output_padding: int = 0, outer_taps: int = 3, pad: Optional[int] = None,
                 prelu_slopes=None, depthwise: bool = False):
        lib = load()
        self._h = ctypes.c_void_p()
        _chk(lib.nw_plan(K, stride, m_outer, m_inner, Cin, Cout, ctypes.byref(self._h)), "nw_plan")
        for attr, val in ((ATTR_MATH, math), (ATTR_DTYPE, dtype), (ATTR_TRANSPOSED, int(transposed)),
                          (ATTR_OUTPUT_PADDING, output_padding), (ATTR_OUTER_TAPS, outer_taps)):
            _chk(lib.nw_plan_set(self._h, attr, val), f"nw_plan_set({attr})")
        if pad is not None:
            _chk(lib.nw_plan_set(self._h, ATTR_PAD, pad), "nw_plan_set(pad)")
        if depthwise:
            _chk(lib.nw_plan_set(self._h, ATTR_DEPTHWISE, 1), "nw_plan_set(depthwise)")
        self._slopes = prelu_slopes  # keep the device buffer alive
        if prelu_slopes is not None:
            _chk(lib.nw_plan_set_prelu(self._h, _ptr(prelu_slopes)), "nw_plan_set_prelu")
        _chk(lib.nw_plan_finalize(self._h), "nw_plan_finalize")
        self.K, self.stride, self.Cin, self.Cout, self.depthwise = K, stride, Cin, Cout, depthwise

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib is not None:
            _lib.nw_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        inf = PlanInfo()
        _chk(load().nw_plan_info(self._h, ctypes.byref(inf)), "nw_plan_info")
        return inf.as_dict()

    def tables(self, which: int) -> List[int]:
        lib = load()
        n = ctypes.c_size_t()
        _chk(lib.nw_plan_tables(self._h, which, None, 0, ctypes.byref(n)), "nw_plan_tables(size)")
        buf = (ctypes.c_longlong * n.value)()
        _chk(lib.nw_plan_tables(self._h, which, buf, n.value, ctypes.byref(n)), "nw_plan_tables")
        return list(buf)

    def output_size(self, H: int, W: int):
        ho, wo = ctypes.c_int(), ctypes.c_int()
        _chk(load().nw_output_size(self._h, H, W, ctypes.byref(ho), ctypes.byref(wo)), "nw_output_size")
        return ho.value, wo.value

    def workspace_size(self, N: int, H: int, W: int, path: str = "nested") -> int:
        lib = load()
        fn = {"nested": lib.nw_workspace_size, "ola": lib.nw_workspace_size_ola,
              "direct": lib.nw_workspace_size_direct, "host": lib.nw_workspace_size_host}[path]
        b = ctypes.c_size_t()
        _chk(fn(self._h, N, H, W, ctypes.byref(b)), f"workspace_size({path})")
        return b.value

    def count_mults(self, N: int, H: int, W: int) -> int:
        c = ctypes.c_ulonglong()
        _chk(load().nw_count_mults(self._h, N, H, W, ctypes.byref(c)), "nw_count_mults")
        return c.value

    def transform_filter(self, w, U, stream=None) -> None:
        _chk(load().nw_transform_filter(self._h, _ptr(w), _ptr(U), _stream(stream)), "nw_transform_filter")

    def forward(self, x, U, y, N: int, H: int, W: int, ws, ws_bytes: int, stream=None) -> None:
        _chk(load().nw_conv_forward(self._h, _ptr(x), _ptr(U), _ptr(y), N, H, W, _ptr(ws), ws_bytes,
                                    _stream(stream)), "nw_conv_forward")

    def forward_host(self, x_host, U, y_host, N: int, H: int, W: int, ws, ws_bytes: int, stream=None) -> None:
        """x_host / y_host: host (ideally pinned) tensors; copies happen inside the call."""
        _chk(load().nw_conv_forward_host(self._h, _ptr(x_host), _ptr(U), _ptr(y_host), N, H, W, _ptr(ws),
                                         ws_bytes, _stream(stream)), "nw_conv_forward_host")

    def ola(self, x, w, y, N: int, H: int, W: int, ws, ws_bytes: int, stream=None) -> None:
        _chk(load().nw_conv_ola(self._h, _ptr(x), _ptr(w), _ptr(y), N, H, W, _ptr(ws), ws_bytes,
                                _stream(stream)), "nw_conv_ola")

    def direct(self, x, w, y, N: int, H: int, W: int, ws, ws_bytes: int, stream=None) -> None:
        _chk(load().nw_conv_direct(self._h, _ptr(x), _ptr(w), _ptr(y), N, H, W, _ptr(ws), ws_bytes,
                                   _stream(stream)), "nw_conv_direct")


def decompose(R: int, S: int, m: int, r: int):
    """Section IV.B decomposition (host only): (reverse-Polish token string, output length M)."""
    lib = load()
    n, M = ctypes.c_size_t(), ctypes.c_int()
    _chk(lib.nw_decompose(R, S, m, r, None, 0, ctypes.byref(n), ctypes.byref(M)), "nw_decompose")
    buf = ctypes.create_string_buffer(n.value + 1)
    _chk(lib.nw_decompose(R, S, m, r, buf, n.value + 1, ctypes.byref(n), ctypes.byref(M)), "nw_decompose")
    return buf.value.decode(), M.value


def launch_count() -> int:
    return int(load().nw_launch_count())


def profile_begin() -> None:
    _chk(load().nw_profile_begin(), "nw_profile_begin")


def profile_end() -> dict:
    """{kernel kind: (launches, total ms)} for launches since profile_begin()."""
    lib = load()
    cap = 32
    names = (ctypes.c_char_p * cap)()
    cnt = (ctypes.c_ulonglong * cap)()
    ms = (ctypes.c_double * cap)()
    n = ctypes.c_size_t()
    _chk(lib.nw_profile_end(names, cnt, ms, cap, ctypes.byref(n)), "nw_profile_end")
    return {names[i].decode(): (int(cnt[i]), float(ms[i])) for i in range(min(n.value, cap))}
