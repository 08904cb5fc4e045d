"""TEST INFRASTRUCTURE ONLY -- ctypes front-end over the parity checkers.

Two interchangeable back-ends with identical C signatures:

* ``port``      -- ``oracle/_build/libqft_oracle.so``: the plain-C restatement
                   (``oracle/qft_oracle.c``), every function citing the reference
                   file:line it follows.
* ``reference`` -- ``oracle/_ref/libqft_ref.so``: the reference's own headers
                   (``/root/reference/proj/include/qft``) compiled unmodified with
                   the reference flags by ``oracle/Makefile``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import
this module.  The product path (``paper_2310_07147_b200``) never does.

Errors mirror the reference's pybind mapping (``test_smoke.py:72-78``):
``std::invalid_argument`` -> ``ValueError``, ``std::out_of_range`` -> ``IndexError``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "libqft_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libqft_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_f = C.c_float
_d = C.c_double

PERCENTILE = 0
RANGE_FRACTION = 1


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class DenseSparse:
    """Host mirror of ``DenseSparseWeight<float>`` (quantize.hpp:62-71)."""

    codes: np.ndarray  # u8 [rows, cols]
    scale: np.ndarray  # f32 [rows]
    zero_point: np.ndarray  # i32 [rows]
    row_ptr: np.ndarray  # i32 [rows+1]
    col_idx: np.ndarray  # i32 [nnz]
    values: np.ndarray  # f32 [nnz]
    t_min: np.ndarray = field(default=None)
    t_max: np.ndarray = field(default=None)
    bit_width: int = 8

    @property
    def rows(self):
        return self.codes.shape[0]

    @property
    def cols(self):
        return self.codes.shape[1]

    @property
    def nnz(self):
        return int(self.row_ptr[-1])

    def byte_size(self):
        """``byte_size(DenseSparseWeight)``, quantize.hpp:353-376."""
        r = self.rows
        return self.codes.size + 8 * r + 4 * (r + 1) + 8 * self.nnz + 8 * r


class Oracle:
    def __init__(self, kind: str = "port"):
        path = {"port": PORT_LIB, "reference": REF_LIB}[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.kind = kind
        self.lib = C.CDLL(path)
        p = "qo_" if kind == "port" else "qr_"
        self._p = p
        L = self.lib

        def fn(name, res, args):
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = args
            return f

        self._last_error = fn("last_error", C.c_char_p, [])
        self._minmax = fn("channel_minmax", _i, [_vp, _i, _i, _vp, _vp])
        self._params = fn("affine_params_from_bounds", _i, [_vp, _vp, _i64, _i, _vp, _vp])
        self._cparams = fn("compute_affine_params", _i, [_vp, _i, _i, _i, _vp, _vp])
        self._quantize = fn("quantize", _i, [_vp, _i, _i, _vp, _vp, _i, _i, _vp])
        self._qstate = fn("quantize_state", _i, [_vp, _i, _i, _i, _vp, _vp, _vp])
        self._dequant = fn("dequantize", _i, [_vp, _i, _i, _vp, _vp, _i, _vp])
        self._accum = fn("accumulate", _i, [_vp, _vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp])
        self._thresh = fn("outlier_thresholds", _i, [_vp, _i, _i, _d, _i, _vp, _vp])
        self._dds = fn("decompose_dense_sparse", _i64,
                       [_vp, _i, _i, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _i64])
        self._dw = fn("decompose_weight", _i64,
                      [_vp, _i, _i, _d, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64])
        self._recon = fn("reconstruct", _i, [_vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp])
        self._lion_apply = fn("lion_apply", None, [_vp, _vp, _vp, _i64, _f, _f, _f, _f])
        self._step = fn("lion_step_layer", _i64,
                        [_i, _i, _i] + [_vp] * 23 + [_i64, _f, _f, _f, _f] + [_vp] * 5)
        synth = L.qo_synth  # both libraries link oracle/synth.c
        synth.restype = None
        synth.argtypes = [_vp, _i64, C.c_uint64, _d, _d]
        self._synth = synth

    # ------------------------------------------------------------------ errors
    def _check(self, rc):
        if rc == -1:
            raise ValueError(self._last_error().decode())
        if rc == -2:
            raise IndexError(self._last_error().decode())
        return rc

    # ------------------------------------------------------------------ inputs
    def synth(self, shape, seed, sigma=0.02, spike_p=0.005):
        out = np.empty(shape, np.float32)
        self._synth(_ptr(out), out.size, seed, sigma, spike_p)
        return out

    # ------------------------------------------------------------------ L0/L1
    def channel_minmax(self, x):
        x = np.ascontiguousarray(x, np.float32)
        r, c = x.shape
        lo = np.empty(r, np.float32)
        hi = np.empty(r, np.float32)
        self._check(self._minmax(_ptr(x), r, c, _ptr(lo), _ptr(hi)))
        return lo, hi

    def affine_params_from_bounds(self, mins, maxs, bit_width=8):
        mins = np.ascontiguousarray(mins, np.float32)
        maxs = np.ascontiguousarray(maxs, np.float32)
        n = mins.size
        if maxs.size != n:
            raise ValueError("affine_params_from_bounds: bad channel count")
        s = np.empty(max(n, 1), np.float32)
        z = np.empty(max(n, 1), np.int32)
        self._check(self._params(_ptr(mins), _ptr(maxs), n, bit_width, _ptr(s), _ptr(z)))
        return s[:n], z[:n]

    def compute_affine_params(self, x, bit_width=8):
        x = np.ascontiguousarray(x, np.float32)
        r, c = x.shape
        s = np.empty(r, np.float32)
        z = np.empty(r, np.int32)
        self._check(self._cparams(_ptr(x), r, c, bit_width, _ptr(s), _ptr(z)))
        return s, z

    def quantize(self, x, scale, zero_point, bit_width=8):
        x = np.ascontiguousarray(x, np.float32)
        scale = np.ascontiguousarray(scale, np.float32)
        zero_point = np.ascontiguousarray(zero_point, np.int32)
        r, c = x.shape
        q = np.empty((r, c), np.uint8)
        self._check(self._quantize(_ptr(x), r, c, _ptr(scale), _ptr(zero_point), scale.size,
                                   bit_width, _ptr(q)))
        return q

    def quantize_state(self, x, bit_width=8):
        x = np.ascontiguousarray(x, np.float32)
        r, c = x.shape
        q = np.empty((r, c), np.uint8)
        s = np.empty(r, np.float32)
        z = np.empty(r, np.int32)
        self._check(self._qstate(_ptr(x), r, c, bit_width, _ptr(q), _ptr(s), _ptr(z)))
        return q, s, z

    def dequantize(self, codes, scale, zero_point):
        codes = np.ascontiguousarray(codes, np.uint8)
        scale = np.ascontiguousarray(scale, np.float32)
        zero_point = np.ascontiguousarray(zero_point, np.int32)
        r, c = codes.shape
        out = np.empty((r, c), np.float32)
        self._check(self._dequant(_ptr(codes), r, c, _ptr(scale), _ptr(zero_point), scale.size,
                                  _ptr(out)))
        return out

    def accumulate(self, codes, scale, zero_point, g, bit_width=8):
        """gradflow.hpp:52-58 -> (codes, scale, zero_point) of the new running sum."""
        codes = np.ascontiguousarray(codes, np.uint8)
        scale = np.ascontiguousarray(scale, np.float32)
        zero_point = np.ascontiguousarray(zero_point, np.int32)
        g = np.ascontiguousarray(g, np.float32)
        r, c = codes.shape
        q = np.empty((r, c), np.uint8)
        s = np.empty(r, np.float32)
        z = np.empty(r, np.int32)
        self._check(self._accum(_ptr(codes), _ptr(scale), _ptr(zero_point), r, c, bit_width,
                                _ptr(g), _ptr(q), _ptr(s), _ptr(z)))
        return q, s, z

    def outlier_thresholds(self, w, fraction, kind=PERCENTILE):
        w = np.ascontiguousarray(w, np.float32)
        r, c = w.shape
        lo = np.empty(r, np.float32)
        hi = np.empty(r, np.float32)
        self._check(self._thresh(_ptr(w), r, c, fraction, kind, _ptr(lo), _ptr(hi)))
        return lo, hi

    def _alloc_dsw(self, r, c, cap, bit_width):
        return DenseSparse(np.empty((r, c), np.uint8), np.empty(r, np.float32),
                           np.empty(r, np.int32), np.empty(r + 1, np.int32),
                           np.empty(max(cap, 1), np.int32), np.empty(max(cap, 1), np.float32),
                           bit_width=bit_width)

    def decompose_dense_sparse(self, w, t_min, t_max, bit_width=8):
        w = np.ascontiguousarray(w, np.float32)
        t_min = np.ascontiguousarray(t_min, np.float32)
        t_max = np.ascontiguousarray(t_max, np.float32)
        r, c = w.shape
        if t_min.size != r or t_max.size != r:
            raise ValueError("decompose_dense_sparse: threshold count must equal rows")
        cap = r * c
        d = self._alloc_dsw(r, c, cap, bit_width)
        nnz = self._check(self._dds(_ptr(w), r, c, _ptr(t_min), _ptr(t_max), bit_width,
                                    _ptr(d.codes), _ptr(d.scale), _ptr(d.zero_point),
                                    _ptr(d.row_ptr), _ptr(d.col_idx), _ptr(d.values), cap))
        d.col_idx = d.col_idx[:nnz].copy()
        d.values = d.values[:nnz].copy()
        d.t_min, d.t_max = t_min.copy(), t_max.copy()
        return d

    def decompose_weight(self, w, fraction, bit_width=8, kind=PERCENTILE):
        w = np.ascontiguousarray(w, np.float32)
        r, c = w.shape
        cap = r * c
        d = self._alloc_dsw(r, c, cap, bit_width)
        d.t_min = np.empty(r, np.float32)
        d.t_max = np.empty(r, np.float32)
        nnz = self._check(self._dw(_ptr(w), r, c, fraction, bit_width, kind, _ptr(d.t_min),
                                   _ptr(d.t_max), _ptr(d.codes), _ptr(d.scale),
                                   _ptr(d.zero_point), _ptr(d.row_ptr), _ptr(d.col_idx),
                                   _ptr(d.values), cap))
        d.col_idx = d.col_idx[:nnz].copy()
        d.values = d.values[:nnz].copy()
        return d

    def reconstruct(self, d: DenseSparse):
        r, c = d.codes.shape
        out = np.empty((r, c), np.float32)
        col = np.ascontiguousarray(d.col_idx, np.int32)
        val = np.ascontiguousarray(d.values, np.float32)
        if col.size == 0:
            col = np.zeros(1, np.int32)
            val = np.zeros(1, np.float32)
        self._check(self._recon(_ptr(np.ascontiguousarray(d.codes)), r, c, _ptr(d.scale),
                                _ptr(d.zero_point), _ptr(d.row_ptr), _ptr(col), _ptr(val),
                                _ptr(out)))
        return out

    # ------------------------------------------------------------------ L4
    def lion_apply(self, w, m, g, lr=1e-4, beta1=0.9, beta2=0.99, wd=0.0):
        w = np.array(w, np.float32, copy=True, order="C")
        m = np.array(m, np.float32, copy=True, order="C")
        g = np.ascontiguousarray(g, np.float32)
        self._lion_apply(_ptr(w), _ptr(m), _ptr(g), w.size, lr, beta1, beta2, wd)
        return w, m

    def lion_step_layer(self, w: DenseSparse, m_codes, m_scale, m_zp, g_codes, g_scale, g_zp,
                        lr=1e-4, beta1=0.9, beta2=0.99, wd=0.0, trace=False):
        """One layer of ``lion_step_quantized`` (optimizer.hpp:103-118).

        Returns ``(new_w: DenseSparse, (m_codes, m_scale, m_zp), trace_dict|None)``."""
        r, c = w.codes.shape
        b = w.bit_width
        cap = r * c
        nw = self._alloc_dsw(r, c, cap, b)
        mq = np.empty((r, c), np.uint8)
        ms = np.empty(r, np.float32)
        mz = np.empty(r, np.int32)
        tr = {k: np.empty((r, c), np.float32) for k in
              ("w_in", "g", "m_in", "w_upd", "m_upd")} if trace else None
        col = np.ascontiguousarray(w.col_idx, np.int32)
        val = np.ascontiguousarray(w.values, np.float32)
        if col.size == 0:
            col, val = np.zeros(1, np.int32), np.zeros(1, np.float32)
        args = [np.ascontiguousarray(g_codes, np.uint8), np.ascontiguousarray(g_scale, np.float32),
                np.ascontiguousarray(g_zp, np.int32), np.ascontiguousarray(m_codes, np.uint8),
                np.ascontiguousarray(m_scale, np.float32), np.ascontiguousarray(m_zp, np.int32),
                np.ascontiguousarray(w.codes), w.scale, w.zero_point, w.t_min, w.t_max,
                w.row_ptr, col, val, mq, ms, mz, nw.codes, nw.scale, nw.zero_point, nw.row_ptr,
                nw.col_idx, nw.values]
        tp = [None] * 5 if tr is None else [tr[k] for k in ("w_in", "g", "m_in", "w_upd", "m_upd")]
        nnz = self._check(self._step(r, c, b, *[_ptr(a) for a in args], cap, lr, beta1, beta2,
                                     wd, *[_ptr(a) for a in tp]))
        nw.col_idx = nw.col_idx[:nnz].copy()
        nw.values = nw.values[:nnz].copy()
        nw.t_min, nw.t_max = w.t_min.copy(), w.t_max.copy()
        return nw, (mq, ms, mz), tr


def available(kind: str) -> bool:
    return os.path.exists({"port": PORT_LIB, "reference": REF_LIB}[kind])


def build(quiet: bool = True) -> None:
    """Compile the checkers (``make -C oracle``).  Building the checker is not using it."""
    import subprocess

    subprocess.run(["make", "-C", HERE] + (["-s"] if quiet else []), check=True,
                   stdout=subprocess.DEVNULL if quiet else None)
