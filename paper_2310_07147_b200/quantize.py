"""Device-side mirror of the reference quantizer/optimizer API (namespace ``qft``,
``/root/reference/proj/include/qft/{quantize,optimizer,gradflow}.hpp``), ``T=float``.

Same names, argument meaning and error behaviour as the reference; tensors are
``torch`` CUDA tensors (PyTorch is only the allocator/stream plumbing here -- all
arithmetic runs in the sm_100a kernels behind the C-ABI).  Value semantics are
kept: functions return new objects, and ``requantize_weight`` /
``lion_step_quantized`` replace the members of the objects they are given,
exactly as the reference mutates through non-const references.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import torch

from . import _native as N

PERCENTILE = "percentile"
RANGE_FRACTION = "range-fraction"
_KINDS = {PERCENTILE: N.PERCENTILE, RANGE_FRACTION: N.RANGE_FRACTION,
          "range_fraction": N.RANGE_FRACTION, 0: N.PERCENTILE, 1: N.RANGE_FRACTION}


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dev(x, dtype=torch.float32) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(x)
    if x.dim() != 2:
        raise ValueError("expected a 2-d tensor")
    if x.device.type != "cuda":
        x = x.to("cuda", non_blocking=False)
    return x.to(dtype).contiguous()


def kind_from_name(kind) -> int:
    if kind not in _KINDS:
        raise ValueError(f"threshold kind must be percentile or range-fraction, got '{kind}'")
    return _KINDS[kind]


# ----------------------------------------------------------------------------- types
@dataclass
class AffineParams:
    """``AffineParams<float>`` (quantize.hpp:26-34)."""

    scale: torch.Tensor        # f32 [channels]
    zero_point: torch.Tensor   # i32 [channels]
    bit_width: int = 8

    def channels(self) -> int:
        return int(self.scale.numel())

    def qmax(self) -> int:
        return (1 << self.bit_width) - 1


@dataclass
class QuantizedTensor:
    """``QuantizedTensor<float>`` affine mode (quantize.hpp:36-46)."""

    rows: int
    cols: int
    data: torch.Tensor         # u8 [rows, cols]
    params: AffineParams

    def size(self) -> int:
        return self.rows * self.cols


@dataclass
class SparseOutliers:
    """Strict CSR (quantize.hpp:48-57); ``row_ptr[0] == 0``."""

    row_ptr: torch.Tensor      # i32 [rows+1]
    col_idx: torch.Tensor      # i32 [nnz]
    values: torch.Tensor       # f32 [nnz]

    def nnz(self) -> int:
        return int(self.values.numel())


@dataclass
class DenseSparseWeight:
    """``DenseSparseWeight<float>`` (quantize.hpp:62-71)."""

    dense: QuantizedTensor
    sparse: SparseOutliers
    t_min: torch.Tensor
    t_max: torch.Tensor
    outlier_fraction: float = 0.0

    def rows(self) -> int:
        return self.dense.rows

    def cols(self) -> int:
        return self.dense.cols


def _require_bit_width(b: int):
    if b < 2 or b > 8:
        raise ValueError(f"bit width must be in [2, 8], got {b}")


# ----------------------------------------------------------------------------- L0/L1
def channel_minmax(x):
    """tensor.hpp:133-148."""
    x = _dev(x)
    r, c = x.shape
    lo = torch.empty(r, dtype=torch.float32, device=x.device)
    hi = torch.empty_like(lo)
    N.check(N.lib.qftc_channel_minmax(_p(x), r, c, _p(lo), _p(hi), _stream()))
    return lo, hi


def affine_params_from_bounds(mins, maxs, bit_width: int) -> AffineParams:
    """quantize.hpp:105-131."""
    _require_bit_width(bit_width)
    mins = torch.as_tensor(mins, dtype=torch.float32).reshape(-1).cuda().contiguous()
    maxs = torch.as_tensor(maxs, dtype=torch.float32).reshape(-1).cuda().contiguous()
    if mins.numel() != maxs.numel() or mins.numel() == 0:
        raise ValueError("affine_params_from_bounds: bad channel count")
    s = torch.empty_like(mins)
    z = torch.empty(mins.numel(), dtype=torch.int32, device=mins.device)
    N.check(N.lib.qftc_affine_params_from_bounds(_p(mins), _p(maxs), mins.numel(), bit_width,
                                                 _p(s), _p(z), _stream()))
    return AffineParams(s, z, bit_width)


def compute_affine_params(x, bit_width: int = 8, channel_wise: bool = True) -> AffineParams:
    """quantize.hpp:133-147."""
    x = _dev(x)
    if x.numel() == 0:
        raise ValueError("compute_affine_params: empty tensor")
    if not channel_wise:
        lo, hi = channel_minmax(x.reshape(1, -1))
        return affine_params_from_bounds(lo, hi, bit_width)
    lo, hi = channel_minmax(x)
    return affine_params_from_bounds(lo, hi, bit_width)


def quantize(x, p: AffineParams) -> QuantizedTensor:
    """quantize.hpp:149-175."""
    x = _dev(x)
    r, c = x.shape
    if p.channels() != 1 and p.channels() != r:
        raise ValueError(f"quantize: channel count {p.channels()} does not match rows {r}")
    q = torch.empty((r, c), dtype=torch.uint8, device=x.device)
    N.check(N.lib.qftc_quantize(_p(x), r, c, _p(p.scale), _p(p.zero_point), p.channels(),
                                p.bit_width, _p(q), _stream()))
    return QuantizedTensor(r, c, q, p)


def quantize_state(x, bit_width: int = 8, check: bool = True) -> QuantizedTensor:
    """quantize.hpp:189-193 (affine mode): fused per-row bounds + params + codes."""
    x = _dev(x)
    r, c = x.shape
    if r == 0 or c == 0:
        raise ValueError("compute_affine_params: empty tensor")
    _require_bit_width(bit_width)
    q = torch.empty((r, c), dtype=torch.uint8, device=x.device)
    s = torch.empty(r, dtype=torch.float32, device=x.device)
    z = torch.empty(r, dtype=torch.int32, device=x.device)
    N.check(N.lib.qftc_quantize_state(_p(x), r, c, bit_width, _p(q), _p(s), _p(z),
                                      1 if check else 0, _stream()))
    return QuantizedTensor(r, c, q, AffineParams(s, z, bit_width))


def dequantize(q: QuantizedTensor, dtype=torch.float32) -> torch.Tensor:
    """quantize.hpp:195-212 (bf16: RNE of the fp32 result)."""
    if q.rows <= 0 or q.cols <= 0:
        raise ValueError("dequantize: empty tensor")
    out = torch.empty((q.rows, q.cols), dtype=dtype, device=q.data.device)
    fn = N.lib.qftc_dequantize if dtype == torch.float32 else N.lib.qftc_dequantize_bf16
    N.check(fn(_p(q.data), q.rows, q.cols, _p(q.params.scale), _p(q.params.zero_point),
               q.params.channels(), _p(out), _stream()))
    return out


def compute_outlier_thresholds(w, fraction: float, kind=PERCENTILE):
    """quantize.hpp:216-247 (exact per-row order statistics by radix select)."""
    w = _dev(w)
    r, c = w.shape
    k = kind_from_name(kind)
    lo = torch.empty(r, dtype=torch.float32, device=w.device)
    hi = torch.empty_like(lo)
    N.check(N.lib.qftc_outlier_thresholds(_p(w), r, c, float(fraction), k, _p(lo), _p(hi),
                                          _stream()))
    return lo, hi


def decompose_dense_sparse(w, t_min, t_max, bit_width: int = 8,
                           capacity: Optional[int] = None) -> DenseSparseWeight:
    """quantize.hpp:253-290.  ``capacity`` bounds the CSR buffer (grown on overflow)."""
    w = _dev(w)
    r, c = w.shape
    t_min = torch.as_tensor(t_min, dtype=torch.float32).reshape(-1).cuda().contiguous()
    t_max = torch.as_tensor(t_max, dtype=torch.float32).reshape(-1).cuda().contiguous()
    if t_min.numel() != r or t_max.numel() != r:
        raise ValueError("decompose_dense_sparse: threshold count must equal rows")
    dev = w.device
    codes = torch.empty((r, c), dtype=torch.uint8, device=dev)
    s = torch.empty(r, dtype=torch.float32, device=dev)
    z = torch.empty(r, dtype=torch.int32, device=dev)
    rp = torch.empty(r + 1, dtype=torch.int32, device=dev)
    cap = int(capacity) if capacity is not None else max(64, r * c // 32)
    while True:
        col = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        val = torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
        nnz = C.c_int64(0)
        rc = N.lib.qftc_decompose_dense_sparse(_p(w), r, c, _p(t_min), _p(t_max), bit_width,
                                               _p(codes), _p(s), _p(z), _p(rp), _p(col),
                                               _p(val), cap, C.byref(nnz), _stream())
        if rc == N.QFTC_EOVERFLOW:
            cap = int(nnz.value)
            continue
        N.check(rc)
        break
    n = int(nnz.value)
    return DenseSparseWeight(QuantizedTensor(r, c, codes, AffineParams(s, z, bit_width)),
                             SparseOutliers(rp, col[:n].clone(), val[:n].clone()),
                             t_min.clone(), t_max.clone())


def decompose_weight(w, fraction: float, bit_width: int = 8,
                     kind=PERCENTILE) -> DenseSparseWeight:
    """quantize.hpp:301-314 (affine mode)."""
    t_min, t_max = compute_outlier_thresholds(w, fraction, kind)
    out = decompose_dense_sparse(w, t_min, t_max, bit_width)
    out.outlier_fraction = float(fraction)
    return out


def requantize_weight(dsw: DenseSparseWeight, w_fp, bit_width: int) -> None:
    """quantize.hpp:318-329: re-split against the CACHED thresholds, in place."""
    nxt = decompose_dense_sparse(w_fp, dsw.t_min, dsw.t_max, bit_width)
    dsw.dense, dsw.sparse = nxt.dense, nxt.sparse


def reconstruct(dsw: DenseSparseWeight, dtype=torch.float32) -> torch.Tensor:
    """quantize.hpp:331-338; ``dtype=torch.bfloat16`` is the on-the-fly expansion for the
    next forward's GEMM operand (network.hpp:208-211 consumer)."""
    d = dsw.dense
    out = torch.empty((d.rows, d.cols), dtype=dtype, device=d.data.device)
    col, val = dsw.sparse.col_idx, dsw.sparse.values
    if col.numel() == 0:
        col = torch.zeros(1, dtype=torch.int32, device=d.data.device)
        val = torch.zeros(1, dtype=torch.float32, device=d.data.device)
    fn = N.lib.qftc_reconstruct if dtype == torch.float32 else N.lib.qftc_reconstruct_bf16
    N.check(fn(_p(d.data), d.rows, d.cols, _p(d.params.scale), _p(d.params.zero_point),
               _p(dsw.sparse.row_ptr), _p(col), _p(val), _p(out), _stream()))
    return out


def byte_size(dsw: DenseSparseWeight) -> int:
    """quantize.hpp:353-376."""
    r = dsw.rows()
    return dsw.dense.size() + 8 * r + 4 * (r + 1) + 8 * dsw.sparse.nnz() + 8 * r


# ----------------------------------------------------------------------------- L3/L4
@dataclass
class LionHyper:
    """``LionHyper<float>`` (optimizer.hpp:15-21)."""

    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.99
    weight_decay: float = 0.0

    def c(self):
        return N.hyper(self.lr, self.beta1, self.beta2, self.weight_decay)


@dataclass
class StackEntry:
    layer_index: int
    grad: QuantizedTensor


class GradientStack:
    """FILO hand-off of quantized per-layer gradients (gradflow.hpp:15-47)."""

    def __init__(self):
        self._entries: List[StackEntry] = []

    def push(self, layer_index: int, grad: QuantizedTensor) -> None:
        self._entries.append(StackEntry(layer_index, grad))

    def pop(self) -> StackEntry:
        if not self._entries:
            raise IndexError("gradient stack: pop on empty stack")
        return self._entries.pop()

    def size(self) -> int:
        return len(self._entries)

    def __len__(self):
        return len(self._entries)

    def empty(self) -> bool:
        return not self._entries

    def at(self, i: int) -> StackEntry:
        """gradflow.hpp:40-43 (bounds-checked)."""
        if i < 0 or i >= len(self._entries):
            raise IndexError("gradient stack: index out of range")
        return self._entries[i]


def accumulate(acc: QuantizedTensor, g_new, out: Optional[QuantizedTensor] = None
               ) -> QuantizedTensor:
    """gradflow.hpp:52-58: the integer-form micro-batch running sum,
    quantize_state(dequantize(acc) + g_new) with fresh per-row params, in one fused row
    kernel.  ``out`` may be ``acc`` itself (in-place update of the stack entry)."""
    g = _dev(g_new)
    if acc.rows != g.shape[0] or acc.cols != g.shape[1]:
        raise ValueError("accumulate: shape mismatch")
    if out is None:
        out = QuantizedTensor(acc.rows, acc.cols, torch.empty_like(acc.data),
                              AffineParams(torch.empty_like(acc.params.scale),
                                           torch.empty_like(acc.params.zero_point),
                                           acc.params.bit_width))
    N.check(N.lib.qftc_accumulate_state(
        _p(acc.data), _p(acc.params.scale), _p(acc.params.zero_point), acc.rows, acc.cols,
        acc.params.bit_width, _p(g), _p(out.data), _p(out.params.scale),
        _p(out.params.zero_point), _stream()))
    return out


@dataclass
class LionState:
    """Quantized momentum per layer (optimizer.hpp:52-67)."""

    momentum: List[QuantizedTensor] = field(default_factory=list)

    @staticmethod
    def init(weights: List[DenseSparseWeight], bit_width: int = 8) -> "LionState":
        st = LionState()
        for w in weights:
            zeros = torch.zeros((w.rows(), w.cols()), dtype=torch.float32, device="cuda")
            st.momentum.append(quantize_state(zeros, bit_width))
        return st


def lion_step_quantized(weights: List[DenseSparseWeight], state: LionState,
                        stack: GradientStack, h: LionHyper, bit_width: int = 8) -> None:
    """optimizer.hpp:85-120: pop layers 1..L, fused dequant -> Lion -> requant per layer.

    Validation order and messages follow the reference (optimizer.hpp:89-102)."""
    L = len(weights)
    if stack.size() != L:
        raise ValueError(f"lion step: stack holds {stack.size()} gradients for {L} layers")
    if len(state.momentum) != L:
        raise ValueError("lion step: momentum count does not match layers")
    hc = h.c()
    for li in range(1, L + 1):
        e = stack.pop()
        if e.layer_index != li:
            raise ValueError(f"lion step: popped layer {e.layer_index}, expected {li}")
        w = weights[li - 1]
        if e.grad.rows != w.rows() or e.grad.cols != w.cols():
            raise ValueError(f"lion step: gradient shape mismatch at layer {li}")
        m = state.momentum[li - 1]
        r, c = w.rows(), w.cols()
        dev = w.dense.data.device
        m_codes = torch.empty((r, c), dtype=torch.uint8, device=dev)
        m_s = torch.empty(r, dtype=torch.float32, device=dev)
        m_z = torch.empty(r, dtype=torch.int32, device=dev)
        w_codes = torch.empty((r, c), dtype=torch.uint8, device=dev)
        rp = torch.empty(r + 1, dtype=torch.int32, device=dev)
        col_in, val_in = w.sparse.col_idx, w.sparse.values
        if col_in.numel() == 0:
            col_in = torch.zeros(1, dtype=torch.int32, device=dev)
            val_in = torch.zeros(1, dtype=torch.float32, device=dev)
        cap = max(64, int(w.sparse.nnz() * 1.25) + r)
        while True:
            col = torch.empty(cap, dtype=torch.int32, device=dev)
            val = torch.empty(cap, dtype=torch.float32, device=dev)
            nnz = C.c_int64(0)
            rc = N.lib.qftc_lion_step(
                r, c, bit_width, _p(e.grad.data), _p(e.grad.params.scale),
                _p(e.grad.params.zero_point), _p(m.data), _p(m.params.scale),
                _p(m.params.zero_point), _p(w.dense.data), _p(w.dense.params.scale),
                _p(w.dense.params.zero_point), _p(w.t_min), _p(w.t_max), _p(w.sparse.row_ptr),
                _p(col_in), _p(val_in), _p(m_codes), _p(m_s), _p(m_z), _p(w_codes), _p(rp),
                _p(col), _p(val), cap, hc, C.byref(nnz), _stream())
            if rc == N.QFTC_EOVERFLOW:
                cap = int(nnz.value)
                continue
            N.check(rc)
            break
        n = int(nnz.value)
        state.momentum[li - 1] = QuantizedTensor(r, c, m_codes, AffineParams(m_s, m_z, bit_width))
        w.dense = QuantizedTensor(r, c, w_codes, w.dense.params)
        w.sparse = SparseOutliers(rp, col[:n].clone(), val[:n].clone())


def lion_apply(w: torch.Tensor, m: torch.Tensor, g: torch.Tensor, h: LionHyper) -> None:
    """Pass-through mode (optimizer.hpp:33-42) on raw fp32 state, in place."""
    if w.shape != g.shape or w.shape != m.shape:
        raise ValueError("lion_apply: shape mismatch")
    N.check(N.lib.qftc_lion_apply(_p(w), _p(m), _p(g), w.numel(), h.c(), _stream()))


def synth(shape, seed: int, sigma: float = 0.02, spike_p: float = 0.005,
          device="cuda") -> torch.Tensor:
    """Deterministic synthetic tensor (device twin of oracle/synth.c)."""
    out = torch.empty(shape, dtype=torch.float32, device=device)
    N.check(N.lib.qftc_synth(_p(out), out.numel(), int(seed) & (2**64 - 1), float(sigma),
                             float(spike_p), _stream()))
    return out
