"""QFTC v1 checkpoints straight from / into the device-resident model state (plus the
opt-in format extensions, version 0x8001: packed sub-byte codes, blockwise momentum scales).

Drop-in for ``qft::save_checkpoint`` / ``qft::load_checkpoint`` (checkpoint.cpp:100-211):
the same byte layout, the same checks in the same order, and the same error texts.
Files written here are byte-identical to the reference's for the same state
(tests/golden/ckpt_*.qftc come from the reference itself).

Layout (little-endian): "QFTC", version u16 (1), layer count u16, bit width u8, quant
mode u8, threshold kind u8, loss u8, one activation u8 per junction, outlier fraction
f32; per layer: rows u32, cols u32, t_min f32[rows], t_max f32[rows], scale f32[rows],
zero_point i32[rows], codes u8[rows*cols], nnz u32, row_ptr i32[rows+1], col_idx
i32[nnz], values f32[nnz], momentum scale f32[rows], zero_point i32[rows], codes
u8[rows*cols]; then the CRC-32 of everything before it.

B200 side: the state never leaves HBM in pieces the host has to assemble.  The CRC is
computed on the GPU over the device arrays in file order (``qftc_crc32``).  The arrays
are copied device -> host (pageable ``.cpu()`` copies, array by array) -> file.  On load the whole file is copied to the
device once and verified there before the state is built.  Pass-through checkpoints
(raw fp32 weights, ``QuantMode::passthrough``) are outside the quantized path and are
refused.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np
import torch

from . import _native as N
from .engine import QftModelState
from .quantize import _stream

MAGIC = b"QFTC"
VERSION = 1
VERSION_EXT = 0x8001   # v1 + the opt-in extensions below (the reference reads only v1; the
                       # high bit keeps the family apart from any future reference version)
EXT_PACKED = 1         # W and momentum codes bit-packed at bit_width bits (lossless)
EXT_MOM_BLOCKS = 2     # momentum with one (scale, zero point) per block of a row (lossy)
AFFINE, PASSTHROUGH = 0, 1


@dataclass
class CheckpointMeta:
    """The ModelConfig fields a checkpoint records (checkpoint.cpp:106-114)."""
    bit_width: int = 8
    quant_mode: int = AFFINE
    threshold_kind: int = 0          # ThresholdKind: 0 percentile, 1 range_fraction
    loss: int = 0                    # LossKind: 0 mse, 1 softmax_cross_entropy
    junctions: Optional[List[int]] = None   # Activation per junction; None: relu (1) everywhere
    outlier_fraction: float = 0.01
    layer_dims: List[int] = field(default_factory=list)


def _crc_device(segments: List[torch.Tensor]) -> int:
    ptrs = (C.c_void_p * max(len(segments), 1))(*[t.data_ptr() for t in segments])
    lens = (C.c_int64 * max(len(segments), 1))(*[t.numel() * t.element_size()
                                                   for t in segments])
    out = C.c_uint32(0)
    N.check(N.lib.qftc_crc32(ptrs, lens, len(segments), C.byref(out), _stream()))
    return int(out.value)


def _dev_bytes(b: bytes, device) -> torch.Tensor:
    return torch.frombuffer(bytearray(b), dtype=torch.uint8).to(device)


def _packed(codes: torch.Tensor, rows: int, cols: int, bits: int) -> torch.Tensor:
    out = torch.empty(rows * ((cols * bits + 7) // 8), dtype=torch.uint8, device=codes.device)
    N.check(N.lib.qftc_pack_codes(C.c_void_p(codes.data_ptr()), rows, cols, bits,
                                  C.c_void_p(out.data_ptr()), _stream()))
    return out


def _unpacked(packed: torch.Tensor, rows: int, cols: int, bits: int) -> torch.Tensor:
    out = torch.empty(rows * cols, dtype=torch.uint8, device=packed.device)
    N.check(N.lib.qftc_unpack_codes(C.c_void_p(packed.data_ptr()), rows, cols, bits,
                                    C.c_void_p(out.data_ptr()), _stream()))
    return out


def _mom_blocks(codes, scale, zp, rows, cols, bits, block, to_blocks: bool):
    nb = rows * ((cols + block - 1) // block) if to_blocks else rows
    dev = codes.device
    oc = torch.empty(rows * cols, dtype=torch.uint8, device=dev)
    os_ = torch.empty(nb, dtype=torch.float32, device=dev)
    oz = torch.empty(nb, dtype=torch.int32, device=dev)
    fn = N.lib.qftc_momentum_to_blocks if to_blocks else N.lib.qftc_momentum_from_blocks
    N.check(fn(C.c_void_p(codes.data_ptr()), C.c_void_p(scale.data_ptr()),
               C.c_void_p(zp.data_ptr()), rows, cols, bits, block, C.c_void_p(oc.data_ptr()),
               C.c_void_p(os_.data_ptr()), C.c_void_p(oz.data_ptr()), _stream()))
    return oc, os_, oz


def save_checkpoint(state: QftModelState, path: str, meta: Optional[CheckpointMeta] = None,
                    packed_codes: bool = False, momentum_block: int = 0):
    """save_checkpoint(model, state, path) (checkpoint.cpp:100-140) for the whole
    device-resident state: layer l of the file is tensor l of ``state``.

    ``meta`` defaults to the config the state records: the one it was loaded with, or
    the outlier fraction / threshold kind it was decomposed with (relu junctions, mse
    loss -- ModelConfig's defaults).  A state that does not know its outlier fraction
    (built by init_from_host without ``fraction``) needs an explicit ``meta``: the
    reference writes cfg.outlier_fraction, so guessing would misreport the file.

    Opt-in format extensions (the file becomes version 0x8001, which
    the reference does not read): ``packed_codes`` bit-packs the W and momentum codes at
    the state's bit width (lossless: 3-bit codes take 3/8 of a byte); ``momentum_block``
    > 0 stores the momentum with one affine (scale, zero point) per block of that many
    elements of a row -- a requantization of the dequantized momentum, lossy; the loader
    brings it back to the per-row quantize_state form.  The header then carries one
    extension-flags byte and the block size (u16) after the outlier fraction."""
    if meta is None:
        meta = getattr(state, "checkpoint_meta", None)
    if meta is None:
        if getattr(state, "outlier_fraction", None) is None:
            raise ValueError("save_checkpoint: the state does not record its outlier fraction; "
                             "pass meta=CheckpointMeta(...)")
        meta = CheckpointMeta(bit_width=state.bit_width, threshold_kind=state.threshold_kind,
                              outlier_fraction=state.outlier_fraction)
    if meta.quant_mode != AFFINE:
        raise NotImplementedError("pass-through checkpoints are outside the quantized path")
    L = state.n
    junc = meta.junctions if meta.junctions is not None else [1] * max(L - 1, 0)
    if len(junc) != max(L - 1, 0):
        raise ValueError("junction count must be num_layers - 1")
    flags = (EXT_PACKED if packed_codes else 0) | (EXT_MOM_BLOCKS if momentum_block > 0 else 0)
    if momentum_block < 0 or momentum_block > 0xFFFF:
        raise ValueError("momentum_block must be in [0, 65535]")
    head = MAGIC + struct.pack("<HHBBBB", VERSION_EXT if flags else VERSION, L, state.bit_width,
                               meta.quant_mode, meta.threshold_kind, meta.loss)
    head += bytes(junc) + struct.pack("<f", meta.outlier_fraction)
    if flags:
        head += struct.pack("<BH", flags, momentum_block)
    dev = state.device
    cur = state.cur
    bw = state.bit_width
    segs: List[torch.Tensor] = [_dev_bytes(head, dev)]
    for i in range(L):
        r, c = state.shapes[i]
        rp, col, val = state.strict_csr(i)
        wc = state._sl(state.w_codes[cur], i).reshape(-1)
        ms, mz = state._rows(state.m_scale[cur], i), state._rows(state.m_zp[cur], i)
        mc = state._sl(state.m_codes[cur], i).reshape(-1)
        if momentum_block > 0:
            mc, ms, mz = _mom_blocks(mc, ms, mz, r, c, bw, momentum_block, True)
        if packed_codes:
            wc, mc = _packed(wc, r, c, bw), _packed(mc, r, c, bw)
        segs += [_dev_bytes(struct.pack("<II", r, c), dev),
                 state._rows(state.t_min, i), state._rows(state.t_max, i),
                 state._rows(state.w_scale, i), state._rows(state.w_zp, i), wc,
                 _dev_bytes(struct.pack("<I", col.numel()), dev), rp, col, val, ms, mz, mc]
    crc = _crc_device(segs)
    try:
        f = open(path, "wb")
    except OSError:
        raise RuntimeError(f"cannot open '{path}' for writing") from None
    with f:
        for t in segs:
            if t.numel():
                f.write(t.contiguous().view(torch.uint8).cpu().numpy().data)
        f.write(struct.pack("<I", crc))


class _Reader:
    """checkpoint.cpp:54-78: bounds-checked little-endian reads."""

    def __init__(self, buf: np.ndarray, start: int, end: int, path: str):
        self.buf, self.p, self.end, self.path = buf, start, end, path

    def _take(self, n: int) -> int:
        if self.p + n > self.end:
            raise RuntimeError(f"checkpoint '{self.path}' is truncated")
        p = self.p
        self.p += n
        return p

    def get(self, fmt: str):
        n = struct.calcsize(fmt)
        return struct.unpack_from(fmt, self.buf, self._take(n))[0]

    def array(self, dtype, n: int) -> np.ndarray:
        dt = np.dtype(dtype)
        p = self._take(n * dt.itemsize)
        a = self.buf[p:p + n * dt.itemsize].view(dt)
        return a if p % dt.itemsize == 0 else a.copy()  # fields are packed, not aligned


def load_checkpoint(path: str, device="cuda") -> Tuple[QftModelState, CheckpointMeta]:
    """load_checkpoint(path) (checkpoint.cpp:142-211): the same checks, in the same
    order, with the same messages; returns the device-resident state and the config
    fields the file records."""
    try:
        buf = np.fromfile(path, dtype=np.uint8)
    except OSError:
        raise RuntimeError(f"cannot open checkpoint '{path}'") from None
    if buf.size < 4 + 4:
        raise RuntimeError(f"checkpoint '{path}' is truncated")
    if bytes(buf[:4]) != MAGIC:
        raise RuntimeError(f"'{path}' is not a checkpoint (bad magic)")
    stored = struct.unpack_from("<I", buf, buf.size - 4)[0]
    body = torch.from_numpy(buf[:-4]).to(device)  # verified where the state will live
    if _crc_device([body]) != stored:
        raise RuntimeError(f"checkpoint '{path}' is corrupt (crc mismatch)")
    del body
    r = _Reader(buf, 4, buf.size - 4, path)
    version = r.get("<H")
    if version not in (VERSION, VERSION_EXT):
        raise RuntimeError(f"checkpoint '{path}' has unsupported version {version}")
    L = r.get("<H")
    if L == 0:
        raise RuntimeError(f"checkpoint '{path}' has no layers")
    meta = CheckpointMeta()
    meta.bit_width = r.get("<B")
    meta.quant_mode = r.get("<B")
    meta.threshold_kind = r.get("<B")
    meta.loss = r.get("<B")
    meta.junctions = [r.get("<B") for _ in range(L - 1)]
    meta.outlier_fraction = float(r.get("<f"))
    flags, block = 0, 0
    if version == VERSION_EXT:
        flags, block = r.get("<B"), r.get("<H")
        if flags & ~(EXT_PACKED | EXT_MOM_BLOCKS) or (bool(flags & EXT_MOM_BLOCKS) != (block > 0)):
            raise RuntimeError(f"checkpoint '{path}' has unsupported extensions")
    if meta.quant_mode != AFFINE:
        raise NotImplementedError("pass-through checkpoints are outside the quantized path")
    bw = meta.bit_width
    if flags and not 2 <= bw <= 8:
        raise RuntimeError(f"checkpoint '{path}' has an invalid bit width")

    def codes_of(rows, cols):
        if flags & EXT_PACKED:
            pk = r.array(np.uint8, rows * ((cols * bw + 7) // 8))
            return _unpacked(torch.from_numpy(np.ascontiguousarray(pk)).to(device), rows, cols,
                             bw).cpu().numpy().reshape(rows, cols)
        return r.array(np.uint8, rows * cols).reshape(rows, cols)

    shapes, tensors = [], []
    for li in range(L):
        rows, cols = r.get("<I"), r.get("<I")
        if not (0 < rows < 2 ** 31 and 0 < cols < 2 ** 31):  # static_cast<int> > 0
            raise RuntimeError(f"checkpoint '{path}' has an empty layer")
        t = dict(t_min=r.array(np.float32, rows), t_max=r.array(np.float32, rows),
                 scale=r.array(np.float32, rows), zero_point=r.array(np.int32, rows),
                 codes=codes_of(rows, cols))
        nnz = r.get("<I")
        t["row_ptr"] = r.array(np.int32, rows + 1)
        t["col_idx"] = r.array(np.int32, nnz)
        t["values"] = r.array(np.float32, nnz)
        if int(t["row_ptr"][-1]) != nnz:
            raise RuntimeError(f"checkpoint '{path}' has inconsistent sparse layout")
        nm = rows * ((cols + block - 1) // block) if block else rows
        t["m_scale"] = r.array(np.float32, nm)
        t["m_zero_point"] = r.array(np.int32, nm)
        t["m_codes"] = codes_of(rows, cols)
        if block:  # back to the per-row quantize_state form (lossy)
            d = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
            mc, ms, mz = _mom_blocks(d(t["m_codes"], None).reshape(-1), d(t["m_scale"], None),
                                     d(t["m_zero_point"], None), rows, cols, bw, block, False)
            t["m_codes"] = mc.cpu().numpy().reshape(rows, cols)
            t["m_scale"], t["m_zero_point"] = ms.cpu().numpy(), mz.cpu().numpy()
        if li == 0:
            meta.layer_dims.append(cols)
        meta.layer_dims.append(rows)
        shapes.append((rows, cols))
        tensors.append(t)
    if r.p != r.end:
        raise RuntimeError(f"checkpoint '{path}' has trailing bytes")
    st = QftModelState(shapes, bit_width=meta.bit_width, device=device)
    st.init_from_host(tensors, fraction=meta.outlier_fraction,
                      kind="percentile" if meta.threshold_kind == 0 else "range_fraction")
    st.checkpoint_meta = meta
    return st, meta
