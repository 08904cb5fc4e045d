"""Device-resident QFT model state and the grouped fused Lion step.

``QftModelState`` holds every weight tensor of a model the way the reference's
``Model<float>`` + ``LionState<float>`` do (DenseSparseWeight: u8 codes, cached
per-row params and thresholds, CSR outliers; momentum: u8 codes + fresh per-row
params), laid out for one B200:

* flat HBM buffers, one per array kind, tensor i a contiguous slice -- the whole
  model's W codes are one 6.7 GB buffer for LLaMA-2-7B, so host<->device
  transfers are single large copies;
* ping-pong sets ``[0]/[1]`` for every array a step rewrites (W codes, m codes,
  m params, row_ptr, CSR arena): step ``k`` reads set ``cur`` and writes
  ``1-cur``, so an overflowing CSR arena can be grown and the step re-run from
  intact inputs;
* tensors grouped by row length; each group is ONE persistent kernel launch
  (``qftc_plan_step``) with its own CSR arena whose ``row_ptr`` values are
  absolute offsets.

The hot path is ``step()``: one launch per width class, no host synchronisation.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _native as N
from .quantize import _p, _stream, compute_outlier_thresholds, kind_from_name

_GRAD_KINDS = {"u8": N.GRAD_U8, "f32": N.GRAD_F32, "bf16": N.GRAD_BF16}


@dataclass
class _Group:
    cols: int
    members: List[int]
    rows: int
    col: List[torch.Tensor]
    val: List[torch.Tensor]
    plan: Optional[C.c_void_p] = None
    nnz: int = 0  # nnz of the arena of the current set


def _cap_for(nnz: int, rows: int) -> int:
    return int(nnz * 1.25) + 8 * rows + 1024


class QftModelState:
    def __init__(self, shapes: Sequence[Tuple[int, int]], bit_width: int = 8,
                 grad_kind: str = "u8", device="cuda"):
        if bit_width < 2 or bit_width > 8:
            raise ValueError(f"bit width must be in [2, 8], got {bit_width}")
        self.shapes = [(int(r), int(c)) for r, c in shapes]
        self.n = len(self.shapes)
        self.bit_width = bit_width
        self.grad_kind = _GRAD_KINDS[grad_kind]
        self.device = torch.device(device)
        self.cur = 0
        self.steps = 0
        sizes = [r * c for r, c in self.shapes]
        self.param_count = int(sum(sizes))
        self.row_count = int(sum(r for r, _ in self.shapes))
        # flat offsets (elements) and row offsets
        self.off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.roff = np.concatenate([[0], np.cumsum([r for r, _ in self.shapes])]).astype(np.int64)
        self.rpoff = self.roff + np.arange(self.n + 1)  # row_ptr slices have rows+1 entries
        dev, P, R = self.device, self.param_count, self.row_count
        u8, f32, i32 = torch.uint8, torch.float32, torch.int32
        self.w_codes = [torch.empty(P, dtype=u8, device=dev) for _ in range(2)]
        self.m_codes = [torch.zeros(P, dtype=u8, device=dev) for _ in range(2)]
        self.w_scale = torch.empty(R, dtype=f32, device=dev)
        self.w_zp = torch.empty(R, dtype=i32, device=dev)
        self.t_min = torch.empty(R, dtype=f32, device=dev)
        self.t_max = torch.empty(R, dtype=f32, device=dev)
        # LionState::init: quantize_state(zeros) -> scale 2^-20, z 0, codes 0
        self.m_scale = [torch.full((R,), 2.0 ** -20, dtype=f32, device=dev) for _ in range(2)]
        self.m_zp = [torch.zeros(R, dtype=i32, device=dev) for _ in range(2)]
        self.row_ptr = [torch.zeros(R + self.n, dtype=i32, device=dev) for _ in range(2)]
        if self.grad_kind == N.GRAD_U8:
            self.g_codes = torch.zeros(P, dtype=u8, device=dev)
            self.g_scale = torch.ones(R, dtype=f32, device=dev)
            self.g_zp = torch.zeros(R, dtype=i32, device=dev)
            self.g_raw = None
        else:
            self.g_codes = self.g_scale = self.g_zp = None
            gdt = f32 if self.grad_kind == N.GRAD_F32 else torch.bfloat16
            self.g_raw = torch.zeros(P, dtype=gdt, device=dev)
        # width classes -> grouped launches
        by_cols: Dict[int, List[int]] = {}
        for i, (_, c) in enumerate(self.shapes):
            by_cols.setdefault(c, []).append(i)
        self.groups: List[_Group] = []
        for c, mem in sorted(by_cols.items()):
            rows = sum(self.shapes[i][0] for i in mem)
            self.groups.append(_Group(c, mem, rows, [None, None], [None, None]))
        self.group_of = {i: gi for gi, g in enumerate(self.groups) for i in g.members}

    # ------------------------------------------------------------------ views
    def _sl(self, flat, i):
        r, c = self.shapes[i]
        return flat[self.off[i]:self.off[i + 1]].view(r, c)

    def _rows(self, flat, i):
        return flat[self.roff[i]:self.roff[i + 1]]

    def _rp(self, flat, i):
        return flat[self.rpoff[i]:self.rpoff[i + 1]]

    def grad_views(self, i):
        """(codes [r,c] u8, scale [r], zero_point [r]) -- the GradientStack entry of tensor i."""
        if self.grad_kind != N.GRAD_U8:
            return self._sl(self.g_raw, i)
        return self._sl(self.g_codes, i), self._rows(self.g_scale, i), self._rows(self.g_zp, i)

    # ------------------------------------------------------------------ init
    def _arena_alloc(self, g: _Group, cap: int, k: int):
        g.col[k] = torch.empty(max(cap, 1), dtype=torch.int32, device=self.device)
        g.val[k] = torch.empty(max(cap, 1), dtype=torch.float32, device=self.device)

    def init_from_weights(self, weight_fn, fraction: float = 0.01, kind="percentile"):
        """Decompose every tensor on the device (decompose_weight, quantize.hpp:301-314).

        ``weight_fn(i)`` returns the fp32 [rows, cols] CUDA tensor of tensor i."""
        k = kind_from_name(kind)
        cur = self.cur
        for g in self.groups:
            cap = _cap_for(int(fraction * g.rows * g.cols) + g.rows, g.rows)
            self._arena_alloc(g, cap, cur)
            base = 0
            for i in g.members:
                r, c = self.shapes[i]
                w = weight_fn(i)
                tmn, tmx = self._rows(self.t_min, i), self._rows(self.t_max, i)
                N.check(N.lib.qftc_outlier_thresholds(_p(w), r, c, float(fraction), k, _p(tmn),
                                                      _p(tmx), _stream()))
                while True:
                    cap_left = g.col[cur].numel() - base
                    nnz = C.c_int64(0)
                    rp = self._rp(self.row_ptr[cur], i)
                    rc = N.lib.qftc_decompose_dense_sparse(
                        _p(w), r, c, _p(tmn), _p(tmx), self.bit_width,
                        _p(self._sl(self.w_codes[cur], i)), _p(self._rows(self.w_scale, i)),
                        _p(self._rows(self.w_zp, i)), _p(rp), _p(g.col[cur][base:]),
                        _p(g.val[cur][base:]), cap_left, C.byref(nnz), _stream())
                    if rc == N.QFTC_EOVERFLOW:
                        self._grow(g, cur, base + int(nnz.value), keep=base)
                        continue
                    N.check(rc)
                    break
                rp += base
                base += int(nnz.value)
                del w
            g.nnz = base
        self._make_plans()

    def init_from_host(self, tensors: Sequence[dict]):
        """Upload reference-layout state (e.g. from the CPU oracle).  Each dict holds
        codes, scale, zero_point, t_min, t_max, row_ptr, col_idx, values (the
        DenseSparseWeight) and optionally m_codes, m_scale, m_zero_point."""
        cur = self.cur
        for g in self.groups:
            nnz = sum(int(tensors[i]["row_ptr"][-1]) for i in g.members)
            self._arena_alloc(g, _cap_for(nnz, g.rows), cur)
            base = 0
            for i in g.members:
                t = tensors[i]
                cp = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a)).to(self.device, dt)
                self._sl(self.w_codes[cur], i).copy_(cp(t["codes"], torch.uint8))
                self._rows(self.w_scale, i).copy_(cp(t["scale"], torch.float32))
                self._rows(self.w_zp, i).copy_(cp(t["zero_point"], torch.int32))
                self._rows(self.t_min, i).copy_(cp(t["t_min"], torch.float32))
                self._rows(self.t_max, i).copy_(cp(t["t_max"], torch.float32))
                rp = np.asarray(t["row_ptr"], np.int64)
                self._rp(self.row_ptr[cur], i).copy_(cp(rp + base, torch.int32))
                n = int(rp[-1])
                if n:
                    g.col[cur][base:base + n].copy_(cp(t["col_idx"], torch.int32))
                    g.val[cur][base:base + n].copy_(cp(t["values"], torch.float32))
                if "m_codes" in t:
                    self._sl(self.m_codes[cur], i).copy_(cp(t["m_codes"], torch.uint8))
                    self._rows(self.m_scale[cur], i).copy_(cp(t["m_scale"], torch.float32))
                    self._rows(self.m_zp[cur], i).copy_(cp(t["m_zero_point"], torch.int32))
                base += n
            g.nnz = base
        self._make_plans()

    def _grow(self, g: _Group, k: int, need: int, keep: int):
        cap = _cap_for(need, g.rows)
        col = torch.empty(cap, dtype=torch.int32, device=self.device)
        val = torch.empty(cap, dtype=torch.float32, device=self.device)
        if keep:
            col[:keep].copy_(g.col[k][:keep])
            val[:keep].copy_(g.val[k][:keep])
        g.col[k], g.val[k] = col, val

    # ------------------------------------------------------------------ plans
    def _descs(self, g: _Group):
        arr = (N.LionTensorC * len(g.members))()
        for j, i in enumerate(g.members):
            r, c = self.shapes[i]
            d = arr[j]
            d.rows, d.cols = r, c
            for k in range(2):
                d.w_codes[k] = self._sl(self.w_codes[k], i).data_ptr()
                d.row_ptr[k] = self._rp(self.row_ptr[k], i).data_ptr()
                d.m_codes[k] = self._sl(self.m_codes[k], i).data_ptr()
                d.m_scale[k] = self._rows(self.m_scale[k], i).data_ptr()
                d.m_zero_point[k] = self._rows(self.m_zp[k], i).data_ptr()
            d.w_scale = self._rows(self.w_scale, i).data_ptr()
            d.w_zero_point = self._rows(self.w_zp, i).data_ptr()
            d.t_min = self._rows(self.t_min, i).data_ptr()
            d.t_max = self._rows(self.t_max, i).data_ptr()
            if self.grad_kind == N.GRAD_U8:
                d.g_codes = self._sl(self.g_codes, i).data_ptr()
                d.g_scale = self._rows(self.g_scale, i).data_ptr()
                d.g_zero_point = self._rows(self.g_zp, i).data_ptr()
            else:
                d.g_raw = self._sl(self.g_raw, i).data_ptr()
        return arr

    def _arena_args(self, g: _Group):
        cols = (C.c_void_p * 2)(*[t.data_ptr() if t is not None else None for t in g.col])
        vals = (C.c_void_p * 2)(*[t.data_ptr() if t is not None else None for t in g.val])
        caps = (C.c_int64 * 2)(*[t.numel() if t is not None else 0 for t in g.col])
        return cols, vals, caps

    def _make_plans(self):
        for g in self.groups:
            nxt = 1 - self.cur
            if g.col[nxt] is None:
                self._arena_alloc(g, _cap_for(g.nnz, g.rows), nxt)
            if g.plan is not None:
                N.lib.qftc_plan_destroy(g.plan)
            arr = self._descs(g)
            cols, vals, caps = self._arena_args(g)
            plan = C.c_void_p()
            N.check(N.lib.qftc_plan_create(C.byref(plan), arr, len(g.members), self.bit_width,
                                           self.grad_kind, cols, vals, caps, _stream()))
            g.plan = plan

    def __del__(self):
        for g in getattr(self, "groups", []):
            if g.plan is not None:
                try:
                    N.lib.qftc_plan_destroy(g.plan)
                except Exception:
                    pass
                g.plan = None

    # ------------------------------------------------------------------ the step
    def launches_per_step(self) -> int:
        return len(self.groups)

    def step(self, lr=1e-4, beta1=0.9, beta2=0.99, weight_decay=0.0, check: bool = False):
        """One quantized Lion step over the whole model (lion_step_quantized,
        optimizer.hpp:85-120): one fused kernel launch per width class, enqueued on
        the current stream without host synchronisation.  ``check=True`` also
        synchronises, validates, and transparently re-runs after growing a CSR arena
        that overflowed (the inputs of the step are intact in the other set)."""
        h = N.hyper(lr, beta1, beta2, weight_decay)
        flip = self.cur
        for g in self.groups:
            N.check(N.lib.qftc_plan_step(g.plan, flip, h, _stream()))
        self.cur = 1 - flip
        self.steps += 1
        if check:
            self._check(flip, h)

    def _check(self, flip, h):
        for g in self.groups:
            while True:
                nnz = C.c_int64(0)
                rc = N.lib.qftc_plan_result(g.plan, C.byref(nnz), _stream())
                if rc == N.QFTC_EOVERFLOW:
                    self._grow(g, 1 - flip, int(nnz.value), keep=0)
                    cols, vals, caps = self._arena_args(g)
                    N.check(N.lib.qftc_plan_set_arena(g.plan, cols, vals, caps))
                    N.check(N.lib.qftc_plan_step(g.plan, flip, h, _stream()))
                    continue
                N.check(rc)
                g.nnz = int(nnz.value)
                break

    def check(self):
        """Synchronise and validate the last step (raises on overflow / bad rows)."""
        for g in self.groups:
            nnz = C.c_int64(0)
            N.check(N.lib.qftc_plan_result(g.plan, C.byref(nnz), _stream()))
            g.nnz = int(nnz.value)

    # ------------------------------------------------------------------ export
    def nnz(self) -> int:
        return int(sum(g.nnz for g in self.groups))

    def export_tensor(self, i: int) -> dict:
        """Reference-layout host copy of tensor i (DenseSparseWeight + momentum)."""
        cur = self.cur
        g = self.groups[self.group_of[i]]
        rp = self._rp(self.row_ptr[cur], i).cpu().numpy().astype(np.int64)
        b, e = int(rp[0]), int(rp[-1])
        return dict(
            codes=self._sl(self.w_codes[cur], i).cpu().numpy(),
            scale=self._rows(self.w_scale, i).cpu().numpy(),
            zero_point=self._rows(self.w_zp, i).cpu().numpy(),
            t_min=self._rows(self.t_min, i).cpu().numpy(),
            t_max=self._rows(self.t_max, i).cpu().numpy(),
            row_ptr=(rp - b).astype(np.int32),
            col_idx=g.col[cur][b:e].cpu().numpy(),
            values=g.val[cur][b:e].cpu().numpy(),
            m_codes=self._sl(self.m_codes[cur], i).cpu().numpy(),
            m_scale=self._rows(self.m_scale[cur], i).cpu().numpy(),
            m_zero_point=self._rows(self.m_zp[cur], i).cpu().numpy(),
        )

    def reconstruct(self, i: int, dtype=torch.float32) -> torch.Tensor:
        """Expand tensor i (dequant + CSR overwrite) to f32 or bf16 for the next forward."""
        cur = self.cur
        g = self.groups[self.group_of[i]]
        r, c = self.shapes[i]
        out = torch.empty((r, c), dtype=dtype, device=self.device)
        fn = N.lib.qftc_reconstruct if dtype == torch.float32 else N.lib.qftc_reconstruct_bf16
        N.check(fn(_p(self._sl(self.w_codes[cur], i)), r, c, _p(self._rows(self.w_scale, i)),
                   _p(self._rows(self.w_zp, i)), _p(self._rp(self.row_ptr[cur], i)),
                   _p(g.col[cur]), _p(g.val[cur]), _p(out), _stream()))
        return out
