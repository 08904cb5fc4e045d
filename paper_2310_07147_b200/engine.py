"""Device-resident QFT model state and the grouped fused Lion step.

``QftModelState`` holds every weight tensor of a model the way the reference's
``Model<float>`` + ``LionState<float>`` do (DenseSparseWeight: u8 codes, cached
per-row params and thresholds, CSR outliers; momentum: u8 codes + fresh per-row
params), laid out for one B200:

* flat HBM buffers, one per array kind, tensor i a contiguous slice -- the whole
  model's W codes are one 6.7 GB buffer for LLaMA-2-7B, so host<->device
  transfers are single large copies;
* ping-pong sets ``[0]/[1]`` for every array a step rewrites (W codes, m codes,
  m params, CSR counts and arena): step ``k`` reads set ``cur`` and writes
  ``1-cur``, so an overflowing CSR slot can be re-planned and the step re-run
  from intact inputs;
* outliers in a SLOTTED CSR: row r owns a 16-byte aligned slot
  ``[row_start[r], row_start[r+1])`` of its group's arena, sized from its count +
  25% + 8; ``row_count[r]`` entries are used.  Rows never wait on each other
  inside the step; the strict reference CSR is produced by compaction
  (``export_tensor``);
* tensors grouped by row length; each group is ONE persistent kernel launch
  (``qftc_plan_step``) with its own arena.

The hot path is ``step()``: one launch per width class, no host synchronisation.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _native as N
from .quantize import _p, _stream, kind_from_name

_GRAD_KINDS = {"u8": N.GRAD_U8, "f32": N.GRAD_F32, "bf16": N.GRAD_BF16}
SLACK = 8
GROWTH_STEPS = 16  # a re-planned slot holds this many steps of the row's last growth


@dataclass
class _Group:
    cols: int
    members: List[int]
    rows: int
    col: List[Optional[torch.Tensor]]
    val: List[Optional[torch.Tensor]]
    plan: Optional[C.c_void_p] = None
    replans: int = 0          # slot re-plans so far: each widens the headroom (_replan)
    layout_idx: Optional[tuple] = None   # cached (rs positions, scan index, contiguous)


class QftModelState:
    def __init__(self, shapes: Sequence[Tuple[int, int]], bit_width: int = 8,
                 grad_kind: str = "u8", device="cuda", pad_to: int = 0,
                 group_contiguous: bool = True):
        """`group_contiguous`: lay the flat buffers out width class by width class (so a
        run of tensors of one launch group is one contiguous range of every array, which
        the chunked host pipeline needs); False keeps the given order (ZeRO-1 shards,
        whose gradient layout is fixed by the reduce-scatter)."""
        if bit_width < 2 or bit_width > 8:
            raise ValueError(f"bit width must be in [2, 8], got {bit_width}")
        self.shapes = [(int(r), int(c)) for r, c in shapes]
        self.n = len(self.shapes)
        self.bit_width = bit_width
        self.grad_kind = _GRAD_KINDS[grad_kind]
        self.device = torch.device(device)
        self.cur = 0
        self.steps = 0
        self.replans = 0
        # the decomposition config the state was built with (DenseSparseWeight::
        # outlier_fraction, quantize.hpp:70; ModelConfig::threshold_kind): recorded by
        # init_from_weights / init_from_host(fraction=...) / load_checkpoint, written by
        # save_checkpoint.  None: unknown (save_checkpoint then requires explicit meta).
        self.outlier_fraction: Optional[float] = None
        self.threshold_kind: int = 0
        self.checkpoint_meta = None
        order = list(range(self.n))
        if group_contiguous:
            order.sort(key=lambda i: (self.shapes[i][1], i))
        self.order = order                       # flat position -> tensor index
        self.pos = {i: p for p, i in enumerate(order)}
        sizes = [self.shapes[i][0] * self.shapes[i][1] for i in order]
        rows_l = [self.shapes[i][0] for i in order]
        self.param_count = int(sum(sizes))
        self.row_count_total = int(sum(rows_l))
        self.off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.roff = np.concatenate([[0], np.cumsum(rows_l)]).astype(np.int64)
        self.rpoff = self.roff + np.arange(self.n + 1)  # row_start slices have rows+1 entries
        self.chunks: List[dict] = []
        dev, P, R = self.device, self.param_count, self.row_count_total
        u8, f32, i32 = torch.uint8, torch.float32, torch.int32
        self.w_codes = [torch.zeros(max(P, pad_to), dtype=u8, device=dev) for _ in range(2)]
        self.m_codes = [torch.zeros(P, dtype=u8, device=dev) for _ in range(2)]
        self.w_scale = torch.empty(R, dtype=f32, device=dev)
        self.w_zp = torch.empty(R, dtype=i32, device=dev)
        self.t_min = torch.empty(R, dtype=f32, device=dev)
        self.t_max = torch.empty(R, dtype=f32, device=dev)
        # LionState::init: quantize_state(zeros) -> scale 2^-20, z 0, codes 0
        self.m_scale = [torch.full((R,), 2.0 ** -20, dtype=f32, device=dev) for _ in range(2)]
        self.m_zp = [torch.zeros(R, dtype=i32, device=dev) for _ in range(2)]
        self.row_start = [torch.zeros(R + self.n, dtype=i32, device=dev) for _ in range(2)]
        self.row_count = [torch.zeros(R, dtype=i32, device=dev) for _ in range(2)]
        if self.grad_kind == N.GRAD_U8:
            self.g_codes = torch.zeros(P, dtype=u8, device=dev)
            self.g_scale = torch.ones(R, dtype=f32, device=dev)
            self.g_zp = torch.zeros(R, dtype=i32, device=dev)
            self.g_raw = None
        else:
            self.g_codes = self.g_scale = self.g_zp = None
            gdt = f32 if self.grad_kind == N.GRAD_F32 else torch.bfloat16
            self.g_raw = torch.zeros(max(P, pad_to), dtype=gdt, device=dev)
        by_cols: Dict[int, List[int]] = {}
        for i in order:
            by_cols.setdefault(self.shapes[i][1], []).append(i)
        self.groups: List[_Group] = []
        for c, mem in sorted(by_cols.items()):
            rows = sum(self.shapes[i][0] for i in mem)
            self.groups.append(_Group(c, mem, rows, [None, None], [None, None]))
        self.group_of = {i: gi for gi, g in enumerate(self.groups) for i in g.members}
        self._plan_order = None

    # ------------------------------------------------------------------ views
    def _sl(self, flat, i):
        r, c = self.shapes[i]
        p = self.pos[i]
        return flat[self.off[p]:self.off[p + 1]].view(r, c)

    def _rows(self, flat, i):
        p = self.pos[i]
        return flat[self.roff[p]:self.roff[p + 1]]

    def _rs(self, flat, i):
        p = self.pos[i]
        return flat[self.rpoff[p]:self.rpoff[p + 1]]

    def grad_views(self, i):
        """The GradientStack entry of tensor i: (codes [r,c] u8, scale [r], zero_point [r]),
        or the raw [r,c] gradient for grad kinds f32/bf16."""
        if self.grad_kind != N.GRAD_U8:
            return self._sl(self.g_raw, i)
        return self._sl(self.g_codes, i), self._rows(self.g_scale, i), self._rows(self.g_zp, i)

    def sink_grad(self, i: int, g: torch.Tensor, accumulate: bool = False):
        """The backward's gradient sink for tensor i (gradflow.hpp:70-84), u8 kind: the
        first micro-batch quantizes its fp32 gradient into the stack entry
        (quantize_state, :77); later ones fold into it in integer form (accumulate,
        :52-58, one fused row kernel, in place)."""
        if self.grad_kind != N.GRAD_U8:
            raise ValueError("sink_grad: the engine keeps raw gradients (grad kind f32/bf16)")
        r, c = self.shapes[i]
        g = g.contiguous()
        if g.dtype != torch.float32 or tuple(g.shape) != (r, c):
            raise ValueError("sink_grad: expected a float32 gradient of the tensor's shape")
        codes, s, z = self.grad_views(i)
        if accumulate:
            N.check(N.lib.qftc_accumulate_state(_p(codes), _p(s), _p(z), r, c, self.bit_width,
                                                _p(g), _p(codes), _p(s), _p(z), _stream()))
        else:
            N.check(N.lib.qftc_quantize_state(_p(g), r, c, self.bit_width, _p(codes), _p(s),
                                              _p(z), 1, _stream()))

    def sink_wgrad(self, i: int, dy: torch.Tensor, x: torch.Tensor, accumulate: bool = False,
                   norm_sq: Optional[torch.Tensor] = None, g_out: Optional[torch.Tensor] = None,
                   check: bool = False):
        """The backward's weight gradient of tensor i with the sink fused into the GEMM
        epilogue (qftc_wgrad_quant; backward_core network.hpp:139 wgrad =
        matmul(transpose(out_grad), in) -> gradflow.hpp:70-84): dy bf16 [T, rows], x bf16
        [T, cols]; the stack entry receives quantize_state(dy^T x) (or, accumulating, the
        integer-form sum) without an fp32 gradient in HBM.  norm_sq: a float64 device
        scalar += sum of squares (backward_core's norm); g_out: the f32 values quantized."""
        if self.grad_kind != N.GRAD_U8:
            raise ValueError("sink_wgrad: the engine keeps raw gradients (grad kind f32/bf16)")
        r, c = self.shapes[i]
        for name, t, w in (("dy", dy, r), ("x", x, c)):
            if t.dtype != torch.bfloat16 or t.dim() != 2 or t.shape[1] != w or not t.is_contiguous():
                raise ValueError(f"sink_wgrad: {name} must be a contiguous bf16 [T, {w}] tensor")
        if dy.shape[0] != x.shape[0]:
            raise ValueError("sink_wgrad: dy and x must have the same number of rows (tokens)")
        ws = getattr(self, "_wg_ws", None)
        need = int(N.lib.qftc_wgrad_workspace_bytes(r))
        if ws is None or ws.numel() < need:
            ws = self._wg_ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        codes, s, z = self.grad_views(i)
        N.check(N.lib.qftc_wgrad_quant(
            _p(dy), _p(x), dy.shape[0], r, c, self.bit_width, int(bool(accumulate)), _p(codes),
            _p(s), _p(z), _p(g_out) if g_out is not None else None,
            _p(norm_sq) if norm_sq is not None else None, _p(ws), int(bool(check)), _stream()))

    # ------------------------------------------------------------------ arenas / slots
    def _alloc(self, cap: int):
        return (torch.empty(max(cap, 4), dtype=torch.int32, device=self.device),
                torch.empty(max(cap, 4), dtype=torch.float32, device=self.device))

    def _ensure(self, g: _Group, k: int, need: int, keep: int):
        if g.col[k] is not None and g.col[k].numel() >= need:
            return
        col, val = self._alloc(int(need * 1.5) + 1024)  # room for a first re-plan
        if keep and g.col[k] is not None:
            col[:keep].copy_(g.col[k][:keep])
            val[:keep].copy_(g.val[k][:keep])
        g.col[k], g.val[k] = col, val

    def _place_strict(self, g: _Group, i: int, k: int, base: int, rp: torch.Tensor,
                      col: torch.Tensor, val: torch.Tensor) -> int:
        """Put tensor i's strict CSR (device row_ptr/col/val) into slots of arena k at
        `base`; returns the new arena end."""
        r = self.shapes[i][0]
        rs = self._rs(self.row_start[k], i)
        total = C.c_int64(0)
        # slot = count + edge codes + 25% + 8: dense elements at code 0 / qmax are
        # the ones requantization can push outside the thresholds (SURVEY.md §0,
        # finding 2: on rows whose threshold sits among spikes dozens move at once)
        codes = self._sl(self.w_codes[k], i)
        qmax = (1 << self.bit_width) - 1
        edge = ((codes == 0) | (codes == qmax)).sum(dim=1, dtype=torch.int32)
        want = (rp[1:] - rp[:-1]) + edge
        N.check(N.lib.qftc_csr_plan_slots(_p(want), None, r, SLACK, _p(rs), C.byref(total),
                                          _stream()))
        rs += base
        end = base + int(total.value)
        self._ensure(g, k, end, keep=base)
        N.check(N.lib.qftc_csr_copy_rows(r, _p(rp), None, _p(col), _p(val), _p(rs),
                                         _p(g.col[k]), _p(g.val[k]), g.col[k].numel(),
                                         _stream()))
        self._rows(self.row_count[k], i).copy_(rp[1:] - rp[:-1])
        return end

    def _mirror_layout(self, g: _Group, src: int):
        """Give the other set the same slot layout and an arena of the same size."""
        dst = 1 - src
        if self._layout(g)[2]:  # contiguous members: one copy of the group's row starts
            p0 = int(self.rpoff[self.pos[g.members[0]]])
            p1 = int(self.rpoff[self.pos[g.members[-1]] + 1])
            self.row_start[dst][p0:p1].copy_(self.row_start[src][p0:p1])
        else:
            for i in g.members:
                self._rs(self.row_start[dst], i).copy_(self._rs(self.row_start[src], i))
        need = g.col[src].numel()
        if g.col[dst] is None or g.col[dst].numel() < need:
            g.col[dst], g.val[dst] = self._alloc(need)

    def _mirror_all(self):
        for g in self.groups:
            self._mirror_layout(g, self.cur)
            if g.plan is not None:
                self._set_arena(g)

    # ------------------------------------------------------------------ init
    def init_from_weights(self, weight_fn, fraction: float = 0.01, kind="percentile"):
        """Decompose every tensor on the device (decompose_weight, quantize.hpp:301-314).

        ``weight_fn(i)`` returns the fp32 [rows, cols] CUDA tensor of tensor i."""
        k = kind_from_name(kind)
        self.outlier_fraction, self.threshold_kind = float(fraction), int(k)
        cur = self.cur
        for g in self.groups:
            base = 0
            for i in g.members:
                r, c = self.shapes[i]
                w = weight_fn(i)
                tmn, tmx = self._rows(self.t_min, i), self._rows(self.t_max, i)
                N.check(N.lib.qftc_outlier_thresholds(_p(w), r, c, float(fraction), k, _p(tmn),
                                                      _p(tmx), _stream()))
                rp = torch.empty(r + 1, dtype=torch.int32, device=self.device)
                cap = int(fraction * r * c) + 4 * r + 1024
                while True:
                    col, val = self._alloc(cap)
                    nnz = C.c_int64(0)
                    rc = N.lib.qftc_decompose_dense_sparse(
                        _p(w), r, c, _p(tmn), _p(tmx), self.bit_width,
                        _p(self._sl(self.w_codes[cur], i)), _p(self._rows(self.w_scale, i)),
                        _p(self._rows(self.w_zp, i)), _p(rp), _p(col), _p(val), cap,
                        C.byref(nnz), _stream())
                    if rc == N.QFTC_EOVERFLOW:
                        cap = int(nnz.value) + 1024
                        continue
                    N.check(rc)
                    break
                base = self._place_strict(g, i, cur, base, rp, col, val)
                del w, col, val
            self._mirror_layout(g, cur)
        self._make_plans()

    def init_from_host(self, tensors: Sequence[dict], fraction: Optional[float] = None,
                       kind="percentile"):
        """Upload reference-layout state (e.g. from the CPU oracle).  Each dict holds
        codes, scale, zero_point, t_min, t_max, row_ptr, col_idx, values (the
        DenseSparseWeight) and optionally m_codes, m_scale, m_zero_point.  `fraction` /
        `kind`: the outlier config the thresholds were computed with (recorded for
        save_checkpoint)."""
        cur = self.cur
        if fraction is not None:
            self.outlier_fraction = float(fraction)
            self.threshold_kind = int(kind_from_name(kind))

        def dv(a, dt):
            return torch.as_tensor(np.ascontiguousarray(a)).to(self.device, dt)

        for g in self.groups:
            base = 0
            for i in g.members:
                t = tensors[i]
                self._sl(self.w_codes[cur], i).copy_(dv(t["codes"], torch.uint8))
                self._rows(self.w_scale, i).copy_(dv(t["scale"], torch.float32))
                self._rows(self.w_zp, i).copy_(dv(t["zero_point"], torch.int32))
                self._rows(self.t_min, i).copy_(dv(t["t_min"], torch.float32))
                self._rows(self.t_max, i).copy_(dv(t["t_max"], torch.float32))
                if "m_codes" in t:
                    self._sl(self.m_codes[cur], i).copy_(dv(t["m_codes"], torch.uint8))
                    self._rows(self.m_scale[cur], i).copy_(dv(t["m_scale"], torch.float32))
                    self._rows(self.m_zp[cur], i).copy_(dv(t["m_zero_point"], torch.int32))
                rp = dv(t["row_ptr"], torch.int32)
                col = dv(np.append(np.asarray(t["col_idx"], np.int32), np.int32(0)), torch.int32)
                val = dv(np.append(np.asarray(t["values"], np.float32), np.float32(0)),
                         torch.float32)
                base = self._place_strict(g, i, cur, base, rp, col, val)
            self._mirror_layout(g, cur)
        self._make_plans()

    # ------------------------------------------------------------------ plans
    def _descs(self, g: _Group, members: Optional[List[int]] = None):
        members = g.members if members is None else members
        arr = (N.LionTensorC * len(members))()
        for j, i in enumerate(members):
            r, c = self.shapes[i]
            d = arr[j]
            d.rows, d.cols = r, c
            for k in range(2):
                d.w_codes[k] = self._sl(self.w_codes[k], i).data_ptr()
                d.row_start[k] = self._rs(self.row_start[k], i).data_ptr()
                d.row_count[k] = self._rows(self.row_count[k], i).data_ptr()
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
        cols = (C.c_void_p * 2)(*[t.data_ptr() for t in g.col])
        vals = (C.c_void_p * 2)(*[t.data_ptr() for t in g.val])
        caps = (C.c_int64 * 2)(*[t.numel() for t in g.col])
        return cols, vals, caps

    def _set_arena(self, g: _Group):
        cols, vals, caps = self._arena_args(g)
        N.check(N.lib.qftc_plan_set_arena(g.plan, cols, vals, caps))
        for ch in self.chunks:
            if ch["group"] is g:
                N.check(N.lib.qftc_plan_set_arena(ch["plan"], cols, vals, caps))

    def make_chunk_plans(self, max_params: int = 256 << 20) -> List[dict]:
        """Split every launch group into runs of consecutive tensors of <= max_params
        (one plan each).  A chunk is one contiguous range of every flat array, so a host
        pipeline can stream chunk i+1 in while chunk i steps and chunk i-1 streams out."""
        for ch in self.chunks:
            N.lib.qftc_plan_destroy(ch["plan"])
        self.chunks = []
        for g in self.groups:
            run, acc = [], 0
            runs = []
            for i in g.members:
                sz = self.shapes[i][0] * self.shapes[i][1]
                if run and acc + sz > max_params:
                    runs.append(run)
                    run, acc = [], 0
                run.append(i)
                acc += sz
            if run:
                runs.append(run)
            for run in runs:
                arr = self._descs(g, run)
                cols, vals, caps = self._arena_args(g)
                plan = C.c_void_p()
                N.check(N.lib.qftc_plan_create(C.byref(plan), arr, len(run), self.bit_width,
                                               self.grad_kind, cols, vals, caps, _stream()))
                p0, p1 = self.pos[run[0]], self.pos[run[-1]] + 1
                self.chunks.append(dict(group=g, members=run, plan=plan, p0=p0, p1=p1))
        return self.chunks

    def chunk_ranges(self, ch: dict, k: int) -> dict:
        """Flat-array ranges of a chunk (element offsets) and its arena range in set k."""
        p0, p1 = ch["p0"], ch["p1"]
        a0 = int(self.row_start[k][int(self.rpoff[p0])].item())
        a1 = int(self.row_start[k][int(self.rpoff[p1]) - 1].item())
        return dict(code=(int(self.off[p0]), int(self.off[p1])),
                    row=(int(self.roff[p0]), int(self.roff[p1])),
                    rs=(int(self.rpoff[p0]), int(self.rpoff[p1])), arena=(a0, a1))

    def step_chunk(self, ch: dict, flip: int, h, stream_handle):
        N.check(N.lib.qftc_plan_step(ch["plan"], flip, h, stream_handle))

    def _make_plans(self):
        for g in self.groups:
            if g.plan is not None:
                N.lib.qftc_plan_destroy(g.plan)
            arr = self._descs(g)
            cols, vals, caps = self._arena_args(g)
            plan = C.c_void_p()
            N.check(N.lib.qftc_plan_create(C.byref(plan), arr, len(g.members), self.bit_width,
                                           self.grad_kind, cols, vals, caps, _stream()))
            g.plan = plan
            self._layout(g)  # the re-plan bookkeeping, off the checked step's path
        self._plan_order = None

    def step_plans(self):
        """The width classes' plans in the order one step launches them concurrently
        (qftc_plans_step): the smaller classes first, each capped at QFT_WIDE_CTAS resident
        CTAs per SM (default 0: no cap), so they can co-reside with the dominant class, which goes last
        and fills the rest of the GPU.  QFT_SERIAL_GROUPS=1 steps the classes one after the
        other on one stream instead."""
        if self._plan_order is None:
            dom = max(self.groups, key=lambda g: g.rows * g.cols)
            order = [g for g in self.groups if g is not dom] + [dom]
            cap = int(os.environ.get("QFT_WIDE_CTAS", "0"))
            for g in order[:-1]:
                N.check(N.lib.qftc_plan_set_ctas_per_sm(g.plan, cap))
            arr = (C.c_void_p * len(order))(*[g.plan.value for g in order])
            self._plan_order = (order, arr)
        return self._plan_order

    def enqueue_step(self, flip: int, h, stream_handle):
        """Enqueue one step over every width class (no host synchronisation)."""
        if len(self.groups) > 1 and os.environ.get("QFT_SERIAL_GROUPS", "0") != "1":
            order, arr = self.step_plans()
            N.check(N.lib.qftc_plans_step(arr, len(order), flip, h, stream_handle))
        else:
            for g in self.groups:
                N.check(N.lib.qftc_plan_step(g.plan, flip, h, stream_handle))

    def __del__(self):
        for ch in getattr(self, "chunks", []):
            try:
                N.lib.qftc_plan_destroy(ch["plan"])
            except Exception:
                pass
        self.chunks = []
        for g in getattr(self, "groups", []):
            if g.plan is not None:
                try:
                    N.lib.qftc_plan_destroy(g.plan)
                except Exception:
                    pass
                g.plan = None

    def ensure_arena_capacity(self, cap: int):
        """Give every group's arenas (both sets) >= cap entries (collectives over arenas
        need a rank-uniform size); keeps the current set's content."""
        for g in self.groups:
            for k in range(2):
                if g.col[k].numel() < cap:
                    col, val = self._alloc(cap)
                    if k == self.cur:
                        n = g.col[k].numel()
                        col[:n].copy_(g.col[k])
                        val[:n].copy_(g.val[k])
                    g.col[k], g.val[k] = col, val
            if g.plan is not None:
                self._set_arena(g)

    # ------------------------------------------------------------------ the step
    def launches_per_step(self) -> int:
        return len(self.groups)

    def step(self, lr=1e-4, beta1=0.9, beta2=0.99, weight_decay=0.0, check: bool = False):
        """One quantized Lion step over the whole model (lion_step_quantized,
        optimizer.hpp:85-120): one fused kernel launch per width class, enqueued on the
        current stream without host synchronisation.  ``check=True`` also synchronises,
        validates, and transparently re-plans CSR slots that overflowed and re-runs
        (the step's inputs are intact in the other set)."""
        h = N.hyper(lr, beta1, beta2, weight_decay)
        flip = self.cur
        self._refuse_if_overflowed("step")
        self.enqueue_step(flip, h, _stream())
        self.cur = 1 - flip
        self.steps += 1
        self._last = (flip, h)
        if check:
            self._check(flip, h)

    def _refuse_if_overflowed(self, what: str):
        """A step enqueued with check=False that overflowed a CSR slot left its output set
        incomplete (every consumer clamps counts to the slot, so nothing reads out of
        bounds, but outliers are missing).  The flag is a mapped host word, visible without
        a synchronisation once that step ran: refuse to build on the state."""
        for g in self.groups:
            if N.lib.qftc_plan_pending_overflow(g.plan):
                raise N.CsrOverflow(
                    f"{what}: a previous step(check=False) overflowed a CSR slot of the "
                    f"{g.cols}-column group; its output is incomplete -- call recover() "
                    "(re-plans and re-runs that step from its intact inputs) before "
                    "feeding the next gradient")

    def recover(self):
        """Repair the last step after an unchecked overflow: re-plan the overflowed
        groups' output slots and re-run the step from its input set (the ping-pong inputs
        and the gradient buffers must still hold that step's inputs)."""
        if getattr(self, "_last", None) is None:
            return
        self._check(*self._last)

    def _layout(self, g: _Group):
        """(row-start positions of the group's tensors in the flat row_start arrays, their
        indices in the group's scanned capacities, members contiguous?) -- built once
        (numpy; 200+ members) and kept on the device."""
        if g.layout_idx is None:
            pos, idx, rb = [], [], 0
            for i in g.members:
                r = self.shapes[i][0]
                p0 = int(self.rpoff[self.pos[i]])
                pos.append(np.arange(p0, p0 + r + 1, dtype=np.int64))
                idx.append(np.arange(rb, rb + r + 1, dtype=np.int64))
                rb += r
            ps = [self.pos[i] for i in g.members]
            contiguous = ps == list(range(ps[0], ps[0] + len(ps)))
            g.layout_idx = (torch.from_numpy(np.concatenate(pos)).to(self.device),
                            torch.from_numpy(np.concatenate(idx)).to(self.device), contiguous)
            # first use of the re-plan's scan / gather / scatter kernels, on scratch of the
            # same sizes: their lazy module loads (~30 ms) stay out of the first checked
            # step that overflows
            caps = torch.zeros(g.rows, dtype=torch.int64, device=self.device)
            cum = torch.zeros(g.rows + 1, dtype=torch.int64, device=self.device)
            torch.cumsum(caps, 0, out=cum[1:])
            scratch = torch.zeros_like(self.row_start[0])
            scratch.index_copy_(0, g.layout_idx[0],
                                cum.index_select(0, g.layout_idx[1]).to(torch.int32))
            int(cum[-1].item())
        return g.layout_idx

    def _replan(self, g: _Group, k: int):
        """Slots of set k re-sized from its (true) counts plus, as at placement
        (_place_strict), the dense elements at code 0 / qmax of the step's output codes:
        only those can become new outliers in a stable-tier step, so the padding keeps the
        no-overflow guarantee of the placement after a replan.  Rows that overflow are
        drifting (a large lr moves codes every step), so a re-planned slot also holds
        GROWTH_STEPS steps of the row's last growth (its count minus the step's input count), and
        every re-plan of the group widens the headroom -- count/4 more per level, the
        slack 8 -> 32 -> 64 entries -- instead of re-planning again the next step.  Batched over the group: one
        row-count pass, one scan, one scatter into the slot starts, one synchronisation."""
        dev = self.device
        rs_pos, scan_idx, contiguous = self._layout(g)
        lvl = min(g.replans, 3)
        # one pass over the output codes per tensor run (qftc_csr_replan_caps): edge codes,
        # growth, headroom -> per-row capacities, no temporaries
        caps = torch.empty(g.rows, dtype=torch.int64, device=dev)
        runs = ([(g.members[0], g.rows)] if contiguous else
                [(i, self.shapes[i][0]) for i in g.members])
        r0 = 0
        for i, rows in runs:
            N.check(N.lib.qftc_csr_replan_caps(
                _p(self._sl(self.w_codes[k], i)), rows, g.cols, self.bit_width,
                _p(self._rows(self.row_count[k], i)), _p(self._rows(self.row_count[1 - k], i)),
                lvl, GROWTH_STEPS, _p(caps[r0:r0 + rows]), _stream()))
            r0 += rows
        cum = torch.zeros(caps.numel() + 1, dtype=torch.int64, device=dev)
        torch.cumsum(caps, 0, out=cum[1:])
        total = int(cum[-1].item())
        if total >= 2 ** 31:
            raise OverflowError(f"CSR arena of the {g.cols}-column group: {total} entries")
        self.row_start[k].index_copy_(0, rs_pos, cum.index_select(0, scan_idx).to(torch.int32))
        g.replans += 1
        if g.col[k].numel() < total:  # grow with headroom: a drifting state re-plans again
            g.col[k], g.val[k] = self._alloc(total + total // 2)

    def _check(self, flip, h):
        out = 1 - flip
        for g in self.groups:
            replanned = False
            while True:
                rc = N.lib.qftc_plan_result(g.plan, None, _stream())
                if rc == N.QFTC_EOVERFLOW:
                    self._replan(g, out)
                    self._set_arena(g)
                    N.check(N.lib.qftc_plan_step(g.plan, flip, h, _stream()))
                    replanned = True
                    self.replans += 1
                    continue
                N.check(rc)
                break
            if replanned:  # the dead input set takes the new layout for the next step
                self._mirror_layout(g, out)
                self._set_arena(g)

    def kernel_names(self) -> List[str]:
        """The main kernel instance each width class ran in the last step (per group,
        e.g. ``rows_kernel<128,5,3,2,4096,8>``; see ``qftc_plan_kernel_name``)."""
        return [N.lib.qftc_plan_kernel_name(g.plan).decode() for g in self.groups]

    def tier_rows(self) -> Tuple[int, int]:
        """(stable-tier rows, general-tier rows) of the last step over all groups
        (synchronises)."""
        st = gen = 0
        for g in self.groups:
            a, b = C.c_int64(0), C.c_int64(0)
            N.check(N.lib.qftc_plan_tier_rows(g.plan, C.byref(a), C.byref(b), _stream()))
            st += a.value
            gen += b.value
        return st, gen

    def tiers(self) -> Tuple[int, int, int]:
        """(stable, GEN, general) rows of the last step over all groups (synchronises):
        the pass-through rows kernel, the requantizing GEN rows kernel, step_kernel."""
        t = [0, 0, 0]
        if not hasattr(N.lib, "qftc_plan_tiers"):  # an older library loaded for an A/B
            a, b = self.tier_rows()
            return a, 0, b
        for g in self.groups:
            arr = (C.c_int64 * 3)()
            N.check(N.lib.qftc_plan_tiers(g.plan, arr, _stream()))
            for k in range(3):
                t[k] += arr[k]
        return t[0], t[1], t[2]

    def check(self):
        """Synchronise and validate the last step (raises on overflow / bad rows)."""
        for g in self.groups:
            N.check(N.lib.qftc_plan_result(g.plan, None, _stream()))

    # ------------------------------------------------------------------ export
    def nnz(self) -> int:
        return int(self.row_count[self.cur].sum().item())

    def group_nnz(self, g: _Group, k: Optional[int] = None) -> int:
        k = self.cur if k is None else k
        return int(sum(self._rows(self.row_count[k], i).sum().item() for i in g.members))

    def strict_csr(self, i: int):
        """Tensor i's outliers as the reference's strict CSR (SparseOutliers,
        quantize.hpp:48-57), compacted from the slotted CSR on the device:
        (row_ptr [rows+1], col_idx [nnz], values [nnz]) device tensors."""
        cur = self.cur
        g = self.groups[self.group_of[i]]
        r = self.shapes[i][0]
        cnt = self._rows(self.row_count[cur], i)
        n = int(cnt.sum().item())
        rp = torch.empty(r + 1, dtype=torch.int32, device=self.device)
        col, val = self._alloc(n)
        nnz = C.c_int64(0)
        N.check(N.lib.qftc_csr_compact(r, _p(self._rs(self.row_start[cur], i)), _p(cnt),
                                       _p(g.col[cur]), _p(g.val[cur]), _p(rp), _p(col), _p(val),
                                       col.numel(), C.byref(nnz), _stream()))
        return rp, col[:n], val[:n]

    def export_tensor(self, i: int) -> dict:
        """Reference-layout host copy of tensor i (DenseSparseWeight + momentum); the
        slotted CSR is compacted into the strict one on the device."""
        cur = self.cur
        rp, col, val = self.strict_csr(i)
        n = col.numel()
        return dict(
            codes=self._sl(self.w_codes[cur], i).cpu().numpy(),
            scale=self._rows(self.w_scale, i).cpu().numpy(),
            zero_point=self._rows(self.w_zp, i).cpu().numpy(),
            t_min=self._rows(self.t_min, i).cpu().numpy(),
            t_max=self._rows(self.t_max, i).cpu().numpy(),
            row_ptr=rp.cpu().numpy(),
            col_idx=col[:n].cpu().numpy(),
            values=val[:n].cpu().numpy(),
            m_codes=self._sl(self.m_codes[cur], i).cpu().numpy(),
            m_scale=self._rows(self.m_scale[cur], i).cpu().numpy(),
            m_zero_point=self._rows(self.m_zp[cur], i).cpu().numpy(),
        )

    def reconstruct_into(self, i: int, out: torch.Tensor, nrows: Optional[int] = None):
        """Expand the first `nrows` rows of tensor i into `out` (f32 or bf16, [nrows, cols])."""
        cur = self.cur
        g = self.groups[self.group_of[i]]
        r, c = self.shapes[i]
        nrows = r if nrows is None else nrows
        N.check(N.lib.qftc_reconstruct_slots(
            _p(self._sl(self.w_codes[cur], i)), nrows, c, _p(self._rows(self.w_scale, i)),
            _p(self._rows(self.w_zp, i)), _p(self._rs(self.row_start[cur], i)),
            _p(self._rows(self.row_count[cur], i)), _p(g.col[cur]), _p(g.val[cur]), _p(out),
            0 if out.dtype == torch.float32 else 1, _stream()))
        return out

    def csr_index(self, i: int) -> torch.Tensor:
        """Tensor i's per-(row, 32-column) CSR slot index (qftc_dequant_gemm_index) for the
        CURRENT state: pass it as ``index=`` to linear / linear_backward while the weights
        are unchanged (the micro-batches between two steps) and the GEMMs skip its rebuild."""
        cur = self.cur
        g = self.groups[self.group_of[i]]
        r, c = self.shapes[i]
        idx = torch.empty(int(N.lib.qftc_dequant_gemm_workspace_bytes(r, c)), dtype=torch.uint8,
                          device=self.device)
        N.check(N.lib.qftc_dequant_gemm_index(
            _p(self._rs(self.row_start[cur], i)), _p(self._rows(self.row_count[cur], i)),
            _p(g.col[cur]), r, c, _p(idx), _stream()))
        return idx

    def linear(self, i: int, x: torch.Tensor, out: Optional[torch.Tensor] = None,
               index: Optional[torch.Tensor] = None) -> torch.Tensor:
        """The forward consumer of tensor i: y = x . W_i^T (network.hpp:113-129), x bf16
        [M, cols] -> y bf16 [M, rows], with W_i dequantized inside the GEMM's operand producer
        (qftc_dequant_gemm: tcgen05 tensor cores read RNE(reconstruct(W_i)) built in shared
        memory from the u8 codes and the CSR outliers; W_i never exists in HBM as bf16)."""
        cur = self.cur
        g = self.groups[self.group_of[i]]
        r, c = self.shapes[i]
        if x.dtype != torch.bfloat16 or x.dim() != 2 or x.shape[1] != c or not x.is_contiguous():
            raise ValueError(f"linear: x must be a contiguous bf16 [M, {c}] tensor")
        y = out if out is not None else torch.empty((x.shape[0], r), dtype=torch.bfloat16,
                                                    device=x.device)
        if index is not None:  # csr_index(i) of the current state
            N.check(N.lib.qftc_dequant_gemm_prebuilt(
                _p(x), x.shape[0], c, _p(self._sl(self.w_codes[cur], i)), r,
                _p(self._rows(self.w_scale, i)), _p(self._rows(self.w_zp, i)),
                _p(g.col[cur]), _p(g.val[cur]), _p(index), _p(y), _stream()))
            return y
        need = int(N.lib.qftc_dequant_gemm_workspace_bytes(r, c))
        ws = getattr(self, "_dq_ws", None)
        if ws is None or ws.numel() < need:
            ws = self._dq_ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        N.check(N.lib.qftc_dequant_gemm(
            _p(x), x.shape[0], c, _p(self._sl(self.w_codes[cur], i)), r,
            _p(self._rows(self.w_scale, i)), _p(self._rows(self.w_zp, i)),
            _p(self._rs(self.row_start[cur], i)), _p(self._rows(self.row_count[cur], i)),
            _p(g.col[cur]), _p(g.val[cur]), _p(y), _p(ws), _stream()))
        return y

    def linear_backward(self, i: int, dy: torch.Tensor, out: Optional[torch.Tensor] = None,
                        index: Optional[torch.Tensor] = None) -> torch.Tensor:
        """The backward's input gradient through tensor i: dx = dy . W_i (network.hpp:145
        backward_core in_grad = matmul(out_grad, w)), dy bf16 [M, rows] -> dx bf16 [M, cols],
        with W_i dequantized inside the GEMM's operand producer (qftc_dequant_gemm_t: the
        tensor cores read RNE(reconstruct(W_i)) as an MN-major operand built in shared memory
        from the u8 codes and the CSR outliers)."""
        cur = self.cur
        g = self.groups[self.group_of[i]]
        r, c = self.shapes[i]
        if dy.dtype != torch.bfloat16 or dy.dim() != 2 or dy.shape[1] != r or not dy.is_contiguous():
            raise ValueError(f"linear_backward: dy must be a contiguous bf16 [M, {r}] tensor")
        dx = out if out is not None else torch.empty((dy.shape[0], c), dtype=torch.bfloat16,
                                                     device=dy.device)
        if index is not None:  # csr_index(i) of the current state
            N.check(N.lib.qftc_dequant_gemm_t_prebuilt(
                _p(dy), dy.shape[0], r, _p(self._sl(self.w_codes[cur], i)), c,
                _p(self._rows(self.w_scale, i)), _p(self._rows(self.w_zp, i)),
                _p(g.col[cur]), _p(g.val[cur]), _p(index), _p(dx), _stream()))
            return dx
        need = int(N.lib.qftc_dequant_gemm_t_workspace_bytes(r, c))
        ws = getattr(self, "_dqt_ws", None)
        if ws is None or ws.numel() < need:
            ws = self._dqt_ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        N.check(N.lib.qftc_dequant_gemm_t(
            _p(dy), dy.shape[0], r, _p(self._sl(self.w_codes[cur], i)), c,
            _p(self._rows(self.w_scale, i)), _p(self._rows(self.w_zp, i)),
            _p(self._rs(self.row_start[cur], i)), _p(self._rows(self.row_count[cur], i)),
            _p(g.col[cur]), _p(g.val[cur]), _p(dx), _p(ws), _stream()))
        return dx

    def expand_table(self, outs: Sequence[torch.Tensor], rows: Optional[Sequence[int]] = None):
        """ctypes table (qftc_expand_tensor[n]) expanding tensor i's first rows[i] rows into
        outs[i] from the CURRENT state; reusable while `cur` and the buffers are unchanged."""
        cur = self.cur
        n = len(self.shapes)
        tab = (N.ExpandTensorC * n)()
        bf16 = None
        for i, (r, c) in enumerate(self.shapes):
            o = outs[i]
            isb = o.dtype == torch.bfloat16
            if bf16 is None:
                bf16 = isb
            if isb != bf16 or o.dtype not in (torch.float32, torch.bfloat16):
                raise ValueError("expand: every output must be f32, or every output bf16")
            g = self.groups[self.group_of[i]]
            t = tab[i]
            t.rows = r if rows is None else int(rows[i])
            t.cols = c
            if o.numel() < t.rows * c:
                raise ValueError(f"expand: output {i} holds {o.numel()} < {t.rows * c} elements")
            t.codes = self._sl(self.w_codes[cur], i).data_ptr()
            t.scale = self._rows(self.w_scale, i).data_ptr()
            t.zero_point = self._rows(self.w_zp, i).data_ptr()
            t.row_start = self._rs(self.row_start[cur], i).data_ptr()
            t.row_count = self._rows(self.row_count[cur], i).data_ptr()
            t.col_idx = g.col[cur].data_ptr()
            t.values = g.val[cur].data_ptr()
            t.out = o.data_ptr()
        return tab, 1 if bf16 else 0

    def expand_plan(self, outs: Sequence[torch.Tensor], rows: Optional[Sequence[int]] = None):
        """An ExpandPlan over every tensor (one launch per run, any number of tensors),
        valid while `cur` and the buffers are unchanged (the ping-pong set flips each step:
        build one plan per set)."""
        tab, bf16 = self.expand_table(outs, rows)
        return ExpandPlan(tab, bf16, keep=(self, list(outs)))

    def expand(self, outs: Sequence[torch.Tensor], rows: Optional[Sequence[int]] = None,
               table=None):
        """Reconstruct every tensor (dense dequant + CSR overwrite, quantize.hpp:331-338)
        into outs (all f32 or all bf16) with one grouped launch -- the weight expansion
        for the next forward (network.hpp:208-211)."""
        self._refuse_if_overflowed("expand")
        tab, bf16 = table if table is not None else self.expand_table(outs, rows)
        N.check(N.lib.qftc_expand(C.cast(tab, C.c_void_p), len(tab), bf16, _stream()))
        return outs

    def reconstruct(self, i: int, dtype=torch.float32) -> torch.Tensor:
        """Expand tensor i (dequant + CSR overwrite) to f32 or bf16 for the next forward."""
        cur = self.cur
        g = self.groups[self.group_of[i]]
        r, c = self.shapes[i]
        out = torch.empty((r, c), dtype=dtype, device=self.device)
        N.check(N.lib.qftc_reconstruct_slots(
            _p(self._sl(self.w_codes[cur], i)), r, c, _p(self._rows(self.w_scale, i)),
            _p(self._rows(self.w_zp, i)), _p(self._rs(self.row_start[cur], i)),
            _p(self._rows(self.row_count[cur], i)), _p(g.col[cur]), _p(g.val[cur]), _p(out),
            0 if dtype == torch.float32 else 1, _stream()))
        return out


class ExpandPlan:
    """A weight expansion whose tensor table lives on the device (qftc_expand_plan): one
    kernel launch per run() for any number of tensors (the forward consumer's bf16 / f32
    weights, network.hpp:199-212)."""

    def __init__(self, table, bf16: int, keep=None):
        self._keep = keep  # the buffers the table points into
        self.n = len(table)
        self.handle = C.c_void_p()
        N.check(N.lib.qftc_expand_plan_create(C.byref(self.handle), table, len(table), int(bf16),
                                              _stream()))

    def run(self, stream=None):
        N.check(N.lib.qftc_expand_plan_run(self.handle, stream if stream is not None else _stream()))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                N.lib.qftc_expand_plan_destroy(h)
            except Exception:
                pass
            self.handle = None
