"""ZeRO-1 row-sharded QFT Lion step over NCCL.

Every quantity of the update is per ROW (scales, zero points, thresholds, the m'
min/max, the CSR segment), so a row-range shard needs no communication inside
the update.  The exchange steps are the data-parallel ones:

1. ``reduce_scatter_tensor(SUM)`` of the fp gradient, laid out SHARD-MAJOR
   ([rank0's rows of every tensor | rank1's rows | ...], each rank block padded to
   the same length) so one collective hands every rank exactly its rows.  The sum
   is taken in fp before quantisation: the reference quantizes the full gradient
   once (gradflow.hpp:77), and quantize_state is per-row, so quantizing the
   shard rows of the summed gradient equals quantizing the full summed gradient.
2. the fused local step on the shard (grad kind f32/bf16: quantize_state(g) ->
   dequantize fused into the kernel); momentum stays sharded (ZeRO-1);
3. ``all_gather_into_tensor`` of the updated W codes, of the CSR row starts and
   counts and of the CSR entries.  By default only the USED entries travel
   (``packed_csr``): every rank packs its slotted arenas densely per width class
   (``qftc_csr_pack``), the ranks agree the largest packed size per class in the same
   all-reduce that carries the overflow flag (no extra host round trip), and each rank
   re-bases its packed row starts by ``rank * packed_size`` so receivers index the
   gathered entries directly.  ``packed_csr=False`` ships the whole slotted arenas
   (fixed rank-uniform capacity; rank k's slot offsets re-based by
   ``k * arena_capacity`` when read).

The local update is pluggable: on GPUs it is :class:`CudaShard` (the fused
sm_100a kernel through the C-ABI); the CPU tests plug the oracle in to check the
collective choreography with gloo.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

Shape = Tuple[int, int]


class ShardLayout:
    """Row ranges of every tensor per rank and the shard-major flat layout."""

    def __init__(self, shapes: Sequence[Shape], world: int):
        self.shapes = [(int(r), int(c)) for r, c in shapes]
        self.world = world
        self.widths = sorted({c for _, c in self.shapes})
        self.members: List[List[Tuple[int, int, int]]] = []   # per rank: (tensor, lo, hi)
        self.numel: List[int] = []
        self.rows: List[int] = []
        for k in range(world):
            mem = []
            for i, (r, c) in enumerate(self.shapes):
                lo, hi = (r * k) // world, (r * (k + 1)) // world
                if hi > lo:
                    mem.append((i, lo, hi))
            self.members.append(mem)
            self.numel.append(sum((hi - lo) * self.shapes[i][1] for i, lo, hi in mem))
            self.rows.append(sum(hi - lo for _, lo, hi in mem))
        self.pad = max(self.numel)                      # elements per rank block
        self.rp_pad = max(self.rows[k] + len(self.members[k]) for k in range(world))
        self.rpad = max(self.rows)
        # element offset of (rank k, j-th member) inside rank k's block
        self.off: List[List[int]] = []
        self.rpoff: List[List[int]] = []
        self.roff: List[List[int]] = []
        for k in range(world):
            o, rp, ro = [0], [0], [0]
            for i, lo, hi in self.members[k]:
                o.append(o[-1] + (hi - lo) * self.shapes[i][1])
                rp.append(rp[-1] + (hi - lo) + 1)
                ro.append(ro[-1] + (hi - lo))
            self.off.append(o)
            self.rpoff.append(rp)
            self.roff.append(ro)

    def shard_shapes(self, k: int) -> List[Shape]:
        return [(hi - lo, self.shapes[i][1]) for i, lo, hi in self.members[k]]

    def pack(self, grads: Sequence[torch.Tensor], out: torch.Tensor) -> torch.Tensor:
        """Write full per-tensor gradients into the shard-major flat buffer."""
        for k in range(self.world):
            base = k * self.pad
            for j, (i, lo, hi) in enumerate(self.members[k]):
                c = self.shapes[i][1]
                out[base + self.off[k][j]: base + self.off[k][j + 1]].copy_(
                    grads[i][lo:hi].reshape(-1))
        return out


class Zero1QftLion:
    """Row-sharded quantized Lion step for one rank of a process group."""

    def __init__(self, shapes: Sequence[Shape], local, group=None, arena_capacity: int = 0,
                 packed_csr: Optional[bool] = None):
        self.group = group
        if packed_csr is None:   # default on; QFT_ZERO1_PACKED=0 ships whole arenas (A/B)
            packed_csr = os.environ.get("QFT_ZERO1_PACKED", "1") != "0"
        self.packed = bool(packed_csr) and hasattr(local, "pack_csr")
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.layout = ShardLayout(shapes, self.world)
        self.local = local
        L = self.layout
        dev = local.device
        self.grad_full = torch.zeros(self.world * L.pad, dtype=local.grad_dtype, device=dev)
        self.codes_full = torch.empty(self.world * L.pad, dtype=torch.uint8, device=dev)
        self.rowstart_full = torch.empty(self.world * L.rp_pad, dtype=torch.int32, device=dev)
        self.count_full = torch.empty(self.world * L.rpad, dtype=torch.int32, device=dev)
        cap = int(arena_capacity) or local.arena_capacity()
        t = torch.tensor([cap], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)   # rank-uniform capacity
        self.cap = int(t.item())
        local.ensure_arena_capacity(self.cap)
        self.col_full = {c: torch.empty(self.world * self.cap, dtype=torch.int32, device=dev)
                         for c in L.widths}
        self.val_full = {c: torch.empty(self.world * self.cap, dtype=torch.float32, device=dev)
                         for c in L.widths}
        self.pcap = {c: 0 for c in L.widths}   # packed entries per rank and class, this step
        self.generation = 0                    # bumps when gathered buffers are reallocated
        self.launches = 0
        self.fused = False
        self._mapped = []

    # ------------------------------------------------------------------ the step
    def reduce_scatter_grads(self):
        dist.reduce_scatter_tensor(self.local.grad_shard(self.layout.pad), self.grad_full,
                                   op=dist.ReduceOp.SUM, group=self.group)

    def _state_parts(self):
        """(name, this rank's source tensor, entries per rank) of everything the all-gather
        ships; with packed_csr the row starts and entries are the packed ones."""
        L = self.layout
        if self.packed:
            rs, ents = self.local.pack_csr(self.pcap, {c: self.rank * self.pcap[c]
                                                       for c in L.widths}, L.rp_pad)
        else:
            rs = self.local.rowstart_shard(L.rp_pad)
            ents = {c: self.local.arena(c, self.cap) for c in L.widths}
        parts = [("codes", self.local.codes_shard(L.pad), L.pad),
                 ("rowstart", rs, L.rp_pad),
                 ("count", self.local.count_shard(L.rpad), L.rpad)]
        for c in L.widths:
            n = self.pcap[c] if self.packed else self.cap
            col, val = ents[c]
            parts += [(f"col{c}", col[:n], n), (f"val{c}", val[:n], n)]
        return parts

    def _full(self, name):
        if name == "grad":
            return self.grad_full
        if name == "codes":
            return self.codes_full
        if name == "rowstart":
            return self.rowstart_full
        if name == "count":
            return self.count_full
        return (self.col_full if name.startswith("col") else self.val_full)[int(name[3:])]

    def all_gather_state(self):
        for name, src, n in self._state_parts():
            if n:
                dist.all_gather_into_tensor(self._full(name)[:self.world * n], src,
                                            group=self.group)

    def gather_bytes_per_rank(self) -> int:
        """Bytes one rank contributes to the state all-gather of the last step."""
        L = self.layout
        n = sum(self.pcap.values()) if self.packed else self.cap * len(L.widths)
        return L.pad + 4 * L.rp_pad + 4 * L.rpad + 8 * n

    def _arena_base(self, k: int) -> int:
        """Offset of rank k's entries in the gathered arena that its row starts omit."""
        return 0 if getattr(self, "packed", False) else k * self.cap

    # ------------------------------------------------------------------ the fused path
    def enable_peer_memory(self):
        """the step over NVLink peer memory instead of NCCL.  Every
        rank maps (CUDA IPC) every peer's full bf16 gradient buffer and gathered buffers.
        The reduce-scatter is fused into the local update: the plans read their rows of
        the summed gradient straight from the peers' buffers and quantize them in one pass
        (``qftc_plan_set_peer_gradients`` -> ``k_rs_grad_quant``); the all-gather is a push
        of the rank's updated shard into every peer's gathered buffers (copy engines over
        the mapped pointers).  Host barriers order the ranks (the gradients are complete
        before anyone reads them; every push lands before anyone reuses a buffer)."""
        from . import _native as N
        names = ["grad", "codes", "rowstart", "count"] + \
                [f"col{c}" for c in self.layout.widths] + [f"val{c}" for c in self.layout.widths]
        buf = self._full
        mine = {}
        for n in names:
            h = C.create_string_buffer(64)
            off = C.c_int64(0)
            N.check(N.lib.qftc_ipc_handle(C.c_void_p(buf(n).data_ptr()), h, C.byref(off)))
            mine[n] = (h.raw, int(off.value))
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=self.group)
        self._close_peers()
        self.peer = []  # per rank: name -> device address
        for k in range(self.world):
            if k == self.rank:
                self.peer.append({n: buf(n).data_ptr() for n in names})
                continue
            d = {}
            for n in names:
                hb, off = allh[k][n]
                base = C.c_void_p()
                N.check(N.lib.qftc_ipc_open(hb, C.byref(base)))
                self._mapped.append(base)
                d[n] = base.value + off
            self.peer.append(d)
        # the local plans read their gradient rows from every rank's grad_full
        st = self.local.state
        esz = self.grad_full.element_size()
        deltas = (C.c_int64 * self.world)(*[
            self.peer[j]["grad"] + self.rank * self.layout.pad * esz - st.g_raw.data_ptr()
            for j in range(self.world)])
        for g in st.groups:
            N.check(N.lib.qftc_plan_set_peer_gradients(g.plan, deltas, self.world))
        self.fused = True
        self._mapped_generation = self.generation

    def _close_peers(self):
        from . import _native as N
        for b in getattr(self, "_mapped", []):
            N.lib.qftc_ipc_close(b)
        self._mapped = []

    def push_state(self):
        """The all-gather as a push: this rank's updated shard into slot `rank` of every
        rank's gathered buffers (mapped peer memory)."""
        from . import _native as N
        k = self.rank
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        parts = self._state_parts()
        for j in range(self.world):
            for name, src, n in parts:
                if not n:
                    continue
                esz = src.element_size()
                N.check(N.lib.qftc_copy_peer(C.c_void_p(self.peer[j][name] + k * n * esz),
                                             C.c_void_p(src.data_ptr()), n * esz, stream))

    def step_fused(self, lr=1e-4, beta1=0.9, beta2=0.99, weight_decay=0.0):
        """reduce-scatter fused into the update, then the push all-gather (enable first)."""
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)          # every rank's gradient is complete
        self.local.step(lr=lr, beta1=beta1, beta2=beta2, weight_decay=weight_decay)
        self.check_local()                      # synchronises; all-reduced overflow flag
        if self.generation != self._mapped_generation:  # gathered buffers reallocated
            self.enable_peer_memory()
        self.push_state()
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)          # every push has landed

    def check_local(self):
        """Every rank learns whether ANY rank's local step overflowed a CSR slot (one
        all-reduced flag): the overflowing ranks re-plan and re-run their step from its
        intact ping-pong inputs, then all ranks re-agree a uniform arena capacity, so the
        all-gather never ships a partial step or cuts off a grown arena."""
        ov = bool(getattr(self.local, "pending_overflow", lambda: False)())
        t = self._flag_and_sizes(ov)
        if t[0]:
            if ov:
                self.local.recover()
            self._agree_capacity()
            if self.packed:
                t = self._flag_and_sizes(False)
        if self.packed:
            self._agree_packed(t[1:])

    def _flag_and_sizes(self, ov: bool) -> List[int]:
        """ONE all-reduce(MAX) of [overflow flag, used entries per width class]."""
        vals = [1 if ov else 0]
        if self.packed:
            nnz = self.local.csr_nnz()
            vals += [int(nnz.get(c, 0)) for c in self.layout.widths]
        t = torch.tensor(vals, dtype=torch.int64, device=self.local.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return [int(x) for x in t.tolist()]

    def _agree_packed(self, maxnnz: Sequence[int]):
        """Per class: the rank-uniform packed size (max used entries, rounded to 32 so every
        rank's segment stays 128-byte aligned); grow the gathered buffers when it no
        longer fits (x1.25 headroom) -- row starts are int32, so world * size < 2^31."""
        dev = self.local.device
        for c, n in zip(self.layout.widths, maxnnz):
            n = (int(n) + 31) & ~31
            if self.world * n >= 2 ** 31:
                raise OverflowError(f"packed CSR all-gather: {self.world} x {n} entries of "
                                    f"width {c} exceed int32 row starts")
            self.pcap[c] = n
            if self.col_full[c].numel() < self.world * n:
                m = min(2 ** 31 - 1, self.world * (n + n // 4 + 32))
                self.col_full[c] = torch.empty(m, dtype=torch.int32, device=dev)
                self.val_full[c] = torch.empty(m, dtype=torch.float32, device=dev)
                self.generation += 1

    def _agree_capacity(self):
        t = torch.tensor([self.local.arena_capacity()], dtype=torch.int64,
                         device=self.local.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        cap = int(t.item())
        if cap > self.cap:
            self.cap = cap
            self.local.ensure_arena_capacity(cap)
            if self.packed:
                return                          # gathered buffers follow the packed sizes
            dev = self.local.device
            for c in self.layout.widths:
                self.col_full[c] = torch.empty(self.world * cap, dtype=torch.int32, device=dev)
                self.val_full[c] = torch.empty(self.world * cap, dtype=torch.float32, device=dev)
            self.generation += 1

    def step(self, lr=1e-4, beta1=0.9, beta2=0.99, weight_decay=0.0):
        self.reduce_scatter_grads()
        self.local.step(lr=lr, beta1=beta1, beta2=beta2, weight_decay=weight_decay)
        self.check_local()
        self.all_gather_state()

    # ------------------------------------------------------------------ the next forward's weights
    def gather_static(self):
        """All-gather the per-row weight params every expansion needs (scale, zero point:
        cached between threshold refreshes, so once), shard-major like the codes."""
        L = self.layout
        dev = self.local.device
        self.wscale_full = torch.empty(self.world * L.rpad, dtype=torch.float32, device=dev)
        self.wzp_full = torch.empty(self.world * L.rpad, dtype=torch.int32, device=dev)
        dist.all_gather_into_tensor(self.wscale_full, self.local.wscale_shard(L.rpad),
                                    group=self.group)
        dist.all_gather_into_tensor(self.wzp_full, self.local.wzp_shard(L.rpad), group=self.group)

    def expand_plan(self, outs: Sequence[torch.Tensor]):
        """ONE grouped expansion launch reading the gathered shard-major buffers directly:
        every (rank, tensor) row range is a table entry (codes, params, row starts, counts
        and the gathered entries -- rank k's arena re-based by k * capacity unless packed),
        writing rows [lo, hi) of the full output tensor (bf16 or f32) -- the next forward's
        weights (network.hpp:199-212).  Valid while ``generation`` is unchanged."""
        from . import _native as N
        from .engine import ExpandPlan
        if not hasattr(self, "wscale_full"):
            self.gather_static()
        L = self.layout
        pieces = [(k, j, ti, lo, hi) for k in range(self.world)
                  for j, (ti, lo, hi) in enumerate(L.members[k])]
        tab = (N.ExpandTensorC * len(pieces))()
        bf16 = outs[0].dtype == torch.bfloat16
        for n, (k, j, ti, lo, hi) in enumerate(pieces):
            r, c = L.shapes[ti]
            o = outs[ti]
            if (o.dtype == torch.bfloat16) != bf16 or o.numel() != r * c:
                raise ValueError(f"expand: output {ti} must be {r}x{c}, one dtype for all")
            t = tab[n]
            t.rows, t.cols = hi - lo, c
            esz = 1
            t.codes = self.codes_full.data_ptr() + (k * L.pad + L.off[k][j]) * esz
            t.scale = self.wscale_full.data_ptr() + 4 * (k * L.rpad + L.roff[k][j])
            t.zero_point = self.wzp_full.data_ptr() + 4 * (k * L.rpad + L.roff[k][j])
            t.row_start = self.rowstart_full.data_ptr() + 4 * (k * L.rp_pad + L.rpoff[k][j])
            t.row_count = self.count_full.data_ptr() + 4 * (k * L.rpad + L.roff[k][j])
            t.col_idx = self.col_full[c].data_ptr() + 4 * self._arena_base(k)
            t.values = self.val_full[c].data_ptr() + 4 * self._arena_base(k)
            t.out = o.data_ptr() + lo * c * o.element_size()
        return ExpandPlan(tab, 1 if bf16 else 0, keep=(self, list(outs)))

    # ------------------------------------------------------------------ views of the gathered state
    def gathered_tensor(self, i: int) -> dict:
        """Reference-layout copy (host numpy) of full tensor i from the gathered buffers."""
        L = self.layout
        r, c = L.shapes[i]
        codes = np.empty((r, c), np.uint8)
        row_ptr = [0]
        cols, vals = [], []
        for k in range(self.world):
            for j, (ti, lo, hi) in enumerate(L.members[k]):
                if ti != i:
                    continue
                base = k * L.pad
                codes[lo:hi] = self.codes_full[base + L.off[k][j]: base + L.off[k][j + 1]] \
                    .cpu().numpy().reshape(hi - lo, c)
                rs = self.rowstart_full[k * L.rp_pad + L.rpoff[k][j]:
                                        k * L.rp_pad + L.rpoff[k][j + 1]].cpu().numpy()
                cnt = self.count_full[k * L.rpad + L.roff[k][j]:
                                      k * L.rpad + L.roff[k][j + 1]].cpu().numpy()
                ca = self.col_full[c][self._arena_base(k):].cpu().numpy()
                va = self.val_full[c][self._arena_base(k):].cpu().numpy()
                for rr in range(hi - lo):
                    a0, n = int(rs[rr]), int(cnt[rr])
                    cols.append(ca[a0:a0 + n])
                    vals.append(va[a0:a0 + n])
                    row_ptr.append(row_ptr[-1] + n)
        return dict(codes=codes, row_ptr=np.asarray(row_ptr, np.int32),
                    col_idx=np.concatenate(cols) if cols else np.zeros(0, np.int32),
                    values=np.concatenate(vals) if vals else np.zeros(0, np.float32))


class CudaShard:
    """Local update on this rank's rows: the fused sm_100a step (QftModelState, raw
    fp gradient kind) with codes and arenas sized for the uniform collectives."""

    def __init__(self, layout: ShardLayout, rank: int, bit_width: int = 8,
                 grad_dtype=torch.float32, device="cuda"):
        from .engine import QftModelState
        self.layout, self.rank = layout, rank
        self.device = torch.device(device)
        self.grad_dtype = grad_dtype
        kind = "f32" if grad_dtype == torch.float32 else "bf16"
        self.state = QftModelState(layout.shard_shapes(rank), bit_width=bit_width,
                                   grad_kind=kind, device=device, pad_to=layout.pad,
                                   group_contiguous=False)

    def arena_capacity(self) -> int:
        return max(int(g.col[self.state.cur].numel()) for g in self.state.groups)

    def ensure_arena_capacity(self, cap: int):
        self.state.ensure_arena_capacity(cap)

    def grad_shard(self, pad: int) -> torch.Tensor:
        return self.state.g_raw[:pad]

    def step(self, **h):
        self.state.step(**h)

    def pending_overflow(self) -> bool:
        """Synchronise and read the plans' overflow flags (mapped host words)."""
        from . import _native as N
        torch.cuda.current_stream(self.device).synchronize()
        return any(N.lib.qftc_plan_pending_overflow(g.plan) for g in self.state.groups)

    def recover(self):
        self.state.recover()

    def codes_shard(self, pad: int) -> torch.Tensor:
        return self.state.w_codes[self.state.cur][:pad]

    def wscale_shard(self, rpad: int) -> torch.Tensor:
        return self._padded(self.state.w_scale, rpad)

    def wzp_shard(self, rpad: int) -> torch.Tensor:
        return self._padded(self.state.w_zp, rpad)

    def _padded(self, t: torch.Tensor, n: int) -> torch.Tensor:
        if t.numel() < n:
            out = torch.zeros(n, dtype=t.dtype, device=self.device)
            out[:t.numel()].copy_(t)
            return out
        return t[:n]

    def rowstart_shard(self, rp_pad: int) -> torch.Tensor:
        return self._padded(self.state.row_start[self.state.cur], rp_pad)

    def count_shard(self, rpad: int) -> torch.Tensor:
        return self._padded(self.state.row_count[self.state.cur], rpad)

    def csr_nnz(self) -> Dict[int, int]:
        """Used CSR entries per width class: one device reduction, one synchronisation."""
        st, widths = self.state, self.layout.widths
        if not hasattr(self, "_wrow"):
            w = np.concatenate([np.full(st.shapes[i][0], widths.index(st.shapes[i][1]), np.int64)
                                for i in st.order])
            self._wrow = torch.from_numpy(w).to(self.device)
        cnt = st.row_count[st.cur][:self._wrow.numel()].to(torch.float64)
        tot = torch.bincount(self._wrow, weights=cnt, minlength=len(widths)).tolist()
        return {c: int(tot[j]) for j, c in enumerate(widths)}

    def pack_csr(self, pcap: Dict[int, int], base: Dict[int, int], rp_pad: int):
        """The used entries of every width class packed densely (a qftc_csr_pack plan: three
        launches for all classes) and the packed row starts + base[class], in the row-start
        layout of rowstart_shard.  Returns (row starts [rp_pad], {class: (col, val)})."""
        from . import _native as N
        st, widths = self.state, self.layout.widths
        nw = len(widths)
        if getattr(self, "_pack_plan", None) is None:
            segs = (N.PackSegmentC * max(1, st.n))()
            for p, i in enumerate(st.order):          # flat positions of the row arrays
                r, c = st.shapes[i]
                segs[p].rows, segs[p].width = r, widths.index(c)
                segs[p].rs_off, segs[p].cnt_off = int(st.rpoff[p]), int(st.roff[p])
            plan = C.c_void_p()
            N.check(N.lib.qftc_csr_pack_plan_create(C.byref(plan), segs, st.n, nw, None))
            self._pack_plan = plan
            self._rs_out = torch.zeros(max(rp_pad, st.row_start[0].numel()), dtype=torch.int32,
                                       device=self.device)
            self._pk = {}
        out = {}
        for c in widths:
            n = max(32, int(pcap.get(c, 0)))
            if c not in self._pk or self._pk[c][0].numel() < n:
                m = n + n // 4
                self._pk[c] = (torch.empty(m, dtype=torch.int32, device=self.device),
                               torch.empty(m, dtype=torch.float32, device=self.device))
            out[c] = self._pk[c]
        k = st.cur
        grp = {g.cols: g for g in st.groups}
        P = C.c_void_p * nw
        col_in = P(*[(grp[c].col[k] if c in grp else out[c][0]).data_ptr() for c in widths])
        val_in = P(*[(grp[c].val[k] if c in grp else out[c][1]).data_ptr() for c in widths])
        col_out = P(*[out[c][0].data_ptr() for c in widths])
        val_out = P(*[out[c][1].data_ptr() for c in widths])
        bases = (C.c_int64 * nw)(*[int(base.get(c, 0)) for c in widths])
        stream = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        N.check(N.lib.qftc_csr_pack_run(self._pack_plan, C.c_void_p(st.row_start[k].data_ptr()),
                                        C.c_void_p(st.row_count[k].data_ptr()),
                                        C.cast(col_in, C.c_void_p), C.cast(val_in, C.c_void_p),
                                        C.cast(col_out, C.c_void_p),
                                        C.cast(val_out, C.c_void_p), bases,
                                        C.c_void_p(self._rs_out.data_ptr()), stream))
        return self._rs_out[:rp_pad], out

    def __del__(self):
        plan = getattr(self, "_pack_plan", None)
        if plan is not None:
            try:
                from . import _native as N
                N.lib.qftc_csr_pack_plan_destroy(plan)
            except Exception:
                pass

    def arena(self, width: int, cap: int):
        g = next((g for g in self.state.groups if g.cols == width), None)
        if g is None:
            z = torch.zeros(cap, dtype=torch.int32, device=self.device)
            return z, z.view(torch.float32)
        k = self.state.cur
        return g.col[k][:cap], g.val[k][:cap]
