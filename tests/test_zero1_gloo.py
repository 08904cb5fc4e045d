"""CPU, world_size 2 over gloo: the ZeRO-1 row-sharded step (reduce-scatter of the fp
gradient -> per-rank update of its rows -> all-gather of codes, row_ptr and CSR
arenas) reassembles exactly the single-process reference step on the summed
gradient.  The local update is the CPU oracle (test double); on GPUs it is the
fused sm_100a kernel (CudaShard).  Gradients are k * 2^-24 with small integers k,
so the fp32 sum is exact in any reduction order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

SHAPES = [(9, 64), (1, 64), (6, 32), (5, 64), (7, 32)]
BW, FRAC = 8, 0.05


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleShard:
    """Local-update test double with CudaShard's buffer interface, computed by the oracle."""

    def __init__(self, layout, rank, port, full_w, full_m):
        from oracle.oracle import DenseSparse
        self.layout, self.rank, self.port = layout, rank, port
        self.device = torch.device("cpu")
        self.grad_dtype = torch.float32
        self.mem = layout.members[rank]
        self.w, self.m = [], []
        for i, lo, hi in self.mem:
            d = full_w[i]
            a, b = int(d.row_ptr[lo]), int(d.row_ptr[hi])
            self.w.append(DenseSparse(d.codes[lo:hi].copy(), d.scale[lo:hi].copy(),
                                      d.zero_point[lo:hi].copy(),
                                      (d.row_ptr[lo:hi + 1] - a).astype(np.int32),
                                      d.col_idx[a:b].copy(), d.values[a:b].copy(),
                                      d.t_min[lo:hi].copy(), d.t_max[lo:hi].copy(), BW))
            mq, ms, mz = full_m[i]
            self.m.append((mq[lo:hi].copy(), ms[lo:hi].copy(), mz[lo:hi].copy()))
        self.g = torch.zeros(layout.pad, dtype=torch.float32)
        self.cap = 0
        self._publish()

    def _publish(self):
        L, k = self.layout, self.rank
        self.codes = torch.zeros(L.pad, dtype=torch.uint8)
        self.rowstart = torch.zeros(L.rp_pad, dtype=torch.int32)
        self.counts = torch.zeros(L.rpad, dtype=torch.int32)
        self.arenas = {}
        base = {c: 0 for c in L.widths}
        cols = {c: [] for c in L.widths}
        vals = {c: [] for c in L.widths}
        for j, (i, lo, hi) in enumerate(self.mem):
            c = L.shapes[i][1]
            d = self.w[j]
            self.codes[L.off[k][j]:L.off[k][j + 1]] = torch.from_numpy(d.codes.reshape(-1))
            # a strict CSR is a slotted one with slot == count
            self.rowstart[L.rpoff[k][j]:L.rpoff[k][j + 1]] = torch.from_numpy(
                d.row_ptr.astype(np.int32) + base[c])
            self.counts[L.roff[k][j]:L.roff[k][j + 1]] = torch.from_numpy(
                np.diff(d.row_ptr).astype(np.int32))
            cols[c].append(d.col_idx)
            vals[c].append(d.values)
            base[c] += d.nnz
        self.nnz = base
        for c in L.widths:
            col = np.concatenate(cols[c]) if cols[c] else np.zeros(0, np.int32)
            val = np.concatenate(vals[c]) if vals[c] else np.zeros(0, np.float32)
            self.arenas[c] = (col, val)

    def arena_capacity(self):
        return max(len(a[0]) for a in self.arenas.values()) * 2 + 64

    def ensure_arena_capacity(self, cap):
        self.cap = cap

    def grad_shard(self, pad):
        return self.g[:pad]

    def step(self, lr, beta1, beta2, weight_decay):
        L, k = self.layout, self.rank
        for j, (i, lo, hi) in enumerate(self.mem):
            c = L.shapes[i][1]
            g = self.g[L.off[k][j]:L.off[k][j + 1]].numpy().reshape(hi - lo, c)
            gq = self.port.quantize_state(g, BW)      # the backward sink, per row
            self.w[j], self.m[j], _ = self.port.lion_step_layer(
                self.w[j], *self.m[j], *gq, lr=lr, beta1=beta1, beta2=beta2, wd=weight_decay)
        self._publish()

    def codes_shard(self, pad):
        return self.codes[:pad]

    def rowstart_shard(self, rp_pad):
        return self.rowstart[:rp_pad]

    def count_shard(self, rpad):
        return self.counts[:rpad]

    def csr_nnz(self):
        return dict(self.nnz)

    def pack_csr(self, pcap, base, rp_pad):
        """A strict CSR is already packed: the row starts only move by base[class]."""
        L, k = self.layout, self.rank
        rs = self.rowstart.clone()
        for j, (i, lo, hi) in enumerate(self.mem):
            rs[L.rpoff[k][j]:L.rpoff[k][j + 1]] += int(base[L.shapes[i][1]])
        return rs[:rp_pad], {c: self.arena(c, max(pcap[c], 1)) for c in L.widths}

    def arena(self, width, cap):
        col, val = self.arenas[width]
        oc = torch.zeros(cap, dtype=torch.int32)
        ov = torch.zeros(cap, dtype=torch.float32)
        oc[:len(col)] = torch.from_numpy(col)
        ov[:len(val)] = torch.from_numpy(val)
        return oc, ov


def _grad(shape, seed, rank):
    rng = np.random.default_rng(seed * 10 + rank)
    return (rng.integers(-2**18, 2**18, size=shape).astype(np.float64) * 2.0**-24).astype(np.float32)


def _worker(rank, world, port_no, q, packed=True):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_2310_07147_b200.zero1 import ShardLayout, Zero1QftLion
        port = Oracle("port")
        full_w = [port.decompose_weight(port.synth(s, 50 + i, 0.02, 0.01), FRAC, BW)
                  for i, s in enumerate(SHAPES)]
        full_m = [port.quantize_state(np.zeros(s, np.float32), BW) for s in SHAPES]
        layout = ShardLayout(SHAPES, world)
        z = Zero1QftLion(SHAPES, OracleShard(layout, rank, port, full_w, full_m),
                         packed_csr=packed)
        assert z.packed == packed
        ref_w, ref_m = list(full_w), list(full_m)
        for step in range(3):
            mine = [torch.from_numpy(_grad(s, 100 * step + i, rank)) for i, s in enumerate(SHAPES)]
            layout.pack(mine, z.grad_full)
            z.step(lr=1e-3, weight_decay=0.01)
            for i, s in enumerate(SHAPES):     # single-process reference on the exact sum
                gsum = sum(_grad(s, 100 * step + i, r).astype(np.float64) for r in range(world))
                gq = port.quantize_state(gsum.astype(np.float32), BW)
                ref_w[i], ref_m[i], _ = port.lion_step_layer(ref_w[i], *ref_m[i], *gq, lr=1e-3,
                                                             wd=0.01)
                got = z.gathered_tensor(i)
                for key in ("codes", "row_ptr", "col_idx", "values"):
                    a, b = got[key], getattr(ref_w[i], key)
                    assert a.shape == b.shape and np.array_equal(a, b), (step, i, key)
            if packed:   # only used entries travel: the largest rank's nnz, 32-aligned
                mine_nnz = z.local.csr_nnz()
                for c in layout.widths:
                    assert z.pcap[c] % 32 == 0 and mine_nnz[c] <= z.pcap[c]
                assert z.gather_bytes_per_rank() < layout.pad + 4 * (layout.rp_pad + layout.rpad) \
                    + 8 * z.cap * len(layout.widths)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("packed", [True, False])
def test_zero1_two_ranks_gloo(packed):
    """packed: only the used CSR entries are all-gathered (row starts re-based per rank);
    not packed: the whole slotted arenas at a rank-uniform capacity."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, q, packed)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}, results


def test_shard_layout_partitions_rows():
    from paper_2310_07147_b200.shapes import llama2_7b
    from paper_2310_07147_b200.zero1 import ShardLayout
    shapes = llama2_7b()
    for world in (2, 4, 8):
        L = ShardLayout(shapes, world)
        assert sum(L.numel) == sum(r * c for r, c in shapes)
        for i, (r, c) in enumerate(shapes):
            covered = sorted((lo, hi) for k in range(world) for ti, lo, hi in L.members[k]
                             if ti == i)
            assert covered[0][0] == 0 and covered[-1][1] == r
            assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
        assert max(L.numel) - min(L.numel) < 0.001 * L.pad  # balanced shards


class _OverflowingShard(OracleShard):
    """Rank 1 reports a CSR slot overflow after its first local step; its recover() grows
    the arena (as a re-plan does), which every rank must then agree on."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.recovered = 0
        self.grow = 0

    def pending_overflow(self):
        return self.rank == 1 and self.recovered == 0

    def recover(self):
        self.recovered += 1
        self.grow = 4096

    def arena_capacity(self):
        return super().arena_capacity() + self.grow


def _overflow_worker(rank, world, port_no, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_2310_07147_b200.zero1 import ShardLayout, Zero1QftLion
        port = Oracle("port")
        full_w = [port.decompose_weight(port.synth(s, 50 + i, 0.02, 0.01), FRAC, BW)
                  for i, s in enumerate(SHAPES)]
        full_m = [port.quantize_state(np.zeros(s, np.float32), BW) for s in SHAPES]
        layout = ShardLayout(SHAPES, world)
        local = _OverflowingShard(layout, rank, port, full_w, full_m)
        z = Zero1QftLion(SHAPES, local, packed_csr=False)
        cap0 = z.cap
        ref_w, ref_m = list(full_w), list(full_m)
        for step in range(2):
            mine = [torch.from_numpy(_grad(s, 100 * step + i, rank)) for i, s in enumerate(SHAPES)]
            layout.pack(mine, z.grad_full)
            z.step(lr=1e-3, weight_decay=0.01)
            for i, s in enumerate(SHAPES):
                gsum = sum(_grad(s, 100 * step + i, r).astype(np.float64) for r in range(world))
                gq = port.quantize_state(gsum.astype(np.float32), BW)
                ref_w[i], ref_m[i], _ = port.lion_step_layer(ref_w[i], *ref_m[i], *gq, lr=1e-3,
                                                             wd=0.01)
                got = z.gathered_tensor(i)
                for key in ("codes", "row_ptr", "col_idx", "values"):
                    assert np.array_equal(got[key], getattr(ref_w[i], key)), (step, i, key)
        # only the overflowing rank re-ran; both agreed the grown, rank-uniform capacity
        assert local.recovered == (1 if rank == 1 else 0)
        assert z.cap > cap0 and local.cap == z.cap
        assert all(t.numel() == world * z.cap for t in z.col_full.values())
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_zero1_overflow_agreement_gloo():
    """Zero1QftLion.check_local: one rank's CSR overflow is all-reduced; that rank
    re-plans and re-runs (recover), all ranks re-agree the arena capacity before the
    all-gather, and the gathered state is still the single-process reference step."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_overflow_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}, results
