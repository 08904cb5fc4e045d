"""configs[3]: the next forward's weights expanded straight from the ZeRO-1 all-gathered,
shard-major buffers (Zero1QftLion.expand_plan: one launch, every (rank, tensor) row range a
table entry with its arena re-based by rank * capacity).  Two ranks' shards are stepped in
one process and their buffers concatenated as all_gather_into_tensor would; the expansion
must equal each shard's own expansion (f32 exact, bf16 the RNE of it) and the oracle's
reconstruct of the single-process reference step."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_expand_from_gathered_shards(cuda, port):
    from paper_2310_07147_b200.zero1 import CudaShard, ShardLayout, Zero1QftLion
    shapes = [(96, 512), (40, 1376), (1, 512), (70, 512)]
    world, bw = 2, 8
    L = ShardLayout(shapes, world)
    shards = []
    for k in range(world):
        sh = CudaShard(L, k, bit_width=bw, grad_dtype=torch.bfloat16)
        ss = L.shard_shapes(k)
        sh.state.init_from_weights(lambda i, k=k, ss=ss: cuda.synth(ss[i], 70 + 10 * k + i, 0.02, 0.005),
                                   0.01)
        for step in range(3):
            sh.state.g_raw.normal_(0.0, 1e-3, generator=torch.Generator("cuda").manual_seed(step + 9 * k))
            sh.state.step(lr=2e-4, check=True)
        shards.append(sh)
    cap = max(s.arena_capacity() for s in shards)
    for s in shards:
        s.ensure_arena_capacity(cap)
    # the all-gathered buffers, built as all_gather_into_tensor lays them out
    z = Zero1QftLion.__new__(Zero1QftLion)
    z.layout, z.world, z.cap, z.local = L, world, cap, shards[0]
    z.codes_full = torch.cat([s.codes_shard(L.pad) for s in shards])
    z.rowstart_full = torch.cat([s.rowstart_shard(L.rp_pad) for s in shards])
    z.count_full = torch.cat([s.count_shard(L.rpad) for s in shards])
    z.wscale_full = torch.cat([s.wscale_shard(L.rpad) for s in shards])
    z.wzp_full = torch.cat([s.wzp_shard(L.rpad) for s in shards])
    z.col_full, z.val_full = {}, {}
    for c in L.widths:
        cols, vals = zip(*[s.arena(c, cap) for s in shards])
        z.col_full[c], z.val_full[c] = torch.cat(cols), torch.cat(vals)
    for dt in (torch.float32, torch.bfloat16):
        outs = [torch.full(sh, float("nan"), dtype=dt, device="cuda") for sh in shapes]
        plan = z.expand_plan(outs)
        plan.run()
        torch.cuda.synchronize()
        for k, s in enumerate(shards):
            ref = [torch.empty(sh, dtype=dt, device="cuda") for sh in L.shard_shapes(k)]
            s.state.expand(ref)
            torch.cuda.synchronize()
            for j, (ti, lo, hi) in enumerate(L.members[k]):
                a = outs[ti][lo:hi].float().cpu().numpy()
                b = ref[j].float().cpu().numpy()
                assert np.array_equal(a, b), f"{dt} rank {k} tensor {ti} rows {lo}:{hi}"
            if dt == torch.float32:  # the oracle's reconstruct of the shard's exported state
                for j, (ti, lo, hi) in enumerate(L.members[k]):
                    e = s.state.export_tensor(j)
                    from oracle.oracle import DenseSparse
                    r_, c_ = L.shard_shapes(k)[j]
                    d = DenseSparse(e["codes"], e["scale"], e["zero_point"], e["row_ptr"],
                                    e["col_idx"], e["values"], e["t_min"], e["t_max"], bw)
                    assert np.array_equal(outs[ti][lo:hi].cpu().numpy(), port.reconstruct(d))
