"""the ZeRO-1 step over peer memory -- the reduce-scatter fused into
the local update (each rank's plans read their rows of the summed bf16 gradient straight
from every rank's buffer through CUDA IPC mappings and quantize them in the same pass,
k_rs_grad_quant), the all-gather a push into every rank's gathered buffers.  Two ranks run
as two processes sharing the one GPU this build has (gloo for the host-side exchange); the
gathered state must equal a single-process step of the full model fed the exact sum."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SHAPES = [(64, 512), (33, 512), (48, 1024), (7, 1024)]
LR, WD, BW = 2.2e-4, 0.01, 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grad(shape, seed, rank):
    rng = np.random.default_rng(seed * 10 + rank)
    g = rng.integers(-128, 128, size=shape).astype(np.float32) * 2.0 ** -14  # bf16-exact
    return torch.from_numpy(g)


def _weights(q, i):
    return q.synth(SHAPES[i], 70 + i, 0.02, 0.005)


def _worker(rank, world, port_no, queue):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2310_07147_b200 as q
        from paper_2310_07147_b200.zero1 import CudaShard, ShardLayout, Zero1QftLion
        layout = ShardLayout(SHAPES, world)
        local = CudaShard(layout, rank, bit_width=BW, grad_dtype=torch.bfloat16)
        mem = layout.members[rank]
        local.state.init_from_weights(lambda j: _weights(q, mem[j][0])[mem[j][1]:mem[j][2]].contiguous(),
                                      0.01)
        z = Zero1QftLion(SHAPES, local)
        z.enable_peer_memory()
        for step in range(4):
            mine = [_grad(s, 100 * step + i, rank).to(torch.bfloat16).cuda()
                    for i, s in enumerate(SHAPES)]
            layout.pack(mine, z.grad_full)
            z.step_fused(lr=LR, weight_decay=WD)
        got = [z.gathered_tensor(i) for i in range(len(SHAPES))]
        kern = [n for n in local.state.kernel_names()]
        if rank == 0:  # the single-process reference step on the exact sum
            ref = q.QftModelState(SHAPES, bit_width=BW, grad_kind="f32")
            ref.init_from_weights(lambda i: _weights(q, i), 0.01)
            for step in range(4):
                for i, s in enumerate(SHAPES):
                    ref.grad_views(i).copy_(sum(_grad(s, 100 * step + i, r) for r in range(world)))
                ref.step(lr=LR, weight_decay=WD, check=True)
            for i in range(len(SHAPES)):
                e = ref.export_tensor(i)
                for k in ("codes", "row_ptr", "col_idx", "values"):
                    assert np.array_equal(got[i][k], e[k]), (i, k)
        z._close_peers()
        queue.put((rank, "ok " + ",".join(kern)))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        queue.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_zero1_fused_peer_memory_two_ranks_one_gpu(cuda):
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, queue)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(queue.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v.startswith("ok") for v in res.values()), res
