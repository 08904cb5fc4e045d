"""The GEN tier: rows that miss only the stable-tier bound (*) (lr large against the row's
weight scale) run the rows kernel with every dense code requantized
(dequant w -> Lion -> outlier test against the cached thresholds -> code,
quantize.hpp:253-290, optimizer.hpp:103-118).  Bytes must equal the oracle, and equal the
general step_kernel (QFT_NO_GEN=1) on the same inputs."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _eq(a, b, what):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    bad = ~((a == b) | (np.isnan(a) & np.isnan(b))) if a.dtype.kind == "f" else a != b
    n = int(bad.sum())
    assert n == 0, f"{what}: {n} mismatches, first at {np.argwhere(bad)[:5].tolist()}"


def _build(cuda, port, shapes, bw, frac=0.01, seed=60):
    eng = cuda.QftModelState(shapes, bit_width=bw)
    host, ora = [], []
    for i, sh in enumerate(shapes):
        d = port.decompose_weight(port.synth(sh, seed + i, 0.02, 0.005), frac, bw)
        host.append(dict(codes=d.codes, scale=d.scale, zero_point=d.zero_point, t_min=d.t_min,
                         t_max=d.t_max, row_ptr=d.row_ptr, col_idx=d.col_idx, values=d.values))
        ora.append([d, port.quantize_state(np.zeros(sh, np.float32), bw)])
    eng.init_from_host(host)
    return eng, ora


KEYS = ("codes", "row_ptr", "col_idx", "values", "m_codes", "m_scale", "m_zero_point")


@pytest.mark.parametrize("cols,bw,lr,wd", [(4096, 8, 2.2e-4, 0.0), (4096, 8, 4e-4, 0.01),
                                           (11008, 8, 2.2e-4, 0.0), (11008, 8, 3e-4, 0.01),
                                           (1024, 4, 1.5e-2, 0.0), (2048, 3, 3e-2, 0.01),
                                           (5120, 8, 3e-4, 0.0), (4096, 4, 8e-3, 0.01)])
def test_gen_tier_matches_oracle(cuda, port, cols, bw, lr, wd):
    shapes = [(40, cols), (13, cols)]
    eng, ora = _build(cuda, port, shapes, bw)
    saw_gen = 0
    for step in range(6):
        for i, sh in enumerate(shapes):
            gq = port.quantize_state(port.synth(sh, 800 + 10 * step + i, 1e-3, 0.01), bw)
            c, s_, z = eng.grad_views(i)
            c.copy_(torch.from_numpy(gq[0]))
            s_.copy_(torch.from_numpy(gq[1]))
            z.copy_(torch.from_numpy(gq[2]))
            d, m = ora[i]
            ora[i] = list(port.lion_step_layer(d, *m, *gq, lr=lr, wd=wd)[:2])
        eng.step(lr=lr, weight_decay=wd, check=True)
        saw_gen += eng.tiers()[1]
        for i in range(len(shapes)):
            got = eng.export_tensor(i)
            d, m = ora[i]
            for k, ref in zip(KEYS, (d.codes, d.row_ptr, d.col_idx, d.values, m[0], m[1], m[2])):
                _eq(got[k], ref, f"cols {cols} b{bw} lr {lr} step {step} tensor {i} {k}")
    assert saw_gen > 0, "no row took the GEN tier"


def test_gen_tier_equals_general_kernel(cuda, port, monkeypatch):
    """Same inputs, GEN tier on and off (QFT_NO_GEN=1 routes those rows to step_kernel):
    identical state after a 20-step trajectory at lr = 2.2e-4 on LLaMA widths."""
    shapes = [(48, 4096), (16, 11008), (24, 4096)]
    res = []
    for off in ("0", "1"):
        monkeypatch.setenv("QFT_NO_GEN", off)
        eng, _ = _build(cuda, port, shapes, 8, seed=91)
        tiers = [0, 0, 0]
        for step in range(20):
            for i, sh in enumerate(shapes):
                gq = port.quantize_state(port.synth(sh, 300 + 7 * step + i, 1e-3, 0.02), 8)
                c, s_, z = eng.grad_views(i)
                c.copy_(torch.from_numpy(gq[0]))
                s_.copy_(torch.from_numpy(gq[1]))
                z.copy_(torch.from_numpy(gq[2]))
            eng.step(lr=2.2e-4, weight_decay=0.01 if step % 2 else 0.0, check=True)
            tiers = [a + b for a, b in zip(tiers, eng.tiers())]
        if off == "0":
            assert tiers[1] > 0
        else:
            assert tiers[1] == 0 and tiers[2] > 0
        res.append([eng.export_tensor(i) for i in range(len(shapes))])
    for i in range(len(shapes)):
        for k in KEYS:
            _eq(res[0][i][k], res[1][i][k], f"tensor {i} {k}: GEN tier vs step_kernel")


@pytest.mark.parametrize("route", ["1", "0"])
def test_few_stable_rows_route_into_gen_list(cuda, port, monkeypatch, route):
    """At a large lr most rows leave the stable tier; when fewer than 1/16 of the rows were
    stable the step before, the step skips the stable launch and its stable rows run in the
    GEN kernel (QFT_NO_ROUTE=1 keeps them in the stable kernel).  Bytes equal the oracle
    either way."""
    monkeypatch.setenv("QFT_NO_ROUTE", "0" if route == "1" else "1")
    shapes = [(40, 4096), (13, 4096)]
    bw, lr, wd = 8, 2.2e-4, 0.01
    eng = cuda.QftModelState(shapes, bit_width=bw)
    host, ora = [], []
    for i, sh in enumerate(shapes):
        w = port.synth(sh, 70 + i, 0.02, 0.005)
        if i == 0:
            w[:2] *= 20.0              # two rows with a coarse scale: stable at this lr
        d = port.decompose_weight(w, 0.01, bw)
        host.append(dict(codes=d.codes, scale=d.scale, zero_point=d.zero_point, t_min=d.t_min,
                         t_max=d.t_max, row_ptr=d.row_ptr, col_idx=d.col_idx, values=d.values))
        ora.append([d, port.quantize_state(np.zeros(sh, np.float32), bw)])
    eng.init_from_host(host)
    tiers = []
    for step in range(4):
        for i, sh in enumerate(shapes):
            gq = port.quantize_state(port.synth(sh, 500 + 10 * step + i, 1e-3, 0.01), bw)
            c, s_, z = eng.grad_views(i)
            c.copy_(torch.from_numpy(gq[0]))
            s_.copy_(torch.from_numpy(gq[1]))
            z.copy_(torch.from_numpy(gq[2]))
            d, m = ora[i]
            ora[i] = list(port.lion_step_layer(d, *m, *gq, lr=lr, wd=wd)[:2])
        eng.step(lr=lr, weight_decay=wd, check=True)
        tiers.append(eng.tiers())
        for i in range(len(shapes)):
            got = eng.export_tensor(i)
            d, m = ora[i]
            for k, ref in zip(KEYS, (d.codes, d.row_ptr, d.col_idx, d.values, m[0], m[1], m[2])):
                _eq(got[k], ref, f"route {route} step {step} tensor {i} {k}")
    assert 0 < tiers[0][0] * 16 < sum(shapes[i][0] for i in range(2)), tiers
    if route == "1":   # the first step had no history; later steps routed
        assert all(t[0] == 0 for t in tiers[1:]), tiers
    else:
        assert all(t[0] > 0 for t in tiers), tiers
