"""Raw (f32 / bf16) gradients on the rows path: k_grad_quant applies the sink's
quantize_state(g) (gradflow.hpp:77; quantize.hpp:189-193) into the plan's u8 entry, then
the rows kernel steps from it.  Bytes must equal the oracle fed quantize_state(g), and the
general raw-gradient kernel (QFT_NO_GRAD_QUANT=1) on the same inputs."""
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


def _grad(port, sh, seed, step, bw=8):
    g = port.synth(sh, seed, 1e-3, 0.0)
    g[0] = 0.0                       # all-zero gradient row (constant channel params)
    g[1] = 2.5e-4                    # constant row
    g[2] *= 1e-30                    # tiny scale
    g[3, ::7] = 0.05 * (step + 1)    # a few large entries: coarse row scale
    # exact ties: bounds -c/1024, (qmax-c)/1024 give s = 2^-10, and every other value is a
    # half-integer multiple of s (bf16-exact) -- round_half_away must go away from zero
    qmax = (1 << bw) - 1
    c = (qmax + 1) // 2
    ties = (np.arange(-c, qmax - c) + 0.5) * 2.0 ** -10
    g[4] = np.resize(ties, sh[1]).astype(np.float32)
    g[4, 0], g[4, 1] = -c * 2.0 ** -10, (qmax - c) * 2.0 ** -10
    g[5, 3::97] = np.nan             # NaN values (not in column 0): code 0
    return g


def _build(cuda, port, shapes, bw, gkind, frac=0.01):
    eng = cuda.QftModelState(shapes, bit_width=bw, grad_kind=gkind)
    host, ora = [], []
    for i, sh in enumerate(shapes):
        d = port.decompose_weight(port.synth(sh, 50 + i, 0.02, 0.005), frac, bw)
        host.append(dict(codes=d.codes, scale=d.scale, zero_point=d.zero_point, t_min=d.t_min,
                         t_max=d.t_max, row_ptr=d.row_ptr, col_idx=d.col_idx, values=d.values))
        ora.append([d, port.quantize_state(np.zeros(sh, np.float32), bw)])
    eng.init_from_host(host)
    return eng, ora


@pytest.mark.parametrize("gkind", ["f32", "bf16"])
@pytest.mark.parametrize("cols,bw,lr,wd", [(4096, 8, 2e-5, 0.0), (4096, 4, 2.2e-4, 0.01),
                                           (11008, 8, 2e-5, 0.01), (11008, 3, 2e-5, 0.0),
                                           (5120, 8, 2.2e-4, 0.0), (1024, 8, 4e-4, 0.01)])
def test_rows_path_raw_gradient_matches_oracle(cuda, port, gkind, cols, bw, lr, wd):
    shapes = [(24, cols), (9, cols)]
    eng, ora = _build(cuda, port, shapes, bw, gkind)
    N = cuda._native
    for g in eng.groups:
        # k_grad_quant + prep + stable rows + GEN rows (when on) + general
        assert N.lib.qftc_plan_launches(g.plan) >= 4, "raw gradient did not take the rows path"
    for step in range(4):
        for i, sh in enumerate(shapes):
            g = _grad(port, sh, 900 + 10 * step + i, step, bw)
            gt = torch.from_numpy(g)
            if gkind == "bf16":
                gt = gt.to(torch.bfloat16)
                g = gt.float().numpy()
            eng.grad_views(i).copy_(gt)
            gq = port.quantize_state(g, bw)
            d, m = ora[i]
            ora[i] = list(port.lion_step_layer(d, *m, *gq, lr=lr, wd=wd)[:2])
        eng.step(lr=lr, weight_decay=wd, check=True)
        assert all(n.startswith("rows_kernel<") for n in eng.kernel_names()), eng.kernel_names()
        for i in range(len(shapes)):
            got = eng.export_tensor(i)
            d, m = ora[i]
            for k, ref in (("codes", d.codes), ("row_ptr", d.row_ptr), ("col_idx", d.col_idx),
                           ("values", d.values), ("m_codes", m[0]), ("m_scale", m[1]),
                           ("m_zero_point", m[2])):
                _eq(got[k], ref, f"{gkind} cols {cols} b{bw} step {step} tensor {i} {k}")


def test_rows_path_raw_gradient_equals_general_kernel(cuda, port, monkeypatch):
    """The same bf16 gradients through k_grad_quant + rows kernel and through the general
    raw-gradient kernel (quantize_state fused per warp-row) give identical state."""
    shapes = [(32, 4096), (16, 4096)]
    bw = 8
    states = []
    for off in ("0", "1"):
        monkeypatch.setenv("QFT_NO_GRAD_QUANT", off)
        eng, _ = _build(cuda, port, shapes, bw, "bf16")
        want = 3 if off == "1" else 4
        if off == "1":
            assert all(cuda._native.lib.qftc_plan_launches(g.plan) == 1 for g in eng.groups)
        else:
            assert all(cuda._native.lib.qftc_plan_launches(g.plan) >= want for g in eng.groups)
        for step in range(3):
            for i, sh in enumerate(shapes):
                eng.grad_views(i).copy_(torch.from_numpy(_grad(port, sh, 77 + step + 5 * i, step))
                                        .to(torch.bfloat16))
            eng.step(lr=2.2e-4, weight_decay=0.01, check=True)
        states.append([eng.export_tensor(i) for i in range(len(shapes))])
    for i in range(len(shapes)):
        for k in ("codes", "row_ptr", "col_idx", "values", "m_codes", "m_scale", "m_zero_point"):
            _eq(states[0][i][k], states[1][i][k], f"tensor {i} {k}: rows path vs general")


def test_rows_path_raw_gradient_nan_column0_raises(cuda, port):
    """A NaN in a gradient row's column 0 is the reference's min > max (quantize.hpp:120):
    the step reports it."""
    shapes = [(8, 4096)]
    eng, _ = _build(cuda, port, shapes, 8, "f32")
    g = _grad(port, shapes[0], 5, 0)
    g[4, 0] = np.nan
    eng.grad_views(0).copy_(torch.from_numpy(g))
    with pytest.raises(ValueError):
        eng.step(lr=2e-5, check=True)
