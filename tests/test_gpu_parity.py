"""GPU parity: every sm_100a kernel against the CPU oracle on identical inputs.

Bar: codes, zero points, row_ptr, col_idx bit-exact; scales,
thresholds, CSR values and post-step fp32 tensors bit-exact (the reference
arithmetic is reproduced, not approximated); bf16 outputs equal the RNE of the
oracle's fp32 value.  Calls go through the C-ABI (via the package's ctypes
binding).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy()


def _eq(a, b, what):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    if a.dtype.kind == "f":
        bad = ~((a == b) | (np.isnan(a) & np.isnan(b)))
    else:
        bad = a != b
    n = int(bad.sum())
    assert n == 0, f"{what}: {n} mismatches, first at {np.argwhere(bad)[:5].tolist()}"


def _rows_zoo(rng, rows, cols, bit_width=8):
    """random rows + the edge cases the reference tests exercise"""
    x = rng.uniform(-2, 2, size=(rows, cols)).astype(np.float32)
    x[0] = 0.0                                   # all-zero channel (acceptance.cpp:173-176)
    x[1] = 3.5                                   # constant channel
    x[2] = 1000.0 + rng.uniform(0, 1e-3, cols).astype(np.float32)   # narrow, far from zero
    x[3] = -7.0 + rng.uniform(0, 1e-4, cols).astype(np.float32)     # |z| huge -> fp64 path
    x[4] = rng.normal(0, 1, cols).astype(np.float32) * 1e-30        # tiny scale
    if rows > 6:
        # planted near-ties: values on (k+0.5)*s grid of the row's own params
        lo, hi = -1.0, 1.0
        qmax = (1 << bit_width) - 1
        s = np.float32((hi - lo) / qmax)
        k = rng.integers(-qmax // 2, qmax // 2, cols)
        v = ((k + 0.5) * s.astype(np.float64)).astype(np.float32)
        jitter = rng.integers(-2, 3, cols)
        v = np.array([np.nextafter(a, np.float32(np.inf) if j > 0 else np.float32(-np.inf))
                      if j else a for a, j in zip(v, jitter)], np.float32)
        v[0], v[1] = lo, hi
        x[5] = v
    return x


def test_synth_device_matches_host(cuda, port):
    for seed, sig, sp in [(1234, 0.02, 0.005), (7, 1e-3, 0.0), (99, 1.0, 0.5)]:
        d = _np(cuda.synth((37, 129), seed, sig, sp))
        h = port.synth((37, 129), seed, sig, sp)
        _eq(d, h, f"synth seed {seed}")


@pytest.mark.parametrize("bw", [2, 3, 4, 8])
@pytest.mark.parametrize("shape", [(64, 256), (33, 100), (7, 4096), (9, 3)])
def test_quantize_state_bitexact(cuda, port, bw, shape):
    rng = np.random.default_rng(bw * 1000 + shape[1])
    x = _rows_zoo(rng, *shape, bit_width=bw) if shape[0] > 5 else \
        rng.normal(size=shape).astype(np.float32)
    q = cuda.quantize_state(torch.from_numpy(x).cuda(), bw)
    cq, cs, cz = port.quantize_state(x, bw)
    _eq(_np(q.params.scale), cs, "scale")
    _eq(_np(q.params.zero_point), cz, "zero_point")
    _eq(_np(q.data), cq, "codes")
    # dequantize f32 and bf16
    deq = cuda.dequantize(q)
    ref = port.dequantize(cq, cs, cz)
    _eq(_np(deq), ref, "dequantize")
    b16 = cuda.dequantize(q, torch.bfloat16)
    _eq(_np(b16.float()), _np(torch.from_numpy(ref).to(torch.bfloat16).float()), "dequant bf16")


@pytest.mark.parametrize("bw", [2, 4, 8])
def test_quantize_given_params_ties(cuda, port, bw):
    """half-away rounding on planted exact ties and +-1..3 ulp neighbours (test_quantize.cpp:102-114)"""
    rng = np.random.default_rng(bw)
    rows, cols = 16, 512
    qmax = (1 << bw) - 1
    scale = rng.uniform(1e-3, 2.0, rows).astype(np.float32)
    zp = rng.integers(-3, qmax + 3, rows).astype(np.int32)
    zp[0] = 3_000_000     # forces the exact fp64 row path (|z| >= 2^21)
    x = np.empty((rows, cols), np.float32)
    for r in range(rows):
        k = rng.integers(-zp[r] - 2, qmax - zp[r] + 2, cols).astype(np.float64)
        v = ((k + 0.5) * np.float64(scale[r])).astype(np.float32)
        steps = rng.integers(-3, 4, cols)
        for j in range(cols):
            for _ in range(abs(int(steps[j]))):
                v[j] = np.nextafter(v[j], np.float32(np.inf if steps[j] > 0 else -np.inf))
        x[r] = v
    x[1, :4] = [np.nan, np.inf, -np.inf, 0.0]
    q = cuda.quantize(torch.from_numpy(x).cuda(),
                      cuda.AffineParams(torch.from_numpy(scale).cuda(),
                                        torch.from_numpy(zp).cuda(), bw))
    _eq(_np(q.data), port.quantize(x, scale, zp, bw), "codes")


def test_half_away_kat(cuda):
    """test_quantize.cpp:102-114: s=1, z=128: 0.5->129, 1.5->130, -0.5->127, -1.5->126, 2.5->131"""
    x = torch.tensor([[0.5, 1.5, -0.5, -1.5, 2.5]], device="cuda")
    p = cuda.AffineParams(torch.tensor([1.0], device="cuda"),
                          torch.tensor([128], dtype=torch.int32, device="cuda"), 8)
    assert _np(cuda.quantize(x, p).data).tolist() == [[129, 130, 127, 126, 131]]


def test_hand_params_kat(cuda):
    """test_quantize.cpp:42-60: [-1,0,2] -> s=3/255, z=85, codes [0,85,255]"""
    q = cuda.quantize_state(torch.tensor([[-1.0, 0.0, 2.0]], device="cuda"), 8)
    assert _np(q.params.zero_point).tolist() == [85]
    assert abs(float(q.params.scale[0]) - 3 / 255) < 1e-8
    assert _np(q.data).tolist() == [[0, 85, 255]]


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("fraction", [0.0, 0.0005, 0.01, 0.05, 0.3])
@pytest.mark.parametrize("shape", [(48, 4096), (17, 100), (5, 1), (3, 2)])
def test_thresholds(cuda, port, kind, fraction, shape):
    w = port.synth(shape, 11 + shape[1], 0.02, 0.005)
    if shape[0] > 4:
        w[4, ::3] = 0.0                           # duplicates / zeros
    lo, hi = cuda.compute_outlier_thresholds(torch.from_numpy(w).cuda(), fraction, kind)
    elo, ehi = port.outlier_thresholds(w, fraction, kind)
    _eq(_np(lo), elo, "t_min")
    _eq(_np(hi), ehi, "t_max")


@pytest.mark.parametrize("bw", [3, 4, 8])
@pytest.mark.parametrize("shape", [(64, 4096), (40, 11008), (13, 80), (6, 7)])
def test_decompose_and_reconstruct(cuda, port, bw, shape):
    w = port.synth(shape, 5 + shape[0], 0.02, 0.005)
    dev = cuda.decompose_weight(torch.from_numpy(w).cuda(), 0.01, bw)
    ref = port.decompose_weight(w, 0.01, bw)
    _eq(_np(dev.t_min), ref.t_min, "t_min")
    _eq(_np(dev.t_max), ref.t_max, "t_max")
    _eq(_np(dev.dense.params.scale), ref.scale, "scale")
    _eq(_np(dev.dense.params.zero_point), ref.zero_point, "zero_point")
    _eq(_np(dev.dense.data), ref.codes, "codes")
    _eq(_np(dev.sparse.row_ptr), ref.row_ptr, "row_ptr")
    _eq(_np(dev.sparse.col_idx), ref.col_idx, "col_idx")
    _eq(_np(dev.sparse.values), ref.values, "values")
    rec = port.reconstruct(ref)
    _eq(_np(cuda.reconstruct(dev)), rec, "reconstruct")
    _eq(_np(cuda.reconstruct(dev, torch.bfloat16).float()),
        _np(torch.from_numpy(rec).to(torch.bfloat16).float()), "reconstruct bf16")
    assert cuda.byte_size(dev) == ref.byte_size()


def test_decompose_hand_csr(cuda):
    """test_quantize.cpp:218-235: row_ptr [0,0,1], col [1], val [100]"""
    w = torch.tensor([[0.1, 0.2], [0.3, 100.0]], device="cuda")
    d = cuda.decompose_dense_sparse(w, torch.tensor([0.1, 0.3]), torch.tensor([0.2, 0.4]), 8)
    assert _np(d.sparse.row_ptr).tolist() == [0, 0, 1]
    assert _np(d.sparse.col_idx).tolist() == [1]
    assert _np(d.sparse.values).tolist() == [100.0]
    assert float(cuda.reconstruct(d)[1, 1]) == 100.0
    assert cuda.byte_size(d) == 56


def _layer(port, shape, seed, bw, frac):
    w = port.synth(shape, seed, 0.02, 0.005)
    dsw = port.decompose_weight(w, frac, bw)
    m = port.quantize_state(np.zeros(shape, np.float32), bw)
    return dsw, m


@pytest.mark.parametrize("wd", [0.0, 0.01])
@pytest.mark.parametrize("bw,frac", [(8, 0.01), (4, 0.01), (3, 0.0045), (8, 0.05)])
@pytest.mark.parametrize("shape", [(64, 4096), (24, 11008), (16, 48), (5, 13)])
def test_lion_step_trajectory(cuda, port, bw, frac, shape, wd):
    """10 quantized Lion steps through the C-ABI single-layer entry, byte-compared each step
    (exercises CSR drift: nnz moves while thresholds stay cached); wd=0 runs the
    saturating sign-update form on proven rows, wd>0 the general form."""
    dsw, m = _layer(port, shape, 100 + shape[1], bw, frac)
    dw = cuda.DenseSparseWeight(
        cuda.QuantizedTensor(shape[0], shape[1], torch.from_numpy(dsw.codes).cuda(),
                             cuda.AffineParams(torch.from_numpy(dsw.scale).cuda(),
                                               torch.from_numpy(dsw.zero_point).cuda(), bw)),
        cuda.SparseOutliers(torch.from_numpy(dsw.row_ptr).cuda(),
                            torch.from_numpy(dsw.col_idx).cuda(),
                            torch.from_numpy(dsw.values).cuda()),
        torch.from_numpy(dsw.t_min).cuda(), torch.from_numpy(dsw.t_max).cuda(), frac)
    st = cuda.LionState([cuda.QuantizedTensor(shape[0], shape[1], torch.from_numpy(m[0]).cuda(),
                                              cuda.AffineParams(torch.from_numpy(m[1]).cuda(),
                                                                torch.from_numpy(m[2]).cuda(),
                                                                bw))])
    h = cuda.LionHyper(lr=2e-3, beta1=0.9, beta2=0.99, weight_decay=wd)
    for step in range(10):
        g = port.synth(shape, 7000 + step, 1e-2, 0.0)
        gq = port.quantize_state(g, bw)
        stack = cuda.GradientStack()
        stack.push(1, cuda.QuantizedTensor(shape[0], shape[1], torch.from_numpy(gq[0]).cuda(),
                                           cuda.AffineParams(torch.from_numpy(gq[1]).cuda(),
                                                             torch.from_numpy(gq[2]).cuda(), bw)))
        cuda.lion_step_quantized([dw], st, stack, h, bw)
        dsw, m, _ = port.lion_step_layer(dsw, *m, *gq, lr=h.lr, beta1=h.beta1, beta2=h.beta2,
                                         wd=h.weight_decay)
        tag = f"step {step}"
        _eq(_np(st.momentum[0].params.scale), m[1], tag + " m scale")
        _eq(_np(st.momentum[0].params.zero_point), m[2], tag + " m zp")
        _eq(_np(st.momentum[0].data), m[0], tag + " m codes")
        _eq(_np(dw.dense.data), dsw.codes, tag + " w codes")
        _eq(_np(dw.sparse.row_ptr), dsw.row_ptr, tag + " row_ptr")
        _eq(_np(dw.sparse.col_idx), dsw.col_idx, tag + " col_idx")
        _eq(_np(dw.sparse.values), dsw.values, tag + " values")


@pytest.mark.parametrize("bw,frac", [(8, 0.01), (8, 0.0045), (4, 0.0045), (3, 0.0045)])
@pytest.mark.parametrize("wd", [0.0, 0.01])
@pytest.mark.parametrize("lr", [2e-5, 1.5e-4, 2.2e-4, 4e-4])
@pytest.mark.parametrize("shape", [(64, 4096), (24, 11008), (40, 48), (24, 5120), (12, 13824)])
def test_lion_step_stable_tier(cuda, port, lr, shape, wd, bw, frac):
    """The rows kernel's stable tier (rowstep.cu): at the paper's lr = 2e-5 every row is
    proven code-stable; lr near sw/2 (~2.2e-4 at 8 bits) splits a tensor between the
    stable tier and the general kernel row by row.  12 steps byte-compared with the
    oracle; the first steps migrate boundary codes (0 / qmax) into the CSR, so the
    candidate path and the old-outlier sparse pass both run.  p = 0.45% puts the
    thresholds inside the spikes, so zero points sit near 0 / qmax and boundary-code
    candidates are common (the tabulated candidate outcomes)."""
    dsw, m = _layer(port, shape, 500 + shape[1], bw, frac)
    dw, st = _dev_layer(cuda, dsw, m, shape, bw, frac)
    h = cuda.LionHyper(lr=lr, beta1=0.9, beta2=0.99, weight_decay=wd)
    for step in range(12):
        g = port.synth(shape, 7700 + step, 1e-2, 0.01 if step % 3 == 0 else 0.0)
        gq = port.quantize_state(g, bw)
        stack = cuda.GradientStack()
        stack.push(1, cuda.QuantizedTensor(shape[0], shape[1], torch.from_numpy(gq[0]).cuda(),
                                           cuda.AffineParams(torch.from_numpy(gq[1]).cuda(),
                                                             torch.from_numpy(gq[2]).cuda(), bw)))
        cuda.lion_step_quantized([dw], st, stack, h, bw)
        dsw, m, _ = port.lion_step_layer(dsw, *m, *gq, lr=h.lr, beta1=h.beta1, beta2=h.beta2,
                                         wd=h.weight_decay)
        tag = f"b{bw} p{frac} lr {lr} step {step}"
        _eq(_np(st.momentum[0].params.scale), m[1], tag + " m scale")
        _eq(_np(st.momentum[0].params.zero_point), m[2], tag + " m zp")
        _eq(_np(st.momentum[0].data), m[0], tag + " m codes")
        _eq(_np(dw.dense.data), dsw.codes, tag + " w codes")
        _eq(_np(dw.sparse.row_ptr), dsw.row_ptr, tag + " row_ptr")
        _eq(_np(dw.sparse.col_idx), dsw.col_idx, tag + " col_idx")
        _eq(_np(dw.sparse.values), dsw.values, tag + " values")


def _dev_layer(cuda, dsw, m, shape, bw, frac):
    dw = cuda.DenseSparseWeight(
        cuda.QuantizedTensor(shape[0], shape[1], torch.from_numpy(dsw.codes).cuda(),
                             cuda.AffineParams(torch.from_numpy(dsw.scale).cuda(),
                                               torch.from_numpy(dsw.zero_point).cuda(), bw)),
        cuda.SparseOutliers(torch.from_numpy(dsw.row_ptr).cuda(),
                            torch.from_numpy(dsw.col_idx).cuda(),
                            torch.from_numpy(dsw.values).cuda()),
        torch.from_numpy(dsw.t_min).cuda(), torch.from_numpy(dsw.t_max).cuda(), frac)
    st = cuda.LionState([cuda.QuantizedTensor(shape[0], shape[1], torch.from_numpy(m[0]).cuda(),
                                              cuda.AffineParams(torch.from_numpy(m[1]).cuda(),
                                                                torch.from_numpy(m[2]).cuda(),
                                                                bw))])
    return dw, st


@pytest.mark.parametrize("wd", [0.0, 0.01])
@pytest.mark.parametrize("bw", [8, 4])
def test_lion_step_edge_rows(cuda, port, bw, wd):
    """Rows that must leave the fast paths, stepped next to ordinary ones: all-zero and
    constant channels, narrow channels far from zero (|z| >= 2^22), tiny scales, planted
    ties (the zoo), and gradients that are zero, 1e-30-scaled (Lion sign products below
    the saturating form's bound), 1e30-scaled or constant per row."""
    shape = (12, 1024)
    rng = np.random.default_rng(11 + bw)
    w = _rows_zoo(rng, shape[0], shape[1], bw)
    dsw = port.decompose_weight(w, 0.01, bw)
    m = port.quantize_state(np.zeros(shape, np.float32), bw)
    dw, st = _dev_layer(cuda, dsw, m, shape, bw, 0.01)
    h = cuda.LionHyper(lr=1e-3, beta1=0.9, beta2=0.99, weight_decay=wd)
    for step in range(6):
        g = port.synth(shape, 8100 + step, 1e-2, 0.0)
        g[0] = 0.0
        g[1] *= np.float32(1e-28)
        g[2] *= np.float32(1e30)
        g[3] = np.float32(0.25)
        g[7] *= np.float32(1e-40 if step % 2 else 1.0)
        gq = port.quantize_state(g, bw)
        stack = cuda.GradientStack()
        stack.push(1, cuda.QuantizedTensor(shape[0], shape[1], torch.from_numpy(gq[0]).cuda(),
                                           cuda.AffineParams(torch.from_numpy(gq[1]).cuda(),
                                                             torch.from_numpy(gq[2]).cuda(), bw)))
        cuda.lion_step_quantized([dw], st, stack, h, bw)
        dsw, m, _ = port.lion_step_layer(dsw, *m, *gq, lr=h.lr, beta1=h.beta1, beta2=h.beta2,
                                         wd=h.weight_decay)
        tag = f"step {step}"
        _eq(_np(st.momentum[0].params.scale), m[1], tag + " m scale")
        _eq(_np(st.momentum[0].params.zero_point), m[2], tag + " m zp")
        _eq(_np(st.momentum[0].data), m[0], tag + " m codes")
        _eq(_np(dw.dense.data), dsw.codes, tag + " w codes")
        _eq(_np(dw.sparse.row_ptr), dsw.row_ptr, tag + " row_ptr")
        _eq(_np(dw.sparse.col_idx), dsw.col_idx, tag + " col_idx")
        _eq(_np(dw.sparse.values), dsw.values, tag + " values")


def test_engine_grouped_step_matches_oracle(cuda, port):
    """A mixed-width model (two width classes, an RMSNorm-like 1xC row) stepped by the
    grouped persistent launch; every tensor byte-compared with the per-layer oracle."""
    shapes = [(32, 4096), (1, 4096), (96, 1024), (16, 4096), (48, 1024)]
    bw, frac = 8, 0.01
    tensors, oracle_state = [], []
    for i, sh in enumerate(shapes):
        dsw, m = _layer(port, sh, 300 + i, bw, frac)
        tensors.append(dict(codes=dsw.codes, scale=dsw.scale, zero_point=dsw.zero_point,
                            t_min=dsw.t_min, t_max=dsw.t_max, row_ptr=dsw.row_ptr,
                            col_idx=dsw.col_idx, values=dsw.values))
        oracle_state.append([dsw, m])
    eng = cuda.QftModelState(shapes, bit_width=bw)
    eng.init_from_host(tensors)
    for step in range(4):
        for i, sh in enumerate(shapes):
            g = port.synth(sh, 9000 + 10 * step + i, 1e-2, 0.0)
            gq = port.quantize_state(g, bw)
            c, s, z = eng.grad_views(i)
            c.copy_(torch.from_numpy(gq[0]))
            s.copy_(torch.from_numpy(gq[1]))
            z.copy_(torch.from_numpy(gq[2]))
            dsw, m = oracle_state[i]
            dsw, m, _ = port.lion_step_layer(dsw, *m, *gq, lr=1e-3, wd=0.0)
            oracle_state[i] = [dsw, m]
        eng.step(lr=1e-3, check=True)
        for i in range(len(shapes)):
            got = eng.export_tensor(i)
            dsw, m = oracle_state[i]
            tag = f"step {step} tensor {i}"
            _eq(got["codes"], dsw.codes, tag + " w codes")
            _eq(got["row_ptr"], dsw.row_ptr, tag + " row_ptr")
            _eq(got["col_idx"], dsw.col_idx, tag + " col_idx")
            _eq(got["values"], dsw.values, tag + " values")
            _eq(got["m_codes"], m[0], tag + " m codes")
            _eq(got["m_scale"], m[1], tag + " m scale")
            _eq(got["m_zero_point"], m[2], tag + " m zp")


def test_engine_expand_grouped(cuda, port):
    """Grouped weight expansion (qftc_expand, one launch for the model) after a step:
    f32 bit-exact with the oracle's reconstruct, bf16 = RNE of it; covers the vector
    path, unaligned widths, a 1xC row and the exact (|z| >= 2^22) dequant rows."""
    shapes = [(32, 4096), (1, 4096), (96, 1024), (9, 100), (6, 7), (8, 1024)]
    bw = 8
    rng = np.random.default_rng(7)
    oracle_state, tensors = [], []
    for i, sh in enumerate(shapes):
        if i == len(shapes) - 1:
            w = _rows_zoo(rng, sh[0], sh[1], bw)
            dsw = port.decompose_weight(w, 0.01, bw)
            m = port.quantize_state(np.zeros(sh, np.float32), bw)
        else:
            dsw, m = _layer(port, sh, 700 + i, bw, 0.01)
        tensors.append(dict(codes=dsw.codes, scale=dsw.scale, zero_point=dsw.zero_point,
                            t_min=dsw.t_min, t_max=dsw.t_max, row_ptr=dsw.row_ptr,
                            col_idx=dsw.col_idx, values=dsw.values))
        oracle_state.append([dsw, m])
    eng = cuda.QftModelState(shapes, bit_width=bw)
    eng.init_from_host(tensors)
    for i, sh in enumerate(shapes):
        gq = port.quantize_state(port.synth(sh, 7100 + i, 1e-2, 0.0), bw)
        c, s, z = eng.grad_views(i)
        c.copy_(torch.from_numpy(gq[0]))
        s.copy_(torch.from_numpy(gq[1]))
        z.copy_(torch.from_numpy(gq[2]))
        dsw, m = oracle_state[i]
        oracle_state[i][0] = port.lion_step_layer(dsw, *m, *gq, lr=1e-3)[0]
    eng.step(lr=1e-3, check=True)
    f32 = [torch.full(sh, float("nan"), device="cuda") for sh in shapes]
    b16 = [torch.zeros(sh, dtype=torch.bfloat16, device="cuda") for sh in shapes]
    eng.expand(f32)
    eng.expand(b16)
    for i in range(len(shapes)):
        rec = port.reconstruct(oracle_state[i][0])
        _eq(_np(f32[i]), rec, f"expand f32 tensor {i}")
        _eq(_np(b16[i].float()), _np(torch.from_numpy(rec).to(torch.bfloat16).float()),
            f"expand bf16 tensor {i}")
    # a row prefix only (the expansion of a partial tensor leaves the rest untouched)
    part = [torch.zeros(sh, device="cuda") for sh in shapes]
    eng.expand(part, rows=[min(2, sh[0]) for sh in shapes])
    for i, sh in enumerate(shapes):
        rec = port.reconstruct(oracle_state[i][0])
        k = min(2, sh[0])
        _eq(_np(part[i][:k]), rec[:k], f"expand prefix tensor {i}")
        assert not bool(part[i][k:].any())
    with pytest.raises(ValueError):
        eng.expand(f32[:-1] + [b16[-1]])


def test_lion_apply_passthrough_bitwise(cuda, port):
    """QuantMode::passthrough pipeline == lion_step_reference bitwise (test_optimizer.cpp:160-187)"""
    rng = np.random.default_rng(5)
    w = rng.uniform(-1, 1, 10001).astype(np.float32)
    m = np.zeros_like(w)
    dw, dm = torch.from_numpy(w).cuda(), torch.from_numpy(m).cuda()
    h = cuda.LionHyper(lr=3e-3, weight_decay=0.01)
    for step in range(25):
        g = rng.uniform(-1, 1, w.size).astype(np.float32)
        cuda.lion_apply(dw, dm, torch.from_numpy(g).cuda(), h)
        w, m = port.lion_apply(w, m, g, lr=3e-3, wd=0.01)
    _eq(_np(dw), w, "w")
    _eq(_np(dm), m, "m")


def test_validation_errors(cuda):
    with pytest.raises(ValueError):
        cuda.quantize_state(torch.zeros(2, 2, device="cuda"), 9)
    with pytest.raises(ValueError):
        cuda.compute_outlier_thresholds(torch.zeros(2, 2, device="cuda"), 0.5)
    with pytest.raises(ValueError):
        cuda.decompose_dense_sparse(torch.zeros(2, 2, device="cuda"), torch.tensor([1.0, 0.0]),
                                    torch.tensor([0.0, 0.0]))
    with pytest.raises(IndexError):
        cuda.GradientStack().pop()
    x = torch.zeros(2, 2, device="cuda")
    x[0, 0] = float("nan")      # NaN in column 0 sticks as the bound -> min > max
    with pytest.raises(ValueError):
        cuda.quantize_state(x, 8)


@pytest.mark.parametrize("gkind", ["f32", "bf16"])
def test_engine_raw_gradient_fused_quantize(cuda, port, gkind):
    """grad kind f32/bf16: the kernel applies the backward sink's quantize_state(g)
    (gradflow.hpp:77) and dequantize in-register; bytes equal the oracle fed the
    quantized gradient."""
    shapes = [(40, 1024), (8, 2048)]
    bw = 8
    eng = cuda.QftModelState(shapes, bit_width=bw, grad_kind=gkind)
    host, ora = [], []
    for i, sh in enumerate(shapes):
        d = port.decompose_weight(port.synth(sh, 40 + i, 0.02, 0.005), 0.01, bw)
        host.append(dict(codes=d.codes, scale=d.scale, zero_point=d.zero_point, t_min=d.t_min,
                         t_max=d.t_max, row_ptr=d.row_ptr, col_idx=d.col_idx, values=d.values))
        ora.append([d, port.quantize_state(np.zeros(sh, np.float32), bw)])
    eng.init_from_host(host)
    for step in range(3):
        for i, sh in enumerate(shapes):
            g = port.synth(sh, 700 + 10 * step + i, 1e-2, 0.0)
            gt = torch.from_numpy(g)
            if gkind == "bf16":
                gt = gt.to(torch.bfloat16)
                g = gt.float().numpy()
            eng.grad_views(i).copy_(gt)
            gq = port.quantize_state(g, bw)
            d, m = ora[i]
            ora[i] = list(port.lion_step_layer(d, *m, *gq, lr=1e-3, wd=0.01)[:2])
        eng.step(lr=1e-3, weight_decay=0.01, check=True)
        for i in range(len(shapes)):
            got = eng.export_tensor(i)
            d, m = ora[i]
            for k, ref in (("codes", d.codes), ("row_ptr", d.row_ptr), ("col_idx", d.col_idx),
                           ("values", d.values), ("m_codes", m[0]), ("m_scale", m[1])):
                _eq(got[k], ref, f"{gkind} step {step} tensor {i} {k}")


def test_engine_slot_overflow_replans(cuda, port):
    """A spike-dominated row moves dozens of edge codes into the sparse set in one step
    (SURVEY finding 2); undersized slots must be re-planned and the step re-run from the
    intact ping-pong inputs, with results still equal to the oracle."""
    sh = (64, 256)
    d = port.decompose_weight(port.synth(sh, 1240, 0.02, 0.02), 0.01, 8)
    eng = cuda.QftModelState([sh], bit_width=8)
    eng.init_from_host([dict(codes=d.codes, scale=d.scale, zero_point=d.zero_point,
                             t_min=d.t_min, t_max=d.t_max, row_ptr=d.row_ptr,
                             col_idx=d.col_idx, values=d.values)])
    # shrink every slot to the bare count: the first step must overflow somewhere
    n = eng.n
    rp = torch.from_numpy(d.row_ptr.astype(np.int64))
    cnt = (rp[1:] - rp[:-1])
    starts = torch.zeros(sh[0] + 1, dtype=torch.int64)
    starts[1:] = torch.cumsum((cnt + 3) // 4 * 4, 0)
    g = eng.groups[0]
    for k in range(2):
        eng.row_start[k][:sh[0] + 1].copy_(starts.to(torch.int32))
    eng.row_count[eng.cur].copy_(cnt.to(torch.int32))
    nnz_slots = int(starts[-1])
    for r in range(sh[0]):
        a, b = int(d.row_ptr[r]), int(d.row_ptr[r + 1])
        s0 = int(starts[r])
        g.col[eng.cur][s0:s0 + b - a].copy_(torch.from_numpy(d.col_idx[a:b]))
        g.val[eng.cur][s0:s0 + b - a].copy_(torch.from_numpy(d.values[a:b]))
    m = port.quantize_state(np.zeros(sh, np.float32), 8)
    gq = port.quantize_state(port.synth(sh, 9, 1e-3, 0.0), 8)
    c, s, z = eng.grad_views(0)
    c.copy_(torch.from_numpy(gq[0]))
    s.copy_(torch.from_numpy(gq[1]))
    z.copy_(torch.from_numpy(gq[2]))
    eng.step(lr=2e-5, check=True)
    d2, m2, _ = port.lion_step_layer(d, *m, *gq, lr=2e-5)
    assert eng.replans >= 1 and d2.nnz > d.nnz and nnz_slots < 2 ** 31
    got = eng.export_tensor(0)
    for k in ("codes", "row_ptr", "col_idx", "values"):
        _eq(got[k], getattr(d2, k), k)
    _eq(got["m_codes"], m2[0], "m_codes")


def test_zero1_world1_nccl_cuda_shard(cuda, port):
    """ZeRO-1 path with the real CUDA local update on a world-size-1 NCCL group:
    reduce-scatter -> fused f32-gradient step -> all-gather of codes/slots/arenas."""
    import socket
    import torch.distributed as dist
    from paper_2310_07147_b200.zero1 import CudaShard, ShardLayout, Zero1QftLion
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port_no = s_.getsockname()[1]
    s_.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port_no}", rank=0,
                            world_size=1)
    try:
        shapes = [(24, 512), (1, 512), (12, 256)]
        layout = ShardLayout(shapes, 1)
        local = CudaShard(layout, 0, bit_width=8)
        host, ora = [], []
        for i, sh in enumerate(shapes):
            d = port.decompose_weight(port.synth(sh, 60 + i, 0.02, 0.005), 0.01, 8)
            host.append(dict(codes=d.codes, scale=d.scale, zero_point=d.zero_point,
                             t_min=d.t_min, t_max=d.t_max, row_ptr=d.row_ptr,
                             col_idx=d.col_idx, values=d.values))
            ora.append([d, port.quantize_state(np.zeros(sh, np.float32), 8)])
        local.state.init_from_host(host)
        z = Zero1QftLion(shapes, local)
        for step in range(2):
            grads = []
            for i, sh in enumerate(shapes):
                g = port.synth(sh, 800 + 10 * step + i, 1e-2, 0.0)
                grads.append(torch.from_numpy(g).cuda())
                d, m = ora[i]
                ora[i] = list(port.lion_step_layer(d, *m, *port.quantize_state(g, 8),
                                                   lr=1e-3)[:2])
            layout.pack(grads, z.grad_full)
            z.step(lr=1e-3)
            local.state.check()
            for i in range(len(shapes)):
                got = z.gathered_tensor(i)
                d = ora[i][0]
                for k in ("codes", "row_ptr", "col_idx", "values"):
                    _eq(got[k], getattr(d, k), f"zero1 step {step} tensor {i} {k}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("grid", [3, 37])
@pytest.mark.parametrize("lr", [2e-5, 2.2e-4])
@pytest.mark.parametrize("model", ["small", "llama_widths"])
def test_rows_kernel_many_rows_per_cta(cuda, port, monkeypatch, grid, lr, model):
    """The rows kernel with a capped grid, so every CTA pipelines many rows through its
    TMA stages and sparse buffers (the other parity tests are small enough to give each
    CTA one row); lr near sw/2 mixes stable rows with rows of the general kernel inside
    one launch.  A small LLaMA-shaped model, 3 steps, every tensor byte-compared with
    the oracle."""
    from paper_2310_07147_b200.shapes import llama
    monkeypatch.setenv("QFT_ROWS_GRID", str(grid))
    # llama_widths: the compile-time-geometry instances (7B and 13B row lengths)
    shapes = llama(512, 1376, 1, 512) if model == "small" else \
        [(40, 4096), (24, 11008), (30, 5120), (20, 13824)]
    bw, frac = 8, 0.01
    st = cuda.QftModelState(shapes, bit_width=bw)
    st.init_from_weights(lambda i: cuda.synth(shapes[i], 1234 + i, 0.02, 0.005), frac)
    ora = []
    for i, sh in enumerate(shapes):
        w = port.synth(sh, 1234 + i, 0.02, 0.005)
        ora.append([port.decompose_weight(w, frac, bw),
                    port.quantize_state(np.zeros(sh, np.float32), bw)])
    for step in range(3):
        for i, sh in enumerate(shapes):
            gq = port.quantize_state(port.synth(sh, 5000 + 100 * step + i, 1e-3, 0.0), bw)
            c, sc, z = st.grad_views(i)
            c.copy_(torch.from_numpy(gq[0]))
            sc.copy_(torch.from_numpy(gq[1]))
            z.copy_(torch.from_numpy(gq[2]))
            d, m = ora[i]
            ora[i] = list(port.lion_step_layer(d, *m, *gq, lr=lr)[:2])
        st.step(lr=lr, check=True)
        for i in range(len(shapes)):
            got = st.export_tensor(i)
            d, m = ora[i]
            tag = f"grid {grid} lr {lr} step {step} tensor {i}"
            _eq(got["codes"], d.codes, tag + " w codes")
            _eq(got["row_ptr"], d.row_ptr, tag + " row_ptr")
            _eq(got["col_idx"], d.col_idx, tag + " col_idx")
            _eq(got["values"], d.values, tag + " values")
            _eq(got["m_codes"], m[0], tag + " m codes")
            _eq(got["m_scale"], m[1], tag + " m scale")
            _eq(got["m_zero_point"], m[2], tag + " m zp")


def _csr_rows(row_ptr, col_idx, values, rows):
    """The CSR entries of the given rows, as (row_ptr, cols, vals) of that sub-matrix."""
    rp, cs, vs = [0], [], []
    for r in rows:
        a, b = int(row_ptr[r]), int(row_ptr[r + 1])
        cs.append(np.asarray(col_idx[a:b]))
        vs.append(np.asarray(values[a:b]))
        rp.append(rp[-1] + (b - a))
    return (np.asarray(rp, np.int32), np.concatenate(cs).astype(np.int32),
            np.concatenate(vs).astype(np.float32))


@pytest.mark.parametrize("lr", [2e-5, 2.2e-4])
def test_full_size_7b_tensors_sampled_rows(cuda, port, lr):
    """Parity at BASELINE.json's full sizes through row independence: the step has no
    cross-row dependency (optimizer.hpp:103-118 is per-row quantize/decompose), so any
    subset of rows stepped by the oracle as its own layer must equal the same rows of
    the full-size GPU step.  The four LLaMA-2-7B matrix shapes (configs[1]; 238 M
    parameters, one grouped engine as in bench.py), three steps; 42 sampled rows per
    tensor (first, last, random) byte-compared -- codes, CSR, momentum -- plus
    whole-tensor invariants (CSR columns ascending and in range, payload code on every
    outlier, CSR values outside the thresholds)."""
    shapes = [(4096, 4096), (11008, 4096), (4096, 11008), (32000, 4096)]
    bw, frac = 8, 0.01
    qmax = (1 << bw) - 1
    st = cuda.QftModelState(shapes, bit_width=bw)
    st.init_from_weights(lambda i: cuda.synth(shapes[i], 4100 + i, 0.02, 0.005), frac)
    rng = np.random.default_rng(7)
    rows = [np.unique(np.r_[0, r - 1, rng.choice(r, 40, replace=False)]) for r, _ in shapes]
    ora = []
    for i, sh in enumerate(shapes):
        w = cuda.synth(sh, 4100 + i, 0.02, 0.005)[torch.from_numpy(rows[i]).cuda()].cpu().numpy()
        ora.append([port.decompose_weight(w, frac, bw),
                    port.quantize_state(np.zeros((len(rows[i]), sh[1]), np.float32), bw)])
        del w
    for step in range(3):
        for i, sh in enumerate(shapes):
            g = cuda.synth(sh, 8100 + 10 * step + i, 1e-3, 0.0)
            q = cuda.quantize_state(g, bw)
            c, sc, z = st.grad_views(i)
            c.copy_(q.data)
            sc.copy_(q.params.scale)
            z.copy_(q.params.zero_point)
            gq = port.quantize_state(g[torch.from_numpy(rows[i]).cuda()].cpu().numpy(), bw)
            del g, q
            d, m = ora[i]
            ora[i] = list(port.lion_step_layer(d, *m, *gq, lr=lr)[:2])
        st.step(lr=lr, check=True)
    for i, (r, c) in enumerate(shapes):
        got = st.export_tensor(i)
        d, m = ora[i]
        rs = rows[i]
        tag = f"lr {lr} {r}x{c}"
        _eq(got["codes"][rs], d.codes, tag + " w codes")
        rp, cs, vs = _csr_rows(got["row_ptr"], got["col_idx"], got["values"], rs)
        _eq(rp, d.row_ptr, tag + " row_ptr")
        _eq(cs, d.col_idx, tag + " col_idx")
        _eq(vs, d.values, tag + " values")
        _eq(got["m_codes"][rs], m[0], tag + " m codes")
        _eq(got["m_scale"][rs], m[1], tag + " m scale")
        _eq(got["m_zero_point"][rs], m[2], tag + " m zp")
        # whole-tensor invariants
        rp_all = np.asarray(got["row_ptr"], np.int64)
        col = np.asarray(got["col_idx"], np.int64)
        val = np.asarray(got["values"], np.float32)
        assert rp_all[0] == 0 and np.all(np.diff(rp_all) >= 0) and rp_all[-1] == col.size
        row_of = np.repeat(np.arange(r), np.diff(rp_all))
        assert col.size == 0 or (col.min() >= 0 and col.max() < c), tag + " column range"
        same_row = row_of[1:] == row_of[:-1]
        assert np.all(col[1:][same_row] > col[:-1][same_row]), tag + " columns ascending"
        tmin = np.asarray(got["t_min"])[row_of]
        tmax = np.asarray(got["t_max"])[row_of]
        assert np.all((val < tmin) | (val > tmax)), tag + " CSR value inside thresholds"
        zp = np.asarray(got["zero_point"], np.int64)[row_of]
        codes = np.asarray(got["codes"])
        assert np.array_equal(codes[row_of, col], np.clip(zp, 0, qmax)), tag + " payload code"
        del got


@pytest.mark.parametrize("bw", [3, 4, 8])
@pytest.mark.parametrize("shape", [(40, 300), (17, 101), (64, 4096)])
@pytest.mark.parametrize("inplace", [False, True])
def test_accumulate_microbatches(cuda, port, bw, shape, inplace):
    """gradflow.hpp:52-58 on the device (fused dequant + add + quantize_state, one row
    kernel), three micro-batches chained, byte-compared with the oracle (itself pinned
    to qft::accumulate in test_oracle.py); in place like the stack entry update."""
    from test_oracle import _acc_inputs
    acc, g = _acc_inputs(port, bw, 5 + shape[1], shape)
    q = cuda.QuantizedTensor(shape[0], shape[1], torch.from_numpy(acc[0]).cuda(),
                             cuda.AffineParams(torch.from_numpy(acc[1]).cuda(),
                                               torch.from_numpy(acc[2]).cuda(), bw))
    ref = acc
    for k in range(3):
        gk = (g * (k + 1)).astype(np.float32)
        q = cuda.accumulate(q, torch.from_numpy(gk).cuda(), out=q if inplace else None)
        ref = port.accumulate(*ref, gk, bw)
        _eq(_np(q.data), ref[0], f"micro-batch {k} codes")
        _eq(_np(q.params.scale), ref[1], f"micro-batch {k} scale")
        _eq(_np(q.params.zero_point), ref[2], f"micro-batch {k} zero_point")


def test_accumulate_nan_column0_raises(cuda, port):
    from test_oracle import _acc_inputs
    acc, g = _acc_inputs(port, 8, 3)
    g[7, 0] = np.nan
    q = cuda.QuantizedTensor(40, 300, torch.from_numpy(acc[0]).cuda(),
                             cuda.AffineParams(torch.from_numpy(acc[1]).cuda(),
                                               torch.from_numpy(acc[2]).cuda(), 8))
    with pytest.raises(ValueError, match="min > max"):
        cuda.accumulate(q, torch.from_numpy(g).cuda())


def test_engine_microbatch_sink_then_step(cuda, port):
    """Three micro-batches sunk into the engine's gradient entries (quantize_state, then
    accumulate in integer form, gradflow.hpp:70-84), then the grouped step; against the
    oracle doing the same per layer (sink + lion_step_layer)."""
    shapes = [(32, 4096), (1, 4096), (48, 1024)]
    bw, frac, lr = 8, 0.01, 1e-3
    eng = cuda.QftModelState(shapes, bit_width=bw)
    eng.init_from_weights(lambda i: cuda.synth(shapes[i], 600 + i, 0.02, 0.005), frac)
    ora = []
    for i, sh in enumerate(shapes):
        w = port.synth(sh, 600 + i, 0.02, 0.005)
        ora.append([port.decompose_weight(w, frac, bw),
                    port.quantize_state(np.zeros(sh, np.float32), bw)])
    for i, sh in enumerate(shapes):
        gq = None
        for mb in range(3):
            g = port.synth(sh, 7000 + 10 * i + mb, 1e-2, 0.0) / np.float32(3.0)
            eng.sink_grad(i, torch.from_numpy(g).cuda(), accumulate=mb > 0)
            gq = port.quantize_state(g, bw) if mb == 0 else port.accumulate(*gq, g, bw)
        d, m = ora[i]
        ora[i] = list(port.lion_step_layer(d, *m, *gq, lr=lr)[:2])
    eng.step(lr=lr, check=True)
    for i in range(len(shapes)):
        got = eng.export_tensor(i)
        d, m = ora[i]
        _eq(got["codes"], d.codes, f"tensor {i} w codes")
        _eq(got["col_idx"], d.col_idx, f"tensor {i} col_idx")
        _eq(got["values"], d.values, f"tensor {i} values")
        _eq(got["m_codes"], m[0], f"tensor {i} m codes")
        _eq(got["m_scale"], m[1], f"tensor {i} m scale")
