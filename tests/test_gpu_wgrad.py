"""§8(f) row 2: the backward's weight gradient with the sink fused into the GEMM epilogue
(qftc_wgrad_quant, tcgen05 + TMA, MN-major operands).  G = dy^T . x (network.hpp:139) is
quantized in the epilogue into the GradientStack entry: quantize_state(G) (gradflow.hpp:77)
or, accumulating, quantize_state(dequantize(entry) + G) (accumulate, gradflow.hpp:52-58).

Parity: the epilogue's quantization is byte-compared with the CPU oracle applied to the
fp32 values the same kernel quantized (g_out); the GEMM itself is checked against a
torch fp32 matmul of the same bf16 inputs (fp32 accumulation order differs: tolerance
below)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [  # (out, in, tokens)
    (128, 256, 64),
    (256, 512, 200),     # tokens not a multiple of the 64-token K block (TMA zero fill)
    (136, 320, 96),      # a partial row block and a partial column tile
    (4096, 4096, 512),   # LLaMA-2-7B q/k/v/o
    (11008, 4096, 128),  # gate/up (86 row blocks)
    (4096, 11008, 128),  # down: a row spans 43 tiles (the cross-CTA bound exchange)
]


def _inputs(o, i, t, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    dy = (torch.randn(t, o, device="cuda", generator=g) * 1e-2).to(torch.bfloat16)
    x = torch.randn(t, i, device="cuda", generator=g).to(torch.bfloat16)
    return dy, x


def _entry(cuda, o, i, bw=8):
    st = cuda.QftModelState([(o, i)], bit_width=bw)
    st.init_from_weights(lambda k: cuda.synth((o, i), 5, 0.02, 0.01), 0.01)
    return st


def _gemm_tol(ref, t):
    # fp32 sums of t bf16 products in a different order: |err| <= t * 2^-23 * sum|terms|
    return 1e-5 * ref.abs().max().item() + ref.abs() * 2.0 ** -20


@pytest.mark.parametrize("o,i,t", SHAPES)
@pytest.mark.parametrize("bw", [8, 4])
def test_wgrad_quant_push_matches_oracle(cuda, port, o, i, t, bw):
    if bw == 4 and o * i > 5_000_000:
        pytest.skip("b=4 covered on the smaller shapes")
    st = _entry(cuda, o, i, bw)
    dy, x = _inputs(o, i, t, o + i + t)
    g = torch.empty(o, i, device="cuda")
    nsq = torch.zeros(1, dtype=torch.float64, device="cuda")
    st.sink_wgrad(0, dy, x, g_out=g, norm_sq=nsq, check=True)
    torch.cuda.synchronize()
    ref = dy.float().t() @ x.float()
    err = (g - ref).abs()
    assert (err <= _gemm_tol(ref, t)).all(), f"GEMM off: max err {err.max().item()}"
    # the epilogue's quantization == quantize_state of the values it quantized, byte for byte
    codes, s, z = st.grad_views(0)
    qo, so, zo = port.quantize_state(g.cpu().numpy(), bw)
    assert np.array_equal(s.cpu().numpy(), so), "scale differs from the oracle"
    assert np.array_equal(z.cpu().numpy(), zo), "zero point differs from the oracle"
    assert np.array_equal(codes.cpu().numpy(), qo), "codes differ from the oracle"
    want = (g.double() ** 2).sum().item()
    assert abs(nsq.item() - want) <= 1e-5 * want


@pytest.mark.parametrize("o,i,t", [(256, 512, 128), (136, 320, 96), (4096, 11008, 64)])
def test_wgrad_quant_accumulate_matches_oracle(cuda, port, o, i, t):
    """Three micro-batches: push, then two integer-form accumulations in place."""
    st = _entry(cuda, o, i)
    scratch = _entry(cuda, o, i)
    dy, x = _inputs(o, i, t, 11)
    st.sink_wgrad(0, dy, x, check=True)
    codes, s, z = st.grad_views(0)
    acc = (codes.cpu().numpy(), s.cpu().numpy(), z.cpu().numpy())
    for mb in range(2):
        dy, x = _inputs(o, i, t, 100 + mb)
        g = torch.empty(o, i, device="cuda")
        scratch.sink_wgrad(0, dy, x, g_out=g)  # the micro-batch's G (same kernel, same order)
        sums = torch.empty(o, i, device="cuda")
        st.sink_wgrad(0, dy, x, accumulate=True, g_out=sums, check=True)
        torch.cuda.synchronize()
        acc = port.accumulate(*acc, g.cpu().numpy(), 8)
        assert np.array_equal(s.cpu().numpy(), acc[1]), f"micro-batch {mb}: scale differs"
        assert np.array_equal(z.cpu().numpy(), acc[2]), f"micro-batch {mb}: zero point differs"
        assert np.array_equal(codes.cpu().numpy(), acc[0]), f"micro-batch {mb}: codes differ"
        # g_out holds dequantize(entry) + G, the values quantized
        qs = port.quantize_state(sums.cpu().numpy(), 8)
        assert np.array_equal(qs[0], acc[0])


def test_wgrad_quant_exact_values_and_ties(cuda, port):
    """One-hot dy: G's rows are x's bf16 rows exactly, on a coarse grid, so many values land
    on or next to the quantizer's half-integers (the exact fallback), plus constant and zero
    rows."""
    o, i, t = 256, 512, 64
    dy = torch.zeros(t, o, device="cuda")
    dy[torch.arange(o, device="cuda") % t, torch.arange(o, device="cuda")] = 1.0
    dy[:, 200:210] = 0.0                    # zero gradient rows
    x = (torch.randint(-64, 64, (t, i), device="cuda").float() / 8.0)
    x[3, :] = 0.75                          # constant row (o = 3, 67, 131, 195)
    dy, x = dy.to(torch.bfloat16), x.to(torch.bfloat16)
    for bw in (8, 3):
        st = _entry(cuda, o, i, bw)
        g = torch.empty(o, i, device="cuda")
        st.sink_wgrad(0, dy, x, g_out=g, check=True)
        torch.cuda.synchronize()
        assert torch.equal(g, dy.float().t() @ x.float())  # exact: one product per element
        codes, s, z = st.grad_views(0)
        qo, so, zo = port.quantize_state(g.cpu().numpy(), bw)
        assert np.array_equal(codes.cpu().numpy(), qo)
        assert np.array_equal(s.cpu().numpy(), so)
        assert np.array_equal(z.cpu().numpy(), zo)


def test_wgrad_quant_nan_in_column0_is_rejected(cuda):
    st = _entry(cuda, 128, 256)
    dy, x = _inputs(128, 256, 64, 3)
    x[5, 0] = float("nan")
    with pytest.raises(ValueError):
        st.sink_wgrad(0, dy, x, check=True)


def test_wgrad_quant_nan_elsewhere_quantizes_to_zero(cuda, port):
    st = _entry(cuda, 128, 256)
    dy, x = _inputs(128, 256, 64, 4)
    x[7, 100] = float("nan")  # column 100 of every row is NaN: never a bound, code 0
    g = torch.empty(128, 256, device="cuda")
    st.sink_wgrad(0, dy, x, g_out=g, check=True)
    torch.cuda.synchronize()
    codes, s, z = st.grad_views(0)
    qo, so, zo = port.quantize_state(g.cpu().numpy(), 8)
    assert np.array_equal(codes.cpu().numpy(), qo) and np.array_equal(s.cpu().numpy(), so)
    assert (codes[:, 100] == 0).all()


def test_wgrad_feeds_the_step(cuda, port):
    """backward (fused sink) -> lion_step_quantized on the GPU == the oracle's step popping
    the same entry."""
    o, i, t = 256, 4096, 128
    st = _entry(cuda, o, i)
    w0 = st.export_tensor(0)
    dy, x = _inputs(o, i, t, 21)
    st.sink_wgrad(0, dy, x, check=True)
    codes, s, z = st.grad_views(0)
    gq = (codes.cpu().numpy(), s.cpu().numpy(), z.cpu().numpy())
    st.step(lr=2e-5, check=True)
    got = st.export_tensor(0)
    d = port.decompose_weight(port.synth((o, i), 5, 0.02, 0.01), 0.01, 8)
    m = port.quantize_state(np.zeros((o, i), np.float32), 8)
    assert np.array_equal(w0["codes"], d.codes)
    d2, m2 = port.lion_step_layer(d, *m, *gq, lr=2e-5)[:2]
    assert np.array_equal(got["codes"], d2.codes)
    assert np.array_equal(got["m_codes"], m2[0])
    assert np.array_equal(got["values"], d2.values)


def test_wgrad_rejects_bad_shapes(cuda):
    st = _entry(cuda, 128, 100)
    dy = torch.zeros(64, 128, dtype=torch.bfloat16, device="cuda")
    x = torch.zeros(64, 100, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(NotImplementedError):
        st.sink_wgrad(0, dy, x)
    st = _entry(cuda, 128, 256)
    with pytest.raises(ValueError):
        st.sink_wgrad(0, dy, torch.zeros(32, 256, dtype=torch.bfloat16, device="cuda"))
