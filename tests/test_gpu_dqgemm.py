"""§8(f) row 1: the forward GEMM with the weight dequantization fused into its operand
producer (qftc_dequant_gemm, tcgen05 + TMA).  y = x . W^T must equal the same GEMM on the
materialised bf16 weights (qftc_expand bf16 = RNE(reconstruct(W)), quantize.hpp:331-338)
up to fp32 accumulation order: within one bf16 rounding of the fp32 reference."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(x, wb):
    return (x.float() @ wb.float().t())


# m <= 256 runs the single-CTA kernel, m > 256 the CTA-pair (cta_group::2) one
@pytest.mark.parametrize("shape,m", [((256, 512), 200), ((384, 1024), 128), ((128, 4096), 77),
                                     ((4096, 4096), 256), ((300, 11008), 130), ((11008, 4096), 64),
                                     ((256, 512), 1000), ((384, 1024), 257), ((4096, 4096), 1024),
                                     ((300, 11008), 600), ((11008, 4096), 513), ((200, 256), 3000)])
def test_dequant_gemm_matches_materialised(cuda, shape, m):
    torch.manual_seed(shape[0] + m)
    st = cuda.QftModelState([shape], bit_width=8)
    st.init_from_weights(lambda i: cuda.synth(shape, 91 + m, 0.02, 0.01), 0.01)
    # a step so the CSR is slotted with real drift
    c, s, z = st.grad_views(0)
    q = cuda.quantize_state(cuda.synth(shape, 7, 1e-3, 0.0), 8)
    c.copy_(q.data); s.copy_(q.params.scale); z.copy_(q.params.zero_point)
    st.step(lr=2e-4, check=True)
    wb = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    st.expand([wb])
    x = (torch.randn(m, shape[1], device="cuda") * 0.5).to(torch.bfloat16)
    y = st.linear(0, x)
    torch.cuda.synchronize()
    ref = _ref(x, wb)
    err = (y.float() - ref).abs()
    tol = ref.abs() * 2.0 ** -7 + 1e-3 * ref.abs().max()
    bad = (err > tol).sum().item()
    assert bad == 0, f"{bad} elements off; max err {err.max().item()} vs |ref| max {ref.abs().max().item()}"
    # the bf16 results themselves agree almost everywhere (only fp32 accumulation-order ties
    # of the final rounding may differ)
    same = (y == ref.to(torch.bfloat16)).float().mean().item()
    assert same > 0.98, f"only {same:.4f} of the bf16 outputs equal the reference's rounding"
    # and the outliers matter: the GEMM on the payload-only dense part differs
    assert st.nnz() > 0


def test_dequant_gemm_rejects_bad_k(cuda):
    st = cuda.QftModelState([(64, 100)], bit_width=8)
    st.init_from_weights(lambda i: cuda.synth((64, 100), 1, 0.02, 0.01), 0.01)
    x = torch.zeros(8, 100, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(NotImplementedError):
        st.linear(0, x)


# tokens <= 256: the single-CTA kernel; > 256: the CTA pair
@pytest.mark.parametrize("shape,m", [((128, 256), 200), ((384, 1024), 512), ((4096, 4096), 256),
                                     ((11008, 4096), 130), ((4096, 11008), 64), ((192, 320), 77),
                                     ((4096, 4096), 1024), ((11008, 4096), 600),
                                     ((4096, 11008), 513), ((192, 320), 300), ((128, 256), 1000)])
def test_dequant_gemm_t_matches_materialised(cuda, shape, m):
    """The backward weight operand: dx = dy . W (network.hpp:145) with W dequantized as an
    MN-major operand (qftc_dequant_gemm_t) == the GEMM on the materialised bf16 weights."""
    torch.manual_seed(shape[1] + m)
    st = cuda.QftModelState([shape], bit_width=8)
    st.init_from_weights(lambda i: cuda.synth(shape, 17 + m, 0.02, 0.01), 0.01)
    c, s, z = st.grad_views(0)
    q = cuda.quantize_state(cuda.synth(shape, 8, 1e-3, 0.0), 8)
    c.copy_(q.data); s.copy_(q.params.scale); z.copy_(q.params.zero_point)
    st.step(lr=2e-4, check=True)  # slotted CSR with drift
    wb = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    st.expand([wb])
    dy = (torch.randn(m, shape[0], device="cuda") * 0.5).to(torch.bfloat16)
    dx = st.linear_backward(0, dy)
    torch.cuda.synchronize()
    ref = dy.float() @ wb.float()
    err = (dx.float() - ref).abs()
    tol = ref.abs() * 2.0 ** -7 + 1e-3 * ref.abs().max()
    bad = (err > tol).sum().item()
    assert bad == 0, f"{bad} elements off; max err {err.max().item()}"
    same = (dx == ref.to(torch.bfloat16)).float().mean().item()
    assert same > 0.98, f"only {same:.4f} of the bf16 outputs equal the reference's rounding"
    # every outlier is in the operand: the GEMM on the payload-only weights differs
    assert st.nnz() > 0


def test_dequant_gemm_t_rejects_bad_shapes(cuda):
    st = cuda.QftModelState([(100, 128)], bit_width=8)
    st.init_from_weights(lambda i: cuda.synth((100, 128), 1, 0.02, 0.01), 0.01)
    dy = torch.zeros(8, 100, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(NotImplementedError):
        st.linear_backward(0, dy)


@pytest.mark.parametrize("shape,m", [((4096, 4096), 200), ((4096, 4096), 600),
                                     ((256, 1024), 1000), ((320, 512), 77)])
def test_dequant_gemms_strict_csr_via_c_abi(cuda, port, shape, m):
    """Both GEMM entry points through the raw C-ABI with a STRICT CSR (row_count = NULL:
    row r's entries are row_ptr[r] .. row_ptr[r+1]) straight from the oracle's
    decompose_weight (quantize.hpp:301-314), single CTA and CTA pair: equal to the GEMMs on
    RNE(reconstruct(W)) (the oracle's fp32 reconstruction rounded to bf16)."""
    import ctypes as C
    N = cuda._native
    r, c = shape
    w = port.synth(shape, 4000 + m, 0.02, 0.005)
    d = port.decompose_weight(w, 0.01, 8)
    wb = torch.from_numpy(port.reconstruct(d)).cuda().to(torch.bfloat16)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    codes, sc, zp = dev(d.codes), dev(d.scale), dev(d.zero_point)
    rp, col, val = dev(d.row_ptr.astype(np.int32)), dev(d.col_idx.astype(np.int32)), dev(d.values)
    vp = lambda t: C.c_void_p(t.data_ptr())
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    # forward: y = x . W^T
    x = (torch.randn(m, c, device="cuda") * 0.5).to(torch.bfloat16)
    y = torch.empty((m, r), dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(int(N.lib.qftc_dequant_gemm_workspace_bytes(r, c)), dtype=torch.uint8, device="cuda")
    N.check(N.lib.qftc_dequant_gemm(vp(x), m, c, vp(codes), r, vp(sc), vp(zp), vp(rp), None,
                                    vp(col), vp(val), vp(y), vp(ws), s))
    # backward: dx = dy . W
    dy = (torch.randn(m, r, device="cuda") * 0.5).to(torch.bfloat16)
    dx = torch.empty((m, c), dtype=torch.bfloat16, device="cuda")
    wst = torch.empty(int(N.lib.qftc_dequant_gemm_t_workspace_bytes(r, c)), dtype=torch.uint8,
                      device="cuda")
    N.check(N.lib.qftc_dequant_gemm_t(vp(dy), m, r, vp(codes), c, vp(sc), vp(zp), vp(rp), None,
                                      vp(col), vp(val), vp(dx), vp(wst), s))
    torch.cuda.synchronize()
    for got, ref, what in ((y, x.float() @ wb.float().t(), "forward"),
                           (dx, dy.float() @ wb.float(), "dx")):
        err = (got.float() - ref).abs()
        tol = ref.abs() * 2.0 ** -7 + 1e-3 * ref.abs().max()
        assert int((err > tol).sum()) == 0, f"{what}: max err {err.max().item()}"
        same = (got == ref.to(torch.bfloat16)).float().mean().item()
        assert same > 0.98, f"{what}: only {same:.4f} equal the reference's rounding"
    assert d.row_ptr[-1] > 0


@pytest.mark.parametrize("shape,m", [((4096, 4096), 600), ((384, 1024), 128), ((11008, 4096), 513)])
def test_dequant_gemms_prebuilt_index_equal(cuda, shape, m):
    """The _prebuilt forms with csr_index(i) (built once per weight version) give the same
    bytes as the calls that rebuild the index, forward and dx; the forward and dx index
    workspaces have the same size (one index serves both)."""
    N = cuda._native
    r, c = shape
    assert (int(N.lib.qftc_dequant_gemm_workspace_bytes(r, c)) ==
            int(N.lib.qftc_dequant_gemm_t_workspace_bytes(r, c)))
    st = cuda.QftModelState([shape], bit_width=8)
    st.init_from_weights(lambda i: cuda.synth(shape, 5 + m, 0.02, 0.01), 0.01)
    cc, s, z = st.grad_views(0)
    q = cuda.quantize_state(cuda.synth(shape, 9, 1e-3, 0.0), 8)
    cc.copy_(q.data); s.copy_(q.params.scale); z.copy_(q.params.zero_point)
    st.step(lr=2e-4, check=True)  # slotted CSR with drift
    x = (torch.randn(m, c, device="cuda") * 0.5).to(torch.bfloat16)
    dy = (torch.randn(m, r, device="cuda") * 0.5).to(torch.bfloat16)
    idx = st.csr_index(0)
    y0, y1 = st.linear(0, x), st.linear(0, x, index=idx)
    d0, d1 = st.linear_backward(0, dy), st.linear_backward(0, dy, index=idx)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1) and torch.equal(d0, d1)
