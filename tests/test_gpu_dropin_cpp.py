"""The drop-in boundary, proven from both host languages the reference offers.

C++: oracle/_ref/dropin_test (oracle/dropin_test.cpp, compiled by oracle/Makefile against
the reference's unmodified headers and linked with the product library) calls
qft::X and qft_b200::X with the same source text on the reference's own Model /
LionState / GradientStack / LionStepTrace and byte-compares everything: the quantizer
surface, >= 5 Lion steps at 8 and 4 bits with and without a trace, the pass-through
model, and the stack validation of test_optimizer.cpp:296-328 including the partially
updated state after a throw.

Python: the same validation cases (test_optimizer.cpp:296-328) through the package's
reference-named API (quantize.lion_step_quantized).
"""
import os
import subprocess

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


def test_cpp_dropin_against_reference(cuda):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin ok" in r.stdout, r.stdout


def _model(cuda, port, dims, seed, bw=8):
    """layers [out x in] decomposed by the oracle, momentum = LionState::init (zeros)"""
    ws, st, ora = [], [], []
    for li in range(len(dims) - 1):
        sh = (dims[li + 1], dims[li])
        d = port.decompose_weight(port.synth(sh, seed + li, 0.5, 0.0), 0.01, bw)
        m = port.quantize_state(np.zeros(sh, np.float32), bw)
        ws.append(cuda.DenseSparseWeight(
            cuda.QuantizedTensor(sh[0], sh[1], torch.from_numpy(d.codes).cuda(),
                                 cuda.AffineParams(torch.from_numpy(d.scale).cuda(),
                                                   torch.from_numpy(d.zero_point).cuda(), bw)),
            cuda.SparseOutliers(torch.from_numpy(d.row_ptr).cuda(),
                                torch.from_numpy(d.col_idx).cuda(),
                                torch.from_numpy(d.values).cuda()),
            torch.from_numpy(d.t_min).cuda(), torch.from_numpy(d.t_max).cuda(), 0.01))
        st.append(cuda.QuantizedTensor(sh[0], sh[1], torch.from_numpy(m[0]).cuda(),
                                       cuda.AffineParams(torch.from_numpy(m[1]).cuda(),
                                                         torch.from_numpy(m[2]).cuda(), bw)))
        ora.append((d, m))
    return ws, cuda.LionState(st), ora


def _q(cuda, port, sh, seed):
    c, s, z = port.quantize_state(port.synth(sh, seed, 1.0, 0.0), 8)
    return cuda.QuantizedTensor(sh[0], sh[1], torch.from_numpy(c).cuda(),
                                cuda.AffineParams(torch.from_numpy(s).cuda(),
                                                  torch.from_numpy(z).cuda(), 8)), (c, s, z)


@pytest.mark.parametrize("case", ["wrong depth", "wrong order", "wrong shape",
                                  "momentum count mismatch", "bad shape below a good layer"])
def test_step_validation_rejects_malformed_stacks(cuda, port, case):
    """test_optimizer.cpp:296-328 through the Python API (layer dims {4, 6, 2}): every
    malformed stack raises ValueError (std::invalid_argument); layers above the bad entry
    are updated before the throw, exactly as the reference's interleaved loop does."""
    ws, st, ora = _model(cuda, port, [4, 6, 2], 10)
    h = cuda.LionHyper(lr=1e-2)
    stack = cuda.GradientStack()
    pushes = {"wrong depth": [(1, (6, 4))],
              "wrong order": [(1, (6, 4)), (2, (2, 6))],
              "wrong shape": [(2, (2, 6)), (1, (5, 5))],
              "momentum count mismatch": [(2, (2, 6)), (1, (6, 4))],
              "bad shape below a good layer": [(2, (3, 3)), (1, (6, 4))]}[case]
    host = {}
    for k, (li, sh) in enumerate(pushes):
        g, gh = _q(cuda, port, sh, 77 + k)
        stack.push(li, g)
        host[li] = gh
    if case == "momentum count mismatch":
        st.momentum.pop()
    before = [w.dense.data.clone() for w in ws]
    with pytest.raises(ValueError):
        cuda.lion_step_quantized(ws, st, stack, h, 8)
    if case == "bad shape below a good layer":
        # layer 1 was popped, validated and updated; layer 2 threw
        d, m = ora[0]
        d2, m2, _ = port.lion_step_layer(d, *m, *host[1], lr=1e-2)
        assert np.array_equal(ws[0].dense.data.cpu().numpy(), d2.codes)
        assert np.array_equal(st.momentum[0].data.cpu().numpy(), m2[0])
        assert torch.equal(ws[1].dense.data, before[1])
        assert stack.size() == 0
    else:
        for w, b in zip(ws, before):
            assert torch.equal(w.dense.data, b)


def test_empty_pop_is_out_of_range(cuda):
    """gradflow.hpp:31: pop on an empty stack -> std::out_of_range (IndexError)."""
    with pytest.raises(IndexError):
        cuda.GradientStack().pop()
