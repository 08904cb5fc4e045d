"""The stable tier's proof, checked on the CPU against the oracle (no GPU code involved).

rowstep.cu (k_step_prep) declares a row "stable" when one Lion step provably cannot move
any dense weight code in [1, qmax-1] (condition (*) in DESIGN.md §2), and tabulates the
outcome of a dense code-0 / code-qmax weight for each sign of d.  Here the same per-row
condition is evaluated in numpy (fp64, the reference's rounding), one reference step is
run by the oracle (optimizer.hpp:103-118), and on every stable row:

* every dense code in [1, qmax-1] is unchanged and not in the new CSR;
* every dense boundary code follows the tabulated outcome selected by
  sign(RN(RN(b1*m) + RN(c1*g))) (code, and outlier or not).
"""
import numpy as np
import pytest

B1, B2 = np.float32(0.9), np.float32(0.99)
C1 = np.float32(np.float32(1.0) - B1)


def _round_half_away(x):
    """std::round on doubles, exactly (quantize.hpp:168)."""
    x = np.asarray(x, np.float64)
    f = np.floor(x)
    up = (x - f) >= 0.5          # x - f is exact for |x| < 2^52
    r = f + up
    neg = x < 0                  # half away from zero: -2.5 -> -3
    fn = np.floor(-x)
    rn = -(fn + (((-x) - fn) >= 0.5))
    return np.where(neg, rn, r)


def _quant_code(x, s, z, qmax):
    """quantize() of one value (quantize.hpp:160-170): fp64 divide, half-away, clip."""
    q = _round_half_away(np.float64(x) / np.float64(s)) + z
    q = np.where(np.isnan(q) | (q <= 0), 0, q)
    return np.minimum(q, qmax).astype(np.int64)


def _stable_rows(d, ms, mz, gs, gz, bw, lr, wd):
    """k_step_prep's stable-tier condition, row by row (fp64)."""
    qmax = (1 << bw) - 1
    sw = d.scale.astype(np.float64)
    zw = d.zero_point.astype(np.float64)
    fast = lambda s, z: (np.abs(z) < 2 ** 22) & (s >= 2.0 ** -126) & (s <= 2.0 ** 100)
    ok = fast(sw, zw) & fast(ms.astype(np.float64), mz) & fast(gs.astype(np.float64), gz)
    ok &= (ms.astype(np.float64) * (qmax + np.abs(mz)) <= 2.0 ** 120)
    ok &= (gs.astype(np.float64) * (qmax + np.abs(gz)) <= 2.0 ** 120)
    ok &= d.t_min <= d.t_max
    ok &= (_round_half_away(d.t_min.astype(np.float64) / sw) + zw) == 0
    ok &= (_round_half_away(d.t_max.astype(np.float64) / sw) + zw) == qmax
    K = qmax + np.abs(zw)
    wmax = sw * K * (1 + 2.0 ** -20)
    D = abs(lr) * (1 + abs(wd) * wmax) * (1 + 2.0 ** -20)
    ok &= D / sw <= 0.5 - (K + 2) * 2.0 ** -21
    return ok


def _outcome(B, S, sw, zw, tmin, tmax, zpay, lr, wd, qmax):
    """The tabulated outcome: w = dequant(B), w' = w - lr*(s + wd*w), s = S - 1."""
    w = np.float32(np.float32(sw) * np.float32(B - zw))
    s = np.float32(S - 1)
    wn = np.float32(w - np.float32(np.float32(lr) * np.float32(s + np.float32(np.float32(wd) * w))))
    o = bool(wn < tmin or wn > tmax)
    return (zpay if o else int(_quant_code(wn, sw, zw, qmax))), o


@pytest.mark.parametrize("bw,frac", [(8, 0.01), (8, 0.0045), (4, 0.0045), (3, 0.0045)])
@pytest.mark.parametrize("lr,wd", [(2e-5, 0.0), (1.5e-4, 0.01), (2.2e-4, 0.0)])
def test_stable_tier_proof_against_oracle(port, bw, frac, lr, wd):
    shape = (24, 2752)
    qmax = (1 << bw) - 1
    w = port.synth(shape, 4242 + bw, 0.02, 0.005)
    d = port.decompose_weight(w, frac, bw)
    m = port.quantize_state(np.zeros(shape, np.float32), bw)
    for k in range(2):  # give the momentum real codes
        gq = port.quantize_state(port.synth(shape, 900 + k, 1e-2, 0.0), bw)
        d, m, _ = port.lion_step_layer(d, *m, *gq, lr=lr, wd=wd)
    gq = port.quantize_state(port.synth(shape, 999, 1e-2, 0.01), bw)
    stable = _stable_rows(d, m[1], m[2], gq[1], gq[2], bw, lr, wd)
    assert stable.any(), "no stable row: the test would be vacuous"
    nd, _, tr = port.lion_step_layer(d, *m, *gq, lr=lr, wd=wd, trace=True)

    checked_dense = checked_boundary = 0
    for r in np.flatnonzero(stable):
        old = set(d.col_idx[d.row_ptr[r]:d.row_ptr[r + 1]].tolist())
        new = set(nd.col_idx[nd.row_ptr[r]:nd.row_ptr[r + 1]].tolist())
        dense = np.ones(shape[1], bool)
        dense[list(old)] = False
        k0 = d.codes[r].astype(np.int64)
        inner = dense & (k0 >= 1) & (k0 <= qmax - 1)
        assert np.array_equal(nd.codes[r][inner], d.codes[r][inner]), f"row {r}: inner code moved"
        assert not (set(np.flatnonzero(inner).tolist()) & new), f"row {r}: inner code left"
        checked_dense += int(inner.sum())
        sw, zw = d.scale[r], int(d.zero_point[r])
        zpay = min(max(zw, 0), qmax)
        for c in np.flatnonzero(dense & ((k0 == 0) | (k0 == qmax))):
            mv, gv = np.float32(tr["m_in"][r, c]), np.float32(tr["g"][r, c])
            dd = np.float32(np.float32(B1 * mv) + np.float32(C1 * gv))
            S = 2 if dd > 0 else (0 if dd < 0 else 1)
            code, o = _outcome(int(k0[c]), S, sw, zw, d.t_min[r], d.t_max[r], zpay, lr, wd, qmax)
            assert int(nd.codes[r, c]) == code, f"row {r} col {c}: code {nd.codes[r, c]} vs {code}"
            assert (int(c) in new) == o, f"row {r} col {c}: outlier class"
            checked_boundary += 1
    assert checked_dense > 0
