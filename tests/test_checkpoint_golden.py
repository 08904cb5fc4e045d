"""QFTC v1 checkpoint golden files (tests/golden/ckpt_*, written by the reference's own
save_checkpoint, tests/golden/make_golden_ckpt.sh), checked on the CPU:

* the file layout and CRC as restated in paper_2310_07147_b200/checkpoint.py's docstring
  (checkpoint.cpp:100-140), parsed here independently with numpy + zlib.crc32;
* the oracle's Lion step reproduces the reference's third step: ckpt_*_a + the
  gradients in ckpt_*_g.bin -> ckpt_*_b, byte for byte.
"""
import os
import struct
import zlib

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = {"ckpt_b8": (1e-3, 0.0), "ckpt_b4": (2e-3, 0.01), "ckpt_b3": (5e-3, 0.0)}


def parse(path):
    buf = open(path, "rb").read()
    assert buf[:4] == b"QFTC"
    assert zlib.crc32(buf[:-4]) == struct.unpack("<I", buf[-4:])[0], "crc"
    p = 4
    ver, L, bw, mode, kind, loss = struct.unpack_from("<HHBBBB", buf, p)
    p += 8
    junc = list(buf[p:p + L - 1])
    p += L - 1
    frac = struct.unpack_from("<f", buf, p)[0]
    p += 4

    def arr(dt, n):
        nonlocal p
        a = np.frombuffer(buf, dt, n, p).copy()
        p += a.nbytes
        return a

    layers = []
    for _ in range(L):
        r, c = struct.unpack_from("<II", buf, p)
        p += 8
        d = dict(rows=r, cols=c, t_min=arr("<f4", r), t_max=arr("<f4", r), scale=arr("<f4", r),
                 zp=arr("<i4", r), codes=arr("u1", r * c).reshape(r, c))
        nnz = struct.unpack_from("<I", buf, p)[0]
        p += 4
        d.update(row_ptr=arr("<i4", r + 1), col=arr("<i4", nnz), val=arr("<f4", nnz),
                 m_scale=arr("<f4", r), m_zp=arr("<i4", r), m_codes=arr("u1", r * c).reshape(r, c))
        layers.append(d)
    assert p == len(buf) - 4, "trailing bytes"
    return dict(version=ver, bw=bw, mode=mode, kind=kind, loss=loss, junctions=junc,
                fraction=frac, layers=layers)


def grads(path, layers):
    raw = open(path, "rb").read()
    p, out = 0, []
    for d in layers:
        r, c = d["rows"], d["cols"]
        s = np.frombuffer(raw, "<f4", r, p).copy(); p += 4 * r
        z = np.frombuffer(raw, "<i4", r, p).copy(); p += 4 * r
        q = np.frombuffer(raw, "u1", r * c, p).copy().reshape(r, c); p += r * c
        out.append((q, s, z))
    assert p == len(raw)
    return out


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_layout_and_crc(name):
    for ab in "ab":
        ck = parse(os.path.join(GOLD, f"{name}_{ab}.qftc"))
        assert ck["version"] == 1 and ck["mode"] == 0
        for d in ck["layers"]:
            assert d["row_ptr"][0] == 0 and d["row_ptr"][-1] == d["col"].size
            assert np.all(np.diff(d["row_ptr"]) >= 0)


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_reproduces_reference_third_step(port, name):
    from oracle.oracle import DenseSparse
    lr, wd = CASES[name]
    a = parse(os.path.join(GOLD, f"{name}_a.qftc"))
    b = parse(os.path.join(GOLD, f"{name}_b.qftc"))
    gs = grads(os.path.join(GOLD, f"{name}_g.bin"), a["layers"])
    for la, lb, g in zip(a["layers"], b["layers"], gs):
        d = DenseSparse(codes=la["codes"], scale=la["scale"], zero_point=la["zp"],
                        t_min=la["t_min"], t_max=la["t_max"], row_ptr=la["row_ptr"],
                        col_idx=la["col"], values=la["val"], bit_width=a["bw"])
        nd, m, _ = port.lion_step_layer(d, la["m_codes"], la["m_scale"], la["m_zp"], *g,
                                        lr=lr, wd=wd)
        np.testing.assert_array_equal(nd.codes, lb["codes"])
        np.testing.assert_array_equal(nd.row_ptr, lb["row_ptr"])
        np.testing.assert_array_equal(nd.col_idx, lb["col"])
        np.testing.assert_array_equal(nd.values.view(np.uint32), lb["val"].view(np.uint32))
        np.testing.assert_array_equal(m[0], lb["m_codes"])
        np.testing.assert_array_equal(m[1].view(np.uint32), lb["m_scale"].view(np.uint32))
        np.testing.assert_array_equal(m[2], lb["m_zp"])
