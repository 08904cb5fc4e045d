"""The opt-in QFTC format extensions: bit-packed sub-byte codes
(lossless) and blockwise momentum scales (lossy), in a version-0x8001 file."""
import ctypes as C
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _np_pack(codes, bits):
    """reference bit packing: LSB-first, each row padded to a byte"""
    rows, cols = codes.shape
    out = np.zeros((rows, (cols * bits + 7) // 8), np.uint8)
    for r in range(rows):
        acc, nb, k = 0, 0, 0
        for v in codes[r]:
            acc |= int(v) << nb
            nb += bits
            while nb >= 8:
                out[r, k] = acc & 0xFF
                acc >>= 8
                nb -= 8
                k += 1
        if nb:
            out[r, k] = acc & 0xFF
    return out


@pytest.mark.parametrize("bits", [2, 3, 4, 5, 7, 8])
@pytest.mark.parametrize("cols", [8, 61, 4096])
def test_pack_unpack_roundtrip(cuda, bits, cols):
    rng = np.random.default_rng(bits * 100 + cols)
    rows = 5
    codes = rng.integers(0, 1 << bits, size=(rows, cols), dtype=np.uint8)
    d = torch.from_numpy(codes).cuda()
    packed = torch.empty(rows * ((cols * bits + 7) // 8), dtype=torch.uint8, device="cuda")
    N = cuda._native
    N.check(N.lib.qftc_pack_codes(C.c_void_p(d.data_ptr()), rows, cols, bits,
                                  C.c_void_p(packed.data_ptr()), None))
    assert np.array_equal(packed.cpu().numpy().reshape(rows, -1), _np_pack(codes, bits))
    back = torch.empty(rows * cols, dtype=torch.uint8, device="cuda")
    N.check(N.lib.qftc_unpack_codes(C.c_void_p(packed.data_ptr()), rows, cols, bits,
                                    C.c_void_p(back.data_ptr()), None))
    assert np.array_equal(back.cpu().numpy().reshape(rows, cols), codes)


def _state(cuda, bw):
    from paper_2310_07147_b200.shapes import llama
    shapes = llama(256, 688, 2, 500)
    st = cuda.QftModelState(shapes, bit_width=bw)
    st.init_from_weights(lambda i: cuda.synth(shapes[i], 31 + i, 0.02, 0.005), 0.01)
    for i, sh in enumerate(shapes):  # momentum with real codes
        q = cuda.quantize_state(cuda.synth(sh, 500 + i, 1e-3, 0.0), bw)
        c, s, z = st.grad_views(i)
        c.copy_(q.data); s.copy_(q.params.scale); z.copy_(q.params.zero_point)
    st.step(lr=2e-4, check=True)
    return st


@pytest.mark.parametrize("bw", [3, 4, 8])
def test_packed_checkpoint_is_lossless_and_smaller(cuda, tmp_path, bw):
    from paper_2310_07147_b200.checkpoint import load_checkpoint, save_checkpoint
    st = _state(cuda, bw)
    p1, p2 = tmp_path / "v1.qftc", tmp_path / "packed.qftc"
    save_checkpoint(st, str(p1))
    save_checkpoint(st, str(p2), packed_codes=True)
    codes_bytes = 2 * sum(r * c for r, c in st.shapes)
    assert os.path.getsize(p1) - os.path.getsize(p2) >= int(codes_bytes * (1 - bw / 8)) - 8 * st.n
    with open(p2, "rb") as f:
        assert f.read(6)[4:] == (0x8001).to_bytes(2, "little")  # the extension family
    st2, meta = load_checkpoint(str(p2))
    for i in range(st.n):
        a, b = st.export_tensor(i), st2.export_tensor(i)
        for k in a:
            assert np.array_equal(a[k], b[k]), (i, k)


def test_blockwise_momentum_checkpoint(cuda, tmp_path):
    """Lossy by definition: W is unchanged, the momentum comes back within the two
    quantization steps it went through (block grid, then the row grid)."""
    from paper_2310_07147_b200.checkpoint import load_checkpoint, save_checkpoint
    st = _state(cuda, 8)
    p = tmp_path / "mblk.qftc"
    save_checkpoint(st, str(p), packed_codes=True, momentum_block=128)
    st2, _ = load_checkpoint(str(p))
    for i in range(st.n):
        a, b = st.export_tensor(i), st2.export_tensor(i)
        for k in ("codes", "scale", "zero_point", "t_min", "t_max", "row_ptr", "col_idx", "values"):
            assert np.array_equal(a[k], b[k]), (i, k)
        ma = (a["m_codes"].astype(np.float64) - a["m_zero_point"][:, None]) * a["m_scale"][:, None]
        mb = (b["m_codes"].astype(np.float64) - b["m_zero_point"][:, None]) * b["m_scale"][:, None]
        # block grid error <= s_block/2 <= s_row/2; then requantized on a row grid no wider
        bound = a["m_scale"][:, None] * 1.01 + 1e-30
        assert np.all(np.abs(ma - mb) <= bound), i
