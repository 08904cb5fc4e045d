"""QFTC v1 checkpoints from / into the device state (paper_2310_07147_b200/checkpoint.py)
against the reference's own files (tests/golden/ckpt_*, see test_checkpoint_golden.py):

* qftc_crc32 (GPU) equals zlib.crc32 over any split of the stream into segments;
* load(reference file) -> save is byte-identical to the reference file;
* load(ckpt_a) + the golden gradients -> one device step -> save is byte-identical to
  the reference's ckpt_b (the step checked through the reference's on-disk format);
* corrupt / truncated / foreign files fail with the reference's messages
  (checkpoint.cpp:142-211).
"""
import ctypes as C
import os
import zlib

import numpy as np
import pytest
import torch

from test_checkpoint_golden import CASES, GOLD, grads, parse

pytestmark = pytest.mark.gpu


def _crc(N, segs):
    ptrs = (C.c_void_p * max(len(segs), 1))(*[t.data_ptr() for t in segs])
    lens = (C.c_int64 * max(len(segs), 1))(*[t.numel() for t in segs])
    out = C.c_uint32(0)
    N.check(N.lib.qftc_crc32(ptrs, lens, len(segs), C.byref(out),
                             C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out.value


def test_crc32_device_matches_zlib(cuda):
    from paper_2310_07147_b200 import _native as N
    rng = np.random.default_rng(3)
    data = rng.integers(0, 256, 3 * 65536 * 7 + 12345, dtype=np.uint8)
    dev = torch.from_numpy(data).cuda()
    assert _crc(N, [dev]) == zlib.crc32(data.tobytes())
    assert _crc(N, []) == zlib.crc32(b"")
    # arbitrary splits: empty, 1 byte, around the 64 KB chunk and 2 KB lane sizes,
    # unaligned starts
    cuts = [0, 0, 1, 2, 7, 2048, 2049, 65535, 65536, 65537, 131075, 400001, 1000000,
            len(data)]
    segs = [dev[a:b] for a, b in zip(cuts[:-1], cuts[1:])]
    assert _crc(N, segs) == zlib.crc32(data.tobytes())
    big = torch.randint(0, 256, (64 << 20,), dtype=torch.uint8, device="cuda")
    assert _crc(N, [big[3:]]) == zlib.crc32(big[3:].cpu().numpy().tobytes())


@pytest.mark.parametrize("name", sorted(CASES))
def test_load_save_roundtrip_is_byte_identical(cuda, tmp_path, name):
    from paper_2310_07147_b200.checkpoint import load_checkpoint, save_checkpoint
    src = os.path.join(GOLD, f"{name}_a.qftc")
    st, meta = load_checkpoint(src)
    out = tmp_path / "re.qftc"
    save_checkpoint(st, str(out), meta)
    assert out.read_bytes() == open(src, "rb").read()


@pytest.mark.parametrize("name", sorted(CASES))
def test_device_step_matches_reference_checkpoint(cuda, tmp_path, name):
    from paper_2310_07147_b200.checkpoint import load_checkpoint, save_checkpoint
    lr, wd = CASES[name]
    st, meta = load_checkpoint(os.path.join(GOLD, f"{name}_a.qftc"))
    layers = parse(os.path.join(GOLD, f"{name}_a.qftc"))["layers"]
    for i, (q, s, z) in enumerate(grads(os.path.join(GOLD, f"{name}_g.bin"), layers)):
        c, sc, zz = st.grad_views(i)
        c.copy_(torch.from_numpy(q))
        sc.copy_(torch.from_numpy(s))
        zz.copy_(torch.from_numpy(z))
    st.step(lr=lr, beta1=0.9, beta2=0.99, weight_decay=wd, check=True)
    out = tmp_path / "b.qftc"
    save_checkpoint(st, str(out), meta)
    want = open(os.path.join(GOLD, f"{name}_b.qftc"), "rb").read()
    got = out.read_bytes()
    if got != want:  # name the first differing field
        a, b = parse(str(out)), parse(os.path.join(GOLD, f"{name}_b.qftc"))
        for li, (x, y) in enumerate(zip(a["layers"], b["layers"])):
            for k in x:
                assert np.array_equal(np.asarray(x[k]), np.asarray(y[k])), f"layer {li} {k}"
    assert got == want


def test_load_errors_match_reference(cuda, tmp_path):
    from paper_2310_07147_b200.checkpoint import load_checkpoint
    good = open(os.path.join(GOLD, "ckpt_b8_a.qftc"), "rb").read()

    def fails(data, msg):
        p = tmp_path / "x.qftc"
        p.write_bytes(data)
        with pytest.raises(RuntimeError, match=msg):
            load_checkpoint(str(p))

    fails(b"QFT", "is truncated")
    fails(b"NOPE" + good[4:], r"is not a checkpoint \(bad magic\)")
    bad = bytearray(good)
    bad[100] ^= 1
    fails(bytes(bad), r"is corrupt \(crc mismatch\)")
    # a consistent CRC over a wrong version / a truncated body / trailing bytes
    import struct

    def with_crc(body):
        return body + struct.pack("<I", zlib.crc32(body))

    body = bytearray(good[:-4])
    body[4] = 2
    fails(with_crc(bytes(body)), "has unsupported version 2")
    fails(with_crc(good[:-4][:-10]), "is truncated")
    fails(with_crc(good[:-4] + b"\0"), "has trailing bytes")
    with pytest.raises(RuntimeError, match="cannot open checkpoint"):
        load_checkpoint(str(tmp_path / "missing.qftc"))


def test_engine_state_roundtrip_then_identical_steps(cuda, tmp_path):
    """A LLaMA-shaped engine state (grouped width classes, slotted CSR) saved, loaded
    and re-saved byte-identically; the loaded copy and the original then take the same
    step and export the same bytes."""
    from paper_2310_07147_b200.checkpoint import CheckpointMeta, load_checkpoint, save_checkpoint
    from paper_2310_07147_b200.shapes import llama
    shapes = llama(512, 1376, 2, 1000)
    st = cuda.QftModelState(shapes, bit_width=8)
    st.init_from_weights(lambda i: cuda.synth(shapes[i], 31 + i, 0.02, 0.005), 0.01)
    for i, sh in enumerate(shapes):  # give the momentum real codes
        q = cuda.quantize_state(cuda.synth(sh, 500 + i, 1e-3, 0.0), 8)
        c, s, z = st.grad_views(i)
        c.copy_(q.data); s.copy_(q.params.scale); z.copy_(q.params.zero_point)
    st.step(lr=2e-4, check=True)
    junc = [(k + 1) % 2 for k in range(len(shapes) - 1)]  # relu / none alternating
    meta = CheckpointMeta(bit_width=8, loss=1, outlier_fraction=0.01, junctions=junc)
    p1, p2 = tmp_path / "a.qftc", tmp_path / "b.qftc"
    save_checkpoint(st, str(p1), meta)
    st2, meta2 = load_checkpoint(str(p1))
    assert meta2.junctions == meta.junctions and meta2.loss == 1
    save_checkpoint(st2, str(p2), meta2)
    assert p1.read_bytes() == p2.read_bytes()
    for s_ in (st, st2):
        for i, sh in enumerate(shapes):
            q = cuda.quantize_state(cuda.synth(sh, 900 + i, 1e-3, 0.0), 8)
            c, s, z = s_.grad_views(i)
            c.copy_(q.data); s.copy_(q.params.scale); z.copy_(q.params.zero_point)
        s_.step(lr=2e-4, check=True)
    for i in range(len(shapes)):
        a, b = st.export_tensor(i), st2.export_tensor(i)
        for k in a:
            assert np.array_equal(a[k], b[k]), f"tensor {i} {k}"
