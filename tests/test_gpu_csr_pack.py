"""qftc_csr_pack (the ZeRO-1 all-gather of only the used CSR entries): random slotted
segments of several width classes -- empty rows, empty segments, rows whose count
overflowed their slot (clamped) -- packed per class in segment order, row starts re-based
by the class's base.  Compared with a numpy restatement."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _restated(segs, rs, cnt, arenas, base):
    out_rs = rs.copy()
    packed = {w: ([], []) for w in arenas}
    fill = {w: 0 for w in arenas}
    for rows, ro, co, w in segs:
        for r in range(rows):
            s = rs[ro + r]
            n = max(0, min(cnt[co + r], rs[ro + r + 1] - s))
            out_rs[ro + r] = base[w] + fill[w]
            packed[w][0].append(arenas[w][0][s:s + n])
            packed[w][1].append(arenas[w][1][s:s + n])
            fill[w] += n
        out_rs[ro + rows] = base[w] + fill[w]
    return out_rs, {w: (np.concatenate(c) if c else np.zeros(0, np.int32),
                        np.concatenate(v) if v else np.zeros(0, np.float32))
                    for w, (c, v) in packed.items()}, fill


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_csr_pack_matches_restatement(cuda, seed):
    N = cuda._native
    rng = np.random.default_rng(seed)
    nw = 3
    seg_rows = [int(x) for x in rng.integers(0, 700, size=11)]
    seg_rows[3] = 0                                     # an empty segment
    seg_rows[5] = 1100                                  # five chunks
    seg_w = [int(x) for x in rng.integers(0, nw, size=len(seg_rows))]
    segs, rs_l, cnt_l = [], [], []
    arena_fill = [0] * nw
    ro = co = 0
    for rows, w in zip(seg_rows, seg_w):
        cap = (rng.integers(0, 40, size=rows) // 4 * 4).astype(np.int32)
        cnt = np.minimum(cap, rng.integers(0, 40, size=rows)).astype(np.int32)
        if rows > 5:
            cnt[1] = cap[1] + 7                         # an overflowed row: clamped to its slot
            cnt[2] = 0
        start = arena_fill[w] + np.concatenate([[0], np.cumsum(cap)]).astype(np.int32)
        arena_fill[w] = int(start[-1]) + 8              # slack between segments
        segs.append((rows, ro, co, w))
        rs_l.append(start)
        cnt_l.append(cnt)
        ro += rows + 1
        co += rows
    rs = np.concatenate(rs_l).astype(np.int32)
    cnt = np.concatenate(cnt_l).astype(np.int32)
    arenas = {w: (rng.integers(0, 1 << 20, size=arena_fill[w] + 4).astype(np.int32),
                  rng.standard_normal(arena_fill[w] + 4).astype(np.float32)) for w in range(nw)}
    base = {w: int(rng.integers(0, 10_000)) for w in range(nw)}
    want_rs, want, fill = _restated(segs, rs, cnt, arenas, base)

    dev = torch.device("cuda")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    rs_t, cnt_t = t(rs), t(cnt)
    ain = {w: (t(arenas[w][0]), t(arenas[w][1])) for w in range(nw)}
    aout = {w: (torch.full((fill[w] + 16,), -1, dtype=torch.int32, device=dev),
                torch.full((fill[w] + 16,), -1.0, dtype=torch.float32, device=dev))
            for w in range(nw)}
    rs_out = torch.full_like(rs_t, -5)
    tab = (N.PackSegmentC * len(segs))()
    for k, (rows, ro, co, w) in enumerate(segs):
        tab[k].rows, tab[k].width, tab[k].rs_off, tab[k].cnt_off = rows, w, ro, co
    plan = C.c_void_p()
    N.check(N.lib.qftc_csr_pack_plan_create(C.byref(plan), tab, len(segs), nw, None))
    P = C.c_void_p * nw
    ptrs = lambda d, k: P(*[d[w][k].data_ptr() for w in range(nw)])  # noqa: E731
    try:
        for _ in range(2):   # a plan runs any number of times
            N.check(N.lib.qftc_csr_pack_run(plan, C.c_void_p(rs_t.data_ptr()),
                                            C.c_void_p(cnt_t.data_ptr()),
                                            C.cast(ptrs(ain, 0), C.c_void_p),
                                            C.cast(ptrs(ain, 1), C.c_void_p),
                                            C.cast(ptrs(aout, 0), C.c_void_p),
                                            C.cast(ptrs(aout, 1), C.c_void_p),
                                            (C.c_int64 * nw)(*[base[w] for w in range(nw)]),
                                            C.c_void_p(rs_out.data_ptr()), None))
    finally:
        torch.cuda.synchronize()
        N.lib.qftc_csr_pack_plan_destroy(plan)
    torch.cuda.synchronize()
    assert np.array_equal(rs_out.cpu().numpy(), want_rs)
    for w in range(nw):
        col, val = aout[w][0].cpu().numpy(), aout[w][1].cpu().numpy()
        n = fill[w]
        assert np.array_equal(col[:n], want[w][0]), w
        assert np.array_equal(val[:n].view(np.int32), want[w][1].view(np.int32)), w
        assert (col[n:] == -1).all(), "wrote past the class's packed size"


def test_csr_pack_rejects_bad_arguments(cuda):
    N = cuda._native
    plan = C.c_void_p()
    tab = (N.PackSegmentC * 1)()
    tab[0].rows, tab[0].width = 4, 3            # class 3 of 2
    with pytest.raises(ValueError):
        N.check(N.lib.qftc_csr_pack_plan_create(C.byref(plan), tab, 1, 2, None))
    with pytest.raises(ValueError):
        N.check(N.lib.qftc_csr_pack_plan_create(C.byref(plan), tab, 1, 9, None))
