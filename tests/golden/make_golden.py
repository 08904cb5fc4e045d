"""Generate the committed golden fixtures from the REAL reference.

Runs ``oracle/_ref/libqft_ref.so`` -- the reference headers
(/root/reference/proj/include/qft) compiled unmodified with the reference flags
by oracle/Makefile -- on small seeded inputs and stores inputs + outputs in
``tests/golden/golden.npz``.  The fixtures travel with the repo, so the oracle
restatement and the GPU kernels are pinned to the reference even where
/root/reference is absent (the GPU box).

    make -C oracle && python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402


def zoo(rng, rows, cols, bw):
    x = rng.uniform(-2, 2, size=(rows, cols)).astype(np.float32)
    x[0] = 0.0
    x[1] = 3.5
    x[2] = 1000.0 + rng.uniform(0, 1e-3, cols).astype(np.float32)
    x[3] = -7.0 + rng.uniform(0, 1e-4, cols).astype(np.float32)
    qmax = (1 << bw) - 1
    s = np.float32(2.0 / qmax)
    k = rng.integers(-qmax // 2, qmax // 2, cols)
    x[4] = ((k + 0.5) * np.float64(s)).astype(np.float32)
    x[4, 0], x[4, 1] = -1.0, 1.0
    return x


def main():
    ref = Oracle("reference")
    out = {}
    rng = np.random.default_rng(20241017)
    # quantize_state over bit widths (incl. planted ties, constant/zero/narrow rows)
    for bw in (2, 3, 4, 8):
        x = zoo(rng, 12, 96, bw)
        q, s, z = ref.quantize_state(x, bw)
        out[f"qs{bw}_x"], out[f"qs{bw}_codes"], out[f"qs{bw}_scale"], out[f"qs{bw}_zp"] = x, q, s, z
        out[f"qs{bw}_deq"] = ref.dequantize(q, s, z)
    # thresholds, both kinds
    w = ref.synth((9, 333), 77, 0.02, 0.005)
    out["th_w"] = w
    for kind in (0, 1):
        for f in (0.0, 0.01, 0.05):
            lo, hi = ref.outlier_thresholds(w, f, kind)
            out[f"th_k{kind}_f{f}_lo"], out[f"th_k{kind}_f{f}_hi"] = lo, hi
    # decompose_weight + reconstruct
    for bw in (3, 8):
        w = ref.synth((16, 160), 500 + bw, 0.02, 0.005)
        d = ref.decompose_weight(w, 0.02, bw)
        p = f"dw{bw}_"
        out[p + "w"] = w
        for k in ("codes", "scale", "zero_point", "row_ptr", "col_idx", "values", "t_min",
                  "t_max"):
            out[p + k] = getattr(d, k)
        out[p + "recon"] = ref.reconstruct(d)
    # a 3-step quantized Lion trajectory with trace (optimizer.hpp:85-120)
    shape, bw = (12, 64), 8
    w = ref.synth(shape, 42, 0.02, 0.005)
    d = ref.decompose_weight(w, 0.05, bw)
    m = ref.quantize_state(np.zeros(shape, np.float32), bw)
    out["ls_w0"] = w
    for step in range(3):
        g = ref.synth(shape, 900 + step, 1e-2, 0.0)
        gq = ref.quantize_state(g, bw)
        d, m, tr = ref.lion_step_layer(d, *m, *gq, lr=2e-3, wd=0.01, trace=True)
        p = f"ls{step}_"
        out[p + "g"] = g
        for k in ("codes", "row_ptr", "col_idx", "values"):
            out[p + k] = getattr(d, k)
        out[p + "m_codes"], out[p + "m_scale"], out[p + "m_zp"] = m
        out[p + "w_upd"], out[p + "m_upd"] = tr["w_upd"], tr["m_upd"]
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print(f"wrote {len(out)} arrays to tests/golden/golden.npz")


if __name__ == "__main__":
    main()
