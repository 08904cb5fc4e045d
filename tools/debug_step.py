"""Debug helper: run the grouped step on a small LLaMA-shaped model (optionally
under compute-sanitizer) and compare every tensor with the CPU oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2310_07147_b200 as q
from paper_2310_07147_b200.shapes import llama
from oracle.oracle import Oracle

hidden, inter, layers, vocab = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (256, 688, 2, 512)))
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
shapes = llama(hidden, inter, layers, vocab)
port = Oracle("port")
st = q.QftModelState(shapes, bit_width=8)
st.init_from_weights(lambda i: q.synth(shapes[i], 1234 + i, 0.02, 0.005), 0.01)
ora = []
for i, sh in enumerate(shapes):
    w = port.synth(sh, 1234 + i, 0.02, 0.005)
    ora.append([port.decompose_weight(w, 0.01, 8), port.quantize_state(np.zeros(sh, np.float32), 8)])
for s in range(steps):
    for i, sh in enumerate(shapes):
        gq = port.quantize_state(port.synth(sh, 5000 + 100 * s + i, 1e-3, 0.0), 8)
        c, sc, z = st.grad_views(i)
        c.copy_(torch.from_numpy(gq[0])); sc.copy_(torch.from_numpy(gq[1])); z.copy_(torch.from_numpy(gq[2]))
        d, m = ora[i]
        ora[i] = list(port.lion_step_layer(d, *m, *gq, lr=2e-5)[:2])
    st.step(lr=2e-5, check=True)
    bad = 0
    for i in range(len(shapes)):
        got = st.export_tensor(i); d, m = ora[i]
        for k, ref in (("codes", d.codes), ("row_ptr", d.row_ptr), ("col_idx", d.col_idx), ("values", d.values), ("m_codes", m[0])):
            if not np.array_equal(got[k], ref):
                bad += 1; print("MISMATCH step", s, "tensor", i, shapes[i], k)
    print("step", s, "ok" if not bad else f"{bad} mismatches", "nnz", st.nnz(), "replans", st.replans, flush=True)
