"""Probe: CSR slot drift at a large lr -- per step the overflowing rows (count above the
slot), the nnz, the largest per-row count increase and the replan levels, on the first
layers of the 7B shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_07147_b200 as q  # noqa: E402
from paper_2310_07147_b200 import _native as N  # noqa: E402
from paper_2310_07147_b200.shapes import llama2_7b  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
lr = float(sys.argv[2]) if len(sys.argv) > 2 else 2.2e-4
shapes = llama2_7b()[:7 * layers]
st = bench.build_state(shapes, q, 1234)
R = st.row_count_total
prev = st.row_count[st.cur][:R].clone()
for step in range(12):
    flip = st.cur
    st.step(**dict(bench.HYPER, lr=lr), check=False)
    torch.cuda.synchronize()
    out = 1 - flip
    ov = any(N.lib.qftc_plan_pending_overflow(g.plan) for g in st.groups)
    cnt = st.row_count[out][:R]
    caps = []
    for i in st.order:                       # flat position order, like row_count
        rs = st._rs(st.row_start[out], i)
        caps.append((rs[1:] - rs[:-1]))
    cap = torch.cat(caps)
    over = cnt > cap
    info = {"step": step, "overflow": bool(ov), "rows_over": int(over.sum()),
            "worst_excess": int((cnt - cap).max()), "nnz": int(cnt.sum()),
            "mean_headroom": float((cap - cnt).float().mean()),
            "max_inc": int((cnt - prev).max()), "levels": [g.replans for g in st.groups]}
    if ov:
        st.recover()
        cnt = st.row_count[out][:R]
    print(json.dumps(info))
    prev = cnt.clone()
