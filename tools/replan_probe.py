"""Probe: where the large-lr (2.2e-4) checked step spends its time on the 7B state --
the step launch group, the overflow check, slot re-plans (_replan), layout mirroring and
the re-run -- host wall time with synchronisation around each piece."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_07147_b200 as q  # noqa: E402
from paper_2310_07147_b200 import engine as E  # noqa: E402
from paper_2310_07147_b200.shapes import llama2_7b  # noqa: E402

st = bench.build_state(llama2_7b(), q, 1234)
hy = dict(bench.HYPER, lr=2.2e-4)
T = {"replan": 0.0, "mirror": 0.0, "set_arena": 0.0, "n_replan": 0}


def wrap(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        T[name] += time.perf_counter() - t0
        if name == "replan":
            T["n_replan"] += 1
        return r
    return w


st._replan = wrap("replan", st._replan)
st._mirror_layout = wrap("mirror", st._mirror_layout)
st._set_arena = wrap("set_arena", st._set_arena)
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    for key in ("replan", "mirror", "set_arena"):
        T[key] = 0.0
    T["n_replan"] = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.step(**hy, check=True)
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t0) * 1e3
    print(f"step {k}: {tot:8.2f} ms  replans {T['n_replan']}  replan {T['replan']*1e3:7.2f}  "
          f"mirror {T['mirror']*1e3:6.2f}  set_arena {T['set_arena']*1e3:6.2f}  nnz {st.nnz()}  "
          f"tiers {st.tiers()}", flush=True)
