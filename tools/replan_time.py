"""Probe: where a large-lr re-plan's time goes (each engine piece timed with a sync)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_07147_b200 as q  # noqa: E402
from paper_2310_07147_b200 import engine as E  # noqa: E402
from paper_2310_07147_b200.shapes import llama2_7b  # noqa: E402

T = {}


def wrap(name):
    f = getattr(E.QftModelState, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        T.setdefault(name, []).append(round(1e3 * (time.perf_counter() - t0), 2))
        return r
    setattr(E.QftModelState, name, g)


for n in ("_replan", "_set_arena", "_mirror_layout", "_alloc"):
    wrap(n)


def wrapf(owner, name, label):
    f = getattr(owner, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        T.setdefault(label, []).append(round(1e3 * (time.perf_counter() - t0), 2))
        return r
    setattr(owner, name, g)


wrapf(q._native.lib, "qftc_csr_replan_caps", "caps")
wrapf(q._native.lib, "qftc_plan_step", "rerun")
wrapf(q._native.lib, "qftc_plan_result", "result")
wrapf(torch, "cumsum", "cumsum")
_step = q._native.lib.qftc_plan_step
st = bench.build_state(llama2_7b(), q, 1234)
hy = dict(bench.HYPER, lr=2.2e-4)
for i in range(12):
    T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.step(**hy, check=True)
    torch.cuda.synchronize()
    print(f"step {i}: {1e3 * (time.perf_counter() - t0):.1f} ms {T}", flush=True)
