"""Probe: per-step timing of the 7B state at lr = 2.2e-4 (checked engine steps), with the
re-plan count after each, then unchecked steps (no host sync) once the slots have grown."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2310_07147_b200 as q  # noqa: E402
from paper_2310_07147_b200.shapes import llama2_7b  # noqa: E402

st = bench.build_state(llama2_7b(), q, 1234)
hy = dict(bench.HYPER, lr=2.2e-4)
s = torch.cuda.current_stream()
for i in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rp = st.replans
    t0 = time.perf_counter()
    e0.record(s)
    st.step(**hy, check=True)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"checked step {i}: {e0.elapsed_time(e1):.2f} ms (wall {1e3*(time.perf_counter()-t0):.2f}) "
          f"replans +{st.replans - rp} tiers {st.tiers()} nnz {st.nnz()}", flush=True)
for i in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    st.step(**hy, check=False)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"unchecked step {i}: {e0.elapsed_time(e1):.2f} ms", flush=True)
    st.check()
