"""Probe: fused dequant GEMM time vs K (M = N = 4096) -- separates the per-K-block cost of
the pipeline from the fixed cost (launch, prologue, epilogue)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2310_07147_b200 as q  # noqa: E402

m = int(os.environ.get("PROBE_M", "4096"))
r = int(os.environ.get("PROBE_N", "4096"))
res = []
for c in (64, 256, 1024, 4096):
    st = q.QftModelState([(r, c)], bit_width=8)
    st.init_from_weights(lambda i: q.synth((r, c), 4242, 0.02, 0.005), 0.01, "percentile")
    x = (torch.randn(m, c, device="cuda") * 0.5).to(torch.bfloat16)
    y = torch.empty((m, r), dtype=torch.bfloat16, device="cuda")
    for _ in range(3):
        st.linear(0, x, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        st.linear(0, x, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    res.append((c, round(ms * 1000, 1)))
print(os.environ.get("TAG", ""), "K -> us:", res)
