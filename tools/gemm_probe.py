"""Probe: one fused dequant GEMM (4096 x 4096 x 4096) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2310_07147_b200 as q  # noqa: E402

r, c, m = 4096, 4096, 4096
st = q.QftModelState([(r, c)], bit_width=8)
st.init_from_weights(lambda i: q.synth((r, c), 4242, 0.02, 0.005), 0.01, "percentile")
x = (torch.randn(m, c, device="cuda") * 0.5).to(torch.bfloat16)
y = torch.empty((m, r), dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    st.linear(0, x, out=y)
torch.cuda.synchronize()
print("ok")
