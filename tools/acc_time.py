"""Time the fused accumulate (gradflow.hpp:52-58) on one B200: 10 warm-up
calls, then 7 repetitions of 10 calls; min and median per call (each call includes its
error-flag synchronisation)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2310_07147_b200 as q  # noqa: E402

r, c = 4096 * 8, 11008   # 360 M elements, 1.8 GB of fp32 gradient (> L2)
g = torch.randn(r, c, device="cuda") * 1e-2
acc = q.quantize_state(torch.randn(r, c, device="cuda") * 1e-2, 8)
for _ in range(10):
    q.accumulate(acc, g, out=acc)
per = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        q.accumulate(acc, g, out=acc)
    e1.record()
    torch.cuda.synchronize()
    per.append(e0.elapsed_time(e1) / 10)
alg = r * c * (1 + 4 + 1) + r * 16
ms = min(per)
print(json.dumps({"accumulate": f"{r}x{c} u8 acc + f32 g -> u8, in place",
                  "ms_min": ms, "ms_median": statistics.median(per),
                  "gbs": alg / ms / 1e6, "frac_of_hbm": alg / ms / 1e6 / 6540.5,
                  "note": "per call incl. the err-flag sync"}))
