"""Time the fused accumulate (gradflow.hpp:52-58) on one B200."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, json, paper_2310_07147_b200 as q
r, c = 4096 * 8, 11008   # 360 M elements (> L2)
g = torch.randn(r, c, device="cuda") * 1e-2
acc = q.quantize_state(torch.randn(r, c, device="cuda") * 1e-2, 8)
for _ in range(3): q.accumulate(acc, g, out=acc)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
n = 10
for _ in range(n): q.accumulate(acc, g, out=acc)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
alg = r * c * (1 + 4 + 1) + r * 16
print(json.dumps({"accumulate": f"{r}x{c} u8 acc + f32 g -> u8, in place", "ms": ms,
                  "gbs": alg / ms / 1e6, "frac_of_hbm": alg / ms / 1e6 / 6540.5,
                  "note": "per call incl. the err-flag sync"}))
