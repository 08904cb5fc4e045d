"""Print the ZeRO-1 fields of a bench --zero1 JSON line (stdin)."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
for k in ("zero1_step", "zero1_fused_step"):
    z = d.get(k, {})
    print(k, json.dumps({a: (round(b, 3) if isinstance(b, float) else b) for a, b in z.items()
                         if a not in ("what", "kernels")}))
