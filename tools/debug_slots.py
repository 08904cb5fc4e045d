import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2310_07147_b200 as q
from paper_2310_07147_b200.shapes import llama
shapes = llama(256, 688, 2, 512)
st = q.QftModelState(shapes, bit_width=8)
st.init_from_weights(lambda i: q.synth(shapes[i], 1234 + i, 0.02, 0.005), 0.01)
for i, sh in enumerate(shapes):
    g = q.synth(sh, 5000 + i, 1e-3, 0.0); gq = q.quantize_state(g, 8)
    c, s, z = st.grad_views(i); c.copy_(gq.data); s.copy_(gq.params.scale); z.copy_(gq.params.zero_point)
torch.cuda.synchronize()
for k in range(2):
    print("set", k, "rs equal", torch.equal(st.row_start[0], st.row_start[1]))
st.step(lr=2e-5)
torch.cuda.synchronize()
for i, sh in enumerate(shapes):
    rs = st._rs(st.row_start[1], i).cpu().numpy(); cap = np.diff(rs)
    c0 = st._rows(st.row_count[0], i).cpu().numpy(); c1 = st._rows(st.row_count[1], i).cpu().numpy()
    over = np.nonzero(c1 > cap)[0]
    if len(over):
        j = over[0]
        print("tensor", i, sh, "overflow rows", len(over), "first", j, "c0", c0[j], "c1", c1[j], "cap", cap[j], "rs", rs[j], rs[j+1])
