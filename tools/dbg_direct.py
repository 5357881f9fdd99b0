import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2305_08819_b200 import smconv as sm, synth
s = tuple(int(v) for v in sys.argv[1].split('x'))
N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
g = synth.rng(9, 1)
X = synth.activations(g, N, IH, IW, IC); W = synth.filters(g, OC, FH, FW, IC)
OH = (IH + 2*ph - FH)//sh + 1; OW = (IW + 2*pw - FW)//sw + 1
dY = synth.activations(g, N, OH, OW, OC)
x, w, dy = (torch.from_numpy(a).cuda() for a in (X, W, dY))
print(sm.plan_describe(0, s), sm.plan_describe(2, s))
y = sm.conv2d_fwd(x, w, (sh, sw), (ph, pw)); torch.cuda.synchronize(); print("fwd ok")
dw = sm.conv2d_bwd_filter(x, dy, (FH, FW), (sh, sw), (ph, pw)); torch.cuda.synchronize(); print("dw ok")
