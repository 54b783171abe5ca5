import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2301_11389_b200 import inputs
from paper_2301_11389_b200.binding import Stencil
shape = tuple(int(x) for x in sys.argv[1].split("x"))
st = Stencil("gradient", shape[::-1], "f32")
u = inputs.generate_torch(shape, "f32", 1)
outs = [torch.zeros_like(u) for _ in range(3)]
st.step([u], outs)
torch.cuda.synchronize()
print("ok", shape, float(outs[0].abs().sum()))
