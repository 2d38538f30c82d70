import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2503_10855_b200 as jb
from paper_2503_10855_b200 import workloads as W
g, st, sx, sy, th = W.edge_filters()
x = np.stack([W.edge_frame(128, 200, seed=s) for s in range(1)])
out = jb.edge_detection(x, g, st, sx, sy, th)
print("ok", out.sum())
