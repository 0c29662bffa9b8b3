import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2011_06636_b200 as srj
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
p = srj.baseline_problem("3d7", n, seed=0, device=torch.device("cuda", 0))
A = p.A
print(A.describe(), flush=True)
b = A.field(p.b); x = A.field(p.x0)
print("S", A.residual_sq(x, b), flush=True)
