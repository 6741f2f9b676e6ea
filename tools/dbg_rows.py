# Development helper: cfg4-shaped batch through the 256-point row kernel variants
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1401_6238_b200 import batched, workloads
from oracle import hankel_oracle as O
H, X = workloads.cfg4()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
H, X = H[:B], X[:B]
dH = torch.from_numpy(np.ascontiguousarray(H)).cuda()
dx = torch.from_numpy(np.ascontiguousarray(np.transpose(X, (0, 2, 1)))).cuda().reshape(B, -1)
os.environ["HK_NO_PP256"] = "1"
ref = batched.bhhb_tvp_partial(dH, [dx, dx], 3, (64,) * 3, (64,) * 3).cpu().numpy()
del os.environ["HK_NO_PP256"]
y = batched.bhhb_tvp_partial(dH, [dx, dx], 3, (64,) * 3, (64,) * 3)
torch.cuda.synchronize()
y = y.cpu().numpy()
print(os.environ.get("HK_ROWS_NG"), os.environ.get("HK_ROWS_NH"), "B", B, "relerr", np.linalg.norm(y - ref) / np.linalg.norm(ref))
