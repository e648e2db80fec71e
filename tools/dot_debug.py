"""Direct check of the tcgen05 DOT kernel (cgx_dot_tc) with a debug dump."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1812_03770_b200 import cg  # noqa: E402

lib = cg.lib()
f = lib.cgx_dot_tc
f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_int]
for (m, n, k, ta, tb) in [(128, 128, 32, 0, 0), (128, 128, 32, 0, 1), (128, 128, 32, 1, 0), (128, 128, 32, 1, 1), (256, 256, 96, 0, 1), (300, 136, 100, 1, 0), (300, 136, 100, 0, 0)]:
    A = torch.randint(-4, 5, ((k, m) if ta else (m, k)), dtype=torch.float32, device="cuda")
    B = torch.randint(-4, 5, ((n, k) if tb else (k, n)), dtype=torch.float32, device="cuda")
    C = torch.full((m, n), -7.0, device="cuda")
    dbg = torch.zeros(64, device="cuda")
    rc = f(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, ta, tb, dbg.data_ptr(), 0)
    ref = (A.T if ta else A).double() @ (B.T if tb else B).double()
    d = dbg.cpu().numpy()
    print(f"m{m} n{n} k{k} ta{ta} tb{tb} rc={rc} max|C-ref|={float((C.double()-ref).abs().max()):g}")
    print("  A raw", d[0:8], "A[0,:8]", (A.T if ta else A)[0, :8].cpu().numpy() if not ta else A[0, :8].cpu().numpy())
    print("  B raw", d[8:16])
    print("  tmem", d[16:17].view(np.uint32), "nk", d[17], "lo32", d[18:19].view(np.uint32), "hi0", d[19])
    print("  C[0,:8]", C[0, :8].cpu().numpy(), "ref", ref[0, :8].cpu().numpy())
    cm = C.cpu().numpy(); rf = ref.cpu().numpy()
    bad = np.argwhere(cm != rf)
    print("  mismatches", len(bad), bad[:5].tolist())
