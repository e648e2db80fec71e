"""Does tcgen05.mma.kind::tf32 truncate fp32 operands to TF32 (ignore the low 13
mantissa bits)?  Runs the 3xTF32 DOT with the hi tile masked explicitly (default)
and with the raw fp32 tile fed as 'hi' (raw_hi = 1): if the tensor core truncates,
both give the same result bit for bit."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1812_03770_b200 import cg  # noqa: E402

f = cg.lib().cgx_dot_tc
f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_int]
torch.manual_seed(0)
for (m, n, k) in [(256, 256, 512), (512, 384, 1000)]:
    A = torch.rand(m, k, device="cuda") * 2 - 1
    B = torch.rand(k, n, device="cuda") * 2 - 1
    C0 = torch.zeros(m, n, device="cuda")
    C1 = torch.zeros(m, n, device="cuda")
    f(A.data_ptr(), B.data_ptr(), C0.data_ptr(), m, n, k, 0, 0, None, 0)
    f(A.data_ptr(), B.data_ptr(), C1.data_ptr(), m, n, k, 0, 0, None, 1)
    ref = A.double() @ B.double()
    e0 = float((C0.double() - ref).abs().max() / ref.abs().max())
    e1 = float((C1.double() - ref).abs().max() / ref.abs().max())
    print(f"{m}x{n}x{k}: masked-hi err {e0:.3e}, raw-hi err {e1:.3e}, bit-identical {bool(torch.equal(C0, C1))}")
