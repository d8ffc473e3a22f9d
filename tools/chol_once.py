"""One hp_chol_inverse at order n (for an ncu launch list): python tools/chol_once.py [n]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1607_05210_b200 import _device as D  # noqa: E402
from paper_1607_05210_b200 import _native as N  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4549
lib = N.load()
st = D._stream()
X = torch.randn(8192, n, dtype=torch.float64, device="cuda")
C = D.DevMat.empty(n, n)
C.tensor().copy_(X.t() @ X)
Linv = D.DevMat.empty(n, n)
ws = D._ws(lib.hp_chol_inverse_workspace_bytes(n))
info = ctypes.c_int(0)
torch.cuda.synchronize()
N.check(lib.hp_chol_inverse(C.ptr, C.ld, n, Linv.ptr, Linv.ld, ctypes.byref(info), ws.data_ptr(), ws.numel(), st),
        "chol_inverse")
torch.cuda.synchronize()
print("info", info.value)
