import ctypes as C, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_1904_03329_b200 import _native as N
N.require_device()
rows = 2_902_330
Y = torch.rand((rows, 32), device="cuda"); F = torch.empty_like(Y)
M = torch.rand((32, 32), device="cuda"); w = torch.rand(32, device="cuda")
G = torch.empty((32, 32), dtype=torch.float64, device="cuda"); inner = torch.empty(1, dtype=torch.float64, device="cuda")
for _ in range(2):
    N.call("hbk_als_update", C.c_void_p(Y.data_ptr()), rows, 32, C.c_void_p(M.data_ptr()), C.c_void_p(w.data_ptr()),
           C.c_void_p(F.data_ptr()), C.c_void_p(G.data_ptr()), C.c_void_p(inner.data_ptr()), N.stream_ptr())
torch.cuda.synchronize()
