import sys, ctypes as C
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1807_01702_b200 import _lib, kernels as K
from paper_1807_01702_b200.params import ConvParams
L = _lib.lib()
w = np.arange(2 * 3 * 1 * 1, dtype=np.float32).reshape(2, 3, 1, 1)
p = ConvParams(3, 2, 1, 1, weights=w)
pc = K.PackedConv(p, torch.float32, cin_store=4)
torch.cuda.synchronize()
print("wp", pc.wp.cpu().numpy().reshape(2, -1)[:, :6])
print("wt", pc.wt.cpu().numpy().reshape(4, -1)[:, :4])
w = np.random.default_rng(0).uniform(-.3, .3, (64, 64, 1, 1)).astype(np.float32)
pc = K.PackedConv(ConvParams(64, 64, 1, 1, weights=w), torch.float32, cin_store=64)
torch.cuda.synchronize()
print("wp", pc.wp.cpu().numpy()[:6], w.reshape(-1)[:6])
print("w32", pc.w32.cpu().numpy().reshape(-1)[:6])
