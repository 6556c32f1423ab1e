import sys, os
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1807_01702_b200 import kernels as K, _lib
from paper_1807_01702_b200.params import ConvParams
print("current stream handle:", torch.cuda.current_stream().cuda_stream)
# dirty the caching allocator with big values, free, then pack
for trial in range(4):
    junk = torch.full((1 << 20,), 25.0, device="cuda"); del junk
    w = np.random.default_rng(trial).uniform(-.3, .3, (64, 64, 1, 1)).astype(np.float32)
    pc = K.PackedConv(ConvParams(64, 64, 1, 1, weights=w), torch.float32, cin_store=64)
    torch.cuda.synchronize()
    print(trial, "w32 ok:", np.array_equal(pc.w32.cpu().numpy(), w), "wp ok:", np.allclose(pc.wp.cpu().numpy()[:4096], w.reshape(-1)))
