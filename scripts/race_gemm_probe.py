import sys; sys.path.insert(0, '/root/repo')
import torch
import paper_2210_03052_b200 as bt
from paper_2210_03052_b200.tensor import gemm_device
bt._lib.require_device()
a = torch.randn(300, 256, device="cuda").to(torch.bfloat16); w = torch.randn(1024, 256, device="cuda").to(torch.bfloat16)
gemm_device(a, w, None, None, 0, bn=int(sys.argv[1])); torch.cuda.synchronize(); print("done", sys.argv[1])
