import torch, math
for (M,N,K) in [(2458,2304,768),(2458,768,768),(2458,3072,768),(2458,768,3072)]:
    A=torch.randn(M,K,device="cuda").to(torch.bfloat16); W=torch.randn(N,K,device="cuda").to(torch.bfloat16)
    for _ in range(3): torch.matmul(A,W.t())
    torch.cuda.synchronize()
