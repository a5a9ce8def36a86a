import sys, torch
sys.path.insert(0, '.')
import paper_1604_06174_b200 as slm
M,N,K=2048,256,2048
for split in (2,4,8):
  for trial in range(2):
    A=torch.randn(K,M,device='cuda').bfloat16(); B=torch.randn(N,K,device='cuda').bfloat16()
    out=torch.empty(split,N,M,device='cuda')
    s=torch.cuda.Stream()
    with torch.cuda.stream(s):
        slm.debug_gemm(1,0,256,M,N,K,A,B,out,stream=s,split=split)
    torch.cuda.synchronize()
    ref=B.float()@A.float()
    print(split, trial, ((out.sum(0)-ref).norm()/ref.norm()).item())
