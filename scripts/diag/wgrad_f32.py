import sys; sys.path.insert(0,'/root/repo')
import torch
from paper_2203_10983_b200 import bns
torch.manual_seed(0)
for (M,K,N) in [(32,128,64),(64,128,64),(1000,256,256)]:
    A=torch.randn(M,K,device='cuda'); D=torch.randn(M,N,device='cuda')
    C=torch.full((K,N),float('nan'),device='cuda')
    S=bns.bns_gemm(bns.BNS_FP32,bns.BNS_GEMM_WGRAD,M,N,K,A,None,K,D,N,C,N)
    torch.cuda.synchronize()
    ref=A.double().t()@D.double()
    err=(C.double()-ref).abs()
    print(M,K,N,'S',S,'relerr',float(err.max()/ref.abs().max()),'nan',int(torch.isnan(C).sum()),'zeros',int((C==0).sum()))
    if M==32:
        print('C[:4,:6]',C[:4,:6].cpu()); print('ref[:4,:6]',ref[:4,:6].cpu())
        # find permutation: for C[0,0] which ref entry matches
        c=C.double()
        for (i,j) in [(0,0),(0,1),(1,0),(5,3),(33,7)]:
            d=(ref-c[i,j]).abs(); k=int(d.argmin()); print((i,j),'->',divmod(k,N),float(d.min()))
