import sys; sys.path.insert(0,'/root/repo')
import torch
from paper_2203_10983_b200 import bns
torch.manual_seed(0)
M,K,N=64,128,64
A=torch.randn(M,K,device='cuda'); D=torch.randn(M,N,device='cuda')
ref=A.double().t()@D.double()
# same product through the FWD path: C[K x N] = At (K x M) . W with W^T = Dt [N][M]
At=A.t().contiguous(); Dt=D.t().contiguous()
C=torch.full((K,N),float('nan'),device='cuda')
bns.bns_gemm(bns.BNS_FP32,bns.BNS_GEMM_FWD,K,N,M,At,None,M,Dt,M,C,N); torch.cuda.synchronize()
print('fwd-path relerr', float((C.double()-ref).abs().max()/ref.abs().max()))
# DX path: C = At . Dt^T with B = Dt [N][K=M]
C2=torch.full((K,N),float('nan'),device='cuda')
bns.bns_gemm(bns.BNS_FP32,bns.BNS_GEMM_DX,K,N,M,At,None,M,Dt,M,C2,N); torch.cuda.synchronize()
print('dx-path relerr', float((C2.double()-ref).abs().max()/ref.abs().max()))
C3=torch.full((K,N),float('nan'),device='cuda')
S=bns.bns_gemm(bns.BNS_FP32,bns.BNS_GEMM_WGRAD,M,N,K,A,None,K,D,N,C3,N); torch.cuda.synchronize()
print('wgrad relerr', float((C3.double()-ref).abs().max()/ref.abs().max()), 'S', S, C3[:2,:4])
Ab=A.bfloat16(); Db=D.bfloat16(); C4=torch.full((K,N),float('nan'),device='cuda')
S=bns.bns_gemm(bns.BNS_BF16,bns.BNS_GEMM_WGRAD,M,N,K,Ab,None,K,Db,N,C4,N); torch.cuda.synchronize()
print('bf16 wgrad relerr', float((C4.double()-Ab.double().t()@Db.double()).abs().max()/ref.abs().max()), 'S', S)
