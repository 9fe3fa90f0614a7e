import os, subprocess, sys, itertools
code = r'''
import sys; sys.path.insert(0,'/root/repo')
import torch
from paper_2203_10983_b200 import bns
torch.manual_seed(0)
M,K,N=64,128,64
A=torch.randn(M,K,device='cuda'); D=torch.randn(M,N,device='cuda')
C=torch.full((K,N),float('nan'),device='cuda')
try:
    bns.bns_gemm(bns.BNS_FP32,bns.BNS_GEMM_WGRAD,M,N,K,A,None,K,D,N,C,N); torch.cuda.synchronize()
    ref=A.double().t()@D.double()
    print('relerr %.3e zeros %d' % (float((C.double()-ref).abs().max()/ref.abs().max()), int((C==0).sum())))
except Exception as e:
    print('ERR', str(e)[:100])
'''
for swz, lay, sbo, lbo in itertools.product([3, 4], [1, 2], [512, 1024, 128], [0, 128]):
    env = dict(os.environ, BNS_TF32_MN_SWZ=str(swz), BNS_TF32_MN_LAYOUT=str(lay), BNS_TF32_MN_SBO=str(sbo), BNS_TF32_MN_LBO=str(lbo))
    try:
        r = subprocess.run([sys.executable, '-c', code], env=env, capture_output=True, text=True, timeout=60)
        out = r.stdout.strip() or r.stderr.strip()[-200:]
    except subprocess.TimeoutExpired:
        out = 'TIMEOUT'
    print(swz, lay, sbo, lbo, out, flush=True)
