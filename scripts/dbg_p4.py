import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch, datagen, oracle
from paper_2203_04071_b200 import _lib as ax
ax.load()
def run(M,N,K,T,A,W,bits=8):
    lut=ax.Lut(bits,T); Kp=(K+15)//16*16
    dA=torch.zeros(M,Kp,dtype=torch.int8,device='cuda'); dA[:,:K]=torch.from_numpy(A).cuda()
    wp=ax.WPack(lut,torch.from_numpy(W).cuda())
    C=torch.full((M,N),-7,dtype=torch.int32,device='cuda')
    ax.axq_lut_gemm_wp(dA.narrow(1,0,K),wp,None,C); torch.cuda.synchronize()
    return C.cpu().numpy(), oracle.lut_gemm(A,W,T,bits)
A=np.array([[3]],np.int8); W=np.array([[5]],np.int8)
for name,T in [("exact",datagen.lut_exact(8)),("randerr",datagen.lut_randerr(8,0,2))]:
    c,r=run(1,1,1,T,A,W); print(name,c,r, "T00",T[0])
A=np.zeros((1,1),np.int8); W=np.array([[5]],np.int8)
c,r=run(1,1,1,datagen.lut_randerr(8,0,2),A,W); print("a=0",c,r)
A=datagen.random_int8(1,(64,32)); W=datagen.random_int8(2,(16,32))
c,r=run(64,16,32,datagen.lut_exact(8),A,W); print("exact 64x16x32 eq", (c==r).all(), c[:2,:4], r[:2,:4])
c,r=run(64,16,32,datagen.lut_randerr(8,0,2),A,W); print("randerr eq", (c==r).all(), c[:2,:4], r[:2,:4])
