import json,sys,os
sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import numpy as np, torch
import pass_probe as PP
import paper_2602_06694_b200 as nq
ctx=nq.context(0); bpw,_,shapes=PP.SHAPES['7b']; rng=np.random.default_rng(5)
ranks={nm:nq.rank_for_target_bpw(n,m,bpw) for nm,n,m in shapes}
steps=[];keep=[]
for b in range(8):
    lay={nm:nq.DeviceLayer.upload_f16(n,m,ranks[nm],*PP.rand_arrays(rng,n,m,ranks[nm]),ctx) for nm,n,m in shapes}
    qkv=nq.DecodeGroup([lay['q'],lay['k'],lay['v']]); gu=nq.DecodeGroup([lay['gate'],lay['up']]); keep+=[lay,qkv,gu]
    d,f=4096,11008; new=lambda n: torch.empty(n,device='cuda',dtype=torch.float16)
    ys=[[new(4096),new(4096),new(4096)],[new(d)],[new(f),new(f)],[new(d)]]
    xs=[torch.randn(d,device='cuda',dtype=torch.float16) for _ in range(3)]+[torch.randn(f,device='cuda',dtype=torch.float16)]
    for u,x,y in zip([qkv,lay['o'],gu,lay['down']],xs,ys): steps.append((u,x,y))
p=nq.DecodePass(steps,ctx)
for _ in range(3): p.launch()
torch.cuda.synchronize()
tr=p.trace().astype(np.int64); G=tr.shape[0]; K=len(steps)
t0=tr[:,0].min(); st=((tr[:,1:1+16*K]-t0)/1e3).reshape(G,K,16)
names={0:'s1start',1:'s1end',2:'s2ready',3:'s2end',4:'tbar',5:'xstaged',6:'pS1done',7:'s1q',8:'s1mma',9:'s2q',10:'s2mma',11:'pS1',12:'tslotfree',13:'tcopy',14:'pS2',15:'pS2done'}
# print step 8..15 medians and max over CTAs
for k in range(8,20):
    row=[]
    for i in [11,6,0,7,8,1,14,15,4,13,2,9,10,3]:
        row.append("%s=%.1f"%(names[i],np.median(st[:,k,i])))
    print(k,' '.join(row))
