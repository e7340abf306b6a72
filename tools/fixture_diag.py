import sys, json, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/oracle')
import oracle as O, paper_2602_06694_b200 as nq
chk=O.restated()
for name in sys.argv[1:]:
    g=np.load(f'/root/repo/tests/golden/admm_{name}.npz')
    n,m,r=int(g['n']),int(g['m']),int(g['r'])
    w=O.synthetic_weight(chk,int(g['seed']),n,m)
    lay,err,st=nq.factorize_layer(w, nq.AdmmConfig(rank=r, max_iters=int(g['max_iters'])))
    d=lay.download()
    def bits(words, rows, cols):
        w8=np.ascontiguousarray(words,'<u4').view(np.uint8)
        return np.unpackbits(w8.reshape(rows,-1),axis=1,bitorder='little')[:,:cols]
    su=(bits(d.u,n,r)==bits(g['u'],n,r)).mean(); sv=(bits(d.v,m,r)==bits(g['v'],m,r)).mean()
    print(json.dumps({"case":name,"gpu_err":err,"ref_err":float(g['rel_err']),"rel":abs(err-float(g['rel_err']))/float(g['rel_err']),
        "gpu_iters":st.iteration,"ref_iters":int(g['iteration']),"sign_u":su,"sign_v":sv,
        "svd_steps":st.stats.get('svd_steps'),"svd_conv":st.stats.get('svd_converged_steps')}), flush=True)
