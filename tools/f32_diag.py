"""fp32 dX error of the fused (lf_cce_forward_backward) and separate paths against the oracle, per shape."""
import sys, os, numpy as np, torch
R=os.environ.get("GRAFT_REPO_ROOT","/root/repo"); sys.path.insert(0,R); sys.path.insert(0,R+"/tests")
import oracle_bind as ob
from gpu_util import instance
import paper_2509_09682_b200 as lf
for (n,d,v) in [(130,256,1000),(300,256,5000),(130,128,1000),(300,64,5000)]:
    X,E,x,Eh,Ch,t = instance(0xB2000031+n+v+d, n, d, v, torch.float32)
    loss,pos,lse = ob.cce_forward(Eh,Ch,t); dX,dC,_,_ = ob.cce_backward(Eh,Ch,t,lse,1.0,0.0)
    fo,fb = lf.cce_forward_backward(X,E,x,1.0,lf.CceConfig())
    so = lf.cce_forward(X,E,x); sb = lf.cce_backward(X,E,x,so.lse,1.0)
    mx = np.abs(dX).max()
    for name,o,g in (("fused",fo,fb),("separate",so,sb)):
        gd = g.grads.d_embeddings.double().cpu().numpy()
        err = np.abs(gd-dX); 
        print(n,d,v,name, "lse", float(np.abs(o.lse.cpu().numpy()-lse).max()), "dX maxerr/max", err.max()/mx, "norm", np.linalg.norm(gd-dX)/np.linalg.norm(dX), "worst excess", float((err - (1e-4*np.abs(dX)+1e-6*mx)).max()))
