import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np, workloads as W
from gpu_util import to_dev, to_np, vec_dev
import paper_2602_19090_b200 as ozr
from oracle import refine as orf, split as osp
c=W.CONFIGS['c2']; n=512
A,_=W.make_matrix(n,c['kind'],c['cnd'],c['seed']); lam0,X0=W.initial_eig(A,'fp64')
ctx=ozr.Context(0)
for th in (1e-4, 1e-12):
    p=ozr.default_params(delta=1e-12, form_R=1, theta_V=th, theta_W=th, theta_U=th)
    Xd,ld=to_dev(X0),vec_dev(lam0)
    rep=ozr.ozr_refine_step(ctx,to_dev(A),Xd,ld,p)
    Rg=to_np(ozr.ozr_last_R(ctx,n))
    Xo,lo,info=orf.sweep(A,X0,lam0,1e-12,theta=p.theta,form_R=True)
    X1=info['X1']
    G64 = X1.T @ X1
    D=np.abs(Rg-info['R']); i,j=np.unravel_index(np.argmax(D),D.shape)
    print(th, rep['kX'], rep['pairs_G'], D.max(), i, j, Rg[i,j], info['R'][i,j], -G64[i,j])
    # symmetry of the GPU R
    print(' asym', np.max(np.abs(Rg-Rg.T)), 'max|R|', np.abs(Rg).max())
