import sys, numpy as np
sys.path.insert(0,'/root/repo')
from paper_2203_11025_b200 import helmgpu as hg
from oracle import oracle as O
def rel(a,b): return float(np.linalg.norm(a-b)/np.linalg.norm(b))
rng=np.random.default_rng(3)
for L,n in [(1,128),(2,128),(4,128)]:
    ctx=hg.Context(0); kap=(0.1+0.3*rng.random((n,n)))
    ctx.set_problem(kap,np.zeros((n,n)),1.0,0.0,1.0); ctx.build_hierarchy(hg.VCycleConfig(levels=2))
    ctx.set_net(0,"solver",L,16,3,0); ctx.init_net_he(0,9)
    x=rng.standard_normal((2,3,n,n)).astype(np.float32)
    y_tc=ctx.net_forward(x); ctx.set_option("tc_conv",0); y_s=ctx.net_forward(x)
    y_o=O.UNet(0,L,16,3,0,seed=9).forward(x)
    print(L, n, "tc-vs-oracle", rel(y_tc,y_o), "simt-vs-oracle", rel(y_s,y_o))
# single conv: 16->16 and 32->32 etc via a 2-level net? use raw layer test through L=1 (enc1 3->16 simt, enc2 16->16 tc, head simt)
