import sys, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
from test_golden import load
from oracle.bind import OracleCase
from paper_2502_17217_b200 import solver as sv
z,m,ph=load('/root/repo/tests/golden/hex_j2.npz')
ev=sv.ResidualEvaluator(m,ph); o=OracleCase(m,ph)
for t in (0.7,):
    ev.set_time(t); o.set_time(t)
for sc in (1e-3, 1e-2, 0.1, 0.3, 1.0):
    u=z['u']*sc
    r=ev.residual(u).cpu().numpy(); ro=o.residual(u)
    print(sc, np.abs(r-ro).max()/np.abs(ro).max())
st=o.law_state(); print(st[0])
ph2=ph; 
u=z['u']
ev.commit(u); o.commit(u)
sg=ev.law_state(); so=o.law_state()
d=np.abs(sg-so).max(axis=0); print('state diff per row', d)
print('gpu', sg[0]); print('orc', so[0])
r=ev.residual(0.5*u).cpu().numpy(); ro=o.residual(0.5*u); print('after commit', np.abs(r-ro).max()/np.abs(ro).max())
