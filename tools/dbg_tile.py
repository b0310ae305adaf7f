import numpy as np, sys
sys.path.insert(0,'.')
from paper_2001_10554_b200 import _native as N
from paper_2001_10554_b200.workloads import haar_2x2
rng=np.random.default_rng(0)
for n in (12,13):
  for cnt in (2,3,5,8):
    st=N.DeviceState(n,n)
    psi=np.zeros(1<<n,complex); psi[0]=1
    st.upload(psi)
    us=np.stack([haar_2x2(rng) for _ in range(cnt)]).view(np.float64).reshape(-1)
    gates=[N.QsGate(0,q%n,-1,0,8*q,0) for q in range(cnt)]
    try:
        st.apply_program(gates, us, fuse=True); st.synchronize(); print(n,cnt,'ok', N.plan_program(n,gates))
    except Exception as e:
        print(n,cnt,'FAIL',e); break
