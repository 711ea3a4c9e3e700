cd tools
for d in ${DBGS:-0 1 2 3}; do echo "dbg=$d"; FCN_TC_DBG=$d python -c "
import sys; sys.argv=['x','cfg5']
import macbench, torch, mac_one
from paper_1811_09953_b200 import _lib, configs, engine, fv, mac_tc
W=configs.WORKLOADS['cfg5']; P=fv.EncryptionParams(W.n,W.primes,(W.t,),W.beta)
name,plan,n_in=macbench.layers('cfg5')[0]
mac,_,_=engine._lower_linear(plan,W.t,W.n,'batched')
k=len(W.primes); x=torch.randint(0,1<<49,(n_in,2,k,W.n),device='cuda',dtype=torch.int64)
tcp=mac_tc.build(mac,n_in,7,2*k*W.n,force=True)
out=torch.empty((4096,2,k,W.n),dtype=torch.int64,device='cuda')
print(macbench.timed(lambda: mac_tc.run(P,tcp,x,out))*1e3, 'ms')
"; done
