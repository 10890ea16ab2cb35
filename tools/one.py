import sys; sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import numpy as np, torch, paper_2601_08082_b200 as tc
from pyoracle import Oracle, parse_levels
o=Oracle()
for (n,b,cfg) in [(8,2,"Pure F64"),(7,2,"[F16, F32]"),(64,8,"[F16, F32]"),(100,7,"[F16, F16, F16, F32]")]:
    a=o.spd_generate(n,1); p=tc.Plan(n,b,cfg); ad=tc.to_device(a); ld=ad.clone()
    st=p.factor_device(ad,ld); torch.cuda.synchronize(); print(n,b,cfg,st.status, flush=True)
