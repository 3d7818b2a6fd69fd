import json, numpy as np, sys, torch
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import test_runtime_gpu as T
torch.backends.cuda.matmul.allow_tf32=False
for case in T.CONFIG1:
    rep,_=T.run_case(case)
    got=np.array(rep.losses); want=np.array(case['losses'])
    rel=np.abs(got-want)/np.abs(want)
    print(case['strategy'], 'max rel %.3g at mb %d'%(rel.max(), rel.argmax()+1), ' '.join('%.1e'%r for r in rel))
