cd $GRAFT_REPO_ROOT
FMG_SYNC_DEBUG=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2511_19036_b200 as P, oracle as O, numpy as np
from fmg_inputs import default_schedule
for d,p,lev in [(2,1,4),(3,1,4)]:
    s=default_schedule(d,p); s['smoother']=1
    g=P.Solver(d,p,lev,P.Schedule.from_dict(s)); g.solve()
    oc=O.CFMG(d,p,lev,O.schedule(d,p,smoother='mcgs')); oc.solve()
    print(d,p,lev,'norm rel', np.max(np.abs(g.norms()-oc.norms())/np.maximum(oc.norms(),1e-300)), [np.array_equal(oc.section(0,l)[0], g.section(0,l)[0]) for l in range(lev)])
" > gpurun_out/g28_dbg.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g28_pytest.log 2>&1; echo pytest=$?
