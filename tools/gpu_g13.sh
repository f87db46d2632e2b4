cd $GRAFT_REPO_ROOT
FMG_SYNC_DEBUG=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2511_19036_b200 as P
s=P.Solver(3,1,6,slabs=2); s.solve(); print('slab solve ok', s.norms()[5,2])
s1=P.Solver(3,1,6); s1.solve(); print('single', s1.norms()[5,2])
" > gpurun_out/g13_dbg.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g13_pytest.log 2>&1; echo pytest=$?
