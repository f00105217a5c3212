cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for e in 1e17 1e19; do MT_TIMING=1 timeout 300 python tools/prof_job.py $e 1 ; done 2>&1 | python -c "
import sys,ast
for l in sys.stdin:
    p=l.split(' ',3)
    if len(p)<4: print(l); continue
    d=ast.literal_eval(p[3]); print(p[0],p[1],p[2],{k:d[k] for k in ('ms_total','ms_update_head','ms_sieve_tail','ms_qgather','ms_setup')}, {k:round(v,1) for k,v in d['kernel_ms'].items()})
"
