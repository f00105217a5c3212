cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -x -q -m gpu -k "production or e10 or reference_values or multi" 2>&1 | tail -5
for e in 1e17 1e19; do timeout 300 python tools/prof_job.py $e 1 ; done 2>&1 | python -c "
import sys,ast
for l in sys.stdin:
    p=l.split(' ',3)
    if len(p)<4: print(l); continue
    d=ast.literal_eval(p[3]); print(p[0],p[1],p[2],{k:d[k] for k in ('ms_total','ms_update_head','ms_sieve_tail','ms_qgather','ms_setup')})
"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sieve2 -s 200 -c 1 -o gpurun_out/r4_sieve2 python tools/prof_job.py 1e17 1 > /dev/null 2>&1
echo done
