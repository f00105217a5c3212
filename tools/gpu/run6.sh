cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -x -q -m gpu -k "production or e10 or reference_values or multi" 2>&1 | tail -3
for big in 17 15 16; do
export MT_S2_BIG_LOG2=$big
echo "big_min 2^$big"
MT_S2_BIG_LOG2=$big timeout 300 python -m pytest tests -x -q -m gpu -k "production" 2>&1 | tail -1
for e in 1e17 1e19; do timeout 300 python tools/prof_job.py $e 1 ; done 2>&1 | python -c "
import sys,ast
for l in sys.stdin:
    p=l.split(' ',3)
    if len(p)<4: print(l); continue
    d=ast.literal_eval(p[3]); print(p[0],p[1],p[2],{k:d[k] for k in ('ms_total','ms_update_head','ms_sieve_tail','ms_qgather','ms_setup')})
"
done
