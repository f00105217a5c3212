cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -3
timeout 2400 python -m pytest tests -x -q -m "slow" --durations=0 2>&1 | tail -12
